# Config-3 phase timers + one ncu --set full capture of k_gmres_persistent (HBM-bound case).
set -x
NCU=/usr/local/cuda/bin/ncu
CFG=c3 KMAX=4 CONC=0 PHASE=tma python tools/c2_phase.py > gpurun_out/c3_phase.txt 2>&1
KMAX=1 python tools/prof_c3.py > gpurun_out/p_c3_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -c 1 -o gpurun_out/prof_c3_full python tools/prof_c3.py > gpurun_out/p_c3_ncu.log 2>&1
