set -x
O=gpurun_out/r2h
mkdir -p $O
run() { CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py 2>&1 | tail -2 | sed "s/^/PH $1 /"; }
run band
SAD_BAND_PERSISTENT=0 run noband
SAD_BAND_ROWS_P=128 run band128
