set -x
O=gpurun_out/r2e
mkdir -p $O
CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py > $O/c3_phase_band.txt 2>&1; tail -4 $O/c3_phase_band.txt
SAD_BAND_PERSISTENT=0 CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py > $O/c3_phase_noband.txt 2>&1; tail -4 $O/c3_phase_noband.txt
timeout 1200 python bench.py --config c3 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 1500 $O/bench_c3.json; tail -3 $O/bench_c3.err
