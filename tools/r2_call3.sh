# round 2, call 3 (after the re-entry): full GPU suite with the new X-parity tests,
# the config-4 headline bench + reference arm, launch list, ncu full captures of the
# SpMM and of the config-4 / config-3 persistent kernel, config-3 phase timers
set -x
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -15 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 2500 $O/bench_c4.json
timeout 600 python bench.py --impl reference > $O/bench_c4_ref.json 2> $O/bench_c4_ref.err; tail -c 800 $O/bench_c4_ref.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --no-c3 --no-cpu-baseline --steps 5 --warmup 3 > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_bulk -s 4 -c 1 -o $O/prof_c4_spmm python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > $O/ncu_full.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -c 2 -o $O/prof_c4_pers python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > $O/ncu_pers.log 2>&1
CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py > $O/c3_phase.txt 2>&1; tail -30 $O/c3_phase.txt
KMAX=1 timeout 600 python tools/prof_c3.py > $O/p_c3_plain.log 2>&1 && \
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -c 1 -o $O/prof_c3_full python tools/prof_c3.py > $O/p_c3_ncu.log 2>&1
ls -la $O
