# round 2, call 2: verification tests, bench (config 4 default), HBM mix calibration,
# ncu launch list + full capture of the SpMM
set -x
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_gpu_apply_host.py tests/test_gpu_race.py -q > gpurun_out/r2/pytest_verify.log 2>&1; tail -15 gpurun_out/r2/pytest_verify.log
timeout 300 python tools/hbm_mix.py > gpurun_out/r2/hbm_mix.txt 2>&1; cat gpurun_out/r2/hbm_mix.txt
timeout 900 python bench.py > gpurun_out/r2/bench_c4b.json 2> gpurun_out/r2/bench_c4b.err; tail -c 1500 gpurun_out/r2/bench_c4b.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_c4b.csv python bench.py --no-c3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2/ncu_launch_b.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_bulk -s 4 -c 1 -o gpurun_out/r2/prof_c4_spmm_b python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/ncu_full_b.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -c 2 -o gpurun_out/r2/prof_c4_pers python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/ncu_pers.log 2>&1
ls -la gpurun_out/r2
