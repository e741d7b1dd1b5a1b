# round 2, first GPU call: new tests, the full GPU suite, the config-4 headline
# bench (with and without the x-diagonal L2 prefetch), launch list + ncu of the SpMM
set -x
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_race.py tests/test_gpu_apply_host.py -x -q > gpurun_out/r2/pytest_new.log 2>&1; tail -3 gpurun_out/r2/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2/bench_c4.json 2> gpurun_out/r2/bench_c4.err; tail -c 3000 gpurun_out/r2/bench_c4.json
SAD_SPMM_XPF=0 timeout 600 python bench.py --no-c3 --no-cpu-baseline > gpurun_out/r2/bench_c4_noxpf.json 2> gpurun_out/r2/bench_c4_noxpf.err; tail -c 600 gpurun_out/r2/bench_c4_noxpf.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_c4.csv python bench.py --no-c3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_bulk -s 4 -c 1 -o gpurun_out/r2/prof_c4_spmm python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/ncu_full.log 2>&1
ls -la gpurun_out/r2
