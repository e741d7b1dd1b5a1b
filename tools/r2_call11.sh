# round 2, call 11: banded SpMM with U by tile size -- tests, whole GPU suite (default and plan forced),
# bench, ncu launch list + full capture
set -x
O=gpurun_out/r2d
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band.log 2>&1; tail -3 $O/pytest_band.log
SAD_SPMM_BAND=1 SAD_BAND_ROWS=128 timeout 900 python -m pytest tests/test_gpu_spmm_band.py tests/test_gpu_kernels.py -q > $O/pytest_band_128.log 2>&1; tail -3 $O/pytest_band_128.log
SAD_SPMM_BAND=1 timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_bandforced.log 2>&1; tail -3 $O/pytest_gpu_bandforced.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 1500 $O/bench_c4.json; tail -3 $O/bench_c4.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv python bench.py --no-c3 --no-cpu-baseline --steps 5 --warmup 3 --c4-steps 2 > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_band -s 4 -c 1 -o $O/prof_c4_band python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 --c4-steps 2 > $O/ncu_band.log 2>&1
ls -la $O
