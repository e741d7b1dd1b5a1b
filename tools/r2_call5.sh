# round 2, call 5: banded-plan SpMM -- parity tests, the whole GPU suite with the plan forced,
# config-4 SpMM timing with and without the plan
set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band.log 2>&1; tail -15 $O/pytest_band.log
SAD_SPMM_BAND=1 timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_bandforced.log 2>&1; tail -8 $O/pytest_gpu_bandforced.log
timeout 900 python bench.py --no-c3 --no-cpu-baseline > $O/bench_c4_band.json 2> $O/bench_c4_band.err; tail -c 1800 $O/bench_c4_band.json; tail -5 $O/bench_c4_band.err
SAD_SPMM_BAND=0 timeout 900 python bench.py --no-c3 --no-cpu-baseline > $O/bench_c4_noband.json 2> $O/bench_c4_noband.err; tail -c 600 $O/bench_c4_noband.json
