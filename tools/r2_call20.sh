set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_adi.py tests/test_gpu_native_adi.py -q -k "intermediate or gap_budget or chunked" > $O/pytest_new.log 2>&1; tail -12 $O/pytest_new.log
