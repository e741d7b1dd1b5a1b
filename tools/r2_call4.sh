# round 2, call 4: preconditioner tests + the tests that lacked their goldens in call 3
set -x
O=gpurun_out/r2b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_precond.py -x -q > $O/pytest_precond.log 2>&1; tail -25 $O/pytest_precond.log
timeout 1200 python -m pytest tests/test_gpu_adi.py tests/test_gpu_kernels.py -q -m gpu > $O/pytest_adi_kernels.log 2>&1; tail -8 $O/pytest_adi_kernels.log
