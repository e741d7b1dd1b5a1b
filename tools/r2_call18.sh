set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_adi.py -x -q -k chunked 2>&1 | tail -3
nproc; free -g | head -2
timeout 900 python tools/download_bench.py c3 c3y c5 2>&1 | tail -8
