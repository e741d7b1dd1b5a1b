timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q -k "edge or override" 2>&1 | tail -15
