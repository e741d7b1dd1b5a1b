timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_cli.py -x -q 2>&1 | tail -3
timeout 900 python tools/_probe.py 2>&1 | grep -E "^PC|Error"
