CONC=1 PHASE=direct timeout 600 python tools/c2_phase.py 2>&1 | grep -E "^concurrent|Error"
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2_newbar.json
SPLITS=0.85 timeout 300 python tools/c2_split.py 2>&1 | grep split
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_adi.py -x -q 2>&1 | tail -3
