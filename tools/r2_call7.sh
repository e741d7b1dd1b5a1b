set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band2.log 2>&1; tail -3 $O/pytest_band2.log
timeout 900 python bench.py --no-c3 --no-cpu-baseline --c4-steps 2 > $O/bench_c4_band2.json 2> $O/bench_c4_band2.err; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2c/bench_c4_band2.json').read().strip().splitlines()[-1])
print('SPMM', d['value'], d['roofline']['frac'], d['ms_per_step'], d['e2e']['value'])
PY
