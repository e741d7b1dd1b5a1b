set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band4.log 2>&1; tail -3 $O/pytest_band4.log
SAD_BAND_ROWS=128 SAD_SPMM_BAND=1 timeout 900 python -m pytest tests/test_gpu_spmm_band.py tests/test_gpu_kernels.py -x -q -k "not tiles" > $O/pytest_band4_128.log 2>&1; tail -3 $O/pytest_band4_128.log
for v in auto 512; do
  if [ $v = auto ]; then unset SAD_BAND_ROWS; else export SAD_BAND_ROWS=$v; fi
  timeout 600 python bench.py --no-c3 --no-cpu-baseline --c4-steps 2 > $O/bench_c4_rt_$v.json 2> $O/bench_c4_rt_$v.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_rt_$v.json').read().strip().splitlines()[-1])
print('SPMM $v', d['value'], d['roofline']['frac'], d['ms_per_step'])
PY
done
