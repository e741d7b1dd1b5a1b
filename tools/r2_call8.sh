set -x
O=gpurun_out/r2c
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band3.log 2>&1; tail -3 $O/pytest_band3.log
for v in default band128 band256; do
  if [ $v = default ]; then unset SAD_LIB_PATH; else export SAD_LIB_PATH=$PWD/tools/bin_$v.so; fi
  timeout 600 python bench.py --no-c3 --no-cpu-baseline --c4-steps 2 > $O/bench_c4_$v.json 2> $O/bench_c4_$v.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_$v.json').read().strip().splitlines()[-1])
print('SPMM $v', d['value'], d['roofline']['frac'], d['ms_per_step'])
PY
done
unset SAD_LIB_PATH
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_band -s 4 -c 1 -o $O/prof_c4_band2 python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 --c4-steps 2 > $O/ncu_band2.log 2>&1
