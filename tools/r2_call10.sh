set -x
O=gpurun_out/r2c
mkdir -p $O
for v in default u3 u4; do
  if [ $v = default ]; then unset SAD_LIB_PATH; else export SAD_LIB_PATH=$PWD/tools/bin_$v.so; fi
  for tr in 256 128; do
  SAD_BAND_ROWS=$tr timeout 600 python bench.py --no-c3 --no-cpu-baseline --c4-steps 2 > $O/bench_c4_u_$v.json 2> $O/bench_c4_u_$v.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_u_$v.json').read().strip().splitlines()[-1])
print('SPMM $v $tr', d['value'], d['roofline']['frac'], d['ms_per_step'])
PY
  done
done
