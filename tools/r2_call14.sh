set -x
O=gpurun_out/r2e
mkdir -p $O
for v in default nobandp noband; do
  unset SAD_BAND_PERSISTENT SAD_SPMM_BAND
  [ $v = nobandp ] && export SAD_BAND_PERSISTENT=0
  [ $v = noband ] && export SAD_SPMM_BAND=0
  timeout 900 python tools/run_config.py c3 --no-verify --reps 2 --profile > $O/run_c3_$v.json 2> $O/run_c3_$v.err
  python - <<PY
import json
d=json.loads(open('$O/run_c3_$v.json').read().strip().splitlines()[0])
print('C3 $v', d['walls_s'], d['outer_steps'], d['sum_inner_A'], d['setup_s'], d['peak_mem_gb'], d.get('profile'))
PY
done
