set -x
O=gpurun_out/r2g
mkdir -p $O
for cap in 108 92; do
SAD_BAND_CAP_KB=$cap timeout 1500 python tools/run_config.py c5 --no-verify --profile > $O/run_c5_cap$cap.json 2> $O/run_c5_cap$cap.err
python - <<PY
import json
d=json.loads(open('$O/run_c5_cap$cap.json').read().strip().splitlines()[0])
p=d['profile']
print('C5 cap$cap', d['walls_s'], p['algorithmic_GBps'], 'A', p['phaseA_ms'], 'C', p['phaseC_ms'], 'spmm', p['spmmA_ms'])
PY
done
SAD_BAND_CAP_KB=108 timeout 900 python bench.py --no-c3 --no-cpu-baseline --steps 3 > $O/bench_c4_cap108.json 2> $O/bench_c4_cap108.err
python - <<PY
import json
d=json.loads(open('$O/bench_c4_cap108.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('PERS cap108', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'], 'A', i['phaseA_ms'], 'C', i['phaseC_ms'])
PY
