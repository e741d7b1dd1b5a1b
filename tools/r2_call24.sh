# round 2, call 24: warp-specialised producer in the persistent kernel's banded SpMM sub-phase
set -x
O=gpurun_out/r2h
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spmm_band.py tests/test_gpu_adi.py tests/test_gpu_race.py -q > $O/pytest_sel.log 2>&1; tail -3 $O/pytest_sel.log
SAD_SPMM_BAND=1 timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_bandforced.log 2>&1; tail -3 $O/pytest_gpu_bandforced.log
for tr in auto 64; do
  if [ $tr = auto ]; then unset SAD_BAND_ROWS_P; else export SAD_BAND_ROWS_P=$tr; fi
  timeout 900 python bench.py --no-c3 --no-cpu-baseline --steps 3 > $O/bench_c4_$tr.json 2> $O/bench_c4_$tr.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_$tr.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('PERS $tr', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'], 'A', i['phaseA_ms'], 'C', i['phaseC_ms'])
PY
done
unset SAD_BAND_ROWS_P
timeout 1500 python tools/run_config.py c5 --no-verify --profile > $O/run_c5.json 2> $O/run_c5.err
python - <<PY
import json
d=json.loads(open('$O/run_c5.json').read().strip().splitlines()[0])
p=d['profile']
print('C5', d['walls_s'], p['algorithmic_GBps'], 'A', p['phaseA_ms'], 'C', p['phaseC_ms'], 'spmm', p['spmmA_ms'])
PY
