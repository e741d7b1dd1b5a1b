# round 2, call 12: banded SpMM inside the persistent kernel (sub-phase A1)
set -x
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band.log 2>&1; tail -5 $O/pytest_band.log
SAD_SPMM_BAND=1 timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_bandforced.log 2>&1; tail -3 $O/pytest_gpu_bandforced.log
for v in auto_auto 64_0 128_2 128_3 ; do
  tr=${v%_*}; st=${v#*_}
  if [ $tr = auto ]; then unset SAD_BAND_ROWS_P; else export SAD_BAND_ROWS_P=$tr; fi
  if [ $st = auto ] || [ $st = 0 ]; then unset SAD_BAND_STAGES_P; else export SAD_BAND_STAGES_P=$st; fi
  timeout 900 python bench.py --no-c3 --no-cpu-baseline --steps 3 > $O/bench_c4_$v.json 2> $O/bench_c4_$v.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_$v.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('PERS $v', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'], 'A', i['phaseA_ms'], 'C', i['phaseC_ms'], 'orth', i['orthogonalisation_gbs'])
PY
done
unset SAD_BAND_ROWS_P SAD_BAND_STAGES_P
SAD_BAND_PERSISTENT=0 timeout 900 python bench.py --no-c3 --no-cpu-baseline --steps 3 > $O/bench_c4_off.json 2> $O/bench_c4_off.err
python - <<PY
import json
d=json.loads(open('$O/bench_c4_off.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('PERS off', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'])
PY
