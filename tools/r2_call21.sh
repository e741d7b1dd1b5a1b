# round 2, call 21: phase C through the TMA ring
set -x
O=gpurun_out/r2g
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spmm_band.py tests/test_gpu_adi.py tests/test_gpu_race.py -q > $O/pytest_sel.log 2>&1; tail -3 $O/pytest_sel.log
for v in 1 0; do
  SAD_RING_C=$v timeout 900 python bench.py --no-c3 --no-cpu-baseline --steps 3 > $O/bench_c4_ringc$v.json 2> $O/bench_c4_ringc$v.err
  python - <<PY
import json
d=json.loads(open('$O/bench_c4_ringc$v.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('PERS ringC=$v', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'], 'A', i['phaseA_ms'], 'C', i['phaseC_ms'], 'orth', i['orthogonalisation_gbs'])
PY
done
