# round 2, call 17: persistent band path restricted to the TMA-ring sweep; c3/c4/c5 checks
set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm_band.py -x -q > $O/pytest_band.log 2>&1; tail -3 $O/pytest_band.log
CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py 2>&1 | tail -2 | sed "s/^/PH c3 /"
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
python - <<PY
import json
d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1])
i=d['inner_solve']
print('C4', d['value'], d['roofline']['frac'], 'PERS', i['kernel_ms'], i['frac'], 'spmm', i['spmm_subphase_ms'], 'A', i['phaseA_ms'], 'C', i['phaseC_ms'], 'c3', d['config3_wall_time']['value'])
PY
timeout 1500 python tools/run_config.py c5 --no-verify --profile > $O/run_c5.json 2> $O/run_c5.err
python - <<PY
import json
d=json.loads(open('$O/run_c5.json').read().strip().splitlines()[0])
print('C5', d['walls_s'], d['outer_steps'], d['sum_inner_A'], d['sum_inner_B'], d['setup_s'], d['peak_mem_gb'], d.get('profile'))
PY
SAD_BAND_PERSISTENT=0 timeout 1500 python tools/run_config.py c5 --no-verify --profile > $O/run_c5_off.json 2> $O/run_c5_off.err
python - <<PY
import json
d=json.loads(open('$O/run_c5_off.json').read().strip().splitlines()[0])
print('C5off', d['walls_s'], d['outer_steps'], d['sum_inner_A'], d['sum_inner_B'], d['setup_s'], d['peak_mem_gb'], d.get('profile'))
PY
