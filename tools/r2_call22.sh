set -x
O=gpurun_out/r2g
mkdir -p $O
run() { CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py 2>&1 | tail -2 | sed "s/^/PH $1 /"; }
SAD_RING_C=1 run ringc1
SAD_RING_C=2 run ringc2
SAD_RING_C=2 SAD_SWEEP=tma run ringc2_sweeptma
timeout 1500 python tools/run_config.py c5 --no-verify --profile > $O/run_c5_ringc.json 2> $O/run_c5_ringc.err
python - <<PY
import json
d=json.loads(open('$O/run_c5_ringc.json').read().strip().splitlines()[0])
print('C5', d['walls_s'], d['outer_steps'], d['sum_inner_A'], d['sum_inner_B'], d.get('profile'))
PY
