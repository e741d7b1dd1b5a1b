CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 900 python tools/c2_phase.py 2>&1 | grep -E "^concurrent|Error"
CONC=1 PHASE=direct timeout 600 python tools/c2_phase.py 2>&1 | grep -E "^concurrent|Error"
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
