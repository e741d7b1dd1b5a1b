CONC=1 PHASE=auto,direct timeout 600 python tools/c2_phase.py 2>&1 | grep -E "^concurrent|Error"
SPLITS=0.85,0.82,0.8 timeout 600 python tools/c2_split.py 2>&1 | grep -E "^split|Error"
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
