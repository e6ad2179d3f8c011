SHAPE=256,256 NSUB=2,2 timeout 60 python tools/time_pc.py 2>&1 | grep -E 'ras_apply|Error' | tail -1
python tools/cmp_ras2d.py
python -m pytest tests -m gpu -x -q -k "ras or schwarz or pc or variants" 2>&1 | tail -2
