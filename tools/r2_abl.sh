for gl in 0 1; do echo "== GL=$gl: $( ( [ $gl = 1 ] && export NKS_RAS2D_GL=1; NKS_RAS2D_PROF=1 SHAPE=256,256 NSUB=2,2 timeout 60 python tools/time_pc.py 2>&1 | grep -E 'cta  [0] |ras_apply|Error' | tail -2 | tr "\n" " ") )"; done
NKS_RAS2D_GL=1 python tools/cmp_ras2d.py
