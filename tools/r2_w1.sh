# one-warp-per-stripe 2D RAS apply (NKS_RAS2D_W1) against the default kernel: time and parity
for v in 0 1; do echo "== W1=$v: $( ( [ $v = 1 ] && export NKS_RAS2D_W1=1; NKS_DEBUG=1 NKS_RAS2D_PROF=1 SHAPE=256,256 NSUB=2,2 timeout 120 python tools/time_pc.py 2>&1 | grep -E 'ras2d rows:|cta  [0] |ras_apply|Error' | tail -3 | tr "\n" " ") )"; done
NKS_RAS2D_W1=1 timeout 300 python tools/cmp_ras2d.py
