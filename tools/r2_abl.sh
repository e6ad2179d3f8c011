for d in 0 128; do echo "== dbg $d: $(NKS_RAS2D_DBG=$d NKS_RAS2D_PROF=1 SHAPE=256,256 NSUB=2,2 timeout 60 python tools/time_pc.py 2>&1 | grep -E 'producer step 4[01]|cta  [0] |ras_apply|Error' | tail -4 | tr '\n' ' ')"; done
python tools/cmp_ras2d.py
