for d in 16 20 48 52; do
  echo "== dbg $d: $(NKS_RAS2D_DBG=$d NKS_RAS2D_PROF=1 CFG=2 timeout 60 python tools/time_pc.py 2>&1 | grep -E 'cta  0|ras_apply' | tail -2 | tr '\n' ' ')"
done
