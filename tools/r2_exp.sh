for d in 4 132; do
  echo "== dbg $d"
  NKS_RAS2D_DBG=$d NKS_RAS2D_PROF=1 CFG=2 timeout 60 python tools/time_pc.py 2>&1 | grep -E 'group 8|cta  0|ras_apply' | tail -3
done
