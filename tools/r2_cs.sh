#!/bin/bash
# Sweep the 2D RAS rows kernel's cluster size (stripes per box) at config 2's geometry.
for cs in ${CS_LIST:-6 8 9 10 11 12 14 16}; do
  echo "== CS $cs: $(NKS_DEBUG=1 NKS_RAS2D_CSMAX=16 NKS_RAS2D_CS=$cs SHAPE=${SHAPE:-512,512} NSUB=${NSUB:-4,4} timeout 120 python tools/cmp_ras2d.py 2>&1 | grep -E 'ras2d rows|nsub' | tr '\n' ' ')"
done
