#!/bin/bash
# Ring depth / group size variants of the 2D RAS rows kernel (libs built with NKS_BUILD_TAG, tools/r2_cs.sh sweep).
for lib in libnks libnks_g2ns8 libnks_g4ns4 libnks_g4ns6 libnks_g8ns3; do
  echo "##### $lib"
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/$lib.so CS_LIST="${CS_LIST:-6 16}" bash tools/r2_cs.sh
done
