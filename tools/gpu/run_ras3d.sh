# 3D RAS apply: one CTA per box vs a cluster of CTAs per box, at config 4's per-GPU share of boxes
cd $GRAFT_REPO_ROOT
TAG=${1:-r3d}
IFS=';' read -ra VS <<< "${VARIANTS:-cs1:-DNKS_RAS3D_CSMAX=1;cs2:-DNKS_RAS3D_CSMAX=2;cs4:-DNKS_RAS3D_CSMAX=4 -DNKS_RAS3D_WIDTH=0}"
for v in "${VS[@]}"; do
  T=${v%%:*}; DEFS=${v#*:}
  NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_${T}_build.log 2>&1 || { echo "$T build failed" >> gpurun_out/${TAG}.log; continue; }
  for g in "256,256,32:8,8,1" "256,256,64:8,8,2" "128,128,128:8,8,8"; do
    echo "== $T $DEFS shape ${g%%:*} nsub ${g#*:}" >> gpurun_out/${TAG}.log
    NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so SHAPE=${g%%:*} NSUB=${g#*:} CFG=4 timeout 300 python tools/time_pc.py >> gpurun_out/${TAG}.log 2>&1
  done
done
