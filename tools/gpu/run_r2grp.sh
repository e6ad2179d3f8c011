# 2D RAS apply: factor-stream transport (NKS_R2_LDGSTS) x steps per group (NKS_R2_G) x group buffers (NKS_R2_NS),
# timed at config 2 + apply parity per variant
cd $GRAFT_REPO_ROOT
TAG=${1:-grp}
VARIANTS=${VARIANTS:-"0 2 4;1 2 4;1 4 2;1 2 3;0 2 4"}
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  set -- $v
  T=l$1g$2n$3
  DEFS="-DNKS_R2_LDGSTS=$1 -DNKS_R2_G=$2 -DNKS_R2_NS=$3"
  NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_${T}_build.log 2>&1 || { echo "$T build failed" >> gpurun_out/${TAG}.log; continue; }
  echo "== LDGSTS $1 G $2 NS $3" >> gpurun_out/${TAG}.log
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" NSUBS="4,4" timeout 300 python tools/ras2d_step_cost.py >> gpurun_out/${TAG}.log 2>&1
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ras2d_apply or ras_bilu0 or fp32" 2>&1 | tail -1 >> gpurun_out/${TAG}.log
done
