# 2D RAS apply compile-time variants (build tags), timed at config 2 with apply parity per variant
#   VARIANTS="tag:-DFOO=1 -DBAR=2;tag2:..."
cd $GRAFT_REPO_ROOT
TAG=${1:-var}
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  T=${v%%:*}; DEFS=${v#*:}
  NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_${T}_build.log 2>&1 || { echo "$T build failed" >> gpurun_out/${TAG}.log; continue; }
  echo "== $T: $DEFS" >> gpurun_out/${TAG}.log
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" NSUBS="4,4" timeout 300 python tools/ras2d_step_cost.py >> gpurun_out/${TAG}.log 2>&1
  [ -n "$PARITY" ] && NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ras2d_apply" 2>&1 | tail -1 >> gpurun_out/${TAG}.log
done
