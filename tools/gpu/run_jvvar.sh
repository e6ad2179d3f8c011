# J.v thread-count variants: micro timing at 2D 512^2, 3D 256^3 / 512^3 + J.v parity
cd $GRAFT_REPO_ROOT
TAG=${1:-jv}
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  T=${v%%:*}; DEFS=${v#*:}
  NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_${T}_build.log 2>&1 || { echo "$T build failed" >> gpurun_out/${TAG}.log; continue; }
  echo "== $T $DEFS" >> gpurun_out/${TAG}.log
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" timeout 600 python tools/micro_fjv.py 2d512 3d256 3d512 >> gpurun_out/${TAG}.log 2>&1
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jv" 2>&1 | tail -1 >> gpurun_out/${TAG}.log
done
