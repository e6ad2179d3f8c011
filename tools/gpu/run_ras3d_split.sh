# 3D RAS apply register variants (chunked neighbour loads + launch bounds) at config 3 and config 4's shares
cd $GRAFT_REPO_ROOT
TAG=${1:-r3s}
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  T=${v%%:*}; DEFS=${v#*:}
  NKS_BUILD_TAG=$T NKS_BUILD_DEFS="$DEFS" python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_${T}_build.log 2>&1 || { echo "$T build failed" >> gpurun_out/${TAG}.log; continue; }
  for g in "128,128,128:8,8,8" "256,256,64:8,8,2" "256,256,256:8,8,8"; do
    echo "== $T $DEFS shape ${g%%:*} nsub ${g#*:}" >> gpurun_out/${TAG}.log
    NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so SHAPE=${g%%:*} NSUB=${g#*:} CFG=4 timeout 300 python tools/time_pc.py >> gpurun_out/${TAG}.log 2>&1
  done
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_$T.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3d" 2>&1 | tail -1 >> gpurun_out/${TAG}.log
done
