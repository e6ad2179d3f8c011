cd $GRAFT_REPO_ROOT
TAG=${1:-prof}
NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_build.log 2>&1 || exit 1
NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE NKS_RAS2D_PROF=1 NSUBS="4,4" \
  timeout 300 python tools/ras2d_step_cost.py > gpurun_out/${TAG}.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}.log
