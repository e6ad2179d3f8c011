# 2D RAS apply ablations (ablation build, timing only: results are wrong when dbg != 0)
#   4 = no DSMEM push, 16 = no halo polls, 32 = no block-row preloads, 64 = no global loads,
#   128 = no copy management after the first groups, 256 = no global stores
cd $GRAFT_REPO_ROOT
TAG=${1:-abl3}
NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_build.log 2>&1 || exit 1
for d in ${DBGS:-0 128 16 144 32 64 260 176 500}; do
  echo "== dbg $d" >> gpurun_out/${TAG}.log
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE NKS_RAS2D_DBG=$d NSUBS="4,4" \
    timeout 300 python tools/ras2d_step_cost.py >> gpurun_out/${TAG}.log 2>&1
done
