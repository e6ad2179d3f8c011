# 2D RAS apply ablations (ablation build): 512 = factor groups copied from L2-resident rows (no HBM stream)
cd $GRAFT_REPO_ROOT
TAG=${1:-abl}
NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_build.log 2>&1 || exit 1
for d in 0 512 544 576 0; do
  echo "== dbg $d" >> gpurun_out/${TAG}.log
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE NKS_RAS2D_DBG=$d NSUBS="4,4;8,8" \
    timeout 300 python tools/ras2d_step_cost.py >> gpurun_out/${TAG}.log 2>&1
done
