cd $GRAFT_REPO_ROOT
TAG=${1:-r2g}
timeout 1200 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_parity.py tests/test_gpu_sharded_step.py -q -rf > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 4 --warmup 3 --no-micro --no-extra > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 600 python tools/ras2d_step_cost.py > gpurun_out/${TAG}_r2cost_default.log 2>&1
NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_abl_build.log 2>&1
for cs in 1 2 8; do
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_RAS2D_CSMAX=$cs timeout 600 python tools/ras2d_step_cost.py > gpurun_out/${TAG}_r2cost_cs$cs.log 2>&1
done
