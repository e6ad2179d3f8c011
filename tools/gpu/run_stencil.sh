# F / J.v two-barrier pipeline: parity (incl. sampled full size and the sharded step) + micro timings
cd $GRAFT_REPO_ROOT
TAG=${1:-r2s}
python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "residual or jv or step_parity_3d or single_particle" \
  > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python -m pytest tests/test_gpu_sharded_step.py tests/test_gpu_neumann.py -q -x >> gpurun_out/${TAG}_pytest.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_pytest.log
REPS=20 timeout 600 python tools/micro_fjv.py 3d128 3d256 3d512 > gpurun_out/${TAG}_micro.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_micro.log
