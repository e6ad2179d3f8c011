cd $GRAFT_REPO_ROOT
TAG=${1:-traj}
python -m paper_2209_08001_b200.build > /dev/null 2>&1 || exit 1
STALL=3 DTS=2.0,1.41421356,1.0 timeout 600 python tools/attempt_cost.py > gpurun_out/${TAG}_attempts.log 2>&1
STALL=0,3 STEPS=9 timeout 1500 python tools/trajectory_check.py > gpurun_out/${TAG}.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "breakdown or gmres or large_dt or adaptive" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-variants --no-extra > gpurun_out/${TAG}_bench.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_bench.log
