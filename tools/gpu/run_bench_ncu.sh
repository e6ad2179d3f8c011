cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
STEPS=${2:-6}
timeout 900 python -m pytest tests/test_gpu_sharded_step.py -q -rf > gpurun_out/${TAG}_pytest_shard.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_shard.log
timeout 1500 python bench.py --steps $STEPS --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 150000 -c 6000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-micro --no-variants \
  --no-extra --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu rc $?" >> gpurun_out/${TAG}_ncu_launch.log
