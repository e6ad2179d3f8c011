cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
STEPS=${2:-6}
timeout 1700 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 1500 python bench.py --steps $STEPS --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python tools/pc_table.py > gpurun_out/${TAG}_pc_table.log 2>&1
echo "pc_table rc $?" >> gpurun_out/${TAG}_pc_table.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 4000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants \
  --no-extra --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch rc $?" >> gpurun_out/${TAG}_ncu_launch.log
