cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
STEPS=${2:-4}
timeout 1700 python -m pytest tests -m gpu -q -s -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps $STEPS --warmup 3 --no-micro > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
