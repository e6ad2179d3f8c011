cd $GRAFT_REPO_ROOT
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 1700 python -m pytest tests -m gpu -q -s -rf > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 6 --warmup 3 > gpurun_out/r2_bench1.log 2>&1
echo "bench rc $?" >> gpurun_out/r2_bench1.log
