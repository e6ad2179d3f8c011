cd $GRAFT_REPO_ROOT
TAG=${1:-r2j}
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe2 tools/tma_probe2.cu -lcuda > gpurun_out/${TAG}_tma_probe2.log 2>&1
timeout 60 /tmp/tma_probe2 >> gpurun_out/${TAG}_tma_probe2.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_tma_probe2.log
timeout 1700 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --steps 6 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --config 3 --sharded --steps 1 --warmup 1 --no-e2e --no-micro --no-variants --no-extra --no-cpu > gpurun_out/${TAG}_bench_c3_sharded.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench_c3_sharded.log
timeout 900 python bench.py --config 3 --sharded --scaling weak --steps 1 --warmup 1 --no-e2e --no-micro --no-variants --no-extra --no-cpu > gpurun_out/${TAG}_bench_c3_weak.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench_c3_weak.log
