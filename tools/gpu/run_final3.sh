# round-2 session-3 final measurements: GPU tests, smoke, bench, ncu launch list + RAS apply capture, config-3 phases
cd $GRAFT_REPO_ROOT
TAG=${1:-r2f4}
timeout 1700 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --steps 6 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 4000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants \
  --no-extra --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch rc $?" >> gpurun_out/${TAG}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 5 -c 1 \
  -o gpurun_out/${TAG}_r2apply python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants --no-extra \
  --no-cpu > gpurun_out/${TAG}_ncu_r2.log 2>&1
echo "ncu r2 rc $?" >> gpurun_out/${TAG}_ncu_r2.log
CFG=3 DT=0.5 timeout 600 python tools/time_step_phases.py > gpurun_out/${TAG}_c3_phases.log 2>&1
echo "rc $?" >> gpurun_out/${TAG}_c3_phases.log
