cd $GRAFT_REPO_ROOT
TAG=${1:-r2l}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 4000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants \
  --no-extra --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch rc $?" >> gpurun_out/${TAG}_ncu_launch.log
timeout 600 ncu --set full --clock-control none -k regex:"k_dcgs" -s 200 -c 3 -o gpurun_out/${TAG}_dcgs python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants --no-extra --no-cpu > gpurun_out/${TAG}_ncu_dcgs.log 2>&1
echo "ncu dcgs rc $?" >> gpurun_out/${TAG}_ncu_dcgs.log
