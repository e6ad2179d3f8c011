cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
# launch list (gpu__time_duration, clock-control none) of the bench's first step: its kernel shares
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 4000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants \
  --no-extra --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch rc $?" >> gpurun_out/${TAG}_ncu_launch.log
# full capture of the 2D RAS apply at config 2 and of F / J.v at 3D 256^3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 5 -c 1 \
  -o gpurun_out/${TAG}_r2apply python bench.py --steps 1 --warmup 0 --no-e2e --no-micro --no-variants --no-extra \
  --no-cpu > gpurun_out/${TAG}_ncu_r2.log 2>&1
echo "ncu r2 rc $?" >> gpurun_out/${TAG}_ncu_r2.log
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_jv_tiled|k_residual_tiled" -s 2 -c 2 \
  -o gpurun_out/${TAG}_fjv python tools/micro_fjv.py 3d256 > gpurun_out/${TAG}_ncu_fjv.log 2>&1
echo "ncu fjv rc $?" >> gpurun_out/${TAG}_ncu_fjv.log
timeout 900 python tools/pc_table.py > gpurun_out/${TAG}_pc_table.log 2>&1
echo "pc_table rc $?" >> gpurun_out/${TAG}_pc_table.log
timeout 1200 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_parity.py -q -rf -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest.log
