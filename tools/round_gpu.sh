# full GPU suite, default bench, launch list and one full ncu capture of the 2D RAS apply
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final5.log 2>&1; tail -3 gpurun_out/gpu_tests_final5.log
python bench.py > gpurun_out/bench_final5.log 2> gpurun_out/bench_final5.err; tail -c 400 gpurun_out/bench_final5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-micro > gpurun_out/ncu_launch_final5.log 2>&1; echo ncu1 $?
bash tools/ncu_r2.sh > /dev/null 2>&1; echo ncu2 $?
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_final5.log 2>&1; tail -2 gpurun_out/smoke_final5.log
