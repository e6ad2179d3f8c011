# one ncu --set full capture of the one-lane-per-row 2D RAS apply at config 2 (tools/time_pc.py)
set -e
CFG=2 timeout 300 python tools/time_pc.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/r2_apply -f python tools/time_pc.py > gpurun_out/ncu_r2.log 2>&1 || true
ncu -i gpurun_out/r2_apply.ncu-rep --page details --csv > gpurun_out/r2_details.csv 2>/dev/null || true
ncu -i gpurun_out/r2_apply.ncu-rep --page raw --csv > gpurun_out/r2_raw.csv 2>/dev/null || true
ncu -i gpurun_out/r2_apply.ncu-rep --page source --csv > gpurun_out/r2_source.csv 2>/dev/null || true
