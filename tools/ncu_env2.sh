#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"env_step" --launch-skip 1 -c 1 \
  -o gpurun_out/r2_env2 -f python tools/prof_actor.py > gpurun_out/r2_ncu_env2.log 2>&1
ncu -i gpurun_out/r2_env2.ncu-rep --page raw --csv > gpurun_out/r2_env2_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_env2.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_env2_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2_env2_raw.csv
python tools/sass_hot.py gpurun_out/r2_env2_sass.csv env_step 30
exit 0
