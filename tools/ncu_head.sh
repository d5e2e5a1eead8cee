#!/bin/bash
# full capture of the actor's fused policy head (source-level stalls)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"head_mma" --launch-skip 1 -c 1 \
  -o gpurun_out/r2_head -f python tools/prof_actor.py > gpurun_out/r2_ncu_head.log 2>&1
ncu -i gpurun_out/r2_head.ncu-rep --page raw --csv > gpurun_out/r2_head_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_head.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_head_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2_head_raw.csv
python tools/sass_hot.py gpurun_out/r2_head_sass.csv head_mma 25
exit 0
