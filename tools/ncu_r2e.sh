#!/bin/bash
# full ncu captures of the actor's env step / head / normalizer kernels (source-level)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"env_step|head_mma|norm_" -c 4 \
  -o gpurun_out/actor2_full -f python tools/prof_actor.py > gpurun_out/ncu_actor2.log 2>&1
ncu -i gpurun_out/actor2_full.ncu-rep --page raw --csv > gpurun_out/actor2_raw.csv 2>/dev/null
ncu -i gpurun_out/actor2_full.ncu-rep --page source --csv > gpurun_out/actor2_source.csv 2>/dev/null
ncu -i gpurun_out/actor2_full.ncu-rep --page details --csv > gpurun_out/actor2_details.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/actor2_raw.csv > gpurun_out/actor2_summary.txt 2>&1
grep -E "==|duration|dram read|dram write|occupancy|L2 %|SM %" gpurun_out/actor2_summary.txt
exit 0
