#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_gemm_kernel -c 1 \
  -o gpurun_out/r2_chain -f python tools/prof_actor.py > gpurun_out/r2_ncu_chain.log 2>&1
ncu -i gpurun_out/r2_chain.ncu-rep --page raw --csv > gpurun_out/r2_chain_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_chain.ncu-rep --page details > gpurun_out/r2_chain_details.txt 2>/dev/null
ncu -i gpurun_out/r2_chain.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_chain_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2_chain_raw.csv | head -16
exit 0
