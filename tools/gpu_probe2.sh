#!/bin/bash
# epilogue phase trace + ncu of the actor's non-GEMM kernels (round 2)
mkdir -p gpurun_out
TRACE_STORE=1 timeout 300 python tools/gemm_trace.py > gpurun_out/gemm_trace.log 2>&1; grep -v "^nvcc\|warn" gpurun_out/gemm_trace.log | tail -6
TRACE_STORE=0 timeout 300 python tools/gemm_trace.py > gpurun_out/gemm_trace0.log 2>&1; tail -6 gpurun_out/gemm_trace0.log
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"head_mma_kernel|norm_partial|norm_finish|env_step_kernel" --launch-skip 8 -c 4 \
  -o gpurun_out/r2_actor2 -f python tools/prof_actor.py > gpurun_out/r2_ncu3.log 2>&1
ncu -i gpurun_out/r2_actor2.ncu-rep --page raw --csv > gpurun_out/r2_actor2_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_actor2.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_actor2_sass.csv 2>/dev/null
ncu -i gpurun_out/r2_actor2.ncu-rep --page details > gpurun_out/r2_actor2_details.txt 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2_actor2_raw.csv
exit 0
