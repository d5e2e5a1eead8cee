#!/bin/bash
# GEMM layout / pairing probe + in-situ ncu captures (round 2)
mkdir -p gpurun_out
timeout 600 python tools/gemm_major.py > gpurun_out/gemm_major.log 2>&1; cat gpurun_out/gemm_major.log
PQLG_PAIR=0 timeout 600 python tools/gemm_major.py > gpurun_out/gemm_major_nopair.log 2>&1; cat gpurun_out/gemm_major_nopair.log
TRACE_STORE=1 timeout 300 python tools/gemm_trace.py > gpurun_out/gemm_trace.log 2>&1; tail -6 gpurun_out/gemm_trace.log
TRACE_STORE=0 timeout 300 python tools/gemm_trace.py > gpurun_out/gemm_trace0.log 2>&1; tail -6 gpurun_out/gemm_trace0.log
bash tools/ncu_r2.sh
exit 0
