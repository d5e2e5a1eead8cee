#!/bin/bash
# round-2 ncu captures (one GPU): the in-update 4-group hidden-layer GEMM
# (launch 5 of the critic update's GEMMs = critic layer 1) and the actor
# step's kernels.  Exports raw + source pages to gpurun_out/.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel \
  --launch-skip 5 --launch-count 1 -o gpurun_out/r2_gemm4_insitu -f \
  python tools/prof_critic.py critic > gpurun_out/r2_ncu1.log 2>&1
ncu -i gpurun_out/r2_gemm4_insitu.ncu-rep --page raw --csv > gpurun_out/r2_gemm4_insitu_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_gemm4_insitu.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_gemm4_insitu_sass.csv 2>/dev/null
ncu -i gpurun_out/r2_gemm4_insitu.ncu-rep --page details > gpurun_out/r2_gemm4_insitu_details.txt 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tf32_kernel|env_step_kernel|norm_update_kernel" --launch-skip 6 -c 6 \
  -o gpurun_out/r2_actor -f python tools/prof_actor.py > gpurun_out/r2_ncu2.log 2>&1
ncu -i gpurun_out/r2_actor.ncu-rep --page raw --csv > gpurun_out/r2_actor_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_actor.ncu-rep --page details > gpurun_out/r2_actor_details.txt 2>/dev/null
rm -f gpurun_out/*.ncu-rep.tmp
ls -la gpurun_out | tail -12
python tools/ncu_summary.py gpurun_out/r2_gemm4_insitu_raw.csv | head -20
exit 0
