#!/bin/bash
# round-2 actor pass: in-graph timing, actor-side tests, full ncu captures of
# the actor's non-GEMM kernels and the policy head (source-level)
mkdir -p gpurun_out
timeout 300 python tools/ab_actor.py > gpurun_out/ab_actor.log 2>&1; tail -4 gpurun_out/ab_actor.log
timeout 900 python -m pytest tests/test_actor_gpu.py tests/test_dp_gpu.py tests/test_evaluate_gpu.py \
  tests/test_sac_gpu.py -q -x > gpurun_out/r2c_pytest.log 2>&1; tail -3 gpurun_out/r2c_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"env_step|norm_|PolicyHead" -c 5 \
  -o gpurun_out/actor_full -f python tools/prof_actor.py > gpurun_out/ncu_actor.log 2>&1
ncu -i gpurun_out/actor_full.ncu-rep --page raw --csv > gpurun_out/actor_full_raw.csv 2>/dev/null
ncu -i gpurun_out/actor_full.ncu-rep --page source --csv > gpurun_out/actor_source.csv 2>/dev/null
ncu -i gpurun_out/actor_full.ncu-rep --page details --csv > gpurun_out/actor_details.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/actor_full_raw.csv > gpurun_out/actor_summary.txt 2>&1
head -c 3000 gpurun_out/actor_summary.txt
exit 0
