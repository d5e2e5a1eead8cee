#!/bin/bash
# GPU-box session: tests, smoke, bench, ncu launch lists and one full capture.
#   bash tools/gpu_check.sh [tests] [bench] [launch] [full] [ref]
# Everything lands in gpurun_out/ (merged back by gpurun).
set -x
what="${*:-tests bench launch full}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
has() { [[ " $what " == *" $1 "* ]]; }
if has tests; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  tail -n 30 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  tail -n 3 gpurun_out/smoke.log
fi
if has bench; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1
  tail -c 4000 gpurun_out/bench.log
fi
if has ref; then
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
  tail -c 1500 gpurun_out/bench_ref.log
fi
if has launch; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_critic.csv python tools/prof_critic.py critic > gpurun_out/ncu1.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_actor.csv python tools/prof_actor.py > gpurun_out/ncu2.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_policy.csv python tools/prof_critic.py policy > gpurun_out/ncu3.log 2>&1
  for f in critic actor policy; do python tools/launch_summary.py gpurun_out/launches_$f.csv; done
fi
if has full; then
  # one full capture of the dominant kernel (hidden-layer forward GEMM, 8192x512x512)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel -c 1 \
    -o gpurun_out/gemm_hidden_full -f python tools/prof_critic.py gemm > gpurun_out/ncu_full.log 2>&1
  ncu -i gpurun_out/gemm_hidden_full.ncu-rep --page raw --csv > gpurun_out/gemm_hidden_full_raw.csv 2>/dev/null
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel -c 1 \
    -o gpurun_out/gemm4_full -f python tools/prof_critic.py gemm4 > gpurun_out/ncu_full4.log 2>&1
  ncu -i gpurun_out/gemm4_full.ncu-rep --page raw --csv > gpurun_out/gemm4_full_raw.csv 2>/dev/null
  # and the critic update's finalize / adam kernels (HBM-bound)
  timeout 900 ncu --set full --clock-control none -k regex:"finalize_kernel|adam_polyak|replay_sample_kernel" -c 3 \
    -o gpurun_out/critic_hbm_full -f python tools/prof_critic.py critic > gpurun_out/ncu_full2.log 2>&1
  ncu -i gpurun_out/critic_hbm_full.ncu-rep --page raw --csv > gpurun_out/critic_hbm_full_raw.csv 2>/dev/null
fi
exit 0
