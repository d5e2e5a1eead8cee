#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ab_actor.py 2>&1 | tail -4
timeout 1500 python -m pytest tests/test_actor_gpu.py tests/test_dp_gpu.py tests/test_sac_gpu.py \
  tests/test_pipeline_gpu.py tests/test_checkpoint_gpu.py tests/test_evaluate_gpu.py tests/test_dropin_gpu.py -q -x 2>&1 | tail -6
exit 0
