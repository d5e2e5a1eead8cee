#!/bin/bash
# round-2 check: drop-in, sampler hook, actor/env/evaluate/pipeline tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dropin_gpu.py tests/test_replay_gpu.py tests/test_actor_gpu.py \
  tests/test_evaluate_gpu.py tests/test_pipeline_gpu.py -q -s > gpurun_out/r2b_pytest.log 2>&1
grep -E "passed|failed|Error|error" gpurun_out/r2b_pytest.log | tail -n 15
exit 0
