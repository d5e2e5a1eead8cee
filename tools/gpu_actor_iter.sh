#!/bin/bash
# actor iteration: actor-side GPU tests + in-graph actor timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_actor_gpu.py tests/test_evaluate_gpu.py tests/test_sac_gpu.py \
  tests/test_dp_gpu.py tests/test_pipeline_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/actor_iter_pytest.log 2>&1
tail -3 gpurun_out/actor_iter_pytest.log
timeout 300 python tools/ab_actor.py > gpurun_out/ab_actor.log 2>&1; cat gpurun_out/ab_actor.log | cut -c1-700
exit 0
