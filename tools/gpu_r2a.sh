#!/bin/bash
# round-2 check: new GPU tests + bench (everything lands in gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dropin_gpu.py tests/test_actor_gpu.py tests/test_evaluate_gpu.py \
  tests/test_pipeline_gpu.py -q -s > gpurun_out/r2a_pytest.log 2>&1
tail -n 25 gpurun_out/r2a_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.log 2> gpurun_out/r2a_bench.err
tail -c 2500 gpurun_out/r2a_bench.log; tail -5 gpurun_out/r2a_bench.err
exit 0
