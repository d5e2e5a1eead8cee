#!/bin/bash
# iteration: full GPU suite, actor / update A/B timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/iter_pytest.log 2>&1; tail -15 gpurun_out/iter_pytest.log
timeout 300 python tools/ab_actor.py 2>&1 | tail -4
[ -n "$UPDATE" ] && timeout 300 python tools/ab_update.py 2>&1 | tail -1
exit 0
