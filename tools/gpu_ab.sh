#!/bin/bash
mkdir -p gpurun_out
PQLG_BRANCHES=0 timeout 300 python tools/ab_update.py 2>&1 | tail -1
PQLG_BRANCHES=1 timeout 300 python tools/ab_update.py 2>&1 | tail -1
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -q -x 2>&1 | tail -5
fi
exit 0
