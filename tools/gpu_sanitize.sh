#!/bin/bash
# compute-sanitizer over the small DDPG / C51 / SAC workload (eager launches)
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_$t.log 2>&1
  echo "== $t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_$t.log | tail -2 | tr '\n' ' ')"
done
exit 0
