#!/bin/bash
# quick GPU check: gpu tests (optionally a subset via PYTEST_K / PYTEST_FILES), GEMM trace + micro, bench
set -x
timeout 1200 python -m pytest ${PYTEST_FILES:-tests} -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -25
timeout 300 python tools/gemm_trace.py 2>&1 | tail -8
timeout 300 python tools/gemm_micro.py 2>&1 | tail -8
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("critic", round(d["value"], 1), "ms", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 1))
print("actor", round(d["actor"]["value"] / 1e6, 2), "M/s ms", round(d["actor"]["ms_per_step"], 4),
      "step-only", round(d["actor"]["actor_step_only"]["ms_per_step"], 4))
print("policy", d["policy_updates"])
print("c51", d.get("c51"))
print("roofline", d["roofline"])
PY
fi
exit 0
