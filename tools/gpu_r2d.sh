#!/bin/bash
# round-2 iteration: full GPU suite, actor in-graph timing, critic/policy kernel lists, quick bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; tail -15 gpurun_out/r2d_pytest.log
timeout 300 python tools/ab_actor.py > gpurun_out/ab_actor.log 2>&1; tail -4 gpurun_out/ab_actor.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/bench_quick.log") if l.startswith("{")][-1])
print("critic", round(d["value"], 1), "ms", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 1))
print("actor", round(d["actor"]["value"] / 1e6, 2), "M/s ms", round(d["actor"]["ms_per_step"], 4),
      "step-only", round(d["actor"]["actor_step_only"]["ms_per_step"], 4))
print("policy", d["policy_updates"]["ms_per_step"], "c51", d["c51"]["critic_updates"]["ms_per_step"], d["c51"]["policy_updates"]["ms_per_step"])
print("sac", d["sac"]["critic_updates"]["ms_per_step"], d["sac"]["policy_updates"]["ms_per_step"])
print("c2", d["other_configs"]["c2"]); print("c1", d["other_configs"]["c1"])
for k in d["roofline"]["kernels"]: print("  ", k)
PY
exit 0
