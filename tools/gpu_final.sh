#!/bin/bash
# round-2 measurement session: GPU suite + smoke, full bench, reference arm,
# ncu launch lists of the three paths
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/final_pytest.log 2>&1; tail -22 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
timeout 1200 python bench.py > gpurun_out/final_bench.log 2>&1; tail -c 600 gpurun_out/final_bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1; tail -c 300 gpurun_out/final_bench_ref.log
for w in critic policy; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final_launches_$w.csv python tools/prof_critic.py $w > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches_actor.csv python tools/prof_actor.py > /dev/null 2>&1
for f in critic policy actor; do python tools/launch_summary.py gpurun_out/final_launches_$f.csv > gpurun_out/final_launches_$f.txt; done
exit 0
