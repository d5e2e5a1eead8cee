# ncu --set full over every kernel of one c3 critic update, one policy update
# and one actor step (+ ingest); raw CSVs for tools/roofline_table.py
set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled \
  --launch-skip 2 --launch-count 20 -o gpurun_out/all_critic -f python tools/prof_one.py critic > gpurun_out/ncu_all_critic.log 2>&1
ncu -i gpurun_out/all_critic.ncu-rep --page raw --csv > gpurun_out/all_critic_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled \
  --launch-skip 2 --launch-count 26 -o gpurun_out/all_policy -f python tools/prof_one.py policy > gpurun_out/ncu_all_policy.log 2>&1
ncu -i gpurun_out/all_policy.ncu-rep --page raw --csv > gpurun_out/all_policy_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled \
  --launch-skip 4 --launch-count 12 -o gpurun_out/all_actor -f python tools/prof_one.py actor > gpurun_out/ncu_all_actor.log 2>&1
ncu -i gpurun_out/all_actor.ncu-rep --page raw --csv > gpurun_out/all_actor_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep; ls -la gpurun_out/
