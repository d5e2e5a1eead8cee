# ncu --set full on the actor-step kernels (env step, normalizer update, n-step emit)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"env_step|norm_update|nstep_emit|PolicyHead" -c 4 -o gpurun_out/actor_full -f python tools/prof_actor.py > gpurun_out/ncu_actor.log 2>&1
ncu -i gpurun_out/actor_full.ncu-rep --page raw --csv > gpurun_out/actor_full_raw.csv 2>/dev/null
ncu -i gpurun_out/actor_full.ncu-rep --page source --csv > gpurun_out/actor_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/actor_full_raw.csv
