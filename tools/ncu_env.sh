# ncu --set full on the synthetic env step only (source-level stalls)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"env_step" -c 1 -o gpurun_out/env_full -f python tools/prof_actor.py > gpurun_out/ncu_env.log 2>&1
ncu -i gpurun_out/env_full.ncu-rep --page raw --csv > gpurun_out/env_full_raw.csv 2>/dev/null
ncu -i gpurun_out/env_full.ncu-rep --page source --csv > gpurun_out/env_source.csv 2>/dev/null
ncu -i gpurun_out/env_full.ncu-rep --page details > gpurun_out/env_details.txt 2>/dev/null
rm -f gpurun_out/env_full.ncu-rep
