# ncu --set full on chosen small kernels of a critic update (first arg: regex, second: mode)
K="${1:-PolicyHead}"
MODE="${2:-critic}"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -c 2 -o gpurun_out/small_full -f python tools/prof_critic.py $MODE > gpurun_out/ncu_small.log 2>&1
ncu -i gpurun_out/small_full.ncu-rep --page raw --csv > gpurun_out/small_full_raw.csv 2>/dev/null
ncu -i gpurun_out/small_full.ncu-rep --page source --csv > gpurun_out/small_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/small_full_raw.csv
