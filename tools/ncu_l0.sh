# ncu --set full on the critic update's 4-group layer-0 launch (K = 231)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"Hidden" --launch-skip 3 --launch-count 1 -o gpurun_out/l0_full -f python tools/prof_critic.py critic > gpurun_out/ncu_l0.log 2>&1
ncu -i gpurun_out/l0_full.ncu-rep --page details > gpurun_out/l0_details.txt 2>/dev/null
ncu -i gpurun_out/l0_full.ncu-rep --page raw --csv > gpurun_out/l0_raw.csv 2>/dev/null
ncu -i gpurun_out/l0_full.ncu-rep --page source --csv --print-source sass > gpurun_out/l0_source.csv 2>/dev/null
rm -f gpurun_out/l0_full.ncu-rep
