# ncu --set full on the C51 critic update's 4-group categorical head launch
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"C51Head" --launch-count 1 -o gpurun_out/c51h -f python tools/prof_critic.py c51 > gpurun_out/ncu_c51h.log 2>&1
ncu -i gpurun_out/c51h.ncu-rep --page details > gpurun_out/c51h_details.txt 2>/dev/null
ncu -i gpurun_out/c51h.ncu-rep --page raw --csv > gpurun_out/c51h_raw.csv 2>/dev/null
rm -f gpurun_out/c51h.ncu-rep
