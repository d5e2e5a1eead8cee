# ncu --set full on the pql_sac-specific kernels (eps stream, Gaussian finish, pick, head backward)
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"eps_|gauss_finish|sac_" -c 8 -o gpurun_out/sac_full -f python tools/prof_sac.py > gpurun_out/ncu_sac.log 2>&1
ncu -i gpurun_out/sac_full.ncu-rep --page raw --csv > gpurun_out/sac_full_raw.csv 2>/dev/null
rm -f gpurun_out/sac_full.ncu-rep
python tools/ncu_summary.py gpurun_out/sac_full_raw.csv
