timeout 900 ncu --set full --clock-control none -k regex:rounds_fused_kernel -s 2 -c 1 -o gpurun_out/fr_full python profiles/k3_rounds.py > /dev/null 2>&1; echo rc=$?
ncu -i gpurun_out/fr_full.ncu-rep --page raw --csv > gpurun_out/fr_full_raw.csv 2>/dev/null
ncu -i gpurun_out/fr_full.ncu-rep --page details --csv > gpurun_out/fr_full_details.csv 2>/dev/null
ls -la gpurun_out/fr_full*
