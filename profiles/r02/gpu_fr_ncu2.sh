timeout 900 ncu --set full --import-source on --clock-control none -k regex:rounds_fused_kernel -c 1 -o gpurun_out/fr2_full python profiles/fused_rounds_bench.py > /dev/null 2>&1; echo rc=$?
ncu -i gpurun_out/fr2_full.ncu-rep --page raw --csv > gpurun_out/fr2_full_raw.csv 2>/dev/null
ncu -i gpurun_out/fr2_full.ncu-rep --page details --csv > gpurun_out/fr2_full_details.csv 2>/dev/null
ncu -i gpurun_out/fr2_full.ncu-rep --page source --csv --print-source sass > gpurun_out/fr2_source.csv 2>/dev/null; echo src rc=$?
ls -la gpurun_out/fr2*
