MOSHPIT_LOGIT_TC=1 timeout 600 python profiles/logistic_tc_bench.py 1024 1024 4096 2 > /dev/null 2>&1 && MOSHPIT_LOGIT_TC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 2 -c 2 -o gpurun_out/tc_src python profiles/logistic_tc_bench.py 1024 1024 4096 2 > /dev/null 2>&1; echo rc=$?
ncu -i gpurun_out/tc_src.ncu-rep --page details --csv > gpurun_out/tc_src_details.csv 2>/dev/null
ncu -i gpurun_out/tc_src.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_src_source.csv 2>/dev/null; echo rc=$?
