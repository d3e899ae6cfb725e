#!/bin/bash
ncu --set full --import-source on --clock-control none -k regex:two_round_step -c 1 -o gpurun_out/two5_full_s1 python profiles/two_round_prof.py 1.0 > gpurun_out/two5_ncu_full.log 2>&1
ncu -i gpurun_out/two5_full_s1.ncu-rep --page details --csv > gpurun_out/two5_full_s1_details.csv 2>/dev/null
ncu -i gpurun_out/two5_full_s1.ncu-rep --page raw --csv > gpurun_out/two5_full_s1_raw.csv 2>/dev/null
ncu -i gpurun_out/two5_full_s1.ncu-rep --page source --csv --print-source cuda > gpurun_out/two5_full_s1_source.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:two_round_step -c 1 -o gpurun_out/two5_full_s0 python profiles/two_round_prof.py 0.0 > /dev/null 2>&1
ncu -i gpurun_out/two5_full_s0.ncu-rep --page source --csv --print-source cuda > gpurun_out/two5_full_s0_source.csv 2>/dev/null
ncu -i gpurun_out/two5_full_s0.ncu-rep --page raw --csv > gpurun_out/two5_full_s0_raw.csv 2>/dev/null
ls -la gpurun_out/two5*
