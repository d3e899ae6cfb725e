#!/bin/bash
python profiles/two_round_prof.py 1.0 > gpurun_out/two2_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/two2_launches_s1.csv python profiles/two_round_prof.py 1.0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/two2_launches_s0.csv python profiles/two_round_prof.py 0.0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:two_round_step -c 1 -o gpurun_out/two2_full_s1 python profiles/two_round_prof.py 1.0 > gpurun_out/two2_ncu_full.log 2>&1
ncu -i gpurun_out/two2_full_s1.ncu-rep --page raw --csv > gpurun_out/two2_full_s1_raw.csv 2>/dev/null
ncu -i gpurun_out/two2_full_s1.ncu-rep --page details --csv > gpurun_out/two2_full_s1_details.csv 2>/dev/null
ls -la gpurun_out | head
