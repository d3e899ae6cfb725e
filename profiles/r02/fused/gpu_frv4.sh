#!/bin/bash
# fused rounds: leaf-row lane mapping + 3 teams with the compact group table -- GPU suite, bench, ncu of the C2 pass
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/frv4_pytest.log; cat gpurun_out/frv4_pytest.log
timeout 300 python profiles/fused_rounds_bench.py > gpurun_out/frv4_bench.json 2>&1; tail -1 gpurun_out/frv4_bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rounds_fused -c 1 -o gpurun_out/frv4_full python profiles/fused_rounds_bench.py > gpurun_out/frv4_ncu.log 2>&1
ncu -i gpurun_out/frv4_full.ncu-rep --page details --csv > gpurun_out/frv4_details.csv 2>&1
ncu -i gpurun_out/frv4_full.ncu-rep --page raw --csv > gpurun_out/frv4_raw.csv 2>&1
rm -f gpurun_out/frv4_full.ncu-rep
