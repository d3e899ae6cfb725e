#!/bin/bash
python -m pytest tests/test_gpu_sgd.py tests/test_gpu_fused_rounds.py -x -q > gpurun_out/two6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/two6_pytest.log
timeout 600 python profiles/two_round_bench.py > gpurun_out/two6_bench.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:two_round_step --log-file gpurun_out/two6_ncu.csv python profiles/two_round_prof.py 1.0 > /dev/null 2>&1
tail -2 gpurun_out/two6_pytest.log; cat gpurun_out/two6_bench.txt
