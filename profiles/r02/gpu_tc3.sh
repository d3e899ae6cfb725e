set -x
timeout 600 python -m pytest tests/test_gpu_logistic.py -x -q 2>&1 | tail -3
MOSHPIT_LOGIT_TC=1 timeout 900 python profiles/logistic_tc_bench.py 1024 1024 4096 10 > gpurun_out/logit_tc.json 2>&1; cat gpurun_out/logit_tc.json
MOSHPIT_LOGIT_TC=1 python profiles/logistic_tc_bench.py 1024 1024 4096 2 > gpurun_out/tc_plain.log 2>&1 && \
MOSHPIT_LOGIT_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tc_gemm" -c 4 --csv --log-file gpurun_out/tc_launches3.csv python profiles/logistic_tc_bench.py 1024 1024 4096 2 > gpurun_out/tc_ncu3.log 2>&1
