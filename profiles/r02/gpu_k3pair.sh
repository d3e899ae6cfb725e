timeout 900 python -m pytest tests/test_gpu_noise.py tests/test_gpu_sgd.py tests/test_gpu_logistic.py -x -q 2>&1 | tail -5
for i in 1 2; do timeout 600 python profiles/k3_rounds.py; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"group_mean_step|group_mean_reg" -c 4 --csv --log-file gpurun_out/k3_pair_ncu.csv python profiles/k3_rounds.py > /dev/null 2>&1
grep -h "step_leaf" gpurun_out/k3_pair_ncu.csv | awk -F'","' '{print $(NF-2), $NF}'
