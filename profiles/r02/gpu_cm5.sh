timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_sgd.py -x -q 2>&1 | tail -3
timeout 600 python profiles/diag_probe.py 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/diag_launches_r02d.csv python profiles/diag_probe.py ncu > /dev/null 2>&1; echo rc=$?
