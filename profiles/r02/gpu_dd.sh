timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sgd.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2
timeout 600 python profiles/diag_probe.py 2>&1 | tail -1
timeout 600 python profiles/r02/c4_diag.py
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__inst_issued.avg.pct_of_peak_sustained_active -k regex:"colmean|dist_rows" --clock-control none --csv --log-file gpurun_out/dd.csv python profiles/diag_probe.py ncu > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time\|lts__t\|dram__bytes" gpurun_out/dd.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-40,90-200 | head -24
