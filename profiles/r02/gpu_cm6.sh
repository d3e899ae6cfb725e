timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "column_means or record or run_moshpit or streamed or report" 2>&1 | tail -2
timeout 600 python profiles/diag_probe.py 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum -k regex:"colmean|dist_rows" --clock-control none --csv --log-file gpurun_out/cm6.csv python profiles/diag_probe.py ncu > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time\|lts__t\|inst_issued" gpurun_out/cm6.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-50,90-200
