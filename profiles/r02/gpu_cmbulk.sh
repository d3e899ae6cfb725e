MOSHPIT_CM_BULK=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sgd.py -x -q -k "column_means or f32_bit_exact or record or report or streamed or fused_paths" 2>&1 | tail -2
for b in 0 1; do echo "== MOSHPIT_CM_BULK=$b"; MOSHPIT_CM_BULK=$b timeout 600 python profiles/diag_probe.py 2>&1 | tail -1 | cut -c1-120; done
MOSHPIT_CM_BULK=1 timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,sm__inst_issued.avg.pct_of_peak_sustained_active -k regex:"colmean" --clock-control none --csv --log-file gpurun_out/cmbulk.csv python profiles/diag_probe.py ncu > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time\|inst_issued" gpurun_out/cmbulk.csv | awk -F'","' '{print substr($5,1,45), $(NF-2), $NF}' | head -12
