set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "concurrent" 2>&1 | tail -1; done
timeout 600 python profiles/diag_probe.py > gpurun_out/diag_time_unrolled.json 2>&1; cat gpurun_out/diag_time_unrolled.json
python profiles/diag_probe.py ncu > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"colmean|dist_rows" --csv --log-file gpurun_out/cm_launches2.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
