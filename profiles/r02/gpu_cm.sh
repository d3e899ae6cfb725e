set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for m in 1 0; do MOSHPIT_COLMEAN_TILES=$m timeout 600 python profiles/diag_probe.py > gpurun_out/diag_time_cm$m.json 2>&1; cat gpurun_out/diag_time_cm$m.json; done
python profiles/diag_probe.py ncu > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"colmean|dist_rows" --csv --log-file gpurun_out/cm_launches.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
