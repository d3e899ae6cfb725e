timeout 1200 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_noise.py tests/test_gpu_logistic.py tests/test_gpu_batch.py -x -q 2>&1 | tail -3
for m in 1 2; do echo "== MOSHPIT_SGD_FUSED_HAT=$m"; MOSHPIT_SGD_FUSED_HAT=$m timeout 600 python profiles/r02/c4_diag.py; done
MOSHPIT_SGD_FUSED_HAT=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16 --csv --log-file gpurun_out/c4diag_vec.csv python profiles/r02/c4_diag.py > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time_duration" gpurun_out/c4diag_vec.csv | awk -F'","' '{print $NF, substr($5,1,50)}'
