timeout 1200 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_noise.py tests/test_gpu_logistic.py -x -q 2>&1 | tail -3
timeout 600 python profiles/r02/c4_diag.py
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/c4diag_launches.csv python profiles/r02/c4_diag.py > /dev/null 2>&1; echo rc=$?
