timeout 1200 python -m pytest tests/test_gpu_sgd.py -x -q 2>&1 | tail -2
timeout 600 python profiles/r02/c4_diag.py
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgd_step_vec -c 3 --csv --log-file gpurun_out/c4diag_vec2.csv python profiles/r02/c4_diag.py > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time_duration" gpurun_out/c4diag_vec2.csv | awk -F'","' '{print $NF, substr($5,1,50)}'
