set -x
timeout 600 python -m pytest tests/test_gpu_logistic.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_logistic.log; cat gpurun_out/pytest_logistic.log
for i in 1 2 3; do python profiles/cold_start.py; done > gpurun_out/cold_start.jsonl 2>&1; cat gpurun_out/cold_start.jsonl
MOSHPIT_LOGIT_TC=1 timeout 900 python profiles/logistic_tc_bench.py 1024 1024 4096 10 > gpurun_out/logit_tc.json 2>&1; cat gpurun_out/logit_tc.json
