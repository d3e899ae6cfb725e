#!/bin/bash
# checkpoint 10 (rounds_record library): GPU suite, smoke, cold start x3, N=1 bench, reference arm
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ck10_pytest_gpu_all.log; cat gpurun_out/ck10_pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2 3; do python profiles/cold_start.py >> gpurun_out/ck10_cold_start.jsonl 2>/dev/null; done
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ck10_bench_n1.json 2> gpurun_out/ck10_bench_n1.err; tail -c 300 gpurun_out/ck10_bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ck10_bench_ref_n1.json 2>&1; tail -c 200 gpurun_out/ck10_bench_ref_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ck10_launches_bench_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sgd --no-full --no-variants > /dev/null 2>&1
cat gpurun_out/ck10_cold_start.jsonl
