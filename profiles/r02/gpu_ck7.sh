#!/bin/bash
# checkpoint 7: GPU suite, smoke, N=1 bench (with the two-round C4), reference arm
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ck7_pytest_gpu_all.log; cat gpurun_out/ck7_pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ck7_bench_n1.json 2> gpurun_out/ck7_bench_n1.err; tail -c 300 gpurun_out/ck7_bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ck7_bench_ref_n1.json 2>&1; tail -c 400 gpurun_out/ck7_bench_ref_n1.json
