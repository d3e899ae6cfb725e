#!/bin/bash
# two-round SGD pass: parity tests, C4 timing, launch list
python -m pytest tests/test_gpu_sgd.py tests/test_gpu_fused_rounds.py tests/test_gpu_noise.py -x -q > gpurun_out/two1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/two1_pytest.log
timeout 600 python profiles/two_round_bench.py > gpurun_out/two1_bench.txt 2>&1
tail -3 gpurun_out/two1_pytest.log; cat gpurun_out/two1_bench.txt
