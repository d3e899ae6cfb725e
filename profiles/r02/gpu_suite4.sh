#!/bin/bash
# the whole GPU suite on a 4-GPU box (the real multi-process shard tests run here)
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/suite4_pytest_gpu_all.log; cat gpurun_out/suite4_pytest_gpu_all.log
