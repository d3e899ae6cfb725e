#!/bin/bash
# partial-sum cross round with the voided-row pulls fused into phase 0:
# emulated tests, real 4-process and world-8 (4 x 2 hosted) checks, sweeps on 2 and 4 GPUs
python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/p3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p3_pytest.log
CROSS=partial timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mgpu/shard_check.py > gpurun_out/p3_check_g4.log 2>&1
CROSS=partial SLABS=4 RANKS_PER_PROC=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tests/mgpu/shard_check.py > gpurun_out/p3_check_w8.log 2>&1
SWEEP="partial:1:0:0,partial:2:0:0,partial:4:0:0,partial:8:0:0,partial:4:148:148" CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 profiles/partial_sweep.py > gpurun_out/p3_sweep_g2.txt 2> gpurun_out/p3_sweep_g2.err
SWEEP="partial:1:0:0,partial:2:0:0,partial:4:0:0,partial:8:0:0,partial:4:148:148,exact:8:0:0" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 profiles/partial_sweep.py > gpurun_out/p3_sweep_g4.txt 2> gpurun_out/p3_sweep_g4.err
tail -2 gpurun_out/p3_pytest.log; tail -1 gpurun_out/p3_check_g4.log; tail -1 gpurun_out/p3_check_w8.log; cat gpurun_out/p3_sweep_g2.txt gpurun_out/p3_sweep_g4.txt
