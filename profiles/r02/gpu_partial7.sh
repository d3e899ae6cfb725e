#!/bin/bash
# SM split of the slab pipeline for the partial-sum cross round (C2, 4 and 2 GPUs)
SWEEP="partial:8:74:74,partial:8:89:59,partial:8:118:30,partial:8:148:148,partial:4:74:74,partial:4:89:59" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 profiles/partial_sweep.py > gpurun_out/p7_sweep_g4.txt 2> gpurun_out/p7_sweep_g4.err
SWEEP="partial:8:74:74,partial:8:89:59,partial:8:118:30,partial:4:89:59" CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 profiles/partial_sweep.py > gpurun_out/p7_sweep_g2.txt 2> gpurun_out/p7_sweep_g2.err
cat gpurun_out/p7_sweep_g4.txt gpurun_out/p7_sweep_g2.txt
