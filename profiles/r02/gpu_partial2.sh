#!/bin/bash
# slab / SM-cap sweep of the partial-sum cross round, C2 on 2 GPUs
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 profiles/partial_sweep.py > gpurun_out/partial_sweep_g2.txt 2> gpurun_out/partial_sweep_g2.err
cat gpurun_out/partial_sweep_g2.txt
