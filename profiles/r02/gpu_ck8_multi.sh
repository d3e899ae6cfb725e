#!/bin/bash
# full bench lines at N = 4 and N = 2 with the partial-sum headline (exact attached)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/ck8_bench_g4.json 2> gpurun_out/ck8_bench_g4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/ck8_bench_g2.json 2> gpurun_out/ck8_bench_g2.err
tail -c 600 gpurun_out/ck8_bench_g4.json; tail -c 600 gpurun_out/ck8_bench_g2.json
