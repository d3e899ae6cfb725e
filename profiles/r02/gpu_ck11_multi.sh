#!/bin/bash
# checkpoint 11 (library with the 3-team temporal blocking): N = 1, 2, 4 bench lines on one 4-GPU box
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ck11_bench_n1.json 2> gpurun_out/ck11_bench_n1.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/ck11_bench_g4.json 2> gpurun_out/ck11_bench_g4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/ck11_bench_g2.json 2> gpurun_out/ck11_bench_g2.err
for f in n1 g2 g4; do python -c "import json,sys; d=json.loads(open('gpurun_out/ck11_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['unit'], d.get('rounds_fused_mode',{}).get('fused',d.get('rounds_fused_mode')) if '$f'=='n1' else '', d.get('clocks'))"; done
