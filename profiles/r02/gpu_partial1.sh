#!/bin/bash
# partial-sum cross round: emulated tests, real 2-process checks, 2-GPU bench (both modes)
set -x
python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/partial_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/partial_pytest.log
for c in partial exact; do
  CROSS=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/mgpu/shard_check.py > gpurun_out/partial_check_g2_$c.log 2>&1
  CROSS=$c SLABS=4 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tests/mgpu/shard_check.py > gpurun_out/partial_check_g2_s4_$c.log 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 --no-coord --no-peer --no-e2e --cross partial > gpurun_out/partial_bench_g2.json 2> gpurun_out/partial_bench_g2.err
tail -3 gpurun_out/partial_pytest.log; tail -2 gpurun_out/partial_check_g2_*.log
