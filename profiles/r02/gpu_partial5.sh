#!/bin/bash
# after: ILP-2 combine / pull, voided-row writes fused into the pull launch
python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/p5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p5_pytest.log
for c in partial exact; do
CROSS=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/mgpu/shard_check.py > gpurun_out/p5_check_g4_$c.log 2>&1
CROSS=$c SLABS=4 RANKS_PER_PROC=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tests/mgpu/shard_check.py > gpurun_out/p5_check_w8_$c.log 2>&1
done
SWEEP="partial:1:0:0,partial:4:0:0,partial:8:0:0,exact:8:0:0" CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 profiles/partial_sweep.py > gpurun_out/p5_sweep_g2.txt 2> gpurun_out/p5_sweep_g2.err
SWEEP="partial:1:0:0,partial:4:0:0,partial:8:0:0,exact:8:0:0" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 profiles/partial_sweep.py > gpurun_out/p5_sweep_g4.txt 2> gpurun_out/p5_sweep_g4.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum --clock-control none --csv -k regex:"partial|shard_pull|move_rows|group_mean|cross_mean" --log-file gpurun_out/p5_ncu_g4_partial.csv python profiles/partial_probe.py 4 partial > gpurun_out/p5_ncu.log 2>&1
tail -2 gpurun_out/p5_pytest.log; tail -n1 gpurun_out/p5_check_*.log; cat gpurun_out/p5_sweep_g2.txt gpurun_out/p5_sweep_g4.txt
