G=$(nvidia-smi -L | wc -l); echo "GPUs: $G"
timeout 1200 python -m pytest tests/test_dist_host.py -m gpu -x -q 2>&1 | tail -2
RANKS_PER_PROC=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tests/mgpu/shard_check.py > gpurun_out/mgpu/world8_hosted.log 2>&1; tail -2 gpurun_out/mgpu/world8_hosted.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  timeout 1500 $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  tail -c 300 gpurun_out/bench_n$n.json; grep -i -m3 "error\|Traceback" gpurun_out/bench_n$n.err
done
