set -x
G=$(nvidia-smi -L | wc -l)
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 $G; do for sl in 1 2; do
  MOSHPIT_SHARD_SLABS=$sl timeout 900 $TR --nproc-per-node $n --master-port 29512 bench.py --gpus $n --steps 20 --warmup 4 --no-coord --no-peer > gpurun_out/bench_g${n}_s${sl}.json 2> gpurun_out/bench_g${n}_s${sl}.err
  tail -c 600 gpurun_out/bench_g${n}_s${sl}.json; grep -i -m3 "error\|Traceback" gpurun_out/bench_g${n}_s${sl}.err
done; done
timeout 900 python bench.py --steps 20 --warmup 5 --no-full --no-sgd --no-cpu > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
tail -c 400 gpurun_out/bench_n1.err
