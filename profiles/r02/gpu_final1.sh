set -x
G=$(nvidia-smi -L | wc -l)
python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_gpu_all.log; cat gpurun_out/pytest_gpu_all.log
for i in 1 2 3; do python profiles/cold_start.py; done > gpurun_out/cold_start.jsonl 2>&1; cat gpurun_out/cold_start.jsonl
CUDA_VISIBLE_DEVICES=0 timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 300 gpurun_out/bench_n1.err
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29514"
for n in 2 4; do
  timeout 1500 $TR --nproc-per-node $n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; tail -c 1200 gpurun_out/bench_n$n.json
done
