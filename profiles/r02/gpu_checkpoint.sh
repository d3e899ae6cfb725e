set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_all.log; cat gpurun_out/pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 300 gpurun_out/bench_n1.err
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
for n in 2 4; do
  timeout 1500 $TR --nproc-per-node $n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; tail -c 300 gpurun_out/bench_n$n.json
done
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29516 --nproc-per-node 4 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_ref_n4.json 2>&1; tail -c 300 gpurun_out/bench_ref_n4.json
