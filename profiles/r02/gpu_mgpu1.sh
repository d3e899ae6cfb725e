set -x
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
G=$(nvidia-smi -L | wc -l)
python -m pytest tests/test_gpu_shard.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_shard.log
cat gpurun_out/pytest_shard.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in "1 1" "1 2" "2 1" "2 2"; do set -- $cfg
  RANKS_PER_PROC=$1 SLABS=$2 timeout 600 $TR --nproc-per-node $G --master-port 29511 tests/mgpu/shard_check.py > gpurun_out/shard_check_g${G}_r$1_s$2.log 2>&1
  tail -8 gpurun_out/shard_check_g${G}_r$1_s$2.log
done
for n in 2 $G; do for sl in 1 2; do
  MOSHPIT_SHARD_SLABS=$sl timeout 900 $TR --nproc-per-node $n --master-port 29512 bench.py --gpus $n --steps 20 --warmup 4 --no-coord --no-peer > gpurun_out/bench_g${n}_s${sl}.json 2> gpurun_out/bench_g${n}_s${sl}.err
  tail -c 1500 gpurun_out/bench_g${n}_s${sl}.json
done; done
