G=$(nvidia-smi -L | wc -l); echo "GPUs: $G"
timeout 1200 python -m pytest tests/test_dist_host.py tests/test_gpu_shard.py -m gpu -x -q 2>&1 | tail -2
RANKS_PER_PROC=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tests/mgpu/shard_check.py > gpurun_out/mgpu/world8_hosted.log 2>&1; tail -2 gpurun_out/mgpu/world8_hosted.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  timeout 1500 $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/bench_n$n.json') if l.startswith('{')][-1])
print($n, d['value'], d['ms_per_step'], d['roofline']['combined_frac_overlapped_bound'], 'e2e', (d.get('e2e') or {}).get('value'), 'c5v', (d.get('peer_sharded_c5v') or {}).get('value'), 'coord', (d.get('coordinate_sharded_weak') or {}).get('value'))
PY
done
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29516 --nproc-per-node 4 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_ref_n4.json 2>&1; tail -c 200 gpurun_out/bench_ref_n4.json
