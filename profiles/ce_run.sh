python -m pytest tests/test_gpu_shard.py -m gpu -x -q 2>&1 | tail -2
python tests/mgpu/shard_check.py --help 2>&1 | head -3
for ce in 1 0; do
MOSHPIT_CROSS_CE=$ce python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$ce bench.py --gpus 2 --mode peer --config C5v --steps 20 --warmup 4 2>gpurun_out/ce$ce.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ce=$ce', d['value'], d['ms_per_step'], r['local']['frac'], json.dumps(r['cross'])[:300], r['combined_frac'])"
done
