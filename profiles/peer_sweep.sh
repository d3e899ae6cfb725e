for c in 3 2 1; do
MOSHPIT_CROSS_CTAS=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$c bench.py --gpus 2 --mode peer --config C2 --steps 40 --warmup 4 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ctas=$c', d['ms_per_step'], r['local']['frac'], json.dumps(r['cross']), r['combined_frac'])"
done
