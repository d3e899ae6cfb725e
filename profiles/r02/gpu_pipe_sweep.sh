# slab-pipeline sweep on N GPUs (C2 peer-sharded): slabs x local/cross SM caps
G=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $G --master-port 29513"
for cfg in "1 0 0" "2 0 0" "2 104 44" "2 96 52" "2 120 28" "4 0 0" "4 104 44" "2 74 74"; do set -- $cfg
  MOSHPIT_SHARD_SLABS=$1 MOSHPIT_PIPE_LOCAL_SMS=$2 MOSHPIT_PIPE_CROSS_SMS=$3 timeout 600 $TR bench.py --gpus $G --steps 20 --warmup 4 --no-coord --no-peer > gpurun_out/pipe_g${G}_s$1_l$2_c$3.json 2> gpurun_out/pipe_g${G}_s$1_l$2_c$3.err
  python -c "
import json
d=json.loads(open('gpurun_out/pipe_g${G}_s$1_l$2_c$3.json').read().strip().splitlines()[-1])
r=d['roofline']
print('G=$G slabs=$1 local=$2 cross=$3', d['value'], d['ms_per_step'], 'local', r['local']['achieved'], 'nvl', r['cross']['achieved_nvlink'], 'A', r['cross']['phase_a_ms'], 'B', r['cross']['phase_b_ms'])" || tail -3 gpurun_out/pipe_g${G}_s$1_l$2_c$3.err
done
