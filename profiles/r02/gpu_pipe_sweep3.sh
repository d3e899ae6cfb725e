G=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $G --master-port 29513"
timeout 600 python -m pytest tests/test_gpu_shard.py -x -q -k slab 2>&1 | tail -1
for cfg in "8 104 44" "12 104 44" "16 104 44" "16 112 36"; do set -- $cfg
  MOSHPIT_SHARD_SLABS=$1 MOSHPIT_PIPE_LOCAL_SMS=$2 MOSHPIT_PIPE_CROSS_SMS=$3 timeout 600 $TR bench.py --gpus $G --steps 20 --warmup 4 --no-coord --no-peer --no-e2e > gpurun_out/pipe3_g${G}_s$1_l$2_c$3.json 2> gpurun_out/pipe3_g${G}_s$1_l$2_c$3.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/pipe3_g${G}_s$1_l$2_c$3.json') if l.startswith('{')][-1])
r=d['roofline']
print('G=$G slabs=$1 local=$2 cross=$3', d['value'], d['ms_per_step'], 'comb_ov', r['combined_frac_overlapped_bound'])" || tail -3 gpurun_out/pipe3_g${G}_s$1_l$2_c$3.err
done
