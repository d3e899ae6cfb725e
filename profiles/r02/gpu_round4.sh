set -x
# per-kernel times of the diagnostics (launch list), then the pipeline sweep on N GPUs
python profiles/diag_probe.py ncu > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/diag_launches_r4.csv python profiles/diag_probe.py ncu > gpurun_out/diag_ncu_r4.log 2>&1
G=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $G --master-port 29513"
for cfg in "4 104 44" "4 112 36" "4 96 52" "8 104 44" "4 88 60" "2 104 44" "1 0 0"; do set -- $cfg
  MOSHPIT_SHARD_SLABS=$1 MOSHPIT_PIPE_LOCAL_SMS=$2 MOSHPIT_PIPE_CROSS_SMS=$3 timeout 600 $TR bench.py --gpus $G --steps 20 --warmup 4 --no-coord --no-peer > gpurun_out/pipe_g${G}_s$1_l$2_c$3.json 2> gpurun_out/pipe_g${G}_s$1_l$2_c$3.err
  python -c "
import json
d=json.loads(open('gpurun_out/pipe_g${G}_s$1_l$2_c$3.json').read().strip().splitlines()[-1])
r=d['roofline']
print('G=$G slabs=$1 local=$2 cross=$3', d['value'], d['ms_per_step'], 'local', r['local']['achieved'], 'nvl', r['cross']['achieved_nvlink'], 'A', r['cross']['phase_a_ms'], 'B', r['cross']['phase_b_ms'], 'comb', r['combined_frac'])" || tail -3 gpurun_out/pipe_g${G}_s$1_l$2_c$3.err
done
