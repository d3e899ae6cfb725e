timeout 900 python -m pytest tests/test_gpu_shard.py -x -q 2>&1 | tail -2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 2 --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 5 --no-coord --no-peer > gpurun_out/bench_n2_e2e.json 2> gpurun_out/bench_n2_e2e.err
python - <<'PY'
import json
line=[l for l in open('gpurun_out/bench_n2_e2e.json') if l.startswith('{')][-1]
d=json.loads(line); print(d['value'], json.dumps(d['e2e']))
PY
grep -i -m3 "error\|Traceback" gpurun_out/bench_n2_e2e.err
