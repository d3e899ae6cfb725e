set -x
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu_all.log; cat gpurun_out/pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 300 gpurun_out/bench_n1.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d['e2e'])[:400]); print(json.dumps(d['e2e_variants'])[:900])"
