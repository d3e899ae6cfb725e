#!/bin/bash
# exact-sum column means + warp-per-column fallback trees: GPU suite, record timing, launch list, N=1 bench
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/cs2_pytest.log; cat gpurun_out/cs2_pytest.log
python profiles/diag_probe.py 2>&1 | tail -n1 > gpurun_out/cs2_on.txt; cat gpurun_out/cs2_on.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"cs_|dist_rows|fold|drift" --log-file gpurun_out/cs2_launches.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/cs2_bench_n1.json 2> gpurun_out/cs2_bench_n1.err
python -c "import json; d=json.loads(open('gpurun_out/cs2_bench_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['value_with_diag']['value'], d['value_with_diag']['ms_per_step'], d['clocks'])"
