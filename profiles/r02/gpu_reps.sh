set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python profiles/diag_probe.py > gpurun_out/diag_time_reps.json 2>&1; cat gpurun_out/diag_time_reps.json
timeout 300 python -c "
import sys,os; sys.path.insert(0,'.'); import json, bench, torch, paper_2103_03239_b200 as mb
print(json.dumps({k: bench.measure_variant(mb, torch, 'C2', 0, 20, 3, **kw) for k, kw in (('value_with_diag', dict(diag='fast')), ('value_f64_exact_diag', dict(f64=True, diag='exact')))}))"
