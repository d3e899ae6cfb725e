"""Trial-batched run_moshpit timing probe (one Table-3 cell: 100 trials of
1024 peers on 32x32, dim 1, p=0.01, 50 rounds): per-call wall time with
EXACT diagnostics and without."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2103_03239_b200 as mb
n, T, R = 1024, 100, 50
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
seeds = [mb.trial_seed(0, "moshpit", n, 0.01, k) for k in range(T)]
x = np.stack([mb.Rng(s).stream("init")._draw(1, n, dt=np.float64).reshape(n, 1) for s in seeds])
g = mb.GridConfig(32, 2, 1)
for diag in ("exact", "none"):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        mb.run_moshpit_batch(g, x, mb.FailureModel(0.01), seeds, R, diagnostics=diag)
        ts.append(time.perf_counter() - t)
    print(diag, "seconds per call", [round(v, 4) for v in ts])

# 16 concurrent callers (the Table-3 sweep shape): wall time of the burst
import concurrent.futures as cf
if len(sys.argv) > 2:
    k = int(sys.argv[2])
    with cf.ThreadPoolExecutor(max_workers=k) as ex:
        list(ex.map(lambda _: mb.run_moshpit_batch(g, x, mb.FailureModel(0.01), seeds, R), range(k)))
        for _ in range(2):
            t = time.perf_counter()
            list(ex.map(lambda _: mb.run_moshpit_batch(g, x, mb.FailureModel(0.01), seeds, R), range(k)))
            print(k, "concurrent calls: seconds", round(time.perf_counter() - t, 4))
