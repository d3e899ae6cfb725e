"""Table-3 Moshpit rows (Table 3 / harness run_experiment): N in
{512,768,900,1024} on 32x32, p in {0,0.001,0.005,0.01}, 100 seeds, dim 1,
round cap 50, thresholds 1e-9 / 1e-4.  GPU: one trial-batched run_moshpit
call per cell.  CPU: the unmodified reference harness run_trial on all host
threads.  Reports must be identical; prints one JSON line."""
import concurrent.futures as cf
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from oracle.oracle import RefHarness  # noqa: E402

NS, PS, SEEDS, CAP = [512, 768, 900, 1024], [0.0, 0.001, 0.005, 0.01], 100, 50


def initial(seed, n):
    s = mb.Rng(seed).stream("init")
    return s._draw(1, n, dt=np.float64).reshape(n, 1)


def main():
    grid = mb.GridConfig(32, 2, 1)
    cells = [(n, p) for n in NS for p in PS]
    # inputs (host RNG, the harness's "init" stream) -- not timed
    data = {}
    for n, p in cells:
        seeds = [mb.trial_seed(0, "moshpit", n, p, k) for k in range(SEEDS)]
        data[(n, p)] = (seeds, np.stack([initial(s, n) for s in seeds]))
    mb.run_moshpit_batch(grid, data[(512, 0.0)][1][:2], mb.FailureModel(0.0),
                         data[(512, 0.0)][0][:2], CAP)  # warm-up
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=len(cells)) as ex:  # cells overlap on the GPU
        res = list(ex.map(lambda c: mb.run_moshpit_batch(grid, data[c][1], mb.FailureModel(c[1]),
                                                         data[c][0], CAP), cells))
    gpu = dict(zip(cells, res))
    t_gpu = time.perf_counter() - t0
    rows = []
    for n, p in cells:
        r9 = [r.rounds_to(1e-9, CAP) for r in gpu[(n, p)]]
        r4 = [r.rounds_to(1e-4, CAP) for r in gpu[(n, p)]]
        rows.append(dict(N=n, p=p, rounds_1e9=round(float(np.mean(r9)), 2),
                         std_1e9=round(float(np.std(r9)), 2), rounds_1e4=round(float(np.mean(r4)), 2),
                         std_1e4=round(float(np.std(r4)), 2)))
    out = {"workload": "Table-3 Moshpit rows: 16 cells x 100 seeds, dim 1, 32x32, cap 50",
           "gpu_seconds": round(t_gpu, 3), "trials": len(cells) * SEEDS, "rows": rows}
    try:
        h = RefHarness()
        jobs = [(n, p, k) for n, p in cells for k in range(SEEDS)]
        threads = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(max_workers=threads) as ex:
            ref = list(ex.map(lambda j: h.run_trial(0, j[0], j[1], j[2], 32, 2, 1, "uniform", CAP),
                              jobs))
        t_cpu = time.perf_counter() - t0
        same = True
        for (n, p, k), want in zip(jobs, ref):
            got = gpu[(n, p)][k]
            same &= np.array_equal(np.array(got.distortion), want["distortion"])
        out.update(cpu_reference_seconds=round(t_cpu, 3), cpu_threads=threads,
                   reports_identical=bool(same), speedup=round(t_cpu / t_gpu, 1))
    except FileNotFoundError as exc:
        out["cpu_reference"] = f"unavailable: {exc}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
