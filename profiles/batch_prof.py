import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2103_03239_b200 as mb
n, T, R = 1024, 100, 50
seeds = [mb.trial_seed(0, "moshpit", n, 0.01, k) for k in range(T)]
x = np.stack([mb.Rng(s).stream("init")._draw(1, n, dt=np.float64).reshape(n, 1) for s in seeds])
import time
t = time.perf_counter()
mb.run_moshpit_batch(mb.GridConfig(32, 2, 1), x, mb.FailureModel(0.01), seeds, R)
print("seconds", time.perf_counter() - t)
