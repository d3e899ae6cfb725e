import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, paper_2103_03239_b200 as mb
D, N = 1 << 20, 1024
sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
tgt = mb.Rng(7).stream("objective").normals(D)
quad = mb.Quadratic(D, 1.0, 0.1, tgt)
cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=6, grid=mb.GridConfig(32, 2, 1), sigma=sigma, n_peers=N)
r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(7), dtype=np.float32, diagnostics="none", noise="device")
print("loop_ms", r.loop_ms, "per step", r.loop_ms / 6)
