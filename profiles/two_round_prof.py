"""C4 SGD (3 steps) for ncu: the two-round pass and the rest of a step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402
import numpy as np  # noqa: E402

sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
D, N = 1 << 20, 1024
tgt = mb.Rng(bench.PROTOCOL_SEED).stream("objective").normals(D)
quad = mb.Quadratic(D, 1.0, 0.1, tgt)
cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=3, grid=mb.GridConfig(32, 2, 1), sigma=sigma,
                         n_peers=N)
r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(bench.PROTOCOL_SEED), dtype=np.float32,
                       diagnostics="none", noise="device")
print("loop ms", r.loop_ms)
