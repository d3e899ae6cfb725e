"""LogisticRegression Moshpit-SGD step loop only (none diagnostics, device
noise) for launch lists / ncu: python profiles/logistic_prof.py [N dim S steps]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2103_03239_b200 as mb  # noqa: E402
n, dim, S, steps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5 else (1024, 1024, 4096, 4)))
M = int(round(n ** 0.5))
lr = mb.LogisticRegression.synthetic(dim, S, 0.01, mb.Rng(17).stream("objective"))
cfg = mb.OptimizerConfig(gamma=0.5, tau=1, steps=steps, grid=mb.GridConfig(M, 2, 1), sigma=0.5, n_peers=n)
r = mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(17), diagnostics="none", noise="device")
print("ms per step", r.loop_ms / steps)
