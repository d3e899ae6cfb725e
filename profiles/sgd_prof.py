"""C4 Moshpit-SGD step timing probe (1024 peers, 32x32, Quadratic D=2^20,
tau=1, inner=2, fp32, device noise, no diagnostics).

    python profiles/sgd_prof.py [sigma] [steps]

Kernel-3 variant via env: MOSHPIT_STEP_KERNEL=old (register/split forms),
MOSHPIT_STEP_MODE=0|1|2 (leaf-streamed form load batches)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, paper_2103_03239_b200 as mb
D, N = 1 << 20, 1024
sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
tgt = mb.Rng(7).stream("objective").normals(D)
quad = mb.Quadratic(D, 1.0, 0.1, tgt)
cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=steps, grid=mb.GridConfig(32, 2, 1), sigma=sigma, n_peers=N)
best = None
for _ in range(2 if steps > 6 else 1):
    r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(7), dtype=np.float32, diagnostics="none", noise="device")
    best = r.loop_ms if best is None else min(best, r.loop_ms)
tag = os.environ.get("MOSHPIT_STEP_KERNEL", "leaf") + "/mode" + os.environ.get("MOSHPIT_STEP_MODE", "auto")
print(f"sigma={sigma} {tag} loop_ms {best:.3f} per step {best / steps:.4f} ms "
      f"hbm_frac {2*2*N*D*4/(best/steps/1e3)/1e9/6552.6:.3f} sigma_hat {r.diagnostics.sigma_hat:.6f}")
