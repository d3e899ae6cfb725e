"""C4 with FAST per-step diagnostics (optimizer.hpp:376, 383-420): ms per SGD
step, sigma = 1 and 0 (bench.measure_sgd_c4)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402

out = {}
for sigma in (1.0, 0.0):
    r = bench.measure_sgd_c4(mb, sigma=sigma, diagnostics="fast")
    out[f"sigma{int(sigma)}_fast"] = {k: r[k] for k in ("ms_per_sgd_step", "hbm_frac", "final_sigma_hat")}
print(json.dumps(out), flush=True)
