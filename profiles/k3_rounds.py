"""C4 (Moshpit SGD, device noise) step time of the library in the current
directory: sigma = 1 and 0, best of 2 x 20 steps (bench.measure_sgd_c4)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402

out = {"lib": mb._capi.LIB_PATH, "extra": os.environ.get("MOSHPIT_NVCC_EXTRA", "")}
for sigma in (1.0, 0.0):
    r = bench.measure_sgd_c4(mb, sigma=sigma)
    out[f"sigma{int(sigma)}"] = {k: r[k] for k in ("ms_per_sgd_step", "hbm_frac", "final_sigma_hat")}
print(json.dumps(out), flush=True)
