"""C4 SGD step with the two-round pass (default) vs kernel 3 + kernel 2
(MOSHPIT_SGD_TWO_ROUND=0), sigma 0 and 1; one JSON line each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402

for flag in ("1", "0"):
    os.environ["MOSHPIT_SGD_TWO_ROUND"] = flag
    for sigma in (0.0, 1.0):
        r = bench.measure_sgd_c4(mb, steps=20, sigma=sigma)
        print(json.dumps({"two_round": flag == "1", "sigma": sigma,
                          "ms_per_sgd_step": r["ms_per_sgd_step"], "hbm_frac_two_round_bytes":
                          r["hbm_frac"], "sigma_hat": r["final_sigma_hat"]}), flush=True)
