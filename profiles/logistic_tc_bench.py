"""Logistic Moshpit SGD step, fp32 state: tensor cores (tcgen05 kind::tf32,
3xTF32; tc_logit.cu) vs the fp64 SIMT kernels on the same fp32 state, and the
fp64 state; device noise, no per-step diagnostics (loop_ms: CUDA events).

    python profiles/logistic_tc_bench.py [N dim samples steps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_2103_03239_b200 as mb  # noqa: E402

n, dim, S, steps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5
                                      else (1024, 1024, 4096, 10)))
M = int(round(n ** 0.5))
lr = mb.LogisticRegression.synthetic(dim, S, 0.01, mb.Rng(17).stream("objective"))
cfg = mb.OptimizerConfig(gamma=0.5, tau=1, steps=steps, grid=mb.GridConfig(M, 2, 1), sigma=0.5,
                         n_peers=n)
out = {"config": dict(n_peers=n, dim=dim, samples=S, steps=steps),
       "gflop_per_step": 4.0 * n * S * dim / 1e9}
for name, dt, tc in (("f32_tensor_cores", np.float32, "1"), ("f32_simt_fp64_math", np.float32, "0"),
                     ("f64_simt", np.float64, "0")):
    os.environ["MOSHPIT_LOGIT_TC"] = tc
    best = None
    for _ in range(2):
        r = mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(17), dtype=dt,
                               diagnostics="none", noise="device")
        best = r.loop_ms if best is None else min(best, r.loop_ms)
    out[name] = {"ms_per_step": round(best / steps, 4),
                 # GFLOP per ms = TFLOP/s (logical flops; 3xTF32 issues 3x on the tensor cores)
                 "tflops_incl_averaging": round(out["gflop_per_step"] / (best / steps), 2),
                 "final_mean_0": float(r.final_mean[0])}
print(json.dumps(out), flush=True)
