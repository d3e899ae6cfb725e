"""Moshpit SGD on LogisticRegression: GPU step-loop time
(loop_ms, CUDA events) vs the unmodified reference on one host core
(oracle/_ref, ref_sgd_logistic), same config, fp64.  Test-side script: the
reference arm is the checker, timed here only as a baseline.

Usage: python profiles/logistic_bench.py [N dim samples steps]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2103_03239_b200 as mb  # noqa: E402


def main():
    n, dim, S, steps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5
                                          else (256, 256, 1024, 20)))
    M = int(round(n ** 0.5))
    l2, gamma, sigma, seed = 0.01, 0.5, 0.5, 17
    lr = mb.LogisticRegression.synthetic(dim, S, l2, mb.Rng(seed).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=gamma, tau=1, steps=steps, grid=mb.GridConfig(M, 2, 1),
                             sigma=sigma, n_peers=n)
    out = {"config": dict(n_peers=n, dim=dim, samples=S, steps=steps, grid=[M, 2])}
    for diag in ("exact", "fast", "none"):
        for noise in ("reference", "device"):
            mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(seed), diagnostics=diag,
                               noise=noise)  # warm-up
            r = mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(seed), diagnostics=diag,
                                   noise=noise)
            out[f"gpu_{diag}_{noise}_ms_per_step"] = r.loop_ms / steps
            if diag == "exact" and noise == "reference":
                gpu_fgap = r.f_gap
    try:
        from oracle.oracle import Checker
        ref = Checker("ref")
        t0 = time.perf_counter()
        want = ref.sgd_logistic(M, 2, n, dim, S, l2, seed, np.zeros(dim), gamma, 1, steps,
                                sigma, seed)
        out["ref_cpu_1core_ms_per_step"] = (time.perf_counter() - t0) * 1e3 / steps
        out["max_rel_f_gap_err"] = float(np.max(np.abs(np.array(gpu_fgap) - want["f_gap"]) /
                                                np.abs(want["f_gap"])))
    except Exception as e:  # noqa: BLE001
        out["ref"] = f"unavailable: {e}"
    # algorithmic flops per step: margins + gradient, 2 flops per (peer, sample, j) each
    out["gflop_per_step"] = 4.0 * n * S * dim / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
