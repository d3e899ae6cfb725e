"""Temporal blocking (Engine.rounds_fused, fused_rounds.cu) against the
per-round path on C2 (1024 peers on 32^2, D = 4 Mi fp32, p = 0.01, 10
rounds) and C1 (256 peers, D = 1 Mi, 2 rounds): CUDA events around the
enqueued rounds (host draws + kernel 1 + the data kernels), best of 3."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402

out = {}
for name, (M, d, n, D, p, R) in {"C2": (32, 2, 1024, 1 << 22, 0.01, 10),
                                 "C1": (16, 2, 256, 1 << 20, 0.0, 2)}.items():
    x = torch.empty((n, D), dtype=torch.float32, device="cuda")
    res = {}
    for mode in ("per_round", "fused"):
        best = None
        for _ in range(3):
            mb.fill_synthetic(x, 0x5EED)
            e = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
            torch.cuda.synchronize()
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if mode == "fused":
                e.rounds_fused(x, R)
            else:
                for _ in range(R):
                    e.round(x)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
            e.close()
        res[mode] = {"ms_total": round(best, 3), "ms_per_round": round(best / R, 4),
                     "peer_vector_gbs_per_round": round(n * D * 4 * R / (best / 1e3) / 1e9, 1)}
    res["hbm_bytes_fused_pass"] = 2 * n * D * 4
    res["speedup"] = round(res["per_round"]["ms_total"] / res["fused"]["ms_total"], 2)
    out[name] = res
    del x
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
