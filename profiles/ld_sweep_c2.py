"""Kernel 2 vs row pitch on C2 (1024 peers on 32^2, D = 4 Mi fp32, p = 0.01):
pitch D (power of two) against D + pad; kernel-2 fraction of the measured HBM
copy peak and the round time (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402

M, d, N, D, p = 32, 2, 1024, 1 << 22, 0.01
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6544.0
for pad in (0, 32, 256, 1024, 4096):
    ld = D + pad
    x = torch.empty((N, ld), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, 0x5EED, dim=D)
    eng = mb.Engine(mb.GridConfig(M, d, 30), N, mb.FailureModel(p), mb.Rng(7), device=0)
    for _ in range(3):
        eng.round(x, dim=D)
    torch.cuda.synchronize()
    eng.set_timing(True)
    r0 = eng.stats()[1]
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        eng.round(x, dim=D)
    e1.record(s)
    torch.cuda.synchronize()
    ms, k = eng.kernel_time()
    rows = eng.stats()[1] - r0
    print(json.dumps({"ld": ld, "pad_floats": pad, "ms_per_round": round(e0.elapsed_time(e1) / 20, 4),
                      "k2_frac": round(2 * 4 * D * rows / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
    eng.close()
    del x
    torch.cuda.empty_cache()
