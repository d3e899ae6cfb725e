"""e2e of run_moshpit (the reference-facing host-buffer call) at C2 in the
modes a caller can hit: fp32 FAST pinned (the bench e2e), fp32 FAST pageable,
fp64 EXACT pageable / pinned (the drop-in's mode), and the diagnostics cost
(DIAG_NONE vs FAST vs EXACT) at a resident size.  Prints one JSON line per
mode."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from paper_2103_03239_b200 import _capi  # noqa: E402

lib = _capi.lib()
M, d, N, R, P = 32, 2, 1024, 10, 0.01
D = int(os.environ.get("E2E_D", 1 << 22))


def host_state(dt, pinned):
    es = np.dtype(dt).itemsize
    if pinned:
        t = torch.empty((N, D), dtype=torch.float32 if es == 4 else torch.float64, pin_memory=True)
        x = t.numpy()
    else:
        x = np.empty((N, D), dtype=dt)
        t = None
    blk = torch.empty((64, D), dtype=torch.float32 if es == 4 else torch.float64, device="cuda")
    for i0 in range(0, N, 64):
        mb.fill_synthetic(blk, 0x5EED, col0=0)
        x[i0:i0 + 64] = blk.cpu().numpy()
    return x, t


def call(x, code, diag, out):
    dist, drift = np.zeros(R), np.zeros(R)
    act = np.zeros(R, dtype=np.uint32)
    a, b = C.c_double(0), C.c_double(0)
    t0 = time.perf_counter()
    _capi.check(lib.moshpit_run_moshpit(code, M, d, R, x.ctypes.data_as(C.c_void_p), N, x.shape[1],
                                        P, 7, R, diag, C.byref(a), dist.ctypes.data_as(C.c_void_p),
                                        drift.ctypes.data_as(C.c_void_p),
                                        act.ctypes.data_as(C.c_void_p), C.byref(b),
                                        out.ctypes.data_as(C.c_void_p) if out is not None else None))
    return time.perf_counter() - t0, dist[-1]


modes = os.environ.get("E2E_MODES", "f32_fast_pinned,f32_fast_pageable,f64_exact_pageable,"
                       "f64_exact_pinned,f64_exact_pageable_noout").split(",")
for m in modes:
    dt = np.float64 if m.startswith("f64") else np.float32
    code = _capi.F64 if dt == np.float64 else _capi.F32
    diag = _capi.DIAG_EXACT if "exact" in m else _capi.DIAG_FAST
    x, keep = host_state(dt, "pinned" in m)
    out = None if m.endswith("noout") else x
    ts = []
    for it in range(3):
        t, dl = call(x, code, diag, out)
        ts.append(round(t, 4))
    bytes_ = N * D * np.dtype(dt).itemsize
    print(json.dumps({"mode": m, "D": D, "seconds": ts, "state_gb": round(bytes_ / 1e9, 2),
                      "peer_vector_gbs_fp32_normalised": round(N * D * 4 * R / min(ts) / 1e9, 1),
                      "final_distortion": dl}), flush=True)
    del x, keep

# diagnostics cost at a resident size (dim <= slab): per round
os.environ["MOSHPIT_SLAB_BYTES"] = str(1 << 40)
Dr = 1 << 18
for dt in (np.float32, np.float64):
    x = np.random.default_rng(0).random((N, Dr)).astype(dt)
    for dg in ("none", "fast", "exact"):
        t = []
        for it in range(3):
            r0 = time.perf_counter()
            mb.run_moshpit(mb.GridConfig(M, d, 1), x, mb.FailureModel(P), mb.Rng(7), R,
                           diagnostics=dg)
            t.append(time.perf_counter() - r0)
        print(json.dumps({"mode": f"resident_{np.dtype(dt).name}_{dg}", "D": Dr,
                          "seconds": [round(v, 4) for v in t]}), flush=True)
