"""e2e variance probe: repeated run_moshpit(C2) calls on pinned host buffers,
slab-streamed vs resident, with a plain H2D/D2H reference."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from paper_2103_03239_b200 import _capi  # noqa: E402

N, D, R = 1024, 1 << 22, 10
host = torch.empty((N, D), dtype=torch.float32, pin_memory=True)
dev = torch.empty((N, D), dtype=torch.float32, device="cuda")
mb.fill_synthetic(dev, 0x5EED)
torch.cuda.synchronize()
t = time.perf_counter(); host.copy_(dev); torch.cuda.synchronize()
print("plain D2H GB/s", round(N * D * 4 / (time.perf_counter() - t) / 1e9, 1))
t = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
print("plain H2D GB/s", round(N * D * 4 / (time.perf_counter() - t) / 1e9, 1))
del dev
torch.cuda.empty_cache()
lib = _capi.lib()
ptr = host.numpy().ctypes.data_as(C.c_void_p)
for mode in ("stream", "resident", "stream"):
    os.environ["MOSHPIT_SLAB_BYTES"] = str(256 << 20) if mode == "stream" else str(1 << 40)
    for it in range(3):
        dist, drift = np.zeros(R), np.zeros(R)
        act = np.zeros(R, dtype=np.uint32)
        a, b = C.c_double(0), C.c_double(0)
        t0 = time.perf_counter()
        _capi.check(lib.moshpit_run_moshpit(0, 32, 2, R, ptr, N, D, 0.01, 7, R, 1, C.byref(a),
                                            dist.ctypes.data_as(C.c_void_p),
                                            drift.ctypes.data_as(C.c_void_p),
                                            act.ctypes.data_as(C.c_void_p), C.byref(b), ptr))
        t1 = time.perf_counter() - t0
        print(mode, it, "s", round(t1, 3), "GB/s", round(N * D * 4 * R / t1 / 1e9, 1), flush=True)
