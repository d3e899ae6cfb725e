"""First-call latency of a fresh process (what a harness-style short process
pays): library load + CUDA context + module load, then the first and the
second small run_moshpit through the C ABI.  Run it as its own process."""
import ctypes as C
import json
import os
import sys
import time

t0 = time.perf_counter()
sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

from paper_2103_03239_b200 import _capi  # noqa: E402

lib = _capi.lib()
t_load = time.perf_counter() - t0
# the driver's share: cuInit + primary context of device 0 (what any CUDA
# program pays before its first kernel), timed through libcuda directly
cu = C.CDLL("libcuda.so.1")
t1 = time.perf_counter()
cu.cuInit(0)
dev, ctx = C.c_int(0), C.c_void_p()
cu.cuDeviceGet(C.byref(dev), 0)
cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev)
t_ctx = time.perf_counter() - t1
n, dim, R = 1024, 1, 50
x = np.random.default_rng(0).random((n, dim))
out = {"lib_bytes": os.path.getsize(_capi.LIB_PATH), "load_s": round(t_load, 4),
       "cuda_primary_context_s": round(t_ctx, 4)}
for k in ("first_call_s", "second_call_s", "third_call_s"):
    dist, drift = np.zeros(R), np.zeros(R)
    act = np.zeros(R, dtype=np.uint32)
    a, b = C.c_double(0), C.c_double(0)
    t1 = time.perf_counter()
    _capi.check(lib.moshpit_run_moshpit(_capi.F64, 32, 2, 1, x.ctypes.data_as(C.c_void_p), n,
                                        dim, 0.01, 7, R, _capi.DIAG_EXACT, C.byref(a),
                                        dist.ctypes.data_as(C.c_void_p),
                                        drift.ctypes.data_as(C.c_void_p),
                                        act.ctypes.data_as(C.c_void_p), C.byref(b), None))
    out[k] = round(time.perf_counter() - t1, 4)
print(json.dumps(out), flush=True)
