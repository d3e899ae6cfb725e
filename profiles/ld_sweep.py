"""Kernel 2 vs row stride: C5-valid slab (4096 peers on 8^4, 6M columns) with
the row pitch padded to different multiples; HBM fraction of kernel 2."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2103_03239_b200 as mb
M, d, N, W = 8, 4, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000
for pad in (4, 1024, 32768, 262144):
    ld = -(-W // pad) * pad
    x = torch.empty((N, ld), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, 0x5EED, dim=W)
    eng = mb.Engine(mb.GridConfig(M, d, 4), N, mb.FailureModel(0.0), mb.Rng(7))
    for _ in range(2):
        eng.round(x, dim=W)
    torch.cuda.synchronize()
    eng.set_timing(True)
    r0 = eng.stats()[1]
    for _ in range(8):
        eng.round(x, dim=W)
    torch.cuda.synchronize()
    ms, k = eng.kernel_time()
    rows = eng.stats()[1] - r0
    print(json.dumps({"W": W, "ld": ld, "pad": pad, "ms_per_launch": round(ms / k, 3),
                      "frac": round(2 * 4 * W * rows / (ms / 1e3) / 1e9 / 6552.6, 4)}))
    eng.close()
    del x
    torch.cuda.empty_cache()
