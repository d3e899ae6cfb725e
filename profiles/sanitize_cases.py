"""Small cases of every data-plane kernel for compute-sanitizer (one tool per
run: racecheck, synccheck, memcheck):  kernel 1 + kernel 2 (register and
bulk/TMA ring variants), the EXACT and FAST diagnostics, the row-pointer
streamed run_moshpit, emulated peer-sharded rounds (world 4, slab pipeline),
the trial batch, the fused SGD step (kernel 3, device noise) and
round_from_groups.  Exits non-zero if any result differs from the CPU oracle.

    compute-sanitizer --tool racecheck python profiles/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from oracle.oracle import Checker  # noqa: E402

o = Checker("oracle")
ok = True


def check(name, good):
    global ok
    print(f"{name}: {'ok' if good else 'MISMATCH'}", flush=True)
    ok = ok and good


M, d, n, p, R, dim = 16, 2, 256, 0.05, 4, 300
init = o.init_state(0x5EED, n, dim, dtype=np.float32)
_, want = o.run_moshpit(M, d, init, p, 7, R)
for kernel in (1, 2):  # register, bulk (cp.async.bulk ring)
    x = torch.zeros((n, 304), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, 0x5EED, dim=dim)
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0,
                    kernel=kernel)
    eng.set_reference(x, diagnostics="exact", dim=dim)
    for _ in range(R):
        eng.round(x, dim=dim)
        eng.record(x, dim=dim)
    torch.cuda.synchronize()
    check(f"engine kernel={kernel}", x[:, :dim].cpu().numpy().tobytes() == want.tobytes())
    eng.close()
x64 = init.astype(np.float64)
for diag in ("exact", "fast"):
    r = mb.run_moshpit(mb.GridConfig(M, d, 1), x64, mb.FailureModel(p), mb.Rng(7), R,
                       diagnostics=diag, return_vectors=True)
    ro, fo = o.run_moshpit(M, d, x64, p, 7, R)
    check(f"run_moshpit f64 {diag}", r.vectors.tobytes() == fo.tobytes())
os.environ["MOSHPIT_SLAB_BYTES"] = "1"  # streamed slabs + pinned staging ring
xs = o.init_state(0x5EED, 64, 70_000, dtype=np.float32)
r1 = mb.run_moshpit(mb.GridConfig(8, 2, 1), xs, mb.FailureModel(0.1), mb.Rng(3), 3,
                    diagnostics="exact", return_vectors=True)
_, w1 = o.run_moshpit(8, 2, xs, 0.1, 3, 3)
check("run_moshpit streamed", r1.vectors.tobytes() == w1.tobytes())
os.environ["MOSHPIT_SLAB_BYTES"] = str(1 << 40)
for slabs in (1, 2):
    sh = mb.Shard(mb.GridConfig(8, 2, 6), 64, mb.FailureModel(0.1), mb.Rng(7), 40, world=4,
                  emulate=True, slabs=slabs)
    sh.fill_synthetic(0x5EED)
    for _ in range(6):
        sh.round()
    got, mask = sh.read()
    _, ws = o.run_moshpit(8, 2, o.init_state(0x5EED, 64, 40, dtype=np.float32), 0.1, 7, 6)
    check(f"emulated shards slabs={slabs}", got.tobytes() == ws.tobytes())
    sh.close()
xb = np.stack([o.init_state(0x5EED + t, 64, 3, dtype=np.float64) for t in range(5)])
rb = mb.run_moshpit_batch(mb.GridConfig(8, 2, 1), xb, mb.FailureModel(0.05), list(range(5)), 6,
                          return_vectors=True)
good = True
for t in range(5):
    _, wb = o.run_moshpit(8, 2, xb[t], 0.05, t, 6)
    good = good and rb[t].vectors.tobytes() == wb.tobytes()
check("trial batch", good)
tgt = mb.Rng(7).stream("objective").normals(512)
cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=4, grid=mb.GridConfig(16, 2, 1), sigma=1.0,
                         n_peers=256)
res = mb.run_moshpit_sgd(cfg, mb.Quadratic(512, 1.0, 0.1, tgt), np.zeros(512), [], mb.Rng(7),
                         dtype=np.float32, diagnostics="none", noise="device")
check("sgd fused step (device noise)", np.isfinite(res.diagnostics.sigma_hat))
xg = np.random.default_rng(1).random((12, 9))
mem, off, vf = np.array([3, 1, 0, 5, 7, 2, 9], np.uint32), np.array([0, 3, 5, 7], np.uint32), \
    np.array([0, 1, 0], np.uint8)
want_g = xg.copy()
for g in range(3):
    rows = mem[off[g]:off[g + 1]]
    out, _ = o.butterfly(xg[rows], failed=np.full(len(rows), vf[g], np.uint8))
    want_g[rows] = out
check("round_from_groups", mb.round_from_groups(xg.copy(), mem, off, vf).tobytes() ==
      want_g.tobytes())
print("SANITIZE CASES", "PASS" if ok else "FAIL", flush=True)
sys.exit(0 if ok else 1)
