"""NVLink traffic of the cross-round kernels, for ncu (one process, no
inter-rank barriers): rank 0 of a 2-GPU peer-sharded C2 trial maps rank 1's
pool directly (moshpit_shard_probe_peers) and runs 4 rounds (2 local, 2 cross)
on GPU 0 alone, so `ncu --metrics nvlrx__bytes.sum,...` can replay the
cross_mean_kernel / shard_pull_kernel launches.  The averages are not valid
(rank 1 never runs); only the traffic is.  Prints the modelled ingress of
one cross round for comparison.

    ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum \
        -k regex:"cross_mean|shard_pull" python profiles/nvlink_ncu.py [C2|C5v-slab]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from paper_2103_03239_b200 import _capi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
M, d, N, D, p = {"C2": (32, 2, 1024, 1 << 22, 0.0),
                 "C5v-slab": (8, 4, 4096, 1 << 21, 0.0)}[cfg]
world = 2
sh = [mb.Shard(mb.GridConfig(M, d, 1), N, mb.FailureModel(p), mb.Rng(7), D, rank=r, world=world,
               device=r) for r in range(world)]
pools = (C.c_void_p * 8)()
for r in range(world):
    ptr, rows, ld = C.c_void_p(), C.c_uint64(), C.c_uint64()
    _capi.check(_capi.lib().moshpit_shard_pool(sh[r]._h, r, C.byref(ptr), C.byref(rows),
                                               C.byref(ld)))
    pools[r] = ptr.value
_capi.check(_capi.lib().moshpit_shard_probe_peers(sh[0]._h, pools))
for r in range(world):
    with torch.cuda.device(r):
        sh[r].fill_synthetic(0x5EED)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
with torch.cuda.device(0):
    for _ in range(2 * d):
        sh[0].round()
    torch.cuda.synchronize()
c = sh[0].stats()
Mg, es = M // world, 4
groups = c[1] // max(c[0], 1)
ingress = groups * es * (D / world) * ((M - Mg) + (world - 1))
print(json.dumps({"config": cfg, "world": world, "cross_rounds": c[0],
                  "active_groups_per_cross_round": groups,
                  "modelled_nvlink_ingress_bytes_per_cross_round": int(ingress),
                  "phase_a_share": round(groups * es * (D / world) * (M - Mg) / ingress, 4)}),
      flush=True)
for x in sh:
    x.close()
