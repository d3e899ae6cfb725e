"""Per-kernel view of one rank's partial-sum cross round, for ncu (one
process, no inter-rank barriers): rank 0 of a `world`-GPU peer-sharded C2
trial (p = 0.01) maps the other ranks' pools directly
(moshpit_shard_probe_peers) and runs 2 local + 2 cross rounds on GPU 0
alone.  The averages are not valid (the other ranks never run); the
kernels' durations and DRAM / NVLink bytes are.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
nvlrx__bytes.sum -k regex:"partial|shard_pull|move_rows|group_mean|cross_mean" \
        python profiles/partial_probe.py 4 partial
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from paper_2103_03239_b200 import _capi  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cross = sys.argv[2] if len(sys.argv) > 2 else "partial"
M, d, N, D, p = 32, 2, 1024, 1 << 22, 0.01
sh = [mb.Shard(mb.GridConfig(M, d, 1), N, mb.FailureModel(p), mb.Rng(7), D, rank=r, world=world,
               device=r, cross=cross) for r in range(world)]
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
for r in range(world):
    torch.cuda.synchronize(r)
models = []
with torch.cuda.device(0):
    prev = (0, 0, 0)
    for _ in range(2 * d):
        sh[0].round()
        torch.cuda.synchronize()
        c = sh[0].stats()
        moved = sh[0].cross_detail(0)[2]
        if c[0] > prev[0]:  # a cross round: modelled NVLink user bytes into rank 0
            groups, mv = c[1] - prev[1], moved - prev[2]
            chunk = 4 * D // world
            if cross == "partial":
                b = groups * chunk * 2 * (world - 1) + 4 * D * mv
            else:
                b = groups * chunk * ((M - M // world) + (world - 1)) + 4 * D * mv
            models.append({"active_groups": groups, "voided_rows_moved_in": mv,
                           "modelled_nvlink_user_bytes": b})
        prev = (c[0], c[1], moved)
print(json.dumps({"world": world, "cross": cross, "cross_rounds": models}), flush=True)
for x in sh:
    x.close()
