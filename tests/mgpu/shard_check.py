"""Real multi-process peer-sharded rounds: torchrun --nproc-per-node P.
Each process hosts RANKS_PER_PROC consecutive ranks (default 1; world =
P * RANKS_PER_PROC, e.g. world 8 on 4 GPUs with 2), with SLABS pipelined
column slabs (default 1).  Every process checks its resident peers' final
vectors bit-for-bit against the CPU oracle (CROSS=partial: the partial-sum
cross round, within 1e-6 relative); exits non-zero on mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2103_03239_b200 as mb  # noqa: E402
from oracle.oracle import Checker  # noqa: E402


def main():
    prank, procs = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", prank))
    per = int(os.environ.get("RANKS_PER_PROC", "1"))
    slabs = int(os.environ.get("SLABS", "1"))
    cross = os.environ.get("CROSS", "exact")
    world = procs * per
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    o = Checker("oracle")
    ok = True
    # (16, 2, ..., 20001): rows of >= 64 KB get the 4 KB row pitch
    for (M, d, p, R, dim) in [(32, 2, 0.01, 10, 4099), (8, 4, 0.05, 8, 1000), (16, 3, 0.0, 6, 64),
                              (8, 1, 0.2, 3, 17), (16, 2, 0.02, 6, 20001), (8, 3, 0.1, 7, 515)]:
        if M % world:
            continue
        n = M ** d
        sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim,
                      rank=prank * per, world=world, device=local, ranks_per_process=per,
                      slabs=slabs, cross=cross)
        sh.connect()
        sh.fill_synthetic(0x5EED)
        for _ in range(R):
            sh.round()
        sh.flush()
        torch.cuda.synchronize()
        got, mask = sh.read()
        init = o.init_state(0x5EED, n, dim, dtype=np.float32)
        _, want = o.run_moshpit(M, d, init, p, 7, R)
        if cross == "partial":
            g, w = got[mask].astype(np.float64), want[mask].astype(np.float64)
            good = bool((np.abs(g - w) <= 1e-6 * np.abs(w)).all())
        else:
            good = got[mask].tobytes() == want[mask].tobytes()
        cnt = torch.tensor([int(mask.sum()), int(good)])
        dist.all_reduce(cnt)
        if prank == 0:
            print(f"M={M} d={d} p={p} R={R} dim={dim} world={world} ({procs} processes x {per} "
                  f"ranks, slabs={slabs}, cross={cross}): resident rows {int(cnt[0])}/{n}, "
                  f"processes {'bit-exact' if cross == 'exact' else 'within 1e-6'} "
                  f"{int(cnt[1])}/{procs}", flush=True)
        ok = ok and int(cnt[0]) == n and int(cnt[1]) == procs
        dist.barrier()
        sh.close()
    dist.destroy_process_group()
    if prank == 0:
        print("SHARD CHECK", "PASS" if ok else "FAIL",
              "(copy-engine cross round)" if os.environ.get("MOSHPIT_CROSS_CE") == "1" else "",
              flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
