"""Slab-pipeline sweep of the peer-sharded C2 round per cross-round mode
(torchrun --nproc-per-node N).  Rank 0 prints one JSON line per setting:
ms per round (max over ranks), value, kernel sums."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    settings = [s.split(":") for s in os.environ.get(
        "SWEEP", "partial:1:0:0,partial:2:0:0,partial:4:0:0,partial:8:0:0,partial:4:148:148,"
                 "partial:8:148:148,exact:8:0:0").split(",")]
    for mode, slabs, lsm, csm in settings:
        for k, v in (("MOSHPIT_PIPE_LOCAL_SMS", lsm), ("MOSHPIT_PIPE_CROSS_SMS", csm)):
            if v != "0":
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        r = bench.run_peer(mb, torch, dist, "C2", 20, 5, rank, world, local, nvlink=True,
                           slabs=int(slabs), cross=mode)
        if rank == 0:
            print(json.dumps({"mode": mode, "slabs": int(slabs), "local_sms": lsm,
                              "cross_sms": csm, "value": r["value"],
                              "ms_per_round": r["ms_per_step"],
                              "combined_frac": r["roofline"]["combined_frac"],
                              "overlapped_frac": r["roofline"]["combined_frac_overlapped_bound"],
                              "local_kernel_ms": r["local_kernel_ms"],
                              "cross_kernel_ms": r["cross_kernel_ms"],
                              "phase_a_ms": r["roofline"]["cross"]["phase_a_ms"],
                              "phase_b_ms": r["roofline"]["cross"]["phase_b_ms"],
                              "nvlink_gb": r["roofline"]["cross"]["nvlink_ingress_gb_per_gpu"]}),
                  flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
