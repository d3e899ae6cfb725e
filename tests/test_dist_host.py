"""CPU, world_size 2 over gloo: the multi-process host logic of the sharded
engine -- handle exchange order/size checks and identical validation on every
rank (the data plane itself needs GPUs: tests/mgpu/shard_check.py)."""
import os
import socket

import pytest
import torch.multiprocessing as tmp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2103_03239_b200 as mb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank]) * 128
        allh = mb.exchange_handles(mine, world)
        res = {"order": [h[0] for h in allh], "sizes": [len(h) for h in allh]}
        errs = []
        for args in [((8, 2, 1), 60, 2), ((6, 2, 1), 36, 4), ((8, 2, 1), 64, 9),
                     ((40, 2, 1), 1600, 2)]:
            (M, d, T), n, w = args
            try:
                mb.Shard(mb.GridConfig(M, d, T), n, mb.FailureModel(), mb.Rng(1), 4, rank=rank,
                         world=w)
                errs.append("none")
            except mb.InvalidArgument:
                errs.append("invalid_argument")
            except mb.CudaError:
                errs.append("cuda")
        gathered = [None] * world
        dist.all_gather_object(gathered, errs)
        res["errs_agree"] = all(g == gathered[0] for g in gathered)
        res["errs"] = errs
        try:
            mb.exchange_handles(mine, world + 1)
            res["bad_world"] = "none"
        except mb.InvalidArgument:
            res["bad_world"] = "invalid_argument"
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_handle_exchange_and_validation():
    world, port = 2, _free_port()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert out[r]["order"] == [0, 1]
        assert out[r]["sizes"] == [128, 128]
        assert out[r]["errs_agree"]
        # every layout above is invalid for peer sharding -> rejected before any device work
        assert out[r]["errs"] == ["invalid_argument"] * 4
        assert out[r]["bad_world"] == "invalid_argument"


@pytest.mark.gpu
@pytest.mark.parametrize("cross", ["exact", "partial"])
def test_real_multi_gpu_shards(cross):
    """One process per GPU over real NVLink: exact cross rounds bit-exact,
    partial-sum cross rounds within 1e-6 relative of the oracle."""
    import subprocess
    import sys

    import torch
    g = torch.cuda.device_count()
    if g < 2:
        pytest.skip("needs >= 2 GPUs (run under gpurun --gpus 2)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={min(g, 8)}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()),
                        os.path.join(root, "tests", "mgpu", "shard_check.py")],
                       capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CROSS=cross))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARD CHECK PASS" in r.stdout
