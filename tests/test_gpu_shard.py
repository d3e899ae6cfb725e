"""Peer-sharded rounds checked on ONE GPU by emulating `world`
ranks as separate row pools (same kernels, same placement, sequential
phases): final vectors must be bit-identical to the single-GPU engine / the
oracle, whatever the world size."""
import numpy as np
import pytest

from tests._util import INIT_SEED, bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible")


@pytest.mark.parametrize("M,d,p,R,dim", [(32, 2, 0.01, 10, 37), (8, 4, 0.0, 8, 9),
                                         (8, 4, 0.05, 6, 16), (16, 3, 0.02, 6, 5),
                                         (8, 2, 0.2, 7, 12), (4, 1, 0.3, 3, 3),
                                         (32, 2, 0.0, 4, 1000)])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("f64", [False, True])
def test_emulated_shards_match_oracle(mb, oracle, M, d, p, R, dim, world, f64):
    if M % world:
        pytest.skip("world must divide M")
    import torch
    n = M ** d
    dt = np.float64 if f64 else np.float32
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim, world=world,
                  emulate=True, dtype=dt)
    sh.fill_synthetic(INIT_SEED)
    crossed = []
    for _ in range(R):
        crossed.append(sh.round()[1])
    torch.cuda.synchronize()
    got, mask = sh.read()
    assert mask.all()
    init = oracle.init_state(INIT_SEED, n, dim, dtype=dt)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(got, want)
    # rounds on axis d-1 (and only those) cross GPUs
    assert crossed == [(t % d) == d - 1 for t in range(R)]
    sh.close()


def test_shard_rejects_unsupported_layouts(mb):
    with pytest.raises(mb.InvalidArgument):  # not a full grid
        mb.Shard(mb.GridConfig(8, 2, 1), 60, mb.FailureModel(), mb.Rng(1), 4, world=2,
                 emulate=True)
    with pytest.raises(mb.InvalidArgument):  # world does not divide M
        mb.Shard(mb.GridConfig(6, 2, 1), 36, mb.FailureModel(), mb.Rng(1), 4, world=4,
                 emulate=True)


@pytest.mark.slow
def test_emulated_c5_valid_slab(mb, oracle):
    """C5-valid (4096 peers on 8^4, 4 rounds) over 8 emulated GPUs, one 2^18-
    coordinate slab: column slices bit-exact vs the oracle."""
    import torch
    M, d, R, dim = 8, 4, 4, 1 << 18
    n = M ** d
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(0.0), mb.Rng(7), dim, world=8,
                  emulate=True)
    sh.fill_synthetic(INIT_SEED)
    for _ in range(R):
        sh.round()
    torch.cuda.synchronize()
    got, mask = sh.read()
    assert mask.all()
    for c0 in (0, dim - 16):
        init = oracle.init_state(INIT_SEED, n, 16, col0=c0, dtype=np.float32)
        _, want = oracle.run_moshpit(M, d, init, 0.0, 7, R)
        assert bits_equal(np.ascontiguousarray(got[:, c0:c0 + 16]), want)
    sh.close()


@pytest.mark.parametrize("M,d,p,R,world", [(32, 2, 0.01, 10, 2), (8, 4, 0.05, 8, 4),
                                           (8, 2, 0.2, 7, 8), (16, 3, 0.0, 6, 4)])
def test_voided_row_moves_counted(mb, oracle, M, d, p, R, world):
    """moshpit_shard_cross_detail counts, per GPU, the voided-group rows whose
    new rank lives on another GPU (the cross round's extra NVLink traffic):
    equal to a replay of the oracle's trace (cells, then x_axis := rank)."""
    import torch
    n = M ** d
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), 4, world=world,
                  emulate=True)
    sh.fill_synthetic(INIT_SEED)
    for _ in range(R):
        sh.round()
    torch.cuda.synchronize()
    got = [sh.cross_detail(k)[2] for k in range(world)]
    sh.close()
    tr = oracle.trace(M, d, n, p, 7, R)
    cells = tr["cells"].astype(np.int64)
    digits = np.stack([(cells // M ** k) % M for k in range(d)], axis=1)
    mg = M // world
    want = [0] * world
    for t in range(R):
        axis = t % d
        off, mem = tr["group_off"][t], tr["members"][t]
        for g in range(int(tr["n_groups"][t])):
            ids = mem[off[g]:off[g + 1]]
            for rank, i in enumerate(ids):
                if axis == d - 1 and tr["void"][t][g]:
                    old, new = digits[i, axis] // mg, rank // mg
                    if old != new:
                        want[new] += 1
                digits[i, axis] = rank
    assert got == want
    if p == 0.0:
        assert sum(got) == 0


@pytest.mark.parametrize("M,d,p,R,dim,world", [(32, 2, 0.01, 6, 37, 2), (8, 4, 0.05, 8, 16, 4),
                                               (8, 2, 0.2, 5, 12, 8)])
def test_emulated_shards_copy_engine_path(mb, oracle, monkeypatch, M, d, p, R, dim, world):
    """The copy-engine cross round (MOSHPIT_CROSS_CE=1: staged remote chunks +
    copy-engine pulls of the chunk means) is bit-identical to the oracle too."""
    import torch
    monkeypatch.setenv("MOSHPIT_CROSS_CE", "1")
    n = M ** d
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim, world=world,
                  emulate=True)
    sh.fill_synthetic(INIT_SEED)
    for _ in range(R):
        sh.round()
    torch.cuda.synchronize()
    got, mask = sh.read()
    assert mask.all()
    init = oracle.init_state(INIT_SEED, n, dim, dtype=np.float32)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(got, want)
    sh.close()


@pytest.mark.parametrize("M,d,p,R,dim,world,slabs", [(32, 2, 0.01, 10, 1000, 2, 2),
                                                     (8, 4, 0.05, 8, 333, 4, 4),
                                                     (16, 3, 0.02, 6, 4099, 8, 3),
                                                     (8, 2, 0.2, 7, 12, 8, 2),
                                                     (32, 2, 0.0, 5, 9, 4, 8)])
def test_emulated_slab_pipeline_matches_oracle(mb, oracle, M, d, p, R, dim, world, slabs):
    """The slab pipeline (column slabs one round apart on their own streams,
    round tables in a ring of slots; read() flushes the lagging slabs) is
    bit-identical to the oracle."""
    import torch
    n = M ** d
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim, world=world,
                  emulate=True, slabs=slabs)
    sh.fill_synthetic(INIT_SEED)
    for _ in range(R):
        sh.round()
    sh.flush()
    torch.cuda.synchronize()
    got, mask = sh.read()
    assert mask.all()
    init = oracle.init_state(INIT_SEED, n, dim, dtype=np.float32)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(got, want)
    sh.close()


def test_shard_round_refuses_without_peers(mb):
    """Real mode (one rank per process, world > 1) without open_peers: an
    InvalidArgument, never a device fault."""
    sh = mb.Shard(mb.GridConfig(8, 2, 2), 64, mb.FailureModel(), mb.Rng(1), 4, rank=0, world=2)
    with pytest.raises(mb.InvalidArgument):
        sh.round()
    sh.close()


@pytest.mark.parametrize("M,d,p,R,dim,world,slabs", [(32, 2, 0.01, 6, 37, 2, 1),
                                                     (8, 4, 0.05, 8, 333, 4, 4),
                                                     (8, 2, 0.2, 7, 12, 8, 2)])
def test_shard_host_rows_round_trip(mb, oracle, M, d, p, R, dim, world, slabs):
    """The multi-GPU end-to-end path: each rank's peers loaded from host rows
    (row_peers gives the placement), rounds, rows stored back and mapped to
    peers by the placement after the rounds -- bit-identical to the oracle."""
    import torch
    n = M ** d
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim, world=world,
                  emulate=True, slabs=slabs)
    init = oracle.init_state(INIT_SEED, n, dim, dtype=np.float32)
    rows = sh.rows()
    keep = []
    for k in range(world):
        peers = sh.row_peers(k)
        host = np.zeros((rows, dim), dtype=np.float32)
        have = peers != 0xFFFFFFFF
        host[have] = init[peers[have]]
        sh.load_rows(host, k)
        keep.append(host)
    for _ in range(R):
        sh.round()
    got = np.full((n, dim), np.nan, dtype=np.float32)
    for k in range(world):
        out = np.zeros((rows, dim), dtype=np.float32)
        sh.store_rows(out, k)
        torch.cuda.synchronize()
        peers = sh.row_peers(k)
        have = peers != 0xFFFFFFFF
        got[peers[have]] = out[have]
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(got, want)
    red, mask = sh.read()
    assert mask.all() and bits_equal(red, want)
    with pytest.raises(mb.InvalidArgument):
        sh.load_rows(np.zeros((rows + 1, dim), dtype=np.float32), 0)
    sh.close()


def _rel_close(got, want, rtol):
    """|got - want| <= rtol * |want| elementwise (the synthetic state is in
    [0, 1), so every mean is positive: no cancellation to excuse)."""
    g, w = got.astype(np.float64), want.astype(np.float64)
    err = np.abs(g - w)
    bad = err > rtol * np.abs(w)
    return not bad.any(), float((err / np.maximum(np.abs(w), 1e-300)).max())


@pytest.mark.parametrize("M,d,p,R,dim", [(32, 2, 0.01, 10, 37), (8, 4, 0.0, 8, 9),
                                         (8, 4, 0.05, 6, 16), (16, 3, 0.02, 6, 5),
                                         (8, 2, 0.2, 7, 12), (32, 2, 0.0, 4, 1000)])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("f64", [False, True])
def test_emulated_partial_cross_within_tolerance(mb, oracle, M, d, p, R, dim, world, f64):
    """cross="partial" (per-GPU partial sums, one partial row per GPU and group
    over NVLink, fp64 combine in rank order): the summation order is not the
    reference's, so north_star's tolerance applies -- within 1e-6 relative of
    the fp32 oracle (1e-13 in fp64) -- while group formation, failures and
    placement stay exact (the same rows are written: every peer present)."""
    if M % world:
        pytest.skip("world must divide M")
    import torch
    n = M ** d
    dt = np.float64 if f64 else np.float32
    sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim, world=world,
                  emulate=True, dtype=dt, cross="partial")
    sh.fill_synthetic(INIT_SEED)
    for _ in range(R):
        sh.round()
    torch.cuda.synchronize()
    got, mask = sh.read()
    sh.close()
    assert mask.all()
    init = oracle.init_state(INIT_SEED, n, dim, dtype=dt)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    ok, worst = _rel_close(got, want, 1e-13 if f64 else 1e-6)
    assert ok, f"max relative error {worst:.3e}"
    if R < d:  # no cross round: the local rounds are the exact kernel 2
        assert bits_equal(got, want)


@pytest.mark.parametrize("M,d,p,R,dim,world,slabs", [(32, 2, 0.01, 10, 1000, 2, 3),
                                                     (8, 4, 0.05, 8, 333, 4, 4),
                                                     (8, 2, 0.2, 7, 12, 8, 2)])
def test_partial_cross_is_deterministic_across_slabs(mb, M, d, p, R, dim, world, slabs):
    """The partial-sum order is fixed (position order per GPU, rank order
    across GPUs): the slab pipeline gives the same bits as slabs = 1."""
    import torch
    n = M ** d
    outs = []
    for s in (1, slabs):
        sh = mb.Shard(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), dim,
                      world=world, emulate=True, slabs=s, cross="partial")
        sh.fill_synthetic(INIT_SEED)
        for _ in range(R):
            sh.round()
        sh.flush()
        torch.cuda.synchronize()
        outs.append(sh.read()[0])
        sh.close()
    assert bits_equal(outs[0], outs[1])


def test_shard_rejects_unknown_cross_mode(mb):
    with pytest.raises(mb.InvalidArgument):
        mb.Shard(mb.GridConfig(8, 2, 1), 64, mb.FailureModel(), mb.Rng(1), 4, world=2,
                 emulate=True, cross="approximate")
