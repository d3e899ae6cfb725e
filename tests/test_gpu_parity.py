"""GPU parity: the sm_100a path (through the C ABI) against the oracle, the
golden vectors from the unmodified reference, and -- at full BASELINE sizes --
size-independent properties.

Bars (written in each test):
  * integer work (group tables, void flags, ranks, keys): bit-exact;
  * fp64 path: bit-exact with the reference (vectors AND TrialReport);
  * fp32 path: bit-exact with the fp32 restatement (same tree, same order);
    within 1e-6 relative of the fp64 reference on uniform inputs
    (north_star tolerance); after d rounds on a full grid every element within
    4 ulp of fp32(global fp64 mean).
"""
import numpy as np
import pytest

from tests._util import INIT_SEED, bits_equal, ulp_diff_f32, unhex, unhexa

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible: the GPU suite cannot run (no CPU fallback exists)")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def engine_run(mb, torch, M, d, n, dim, p, seed, rounds, dtype=None, ld=None, col0=0,
               kernel=0, tables=False):
    dtype = dtype or torch.float32
    vec = 4 if dtype == torch.float32 else 2
    ld = ld or max(vec, (dim + vec - 1) // vec * vec)
    x = torch.zeros((n, ld), dtype=dtype, device="cuda")
    mb.fill_synthetic(x, INIT_SEED, dim=dim, col0=col0)
    eng = mb.Engine(mb.GridConfig(M, d, rounds), n, mb.FailureModel(p), mb.Rng(seed),
                    kernel=kernel)
    tabs = []
    for _ in range(rounds):
        eng.round(x, dim=dim)
        if tables:
            tabs.append(eng.tables())
    torch.cuda.synchronize()
    stats = eng.stats()
    eng.close()
    return x, tabs, stats


# ---------------------------------------------------------------------------
# Kernel 1: integer plane
# ---------------------------------------------------------------------------
def test_form_groups_gpu_matches_golden(mb, golden):
    for g in golden["form_groups"]:
        peers = [mb.MatchPeer(i, mb.GroupKey(k), int(t)) for i, k, t in
                 zip(g["ids"], g["keys"], g["ts"])]
        groups = mb.form_groups_uncontested(peers, g["cap"])
        flat = [m for gr in groups for m in gr.members]
        assert flat == g["members"]
        off = np.cumsum([0] + [len(gr.members) for gr in groups]).tolist()
        assert off == g["group_off"]
        assert all(gr.leader == gr.members[0] for gr in groups)


@pytest.mark.parametrize("n,klen,kmax,cap", [(1, 1, 4, 8), (7, 0, 1, 3), (300, 1, 8, 16),
                                             (1000, 2, 5, 7), (5000, 1, 300, 32),
                                             (20000, 2, 40, 0xFFFFFFFF)])
def test_form_groups_gpu_matches_oracle(mb, oracle, n, klen, kmax, cap):
    gen = np.random.default_rng(n + klen)
    ids = gen.permutation(4 * n)[:n].astype(np.uint32)
    keys = gen.integers(0, kmax, (n, klen)).astype(np.uint32)
    ts = gen.integers(0, 2**48, n).astype(np.uint64)
    ts[::5] = ts[0]  # ties on the timestamp: the id decides
    m_ref, off_ref = oracle.form_groups(ids, keys, ts, cap)
    peers = [mb.MatchPeer(int(i), mb.GroupKey(list(map(int, k))), int(t))
             for i, k, t in zip(ids, keys, ts)]
    groups = mb.form_groups_uncontested(peers, cap)
    assert [m for g in groups for m in g.members] == m_ref.tolist()
    assert np.cumsum([0] + [len(g.members) for g in groups]).tolist() == off_ref.tolist()


@pytest.mark.parametrize("M,d,n,p,R", [(32, 2, 1024, 0.01, 10), (16, 3, 4096, 0.0, 3),
                                       (8, 4, 4096, 0.05, 4), (16, 2, 256, 0.0, 2),
                                       (5, 2, 24, 0.1, 10), (4, 3, 50, 0.2, 8),
                                       (8, 1, 8, 0.3, 3), (32, 2, 512, 0.0, 12),
                                       (2, 10, 1024, 0.02, 5), (3, 3, 27, 0.2, 7),
                                       (64, 2, 4000, 0.01, 3)])
def test_engine_tables_match_oracle_trace(mb, oracle, torch, M, d, n, p, R):
    """Group tables, void flags, ranks and next keys: bit-exact per round."""
    t = oracle.trace(M, d, n, p, 7, R)
    _, tabs, _ = engine_run(mb, torch, M, d, n, 4, p, 7, R, tables=True)
    for r in range(R):
        g = int(t["n_groups"][r])
        assert tabs[r]["n_groups"] == g
        assert tabs[r]["group_off"].tolist() == t["group_off"][r][: g + 1].tolist()
        assert tabs[r]["members"].tolist() == t["members"][r].tolist()
        assert tabs[r]["void"].tolist() == t["void"][r][:g].tolist()
        assert tabs[r]["rank"].tolist() == t["rank"][r].tolist()
    if d > 1:
        assert tabs[-1]["keys"].tolist() == t["keys_final"].tolist()


# ---------------------------------------------------------------------------
# fp64: bit parity with the reference
# ---------------------------------------------------------------------------
def test_run_moshpit_f64_bit_exact_vs_golden(mb, oracle, golden):
    for c in golden["run_moshpit"]:
        x = oracle.init_state(INIT_SEED, c["n"], c["dim"], dtype=np.float64)
        rep = mb.run_moshpit(mb.GridConfig(c["M"], c["d"], 1), x, mb.FailureModel(c["p"]),
                             mb.Rng(c["seed"]), c["rounds"], return_vectors=True)
        assert rep.initial_distortion == unhex(c["initial_distortion"]), c
        assert bits_equal(np.array(rep.distortion), unhexa(c["distortion"])), c
        assert bits_equal(np.array(rep.mean_drift), unhexa(c["mean_drift"])), c
        assert rep.active_counts == c["active_counts"]
        assert rep.cost_units == unhex(c["cost_units"])
        if c["final"] is not None:
            assert bits_equal(rep.vectors.reshape(-1), unhexa(c["final"]))
        for i, row in zip(c["final_rows"], c["final_rows_values"]):
            assert bits_equal(rep.vectors[i], unhexa(row))


@pytest.mark.parametrize("M,d,n,p,R,dim", [(3, 2, 9, 0.0, 4, 2), (5, 2, 24, 0.1, 10, 3),
                                           (4, 3, 50, 0.2, 8, 5), (8, 1, 8, 0.3, 3, 4),
                                           (7, 2, 40, 0.5, 6, 3), (2, 5, 32, 0.1, 9, 2),
                                           (40, 2, 1600, 0.01, 3, 7), (33, 2, 1000, 0.0, 2, 5),
                                           (16, 2, 256, 0.05, 3, 70001)])
def test_run_moshpit_f64_equals_reference(mb, ref, M, d, n, p, R, dim):
    x = np.random.default_rng(n * 31 + d).random((n, dim))
    rr, fr = ref.run_moshpit(M, d, x, p, 1000 + n, R)
    rep = mb.run_moshpit(mb.GridConfig(M, d, 1), x, mb.FailureModel(p), mb.Rng(1000 + n), R,
                         return_vectors=True)
    assert rep.initial_distortion == rr["initial_distortion"]
    assert bits_equal(np.array(rep.distortion), rr["distortion"])
    assert bits_equal(np.array(rep.mean_drift), rr["mean_drift"])
    assert rep.active_counts == rr["active_counts"].tolist()
    assert bits_equal(rep.vectors, fr)


def test_reference_protocol_properties_on_gpu(mb):
    # test_protocols.cpp:45-55 full grid exact in d rounds
    x = mb.Rng(10).stream("init")
    init = np.array([[x.uniform() for _ in range(2)] for _ in range(9)])
    rep = mb.run_moshpit(mb.GridConfig(3, 2, 1), init, mb.FailureModel(), mb.Rng(99), 4)
    assert rep.distortion[0] > 1e-24 and rep.distortion[1] <= 1e-24 and rep.distortion[3] <= 1e-24
    # :57-63 single peer
    rep = mb.run_moshpit(mb.GridConfig(4, 2, 1), [[3.0, 4.0]], mb.FailureModel(), mb.Rng(1), 3)
    assert rep.initial_distortion == 0.0 and rep.rounds_to(1e-9, 50) == 0
    # :72-88 mean conservation under failures
    for trial in range(5):
        s = mb.Rng(11).stream("init", trial)
        init = np.array([[s.uniform() for _ in range(3)] for _ in range(24)])
        rep = mb.run_moshpit(mb.GridConfig(5, 2, 1), init, mb.FailureModel(trial * 0.05),
                             mb.Rng(1000 + trial), 10)
        assert max(rep.mean_drift) <= 1e-12
    # :113-122 converges for p < 1
    for s_ in range(20):
        s = mb.Rng(13).stream("init", s_)
        init = np.array([[s.uniform()] for _ in range(12)])
        rep = mb.run_moshpit(mb.GridConfig(4, 2, 1), init, mb.FailureModel(0.2),
                             mb.Rng(4000 + s_), 50)
        assert rep.distortion[-1] < rep.initial_distortion
    # acceptance.cpp:103-122: N=1024, M=32, p=0 needs exactly 2 rounds every seed
    for seed in range(3):
        s = mb.Rng(seed).stream("init")
        init = np.array([[s.uniform()] for _ in range(1024)])
        rep = mb.run_moshpit(mb.GridConfig(32, 2, 1), init, mb.FailureModel(), mb.Rng(seed), 4)
        assert rep.rounds_to(1e-9, 50) == 2


def test_all_failed_round_leaves_state(mb):
    x = np.random.default_rng(1).random((16, 3))
    rep = mb.run_moshpit(mb.GridConfig(4, 2, 1), x, mb.FailureModel(1.0), mb.Rng(3), 3,
                         return_vectors=True)
    assert bits_equal(rep.vectors, x)
    assert rep.active_counts == [0, 0, 0]


# ---------------------------------------------------------------------------
# fp32: bit parity with the fp32 restatement, tolerance vs fp64
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("M,d,n,p,R,dim", [(16, 2, 256, 0.0, 2, 64), (32, 2, 1024, 0.01, 10, 37),
                                           (16, 3, 4096, 0.0, 3, 8), (8, 4, 4096, 0.0, 4, 9),
                                           (5, 2, 24, 0.1, 10, 3), (40, 2, 1600, 0.02, 4, 13),
                                           (8, 1, 8, 0.3, 3, 1),
                                           # column means over the representative map:
                                           # distinct rows within / past the staged budget
                                           (32, 2, 1024, 0.01, 4, 68), (32, 2, 1024, 0.2, 3, 36),
                                           (8, 2, 64, 0.05, 5, 20),
                                           # wide rows: the EXACT drift chain runs in column
                                           # segments beside the means
                                           (16, 2, 256, 0.05, 3, 70001), (8, 2, 64, 0.0, 2, 131072)])
def test_run_moshpit_f32_bit_exact_vs_oracle(mb, oracle, M, d, n, p, R, dim):
    x = oracle.init_state(INIT_SEED, n, dim, dtype=np.float32)
    ro, fo = oracle.run_moshpit(M, d, x, p, 7, R)
    exact = mb.run_moshpit(mb.GridConfig(M, d, 1), x, mb.FailureModel(p), mb.Rng(7), R,
                           diagnostics="exact", return_vectors=True)
    assert bits_equal(exact.vectors, fo)
    assert exact.initial_distortion == ro["initial_distortion"]
    assert bits_equal(np.array(exact.distortion), ro["distortion"])
    assert bits_equal(np.array(exact.mean_drift), ro["mean_drift"])
    assert exact.active_counts == ro["active_counts"].tolist()
    fast = mb.run_moshpit(mb.GridConfig(M, d, 1), x, mb.FailureModel(p), mb.Rng(7), R,
                          return_vectors=True)
    assert bits_equal(fast.vectors, fo)
    # FAST diagnostics: fixed-order chunked fp64 sums; tolerance 1e-12 relative
    np.testing.assert_allclose(fast.distortion, ro["distortion"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(fast.mean_drift, ro["mean_drift"], rtol=1e-9, atol=1e-18)


def test_f32_within_1e6_of_fp64_reference(mb, oracle):
    x = oracle.init_state(INIT_SEED, 1024, 96, dtype=np.float32)
    _, f64 = oracle.run_moshpit(32, 2, x.astype(np.float64), 0.01, 7, 10)
    rep = mb.run_moshpit(mb.GridConfig(32, 2, 1), x, mb.FailureModel(0.01), mb.Rng(7), 10,
                         return_vectors=True)
    rel = np.abs(rep.vectors.astype(np.float64) - f64) / np.abs(f64)
    assert rel.max() <= 1e-6  # north_star fp32 tolerance


# ---------------------------------------------------------------------------
# Standalone data-plane entry points
# ---------------------------------------------------------------------------
def test_butterfly_gpu_matches_golden(mb, golden):
    for b in golden["butterfly"]:
        x = unhexa(b["inputs"]).reshape(b["n"], b["dim"])
        out = mb.butterfly_allreduce(x, mb.PartitionWeights.uniform(b["n"]), b["failed"])
        assert out.completed == b["completed"]
        assert out.chunks == list(range(b["n"]))
        assert bits_equal(out.vectors.reshape(-1), unhexa(b["out"]))


@pytest.mark.parametrize("n", [1, 2, 5, 8, 9, 16, 17, 31, 32, 33, 40, 64, 100])
def test_butterfly_gpu_f32_f64_all_group_sizes(mb, oracle, n):
    gen = np.random.default_rng(n)
    for dt in (np.float32, np.float64):
        x = gen.standard_normal((n, 23)).astype(dt)
        want, _ = oracle.butterfly(x)
        got = mb.butterfly_allreduce(x, mb.PartitionWeights.uniform(n))
        assert got.completed and bits_equal(got.vectors, want)
    # partition choice does not change the result (test_allreduce.cpp:67-73)
    inp = np.array([[1.0, 2.0, 3.0, 10.0], [3.0, 4.0, 5.0, 20.0]])
    a = mb.butterfly_allreduce(inp, mb.PartitionWeights.uniform(2))
    b = mb.butterfly_allreduce(inp, mb.PartitionWeights([0.9, 0.1]))
    assert bits_equal(a.vectors, b.vectors)


def test_group_mean_distortion_mean_of(mb, ref):
    assert mb.group_mean([[1.0, 2.0], [3.0, 6.0]]).tolist() == [2.0, 4.0]
    assert mb.distortion([[1.0], [3.0]], [2.0]) == 1.0
    assert mb.distortion([[5.0, 5.0], [5.0, 5.0]], [5.0, 5.0]) == 0.0
    gen = np.random.default_rng(3)
    x = gen.standard_normal((777, 19))
    assert bits_equal(mb.mean_of(x), ref.mean_of(x))
    r = gen.standard_normal(19)
    assert mb.distortion(x, r) == ref.distortion(x, r)


def test_moshpit_average_gpu_matches_golden(mb, oracle, golden):
    for c in golden["moshpit_average"]:
        x = oracle.init_state(INIT_SEED, c["n"], c["dim"], dtype=np.float64)
        y = mb.moshpit_average(x.copy(), mb.GridConfig(c["M"], c["d"], 1), c["rounds"],
                               mb.Rng(c["seed"]).stream(c["name"]))
        assert bits_equal(y.reshape(-1), unhexa(c["out"]))
        x32 = x.astype(np.float32)
        want = oracle.moshpit_average(x32, c["M"], c["d"], c["rounds"], c["seed"], c["name"])
        got = mb.moshpit_average(x32.copy(), mb.GridConfig(c["M"], c["d"], 1), c["rounds"],
                                 mb.Rng(c["seed"]).stream(c["name"]))
        assert bits_equal(got, want)


# ---------------------------------------------------------------------------
# Device-resident engine: padded strides, both precisions, both kernels
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dim,ldpad", [(1, 0), (3, 4), (5, 0), (64, 8), (1027, 4), (4099, 0)])
@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("kernel", [1, 2])
def test_engine_padded_rows_match_oracle(mb, oracle, torch, dim, ldpad, f64, kernel):
    M, d, n, p, R = 16, 2, 256, 0.05, 4
    dt = torch.float64 if f64 else torch.float32
    vec = 2 if f64 else 4
    ld = (dim + vec - 1) // vec * vec + ldpad
    x, _, _ = engine_run(mb, torch, M, d, n, dim, p, 7, R, dtype=dt, ld=ld, kernel=kernel)
    init = oracle.init_state(INIT_SEED, n, dim, dtype=np.float64 if f64 else np.float32)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(x[:, :dim].cpu().numpy(), want)


@pytest.mark.parametrize("M,d,n,p,R", [(32, 2, 1024, 0.01, 10), (8, 4, 4096, 0.02, 4),
                                       (16, 3, 4096, 0.0, 3), (32, 2, 700, 0.05, 6),
                                       (5, 3, 125, 0.1, 5)])
def test_bulk_kernel_equals_register_kernel(mb, torch, M, d, n, p, R):
    """Kernel-2 variants (register tree vs cp.async.bulk ring): bit-identical."""
    dim = 70001
    a, _, sa = engine_run(mb, torch, M, d, n, dim, p, 7, R, kernel=1)
    b, _, sb = engine_run(mb, torch, M, d, n, dim, p, 7, R, kernel=2)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    assert sa == sb


def test_bulk_kernel_rejects_groups_over_32(mb, torch):
    with pytest.raises(mb.InvalidArgument):
        engine_run(mb, torch, 64, 2, 200, 8, 0.0, 7, 1, kernel=2)


def _slice_check(mb, oracle, x, M, d, n, p, seed, R, cols):
    for c0 in cols:
        init = oracle.init_state(INIT_SEED, n, 16, col0=c0, dtype=np.float32)
        _, want = oracle.run_moshpit(M, d, init, p, seed, R)
        got = x[:, c0:c0 + 16].cpu().numpy()
        assert bits_equal(got, want), f"column slice {c0}"


def _exact_mean_check(torch, x0_mean, x, dim):
    """Full grid after d rounds: every element within 4 ulp of fp32(global
    fp64 mean); distortion/D <= 1e-15."""
    target = x0_mean.to(torch.float32)
    worst = 0
    for i0 in range(0, x.shape[0], 128):
        blk = x[i0:i0 + 128, :dim]
        diff = (blk.view(torch.int32).to(torch.int64) -
                target.view(torch.int32).to(torch.int64)[None, :]).abs().max().item()
        worst = max(worst, diff)
    assert worst <= 4, worst
    dist = 0.0
    for i0 in range(0, x.shape[0], 128):
        blk = x[i0:i0 + 128, :dim].double() - x0_mean[None, :]
        dist += (blk * blk).sum().item()
    assert dist / x.shape[0] / dim <= 1e-15


def _column_mean(torch, x, dim):
    acc = torch.zeros(dim, dtype=torch.float64, device=x.device)
    for i0 in range(0, x.shape[0], 64):
        acc += x[i0:i0 + 64, :dim].double().sum(0)
    return acc / x.shape[0]


@pytest.mark.slow
def test_c1_full_size(mb, oracle, torch):
    """C1: 256 peers, 16x16, D=2^20 fp32, p=0, 2 rounds -> exact mean."""
    M, d, n, dim, R = 16, 2, 256, 1 << 20, 2
    x = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED)
    m0 = _column_mean(torch, x, dim)
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(0.0), mb.Rng(7))
    for _ in range(R):
        eng.round(x)
    torch.cuda.synchronize()
    _slice_check(mb, oracle, x, M, d, n, 0.0, 7, R, [0, 12345 * 16, dim - 16])
    _exact_mean_check(torch, m0, x, dim)


@pytest.mark.slow
def test_c2_full_size(mb, oracle, torch):
    """C2: 1024 peers, 32x32, D=2^22 fp32, p=0.01, 10 rounds (17.2 GB state)."""
    M, d, n, dim, R, p = 32, 2, 1024, 1 << 22, 10, 0.01
    x = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED)
    m0 = _column_mean(torch, x, dim)
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7))
    for _ in range(R):
        eng.round(x)
    torch.cuda.synchronize()
    _slice_check(mb, oracle, x, M, d, n, p, 7, R, [0, 777 * 16, dim - 16])
    # mean conservation (test_protocols.cpp:72-88, fp32-scaled)
    m1 = _column_mean(torch, x, dim)
    drift = ((m1 - m0).norm() / m0.norm()).item()
    assert drift <= 1e-6
    del x
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("M,d,n,R", [(16, 3, 4096, 3), (8, 4, 4096, 4)])
def test_c3_c5_slab(mb, oracle, torch, M, d, n, R):
    """C3 (16^3) and C5-valid (4096 on 8^4): one resident D-slab of 2^20
    coordinates (coordinates are independent) -> exact mean."""
    dim = 1 << 20
    x = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED, col0=3 << 20)
    m0 = _column_mean(torch, x, dim)
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(0.0), mb.Rng(7))
    for _ in range(R):
        eng.round(x)
    torch.cuda.synchronize()
    for c0 in [0, dim - 16]:
        init = oracle.init_state(INIT_SEED, n, 16, col0=(3 << 20) + c0, dtype=np.float32)
        _, want = oracle.run_moshpit(M, d, init, 0.0, 7, R)
        assert bits_equal(x[:, c0:c0 + 16].cpu().numpy(), want)
    _exact_mean_check(torch, m0, x, dim)
    del x
    torch.cuda.empty_cache()


def test_native_library_is_loaded_in_process(mb):
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libmoshpit_b200.so" in maps


@pytest.mark.parametrize("f64,diag", [(False, "fast"), (False, "exact"), (True, "exact"),
                                      (False, "none")])
def test_streamed_run_moshpit_equals_resident(mb, oracle, monkeypatch, f64, diag):
    """run_moshpit on host buffers streams D-slabs (H2D || rounds || D2H)
    once the state exceeds the slab budget; vectors and TrialReport must be
    bit-identical to the resident path (coordinates independent)."""
    n, dim, R = 256, 200_003, 4
    dt = np.float64 if f64 else np.float32
    x = oracle.init_state(INIT_SEED, n, dim, dtype=dt)
    grid, fm = mb.GridConfig(16, 2, 1), mb.FailureModel(0.05)
    monkeypatch.setenv("MOSHPIT_SLAB_BYTES", "1")  # 64 Ki-column slabs -> 4 slabs, ring reused
    a = mb.run_moshpit(grid, x, fm, mb.Rng(7), R, diagnostics=diag, return_vectors=True)
    monkeypatch.setenv("MOSHPIT_SLAB_BYTES", str(1 << 40))  # resident
    b = mb.run_moshpit(grid, x, fm, mb.Rng(7), R, diagnostics=diag, return_vectors=True)
    assert bits_equal(a.vectors, b.vectors)
    for k in ("distortion", "mean_drift"):
        assert bits_equal(np.array(getattr(a, k)), np.array(getattr(b, k))), k
    assert bits_equal(np.array([a.initial_distortion]), np.array([b.initial_distortion]))
    assert a.active_counts == b.active_counts
    if not f64:
        init = oracle.init_state(INIT_SEED, n, 64, col0=131_000, dtype=dt)
        _, want = oracle.run_moshpit(16, 2, init, 0.05, 7, R)
        assert bits_equal(np.ascontiguousarray(a.vectors[:, 131_000:131_064]), want)


def test_concurrent_callers_are_independent(mb, oracle):
    """harness::run_experiment calls run_moshpit from many threads at once
    (harness.hpp:240-248): concurrent calls through the C ABI (ctypes releases
    the GIL) must equal the sequential results bit for bit."""
    import concurrent.futures as cf
    cases = [(16, 2, 256, 0.05, 6, 33), (32, 2, 1024, 0.01, 4, 17), (8, 3, 512, 0.0, 3, 9),
             (5, 2, 25, 0.2, 10, 4)] * 3
    def run(c):
        M, d, n, p, R, dim = c
        x = oracle.init_state(INIT_SEED + n, n, dim, dtype=np.float64)
        r = mb.run_moshpit(mb.GridConfig(M, d, 1), x, mb.FailureModel(p), mb.Rng(n), R,
                           return_vectors=True)
        return r.vectors, np.array(r.distortion)
    seq = [run(c) for c in cases]
    with cf.ThreadPoolExecutor(max_workers=6) as ex:
        par = list(ex.map(run, cases))
    for (va, da), (vb, db) in zip(seq, par):
        assert bits_equal(va, vb) and bits_equal(da, db)


@pytest.mark.parametrize("f64", [False, True])
def test_run_moshpit_rows_equals_contiguous(mb, oracle, monkeypatch, f64):
    """moshpit_run_moshpit_rows (the drop-in's row-pointer entry: host threads
    pack the caller's rows into a pinned ring, no flattened copy) gives the
    same TrialReport bits as the contiguous call, streamed and resident."""
    import ctypes as C
    from paper_2103_03239_b200 import _capi
    n, dim, R = 256, 200_003, 4
    dt = np.float64 if f64 else np.float32
    x = oracle.init_state(INIT_SEED, n, dim, dtype=dt)
    rows = [np.array(x[i]) for i in range(n)]  # separate pageable allocations
    ptrs = (C.c_void_p * n)(*[r.ctypes.data for r in rows])
    grid, fm = mb.GridConfig(16, 2, 1), mb.FailureModel(0.05)
    for slab in ("1", str(1 << 40)):  # 4 streamed slabs, then resident
        monkeypatch.setenv("MOSHPIT_SLAB_BYTES", slab)
        want = mb.run_moshpit(grid, x, fm, mb.Rng(7), R, diagnostics="exact")
        dist, drift = np.zeros(R), np.zeros(R)
        act = np.zeros(R, dtype=np.uint32)
        init_d, cost = C.c_double(0), C.c_double(0)
        _capi.check(_capi.lib().moshpit_run_moshpit_rows(
            _capi.F64 if f64 else _capi.F32, 16, 2, 1, ptrs, n, dim, 0.05, 7, R, _capi.DIAG_EXACT,
            C.byref(init_d), dist.ctypes.data_as(C.c_void_p), drift.ctypes.data_as(C.c_void_p),
            act.ctypes.data_as(C.c_void_p), C.byref(cost)))
        assert bits_equal(dist, np.array(want.distortion))
        assert bits_equal(drift, np.array(want.mean_drift))
        assert bits_equal(np.array([init_d.value]), np.array([want.initial_distortion]))
        assert list(act) == want.active_counts
        assert cost.value == want.cost_units


def test_engine_alternating_streams(mb, oracle, torch):
    """Engine.round on a different stream each call: the engine orders each
    round after the previous one (event + stream wait), so the result equals
    the single-stream run bit for bit (cross-stream table reuse)."""
    M, d, n, p, R, dim = 32, 2, 1024, 0.05, 6, 1 << 16
    x0 = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x0, INIT_SEED)
    a = x0.clone()
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    for _ in range(R):
        eng.round(a)
    torch.cuda.synchronize()
    eng.close()
    b = x0.clone()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(3)]
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    for r in range(R):
        # no caller-side ordering at all: round r+1 on another stream must
        # still start after round r (its tables and its state writes)
        eng.round(b, stream=streams[r % 3])
    torch.cuda.synchronize()
    rounds, _ = eng.stats()
    eng.close()
    assert rounds == R
    assert torch.equal(a, b)


@pytest.mark.parametrize("f64,diag", [(False, "fast"), (True, "exact"), (False, "exact")])
def test_engine_device_report_equals_run_moshpit(mb, torch, f64, diag):
    """Engine.set_reference / record / report (record_round on the device,
    protocols.hpp:68-84) give the same TrialReport bits as run_moshpit on host
    buffers with the same mode."""
    M, d, n, p, R, dim = 16, 2, 256, 0.05, 5, 70_001
    tdt = torch.float64 if f64 else torch.float32
    x = torch.zeros((n, 70_004), dtype=tdt, device="cuda")  # padded rows: ld 16-byte aligned
    mb.fill_synthetic(x, INIT_SEED, dim=dim)
    host = np.ascontiguousarray(x[:, :dim].cpu().numpy())
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    eng.set_reference(x, diagnostics=diag, dim=dim)
    for _ in range(R):
        eng.round(x, dim=dim)
        eng.record(x, dim=dim)
    init, dist, drift = eng.report()
    eng.close()
    want = mb.run_moshpit(mb.GridConfig(M, d, 1), host, mb.FailureModel(p), mb.Rng(7), R,
                          diagnostics=diag)
    assert bits_equal(np.array([init]), np.array([want.initial_distortion]))
    assert bits_equal(np.array(dist), np.array(want.distortion))
    assert bits_equal(np.array(drift), np.array(want.mean_drift))


@pytest.mark.parametrize("trial", range(6))
@pytest.mark.parametrize("cap", [0, 3])
def test_round_from_contested_groups_matches_reference(mb, ref, oracle, torch, trial, cap):
    """the unmodified reference's CONTESTED form_groups
    (skewed arrivals + FailStop, matchmaking.hpp:104-294) feeds the GPU data
    plane through moshpit_round_from_groups; the vectors after the round are
    bit-identical to the reference's butterfly_allreduce per sealed group (fp64),
    and the fp32 path to the fp32 restatement's butterfly."""
    rng = np.random.default_rng(100 + trial)
    n, dim = 6 + 5 * trial, 37
    x = rng.random((n, dim))
    mem, off, vf, want = ref.contested_round(1000 + trial, x, nkeys=3, cap=cap)
    assert len(off) > 1
    got = mb.round_from_groups(x.copy(), mem, off, vf)
    assert bits_equal(got, want)
    # device form, padded rows, fp32 vs the restatement group by group
    x32 = x.astype(np.float32)
    t = torch.zeros((n, 40), dtype=torch.float32, device="cuda")
    t[:, :dim] = torch.from_numpy(x32).cuda()
    mb.round_from_groups(t, mem, off, vf, dim=dim)
    torch.cuda.synchronize()
    want32 = x32.copy()
    for g in range(len(off) - 1):
        rows = mem[off[g]:off[g + 1]]
        out, done = oracle.butterfly(x32[rows], failed=np.full(len(rows), vf[g], np.uint8))
        want32[rows] = out
    assert bits_equal(t[:, :dim].cpu().numpy(), want32)


def test_round_from_groups_validates_like_the_reference(mb):
    x = np.zeros((4, 3))
    with pytest.raises(mb.InvalidArgument):  # empty group (allreduce.hpp:83)
        mb.round_from_groups(x, [0, 1], [0, 0, 2])
    with pytest.raises(mb.OutOfRange):
        mb.round_from_groups(x, [0, 7], [0, 2])
    with pytest.raises(mb.InvalidArgument):  # a row in two groups
        mb.round_from_groups(x, [0, 1, 1], [0, 2, 3])


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 16, 17, 31, 100, 255, 256, 257, 777, 1000, 1024,
                               1025])
def test_column_means_equal_reference(mb, ref, n):
    """mean_of on the GPU (the column means every diagnostic uses) equals the
    unmodified reference's pairwise tree bit for bit for group sizes around
    every leaf / split boundary (core.hpp:72-81, 128-133)."""
    x = np.random.default_rng(n).standard_normal((n, 45))
    assert bits_equal(mb.mean_of(x), ref.mean_of(x))


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512, 1024, 4096])
@pytest.mark.parametrize("dim", [2, 66, 1030])
def test_column_means_staged_tree_equal_reference(mb, ref, n, dim):
    """n = 8 * 2^K with 16-byte rows: the cp.async-staged binary-counter
    evaluation of the tree (diag_kernel.cu colmean_staged), with column
    vectors past the row end in the last CTA, bit for bit."""
    x = np.random.default_rng(n + dim).standard_normal((n, dim))
    assert bits_equal(mb.mean_of(x), ref.mean_of(x))


@pytest.mark.parametrize("n", [8, 256, 1024, 1000])
def test_column_means_row_gather_equal_reference(mb, ref, n):
    """group_mean over a member list with repeated rows (the representative
    gather the diagnostics use after a round): tree element i is row
    members[i]."""
    import ctypes as C
    rng = np.random.default_rng(n)
    x = rng.standard_normal((300, 66))
    mem = rng.integers(0, 300, n).astype(np.uint32)
    out = np.zeros(66)
    mb.check(mb._capi.lib().moshpit_group_mean(
        1, x.ctypes.data_as(C.c_void_p), 300, 66, mem.ctypes.data_as(C.c_void_p), n,
        out.ctypes.data_as(C.c_void_p)))
    assert bits_equal(out, ref.mean_of(x[mem]))


@pytest.mark.parametrize("diag", ["fast", "exact"])
def test_engine_round_record_equals_round_then_record(mb, torch, diag):
    """round_record reads one representative row per averaged group (every
    member holds the same mean); the report must equal round() + record()
    bit for bit (which read every row)."""
    M, d, n, p, R, dim = 32, 2, 1024, 0.05, 5, 4096
    x0 = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x0, INIT_SEED)
    reports = []
    for combined in (False, True):
        x = x0.clone()
        eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
        eng.set_reference(x, diagnostics=diag)
        for _ in range(R):
            if combined:
                eng.round_record(x)
            else:
                eng.round(x)
                eng.record(x)
        reports.append(eng.report())
        eng.close()
    (i0, d0, f0), (i1, d1, f1) = reports
    assert bits_equal(np.array([i0]), np.array([i1]))
    assert bits_equal(np.array(d0), np.array(d1))
    assert bits_equal(np.array(f0), np.array(f1))


@pytest.mark.parametrize("f64,diag,M,d,n,p,R,dim", [
    (False, "fast", 16, 2, 256, 0.05, 7, 70_001),
    (False, "fast", 32, 2, 1024, 0.01, 6, 8_195),
    (True, "fast", 8, 3, 400, 0.2, 5, 4_099),
    (False, "fast", 5, 2, 25, 0.3, 9, 37),
    (False, "exact", 16, 2, 256, 0.05, 4, 1_000),
])
def test_engine_rounds_record_equals_run_moshpit(mb, torch, f64, diag, M, d, n, p, R, dim):
    """Engine.rounds_record (R rounds + record_round in one call; FAST reuses
    the voided rows' cached row partials and re-reads only the averaged
    groups' representatives) gives the TrialReport bits and vectors of
    run_moshpit on host buffers, and of R round_record calls."""
    tdt = torch.float64 if f64 else torch.float32
    pad = (dim + 3) // 4 * 4
    x = torch.zeros((n, pad), dtype=tdt, device="cuda")
    mb.fill_synthetic(x, INIT_SEED, dim=dim)
    host = np.ascontiguousarray(x[:, :dim].cpu().numpy())
    y = x.clone()
    outs = []
    for mode in ("rounds", "each"):
        z = x if mode == "rounds" else y
        eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
        eng.set_reference(z, diagnostics=diag, dim=dim)
        if mode == "rounds":
            act = eng.rounds_record(z, R, dim=dim)
        else:
            act = [eng.round_record(z, dim=dim) for _ in range(R)]
        outs.append((eng.report(), act))
        eng.close()
    torch.cuda.synchronize()
    (init_a, dist_a, drift_a), act_a = outs[0]
    (init_b, dist_b, drift_b), act_b = outs[1]
    assert act_a == act_b
    assert bits_equal(np.array(dist_a), np.array(dist_b))
    assert bits_equal(np.array(drift_a), np.array(drift_b))
    assert torch.equal(x, y)
    want = mb.run_moshpit(mb.GridConfig(M, d, 1), host, mb.FailureModel(p), mb.Rng(7), R,
                          diagnostics=diag, return_vectors=True)
    assert bits_equal(np.array([init_a]), np.array([want.initial_distortion]))
    assert bits_equal(np.array(dist_a), np.array(want.distortion))
    assert bits_equal(np.array(drift_a), np.array(want.mean_drift))
    assert bits_equal(np.ascontiguousarray(x[:, :dim].cpu().numpy()), want.vectors)


@pytest.mark.parametrize("diag", ["fast", "exact"])
def test_engine_record_exact_column_sums_fallback(mb, torch, diag):
    """fp32 column means by exact sums of the distinct rows (launch_colmean_
    exactsum) equal the reference tree's bits: columns whose exponent range
    fits take the exact sum, columns spanning 40 binades, tiny/huge mixes and
    subnormals take the tree (the fallback list) -- all against run_moshpit's
    tree on host buffers."""
    M, d, n, p, R, dim = 32, 2, 1024, 0.01, 3, 1000
    x = torch.zeros((n, dim), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED, dim=dim)
    i = torch.arange(n, device="cuda", dtype=torch.float32)
    x[:, 5] *= torch.pow(2.0, (i % 40) - 20)          # 40 binades: tree
    x[:, 6] = torch.where(i % 97 == 0, x[:, 6] * 1e-30, x[:, 6])  # tiny among O(1): tree
    x[:, 7] = torch.where(i % 13 == 0, x[:, 7] * 1e-40, x[:, 7])  # subnormals: tree
    x[:, 8] *= torch.pow(2.0, (i % 8) - 4)            # 8 binades: exact sum
    host = np.ascontiguousarray(x.cpu().numpy())
    eng = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    eng.set_reference(x, diagnostics=diag, dim=dim)
    eng.rounds_record(x, R, dim=dim)
    init_a, dist_a, drift_a = eng.report()
    eng.close()
    torch.cuda.synchronize()
    want = mb.run_moshpit(mb.GridConfig(M, d, 1), host, mb.FailureModel(p), mb.Rng(7), R,
                          diagnostics=diag, return_vectors=True)
    assert bits_equal(np.array(dist_a), np.array(want.distortion))
    assert bits_equal(np.array(drift_a), np.array(want.mean_drift))
    assert bits_equal(np.ascontiguousarray(x.cpu().numpy()), want.vectors)
