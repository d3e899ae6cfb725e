"""GPU Moshpit SGD (optimizer.hpp:231-242, 297-439, Quadratic objective).

Bars: fp64 + reference noise stream + EXACT diagnostics -> bit-identical to
the reference (golden vectors and oracle/_ref); fp32 -> bit-identical to the
fp32 restatement; FAST diagnostics within 1e-12 relative; device (Philox)
noise -> the reference's own statistical properties (test_optimizer.cpp)."""
import numpy as np
import pytest

from tests._util import bits_equal, unhex, unhexa

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible")


def _cfg(mb, c):
    cfg = mb.OptimizerConfig(gamma=c["gamma"], tau=c["tau"], steps=c["steps"],
                             grid=mb.GridConfig(c["M"], c["d"], 1), sigma=c["sigma"],
                             n_peers=c["n"])
    quad = mb.Quadratic(c["dim"], c["L"], c["mu"], unhexa(c["target"]))
    sched = [mb.MembershipEvent(s, dd) for s, dd in c["schedule"]]
    return cfg, quad, sched


def test_sgd_f64_bit_exact_vs_golden(mb, golden):
    for c in golden["sgd_quadratic"]:
        cfg, quad, sched = _cfg(mb, c)
        r = mb.run_moshpit_sgd(cfg, quad, np.zeros(c["dim"]), sched, mb.Rng(c["seed"]))
        assert bits_equal(np.array(r.f_gap), unhexa(c["f_gap"])), c["seed"]
        assert bits_equal(np.array(r.grad_norm_sq), unhexa(c["grad_norm_sq"]))
        assert bits_equal(np.array(r.f_gap_weighted), unhexa(c["f_gap_weighted"]))
        assert bits_equal(np.array(r.diagnostics.dispersion), unhexa(c["dispersion"]))
        assert bits_equal(r.final_mean, unhexa(c["final_mean"]))
        assert r.diagnostics.delta_aq_hat == unhex(c["delta_aq_hat"])
        assert r.diagnostics.sigma_hat == unhex(c["sigma_hat"])
        assert r.diagnostics.delta_pv2_hat == unhex(c["delta_pv2_hat"])
        assert r.diagnostics.n_min == c["n_min"]


def test_local_step_matches_golden(mb, golden):
    for c in golden["local_step"]:
        th = np.array(c["theta"], dtype=np.float64)
        quad = mb.Quadratic(c["dim"], c["L"], c["mu"], c["target"])
        s = mb.Rng(c["seed"]).stream(c["name"])
        mb.local_step(th, quad, c["gamma"], c["sigma"], s)
        assert bits_equal(th, unhexa(c["out"]))
    # test_optimizer.cpp:60-69
    th = np.zeros(2)
    mb.local_step(th, mb.Quadratic(2, 2.0, 2.0, [1.0, 1.0]), 0.25, 0.0, mb.Rng(23).stream("n"))
    assert th.tolist() == [0.5, 0.5]


@pytest.mark.parametrize("sigma,tau,sched", [(0.0, 1, ()), (1.0, 3, ()),
                                             (0.5, 2, ((5, -3), (12, 2)))])
def test_sgd_f32_bit_exact_vs_oracle(mb, oracle, sigma, tau, sched):
    dim, n = 37, 12
    tgt = oracle.stream_draws(11, "objective", dim, "normal")
    res = oracle.sgd_quadratic(4, 2, n, dim, 2.0, 0.5, tgt, np.zeros(dim), 0.05, tau, 20, sigma,
                               99, schedule=sched, dtype=np.float32)
    cfg = mb.OptimizerConfig(gamma=0.05, tau=tau, steps=20, grid=mb.GridConfig(4, 2, 1),
                             sigma=sigma, n_peers=n)
    r = mb.run_moshpit_sgd(cfg, mb.Quadratic(dim, 2.0, 0.5, tgt), np.zeros(dim),
                           [mb.MembershipEvent(*e) for e in sched], mb.Rng(99), dtype=np.float32,
                           return_thetas=True)
    assert bits_equal(r.final_thetas, res["final_thetas"])
    assert bits_equal(np.array(r.f_gap), res["f_gap"])
    assert bits_equal(np.array(r.diagnostics.dispersion), res["dispersion"])
    fast = mb.run_moshpit_sgd(cfg, mb.Quadratic(dim, 2.0, 0.5, tgt), np.zeros(dim),
                              [mb.MembershipEvent(*e) for e in sched], mb.Rng(99),
                              dtype=np.float32, diagnostics="fast")
    np.testing.assert_allclose(fast.f_gap, res["f_gap"], rtol=1e-12)
    np.testing.assert_allclose(fast.diagnostics.dispersion, res["dispersion"], rtol=1e-12,
                               atol=1e-300)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n,M,tau,sched", [(64, 8, 1, ()), (32, 8, 2, ()), (256, 16, 1, ()),
                                           (64, 8, 1, ((5, -32), (9, 32)))])
def test_sgd_diagnostics_fused_paths_vs_oracle(mb, oracle, dt, n, M, tau, sched):
    """n = 8 * 2^K peers with 16-byte rows: the noise-free step fused into the
    post-step mean (hat theta) and the representative-row mean / dispersion
    after each averaging pass -- EXACT diagnostics bit-exact vs the oracle,
    FAST within its tolerance (membership events take n off the power of 2
    and back)."""
    dim = 40
    tgt = oracle.stream_draws(11, "objective", dim, "normal")
    res = oracle.sgd_quadratic(M, 2, n, dim, 2.0, 0.5, tgt, np.zeros(dim), 0.05, tau, 16, 0.0,
                               99, schedule=sched, dtype=dt)
    cfg = mb.OptimizerConfig(gamma=0.05, tau=tau, steps=16, grid=mb.GridConfig(M, 2, 1),
                             sigma=0.0, n_peers=n)
    ev = [mb.MembershipEvent(*e) for e in sched]
    r = mb.run_moshpit_sgd(cfg, mb.Quadratic(dim, 2.0, 0.5, tgt), np.zeros(dim), ev, mb.Rng(99),
                           dtype=dt, return_thetas=True)
    assert bits_equal(r.final_thetas, res["final_thetas"])
    assert bits_equal(np.array(r.f_gap), res["f_gap"])
    assert bits_equal(np.array(r.grad_norm_sq), res["grad_norm_sq"])
    assert bits_equal(np.array(r.diagnostics.dispersion), res["dispersion"])
    fast = mb.run_moshpit_sgd(cfg, mb.Quadratic(dim, 2.0, 0.5, tgt), np.zeros(dim), ev,
                              mb.Rng(99), dtype=dt, diagnostics="fast", return_thetas=True)
    assert bits_equal(fast.final_thetas, res["final_thetas"])
    np.testing.assert_allclose(fast.f_gap, res["f_gap"], rtol=1e-12)
    np.testing.assert_allclose(fast.diagnostics.dispersion, res["dispersion"], rtol=1e-12,
                               atol=1e-300)


def test_sgd_validation_matches_reference(mb):
    quad = mb.Quadratic(2, 2.0, 1.0, [1.0, 1.0])
    cfg = mb.OptimizerConfig(gamma=0.1, tau=2, steps=20, grid=mb.GridConfig(4, 2, 1), sigma=0.5,
                             n_peers=8)
    r = mb.run_moshpit_sgd(cfg, quad, np.zeros(2), [mb.MembershipEvent(5, -3),
                                                    mb.MembershipEvent(12, 2)], mb.Rng(777))
    assert r.diagnostics.n_min == 5 and len(r.f_gap) == 20   # test_optimizer.cpp:160-176
    with pytest.raises(ValueError):                            # :177-180
        mb.run_moshpit_sgd(cfg, quad, np.zeros(2), [mb.MembershipEvent(3, -8)], mb.Rng(1))
    with pytest.raises(ValueError):
        mb.Quadratic(2, 1.0, 2.0, [0.0, 0.0])
    bad = mb.OptimizerConfig(gamma=0.0, grid=mb.GridConfig(2, 2, 1), n_peers=4)
    with pytest.raises(ValueError):
        mb.run_moshpit_sgd(bad, quad, np.zeros(2), [], mb.Rng(1))
    with pytest.raises(mb.ReferenceRuntimeError):  # non-finite gradient
        huge = mb.Quadratic(2, 1e308, 1e308, [0.0, 0.0])
        c2 = mb.OptimizerConfig(gamma=1e10, steps=3, grid=mb.GridConfig(2, 2, 1), n_peers=4)
        mb.run_moshpit_sgd(c2, huge, np.full(2, 1e300), [], mb.Rng(1))


def test_tau1_sigma0_equals_gradient_descent(mb):
    # test_optimizer.cpp:71-98
    s = mb.Rng(24).stream("target")
    quad = mb.Quadratic(4, 5.0, 0.5, s.normals(4))
    cfg = mb.OptimizerConfig(gamma=0.05, tau=1, steps=60, grid=mb.GridConfig(4, 2, 1),
                             sigma=0.0, n_peers=9)
    r = mb.run_moshpit_sgd(cfg, quad, np.full(4, 2.0), [], mb.Rng(500), noise="device")
    c = np.array([0.5 + 4.5 * j / 3 for j in range(4)])
    th = np.full(4, 2.0)
    for k in range(60):
        th = th - 0.05 * (c * (th - quad.target))
        f = float(np.sum(0.5 * c * (th - quad.target) ** 2))
        assert abs(r.f_gap[k] - f) <= 1e-12
        assert r.diagnostics.dispersion[k] <= 1e-24
    assert np.allclose(r.final_mean, th, atol=1e-12)


def test_device_noise_statistics(mb):
    """Philox noise: sigma_hat ~ sigma, and the reference's V_k bound
    (test_optimizer.cpp:100-130) and N-doubling property (:132-158)."""
    cfg = mb.OptimizerConfig(gamma=0.02, tau=4, steps=80, grid=mb.GridConfig(4, 2, 1), sigma=1.0,
                             n_peers=12)
    quad = mb.Quadratic(3, 10.0, 1.0, np.ones(3))
    n_seeds = 60
    mean_vk = np.zeros(80)
    worst_aq, sigma_hat = 0.0, 0.0
    for s in range(n_seeds):
        r = mb.run_moshpit_sgd(cfg, quad, np.zeros(3), [], mb.Rng(8000 + s), noise="device",
                               diagnostics="fast")
        mean_vk += np.array(r.diagnostics.dispersion) / n_seeds
        worst_aq = max(worst_aq, r.diagnostics.delta_aq_hat)
        sigma_hat += r.diagnostics.sigma_hat / n_seeds
    assert abs(sigma_hat - 1.0) < 0.1
    bound = 2 * 0.02 ** 2 * (4 * worst_aq ** 2 + 3 * sigma_hat ** 2)
    assert (mean_vk <= 1.5 * bound).all()

    def steady(n_peers):
        c = mb.OptimizerConfig(gamma=0.05, tau=1, steps=200, grid=mb.GridConfig(8, 2, 1),
                               sigma=1.0, n_peers=n_peers)
        q = mb.Quadratic(2, 4.0, 1.0, np.full(2, 0.5))
        acc = 0.0
        for s in range(30):
            r = mb.run_moshpit_sgd(c, q, np.zeros(2), [], mb.Rng(9000 + s), noise="device",
                                   diagnostics="fast")
            acc += float(np.mean(r.f_gap[150:]))
        return acc / 30
    assert steady(16) < steady(8)


@pytest.mark.slow
def test_c4_shaped_run_device_noise(mb):
    """C4: 1024 peers on 32x32, Quadratic(D=2^16, L=1, mu=0.1), gamma=0.1,
    tau=1, sigma=1, device noise, FAST diagnostics: converges and stays
    consistent (dispersion after exact 2-round averaging ~ fp rounding)."""
    D = 1 << 16
    s = mb.Rng(7).stream("objective")
    quad = mb.Quadratic(D, 1.0, 0.1, s.normals(D))
    cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=20, grid=mb.GridConfig(32, 2, 1), sigma=1.0,
                             n_peers=1024)
    r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(7), noise="device",
                           diagnostics="fast", dtype=np.float32)
    assert r.f_gap[-1] < 0.5 * r.f_gap[0]
    assert max(r.diagnostics.dispersion) < 1e-9  # full grid, tau=1: exact average each step
    assert abs(r.diagnostics.sigma_hat - 1.0) < 0.01


@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("sigma,tau,M,d,n", [(0.0, 1, 4, 2, 16), (1.0, 1, 8, 2, 64),
                                             (0.7, 3, 4, 3, 50), (1.0, 1, 40, 2, 1600),
                                             # groups of 7 / 13 / <= 31: whole 4-member
                                             # batches (interleaved Philox) + partial ones
                                             (1.0, 1, 7, 2, 49), (1.0, 1, 13, 2, 150),
                                             (0.5, 2, 31, 2, 900)])
def test_fused_kernel3_equals_unfused(mb, f64, sigma, tau, M, d, n):
    """Kernel 3 (local step fused into averaging round 1) == step kernel +
    averaging, bit for bit, with the same device noise."""
    dim = 45
    tgt = mb.Rng(3).stream("objective").normals(dim)
    cfg = mb.OptimizerConfig(gamma=0.05, tau=tau, steps=12, grid=mb.GridConfig(M, d, 1),
                             sigma=sigma, n_peers=n)
    quad = mb.Quadratic(dim, 2.0, 0.2, tgt)
    dt = np.float64 if f64 else np.float32
    a = mb.run_moshpit_sgd(cfg, quad, np.zeros(dim), [], mb.Rng(5), dtype=dt, noise="device",
                           diagnostics="none", return_thetas=True)
    b = mb.run_moshpit_sgd(cfg, quad, np.zeros(dim), [], mb.Rng(5), dtype=dt, noise="device",
                           diagnostics="fast", return_thetas=True)
    assert bits_equal(a.final_thetas, b.final_thetas)
    assert bits_equal(a.final_mean, b.final_mean)
    assert np.isnan(a.f_gap).all()
    if sigma > 0:
        assert abs(a.diagnostics.sigma_hat - b.diagnostics.sigma_hat) <= 1e-9 * b.diagnostics.sigma_hat


@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("sigma,tau,M,n,dim,sched", [
    (1.0, 1, 32, 1024, 1029, []),                  # C4-shaped: 32 groups of 32
    (0.0, 1, 32, 1024, 64, []),
    (1.0, 2, 8, 64, 45, [(3, -5), (7, 2)]),        # partial grids after membership events
    (0.7, 1, 13, 150, 37, [(4, 9)]),               # groups of 13 / ragged lines
    (1.0, 1, 31, 900, 18, [(2, -100), (9, 61)]),   # leaves of 7-8 members, 4-member batches
    (1.0, 3, 5, 25, 9, []),
])
def test_two_round_pass_equals_kernel3_plus_kernel2(mb, monkeypatch, f64, sigma, tau, M, n,
                                                    dim, sched):
    """The SGD averaging step with two rounds in ONE pass over the state
    (step + round 1 into shared memory, round 2 from there; the default for
    d = 2, M <= 32) is bit-identical to kernel 3 + kernel 2
    (MOSHPIT_SGD_TWO_ROUND=0), device noise included."""
    tgt = mb.Rng(3).stream("objective").normals(dim)
    cfg = mb.OptimizerConfig(gamma=0.05, tau=tau, steps=9, grid=mb.GridConfig(M, 2, 1),
                             sigma=sigma, n_peers=n)
    quad = mb.Quadratic(dim, 2.0, 0.2, tgt)
    dt = np.float64 if f64 else np.float32
    ev = [mb.MembershipEvent(*e) for e in sched]
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("MOSHPIT_SGD_TWO_ROUND", flag)
        outs.append(mb.run_moshpit_sgd(cfg, quad, np.zeros(dim), ev, mb.Rng(5), dtype=dt,
                                       noise="device", diagnostics="none", return_thetas=True))
    a, b = outs
    assert bits_equal(a.final_thetas, b.final_thetas)
    assert bits_equal(a.final_mean, b.final_mean)
    if sigma > 0:
        assert abs(a.diagnostics.sigma_hat - b.diagnostics.sigma_hat) <= 1e-9 * b.diagnostics.sigma_hat
