"""GPU Moshpit SGD on LogisticRegression (optimizer.hpp:75-146, 231-242,
297-439).

Bars: the summation orders are the reference's, but exp/log1p come from
CUDA's libdevice rather than glibc, which may differ in the last bit for
some arguments.  So fp64 parity is a tolerance: value / gradient within
RTOL_EVAL = 1e-13 relative (per-element, scaled by the vector's max), and
whole SGD runs within RTOL_RUN = 1e-10 of the unmodified reference's golden
vectors (the contraction of a strongly convex problem keeps 1-ulp gradient
differences from growing).  fp32 state: within 1e-4 of the fp64 reference.
Device (Philox) noise: the reference's statistical properties."""
import numpy as np
import pytest

from tests._util import unhex, unhexa

pytestmark = pytest.mark.gpu

RTOL_EVAL = 1e-13
RTOL_RUN = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible")


def _close(a, b, rtol):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = max(np.max(np.abs(b)) if b.size else 0.0, 1e-300)
    return a.shape == b.shape and bool(np.all(np.abs(a - b) <= rtol * scale))


def _lr(mb, c):
    return mb.LogisticRegression.synthetic(c["dim"], c["samples"], c["l2"],
                                           mb.Rng(c["data_seed"]).stream("objective"))


def test_logistic_eval_vs_golden(mb, golden):
    for c in golden["logistic_eval"]:
        lr = _lr(mb, c)
        th = unhexa(c["theta"])
        assert _close([lr.value(th)], [unhex(c["value"])], RTOL_EVAL)
        assert _close(lr.gradient(th), unhexa(c["grad"]), RTOL_EVAL)


def test_logistic_eval_vs_reference_both_tails(mb, ref):
    rng = np.random.default_rng(9)
    for S, dim in [(1, 1), (7, 3), (300, 40), (1000, 5)]:
        xs = rng.normal(size=(S, dim)) * 3
        ys = np.where(rng.random(S) < 0.5, -1.0, 1.0)
        th = rng.normal(size=dim) * 5
        lr = mb.LogisticRegression(xs, ys, 0.05)
        v, g, sm = ref.logistic_eval(xs, ys, 0.05, th)
        assert _close([lr.value(th)], [v], RTOL_EVAL)
        assert _close(lr.gradient(th), g, RTOL_EVAL)
        assert lr.smoothness() == sm


def test_sgd_logistic_f64_vs_golden(mb, golden):
    for c in golden["sgd_logistic"]:
        lr = _lr(mb, c)
        cfg = mb.OptimizerConfig(gamma=c["gamma"], tau=c["tau"], steps=c["steps"],
                                 grid=mb.GridConfig(c["M"], c["d"], 1), sigma=c["sigma"],
                                 n_peers=c["n"])
        r = mb.run_moshpit_sgd(cfg, lr, np.zeros(c["dim"]), [], mb.Rng(c["seed"]))
        for k, got in (("f_gap", r.f_gap), ("grad_norm_sq", r.grad_norm_sq),
                       ("f_gap_weighted", r.f_gap_weighted),
                       ("dispersion", r.diagnostics.dispersion), ("final_mean", r.final_mean)):
            want = unhexa(c[k])
            if k == "final_mean":
                assert _close(got, want, RTOL_RUN), k
                continue
            # per step, relative; squared roundoff-level quantities (dispersion
            # at sigma=0 is ~1e-34) get an absolute floor of (1e-12)^2
            err = np.abs(np.asarray(got) - want)
            assert np.all(err <= RTOL_RUN * np.abs(want) + 1e-24), (k, err.max())
        assert r.diagnostics.sigma_hat == unhex(c["sigma_hat"])  # host noise stream: exact
        assert _close([r.diagnostics.delta_aq_hat], [unhex(c["delta_aq_hat"])], 1e-6)


@pytest.mark.parametrize("M,n,dim,S", [(16, 256, 64, 512), (12, 130, 70, 333)])
def test_sgd_logistic_matches_reference_larger(mb, ref, M, n, dim, S):
    """Larger runs through the tiled step kernels: tile-aligned (N=256 peers
    on 16x16, 64 features, 512 samples) and ragged in every dimension."""
    d, l2 = 2, 0.02
    want = ref.sgd_logistic(M, d, n, dim, S, l2, 41, np.zeros(dim), 0.5, 2, 16, 0.3, 41)
    lr = mb.LogisticRegression.synthetic(dim, S, l2, mb.Rng(41).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=0.5, tau=2, steps=16, grid=mb.GridConfig(M, d, 1), sigma=0.3,
                             n_peers=n)
    r = mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(41))
    assert _close(r.f_gap, want["f_gap"], RTOL_RUN)
    assert _close(r.f_gap_weighted, want["f_gap_weighted"], RTOL_RUN)
    assert _close(r.final_mean, want["final_mean"], RTOL_RUN)
    assert np.all(np.diff(r.f_gap) < 0.05)


def test_sgd_logistic_f32_close_to_reference(mb, golden):
    c = golden["sgd_logistic"][0]
    lr = _lr(mb, c)
    cfg = mb.OptimizerConfig(gamma=c["gamma"], tau=c["tau"], steps=c["steps"],
                             grid=mb.GridConfig(c["M"], c["d"], 1), sigma=c["sigma"],
                             n_peers=c["n"])
    r = mb.run_moshpit_sgd(cfg, lr, np.zeros(c["dim"]), [], mb.Rng(c["seed"]), dtype=np.float32)
    assert _close(r.f_gap, unhexa(c["f_gap"]), 1e-4)
    assert _close(r.final_mean, unhexa(c["final_mean"]), 1e-4)


def test_sgd_logistic_diag_none_same_iterates(mb):
    lr = mb.LogisticRegression.synthetic(10, 80, 0.05, mb.Rng(3).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=0.2, tau=2, steps=12, grid=mb.GridConfig(4, 2, 1), sigma=0.5,
                             n_peers=16)
    a = mb.run_moshpit_sgd(cfg, lr, np.zeros(10), [], mb.Rng(5), diagnostics="none",
                           return_thetas=True)
    b = mb.run_moshpit_sgd(cfg, lr, np.zeros(10), [], mb.Rng(5), return_thetas=True)
    assert np.array_equal(a.final_thetas, b.final_thetas)
    assert np.array_equal(a.final_mean, b.final_mean)
    assert np.isnan(a.f_gap).all() and not np.isnan(b.f_gap).any()
    assert a.diagnostics.sigma_hat == b.diagnostics.sigma_hat


@pytest.mark.parametrize("dtype", [np.float64, np.float32])  # fp32: the tensor-core path
def test_sgd_logistic_device_noise_statistics(mb, dtype):
    """Philox noise: sigma_hat ~ sigma (test_optimizer.cpp's sigma check),
    loss decreases, peers agree after averaging."""
    lr = mb.LogisticRegression.synthetic(32, 256, 0.05, mb.Rng(8).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=0.3, tau=1, steps=40, grid=mb.GridConfig(8, 2, 1), sigma=1.0,
                             n_peers=64)
    r = mb.run_moshpit_sgd(cfg, lr, np.zeros(32), [], mb.Rng(2), noise="device", dtype=dtype)
    assert abs(r.diagnostics.sigma_hat - 1.0) < 0.05
    assert r.f_gap[-1] < r.f_gap[0]
    f0 = lr.value(np.zeros(32))
    assert r.f_gap[-1] < f0


def test_sgd_logistic_membership_schedule(mb):
    lr = mb.LogisticRegression.synthetic(6, 40, 0.1, mb.Rng(4).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=0.2, tau=1, steps=15, grid=mb.GridConfig(4, 2, 1), sigma=0.2,
                             n_peers=12)
    sched = [mb.MembershipEvent(3, -5), mb.MembershipEvent(8, 4)]
    r = mb.run_moshpit_sgd(cfg, lr, np.zeros(6), sched, mb.Rng(6), return_thetas=True)
    assert r.diagnostics.n_min == 7
    assert r.final_thetas.shape == (11, 6)
    assert np.all(np.isfinite(r.f_gap))


def test_local_step_logistic_vs_oracle(mb, oracle):
    xs, ys = oracle.logistic_dataset(5, 30, 77)
    lr = mb.LogisticRegression(xs, ys, 0.1)
    th = np.linspace(-1, 1, 5)
    _, g, _ = oracle.logistic_eval(xs, ys, 0.1, th)
    want = th - 0.25 * g
    got = mb.local_step(th.copy(), lr, 0.25, 0.0, mb.Rng(1).stream("noise"))
    assert _close(got, want, RTOL_EVAL)
    # with noise: the stream advances exactly as the reference's (dim normals)
    s1, s2 = mb.Rng(2).stream("noise"), mb.Rng(2).stream("noise")
    got = mb.local_step(th.copy(), lr, 0.25, 1.0, s1)
    nz = np.array([s2.normal() for _ in range(5)]) * (1.0 / np.sqrt(5))
    assert _close(got, th - 0.25 * (g + nz), RTOL_EVAL)
    assert s1() == s2()


def test_logistic_errors(mb):
    lr = mb.LogisticRegression(np.ones((2, 3)), [1.0, -1.0], 0.1)
    cfg = mb.OptimizerConfig(gamma=0.1, steps=2, grid=mb.GridConfig(4, 2, 1), n_peers=4)
    with pytest.raises(ValueError):
        mb.run_moshpit_sgd(cfg, lr, np.zeros(2), [], mb.Rng(1))
    with pytest.raises(ValueError):
        mb.run_moshpit_sgd(mb.OptimizerConfig(gamma=0.0, n_peers=4), lr, np.zeros(3), [],
                           mb.Rng(1))
    bad = mb.LogisticRegression(np.array([[1.0]]), [1.0], 0.0)
    with pytest.raises(mb.MoshpitError):  # non-finite gradient -> runtime_error (:368-369)
        mb.run_moshpit_sgd(mb.OptimizerConfig(gamma=0.1, steps=3, grid=mb.GridConfig(2, 1, 1),
                                              n_peers=1), bad, np.array([np.nan]), [], mb.Rng(1))


def test_logistic_gradient_matches_finite_differences(mb):
    """test_optimizer.cpp:30-44 / acceptance.cpp criterion 9(d): the GPU
    gradient agrees with central differences of the GPU value at 1e-6."""
    stream = mb.Rng(21).stream("theta")
    stream.normals(6)
    lr = mb.LogisticRegression.synthetic(5, 80, 0.05, stream)
    for _ in range(10):
        th = stream.normals(5)
        g = lr.gradient(th)
        for j in range(5):
            h = 1e-6 * max(1.0, abs(th[j]))
            lo, hi = th.copy(), th.copy()
            lo[j] -= h
            hi[j] += h
            fd = (lr.value(hi) - lr.value(lo)) / (2.0 * h)
            assert abs(g[j] - fd) / max(abs(g[j]), abs(fd), 1e-8) <= 1e-6


def test_sgd_logistic_fast_diagnostics(mb, golden):
    """FAST differs from EXACT only in the dispersion's summation order."""
    c = golden["sgd_logistic"][1]
    lr = _lr(mb, c)
    cfg = mb.OptimizerConfig(gamma=c["gamma"], tau=c["tau"], steps=c["steps"],
                             grid=mb.GridConfig(c["M"], c["d"], 1), sigma=c["sigma"],
                             n_peers=c["n"])
    a = mb.run_moshpit_sgd(cfg, lr, np.zeros(c["dim"]), [], mb.Rng(c["seed"]), diagnostics="fast")
    b = mb.run_moshpit_sgd(cfg, lr, np.zeros(c["dim"]), [], mb.Rng(c["seed"]))
    assert np.array_equal(a.f_gap, b.f_gap) and np.array_equal(a.final_mean, b.final_mean)
    assert np.array_equal(a.f_gap_weighted, b.f_gap_weighted)
    d_a, d_b = np.array(a.diagnostics.dispersion), np.array(b.diagnostics.dispersion)
    assert np.all(np.abs(d_a - d_b) <= 1e-12 * np.abs(d_b) + 1e-30)


@pytest.mark.parametrize("sigma", [0.0, 0.5])
def test_sgd_logistic_f32_tensor_cores(mb, monkeypatch, sigma):
    """fp32 state: the two GEMMs of the logistic step run on tcgen05 (kind::tf32,
    3xTF32 split; tc_logit.cu).  Same run with the tensor cores off (the fp64
    SIMT kernels on the fp32 state) and with fp64 state: fp32-level agreement
    (north_star: 1e-6 relative per step; over the run's steps the fp32
    iterates drift further, so the run is checked at 1e-4 against fp64)."""
    dim, S, n = 256, 512, 256
    lr = mb.LogisticRegression.synthetic(dim, S, 0.05, mb.Rng(11).stream("objective"))
    cfg = mb.OptimizerConfig(gamma=0.5, tau=1, steps=6, grid=mb.GridConfig(16, 2, 1),
                             sigma=sigma, n_peers=n)
    run = lambda dt: mb.run_moshpit_sgd(cfg, lr, np.zeros(dim), [], mb.Rng(5), dtype=dt,
                                        return_thetas=True)
    monkeypatch.setenv("MOSHPIT_LOGIT_TC", "1")
    tc = run(np.float32)
    monkeypatch.setenv("MOSHPIT_LOGIT_TC", "0")
    simt = run(np.float32)
    f64 = run(np.float64)
    scale = np.abs(f64.final_thetas).max()
    assert np.abs(tc.final_thetas - simt.final_thetas).max() <= 2e-5 * scale
    assert np.abs(tc.final_thetas - f64.final_thetas).max() <= 1e-4 * scale
    assert _close(tc.f_gap, f64.f_gap, 1e-4)
    assert not np.array_equal(tc.final_thetas, simt.final_thetas)  # a different kernel ran


def test_local_step_logistic_tensor_cores_one_step(mb, oracle, monkeypatch):
    """One fp32 local step of 256 peers on the tensor cores vs the fp64
    reference gradient (the oracle): within fp32 rounding (1e-6 relative)."""
    import torch  # noqa: F401
    dim, S, n = 128, 256, 256
    xs, ys = oracle.logistic_dataset(dim, S, 91)
    lr = mb.LogisticRegression(xs, ys, 0.1)
    rng = np.random.default_rng(3)
    th = rng.normal(size=(n, dim)) * 0.1
    monkeypatch.setenv("MOSHPIT_LOGIT_TC", "1")
    cfg = mb.OptimizerConfig(gamma=0.25, tau=1000, steps=1, grid=mb.GridConfig(16, 2, 1),
                             sigma=0.0, n_peers=n)
    # one step with no averaging (tau > steps): theta_1 = theta_0 - gamma grad(theta_0)
    r = mb.run_moshpit_sgd(cfg, lr, th[0], [], mb.Rng(1), dtype=np.float32, return_thetas=True,
                           diagnostics="none")
    _, g, _ = oracle.logistic_eval(xs, ys, 0.1, th[0])
    want = th[0] - 0.25 * g
    got = r.final_thetas[0]
    assert np.abs(got - want).max() <= 1e-6 * max(1.0, np.abs(want).max())
