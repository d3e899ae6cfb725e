"""Temporal blocking (fused_rounds.cu, SURVEY 8d "run_rounds_fused"): R rounds
-- and, in Moshpit SGD, the local step before them -- in one pass over the
state must give the same bits as the per-round path."""
import numpy as np
import pytest

from tests._util import INIT_SEED, bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("M,d,n,p,R,dim", [(32, 2, 1024, 0.01, 10, 1000),
                                           (16, 2, 256, 0.05, 7, 37),
                                           (8, 3, 512, 0.02, 12, 4099),
                                           (5, 2, 24, 0.1, 10, 3),
                                           (40, 2, 1600, 0.02, 4, 70),
                                           (32, 2, 1000, 0.0, 3, 16)])
def test_rounds_fused_equals_per_round(mb, oracle, torch, M, d, n, p, R, dim, f64):
    """Groups of 5..40 (the leaf form and the runtime tree), voided groups,
    partial grids, column tails, chunked passes (n = 1600: one round per
    pass), fp32 and fp64; against R engine rounds and the oracle."""
    dt = torch.float64 if f64 else torch.float32
    ld = (dim + 3) // 4 * 4 + 4
    x0 = torch.empty((n, ld), dtype=dt, device="cuda")
    mb.fill_synthetic(x0, INIT_SEED, dim=dim)
    a, b = x0.clone(), x0.clone()
    e1 = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    act1 = [e1.round(a, dim=dim) for _ in range(R)]
    e2 = mb.Engine(mb.GridConfig(M, d, R), n, mb.FailureModel(p), mb.Rng(7), device=0)
    act2 = e2.rounds_fused(b, R, dim=dim)
    torch.cuda.synchronize()
    assert act1 == act2
    assert bits_equal(a[:, :dim].cpu().numpy(), b[:, :dim].cpu().numpy())
    init = oracle.init_state(INIT_SEED, n, dim, dtype=np.float64 if f64 else np.float32)
    _, want = oracle.run_moshpit(M, d, init, p, 7, R)
    assert bits_equal(b[:, :dim].cpu().numpy(), want)
    e1.close()
    e2.close()


def test_rounds_fused_refuses_too_many_peers(mb, torch):
    x = torch.zeros((4096, 8), dtype=torch.float32, device="cuda")
    e = mb.Engine(mb.GridConfig(16, 3, 1), 4096, mb.FailureModel(), mb.Rng(1), device=0)
    with pytest.raises(mb.InvalidArgument):
        e.rounds_fused(x, 1)
    e.close()


@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("sigma,tau,M,n,dim", [(0.0, 1, 8, 64, 45), (1.0, 1, 8, 64, 45),
                                               (1.0, 2, 32, 1024, 1003), (0.7, 1, 13, 150, 16),
                                               (0.5, 1, 40, 1600, 12)])
def test_sgd_fused_rounds_equal_kernel3(mb, monkeypatch, f64, sigma, tau, M, n, dim):
    """Moshpit SGD without diagnostics: the step + both inner rounds in one
    pass == kernel 3 (step + round 1) + kernel 2 (round 2), same device noise."""
    tgt = mb.Rng(3).stream("objective").normals(dim)
    cfg = mb.OptimizerConfig(gamma=0.05, tau=tau, steps=6, grid=mb.GridConfig(M, 2, 1),
                             sigma=sigma, n_peers=n)
    quad = mb.Quadratic(dim, 2.0, 0.2, tgt)
    dt = np.float64 if f64 else np.float32
    runs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("MOSHPIT_SGD_FUSED_ROUNDS", fused)
        runs.append(mb.run_moshpit_sgd(cfg, quad, np.zeros(dim), [], mb.Rng(5), dtype=dt,
                                       noise="device", diagnostics="none", return_thetas=True))
    a, b = runs
    assert bits_equal(a.final_thetas, b.final_thetas)
    assert bits_equal(a.final_mean, b.final_mean)
    if sigma > 0:
        assert abs(a.diagnostics.sigma_hat - b.diagnostics.sigma_hat) <= 1e-9 * b.diagnostics.sigma_hat
