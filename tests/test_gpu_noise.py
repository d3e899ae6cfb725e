"""Device (Philox) noise: the normals every device-noise kernel adds
(coordinate j of peer i at step k; csrc/philox.cuh) are standard normal and
independent across coordinates, pairs and peers.  The fused kernel 3 draws
the same normals bit for bit (test_gpu_sgd.py::test_fused_kernel3_equals_unfused);
here the standalone step exposes them: Quadratic(L = mu = 0) has zero
gradient, so one local step from theta = 0 with gamma = 1 and
sigma = sqrt(D) (coord_std = 1) leaves theta = -z exactly."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _normals(mb, n, D, dtype, seed=11):
    quad = mb.Quadratic(D, 0.0, 0.0, np.zeros(D))
    cfg = mb.OptimizerConfig(gamma=1.0, tau=2, steps=1, grid=mb.GridConfig(8, 2, 1),
                             sigma=math.sqrt(D), n_peers=n)
    r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(seed), dtype=dtype,
                           noise="device", diagnostics="none", return_thetas=True)
    return -np.asarray(r.final_thetas, dtype=np.float64)


@pytest.fixture(scope="module")
def z32(mb):
    return _normals(mb, 64, 1 << 16, np.float32)


def test_noise_is_standard_normal(z32):
    from scipy.special import ndtr
    z = z32.ravel()
    N = z.size
    assert abs(z.mean()) < 5 / math.sqrt(N)
    assert abs(z.var() - 1) < 5 * math.sqrt(2 / N)
    sk = np.mean(z ** 3)
    ku = np.mean(z ** 4)
    assert abs(sk) < 5 * math.sqrt(6 / N)
    assert abs(ku - 3) < 5 * math.sqrt(96 / N)
    zs = np.sort(z)
    cdf = ndtr(zs)
    ks = max(np.max(np.arange(1, N + 1) / N - cdf), np.max(cdf - np.arange(N) / N))
    assert ks < 2.0 / math.sqrt(N)
    # tails: P(|z| > 3) = 2.70e-3, P(|z| > 4) = 6.33e-5; radius cut at
    # sqrt(48 ln 2) = 5.77 (24-bit radius draws)
    for thr, p in ((3.0, 2.6998e-3), (4.0, 6.3342e-5)):
        c = int(np.sum(np.abs(z) > thr))
        assert abs(c - N * p) < 5 * math.sqrt(N * p) + 1
    assert 4.5 < np.abs(z).max() <= 5.78


def test_noise_pairs_and_neighbours_independent(z32):
    z = z32
    N = z.size
    tol = 5 / math.sqrt(N)
    flat = z.ravel()
    for lag in (1, 2, 3, 4, 8):  # within a Box-Muller pair (1), a Philox quad, across
        a, b = flat[:-lag], flat[lag:]
        assert abs(np.mean(a * b)) < tol * 1.5, lag
    # across peers at the same coordinate
    assert abs(np.mean(z[:-1] * z[1:])) < tol * 1.5
    # Box-Muller pairs: r^2 ~ Exp(mean 2), the angle uniform
    p = flat.reshape(-1, 2)
    r2 = p[:, 0] ** 2 + p[:, 1] ** 2
    M = r2.size
    assert abs(r2.mean() - 2) < 5 * 2 / math.sqrt(M)
    f = np.mean(r2 > 10.0)
    assert abs(f - math.exp(-5)) < 5 * math.sqrt(math.exp(-5) / M)
    ang = np.arctan2(p[:, 1], p[:, 0])
    h, _ = np.histogram(ang, bins=32, range=(-math.pi, math.pi))
    chi2 = float(np.sum((h - M / 32) ** 2 / (M / 32)))
    assert chi2 < 31 + 5 * math.sqrt(62)


def test_noise_same_normals_in_both_precisions(mb, z32):
    """The fp64 state draws the same float normals (then scales them in fp64)."""
    z64 = _normals(mb, 64, 1 << 16, np.float64)
    assert np.array_equal(z64, z32)


def test_noise_depends_on_seed_step_and_peer(mb, z32):
    other = _normals(mb, 64, 1 << 16, np.float32, seed=12)
    assert np.mean(other == z32) < 1e-3
    assert np.mean(z32[0] == z32[1]) < 1e-3
