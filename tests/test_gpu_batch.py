"""Trial-batched run_moshpit: a batch of trials must equal,
report by report and bit for bit, the unmodified reference harness's
run_trial (harness.hpp:157-189) for the Moshpit protocol."""
import os

import numpy as np
import pytest

from tests._util import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device(mb):
    if mb.device_count() == 0:
        pytest.fail("no CUDA device visible")


@pytest.fixture(scope="module")
def refh():
    from oracle.oracle import REF_HARNESS_SO, RefHarness
    if not os.path.exists(REF_HARNESS_SO):
        pytest.skip("reference harness shim not built")
    return RefHarness()


def harness_initial(mb, seed, n, dim, init):
    s = mb.Rng(seed).stream("init")
    if init == "normal":
        return np.array([s.normals(dim) for _ in range(n)])
    return np.array([[s.uniform() for _ in range(dim)] for _ in range(n)])


@pytest.mark.parametrize("n,p,dim,init", [(1024, 0.0, 1, "uniform"), (768, 0.005, 1, "uniform"),
                                          (900, 0.01, 2, "normal"), (512, 0.001, 1, "uniform")])
def test_batch_equals_reference_harness(mb, refh, n, p, dim, init):
    grid, seeds_idx, cap = mb.GridConfig(32, 2, 1), range(6), 50
    seeds = [mb.trial_seed(0, "moshpit", n, p, k) for k in seeds_idx]
    assert seeds == [refh.trial_seed(0, n, p, k) for k in seeds_idx]
    x = np.stack([harness_initial(mb, s, n, dim, init) for s in seeds])
    reps = mb.run_moshpit_batch(grid, x, mb.FailureModel(p), seeds, cap)
    for k, rep in zip(seeds_idx, reps):
        want = refh.run_trial(0, n, p, k, 32, 2, dim, init, cap)
        assert rep.initial_distortion == want["initial_distortion"]
        assert bits_equal(np.array(rep.distortion), want["distortion"])
        assert bits_equal(np.array(rep.mean_drift), want["mean_drift"])
        assert rep.active_counts == want["active_counts"].tolist()


# (n, R): blocks of 4 rounds hold n*rounds draws per stream; >= 512 take the
# lane-parallel jump-ahead draws, fewer the serial chain.  (130, 9) mixes
# both in one call (520, 520, then 130 draws), (100, 3) is serial only.
@pytest.mark.parametrize("n,R", [(500, 7), (130, 9), (100, 3)])
@pytest.mark.parametrize("f64", [False, True])
def test_batch_equals_single_trials(mb, oracle, f64, n, R):
    dt = np.float64 if f64 else np.float32
    M, d, dim, p = 8, 3, 37, 0.05
    seeds = [11, 12, 13, 2**40 + 5, 7]
    x = np.stack([oracle.init_state(1000 + t, n, dim, dtype=dt) for t in range(len(seeds))])
    reps = mb.run_moshpit_batch(mb.GridConfig(M, d, 1), x, mb.FailureModel(p), seeds, R,
                                return_vectors=True)
    for t, s in enumerate(seeds):
        one = mb.run_moshpit(mb.GridConfig(M, d, 1), x[t], mb.FailureModel(p), mb.Rng(s), R,
                             diagnostics="exact", return_vectors=True)
        assert bits_equal(reps[t].vectors, one.vectors)
        assert bits_equal(np.array(reps[t].distortion), np.array(one.distortion))
        assert reps[t].active_counts == one.active_counts


def test_table3_moshpit_rows_reproduce_reference(mb, refh):
    """acceptance.cpp:103-122 on the batch path: N=1024, M=32, p=0 needs
    exactly 2 rounds to 1e-9 on every seed."""
    n, seeds = 1024, [mb.trial_seed(0, "moshpit", 1024, 0.0, k) for k in range(100)]
    x = np.stack([harness_initial(mb, s, n, 1, "uniform") for s in seeds])
    reps = mb.run_moshpit_batch(mb.GridConfig(32, 2, 1), x, mb.FailureModel(0.0), seeds, 50)
    assert all(r.rounds_to(1e-9, 50) == 2 for r in reps)
