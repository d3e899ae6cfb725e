"""CPU: the C-ABI library loads, exports every declared symbol, and its host
logic (RNG, key arithmetic, validation with the reference's error classes)
matches the reference -- no compute call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests._util import bits_equal, unhexa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "moshpit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moshpit_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(mb):
    lib = mb.lib()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding prototypes cover the same set
    from paper_2103_03239_b200 import _capi
    assert sorted(_capi.PROTOTYPES) == names


def test_library_is_sm100a(mb):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", mb._capi.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_rng_matches_golden(mb, golden):
    for g in golden["rng"]:
        idx = None if g["index"] < 0 else g["index"]
        s = mb.Rng(int(g["seed"])).stream(g["name"], idx)
        assert [str(int(v)) for v in s.next_n(16)] == g["next"]
        s = mb.Rng(int(g["seed"])).stream(g["name"], idx)
        assert bits_equal(np.array([s.uniform() for _ in range(8)]), unhexa(g["uniform"]))
        s = mb.Rng(int(g["seed"])).stream(g["name"], idx)
        assert bits_equal(np.array([s.normal() for _ in range(9)]), unhexa(g["normal"]))
        s = mb.Rng(int(g["seed"])).stream(g["name"], idx)
        assert [s.below(1000) for _ in range(8)] == g["below"]


def test_named_streams_deterministic_and_independent(mb):
    # test_core.cpp:66-86
    a, b, c = mb.Rng(7), mb.Rng(7), mb.Rng(8)
    s1, s2, s3, s4 = a.stream("x"), b.stream("x"), a.stream("y"), c.stream("x")
    v1, v2, v3, v4 = s1.next_n(64), s2.next_n(64), s3.next_n(64), s4.next_n(64)
    assert (v1 == v2).all() and not (v1 == v3).all() and not (v1 == v4).all()
    assert a.stream("z", 0)() != a.stream("z", 1)()


def test_bernoulli_edges_and_ranges(mb):
    s = mb.Rng(9).stream("coin")
    assert not any(s.bernoulli(0.0) for _ in range(100))
    assert all(s.bernoulli(1.0) for _ in range(100))
    s = mb.Rng(3).stream("range")
    for _ in range(200):
        assert 0.0 <= s.uniform() < 1.0
        assert s.below(7) < 7
    v = list(range(50))
    mb.Rng(5).stream("perm").shuffle(v)
    assert sorted(v) == list(range(50))


def test_key_arithmetic_matches_golden(mb, golden):
    for k in golden["initial_index"]:
        assert mb.initial_index(k["cell"], mb.GridConfig(k["M"], k["d"], 1)).indices == k["key"]
    for k in golden["next_group_key"]:
        g = mb.GridConfig(k["M"], len(k["key"]) + 1, 1)
        assert mb.next_group_key(mb.GroupKey(k["key"]), k["chunk"], g).indices == k["out"]


def test_reference_key_kats_and_errors(mb):
    g = mb.GridConfig(3, 3, 1)
    assert mb.initial_index(0, g).indices == [0, 0]
    assert mb.initial_index(5, g).indices == [1, 0]
    assert mb.initial_index(26, g).indices == [2, 2]
    with pytest.raises(mb.OutOfRange):
        mb.initial_index(27, g)
    assert mb.initial_index(2, mb.GridConfig(5, 1, 1)).indices == []
    g4 = mb.GridConfig(4, 3, 1)
    assert mb.next_group_key(mb.GroupKey([1, 2]), 3, g4).indices == [2, 3]
    with pytest.raises(IndexError):
        mb.next_group_key(mb.GroupKey([1, 2]), 4, g4)
    assert mb.next_group_key(mb.GroupKey([]), 2, mb.GridConfig(4, 1, 1)).indices == []
    # every initial key has exactly M cells in its preimage (test_matchmaking.cpp:51-58)
    from collections import Counter
    cnt = Counter(tuple(mb.initial_index(c, g4).indices) for c in range(g4.capacity()))
    assert len(cnt) == 16 and set(cnt.values()) == {4}


def test_grid_and_failure_validation(mb):
    mb.GridConfig(3, 2, 1).validate()
    assert mb.GridConfig(3, 2, 1).capacity() == 9
    assert mb.GridConfig(2, 10, 1).capacity() == 1024
    for bad in [(0, 2, 1), (3, 0, 1), (3, 2, 0)]:
        with pytest.raises(ValueError):
            mb.GridConfig(*bad).validate()
    with pytest.raises(ValueError):
        mb.FailureModel(-0.1).validate()
    with pytest.raises(ValueError):
        mb.FailureModel(1.5).validate()


def test_chunk_sizes_and_weights(mb, golden):
    for c in golden["chunk_sizes"]:
        assert mb.chunk_sizes(c["dim"], mb.PartitionWeights(c["w"])) == c["sizes"]
    mb.PartitionWeights.uniform(5).validate()
    with pytest.raises(ValueError):
        mb.PartitionWeights([0.5, 0.6]).validate()
    with pytest.raises(ValueError):
        mb.PartitionWeights([1.5, -0.5]).validate()
    with pytest.raises(ValueError):
        mb.chunk_sizes(4, mb.PartitionWeights([0.5, 0.6]))


def test_complexity_estimate_matches_reference(mb, golden):
    from tests._util import unhex
    for c in golden["run_moshpit"]:
        assert mb.complexity_estimate(c["rounds"], c["n"], c["M"], c["dim"]) == unhex(c["cost_units"])


def test_validation_happens_before_the_device(mb):
    """Argument errors surface with the reference's classes even without a GPU
    (protocols.hpp:112-117, allreduce.hpp:82-89, core.hpp:92)."""
    x = np.ones((5, 1))
    with pytest.raises(ValueError):  # N > M^d (test_protocols.cpp:65-70)
        mb.run_moshpit(mb.GridConfig(2, 2, 1), x, mb.FailureModel(), mb.Rng(1), 1)
    with pytest.raises(ValueError):
        mb.run_moshpit(mb.GridConfig(0, 2, 1), x, mb.FailureModel(), mb.Rng(1), 1)
    with pytest.raises(ValueError):
        mb.run_moshpit(mb.GridConfig(4, 2, 1), x, mb.FailureModel(2.0), mb.Rng(1), 1)
    with pytest.raises(ValueError):
        mb.run_moshpit(mb.GridConfig(4, 2, 1), [], mb.FailureModel(), mb.Rng(1), 1)
    with pytest.raises(ValueError):  # C5 as written: 8192 peers on 8^4
        mb.run_moshpit(mb.GridConfig(8, 4, 4), np.zeros((8192, 1)), mb.FailureModel(),
                       mb.Rng(7), 4)
    with pytest.raises(ValueError):
        mb.butterfly_allreduce([], mb.PartitionWeights([]))
    with pytest.raises(ValueError):
        mb.butterfly_allreduce([[1.0], [2.0]], mb.PartitionWeights([1.0]))
    with pytest.raises(ValueError):
        mb.butterfly_allreduce([[1.0], [2.0, 3.0]], mb.PartitionWeights.uniform(2))
    with pytest.raises(ValueError):
        mb.group_mean([])
    assert mb.distortion([], [1.0]) == 0.0
    with pytest.raises(ValueError):
        mb.distortion([[1.0], [1.0, 2.0]], [2.0])


def test_void_path_needs_no_device(mb):
    # allreduce.hpp:95-102: any failure voids the group; outputs = inputs
    # (test_allreduce.cpp:75-82).  No arithmetic, so it runs on CPU too.
    inputs = [[1.0], [2.0], [3.0]]
    out = mb.butterfly_allreduce(inputs, mb.PartitionWeights.uniform(3), [False, True, False])
    assert not out.completed
    assert out.vectors.tolist() == inputs
    assert out.chunks == [0, 1, 2]


def test_compute_without_device_fails_loudly(mb):
    if mb.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(mb.CudaError):
        mb.group_mean([[1.0, 2.0], [3.0, 6.0]])
    with pytest.raises(mb.CudaError):
        mb.run_moshpit(mb.GridConfig(3, 2, 1), np.ones((9, 2)), mb.FailureModel(), mb.Rng(1), 2)


def test_trial_seed_matches_reference_harness(mb):
    from oracle.oracle import REF_HARNESS_SO, RefHarness
    if not os.path.exists(REF_HARNESS_SO):
        pytest.skip("reference harness shim not built")
    h = RefHarness()
    for n, p, k in [(1024, 0.0, 0), (768, 0.005, 17), (512, 0.01, 99), (900, 1e-3, 3)]:
        assert mb.trial_seed(0, "moshpit", n, p, k) == h.trial_seed(0, n, p, k)
        assert mb.trial_seed(12345, "moshpit", n, p, k) == h.trial_seed(12345, n, p, k)


def test_logistic_synthetic_and_smoothness_on_host(mb, golden, oracle):
    """LogisticRegression::synthetic draws (optimizer.hpp:89-104) and the
    smoothness bound (:82-86) are host setup: bit-exact without a device."""
    from tests._util import bits_equal, unhex
    for c in golden["logistic_eval"]:
        lr = mb.LogisticRegression.synthetic(c["dim"], c["samples"], c["l2"],
                                             mb.Rng(c["data_seed"]).stream("objective"))
        xs, ys = oracle.logistic_dataset(c["dim"], c["samples"], c["data_seed"])
        assert bits_equal(lr.xs, xs) and bits_equal(lr.ys, ys)
        assert lr.smoothness() == unhex(c["smoothness"])
        assert lr.strong_convexity() == c["l2"] and lr.optimum_value() == 0.0
    with pytest.raises(ValueError):  # optimizer.hpp:80-81
        mb.LogisticRegression(np.zeros((0, 3)), [], 0.1)
    with pytest.raises(ValueError):
        mb.LogisticRegression(np.zeros((2, 3)), [1.0], 0.1)
