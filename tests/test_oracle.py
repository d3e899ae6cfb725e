"""CPU: the oracle (C restatement) is pinned to the reference.

Two anchors: the committed golden vectors (tests/golden/golden.json, made by
gen_golden.py from the unmodified reference) and, where it is built here, the
reference itself (oracle/_ref).  Bit-exact throughout (fp64).
"""
import numpy as np
import pytest

from tests._util import INIT_SEED, bits_equal, unhex, unhexa


def test_rng_streams_match_golden(oracle, golden):
    for g in golden["rng"]:
        seed, name, idx = int(g["seed"]), g["name"], g["index"]
        nxt = oracle.stream_draws(seed, name, 16, "next", idx)
        assert [str(int(v)) for v in nxt] == g["next"]
        assert bits_equal(oracle.stream_draws(seed, name, 8, "uniform", idx), unhexa(g["uniform"]))
        assert bits_equal(oracle.stream_draws(seed, name, 9, "normal", idx), unhexa(g["normal"]))
        assert [int(v) for v in oracle.stream_draws(seed, name, 8, "below", idx, arg=1000)] == g["below"]


def test_initial_index_and_next_key_match_golden(oracle, golden):
    for k in golden["initial_index"]:
        assert oracle.initial_index(k["cell"], k["M"], k["d"]) == k["key"]
    for k in golden["next_group_key"]:
        assert oracle.next_group_key(k["key"], k["chunk"], k["M"]) == k["out"]


def test_reference_kats(oracle):
    # test_matchmaking.cpp:39-68
    assert oracle.initial_index(0, 3, 3) == [0, 0]
    assert oracle.initial_index(5, 3, 3) == [1, 0]
    assert oracle.initial_index(26, 3, 3) == [2, 2]
    with pytest.raises(IndexError):
        oracle.initial_index(27, 3, 3)
    assert oracle.initial_index(2, 5, 1) == []
    assert oracle.next_group_key([1, 2], 3, 4) == [2, 3]
    with pytest.raises(IndexError):
        oracle.next_group_key([1, 2], 4, 4)
    # test_allreduce.cpp:19-25
    assert oracle.chunk_sizes(8, [0.5, 0.25, 0.125, 0.125]) == [4, 2, 1, 1]
    assert oracle.chunk_sizes(4, [0.0, 0.0, 1.0]) == [0, 0, 4]
    # test_core.cpp:32-48
    assert oracle.group_mean(np.array([[1.0, 2.0], [3.0, 6.0]])).tolist() == [2.0, 4.0]
    assert oracle.distortion(np.array([[1.0], [3.0]]), [2.0]) == 1.0
    assert oracle.distortion(np.array([[5.0, 5.0], [5.0, 5.0]]), [5.0, 5.0]) == 0.0
    # SPEC distortion example [1,2,3,4], ref 2.5 -> 1.25
    assert oracle.distortion(np.array([[1.0], [2.0], [3.0], [4.0]]), [2.5]) == 1.25


def test_form_groups_match_golden(oracle, golden):
    for g in golden["form_groups"]:
        ts = np.array([int(v) for v in g["ts"]], dtype=np.uint64)
        keys = np.array(g["keys"], dtype=np.uint32).reshape(len(g["ids"]), -1)
        m, off = oracle.form_groups(g["ids"], keys, ts, g["cap"])
        assert m.tolist() == g["members"]
        assert off.tolist() == g["group_off"]


def test_chunk_sizes_match_golden(oracle, golden):
    for c in golden["chunk_sizes"]:
        assert oracle.chunk_sizes(c["dim"], c["w"]) == c["sizes"]


def test_butterfly_matches_golden(oracle, golden):
    for b in golden["butterfly"]:
        x = unhexa(b["inputs"]).reshape(b["n"], b["dim"])
        y, done = oracle.butterfly(x, b["failed"])
        assert done == b["completed"]
        assert bits_equal(y.reshape(-1), unhexa(b["out"]))


def test_run_moshpit_matches_golden(oracle, golden):
    for c in golden["run_moshpit"]:
        x = oracle.init_state(INIT_SEED, c["n"], c["dim"], dtype=np.float64)
        rep, fin = oracle.run_moshpit(c["M"], c["d"], x, c["p"], c["seed"], c["rounds"])
        assert rep["initial_distortion"] == unhex(c["initial_distortion"])
        assert bits_equal(rep["distortion"], unhexa(c["distortion"]))
        assert bits_equal(rep["mean_drift"], unhexa(c["mean_drift"]))
        assert rep["active_counts"].tolist() == c["active_counts"]
        assert rep["cost_units"] == unhex(c["cost_units"])
        if c["final"] is not None:
            assert bits_equal(fin.reshape(-1), unhexa(c["final"]))
        for i, row in zip(c["final_rows"], c["final_rows_values"]):
            assert bits_equal(fin[i], unhexa(row))


def test_moshpit_average_matches_golden(oracle, golden):
    for c in golden["moshpit_average"]:
        x = oracle.init_state(INIT_SEED, c["n"], c["dim"], dtype=np.float64)
        y = oracle.moshpit_average(x, c["M"], c["d"], c["rounds"], c["seed"], c["name"])
        assert bits_equal(y.reshape(-1), unhexa(c["out"]))


@pytest.mark.parametrize("M,d,n,p,R,dim", [(3, 2, 9, 0.0, 4, 2), (5, 2, 24, 0.1, 10, 3),
                                           (4, 3, 50, 0.2, 8, 5), (8, 1, 8, 0.3, 3, 4),
                                           (7, 2, 40, 0.5, 6, 3), (2, 5, 32, 0.1, 9, 2)])
def test_oracle_equals_reference(oracle, ref, M, d, n, p, R, dim):
    x = np.random.default_rng(n * 31 + d).random((n, dim))
    ro, fo = oracle.run_moshpit(M, d, x, p, 1000 + n, R)
    rr, fr = ref.run_moshpit(M, d, x, p, 1000 + n, R)
    for k in ro:
        assert bits_equal(np.asarray(ro[k]), np.asarray(rr[k])), k
    assert bits_equal(fo, fr)


def test_restated_reference_loop_equals_stock_run_moshpit(ref):
    x = np.random.default_rng(5).random((30, 2))
    a, _ = ref.run_moshpit(6, 2, x, 0.05, 12, 20)
    b, _ = ref.run_moshpit(6, 2, x, 0.05, 12, 20, vectors=False)
    for k in a:
        assert bits_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_fp32_oracle_is_close_to_fp64_reference(oracle):
    x = oracle.init_state(INIT_SEED, 256, 64, dtype=np.float32)
    _, f32 = oracle.run_moshpit(16, 2, x, 0.0, 7, 2)
    _, f64 = oracle.run_moshpit(16, 2, x.astype(np.float64), 0.0, 7, 2)
    rel = np.abs(f32.astype(np.float64) - f64) / np.abs(f64)
    assert rel.max() <= 1e-6


def test_oracle_trace_is_consistent(oracle):
    t = oracle.trace(32, 2, 1024, 0.01, 7, 10)
    for r in range(10):
        g = int(t["n_groups"][r])
        off = t["group_off"][r][: g + 1]
        assert off[0] == 0 and off[-1] == 1024
        assert np.all(np.diff(off) == 32)  # full grid: every group exactly M
        assert sorted(t["members"][r].tolist()) == list(range(1024))


def _sgd_case(c):
    from tests._util import unhexa as U
    return dict(M=c["M"], d=c["d"], n_peers=c["n"], dim=c["dim"], L=c["L"], mu=c["mu"],
                target=U(c["target"]), theta0=np.zeros(c["dim"]), gamma=c["gamma"], tau=c["tau"],
                steps=c["steps"], sigma=c["sigma"], seed=c["seed"],
                schedule=[tuple(e) for e in c["schedule"]])


def test_sgd_oracle_matches_golden(oracle, golden):
    for c in golden["sgd_quadratic"]:
        res = oracle.sgd_quadratic(**_sgd_case(c))
        for k in ("f_gap", "grad_norm_sq", "f_gap_weighted", "dispersion", "final_mean"):
            assert bits_equal(res[k], unhexa(c[k])), k
        assert res["delta_aq_hat"] == unhex(c["delta_aq_hat"])
        assert res["sigma_hat"] == unhex(c["sigma_hat"])
        assert res["delta_pv2_hat"] == unhex(c["delta_pv2_hat"])
        assert res["n_min"] == c["n_min"]


def test_sgd_oracle_equals_reference_with_schedule(oracle, ref):
    tgt = ref.stream_draws(24, "target", 3, "normal")
    kw = dict(M=4, d=2, n_peers=12, dim=3, L=10.0, mu=1.0, target=tgt, theta0=np.zeros(3),
              gamma=0.02, tau=3, steps=30, sigma=0.7, seed=31, schedule=((4, -5), (9, 6)))
    a, b = oracle.sgd_quadratic(**kw), ref.sgd_quadratic(**kw)
    for k in ("f_gap", "grad_norm_sq", "f_gap_weighted", "dispersion", "final_mean"):
        assert bits_equal(a[k], b[k]), k
    assert a["sigma_hat"] == b["sigma_hat"] and a["n_min"] == b["n_min"] == 7


# ---- LogisticRegression (optimizer.hpp:75-146), SURVEY 8f rank 3 ----------------
def test_logistic_oracle_matches_golden(oracle, golden):
    """The oracle's synthetic dataset, value, gradient and smoothness are
    bit-identical to the unmodified reference's (golden vectors)."""
    for c in golden["logistic_eval"]:
        xs, ys = oracle.logistic_dataset(c["dim"], c["samples"], c["data_seed"])
        assert set(np.unique(ys).tolist()) <= {-1.0, 1.0}
        v, g, sm = oracle.logistic_eval(xs, ys, c["l2"], unhexa(c["theta"]))
        assert v == unhex(c["value"])
        assert bits_equal(g, unhexa(c["grad"]))
        assert sm == unhex(c["smoothness"])


def test_logistic_oracle_equals_reference_eval(oracle, ref):
    rng = np.random.default_rng(5)
    for S, dim in [(1, 1), (7, 3), (64, 33)]:
        xs = rng.normal(size=(S, dim)) * 3
        ys = np.where(rng.random(S) < 0.5, -1.0, 1.0)
        th = rng.normal(size=dim) * 5  # both tails of the stable softplus
        a, b = oracle.logistic_eval(xs, ys, 0.05, th), ref.logistic_eval(xs, ys, 0.05, th)
        assert a[0] == b[0] and bits_equal(a[1], b[1]) and a[2] == b[2]


def test_sgd_logistic_oracle_matches_golden(oracle, golden):
    for c in golden["sgd_logistic"]:
        res = oracle.sgd_logistic(c["M"], c["d"], c["n"], c["dim"], c["samples"], c["l2"],
                                  c["data_seed"], np.zeros(c["dim"]), c["gamma"], c["tau"],
                                  c["steps"], c["sigma"], c["seed"])
        for k in ("f_gap", "grad_norm_sq", "f_gap_weighted", "dispersion", "final_mean"):
            assert bits_equal(res[k], unhexa(c[k])), k
        assert res["delta_aq_hat"] == unhex(c["delta_aq_hat"])
        assert res["sigma_hat"] == unhex(c["sigma_hat"])
        assert res["delta_pv2_hat"] == unhex(c["delta_pv2_hat"])
