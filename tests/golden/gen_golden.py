"""Generate tests/golden/golden.json from the UNMODIFIED reference.

    python tests/golden/gen_golden.py

Runs the reference headers compiled into oracle/_ref/libmoshpit_ref.so
(oracle/Makefile builds it from /root/reference/proj/include) and records
known-answer vectors for the hot path: RNG streams, initial_index /
next_group_key, form_groups_uncontested, chunk_sizes, butterfly_allreduce,
run_moshpit TrialReports + final vectors (through ref_run_moshpit_vectors,
whose report is asserted equal to the stock run_moshpit here), and
moshpit_average.  Doubles are stored as IEEE-754 hex bit patterns so
comparisons are bit-exact.  The fixtures travel with the repo; the reference
tree does not.
"""
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Checker  # noqa: E402

INIT_SEED = 0x5EED


def hx(x):
    return struct.pack("<d", float(x)).hex()


def hxa(a):
    return [hx(v) for v in np.asarray(a, dtype=np.float64).reshape(-1)]


def C_eval(r, dim, S, l2, dseed, th):
    import ctypes as C
    v, sm = C.c_double(0), C.c_double(0)
    g = np.zeros(dim)
    rc = r._logistic_synthetic_eval(dim, S, l2, dseed, b"objective",
                                    th.ctypes.data_as(C.c_void_p), C.byref(v),
                                    g.ctypes.data_as(C.c_void_p), C.byref(sm))
    assert rc == 0
    return v.value, g, sm.value


def main():
    r = Checker("ref")
    out = {"source": "oracle/_ref (unmodified reference headers via ref_shim.cpp)",
           "init": "x(i,j) = (splitmix64(0x5EED ^ (i<<32) ^ j) >> 40) * 2^-24"}

    rng = []
    for seed, name, index in [(7, "priorities", -1), (7, "failures", -1), (7, "cells", -1),
                              (0, "init", -1), (12345, "averaging", -1), (3, "keys", 5),
                              (99, "trial", 0), (2**63 + 11, "noise", -1)]:
        rng.append(dict(seed=str(seed), name=name, index=index,
                        next=[str(int(v)) for v in r.stream_draws(seed, name, 16, "next", index)],
                        uniform=hxa(r.stream_draws(seed, name, 8, "uniform", index)),
                        normal=hxa(r.stream_draws(seed, name, 9, "normal", index)),
                        below=[int(v) for v in r.stream_draws(seed, name, 8, "below", index,
                                                              arg=1000)]))
    out["rng"] = rng

    kat = []
    for M, d in [(3, 3), (4, 3), (5, 1), (16, 2), (8, 4), (2, 10)]:
        cap = M ** d
        for cell in sorted({0, 1, cap // 3, cap // 2, cap - 1}):
            kat.append(dict(M=M, d=d, cell=cell, key=r.initial_index(cell, M, d)))
    out["initial_index"] = kat
    out["next_group_key"] = [dict(M=4, key=[1, 2], chunk=3, out=r.next_group_key([1, 2], 3, 4)),
                             dict(M=16, key=[5, 9, 15], chunk=0,
                                  out=r.next_group_key([5, 9, 15], 0, 16)),
                             dict(M=4, key=[], chunk=2, out=[])]

    gen = np.random.default_rng(2103)
    groups = []
    for t in range(12):
        n = int(gen.integers(1, 60))
        klen = int(gen.integers(0, 3))
        ids = gen.permutation(5000)[:n].astype(np.uint32)
        keys = gen.integers(0, 4, (n, klen)).astype(np.uint32)
        ts = gen.integers(0, 2**48, n).astype(np.uint64)
        if t % 3 == 0:
            ts[: n // 2] = ts[0]  # timestamp ties -> id breaks them
        cap = int(gen.integers(1, 9)) if t % 2 else 0xFFFFFFFF
        m, off = r.form_groups(ids, keys, ts, cap)
        groups.append(dict(ids=ids.tolist(), keys=keys.tolist(), ts=[str(int(v)) for v in ts],
                           cap=cap, members=m.tolist(), group_off=off.tolist()))
    out["form_groups"] = groups

    out["chunk_sizes"] = [dict(dim=8, w=[0.5, 0.25, 0.125, 0.125],
                               sizes=r.chunk_sizes(8, [0.5, 0.25, 0.125, 0.125])),
                          dict(dim=4, w=[0.0, 0.0, 1.0], sizes=r.chunk_sizes(4, [0.0, 0.0, 1.0])),
                          dict(dim=7, w=[1 / 3] * 3, sizes=r.chunk_sizes(7, [1 / 3] * 3))]

    bfly = []
    for n, dim, fail in [(1, 6, None), (2, 6, None), (5, 6, None), (8, 6, None), (13, 5, None),
                         (32, 3, None), (3, 1, [0, 1, 0])]:
        x = gen.standard_normal((n, dim))
        y, done = r.butterfly(x, fail)
        bfly.append(dict(inputs=hxa(x), n=n, dim=dim, failed=fail, out=hxa(y), completed=done))
    out["butterfly"] = bfly

    runs = []
    init = Checker("oracle").init_state
    for M, d, n, dim, p, seed, R in [(3, 2, 9, 2, 0.0, 99, 4), (16, 2, 256, 8, 0.0, 7, 2),
                                     (32, 2, 1024, 4, 0.01, 7, 10), (16, 3, 4096, 2, 0.0, 7, 3),
                                     (8, 4, 4096, 2, 0.0, 7, 4), (5, 2, 24, 3, 0.1, 1000, 10),
                                     (4, 3, 50, 5, 0.2, 12, 8), (8, 1, 8, 4, 0.3, 5, 3),
                                     (32, 2, 512, 3, 0.0, 3, 12), (6, 2, 30, 2, 0.05, 12, 20)]:
        x = init(INIT_SEED, n, dim, dtype=np.float64)
        rep, fin = r.run_moshpit(M, d, x, p, seed, R)
        stock, _ = r.run_moshpit(M, d, x, p, seed, R, vectors=False)
        for k in rep:
            assert np.array_equal(np.asarray(rep[k]), np.asarray(stock[k])), k
        runs.append(dict(M=M, d=d, n=n, dim=dim, p=p, seed=seed, rounds=R,
                         initial_distortion=hx(rep["initial_distortion"]),
                         distortion=hxa(rep["distortion"]), mean_drift=hxa(rep["mean_drift"]),
                         active_counts=[int(a) for a in rep["active_counts"]],
                         cost_units=hx(rep["cost_units"]),
                         final=hxa(fin) if n * dim <= 4096 else None,
                         final_rows=[0, n // 2, n - 1],
                         final_rows_values=[hxa(fin[i]) for i in (0, n // 2, n - 1)]))
    out["run_moshpit"] = runs

    x = init(INIT_SEED, 14, 3, dtype=np.float64)
    out["moshpit_average"] = [dict(M=4, d=2, rounds=2, seed=5, name="averaging", n=14, dim=3,
                                   out=hxa(r.moshpit_average(x, 4, 2, 2, 5)))]
    x = init(INIT_SEED, 60, 2, dtype=np.float64)
    out["moshpit_average"].append(dict(M=4, d=3, rounds=3, seed=8, name="averaging", n=60, dim=2,
                                       out=hxa(r.moshpit_average(x, 4, 3, 3, 8))))

    sgd = []
    for (M, d, n, dim, L, mu, gamma, tau, K, sigma, sched, seed) in [
            (4, 2, 9, 4, 5.0, 0.5, 0.05, 1, 60, 0.0, (), 500),
            (4, 2, 12, 3, 10.0, 1.0, 0.02, 4, 40, 1.0, (), 8000),
            (8, 2, 16, 2, 4.0, 1.0, 0.05, 1, 30, 1.0, (), 9000),
            (4, 2, 8, 2, 2.0, 1.0, 0.1, 2, 20, 0.5, ((5, -3), (12, 2)), 777),
            (32, 2, 1024, 8, 1.0, 0.1, 0.1, 1, 6, 1.0, (), 7)]:
        tgt = r.stream_draws(seed, "objective", dim, "normal")
        th0 = np.zeros(dim)
        res = r.sgd_quadratic(M, d, n, dim, L, mu, tgt, th0, gamma, tau, K, sigma, seed,
                              schedule=sched)
        sgd.append(dict(M=M, d=d, n=n, dim=dim, L=L, mu=mu, gamma=gamma, tau=tau, steps=K,
                        sigma=sigma, schedule=[list(e) for e in sched], seed=seed,
                        target=hxa(tgt), f_gap=hxa(res["f_gap"]),
                        grad_norm_sq=hxa(res["grad_norm_sq"]),
                        f_gap_weighted=hxa(res["f_gap_weighted"]),
                        dispersion=hxa(res["dispersion"]), final_mean=hxa(res["final_mean"]),
                        delta_aq_hat=hx(res["delta_aq_hat"]), sigma_hat=hx(res["sigma_hat"]),
                        delta_pv2_hat=hx(res["delta_pv2_hat"]), n_min=res["n_min"]))
    out["sgd_quadratic"] = sgd
    th = np.array([0.0, 0.0])
    out["local_step"] = [dict(dim=2, L=2.0, mu=2.0, target=[1.0, 1.0], gamma=0.25, sigma=0.0,
                              seed=23, name="n", theta=[0.0, 0.0],
                              out=hxa(r.local_step_quadratic(th, 2.0, 2.0, [1.0, 1.0], 0.25, 0.0,
                                                             23, "n"))),
                         dict(dim=5, L=3.0, mu=0.5, target=[0.1, -0.2, 0.3, 0.4, -0.5], gamma=0.1,
                              sigma=2.0, seed=4, name="noise", theta=[1.0, 2.0, 3.0, 4.0, 5.0],
                              out=hxa(r.local_step_quadratic(np.arange(1.0, 6.0), 3.0, 0.5,
                                                             [0.1, -0.2, 0.3, 0.4, -0.5], 0.1,
                                                             2.0, 4, "noise")))]

    # LogisticRegression (optimizer.hpp:75-146): synthetic(dim, samples, l2,
    # Rng(data_seed).stream("objective")) evaluated at theta, and
    # run_moshpit_sgd over it -- both from the unmodified reference.
    logit = []
    for (dim, S, l2, dseed) in [(4, 32, 0.01, 11), (16, 200, 0.1, 12), (1, 5, 0.0, 13)]:
        th = r.stream_draws(dseed, "theta", dim, "normal")
        v, g, sm = C_eval(r, dim, S, l2, dseed, th)
        logit.append(dict(dim=dim, samples=S, l2=l2, data_seed=dseed, theta=hxa(th),
                          value=hx(v), grad=hxa(g), smoothness=hx(sm)))
    out["logistic_eval"] = logit
    lsgd = []
    for (M, d, n, dim, S, l2, gamma, tau, K, sigma, seed) in [
            (4, 2, 9, 4, 32, 0.01, 0.2, 1, 25, 0.0, 31),
            (4, 2, 12, 8, 64, 0.1, 0.1, 3, 20, 1.0, 32),
            (8, 2, 40, 16, 100, 0.05, 0.3, 1, 10, 0.5, 33)]:
        res = r.sgd_logistic(M, d, n, dim, S, l2, seed, np.zeros(dim), gamma, tau, K, sigma,
                             seed)
        lsgd.append(dict(M=M, d=d, n=n, dim=dim, samples=S, l2=l2, gamma=gamma, tau=tau,
                         steps=K, sigma=sigma, seed=seed, data_seed=seed,
                         f_gap=hxa(res["f_gap"]), grad_norm_sq=hxa(res["grad_norm_sq"]),
                         f_gap_weighted=hxa(res["f_gap_weighted"]),
                         dispersion=hxa(res["dispersion"]), final_mean=hxa(res["final_mean"]),
                         delta_aq_hat=hx(res["delta_aq_hat"]), sigma_hat=hx(res["sigma_hat"]),
                         delta_pv2_hat=hx(res["delta_pv2_hat"])))
    out["sgd_logistic"] = lsgd

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
