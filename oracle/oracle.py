"""ctypes view of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two libraries share one calling convention:
  * ``oracle/liboracle.so`` -- the C restatement (``orc_*``), both precisions;
  * ``oracle/_ref/libmoshpit_ref.so`` -- the unmodified reference headers
    behind ``ref_shim.cpp`` (``ref_*``), fp64 only.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoshpit_ref.so")

ERR = {-1: ValueError, -2: IndexError, -3: RuntimeError, -4: RuntimeError}


def _check(rc, what):
    if rc < 0:
        raise ERR.get(rc, RuntimeError)(f"{what} failed with status {rc}")
    return rc


def build(quiet=True):
    """Compile liboracle.so (and _ref when the reference tree is present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class _Rng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4), ("have_spare", C.c_int), ("spare", C.c_double)]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


u64, u32, i64, dbl, vp, cstr = C.c_uint64, C.c_uint32, C.c_int64, C.c_double, C.c_void_p, C.c_char_p


class Checker:
    """One of the two CPU checkers.  ``kind`` is 'oracle' or 'ref'."""

    def __init__(self, kind="oracle"):
        self.kind = kind
        path = ORACLE_SO if kind == "oracle" else REF_SO
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.pre = "orc_" if kind == "oracle" else "ref_"
        f = self._fn
        f("stream_draws", None, [u64, cstr, i64, C.c_int, u64, dbl, u64, vp])
        f("initial_index", C.c_int, [u64, u32, u32, vp])
        f("next_group_key", C.c_int, [vp, u32, u32, u32, vp])
        f("form_groups_uncontested", i64, [u64, vp, vp, u32, vp, u32, vp, vp])
        f("chunk_sizes", C.c_int, [u64, vp, u64, vp])
        f("complexity_estimate", dbl, [u32, u32, u32, u32])
        if kind == "oracle":
            for sfx, real in (("f64", dbl), ("f32", C.c_float)):
                f(f"pairwise_sum_{sfx}", real, [vp, u64])
                f(f"group_mean_{sfx}", C.c_int, [vp, u64, u64, vp, vp])
                f(f"butterfly_{sfx}", C.c_int, [vp, u64, u64, vp, vp, vp])
                f(f"distortion_{sfx}", dbl, [vp, u64, u64, vp])
                f(f"mean_of_{sfx}", C.c_int, [vp, u64, u64, vp])
                f(f"run_moshpit_{sfx}", C.c_int,
                  [u32, u32, u32, vp, u64, u64, dbl, u64, u32, vp, vp, vp, vp, vp, vp])
                f(f"moshpit_average_{sfx}", C.c_int, [vp, u64, u64, u32, u32, u32, vp])
            f("moshpit_trace", C.c_int,
              [u32, u32, u64, dbl, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp])
            f("init_value", dbl, [u64, u64, u64])
            for sfx in ("f64", "f32"):
                f(f"sgd_quadratic_{sfx}", C.c_int,
                  [u32, u32, u32, u32, u64, dbl, dbl, vp, vp, dbl, u32, u32, dbl, u32, u64, vp,
                   vp, u64, vp, vp, vp, vp, vp, vp, vp])
            f("rng_stream", None, [vp, u64, cstr])
            f("logistic_synthetic", None, [u64, u64, vp, vp, vp])
            f("logistic_value", dbl, [vp, vp, u64, u64, dbl, vp])
            f("logistic_gradient", None, [vp, vp, u64, u64, dbl, vp, vp])
            f("logistic_smoothness", dbl, [vp, u64, u64, dbl])
            f("sgd_logistic_f64", C.c_int,
              [u32, u32, u32, u32, u64, vp, vp, u64, dbl, vp, dbl, u32, u32, dbl, u32, u64, vp,
               vp, vp, vp, vp, vp, vp])
        else:
            f("pairwise_sum", dbl, [vp, u64])
            f("group_mean", C.c_int, [vp, u64, u64, vp, vp])
            f("butterfly", C.c_int, [vp, u64, u64, vp, vp, vp, vp])
            f("contested_round", C.c_int, [u64, u32, u32, u32, vp, u64, vp, vp, vp, vp, vp])
            f("distortion", dbl, [vp, u64, u64, vp])
            f("mean_of", C.c_int, [vp, u64, u64, vp])
            f("run_moshpit", C.c_int,
              [u32, u32, u32, vp, u64, u64, dbl, u64, u32, vp, vp, vp, vp, vp])
            f("run_moshpit_vectors", C.c_int,
              [u32, u32, u32, vp, u64, u64, dbl, u64, u32, vp, vp, vp, vp, vp, vp])
            f("moshpit_average", C.c_int, [vp, u64, u64, u32, u32, u32, u64, cstr])
            f("sgd_quadratic", C.c_int,
              [u32, u32, u32, u32, u64, dbl, dbl, vp, vp, dbl, u32, u32, dbl, u32, u64, vp,
               vp, u64, vp, vp, vp, vp, vp, vp])
            f("local_step_quadratic", C.c_int, [vp, u64, dbl, dbl, vp, dbl, dbl, u64, cstr])
            f("logistic_eval", C.c_int, [vp, vp, u64, u64, dbl, vp, vp, vp, vp])
            f("logistic_synthetic_eval", C.c_int, [u64, u64, dbl, u64, cstr, vp, vp, vp, vp])
            f("sgd_logistic", C.c_int,
              [u32, u32, u32, u32, u64, u64, dbl, u64, cstr, vp, dbl, u32, u32, dbl, u32, u64,
               vp, vp, vp, vp, vp, vp])
            f("slice_bench", C.c_int,
              [u32, u32, u64, u64, u64, u64, u64, u64, dbl, u32, u32, vp, vp, vp])

    def _fn(self, name, res, args):
        fn = getattr(self.lib, self.pre + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    # ---- rng ---------------------------------------------------------------
    def stream_draws(self, root, name, n, kind="next", index=-1, arg=0, p=0.0):
        k = {"next": 0, "uniform": 1, "below": 2, "normal": 3, "bernoulli": 4}[kind]
        dt = {0: np.uint64, 1: np.float64, 2: np.uint64, 3: np.float64, 4: np.uint8}[k]
        out = np.zeros(max(n, 1), dtype=dt)
        self._stream_draws(root, name.encode(), index, k, arg, p, n, _p(out))
        return out[:n]

    # ---- keys / grouping -----------------------------------------------------
    def initial_index(self, cell, M, d):
        key = np.zeros(max(d - 1, 1), dtype=np.uint32)
        _check(self._initial_index(cell, M, d, _p(key)), "initial_index")
        return [int(x) for x in key[: d - 1]]

    def next_group_key(self, key, chunk, M):
        k = np.asarray(key, dtype=np.uint32).reshape(-1)
        out = np.zeros(max(len(k), 1), dtype=np.uint32)
        _check(self._next_group_key(_p(k) if len(k) else None, len(k), chunk, M, _p(out)),
               "next_group_key")
        return [int(x) for x in out[: len(k)]]

    def form_groups(self, ids, keys, ts, cap=0xFFFFFFFF):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        n = len(ids)
        keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(n, -1)
        ts = np.ascontiguousarray(ts, dtype=np.uint64)
        members = np.zeros(max(n, 1), dtype=np.uint32)
        off = np.zeros(n + 1, dtype=np.uint32)
        g = _check(self._form_groups_uncontested(n, _p(ids), _p(keys), keys.shape[1], _p(ts),
                                                 cap, _p(members), _p(off)), "form_groups")
        return members[:n], off[: g + 1]

    def chunk_sizes(self, dim, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.zeros(max(len(w), 1), dtype=np.uint64)
        _check(self._chunk_sizes(dim, _p(w), len(w), _p(out)), "chunk_sizes")
        return [int(x) for x in out[: len(w)]]

    def complexity_estimate(self, t, n, m, dim):
        return self._complexity_estimate(t, n, m, dim)

    # ---- real-valued ----------------------------------------------------------
    def _sfx(self, dtype):
        if self.kind == "ref":
            if np.dtype(dtype) != np.float64:
                raise TypeError("the reference is fp64 only")
            return ""
        return "_f64" if np.dtype(dtype) == np.float64 else "_f32"

    def pairwise_sum(self, xs):
        xs = np.ascontiguousarray(xs)
        return getattr(self, "_pairwise_sum" + self._sfx(xs.dtype))(_p(xs), len(xs))

    def group_mean(self, rows, members=None):
        rows = np.ascontiguousarray(rows)
        n = len(members) if members is not None else rows.shape[0]
        m = None if members is None else np.ascontiguousarray(members, dtype=np.uint32)
        out = np.zeros(rows.shape[1], dtype=rows.dtype)
        _check(getattr(self, "_group_mean" + self._sfx(rows.dtype))(
            _p(rows), n, rows.shape[1], _p(m), _p(out)), "group_mean")
        return out

    def butterfly(self, inputs, failed=None):
        x = np.ascontiguousarray(inputs)
        n, dim = x.shape
        f = None if failed is None else np.ascontiguousarray(failed, dtype=np.uint8)
        out = np.zeros_like(x)
        done = C.c_int(0)
        if self.kind == "ref":
            chunks = np.zeros(n, dtype=np.uint32)
            _check(self._butterfly(_p(x), n, dim, _p(f), _p(out), C.byref(done), _p(chunks)),
                   "butterfly")
        else:
            _check(getattr(self, "_butterfly" + self._sfx(x.dtype))(
                _p(x), n, dim, _p(f), _p(out), C.byref(done)), "butterfly")
        return out, bool(done.value)

    def contested_round(self, trial_seed, x, nkeys=3, cap=0):
        """The unmodified reference's contested form_groups (skewed arrivals,
        FailStop) + butterfly_allreduce per sealed group (ref only):
        returns (members, group_off, void_flags, vectors after the round)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, dim = x.shape
        mem = np.zeros(n, dtype=np.uint32)
        off = np.zeros(n + 1, dtype=np.uint32)
        vf = np.zeros(n, dtype=np.uint8)
        ng = C.c_uint32(0)
        out = np.zeros_like(x)
        _check(self._contested_round(trial_seed, n, nkeys, cap, _p(x), dim, _p(mem), _p(off),
                                     C.byref(ng), _p(vf), _p(out)), "contested_round")
        g = ng.value
        return mem[:off[g]], off[:g + 1], vf[:g], out

    def distortion(self, peers, ref):
        x = np.ascontiguousarray(peers)
        r = np.ascontiguousarray(ref, dtype=np.float64)
        return getattr(self, "_distortion" + self._sfx(x.dtype))(_p(x), x.shape[0], x.shape[1], _p(r))

    def mean_of(self, peers):
        x = np.ascontiguousarray(peers)
        out = np.zeros(x.shape[1], dtype=x.dtype)
        _check(getattr(self, "_mean_of" + self._sfx(x.dtype))(_p(x), x.shape[0], x.shape[1], _p(out)),
               "mean_of")
        return out

    def run_moshpit(self, M, d, initial, p, seed, rounds, T=1, vectors=True):
        x = np.ascontiguousarray(initial)
        n, dim = x.shape
        R = max(rounds, 1)
        init_d = C.c_double(0)
        cost = C.c_double(0)
        dist = np.zeros(R)
        drift = np.zeros(R)
        act = np.zeros(R, dtype=np.uint32)
        final = np.zeros_like(x) if vectors else None
        if self.kind == "ref":
            if vectors:
                rc = self._run_moshpit_vectors(M, d, T, _p(x), n, dim, p, seed, rounds,
                                               C.byref(init_d), _p(dist), _p(drift), _p(act),
                                               C.byref(cost), _p(final))
            else:
                rc = self._run_moshpit(M, d, T, _p(x), n, dim, p, seed, rounds, C.byref(init_d),
                                       _p(dist), _p(drift), _p(act), C.byref(cost))
        else:
            rc = getattr(self, "_run_moshpit" + self._sfx(x.dtype))(
                M, d, T, _p(x), n, dim, p, seed, rounds, C.byref(init_d), _p(dist), _p(drift),
                _p(act), C.byref(cost), _p(final))
        _check(rc, "run_moshpit")
        rep = dict(initial_distortion=init_d.value, distortion=dist[:rounds],
                   mean_drift=drift[:rounds], active_counts=act[:rounds], cost_units=cost.value)
        return rep, final

    def moshpit_average(self, thetas, M, d, rounds, seed, name="averaging"):
        x = np.ascontiguousarray(thetas).copy()
        n, dim = x.shape
        if self.kind == "ref":
            _check(self._moshpit_average(_p(x), n, dim, M, d, rounds, seed, name.encode()),
                   "moshpit_average")
        else:
            st = _Rng()
            self._rng_stream(C.byref(st), seed, name.encode())
            _check(getattr(self, "_moshpit_average" + self._sfx(x.dtype))(
                _p(x), n, dim, M, d, rounds, C.byref(st)), "moshpit_average")
        return x

    def sgd_quadratic(self, M, d, n_peers, dim, L, mu, target, theta0, gamma, tau, steps, sigma,
                      seed, inner_rounds=0, schedule=(), T=1, dtype=np.float64):
        """run_moshpit_sgd(Quadratic(dim, L, mu, target)); returns a dict."""
        tgt = np.ascontiguousarray(target, dtype=np.float64)
        th0 = np.ascontiguousarray(theta0, dtype=np.float64)
        evs = np.array([e[0] for e in schedule], dtype=np.uint32)
        evd = np.array([e[1] for e in schedule], dtype=np.int32)
        K = max(steps, 1)
        out = {k: np.zeros(K) for k in ("f_gap", "grad_norm_sq", "f_gap_weighted", "dispersion")}
        fm = np.zeros(max(dim, 1))
        diag = np.zeros(6)
        n_max = n_peers + sum(max(e[1], 0) for e in schedule)
        args = [M, d, T, n_peers, dim, L, mu, _p(tgt), _p(th0), gamma, tau, steps, sigma,
                inner_rounds, seed, _p(evs) if len(evs) else None, _p(evd) if len(evd) else None,
                len(evs), _p(out["f_gap"]), _p(out["grad_norm_sq"]), _p(out["f_gap_weighted"]),
                _p(out["dispersion"]), _p(fm), _p(diag)]
        fin = None
        if self.kind == "ref":
            _check(self._sgd_quadratic(*args), "sgd_quadratic")
        else:
            fin = np.zeros((n_max, max(dim, 1)), dtype=dtype)
            _check(getattr(self, "_sgd_quadratic" + self._sfx(dtype))(*args, _p(fin)),
                   "sgd_quadratic")
            fin = fin[: int(diag[5]), :dim]
        res = {k: v[:steps] for k, v in out.items()}
        res.update(final_mean=fm[:dim], delta_aq_hat=diag[0], sigma_hat=diag[1],
                   delta_pv1_hat=diag[2], delta_pv2_hat=diag[3], n_min=int(diag[4]),
                   final_thetas=fin)
        return res

    def local_step_quadratic(self, theta, L, mu, target, gamma, sigma, seed, name):
        th = np.ascontiguousarray(theta, dtype=np.float64).copy()
        tgt = np.ascontiguousarray(target, dtype=np.float64)
        _check(self._local_step_quadratic(_p(th), len(th), L, mu, _p(tgt), gamma, sigma, seed,
                                          name.encode()), "local_step")
        return th

    # ---- LogisticRegression (optimizer.hpp:75-146) --------------------------------
    def logistic_dataset(self, dim, samples, data_seed, name="objective"):
        """LogisticRegression::synthetic over Rng(data_seed).stream(name) (oracle)."""
        st = _Rng()
        self._rng_stream(C.byref(st), data_seed, name.encode())
        xs = np.zeros((samples, max(dim, 1)))
        ys = np.zeros(max(samples, 1))
        self._logistic_synthetic(dim, samples, C.byref(st), _p(xs), _p(ys))
        return xs[:, :dim].copy(), ys[:samples].copy()

    def logistic_eval(self, xs, ys, l2, theta):
        """(value, gradient, smoothness) of LogisticRegression(xs, ys, l2) at theta."""
        x = np.ascontiguousarray(xs, dtype=np.float64)
        y = np.ascontiguousarray(ys, dtype=np.float64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        S, dim = x.shape
        g = np.zeros(max(dim, 1))
        if self.kind == "ref":
            v, sm = C.c_double(0), C.c_double(0)
            _check(self._logistic_eval(_p(x), _p(y), S, dim, l2, _p(th), C.byref(v), _p(g),
                                       C.byref(sm)), "logistic_eval")
            return v.value, g[:dim], sm.value
        v = self._logistic_value(_p(x), _p(y), S, dim, l2, _p(th))
        self._logistic_gradient(_p(x), _p(y), S, dim, l2, _p(th), _p(g))
        return v, g[:dim], self._logistic_smoothness(_p(x), S, dim, l2)

    def sgd_logistic(self, M, d, n_peers, dim, samples, l2, data_seed, theta0, gamma, tau, steps,
                     sigma, seed, inner_rounds=0, T=1, name="objective"):
        """run_moshpit_sgd(LogisticRegression::synthetic(dim, samples, l2,
        Rng(data_seed).stream(name))); returns a dict (fp64, no schedule)."""
        th0 = np.ascontiguousarray(theta0, dtype=np.float64)
        K = max(steps, 1)
        out = {k: np.zeros(K) for k in ("f_gap", "grad_norm_sq", "f_gap_weighted", "dispersion")}
        fm = np.zeros(max(dim, 1))
        diag = np.zeros(6)
        tail = [_p(th0), gamma, tau, steps, sigma, inner_rounds, seed, _p(out["f_gap"]),
                _p(out["grad_norm_sq"]), _p(out["f_gap_weighted"]), _p(out["dispersion"]),
                _p(fm), _p(diag)]
        fin = None
        if self.kind == "ref":
            _check(self._sgd_logistic(M, d, T, n_peers, dim, samples, l2, data_seed,
                                      name.encode(), *tail), "sgd_logistic")
        else:
            xs, ys = self.logistic_dataset(dim, samples, data_seed, name)
            fin = np.zeros((n_peers, max(dim, 1)))
            _check(self._sgd_logistic_f64(M, d, T, n_peers, dim, _p(xs), _p(ys), samples, l2,
                                          *tail, _p(fin)), "sgd_logistic")
            fin = fin[: int(diag[5]), :dim]
        res = {k: v[:steps] for k, v in out.items()}
        res.update(final_mean=fm[:dim], delta_aq_hat=diag[0], sigma_hat=diag[1],
                   delta_pv1_hat=diag[2], delta_pv2_hat=diag[3], n_min=int(diag[4]),
                   final_thetas=fin)
        return res

    # ---- oracle-only ------------------------------------------------------------
    def trace(self, M, d, n, p, seed, rounds):
        """Per-round integer plane of run_moshpit (group tables, voids, ranks)."""
        R = max(rounds, 1)
        members = np.zeros((R, n), dtype=np.uint32)
        off = np.zeros((R, n + 1), dtype=np.uint32)
        ng = np.zeros(R, dtype=np.uint32)
        void = np.zeros((R, n), dtype=np.uint8)
        rank = np.zeros((R, n), dtype=np.uint32)
        act = np.zeros(R, dtype=np.uint32)
        keys = np.zeros((n, max(d - 1, 1)), dtype=np.uint32)
        cells = np.zeros(n, dtype=np.uint64)
        _check(self._moshpit_trace(M, d, n, p, seed, rounds, _p(members), _p(off), _p(ng),
                                   _p(void), _p(rank), _p(act), _p(keys), _p(cells)), "trace")
        return dict(members=members[:rounds], group_off=off[:rounds], n_groups=ng[:rounds],
                    void=void[:rounds], rank=rank[:rounds], active=act[:rounds],
                    keys_final=keys[:, : d - 1], cells=cells)

    def init_state(self, seed, n, dim, col0=0, dtype=np.float32):
        """Counter-based synthetic init, vectorised in numpy."""
        i = np.arange(n, dtype=np.uint64)[:, None]
        j = np.arange(col0, col0 + dim, dtype=np.uint64)[None, :]
        with np.errstate(over="ignore"):
            s = np.uint64(seed) ^ (i << np.uint64(32)) ^ j
            z = s + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return ((z >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(dtype)

    def slice_bench(self, M, d, n, width, slices, col0, init_seed, seed, p, rounds, threads):
        run_s, init_s, chk = C.c_double(0), C.c_double(0), C.c_double(0)
        _check(self._slice_bench(M, d, n, width, slices, col0, init_seed, seed, p, rounds,
                                 threads, C.byref(run_s), C.byref(init_s), C.byref(chk)),
               "slice_bench")
        return run_s.value, init_s.value, chk.value


REF_HARNESS_SO = os.path.join(HERE, "_ref", "libmoshpit_ref_harness.so")


class RefHarness:
    """The unmodified reference harness (trial_rng, run_trial) -- test only."""

    def __init__(self):
        if not os.path.exists(REF_HARNESS_SO):
            raise FileNotFoundError(REF_HARNESS_SO)
        self.lib = C.CDLL(REF_HARNESS_SO)
        self.lib.refh_trial_seed.restype = u64
        self.lib.refh_trial_seed.argtypes = [u64, u32, dbl, u32]
        self.lib.refh_run_trial.restype = C.c_int
        self.lib.refh_run_trial.argtypes = [u64, u32, dbl, u32, u32, u32, u32, C.c_int, u32, vp,
                                            vp, vp, vp]

    def trial_seed(self, seed_base, n, p, seed_index):
        return int(self.lib.refh_trial_seed(seed_base, n, p, seed_index))

    def run_trial(self, seed_base, n, p, seed_index, M, d, dim, init="uniform", round_cap=50):
        init_d = C.c_double(0)
        dist, drift = np.zeros(round_cap), np.zeros(round_cap)
        act = np.zeros(round_cap, dtype=np.uint32)
        _check(self.lib.refh_run_trial(seed_base, n, p, seed_index, M, d, dim,
                                       1 if init == "normal" else 0, round_cap, C.byref(init_d),
                                       _p(dist), _p(drift), _p(act)), "run_trial")
        return dict(initial_distortion=init_d.value, distortion=dist, mean_drift=drift,
                    active_counts=act)
