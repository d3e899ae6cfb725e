"""B200-native Moshpit averaging engine (arXiv 2103.03239), Python face.

Mirrors the reference's public API (proj/include/moshpit/: ``GridConfig``,
``GroupKey``, ``FailureModel``, ``Rng``/``RngStream``, ``initial_index``,
``next_group_key``, ``MatchPeer``/``SealedGroup``/``form_groups_uncontested``,
``PartitionWeights``/``butterfly_allreduce``, ``group_mean``, ``distortion``,
``mean_of``, ``TrialReport``/``run_moshpit``, ``moshpit_average``) with the
same argument meaning and error classes, over the C ABI of
``libmoshpit_b200.so`` (include/moshpit_b200.h).  The data plane runs on the
GPU; there is no CPU fallback.  ``Engine`` is the device-resident
performance path (peer state in a CUDA tensor, one call per round).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import (CudaError, InvalidArgument, MoshpitError, OutOfRange,  # noqa: F401
                    ReferenceRuntimeError, check, lib)

UINT32_MAX = 0xFFFFFFFF

__all__ = [
    "GridConfig", "GroupKey", "FailureModel", "Rng", "RngStream", "initial_index",
    "next_group_key", "MatchPeer", "SealedGroup", "Priority", "form_groups_uncontested",
    "PartitionWeights", "chunk_sizes", "AllReduceOutcome", "butterfly_allreduce",
    "group_mean", "distortion", "mean_of", "TrialReport", "run_moshpit", "moshpit_average",
    "complexity_estimate", "Engine", "fill_synthetic", "InvalidArgument", "OutOfRange",
    "CudaError", "MoshpitError", "device_count", "Shard", "Quadratic", "OptimizerConfig",
    "MembershipEvent", "SgdResult", "AssumptionDiagnostics", "local_step", "run_moshpit_sgd",
    "run_moshpit_batch", "trial_seed", "LogisticRegression",
]


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dtype_code(dt):
    dt = np.dtype(dt)
    if dt == np.float32:
        return _capi.F32
    if dt == np.float64:
        return _capi.F64
    raise InvalidArgument(f"unsupported dtype {dt}; use float32 or float64")


def device_count() -> int:
    n = C.c_int(0)
    check(lib().moshpit_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# core.hpp:19-66
# ---------------------------------------------------------------------------
@dataclass
class GridConfig:
    peers_per_axis: int = 1  # M
    dims: int = 1            # d
    rounds: int = 1          # T

    def validate(self):
        check(lib().moshpit_grid_validate(self.peers_per_axis, self.dims, self.rounds))

    def capacity(self) -> int:
        return int(lib().moshpit_grid_capacity(self.peers_per_axis, self.dims))


@dataclass(order=True)
class GroupKey:
    indices: List[int] = field(default_factory=list)


@dataclass
class FailureModel:
    p_round: float = 0.0
    churn: list = field(default_factory=list)

    def validate(self):
        if self.p_round < 0.0 or self.p_round > 1.0:
            raise InvalidArgument("FailureModel: p_round must be in [0,1]")


# ---------------------------------------------------------------------------
# rng.hpp:31-127
# ---------------------------------------------------------------------------
class RngStream:
    """xoshiro256** stream with the reference's exact output sequence."""

    def __init__(self, state: _capi.RngState):
        self.state = state

    def _draw(self, kind, n, arg=0, p=0.0, dt=np.uint64):
        out = np.zeros(max(n, 1), dtype=dt)
        check(lib().moshpit_rng_draws(C.byref(self.state), kind, arg, p, n, _p(out)))
        return out[:n]

    def __call__(self) -> int:
        return int(self._draw(0, 1)[0])

    def next_n(self, n) -> np.ndarray:
        return self._draw(0, n)

    def uniform(self) -> float:
        return float(self._draw(1, 1, dt=np.float64)[0])

    def below(self, n: int) -> int:
        return int(self._draw(2, 1, arg=n)[0])

    def normal(self) -> float:
        return float(self._draw(3, 1, dt=np.float64)[0])

    def normals(self, n) -> np.ndarray:
        return self._draw(3, n, dt=np.float64)

    def bernoulli(self, p: float) -> bool:
        return bool(self._draw(4, 1, p=p, dt=np.uint8)[0])

    def shuffle(self, v: list):
        for i in range(len(v), 1, -1):
            j = self.below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


class Rng:
    def __init__(self, seed: int):
        self._seed = int(seed) & 0xFFFFFFFFFFFFFFFF

    def seed(self) -> int:
        return self._seed

    def stream(self, name: str, index: Optional[int] = None) -> RngStream:
        st = _capi.RngState()
        check(lib().moshpit_rng_stream(self._seed, name.encode(),
                                       -1 if index is None else int(index), C.byref(st)))
        return RngStream(st)


# ---------------------------------------------------------------------------
# matchmaking.hpp:20-25, 46-90, 300-323
# ---------------------------------------------------------------------------
def initial_index(peer_cell: int, grid: GridConfig) -> GroupKey:
    out = np.zeros(max(grid.dims - 1, 1), dtype=np.uint32)
    check(lib().moshpit_initial_index(peer_cell, grid.peers_per_axis, grid.dims, _p(out)))
    return GroupKey([int(x) for x in out[: grid.dims - 1]])


def next_group_key(prev: GroupKey, new_chunk: int, grid: GridConfig) -> GroupKey:
    k = np.asarray(prev.indices, dtype=np.uint32)
    out = np.zeros(max(len(k), 1), dtype=np.uint32)
    check(lib().moshpit_next_group_key(_p(k) if len(k) else None, len(k), new_chunk,
                                       grid.peers_per_axis, _p(out)))
    return GroupKey([int(x) for x in out[: len(k)]])


@dataclass(order=True)
class Priority:
    timestamp: int = 0
    peer: int = 0


@dataclass
class MatchPeer:
    id: int = 0
    key: GroupKey = field(default_factory=GroupKey)
    timestamp: int = 0
    arrival: int = 0


@dataclass
class SealedGroup:
    leader: int = 0
    members: List[int] = field(default_factory=list)


def form_groups_uncontested(peers: Sequence[MatchPeer],
                            max_group_size: int = UINT32_MAX) -> List[SealedGroup]:
    """Closed-form grouping on the GPU (kernel 1)."""
    n = len(peers)
    if n == 0:
        return []
    klens = {len(p.key.indices) for p in peers}
    if len(klens) != 1:
        raise InvalidArgument("form_groups_uncontested: keys of different lengths")
    klen = klens.pop()
    ids = np.array([p.id for p in peers], dtype=np.uint32)
    keys = np.array([p.key.indices for p in peers], dtype=np.uint32).reshape(n, klen)
    ts = np.array([p.timestamp for p in peers], dtype=np.uint64)
    members = np.zeros(n, dtype=np.uint32)
    off = np.zeros(n + 1, dtype=np.uint32)
    ng = C.c_uint64(0)
    check(lib().moshpit_form_groups_uncontested(n, _p(ids), _p(keys) if klen else None, klen,
                                                _p(ts), max_group_size, _p(members), _p(off),
                                                C.byref(ng)))
    groups = []
    for g in range(ng.value):
        m = [int(x) for x in members[off[g]:off[g + 1]]]
        groups.append(SealedGroup(leader=m[0], members=m))
    return groups


# ---------------------------------------------------------------------------
# allreduce.hpp:15-121
# ---------------------------------------------------------------------------
@dataclass
class PartitionWeights:
    w: List[float] = field(default_factory=list)

    def validate(self):
        total = 0.0
        for wi in self.w:
            if wi < 0.0:
                raise InvalidArgument("PartitionWeights: w >= 0")
            total += wi
        if abs(total - 1.0) > 1e-9:
            raise InvalidArgument("PartitionWeights: weights must sum to 1")

    @staticmethod
    def uniform(n: int) -> "PartitionWeights":
        return PartitionWeights([1.0 / n] * n)


def chunk_sizes(dim: int, weights: PartitionWeights) -> List[int]:
    w = np.asarray(weights.w, dtype=np.float64)
    out = np.zeros(max(len(w), 1), dtype=np.uint64)
    check(lib().moshpit_chunk_sizes(dim, _p(w), len(w), _p(out)))
    return [int(x) for x in out[: len(w)]]


@dataclass
class AllReduceOutcome:
    completed: bool = False
    vectors: Optional[np.ndarray] = None
    chunks: List[int] = field(default_factory=list)


def _rows(x, dtype=None):
    if isinstance(x, np.ndarray):
        a = x
    else:
        lens = {len(v) for v in x}
        if len(lens) > 1:
            raise InvalidArgument("dimension mismatch")
        a = np.asarray(x)
    if dtype is not None:
        a = a.astype(dtype, copy=False)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    if a.ndim == 1:
        a = a.reshape(len(a), -1) if len(a) else a.reshape(0, 0)
    return np.ascontiguousarray(a)


def butterfly_allreduce(inputs, weights: PartitionWeights,
                        failed: Optional[Sequence[bool]] = None) -> AllReduceOutcome:
    if len(inputs) == 0:
        raise InvalidArgument("butterfly_allreduce: empty group")
    x = _rows(inputs)
    n, dim = x.shape
    w = np.asarray(weights.w, dtype=np.float64)
    f = None if not failed else np.asarray(failed, dtype=np.uint8)
    out = np.zeros_like(x)
    chunks = np.zeros(n, dtype=np.uint32)
    done = C.c_int32(0)
    check(lib().moshpit_butterfly_allreduce(_dtype_code(x.dtype), _p(x), n, dim, _p(w), len(w),
                                            _p(f), _p(out), _p(chunks), C.byref(done)))
    return AllReduceOutcome(bool(done.value), out, [int(c) for c in chunks])


# ---------------------------------------------------------------------------
# core.hpp:91-133
# ---------------------------------------------------------------------------
def group_mean(members) -> np.ndarray:
    if len(members) == 0:
        raise InvalidArgument("group_mean: empty group")
    x = _rows(members)
    out = np.zeros(x.shape[1], dtype=x.dtype)
    check(lib().moshpit_group_mean(_dtype_code(x.dtype), _p(x), x.shape[0], x.shape[1], None,
                                   x.shape[0], _p(out)))
    return out


def mean_of(peers) -> np.ndarray:
    return group_mean(peers)


def distortion(peers, reference_mean) -> float:
    if len(peers) == 0:
        return 0.0
    x = _rows(peers)
    ref = np.ascontiguousarray(reference_mean, dtype=np.float64).reshape(-1)
    if x.shape[1] != len(ref):
        raise InvalidArgument("distortion: dimension mismatch")
    out = C.c_double(0.0)
    check(lib().moshpit_distortion(_dtype_code(x.dtype), _p(x), x.shape[0], x.shape[1],
                                   _p(ref), C.byref(out)))
    return out.value


def complexity_estimate(t_rounds, n_peers, m, dim) -> float:
    return lib().moshpit_complexity_estimate(t_rounds, n_peers, m, dim)


# ---------------------------------------------------------------------------
# protocols.hpp:49-179
# ---------------------------------------------------------------------------
@dataclass
class TrialReport:
    initial_distortion: float = 0.0
    distortion: List[float] = field(default_factory=list)
    mean_drift: List[float] = field(default_factory=list)
    active_counts: List[int] = field(default_factory=list)
    cost_units: float = 0.0
    vectors: Optional[np.ndarray] = None  # extension: final peer vectors

    def rounds_to(self, threshold: float, cap: int) -> int:
        if self.initial_distortion <= threshold:
            return 0
        for t in range(min(len(self.distortion), cap)):
            if self.distortion[t] <= threshold:
                return t + 1
        return cap


_DIAG = {"none": _capi.DIAG_NONE, "fast": _capi.DIAG_FAST, "exact": _capi.DIAG_EXACT}


def run_moshpit(grid: GridConfig, initial, failure: FailureModel, rng: Rng, rounds: int, *,
                dtype=None, diagnostics: Optional[str] = None,
                return_vectors: bool = False) -> TrialReport:
    """protocols::run_moshpit on the GPU.

    ``dtype`` float64 (default for lists / float64 arrays) is bit-identical to
    the reference; float32 is the performance path.  ``diagnostics`` defaults
    to "exact" (reference summation order) for float64 and "fast" for
    float32.
    """
    if len(initial) == 0:
        grid.validate()
        failure.validate()
        raise InvalidArgument("run_moshpit: no peers")
    x = _rows(initial, dtype)
    n, dim = x.shape
    code = _dtype_code(x.dtype)
    if diagnostics is None:
        diagnostics = "exact" if code == _capi.F64 else "fast"
    R = max(int(rounds), 1)
    dist = np.zeros(R)
    drift = np.zeros(R)
    act = np.zeros(R, dtype=np.uint32)
    init_d = C.c_double(0)
    cost = C.c_double(0)
    final = np.zeros_like(x) if return_vectors else None
    check(lib().moshpit_run_moshpit(code, grid.peers_per_axis, grid.dims, grid.rounds, _p(x), n,
                                    dim, failure.p_round, rng.seed(), int(rounds),
                                    _DIAG[diagnostics], C.byref(init_d), _p(dist), _p(drift),
                                    _p(act), C.byref(cost), _p(final)))
    return TrialReport(init_d.value, list(dist[:rounds]), list(drift[:rounds]),
                       [int(a) for a in act[:rounds]], cost.value, final)


def round_from_groups(state, members, group_off, void_flags=None, dim: Optional[int] = None,
                      stream=None):
    """One round over an externally formed group table:
    ``state`` a CUDA tensor [n_rows, ld] averaged in place, or a host numpy
    array [n_rows, dim] (copied in and out).  ``members``/``group_off`` as in
    a CSR table of the groups in priority order; ``void_flags[g]`` voids g."""
    mem = np.ascontiguousarray(members, dtype=np.uint32)
    off = np.ascontiguousarray(group_off, dtype=np.uint32)
    ng = max(len(off) - 1, 0)
    vf = None if void_flags is None else np.ascontiguousarray(void_flags, dtype=np.uint8)
    if isinstance(state, np.ndarray):
        if not state.flags.c_contiguous or state.dtype not in (np.float32, np.float64):
            raise InvalidArgument("round_from_groups: C-contiguous float32/float64 rows")
        check(lib().moshpit_round_from_groups_host(_dtype_code(state.dtype), _p(state),
                                                   state.shape[0], state.shape[1], _p(mem),
                                                   _p(off), ng, _p(vf)))
        return state
    import torch
    code, ptr, ld = _tensor_args(state)
    s = stream if stream is not None else torch.cuda.current_stream(state.device)
    check(lib().moshpit_round_from_groups(code, ptr, state.shape[0],
                                          state.shape[1] if dim is None else dim, ld, _p(mem),
                                          _p(off), ng, _p(vf), s.cuda_stream))
    return state


def trial_seed(seed_base: int, protocol: str, n: int, p: float, seed_index: int) -> int:
    """harness::trial_rng (harness.hpp:145-155) root seed."""
    return int(lib().moshpit_trial_seed(seed_base, protocol.encode(), n, p, seed_index))


def run_moshpit_batch(grid: GridConfig, initial, failure: FailureModel, seeds: Sequence[int],
                      rounds: int, *, diagnostics: str = "exact",
                      return_vectors: bool = False) -> List[TrialReport]:
    """Trial-batched protocols::run_moshpit: ``initial`` is [trials, n, dim];
    trial t runs with Rng(seeds[t]).  Equal, report by report, to calling
    run_moshpit per trial -- but one launch per kernel per round for all."""
    x = np.ascontiguousarray(initial)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    T, n, dim = x.shape
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    if len(sd) != T:
        raise InvalidArgument("run_moshpit_batch: one seed per trial")
    R = max(rounds, 1)
    init_d = np.zeros(max(T, 1))
    dist = np.zeros((max(T, 1), R))
    drift = np.zeros((max(T, 1), R))
    act = np.zeros((max(T, 1), R), dtype=np.uint32)
    cost = np.zeros(max(T, 1))
    fin = np.zeros_like(x) if return_vectors else None
    check(lib().moshpit_run_moshpit_batch(_dtype_code(x.dtype), grid.peers_per_axis, grid.dims,
                                          grid.rounds, T, _p(x), n, dim, failure.p_round, _p(sd),
                                          rounds, _DIAG[diagnostics], _p(init_d), _p(dist),
                                          _p(drift), _p(act), _p(cost), _p(fin)))
    out = []
    for t in range(T):
        out.append(TrialReport(float(init_d[t]), list(dist[t, :rounds]), list(drift[t, :rounds]),
                               [int(a) for a in act[t, :rounds]], float(cost[t]),
                               None if fin is None else fin[t]))
    return out


def moshpit_average(thetas, grid: GridConfig, rounds: int, stream: RngStream):
    """optimizer::detail::moshpit_average on the GPU; returns the averaged
    array (in place when ``thetas`` is a C-contiguous float array)."""
    x = thetas if (isinstance(thetas, np.ndarray) and thetas.flags.c_contiguous
                   and thetas.dtype in (np.float32, np.float64)) else _rows(thetas)
    n = x.shape[0]
    dim = x.shape[1] if x.ndim == 2 else 0
    check(lib().moshpit_moshpit_average(_dtype_code(x.dtype), _p(x), n, dim,
                                        grid.peers_per_axis, grid.dims, rounds,
                                        C.byref(stream.state)))
    return x


# ---------------------------------------------------------------------------
# optimizer.hpp:31-72, 186-227, 231-242, 297-439 (Quadratic objective)
# ---------------------------------------------------------------------------
class Quadratic:
    """Axis-aligned quadratic with curvature interpolated mu -> L."""

    def __init__(self, dim: int, l: float, mu: float, target):
        if l < mu or mu < 0.0:
            raise InvalidArgument("Quadratic: need L >= mu >= 0")
        t = np.ascontiguousarray(target, dtype=np.float64).reshape(-1)
        if len(t) != dim:
            raise InvalidArgument("Quadratic: target dimension mismatch")
        self._dim, self.l, self.mu, self.target = int(dim), float(l), float(mu), t

    def dim(self):
        return self._dim

    def smoothness(self):
        return self.l

    def strong_convexity(self):
        return self.mu

    def optimum_value(self):
        return 0.0

    def optimum(self):
        return self.target


class LogisticRegression:
    """L2-regularised logistic regression (optimizer.hpp:75-146): value and
    gradient evaluate on the GPU in the reference's summation orders."""

    def __init__(self, xs, ys, l2: float):
        x = np.ascontiguousarray(xs, dtype=np.float64)
        y = np.ascontiguousarray(ys, dtype=np.float64).reshape(-1)
        if x.ndim != 2 or x.shape[0] == 0 or x.shape[0] != len(y):
            raise InvalidArgument("LogisticRegression: bad dataset")
        self.xs, self.ys, self.l2 = x, y, float(l2)
        sm = C.c_double(0.0)
        check(lib().moshpit_logistic_eval(_p(x), _p(y), len(y), x.shape[1], self.l2, None, None,
                                          None, C.byref(sm)))
        self._l = sm.value

    @staticmethod
    def synthetic(dim: int, samples: int, l2: float, stream: RngStream) -> "LogisticRegression":
        xs = np.zeros((samples, dim))
        ys = np.zeros(samples)
        check(lib().moshpit_logistic_synthetic(dim, samples, C.byref(stream.state), _p(xs),
                                               _p(ys)))
        return LogisticRegression(xs, ys, l2)

    def _eval(self, theta, want_grad):
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
        v = C.c_double(0.0)
        g = np.zeros(max(self.dim(), 1)) if want_grad else None
        check(lib().moshpit_logistic_eval(_p(self.xs), _p(self.ys), len(self.ys), self.dim(),
                                          self.l2, _p(th), C.byref(v), _p(g), None))
        return v.value, (g[:self.dim()] if want_grad else None)

    def value(self, theta) -> float:
        return self._eval(theta, False)[0]

    def gradient(self, theta) -> np.ndarray:
        return self._eval(theta, True)[1]

    def dim(self):
        return self.xs.shape[1]

    def smoothness(self):
        return self._l

    def strong_convexity(self):
        return self.l2

    def optimum_value(self):
        return 0.0


@dataclass
class OptimizerConfig:
    gamma: float = 0.1
    tau: int = 1
    steps: int = 100
    grid: GridConfig = field(default_factory=GridConfig)
    sigma: float = 0.0
    n_peers: int = 1
    inner_rounds: int = 0

    def validate(self):
        if self.gamma <= 0.0:
            raise InvalidArgument("OptimizerConfig: gamma > 0")
        if self.tau < 1:
            raise InvalidArgument("OptimizerConfig: tau >= 1")
        if self.sigma < 0.0:
            raise InvalidArgument("OptimizerConfig: sigma >= 0")
        self.grid.validate()
        if self.n_peers < 1 or self.n_peers > self.grid.capacity():
            raise InvalidArgument("OptimizerConfig: 1 <= N <= M^d")


@dataclass
class MembershipEvent:
    step: int = 0
    delta: int = 0


@dataclass
class AssumptionDiagnostics:
    dispersion: List[float] = field(default_factory=list)
    delta_aq_hat: float = 0.0
    sigma_hat: float = 0.0
    delta_pv1_hat: float = 0.0
    delta_pv2_hat: float = 0.0
    n_min: int = 0


@dataclass
class SgdResult:
    f_gap: List[float] = field(default_factory=list)
    grad_norm_sq: List[float] = field(default_factory=list)
    f_gap_weighted: List[float] = field(default_factory=list)
    final_mean: Optional[np.ndarray] = None
    diagnostics: AssumptionDiagnostics = field(default_factory=AssumptionDiagnostics)
    final_thetas: Optional[np.ndarray] = None  # extension
    loop_ms: float = 0.0  # extension: device time of the step loop


def local_step(theta: np.ndarray, objective, gamma: float, sigma: float,
               noise: RngStream) -> np.ndarray:
    """optimizer::local_step on the GPU (in place for float arrays)."""
    x = theta if (isinstance(theta, np.ndarray) and theta.dtype in (np.float32, np.float64)
                  and theta.flags.c_contiguous) else np.ascontiguousarray(theta, np.float64)
    if isinstance(objective, LogisticRegression):
        check(lib().moshpit_local_step_logistic(_dtype_code(x.dtype), _p(x), len(x),
                                                _p(objective.xs), _p(objective.ys),
                                                len(objective.ys), objective.l2, gamma, sigma,
                                                C.byref(noise.state)))
        return x
    if not isinstance(objective, Quadratic):
        raise InvalidArgument("local_step: objective must be Quadratic or LogisticRegression")
    check(lib().moshpit_local_step_quadratic(_dtype_code(x.dtype), _p(x), len(x), objective.l,
                                             objective.mu, _p(objective.target), gamma, sigma,
                                             C.byref(noise.state)))
    return x


def run_moshpit_sgd(config: OptimizerConfig, objective, theta0,
                    schedule: Sequence[MembershipEvent], rng: Rng, *, dtype=np.float64,
                    diagnostics: str = "exact", noise: str = "reference",
                    return_thetas: bool = False) -> SgdResult:
    """optimizer::run_moshpit_sgd on the GPU.  float64 + diagnostics="exact" +
    noise="reference" is bit-identical to the reference; noise="device" uses
    Philox normals on the GPU (statistical parity, no O(N*D) host draws)."""
    th0 = np.ascontiguousarray(theta0, dtype=np.float64).reshape(-1)
    if len(th0) != objective.dim():
        config.validate()
        raise InvalidArgument("run_moshpit_sgd: theta0 dimension mismatch")
    K = max(config.steps, 1)
    out = {k: np.zeros(K) for k in ("f_gap", "g", "fw", "disp")}
    dim = objective.dim()
    fm = np.zeros(max(dim, 1))
    d6 = np.zeros(6)
    evs = np.array([e.step for e in schedule], dtype=np.uint32)
    evd = np.array([e.delta for e in schedule], dtype=np.int32)
    n_max = config.n_peers + sum(max(e.delta, 0) for e in schedule)
    fin = np.zeros((n_max, max(dim, 1)), dtype=dtype) if return_thetas else None
    loop_ms = C.c_double(0.0)
    g = config.grid
    tail = (_p(th0), config.gamma, config.tau, config.steps, config.sigma, config.inner_rounds,
            rng.seed(), _p(evs) if len(evs) else None, _p(evd) if len(evd) else None, len(evs),
            _DIAG[diagnostics], {"reference": 0, "device": 1}[noise], _p(out["f_gap"]),
            _p(out["g"]), _p(out["fw"]), _p(out["disp"]), _p(fm), _p(d6), _p(fin),
            C.byref(loop_ms))
    if isinstance(objective, LogisticRegression):
        check(lib().moshpit_run_moshpit_sgd_logistic(
            _dtype_code(dtype), g.peers_per_axis, g.dims, g.rounds, config.n_peers, dim,
            _p(objective.xs), _p(objective.ys), len(objective.ys), objective.l2, *tail))
    elif isinstance(objective, Quadratic):
        check(lib().moshpit_run_moshpit_sgd_quadratic(
            _dtype_code(dtype), g.peers_per_axis, g.dims, g.rounds, config.n_peers, dim,
            objective.l, objective.mu, _p(objective.target), *tail))
    else:
        raise InvalidArgument("run_moshpit_sgd: objective must be Quadratic or "
                              "LogisticRegression")
    n_fin = int(d6[5])
    diag = AssumptionDiagnostics(list(out["disp"][:config.steps]), d6[0], d6[1], d6[2], d6[3],
                                 int(d6[4]))
    return SgdResult(list(out["f_gap"][:config.steps]), list(out["g"][:config.steps]),
                     list(out["fw"][:config.steps]), fm[:dim], diag,
                     None if fin is None else fin[:n_fin, :dim], loop_ms.value)


# ---------------------------------------------------------------------------
# Device-resident engine (torch tensors or raw device pointers)
# ---------------------------------------------------------------------------
def _tensor_args(state):
    import torch  # plumbing only: device memory and streams
    if not isinstance(state, torch.Tensor) or not state.is_cuda:
        raise InvalidArgument("state must be a CUDA tensor")
    if state.dtype == torch.float32:
        code = _capi.F32
    elif state.dtype == torch.float64:
        code = _capi.F64
    else:
        raise InvalidArgument("state dtype must be float32 or float64")
    if state.dim() != 2 or state.stride(1) != 1:
        raise InvalidArgument("state must be [n, ld] with unit column stride")
    return code, state.data_ptr(), state.stride(0)


def fill_synthetic(state, seed: int, dim: Optional[int] = None, col0: int = 0, stream=None):
    import torch
    code, ptr, ld = _tensor_args(state)
    s = stream if stream is not None else torch.cuda.current_stream(state.device)
    check(lib().moshpit_fill_synthetic(code, ptr, state.shape[0],
                                       state.shape[1] if dim is None else dim, ld, seed, col0,
                                       s.cuda_stream))


class Engine:
    """One Moshpit trial resident on a GPU (protocols.hpp:123-173 round loop)."""

    def __init__(self, grid: GridConfig, n_peers: int, failure: FailureModel, rng: Rng,
                 device: int = 0, kernel: int = _capi.KERNEL_AUTO):
        self.grid, self.n = grid, int(n_peers)
        h = C.c_void_p()
        check(lib().moshpit_engine_create(grid.peers_per_axis, grid.dims, self.n,
                                          failure.p_round, rng.seed(), device, C.byref(h)))
        self._h = h
        self.device = device
        if kernel != _capi.KERNEL_AUTO:
            check(lib().moshpit_engine_set_kernel(self._h, kernel))

    def close(self):
        if getattr(self, "_h", None):
            lib().moshpit_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_kernel(self, variant: int):
        check(lib().moshpit_engine_set_kernel(self._h, variant))

    def round(self, state, dim: Optional[int] = None, stream=None) -> int:
        """Enqueue one round on ``stream`` (default: torch's current stream)."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        act = C.c_uint32(0)
        check(lib().moshpit_engine_round(self._h, code, ptr,
                                         state.shape[1] if dim is None else dim, ld,
                                         s.cuda_stream, C.byref(act)))
        return act.value

    def rounds_fused(self, state, rounds: int, dim: Optional[int] = None, stream=None):
        """Enqueue ``rounds`` rounds in one pass over the state (temporal
        blocking; n <= 1800): the same results as ``rounds`` calls of
        round().  Returns the per-round active (non-failed) peer counts."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        act = np.zeros(max(int(rounds), 1), dtype=np.uint32)
        check(lib().moshpit_engine_rounds_fused(self._h, code, ptr,
                                                state.shape[1] if dim is None else dim, ld,
                                                int(rounds), s.cuda_stream, _p(act)))
        return act[:int(rounds)].tolist()

    def round_raw(self, dtype_code: int, ptr: int, dim: int, ld: int, stream_handle: int) -> int:
        act = C.c_uint32(0)
        check(lib().moshpit_engine_round(self._h, dtype_code, ptr, dim, ld, stream_handle,
                                         C.byref(act)))
        return act.value

    def set_timing(self, enable: bool):
        check(lib().moshpit_engine_set_timing(self._h, 1 if enable else 0))

    def kernel_time(self):
        """(summed device ms, launches) of kernel 2 since the last call."""
        ms, k = C.c_double(0), C.c_uint64(0)
        check(lib().moshpit_engine_kernel_time(self._h, C.byref(ms), C.byref(k)))
        return ms.value, k.value

    def set_reference(self, state, diagnostics: str = "fast", dim: Optional[int] = None,
                      stream=None):
        """record_round's reference = mean_of(state) and the initial
        distortion, on the device (protocols.hpp:119, 68-84)."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        check(lib().moshpit_engine_set_reference(self._h, code, ptr,
                                                 state.shape[1] if dim is None else dim, ld,
                                                 _DIAG[diagnostics], s.cuda_stream))

    def round_record(self, state, dim: Optional[int] = None, stream=None) -> int:
        """One round and its record_round (reads one representative row per
        averaged group: same bits as round() + record())."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        act = C.c_uint32(0)
        check(lib().moshpit_engine_round_record(self._h, code, ptr,
                                                state.shape[1] if dim is None else dim, ld,
                                                s.cuda_stream, C.byref(act)))
        return act.value

    def rounds_record(self, state, rounds: int, dim: Optional[int] = None,
                      stream=None) -> List[int]:
        """``rounds`` x (round + record_round) in one call (the run_moshpit
        loop on the device): with FAST diagnostics the voided rows' cached row
        partials are reused, only the averaged groups' representatives are
        re-read; same bits as ``rounds`` round_record() calls."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        act = (C.c_uint32 * max(int(rounds), 1))()
        check(lib().moshpit_engine_rounds_record(self._h, code, ptr,
                                                 state.shape[1] if dim is None else dim, ld,
                                                 int(rounds), s.cuda_stream, act))
        return list(act)[:int(rounds)]

    def record(self, state, dim: Optional[int] = None, stream=None):
        """Append this round's (distortion, mean_drift) to the device log."""
        import torch
        code, ptr, ld = _tensor_args(state)
        s = stream if stream is not None else torch.cuda.current_stream(state.device)
        check(lib().moshpit_engine_record(self._h, code, ptr,
                                          state.shape[1] if dim is None else dim, ld,
                                          s.cuda_stream))

    def report(self):
        """(initial_distortion, [distortion], [mean_drift]) recorded so far."""
        cnt = C.c_uint64(0)
        init = C.c_double(0)
        check(lib().moshpit_engine_report(self._h, C.byref(init), None, None, 0, C.byref(cnt)))
        k = cnt.value
        dist, drift = np.zeros(max(k, 1)), np.zeros(max(k, 1))
        check(lib().moshpit_engine_report(self._h, C.byref(init), _p(dist), _p(drift), k,
                                          C.byref(cnt)))
        return init.value, list(dist[:k]), list(drift[:k])

    def stats(self):
        r, rows = C.c_uint64(0), C.c_uint64(0)
        check(lib().moshpit_engine_stats(self._h, C.byref(r), C.byref(rows)))
        return r.value, rows.value

    def tables(self):
        n, klen = self.n, self.grid.dims - 1
        members = np.zeros(n, dtype=np.uint32)
        off = np.zeros(n + 1, dtype=np.uint32)
        ng = C.c_uint32(0)
        void = np.zeros(n, dtype=np.uint8)
        ranks = np.zeros(n, dtype=np.uint32)
        keys = np.zeros((n, max(klen, 1)), dtype=np.uint32)
        check(lib().moshpit_engine_tables(self._h, _p(members), _p(off), C.byref(ng), _p(void),
                                          _p(ranks), _p(keys)))
        g = ng.value
        return dict(members=members, group_off=off[: g + 1], n_groups=g, void=void[:g],
                    rank=ranks, keys=keys[:, :klen])


# ---------------------------------------------------------------------------
# Peer-sharded multi-GPU engine
# ---------------------------------------------------------------------------
def exchange_handles(mine: bytes, procs: int, group=None) -> List[bytes]:
    """All-gather one fixed-size handle blob per process, in process order."""
    import torch.distributed as dist
    if dist.get_world_size(group) != procs:
        raise InvalidArgument("process group size differs from the shard's process count")
    allh = [None] * procs
    dist.all_gather_object(allh, mine, group=group)
    if any(len(h) != len(mine) for h in allh):
        raise InvalidArgument("processes disagree on the handle size")
    return allh


class Shard:
    """The ranks of a peer-sharded Moshpit trial hosted by this process.

    Real multi-process use (one process per GPU, torch.distributed for the
    one-time handle exchange only)::

        sh = Shard(grid, n, failure, rng, dim, rank=r, world=w, device=local)
        sh.connect(process_group)        # all_gather of CUDA IPC handles
        sh.fill_synthetic(seed)          # or sh.load_rows(host) (sh.row_peers(): the placement)
        for _ in range(rounds): sh.round()
        sh.flush()                       # slabs > 1: finish the lagging slabs
        sh.store_rows(host)              # optional: the rows back to the host

    ``ranks_per_process=k`` hosts ranks [rank, rank+k) here (rank a multiple of
    k; e.g. world 8 on 4 GPUs); ``emulate=True`` hosts all ``world`` ranks on
    one GPU.  ``slabs=S`` pipelines S column slabs one round apart so NVLink
    cross rounds overlap HBM-bound local rounds (bit-identical results).
    ``cross="exact"`` (default) runs the reference tree over the members' raw
    chunks in cross rounds (bit-exact); ``cross="partial"`` ships one partial
    sum per GPU and group instead (fixed order, fp64 combine; within 1e-6
    relative in fp32 -- the summation order is not the reference's).
    """

    def __init__(self, grid: GridConfig, n_peers: int, failure: FailureModel, rng: Rng,
                 dim: int, rank: int = 0, world: int = 1, emulate: bool = False,
                 device: int = 0, dtype=np.float32, ranks_per_process: int = 1,
                 slabs: int = 1, cross: str = "exact"):
        self.grid, self.n, self.dim = grid, int(n_peers), int(dim)
        self.world, self.emulate = world, emulate
        self.nhost = world if emulate else int(ranks_per_process)
        self.rank = 0 if emulate else rank
        self.procs = world // self.nhost
        self.device = int(device)
        self.dtype = np.dtype(dtype)
        self.slabs = int(slabs)
        self._loading = []  # host buffers of load_rows copies possibly in flight
        h = C.c_void_p()
        check(lib().moshpit_shard_create_ex(_dtype_code(self.dtype), grid.peers_per_axis,
                                            grid.dims, self.n, failure.p_round, rng.seed(),
                                            self.dim, self.rank, self.nhost, world, self.slabs,
                                            device, C.byref(h)))
        self._h = h
        if cross not in ("exact", "partial"):
            self.close()
            raise InvalidArgument(f"Shard: cross must be 'exact' or 'partial', not {cross!r}")
        self.cross = cross
        check(lib().moshpit_shard_set_cross_mode(self._h, 1 if cross == "partial" else 0))

    def close(self):
        if getattr(self, "_h", None):
            lib().moshpit_shard_destroy(self._h)
            self._h = None
        self._loading = []

    __del__ = close

    def ipc_handles(self) -> bytes:
        buf = (C.c_char * (128 * self.nhost))()
        check(lib().moshpit_shard_ipc_handles(self._h, buf))
        return bytes(buf)

    def open_peers(self, handles: Sequence[bytes]):
        blob = b"".join(handles)
        if len(blob) != 128 * self.world:
            raise InvalidArgument("open_peers: need 128 bytes per rank")
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        check(lib().moshpit_shard_open_peers(self._h, buf))

    def connect(self, group=None):
        """Exchange CUDA IPC handles over torch.distributed (plumbing only)."""
        self.open_peers(exchange_handles(self.ipc_handles(), self.procs, group))

    def flush(self, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().moshpit_shard_flush(self._h, s.cuda_stream))

    def fill_synthetic(self, seed: int, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().moshpit_shard_fill_synthetic(self._h, seed, s.cuda_stream))

    def round(self, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        act, crossed = C.c_uint32(0), C.c_int32(0)
        check(lib().moshpit_shard_round(self._h, s.cuda_stream, C.byref(act), C.byref(crossed)))
        return act.value, bool(crossed.value)

    def read(self):
        out = np.zeros((self.n, self.dim), dtype=self.dtype)
        mask = np.zeros(self.n, dtype=np.uint8)
        check(lib().moshpit_shard_read(self._h, _p(out), _p(mask)))
        self._loading = []
        return out, mask.astype(bool)

    def _rank(self, k):
        return self.rank if k is None else k

    def rows(self) -> int:
        """Rows of each rank's pool (its resident peers)."""
        ptr, rows, ld = C.c_void_p(), C.c_uint64(0), C.c_uint64(0)
        check(lib().moshpit_shard_pool(self._h, self.rank, C.byref(ptr), C.byref(rows),
                                       C.byref(ld)))
        return rows.value

    def row_peers(self, k: Optional[int] = None) -> np.ndarray:
        """The peer held by each row of rank k's pool (-1 as 0xffffffff: none)."""
        out = np.zeros(self.rows(), dtype=np.uint32)
        check(lib().moshpit_shard_row_peers(self._h, self._rank(k), _p(out)))
        self._loading = []
        return out

    def load_rows(self, host: np.ndarray, k: Optional[int] = None, stream=None):
        """Host rows -> rank k's pool (row r holds row_peers(k)[r]); `host`
        is rows() x dim (pinned memory for full PCIe rate), asynchronous on
        `stream` -- keep `host` alive until the stream passes the copy."""
        if host.dtype != self.dtype or host.ndim != 2 or host.shape[0] != self.rows() \
                or host.shape[1] < self.dim:
            raise InvalidArgument("shard: host rows must be rows() x dim of the shard dtype")
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().moshpit_shard_load_rows(self._h, self._rank(k), _p(host), host.strides[0],
                                            s.cuda_stream))
        # the copy may still be in flight: hold the buffer until a call that
        # synchronises the device (row_peers, read, close)
        self._loading.append(host)

    def store_rows(self, host: np.ndarray, k: Optional[int] = None, stream=None):
        """Rank k's pool -> host rows (after the lagging slabs finish)."""
        if host.dtype != self.dtype or host.ndim != 2 or host.shape[0] != self.rows() \
                or host.shape[1] < self.dim or not host.flags.writeable:
            raise InvalidArgument("shard: host rows must be rows() x dim of the shard dtype")
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().moshpit_shard_store_rows(self._h, self._rank(k), _p(host), host.strides[0],
                                             s.cuda_stream))

    def set_timing(self, enable: bool):
        check(lib().moshpit_shard_set_timing(self._h, 1 if enable else 0))

    def stats(self, k: int = 0):
        """(cross rounds, active groups over cross rounds, local active rows)."""
        a, b, c = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        check(lib().moshpit_shard_stats(self._h, k, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def cross_detail(self, k: int = 0):
        """(phase A ms, phase B ms) of the cross rounds timed by the last
        kernel_time() call, and voided rows moved into rank k so far."""
        a, b, m = C.c_double(0), C.c_double(0), C.c_uint64(0)
        check(lib().moshpit_shard_cross_detail(self._h, k, C.byref(a), C.byref(b), C.byref(m)))
        return a.value, b.value, m.value

    def kernel_time(self):
        lm, ln, cm, cn = C.c_double(0), C.c_uint64(0), C.c_double(0), C.c_uint64(0)
        check(lib().moshpit_shard_kernel_time(self._h, C.byref(lm), C.byref(ln), C.byref(cm),
                                              C.byref(cn)))
        return lm.value, ln.value, cm.value, cn.value
