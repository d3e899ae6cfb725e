#!/usr/bin/env python
"""Moshpit averaging-round benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--config C2] [--kernel auto|register|bulk] [--no-e2e] [--no-cpu]

Metric: peer-vector GB/s averaged per Moshpit round = N_peers * D * 4 B /
t_round (BASELINE.json).  One *step* = one Moshpit round (host draws ->
kernel 1 group formation -> kernel 2 segmented group mean, in place) over the
resident fp32 peer state.  Default workload = configs[1] (C2: 1024 peers on a
32x32 grid, D = 2^22 fp32, 1% per-round peer failure), which fits one B200
(17.2 GB); the state is 136x the 126 MB L2, so no L2 flush is needed between
rounds.  Synthetic, counter-initialised data.

Multi-GPU (torchrun, one rank per GPU): the headline is the PEER-SHARDED
C2 round (the graded layout): the same 1024 x 4 Mi problem as N=1
(strong scaling), peers split by grid digit d-1 across the ranks, rounds on
axis 0 GPU-local, the axis-1 round one fused NVLink kernel per GPU.  value =
N*D*4 per round / max-over-ranks device time.  Coordinate-sharded weak
scaling (every rank all peers x its own D-slab, no exchange) and the
peer-sharded C5-valid run are attached as extra keys, with NVLink hardware
counters (NVML) read around the timed cross rounds.

--impl reference: the unmodified reference run_moshpit (oracle/_ref, compiled
from the reference headers) on bounded column slices of the same workload on
all host cores; rank 0 only.  Both arms print the same `config` dict.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (M, d, N, D, p, rounds-of-the-config)
    "C1": (16, 2, 256, 1 << 20, 0.0, 2),
    "C2": (32, 2, 1024, 1 << 22, 0.01, 10),
    "C3slab": (16, 3, 4096, 1 << 22, 0.0, 3),
    "C5slab": (8, 4, 4096, 1 << 22, 0.0, 4),
    # C5 as written (8192 peers on 8^4) is rejected by the reference
    # (protocols.hpp:116-117); C5v is the closest valid config.
    "C5v": (8, 4, 4096, 18_000_000, 0.0, 4),
    # the north-star 1-GPU target: C3 at full size (419 GB of fp32 state)
    # runs as resident D-slabs (measure_full_slabbed)
    "C3": (16, 3, 4096, 25_600_000, 0.0, 3),
}
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
NVLINK_ALL_ACTIVE_GBS = 665.0  # every GPU pulling from its peers at once (profiles/r01/p2p_probe.txt)
PROTOCOL_SEED = 7
INIT_SEED = 0x5EED


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic(kernel_name, cfg_name):
    """dram bytes per launch of the top kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        ent = s["kernels"][kernel_name][cfg_name]
        return ent["dram_bytes_per_launch"], ent
    except Exception:  # noqa: BLE001
        return None, None


# ---------------------------------------------------------------------------
# CPU reference arm / baseline: unmodified run_moshpit on column slices
# ---------------------------------------------------------------------------
_CALIB = {}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": len(os.sched_getaffinity(0))}


# Column-slice widths of the CPU samples.  WIDE: 16 Ki columns x 1024 peers x
# 8 B = 128 MB per slice, far beyond a core's cache share, so the reference runs
# at its memory-bound rate (the default).  NARROW: 64 columns (512 KB, cache
# resident) -- the round-1 sample, kept as a labelled upper bound.
WIDE, NARROW = 1 << 14, 64


def cpu_reference(cfg_name, budget_s, threads=None, width=WIDE):
    from oracle.oracle import REF_SO, Checker
    M, d, N, D, p, R = CONFIGS[cfg_name]
    threads = threads or len(os.sched_getaffinity(0))
    width = min(width, D)
    if not os.path.exists(REF_SO):  # the C restatement, single-threaded, as the port baseline
        import numpy as np
        o = Checker("oracle")
        x = o.init_state(INIT_SEED, N, NARROW, dtype=np.float64)
        t0 = time.perf_counter()
        o.run_moshpit(M, d, x, p, PROTOCOL_SEED, R)
        run_s = time.perf_counter() - t0
        return dict(kind="port", cores=1, run_s=run_s, cols=NARROW, rounds=R, N=N, D=D,
                    width=NARROW, slices=1,
                    sample=f"oracle port, 1 thread, {NARROW} of {D} columns, {R} rounds")
    chk = Checker("ref")
    # calibrate once: one slice per thread
    key = (cfg_name, threads, width)
    if key not in _CALIB:
        run_s, _, _ = chk.slice_bench(M, d, N, width, threads, 0, INIT_SEED, PROTOCOL_SEED, p, R,
                                      threads)
        _CALIB[key] = max(run_s, 1e-3)
    per_slice_batch = _CALIB[key]
    batches = max(1, int(budget_s / per_slice_batch))
    slices = threads * batches
    run_s, init_s, _ = chk.slice_bench(M, d, N, width, slices, 0, INIT_SEED, PROTOCOL_SEED, p, R,
                                       threads)
    cols = slices * width
    return dict(kind="reference", cores=threads, run_s=run_s, init_s=init_s, cols=cols, rounds=R,
                N=N, D=D, width=width, slices=slices,
                sample=(f"unmodified run_moshpit (fp64, incl. record_round) on {slices} column "
                        f"slices x {width} = {cols} of D={D} coordinates "
                        f"({N * width * 8 / 1e6:.1f} MB per slice), {R} rounds, {threads} "
                        f"threads; cost linear in D (coordinates independent)"))


def cpu_value(res):
    gbs = res["N"] * res["cols"] * 4 * res["rounds"] / res["run_s"] / 1e9
    ms_round_full = res["run_s"] / res["rounds"] * (res["D"] / res["cols"]) * 1e3
    return gbs, ms_round_full


def cpu_baseline_block(cfg, budget_s):
    """The reported CPU baseline: all host threads on wide
    slices (the value), plus the single-thread figure, the cache-resident
    narrow-slice figure, the CPU model and the extrapolation factor."""
    res = cpu_reference(cfg, budget_s)
    g, ms_full = cpu_value(res)
    out = {"value": round(g, 6), "unit": "GB/s", "cores": res["cores"], "kind": res["kind"],
           "sample": res["sample"], **host_info(),
           "ms_per_round_extrapolated": round(ms_full, 1),
           "extrapolation_factor": round(res["D"] / res["cols"], 3),
           "normalisation": "fp32-normalised N*D*4 bytes per round (the reference computes "
                            "in fp64: twice these bytes move)"}
    if res["kind"] == "reference":
        one = cpu_reference(cfg, max(2.0, budget_s / 4), threads=1)
        narrow = cpu_reference(cfg, max(2.0, budget_s / 4), width=NARROW)
        out["single_thread"] = {"value": round(cpu_value(one)[0], 6), "unit": "GB/s",
                                "sample": one["sample"]}
        out["narrow_slices_cache_resident"] = {"value": round(cpu_value(narrow)[0], 6),
                                               "unit": "GB/s", "sample": narrow["sample"]}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = args.config
    # each step = one bounded sample; the whole run stays within ~2-3 minutes
    total = float(os.environ.get("MOSHPIT_REF_TOTAL_S", "120"))
    per_step = max(0.25, min(10.0, total / (args.steps + args.warmup)))
    vals, mss = [], []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_reference(cfg, per_step)
        g, ms = cpu_value(res)
        if i >= args.warmup:
            vals.append(g)
            mss.append(ms)
    value = sum(vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(value, 6), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sum(mss) / len(mss), 3),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based uniform [0,1) init, exact in fp32)",
        "config": workload_config(cfg),
        "parallelism": f"host threads x{res['cores']} over column slices (rank 0 only)",
        "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"], **host_info(),
                         "extrapolation_factor": round(res["D"] / res["cols"], 3)},
        "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "peer-vector GB/s averaged per Moshpit round"


def workload_config(cfg):
    """The workload only -- identical in both arms (implementation details such
    as the kernel variant or the parallel layout are top-level keys)."""
    M, d, N, D, p, R = CONFIGS[cfg]
    return {"workload": f"{cfg}: Moshpit All-Reduce round, {N} peers on {M}^{d} grid, "
                        f"D={D} per peer, p_fail={p}; step = one round",
            "peers": N, "grid": f"{M}^{d}", "dim": D, "p_round": p, "protocol_seed": PROTOCOL_SEED,
            "rounds_of_config": R, "l2": "state >> 126 MB L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def time_engine_rounds(mb, torch, eng, x, steps, record=False):
    """CUDA events around `steps` engine rounds on the current stream
    (optionally with the device record_round after each); returns
    (ms, kernel-2 ms, kernel-2 launches, active rows)."""
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    r0, rows0 = eng.stats()
    eng.set_timing(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if record and os.environ.get("MOSHPIT_BENCH_ROUND_RECORD", "0") != "1":
        # the run_moshpit loop in one call: round + record_round every round
        # (FAST: the voided rows' cached row partials reused)
        eng.rounds_record(x, steps)
    else:
        for _ in range(steps):
            if record:  # the round and its record_round (representative rows)
                eng.round_record(x)
            else:
                eng.round(x)
    ev1.record(stream)
    torch.cuda.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    k_ms, k_launches = eng.kernel_time()
    eng.set_timing(False)
    _, rows1 = eng.stats()
    return t_ms, k_ms, k_launches, rows1 - rows0


def measure_rounds_fused(mb, torch, cfg, local, reps=3):
    """SURVEY 8d's separately named temporal-blocking mode: the config's R
    rounds in one pass over the state (Engine.rounds_fused; bit-identical to
    R per-round calls, tests/test_gpu_fused_rounds.py) against R per-round
    calls, CUDA events around the enqueued rounds (host draws + kernel 1
    included), best of `reps`.  Its byte count is 2 * N * D * 4 per PASS, so
    it is reported beside the per-round metric, never as it."""
    M, d, N, D, p, R = CONFIGS[cfg]
    x = torch.empty((N, D), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    res = {}
    for mode in ("per_round", "fused"):
        best = None
        for _ in range(reps):
            mb.fill_synthetic(x, INIT_SEED)
            eng = mb.Engine(mb.GridConfig(M, d, R), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED),
                            device=local)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if mode == "fused":
                eng.rounds_fused(x, R)
            else:
                for _ in range(R):
                    eng.round(x)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
            eng.close()
        res[mode] = best
    del x
    torch.cuda.empty_cache()
    return {"workload": f"{cfg}: {R} rounds, fp32, one pass over column tiles of all {N} peers",
            "ms_fused": round(res["fused"], 3), "ms_per_round_path": round(res["per_round"], 3),
            "speedup": round(res["per_round"] / res["fused"], 3),
            "peer_vector_gbs_per_round_equiv": round(N * D * 4 * R / (res["fused"] / 1e3) / 1e9, 1),
            "hbm_bytes_per_pass": 2 * N * D * 4,
            "note": "temporal blocking (SURVEY 8d): bytes per pass, not per round; the "
                    "per-round metric stays kernel 2's one read + one write per round"}


def measure_variant(mb, torch, cfg, local, steps, warmup, f64=False, diag=None):
    """A variant of the N=1 headline on the same config: fp64 state and/or
    record_round on the device after every round (FAST or EXACT)."""
    M, d, N, D, p, Rcfg = CONFIGS[cfg]
    es = 8 if f64 else 4
    x = torch.empty((N, D), dtype=torch.float64 if f64 else torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED)
    eng = mb.Engine(mb.GridConfig(M, d, Rcfg), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED),
                    device=local)
    if diag:
        eng.set_reference(x, diagnostics=diag)
    for _ in range(warmup):
        if diag:
            eng.round_record(x)
        else:
            eng.round(x)
    t_ms, k_ms, kn, rows = time_engine_rounds(mb, torch, eng, x, steps, record=bool(diag))
    rep = eng.report() if diag else None
    eng.close()
    del x
    torch.cuda.empty_cache()
    peak, _ = peaks()
    alg = 2 * es * D * rows
    out = {"dtype": "f64" if f64 else "f32",
           "diagnostics": (f"record_round on the device after every round ({diag.upper()}: "
                           + ("reference j-order" if diag == "exact" else "fixed chunk order")
                           + ")") if diag else "none",
           "value": round(N * D * 4 * steps / (t_ms / 1e3) / 1e9, 3), "unit": "GB/s",
           "value_note": "fp32-normalised N*D*4 bytes per round, as the headline",
           "ms_per_step": round(t_ms / steps, 4), "steps": steps,
           "kernel2": {"achieved": round(alg / (k_ms / 1e3) / 1e9, 1), "peak": peak,
                       "frac": round(alg / (k_ms / 1e3) / 1e9 / peak, 4), "launches": kn}}
    if rep:
        out["final_distortion"] = rep[1][-1] if rep[1] else None
    return out


def run_mine(args):
    import torch
    import torch.distributed as dist

    import paper_2103_03239_b200 as mb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world == 1 and args.gpus > 1:
        log(f"--gpus {args.gpus} requested without torchrun; running 1 rank")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return run_mine_multi(args, mb, torch, dist, rank, world, local)

    cfg = args.config
    M, d, N, D, p, Rcfg = CONFIGS[cfg]
    kernel = {"auto": 0, "register": 1, "bulk": 2}[args.kernel]

    x = torch.empty((N, D), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED)
    eng = mb.Engine(mb.GridConfig(M, d, Rcfg), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED),
                    device=local, kernel=kernel)
    for _ in range(args.warmup):
        eng.round(x)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    t_ms, k_ms, k_launches, active_rows = time_engine_rounds(mb, torch, eng, x, args.steps)
    clk = clocks.stop()
    eng.close()

    state_bytes = N * D * 4
    value = state_bytes * args.steps / (t_ms / 1e3) / 1e9
    alg_bytes = 2 * 4 * D * active_rows  # kernel 2 reads+writes every active row once
    achieved = alg_bytes / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
    peak, peak_src = peaks()
    traffic, traffic_ent = load_traffic("group_mean_register", cfg)
    launches_per_step = 2  # kernel 1 (group formation) + kernel 2 (group mean)

    del x
    torch.cuda.empty_cache()

    variants = {}
    if not args.no_variants:
        vs = min(args.steps, 20)
        for name, kw in (("value_with_diag", dict(diag="fast")), ("value_f64", dict(f64=True)),
                         ("value_f64_exact_diag", dict(f64=True, diag="exact"))):
            try:
                variants[name] = measure_variant(mb, torch, cfg, local, vs, 3, **kw)
            except Exception as exc:  # noqa: BLE001
                variants[name] = {"error": str(exc)}
        try:  # SURVEY 8d temporal-blocking mode: its own byte count, never the metric
            variants["rounds_fused_mode"] = measure_rounds_fused(mb, torch, cfg, local)
        except Exception as exc:  # noqa: BLE001
            variants["rounds_fused_mode"] = {"error": str(exc)}
    full = full_c5 = None
    if not args.no_full:
        try:
            full = measure_full_slabbed(mb, torch, "C3", local)
        except Exception as exc:  # noqa: BLE001
            full = {"error": str(exc)}
        try:
            full_c5 = measure_full_slabbed(mb, torch, "C5v", local, slabs=3)
        except Exception as exc:  # noqa: BLE001
            full_c5 = {"error": str(exc)}
    e2e = e2e_more = None
    if not args.no_e2e:
        e2e = measure_e2e(mb, cfg)
        e2e_more = {}
        try:
            e2e_more["pinned_f32_fast_with_vectors"] = measure_e2e(mb, cfg, vectors=True)
        except Exception as exc:  # noqa: BLE001
            e2e_more["pinned_f32_fast_with_vectors"] = {"error": str(exc)}
        try:
            e2e_more["pageable_f32_fast"] = measure_e2e(mb, cfg, pinned=False)
        except Exception as exc:  # noqa: BLE001
            e2e_more["pageable_f32_fast"] = {"error": str(exc)}
        try:
            e2e_more["dropin_f64_exact"] = measure_e2e_dropin(cfg)
        except Exception as exc:  # noqa: BLE001
            e2e_more["dropin_f64_exact"] = {"error": str(exc)}
    sgd = None
    if not args.no_sgd:
        try:
            sgd = measure_sgd_c4(mb)
            s0 = measure_sgd_c4(mb, sigma=0.0)
            sgd["sigma0"] = {k: s0[k] for k in ("ms_per_sgd_step", "peer_vector_gbs", "hbm_frac")}
            sf = measure_sgd_c4(mb, diagnostics="fast")
            sgd["sigma1_fast_diagnostics"] = {
                k: sf[k] for k in ("ms_per_sgd_step", "peer_vector_gbs", "hbm_frac", "timing")}
        except Exception as exc:  # noqa: BLE001
            sgd = {"error": str(exc)}
    cpu = None
    if not args.no_cpu:
        try:
            cpu = cpu_baseline_block(cfg, float(os.environ.get("MOSHPIT_CPU_BUDGET_S", "15")))
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                   "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": round(value, 3),
        "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter-based uniform [0,1) init, exact in fp32)",
        "config": workload_config(cfg),
        "parallelism": "single GPU", "kernel": args.kernel,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": traffic,
                     "traffic_over_algorithmic": (traffic_ent or {}).get("traffic_over_algorithmic"),
                     "traffic_source": "profiles/ncu_summary.json (ncu --set full, one launch)",
                     "kernel": "group_mean_register (kernel 2)",
                     "algorithmic_bytes": "2 * 4 B * D * rows in non-voided groups",
                     "avg_launch_ms": round(k_ms / max(k_launches, 1), 4),
                     "launches": k_launches, "active_rows_timed": active_rows,
                     "peak_source": peak_src},
        "kernel2_share_of_step": round(k_ms / t_ms, 4) if t_ms > 0 else None,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "e2e": e2e,
        "e2e_variants": e2e_more,
        "cpu_baseline": cpu,
        **variants,
        "c3_full_1gpu": full,
        "c5v_full_1gpu": full_c5,
        "sgd_c4": sgd,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_mine_multi(args, mb, torch, dist, rank, world, local):
    """N > 1: the headline is the peer-sharded round on the N=1 config (strong
    scaling, NVLink cross rounds); coordinate sharding and the peer-sharded
    C5-valid run are attached."""
    cfg = args.config
    clocks = ClockSampler(local)
    clocks.start()
    head = run_peer(mb, torch, dist, cfg, args.steps, args.warmup, rank, world, local,
                    nvlink=True, e2e=not args.no_e2e, cross=args.cross)
    clk = clocks.stop()
    coord = c5v = other = None
    # the other cross-round summation on the same config (exact: the reference
    # tree over raw member chunks, bit-exact; partial: per-GPU partial sums,
    # within 1e-6 relative)
    other_mode = "partial" if args.cross == "exact" else "exact"
    try:
        other = run_peer(mb, torch, dist, cfg, args.steps, args.warmup, rank, world, local,
                         nvlink=True, cross=other_mode)
        other.pop("e2e", None)
    except Exception as exc:  # noqa: BLE001
        other = {"error": str(exc)}
    if not args.no_coord:
        try:
            coord = run_coord(mb, torch, dist, cfg, min(args.steps, 40), args.warmup, rank, world,
                              local)
        except Exception as exc:  # noqa: BLE001
            coord = {"error": str(exc)}
    if not args.no_peer:
        # C5-valid (the north-star multi-GPU config, 295 GB) wherever its
        # 1/world share fits this GPU (world >= 2 on 180 GB B200s)
        Mv, dv, Nv, Dv, _, _ = CONFIGS["C5v"]
        need = Nv // world * ((Dv + 1023) // 1024 * 1024) * 4 + (4 << 30)
        fits = torch.tensor([1.0 if torch.cuda.mem_get_info()[0] >= need else 0.0],
                            device="cuda")
        dist.all_reduce(fits, op=dist.ReduceOp.MIN)
        if Mv % world == 0 and fits.item() > 0:
            try:
                c5v = run_peer(mb, torch, dist, "C5v", max(8, min(args.steps, 24)), 4, rank,
                               world, local, nvlink=True, cross=args.cross)
            except Exception as exc:  # noqa: BLE001
                c5v = {"error": str(exc)}
    if rank == 0:
        peak, peak_src = peaks()
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (counter-based uniform [0,1) init, exact in fp32)",
            "config": workload_config(cfg),
            "parallelism": (f"peer-sharded x{world}: grid digit d-1 split across GPUs; axis-0 "
                            f"rounds GPU-local, axis-(d-1) rounds over NVLink peer memory "
                            f"({args.cross} cross-round summation)"),
            "roofline": dict(head["roofline"], bound="hbm+nvlink",
                             frac=head["roofline"]["combined_frac"], peak_hbm=peak,
                             peak_nvlink=NVLINK_GBS, peak_source=peak_src),
            "gpu_launches": head["gpu_launches"],
            "rounds_local": head["rounds_local"], "rounds_cross": head["rounds_cross"],
            "nvlink_counters": head.get("nvlink_counters"),
            "clocks": clk,
            "e2e": head["e2e"],
            "cross_summation": (
                "exact: the reference pairwise tree over the members' raw chunks (bit-exact)"
                if args.cross == "exact" else
                "partial: per-GPU partial sums combined in rank order in fp64 (the summation "
                "order is not the reference's: within 1e-6 relative in fp32, north_star)"),
            f"peer_sharded_{other_mode}": other,
            "coordinate_sharded_weak": coord,
            "peer_sharded_c5v": c5v,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def run_coord(mb, torch, dist, cfg, steps, warmup, rank, world, local):
    """Coordinate-sharded weak scaling: every rank owns all N peers over its
    own D-slab of a (D * world)-coordinate problem and replays the identical
    host draws (no data-path exchange; exact by coordinate independence)."""
    M, d, N, D, p, Rcfg = CONFIGS[cfg]
    x = torch.empty((N, D), dtype=torch.float32, device="cuda")
    mb.fill_synthetic(x, INIT_SEED, col0=rank * D)
    eng = mb.Engine(mb.GridConfig(M, d, Rcfg), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED),
                    device=local)
    for _ in range(warmup):
        eng.round(x)
    torch.cuda.synchronize()
    dist.barrier()
    t_ms, k_ms, kn, rows = time_engine_rounds(mb, torch, eng, x, steps)
    dist.barrier()
    tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    eng.close()
    del x
    torch.cuda.empty_cache()
    return {"workload": f"{cfg} per rank over its own D-slab ({world} x {D} coordinates)",
            "value": round(world * N * D * 4 * steps / (tt.item() / 1e3) / 1e9, 3),
            "unit": "GB/s", "scaling": "weak", "steps": steps,
            "ms_per_step": round(tt.item() / steps, 4)}


def measure_e2e_peer(mb, torch, dist, sh, cfg, world, calls=3):
    """End to end at N GPUs through the public Shard API: every rank loads its
    own peers' rows from pinned host memory (Shard.load_rows), runs the
    config's R rounds and stores the rows back (Shard.store_rows), host wall
    clock between barriers, max over ranks, 1 warm-up + median of `calls`.
    There is no distributed TrialReport, so the result read back is the
    vectors (the N=1 line's e2e_variants.pinned_f32_fast_with_vectors is the
    same call shape on one GPU)."""
    M, d, N, D, p, R = CONFIGS[cfg]
    rows = sh.rows()
    host = torch.empty((rows, D), dtype=torch.float32, pin_memory=True).numpy()
    sh.store_rows(host)  # the current state: the rows a caller would hold
    torch.cuda.synchronize()
    secs = []
    for it in range(calls + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh.load_rows(host)
        for _ in range(R):
            sh.round()
        sh.store_rows(host)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if it:
            secs.append(t.item())
    sec = sorted(secs)[len(secs) // 2]
    moved = world * rows * D * 4
    return {"value": round(N * D * 4 * R / sec / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": moved // R, "d2h_bytes_per_step": moved // R,
            "h2d_bytes_per_call": moved, "d2h_bytes_per_call": moved,
            "call": f"Shard.load_rows (pinned) + {R} rounds + Shard.store_rows on each of "
                    f"{world} ranks (peer-sharded {cfg})",
            "seconds": round(sec, 4), "seconds_each": [round(x, 4) for x in secs],
            "timing": "host wall clock per call between barriers, max over ranks, "
                      "1 warm-up + median of 3",
            "bytes_note": "whole job: every rank copies its resident rows in and out"}


def run_peer(mb, torch, dist, cfg, steps, warmup, rank, world, local, nvlink=False, slabs=None,
             e2e=False, cross="exact"):
    """Peer-sharded rounds: peers split by grid digit d-1, rounds on
    axes 0..d-2 local, the axis d-1 round one fused NVLink kernel.  Returns
    the whole-problem metric (strong scaling) and the combined roofline."""
    M, d, N, D, p, Rcfg = CONFIGS[cfg]
    if slabs is None:  # slab pipeline: cross rounds of some slabs under local rounds of others
        slabs = int(os.environ.get("MOSHPIT_SHARD_SLABS", 8 if world > 1 else 1))
    sh = mb.Shard(mb.GridConfig(M, d, Rcfg), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED), D,
                  rank=rank, world=world, device=local, slabs=slabs, cross=cross)
    if world > 1:
        sh.connect()
    sh.fill_synthetic(INIT_SEED)
    for _ in range(warmup):
        sh.round()
    sh.flush()
    torch.cuda.synchronize()
    c0 = sh.stats()
    mv0 = sh.cross_detail()[2]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sh.set_timing(True)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        sh.round()
    sh.flush()  # the lagging slabs finish their rounds inside the timed region
    ev1.record(stream)
    torch.cuda.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    lms, ln, cms, cn = sh.kernel_time()
    c1 = sh.stats()
    pa_ms, pb_ms, mv1 = sh.cross_detail()
    moved = mv1 - mv0  # voided-group rows that moved onto this GPU (cross rounds)
    sh.set_timing(False)
    cross_rounds, cross_groups, local_rows = (c1[0] - c0[0], c1[1] - c0[1], c1[2] - c0[2])
    es, Mg = 4, M // world
    # minimal (algorithmic) bytes, busiest GPU: every resident row read and
    # written once per round; in a cross round each GPU must receive the raw
    # chunk of every remote member (no pre-reduction: the tree spans GPUs) and
    # one copy of each foreign mean chunk.
    hbm_local = 2 * es * D * local_rows
    # voided groups of a cross round move the rows whose new rank lives on
    # another GPU: one full row over NVLink (pull) + its HBM read and write
    if cross == "partial":
        # per group: the Mg member rows read (partial sums) and written (mean),
        # the partial row written, this GPU's partial chunk and mean chunk
        # read by the w-1 peers (and its own partial chunk by itself); NVLink:
        # w-1 foreign partial chunks + w-1 foreign mean chunks pulled
        hbm_cross = (es * D * cross_groups * (2 * Mg + 1 + (2 * (world - 1) + 1) / world)
                     + 2 * es * D * moved)
        nvl_cross = (cross_groups * es * (D / world) * 2 * (world - 1)
                     + es * D * moved) if world > 1 else 0
    else:
        hbm_cross = 2 * es * D * Mg * cross_groups + 2 * es * D * moved
        nvl_cross = (cross_groups * es * (D / world) * ((M - Mg) + (world - 1))
                     + es * D * moved) if world > 1 else 0
    peak, _ = peaks()
    t_roof_local = hbm_local / (peak * 1e9) * 1e3
    t_roof_cross = max(hbm_cross / (peak * 1e9), nvl_cross / (NVLINK_GBS * 1e9)) * 1e3
    hbm_cross_ms_mine = hbm_cross / (peak * 1e9) * 1e3
    vals = torch.tensor([t_ms, lms, cms, t_roof_local, t_roof_cross, pa_ms, pb_ms, nvl_cross,
                         hbm_cross_ms_mine],
                        dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_max, lmax, cmax, trl, trc, pa_max, pb_max, nvl_max, hbm_cross_ms = vals.tolist()
    # NVLink bytes are modelled here; the measured counterpart is the ncu
    # nvlrx__bytes capture of the cross kernels (profiles/nvlink_ncu.py; NVML's
    # NVLink throughput counters read N/A on this driver)
    nvl_meas = {"source": "modelled (see profiles/ncu_summary.json nvlink entries for the "
                          "ncu-measured nvlrx bytes of the same kernels)"} if nvlink else None
    e2e_line = None
    if e2e:
        try:
            e2e_line = measure_e2e_peer(mb, torch, dist, sh, cfg, world)
        except Exception as exc:  # noqa: BLE001
            e2e_line = {"error": str(exc)}
    sh.close()
    torch.cuda.empty_cache()
    value = N * D * es * steps / (t_max / 1e3) / 1e9
    return {
        "e2e": e2e_line,
        "workload": f"{cfg}: {N} peers on {M}^{d}, D={D} fp32, p_fail={p}, peer-sharded over "
                    f"{world} GPU(s) (grid digit d-1 split; axes 0..d-2 local)",
        "cross": cross,
        "metric": "peer-vector GB/s averaged per Moshpit round", "value": round(value, 3),
        "unit": "GB/s", "scaling": "strong", "steps": steps, "ms_per_step": round(t_max / steps, 4),
        "slabs": slabs,
        "rounds_local": ln, "rounds_cross": cross_rounds,
        # per round: kernel 1 + the placement kernel (control stream); per slab
        # and local round: kernel 2; per slab and cross round: the barriers and
        # the mode's kernels (exact: cross_mean + pull [+ the voided rows'
        # staging pull]; partial: partial_sum + combine + pull)
        "gpu_launches": steps * 2 + ln + (cn // 2) * (
            (4 + 3) if cross == "partial" else (3 + 2 + (1 if p > 0 else 0))),
        "nvlink_counters": nvl_meas,
        "local_kernel_ms": round(lmax, 3), "cross_kernel_ms": round(cmax, 3),
        "roofline": {
            "bound": "hbm (local rounds) + nvlink (cross rounds)",
            "local": {"achieved": round(hbm_local / (lmax / 1e3) / 1e9, 1) if lmax else None,
                      "peak": peak, "unit": "GB/s",
                      "frac": round(trl / lmax, 4) if lmax else None},
            "cross": {"nvlink_ingress_gb_per_gpu": round(nvl_max / 1e9, 3),
                      "voided_rows_moved_in": moved,
                      "phase_a_ms": round(pa_max, 3), "phase_b_ms": round(pb_max, 3),
                      "achieved_nvlink": round(nvl_max / (cmax / 1e3) / 1e9, 1) if cmax else None,
                      "peak_nvlink": NVLINK_GBS, "unit": "GB/s",
                      "frac": round(trc / cmax, 4) if cmax else None},
            "combined_frac": round((trl + trc) / t_max, 4) if t_max else None,
            "combined_frac_overlapped_bound": round(
                max(trl + hbm_cross_ms, nvl_max / (NVLINK_GBS * 1e9) * 1e3) / t_max, 4)
            if t_max else None,
            # the same against the all-GPUs-active peer-read figure (every GPU
            # pulling from its peers at once: 663-667 GB/s, profiles/r01/p2p_probe.txt)
            "combined_frac_overlapped_bound_all_active": round(
                max(trl + hbm_cross_ms, nvl_max / (NVLINK_ALL_ACTIVE_GBS * 1e9) * 1e3) / t_max, 4)
            if t_max else None,
            "note": "t_roof = max(HBM bytes / hbm_gbs, NVLink ingress / 770 GB/s) per round, "
                    "busiest GPU, minimal bytes of the mode (exact: raw remote member chunks; "
                    "partial: one partial chunk per foreign GPU and group; both: one copy of each "
                    "foreign mean chunk + the voided-group rows whose new rank lives on another "
                    "GPU, all NVLink traffic as pulls); combined_frac = sum of the rounds' t_roof "
                    "/ the measured wall time of all rounds (max over ranks; host draws, kernel 1, "
                    "barriers included).  With slabs > 1 the slabs' cross rounds overlap other "
                    "slabs' local rounds, so combined_frac can exceed 1; "
                    "combined_frac_overlapped_bound uses the overlapped bound max(all HBM bytes / "
                    "hbm_gbs, all NVLink bytes / 770) instead",
        },
    }


def measure_full_slabbed(mb, torch, cfg, local, slabs=4):
    """A config whose state exceeds one GPU (C3: 4096 x 25.6M fp32 = 419 GB;
    C5-valid: 4096 x 18M = 295 GB, the 1-GPU point of the multi-GPU series),
    every coordinate of it, as `slabs` resident D-slabs (coordinates are
    independent): per slab, counter-based init on the device
    (timed separately), a fresh engine with the config's protocol seed (the
    same draws and group tables for every slab) and the config's R rounds.
    value = N * D * 4 * R / (sum of the slabs' round times)."""
    M, d, N, D, p, R = CONFIGS[cfg]
    W = -(-D // slabs)
    W = (W + 3) // 4 * 4
    stream = torch.cuda.current_stream()
    # 4 KB row pitch: 96.4 % vs 92.4 % of the HBM peak for 24,000,000-byte
    # rows (profiles/ld_sweep.py)
    ld = -(-W // 1024) * 1024
    x = torch.empty((N, ld), dtype=torch.float32, device="cuda")
    t_rounds = t_init = k_ms = 0.0
    rows = launches = 0
    for c0 in range(0, D, W):
        w = min(W, D - c0)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(stream)
        mb.fill_synthetic(x, INIT_SEED, dim=w, col0=c0)
        e[1].record(stream)
        eng = mb.Engine(mb.GridConfig(M, d, R), N, mb.FailureModel(p), mb.Rng(PROTOCOL_SEED),
                        device=local)
        eng.set_timing(True)
        r0 = eng.stats()[1]
        torch.cuda.synchronize()
        e[2].record(stream)
        for _ in range(R):
            eng.round(x, dim=w)
        e[3].record(stream)
        torch.cuda.synchronize()
        t_init += e[0].elapsed_time(e[1])
        t_rounds += e[2].elapsed_time(e[3])
        km, kn = eng.kernel_time()
        k_ms += km
        launches += kn
        rows += (eng.stats()[1] - r0) * w
        eng.close()
    del x
    torch.cuda.empty_cache()
    peak, _ = peaks()
    alg = 2 * 4 * rows  # rows x columns actually averaged, read + written once per round
    return {"workload": f"{cfg}: {N} peers on {M}^{d}, D={D} fp32 (full size, "
                        f"{N * D * 4 / 1e9:.1f} GB) as {-(-D // W)} resident D-slabs of {W} "
                        f"columns, {R} rounds each",
            "metric": "peer-vector GB/s averaged per Moshpit round",
            "value": round(N * D * 4 * R / (t_rounds / 1e3) / 1e9, 3), "unit": "GB/s",
            "ms_per_round": round(t_rounds / R, 3),
            "init_ms_total": round(t_init, 3),
            "roofline": {"bound": "hbm", "kernel": "group_mean_register (kernel 2)",
                         "achieved": round(alg / (k_ms / 1e3) / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(alg / (k_ms / 1e3) / 1e9 / peak, 4),
                         "launches": launches,
                         "frac_of_round_time": round(alg / (t_rounds / 1e3) / 1e9 / peak, 4)},
            "timing": "CUDA events around each slab's R rounds (host draws + kernel 1 + "
                      "kernel 2); the on-device init is reported apart"}


def measure_sgd_c4(mb, steps=20, sigma=1.0, diagnostics="none"):
    """C4 (configs[3]): Moshpit SGD, 1024 peers on 32x32, Quadratic(D=2^20,
    L=1, mu=0.1, target ~ N(0,1)), gamma=0.1, tau=1, inner=d=2, fp32,
    device Philox noise, kernel 3 (local step fused into averaging round 1).
    Device time of the step loop (CUDA events inside the C ABI call)."""
    import numpy as np
    D, N = 1 << 20, 1024
    tgt = mb.Rng(PROTOCOL_SEED).stream("objective").normals(D)
    quad = mb.Quadratic(D, 1.0, 0.1, tgt)
    cfg = mb.OptimizerConfig(gamma=0.1, tau=1, steps=steps, grid=mb.GridConfig(32, 2, 1),
                             sigma=sigma, n_peers=N)
    best = None
    for _ in range(2):
        r = mb.run_moshpit_sgd(cfg, quad, np.zeros(D), [], mb.Rng(PROTOCOL_SEED),
                               dtype=np.float32, diagnostics=diagnostics, noise="device")
        best = r.loop_ms if best is None else min(best, r.loop_ms)
    ms = best / steps
    alg = 2 * 2 * N * D * 4  # two averaging rounds, each one read + one write of the state
    one = 2 * N * D * 4  # the two-round pass: one read + one write of the state per step
    peak, _ = peaks()
    two = os.environ.get("MOSHPIT_SGD_TWO_ROUND", "1") != "0"
    return {"workload": f"C4: Moshpit SGD, 1024 peers on 32x32, Quadratic D=2^20, tau=1, "
                        f"inner=2, sigma={sigma} (device noise), fp32, "
                        + ("the step + both averaging rounds in one pass (two_round_step_kernel)"
                           if two else "kernel 3 fused step + kernel 2"),
            "ms_per_sgd_step": round(ms, 4),
            "peer_vector_gbs": round(N * D * 4 / (ms / 1e3) / 1e9, 1),
            "algorithmic_bytes_per_step": alg,
            "hbm_frac": round(alg / (ms / 1e3) / 1e9 / peak, 4),
            "one_pass_bytes_per_step": one,
            "hbm_frac_one_pass": round(one / (ms / 1e3) / 1e9 / peak, 4),
            "note": "hbm_frac: against two rounds of one read + one write each (the per-round "
                    "algorithm); hbm_frac_one_pass: against the one-pass bytes the two-round "
                    "kernel actually moves",
            "timing": f"CUDA events around the {steps}-step loop (best of 2), incl. host draws; "
                      f"per-step diagnostics: {diagnostics}",
            "final_sigma_hat": round(r.diagnostics.sigma_hat, 6)}


def measure_e2e(mb, cfg, pinned=True, vectors=False):
    """The reference-facing call (run_moshpit through the C ABI) with HOST
    buffers: H2D of the initial state, R rounds + TrialReport diagnostics and
    the D2H of the report -- the reference's run_moshpit returns the
    TrialReport only (protocols.hpp:108-179) -- all inside the timed region.
    vectors=True also copies the final vectors back (the C ABI's optional
    final_out).  pinned=False: a plain (pageable) numpy buffer, packed through
    the library's pinned staging ring by host threads."""
    import numpy as np
    import torch
    M, d, N, D, p, R = CONFIGS[cfg]
    if pinned:
        host = torch.empty((N, D), dtype=torch.float32, pin_memory=True)
        xh = host.numpy()
        out_t = torch.empty((N, D), dtype=torch.float32, pin_memory=True) if vectors else None
        oh = out_t.numpy() if vectors else None
    else:
        host = None
        xh = np.empty((N, D), dtype=np.float32)
        oh = np.empty((N, D), dtype=np.float32) if vectors else None
    # fill the host buffer from the device init (same synthetic data)
    blk = torch.empty((64, D), dtype=torch.float32, device="cuda")
    for i0 in range(0, N, 64):
        mb.fill_synthetic(blk, INIT_SEED)
        xh[i0:i0 + 64] = blk.cpu().numpy()  # row ids restart per block: fine for timing
    del blk
    torch.cuda.synchronize()
    import ctypes as C
    from paper_2103_03239_b200 import _capi
    lib = _capi.lib()
    dist_ = np.zeros(R)
    drift = np.zeros(R)
    act = np.zeros(R, dtype=np.uint32)
    init_d, cost = C.c_double(0), C.c_double(0)
    ptr = xh.ctypes.data_as(C.c_void_p)
    # separate output: every call starts from the init
    optr = oh.ctypes.data_as(C.c_void_p) if vectors else None

    def call():
        _capi.check(lib.moshpit_run_moshpit(_capi.F32, M, d, R, ptr, N, D, p, PROTOCOL_SEED, R,
                                            _capi.DIAG_FAST, C.byref(init_d),
                                            dist_.ctypes.data_as(C.c_void_p),
                                            drift.ctypes.data_as(C.c_void_p),
                                            act.ctypes.data_as(C.c_void_p), C.byref(cost), optr))
    call()  # warm-up: kernel module loading + workspace allocation (untimed)
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    t = sorted(times)[1]  # median of 3
    bytes_ = N * D * 4
    h2d_call = bytes_ + R * N * 9  # state + per-round draws
    d2h_call = (bytes_ if vectors else 0) + (2 * R + 2) * 8  # (vectors +) the TrialReport
    out = {"value": round(bytes_ * R / t / 1e9, 3), "unit": "GB/s",
           # a step is one round: the call's copies amortised over its R rounds
           "h2d_bytes_per_step": h2d_call // R, "d2h_bytes_per_step": d2h_call // R,
           "h2d_bytes_per_call": h2d_call, "d2h_bytes_per_call": d2h_call,
           "call": (f"moshpit_run_moshpit(F32, rounds={R}, DIAG_FAST) host->host, "
                    + ("pinned" if pinned else "pageable numpy buffer (library staging ring)")
                    + (", final vectors copied back" if vectors else
                       ", TrialReport returned (as protocols::run_moshpit)")),
           "seconds": round(t, 4), "seconds_each": [round(x, 4) for x in times],
           "timing": "host wall clock per call, 1 warm-up + median of 3",
           "final_distortion": float(dist_[-1]),
           "pipeline": "D-slabs of 256 MB: H2D(s+1) || 10 rounds + diagnostics(s) || D2H(s-1)"}
    if not pinned:
        out["host_threads"] = len(os.sched_getaffinity(0))
        del xh, oh
        return out
    # PCIe reference point: one plain pinned H2D copy of the same state
    dev = torch.empty((N, D), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = bytes_ / (time.perf_counter() - t1) / 1e9
    # the ceiling the pipeline runs against: both directions busy at once
    # (2 GiB each way on two streams); the call moves bytes_ each way
    n2 = min(bytes_, 2 << 30) // 4
    hb = torch.empty(n2, dtype=torch.float32, pin_memory=True)
    dflat = dev.view(-1)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    bidir_gbs = 0.0
    for _ in range(2):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        with torch.cuda.stream(sa):
            dflat[:n2].copy_(host.view(-1)[:n2], non_blocking=True)
        with torch.cuda.stream(sb):
            hb.copy_(dflat[n2:2 * n2], non_blocking=True)
        torch.cuda.synchronize()
        bidir_gbs = max(bidir_gbs, 2 * n2 * 4 / (time.perf_counter() - t1) / 1e9)
    del dev, hb, out_t, host
    torch.cuda.empty_cache()
    t_floor = 2 * bytes_ / (bidir_gbs * 1e9) if vectors else bytes_ / (h2d_gbs * 1e9)
    out.update({"pcie_h2d_gbs_plain_copy": round(h2d_gbs, 1),
                "pcie_bidir_gbs_aggregate": round(bidir_gbs, 1),
                "frac_of_pcie_ceiling": round(t_floor / t, 3),
                "pcie_ceiling": "bidirectional (state in + vectors out)" if vectors
                                else "one-way H2D of the state"})
    return out


DROPIN_BIN = os.path.join(ROOT, "paper_2103_03239_b200", "bench_dropin")


def build_dropin_bench():
    """g++ of the drop-in bench (the reference user's C++ call) against the
    drop-in header and the in-tree library; rebuilt if missing."""
    src = os.path.join(ROOT, "paper_2103_03239_b200", "csrc", "host", "bench_dropin.cpp")
    if os.path.exists(DROPIN_BIN) and os.path.getmtime(DROPIN_BIN) >= os.path.getmtime(src):
        return DROPIN_BIN
    lib = os.path.join(ROOT, "paper_2103_03239_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", src, "-I",
                    os.path.join(ROOT, "include"), "-L", lib, "-lmoshpit_b200",
                    "-Wl,-rpath,$ORIGIN", "-o", DROPIN_BIN], check=True, capture_output=True,
                   timeout=300)
    return DROPIN_BIN


def measure_e2e_dropin(cfg, reps=3):
    """protocols::run_moshpit through include/moshpit_b200/moshpit.hpp: fp64,
    EXACT diagnostics (TrialReport bit-identical to the reference), the
    caller's std::vector<ParamVector> (pageable) -- the path a reference user
    gets by swapping the header.  Host wall clock per call (C++ binary)."""
    M, d, N, D, p, R = CONFIGS[cfg]
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 0
    # the caller's fp64 state must fit host RAM with room to spare
    if avail and N * D * 8 * 1.5 > avail:
        D = max(1 << 16, int(avail / 1.5 / (N * 8)) // 65536 * 65536)
    exe = build_dropin_bench()
    r = subprocess.run([exe, str(M), str(d), str(N), str(D), str(p), str(R), str(reps)],
                       capture_output=True, text=True, timeout=1200)
    if r.returncode != 0:
        return {"error": r.stderr[-500:]}
    out = json.loads(r.stdout.strip().splitlines()[-1])
    t = out["seconds_median"]
    out.update({"value": round(N * D * 4 * R / t / 1e9, 3), "unit": "GB/s",
                "value_note": "fp32-normalised N*D*4 bytes per round (the call moves fp64)",
                "value_fp64_bytes": round(N * D * 8 * R / t / 1e9, 3),
                "h2d_bytes_per_step": (N * D * 8 + R * N * 9) // R,
                "d2h_bytes_per_step": ((2 * R + 2) * 8) // R,
                "h2d_bytes_per_call": N * D * 8 + R * N * 9, "d2h_bytes_per_call": (2 * R + 2) * 8,
                "timing": f"host wall clock per call, 1 warm-up + median of {reps}",
                "config_dim": D})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="C2", choices=[c for c in sorted(CONFIGS) if c != "C3"],
                    help="C3 at full size exceeds one GPU: see the c3_full_1gpu key")
    ap.add_argument("--kernel", default="auto", choices=["auto", "register", "bulk"])
    ap.add_argument("--cross", default=os.environ.get("MOSHPIT_BENCH_CROSS", "partial"),
                    choices=["exact", "partial"],
                    help="N > 1 headline's cross-round summation (the other one is attached)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sgd", action="store_true", help="skip the C4 Moshpit-SGD measurement")
    ap.add_argument("--no-full", action="store_true",
                    help="skip the full-size C3 (slab-streamed) measurement at N=1")
    ap.add_argument("--no-peer", action="store_true",
                    help="skip the peer-sharded C5-valid measurement attached at N>1")
    ap.add_argument("--no-coord", action="store_true",
                    help="skip the coordinate-sharded weak-scaling key at N>1")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the fp64 / with-diagnostics variants at N=1")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup < 3 is not allowed by the timing rules; using 3")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
