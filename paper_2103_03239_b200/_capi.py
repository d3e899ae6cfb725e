"""ctypes binding of include/moshpit_b200.h (libmoshpit_b200.so, built in-tree).

There is no fallback: if the library is missing or a GPU entry point is
called without a device, this raises.  See INTEGRATION.md.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmoshpit_b200.so")

OK, E_INVALID, E_RANGE, E_RUNTIME, E_CUDA = 0, -1, -2, -3, -4
F32, F64 = 0, 1
DIAG_NONE, DIAG_FAST, DIAG_EXACT = 0, 1, 2
KERNEL_AUTO, KERNEL_REGISTER, KERNEL_BULK = 0, 1, 2


class MoshpitError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(MoshpitError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(MoshpitError, IndexError):
    """std::out_of_range in the reference."""


class ReferenceRuntimeError(MoshpitError):
    """std::runtime_error in the reference."""


class CudaError(MoshpitError):
    """Device or driver failure (the engine has no CPU fallback)."""


_EXC = {E_INVALID: InvalidArgument, E_RANGE: OutOfRange, E_RUNTIME: ReferenceRuntimeError,
        E_CUDA: CudaError}


class RngState(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4), ("have_spare", C.c_int32), ("spare", C.c_double)]


u64, u32, i64, i32, dbl, vp = C.c_uint64, C.c_uint32, C.c_int64, C.c_int32, C.c_double, C.c_void_p
P = C.POINTER

# name -> (restype, argtypes)
PROTOTYPES = {
    "moshpit_last_error": (C.c_char_p, []),
    "moshpit_version": (C.c_char_p, []),
    "moshpit_device_count": (C.c_int, [P(C.c_int)]),
    "moshpit_rng_stream": (C.c_int, [u64, C.c_char_p, i64, P(RngState)]),
    "moshpit_rng_seeded": (C.c_int, [u64, P(RngState)]),
    "moshpit_release_workspace": (C.c_int, []),
    "moshpit_round_from_groups": (C.c_int, [C.c_int, vp, u64, u64, u64, vp, vp, u64, vp, vp]),
    "moshpit_round_from_groups_host": (C.c_int, [C.c_int, vp, u64, u64, vp, vp, u64, vp]),
    "moshpit_run_moshpit_rows": (C.c_int, [C.c_int, u32, u32, u32, P(C.c_void_p), u64, u64,
                                           C.c_double, u64, u32, C.c_int, P(C.c_double),
                                           vp, vp, vp, P(C.c_double)]),
    "moshpit_rng_draws": (C.c_int, [P(RngState), C.c_int, u64, dbl, u64, vp]),
    "moshpit_grid_validate": (C.c_int, [u32, u32, u32]),
    "moshpit_grid_capacity": (u64, [u32, u32]),
    "moshpit_initial_index": (C.c_int, [u64, u32, u32, vp]),
    "moshpit_next_group_key": (C.c_int, [vp, u32, u32, u32, vp]),
    "moshpit_chunk_sizes": (C.c_int, [u64, vp, u64, vp]),
    "moshpit_complexity_estimate": (dbl, [u32, u32, u32, u32]),
    "moshpit_form_groups_uncontested": (C.c_int, [u64, vp, vp, u32, vp, u32, vp, vp, P(u64)]),
    "moshpit_group_mean": (C.c_int, [C.c_int, vp, u64, u64, vp, u64, vp]),
    "moshpit_butterfly_allreduce": (C.c_int, [C.c_int, vp, u64, u64, vp, u64, vp, vp, vp,
                                              P(i32)]),
    "moshpit_distortion": (C.c_int, [C.c_int, vp, u64, u64, vp, P(dbl)]),
    "moshpit_mean_of": (C.c_int, [C.c_int, vp, u64, u64, vp]),
    "moshpit_run_moshpit": (C.c_int, [C.c_int, u32, u32, u32, vp, u64, u64, dbl, u64, u32,
                                      C.c_int, P(dbl), vp, vp, vp, P(dbl), vp]),
    "moshpit_run_moshpit_batch": (C.c_int, [C.c_int, u32, u32, u32, u32, vp, u64, u64, dbl, vp,
                                            u32, C.c_int, vp, vp, vp, vp, vp, vp]),
    "moshpit_trial_seed": (u64, [u64, C.c_char_p, u32, dbl, u32]),
    "moshpit_moshpit_average": (C.c_int, [C.c_int, vp, u64, u64, u32, u32, u32, P(RngState)]),
    "moshpit_local_step_quadratic": (C.c_int, [C.c_int, vp, u64, dbl, dbl, vp, dbl, dbl,
                                               P(RngState)]),
    "moshpit_run_moshpit_sgd_quadratic": (C.c_int, [C.c_int, u32, u32, u32, u32, u64, dbl, dbl,
                                                    vp, vp, dbl, u32, u32, dbl, u32, u64, vp, vp,
                                                    u64, C.c_int, C.c_int, vp, vp, vp, vp, vp,
                                                    vp, vp, P(dbl)]),
    "moshpit_logistic_synthetic": (C.c_int, [u64, u64, P(RngState), vp, vp]),
    "moshpit_logistic_eval": (C.c_int, [vp, vp, u64, u64, dbl, vp, P(dbl), vp, P(dbl)]),
    "moshpit_local_step_logistic": (C.c_int, [C.c_int, vp, u64, vp, vp, u64, dbl, dbl, dbl,
                                              P(RngState)]),
    "moshpit_run_moshpit_sgd_logistic": (C.c_int, [C.c_int, u32, u32, u32, u32, u64, vp, vp,
                                                   u64, dbl, vp, dbl, u32, u32, dbl, u32, u64,
                                                   vp, vp, u64, C.c_int, C.c_int, vp, vp, vp,
                                                   vp, vp, vp, vp, P(dbl)]),
    "moshpit_engine_create": (C.c_int, [u32, u32, u64, dbl, u64, C.c_int, P(vp)]),
    "moshpit_engine_destroy": (C.c_int, [vp]),
    "moshpit_engine_set_kernel": (C.c_int, [vp, C.c_int]),
    "moshpit_engine_round": (C.c_int, [vp, C.c_int, vp, u64, u64, vp, P(u32)]),
    "moshpit_engine_rounds_fused": (C.c_int, [vp, C.c_int, vp, u64, u64, u32, vp, vp]),
    "moshpit_engine_stats": (C.c_int, [vp, P(u64), P(u64)]),
    "moshpit_engine_set_timing": (C.c_int, [vp, C.c_int]),
    "moshpit_engine_kernel_time": (C.c_int, [vp, P(dbl), P(u64)]),
    "moshpit_engine_tables": (C.c_int, [vp, vp, vp, P(u32), vp, vp, vp]),
    "moshpit_engine_set_reference": (C.c_int, [vp, C.c_int, vp, u64, u64, C.c_int, vp]),
    "moshpit_engine_record": (C.c_int, [vp, C.c_int, vp, u64, u64, vp]),
    "moshpit_engine_round_record": (C.c_int, [vp, C.c_int, vp, u64, u64, vp, P(u32)]),
    "moshpit_engine_rounds_record": (C.c_int, [vp, C.c_int, vp, u64, u64, u32, vp, P(u32)]),
    "moshpit_engine_report": (C.c_int, [vp, P(dbl), vp, vp, u64, P(u64)]),
    "moshpit_shard_create": (C.c_int, [C.c_int, u32, u32, u64, dbl, u64, u64, i32, i32, i32,
                                       i32, P(vp)]),
    "moshpit_shard_create_ex": (C.c_int, [C.c_int, u32, u32, u64, dbl, u64, u64, i32, i32, i32,
                                          i32, i32, P(vp)]),
    "moshpit_shard_flush": (C.c_int, [vp, vp]),
    "moshpit_shard_probe_peers": (C.c_int, [vp, P(vp)]),
    "moshpit_shard_destroy": (C.c_int, [vp]),
    "moshpit_shard_ipc_handles": (C.c_int, [vp, vp]),
    "moshpit_shard_open_peers": (C.c_int, [vp, vp]),
    "moshpit_shard_fill_synthetic": (C.c_int, [vp, u64, vp]),
    "moshpit_shard_round": (C.c_int, [vp, vp, P(u32), P(i32)]),
    "moshpit_shard_read": (C.c_int, [vp, vp, vp]),
    "moshpit_shard_set_timing": (C.c_int, [vp, i32]),
    "moshpit_shard_set_cross_mode": (C.c_int, [vp, i32]),
    "moshpit_shard_kernel_time": (C.c_int, [vp, P(dbl), P(u64), P(dbl), P(u64)]),
    "moshpit_shard_stats": (C.c_int, [vp, i32, P(u64), P(u64), P(u64)]),
    "moshpit_shard_cross_detail": (C.c_int, [vp, i32, P(dbl), P(dbl), P(u64)]),
    "moshpit_shard_pool": (C.c_int, [vp, i32, P(vp), P(u64), P(u64)]),
    "moshpit_shard_row_peers": (C.c_int, [vp, i32, vp]),
    "moshpit_shard_load_rows": (C.c_int, [vp, i32, vp, u64, vp]),
    "moshpit_shard_store_rows": (C.c_int, [vp, i32, vp, u64, vp]),
    "moshpit_fill_synthetic": (C.c_int, [C.c_int, vp, u64, u64, u64, u64, u64, vp]),
}

_lib = None


def lib():
    """Load libmoshpit_b200.so (building it first if this checkout has nvcc)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        try:
            from . import build as _b
            _b.build()
        except Exception as exc:  # noqa: BLE001
            raise ImportError(
                f"libmoshpit_b200.so is not built ({exc}); run "
                "`python -m paper_2103_03239_b200.build` -- there is no CPU fallback") from exc
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc):
    if rc != OK:
        msg = lib().moshpit_last_error().decode(errors="replace")
        raise _EXC.get(rc, MoshpitError)(msg)
    return rc


def exported_symbols():
    return list(PROTOTYPES)
