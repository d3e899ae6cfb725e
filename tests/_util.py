"""Shared helpers for the parity tests."""
import numpy as np

INIT_SEED = 0x5EED


def unhex(h):
    return np.frombuffer(bytes.fromhex(h), dtype="<f8")[0]


def unhexa(hs):
    if not hs:
        return np.zeros(0)
    return np.frombuffer(b"".join(bytes.fromhex(h) for h in hs), dtype="<f8").copy()


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    return a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes()


def ulp_diff_f32(a, b):
    ai = np.ascontiguousarray(a, dtype=np.float32).view(np.int32).astype(np.int64)
    bi = np.ascontiguousarray(b, dtype=np.float32).view(np.int32).astype(np.int64)
    return np.abs(ai - bi)
