"""ctypes wrapper of the C oracle (oracle/adt_oracle.c) — TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle_adt.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        lib = ctypes.CDLL(LIB)
        lib.oracle_pack.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        lib.oracle_unpack.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        lib.oracle_sumsq.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        lib.oracle_sumsq.restype = ctypes.c_double
        _lib = lib
    return _lib


def pack(x, r: int) -> bytes:
    w = np.ascontiguousarray(x, dtype=np.float32).reshape(-1).view(np.uint32)
    out = np.empty(w.size * r, np.uint8)
    if load().oracle_pack(w.ctypes.data, w.size, r, out.ctypes.data):
        raise ValueError("round_to must be an integer in [1, 4]")
    return out.tobytes()


def unpack(payload: bytes, n: int, r: int) -> np.ndarray:
    src = np.frombuffer(payload, np.uint8)
    if src.size != n * r:
        raise ValueError("payload length mismatch")
    out = np.empty(n, np.uint32)
    if load().oracle_unpack(src.ctypes.data, n, r, out.ctypes.data):
        raise ValueError("round_to must be an integer in [1, 4]")
    return out.view(np.float32)


def sumsq(x) -> float:
    a = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    return float(load().oracle_sumsq(a.ctypes.data, a.size))
