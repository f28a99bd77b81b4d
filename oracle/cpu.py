"""TEST INFRASTRUCTURE — ctypes loader for the C restatement
(``oracle/teal_oracle.c``) of the reference CPU GEMV (kernel.py:30-44)."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle_teal.so"
_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < (HERE / "teal_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "-s"], check=True,
                       capture_output=True, text=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        f32p = ctypes.POINTER(ctypes.c_float)
        ll = ctypes.c_longlong
        L.oracle_skip_gemv.argtypes = [f32p, f32p, ll, ll, ctypes.c_double, f32p]
        L.oracle_skip_gemv.restype = ll
        L.oracle_skip_gemv_mt.argtypes = [f32p, f32p, ll, ll, ctypes.c_double, f32p, ctypes.c_int]
        L.oracle_skip_gemv_mt.restype = ll
        L.oracle_skip_gemv_bf16_mt.argtypes = [f32p, ctypes.c_void_p, ll, ll, ctypes.c_double, f32p, ctypes.c_int]
        L.oracle_skip_gemv_bf16_mt.restype = ll
        L.oracle_gemv_dense.argtypes = [f32p, f32p, ll, ll, f32p]
        L.oracle_gemv_dense.restype = None
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def skip_gemv(x, w_in_major, t, threads: int = 1):
    """C port of `_skip_gemv` (kernel.py:30-44); returns (y, used)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w_in_major, dtype=np.float32)
    m, n = w.shape
    y = np.empty(n, dtype=np.float32)
    if threads <= 1:
        used = lib().oracle_skip_gemv(_fp(x), _fp(w), m, n, float(t), _fp(y))
    else:
        used = lib().oracle_skip_gemv_mt(_fp(x), _fp(w), m, n, float(t), _fp(y), threads)
    return y, int(used)


def skip_gemv_bf16(x, w_bits_in_major, t, threads: int = 1):
    """Same loop over bf16 rows (uint16 bit patterns) widened exactly to fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w_bits_in_major, dtype=np.uint16)
    m, n = w.shape
    y = np.empty(n, dtype=np.float32)
    used = lib().oracle_skip_gemv_bf16_mt(_fp(x), w.ctypes.data, m, n, float(t), _fp(y), max(1, threads))
    return y, int(used)


def gemv_dense(x, w_in_major):
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w_in_major, dtype=np.float32)
    m, n = w.shape
    y = np.empty(n, dtype=np.float32)
    lib().oracle_gemv_dense(_fp(x), _fp(w), m, n, _fp(y))
    return y


def max_threads() -> int:
    return int(lib().oracle_max_threads())
