"""TEST INFRASTRUCTURE — ctypes loader for the C restatement
(``oracle/teal_oracle.c``) of the reference CPU GEMV (kernel.py:30-44)."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle_teal.so"          # x86-64-v2 (any x86-64 host)
LIB_V3 = HERE / "build" / "liboracle_teal_v3.so"    # AVX2 / FMA hosts
LIB_V4 = HERE / "build" / "liboracle_teal_v4.so"    # AVX-512 hosts
_lib = None


def build(force: bool = False) -> Path:
    libs = (LIB, LIB_V3, LIB_V4)
    src = (HERE / "teal_oracle.c").stat().st_mtime
    if force or any(not p.exists() or p.stat().st_mtime < src for p in libs):
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "-s"], check=True,
                       capture_output=True, text=True)
    return LIB


def isa_level() -> str:
    """Widest x86-64 level the host supports (numba compiles the reference
    for the host CPU the same way)."""
    try:
        flags = set()
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        return "v2"
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl", "avx2", "fma", "bmi2"} <= flags:
        return "v4"
    if {"avx2", "fma", "bmi2", "movbe"} <= flags:
        return "v3"
    return "v2"


def lib_path() -> Path:
    lv = isa_level()
    p = {"v4": LIB_V4, "v3": LIB_V3}.get(lv, LIB)
    return p if p.exists() else LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(lib_path()))
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
