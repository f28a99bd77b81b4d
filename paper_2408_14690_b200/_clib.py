"""ctypes binding of the C ABI declared in ``include/teal_b200.h``.

This is the binding a Python caller of the reference would add: plain
pointers and sizes, int status, ``teal_last_error()`` for the message.  The
library is loaded from the in-tree ``lib/libteal_b200.so``; there is no CPU
fallback — if it is missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libteal_b200.so"

TEAL_OK, TEAL_EINVAL, TEAL_ECUDA = 0, 1, 2
TEAL_F32, TEAL_BF16, TEAL_I8, TEAL_I4, TEAL_F64 = 0, 1, 2, 3, 4
PRO_PLAIN, PRO_RMSNORM = 0, 1
EPI_STORE, EPI_RESID, EPI_SILU, EPI_QKV = 0, 1, 2, 3

c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


class TealSeg(ctypes.Structure):
    _fields_ = [
        ("w", c_vp), ("ldw", c_i64), ("n", c_i64), ("t32", ctypes.c_float),
        ("y", c_vp), ("col_scale", c_vp), ("dbg_bits", c_vp), ("kept", c_vp),
    ]


class TealGemvArgs(ctypes.Structure):
    _fields_ = [
        ("w_dtype", ctypes.c_int), ("x_dtype", ctypes.c_int), ("x", c_vp), ("m", c_i64),
        ("nseg", ctypes.c_int), ("seg", TealSeg * 3),
        ("prologue", ctypes.c_int), ("norm_scale", c_vp), ("ss_part", c_vp), ("ss_count", ctypes.c_int),
        ("eps", ctypes.c_float), ("dbg_h", c_vp),
        ("epilogue", ctypes.c_int), ("resid", c_vp), ("ss_out", c_vp), ("inter", c_vp),
        ("q_out", c_vp), ("k_cache", c_vp), ("v_cache", c_vp), ("kv_dtype", ctypes.c_int),
        ("max_seq", c_i64), ("pos", c_vp), ("head_dim", ctypes.c_int),
        ("rope_cos", c_vp), ("rope_sin", c_vp),
        ("ctas", ctypes.c_int), ("ws", c_vp), ("tickets", c_vp),
    ]


class TealGemvBatchedArgs(ctypes.Structure):
    _fields_ = [("w", c_vp), ("scale", c_vp), ("x", c_vp), ("y", c_vp), ("mask", c_vp), ("kept", c_vp),
                ("ws", c_vp), ("tickets", c_vp), ("m", c_i64), ("n", c_i64), ("ldw", c_i64),
                ("w_dtype", ctypes.c_int), ("group", ctypes.c_int), ("B", ctypes.c_int), ("t32", ctypes.c_float),
                ("ctas", ctypes.c_int), ("pad_", ctypes.c_int)]


class TealPrefillArgs(ctypes.Structure):
    _fields_ = [("w", c_vp), ("m", c_i64), ("n", c_i64), ("ldw", c_i64), ("x_hi", c_vp), ("x_lo", c_vp),
                ("T", c_i64), ("ldx", c_i64), ("y", c_vp), ("ldy", c_i64), ("accumulate", ctypes.c_int),
                ("splits", ctypes.c_int), ("ws", c_vp), ("tickets", c_vp)]


# (name, restype, argtypes) for every exported symbol of include/teal_b200.h
_SIGNATURES = [
    ("teal_last_error", ctypes.c_char_p, []),
    ("teal_abi_version", ctypes.c_int, []),
    ("teal_device_sm_count", ctypes.c_int, [ctypes.c_int]),
    ("teal_threshold", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, ctypes.c_float, c_vp, c_vp, c_vp, c_vp]),
    ("teal_threshold_batched", ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.c_float, c_vp, c_vp, c_vp]),
    ("teal_gemv_workspace", ctypes.c_int, [ctypes.POINTER(TealGemvArgs), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    ("teal_gemv_tile_width", ctypes.c_int, [ctypes.POINTER(TealGemvArgs)]),
    ("teal_debug_timeline", ctypes.c_int, [c_vp, ctypes.c_int]),
    ("teal_fused_gemv", ctypes.c_int, [ctypes.POINTER(TealGemvArgs), c_vp]),
    ("teal_sparse_gemv", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_i64, c_i64, c_vp, ctypes.c_int,
                                        ctypes.c_float, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp]),
    ("teal_dense_gemv", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_i64, c_i64, c_vp, ctypes.c_int,
                                       c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp]),
    ("teal_hist_record", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, ctypes.c_double, ctypes.c_int,
                                        c_vp, c_vp, c_vp, c_vp]),
    ("teal_hist_threshold", ctypes.c_int, [c_vp, ctypes.c_int, c_vp, ctypes.c_double, c_vp, ctypes.c_int,
                                           c_vp, c_vp]),
    ("teal_decode_attention", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, c_i64, c_vp, ctypes.c_int, c_vp, c_vp, c_vp,
                                             ctypes.c_int, c_vp]),
    ("teal_load_residual", ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_i64, c_vp, c_vp, ctypes.c_int, c_vp, c_vp]),
    ("teal_argmax", ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    ("teal_output_sparse_gemv", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_i64, c_i64, c_vp, c_vp, ctypes.c_float,
                                               c_vp, c_vp, c_vp, c_vp]),
    ("teal_prefill_gate", ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, ctypes.c_float, c_i64, c_vp, c_vp, c_i64,
                                         c_vp, c_vp]),
    ("teal_prefill_workspace", ctypes.c_int, [ctypes.POINTER(TealPrefillArgs), ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    ("teal_prefill_gemm", ctypes.c_int, [ctypes.POINTER(TealPrefillArgs), c_vp]),
    ("teal_prefill_rope_cache", ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, c_i64, c_vp, c_vp, c_vp, c_vp, ctypes.c_int,
                                               c_i64, c_vp]),
    ("teal_batch_attention", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, c_i64, c_vp, ctypes.c_int, c_vp, c_vp, c_vp, ctypes.c_int,
                                            c_vp]),
    ("teal_batch_embed", ctypes.c_int, [c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_i64, c_vp, c_vp, c_vp]),
    ("teal_batch_rmsnorm", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_float, ctypes.c_int, c_i64, c_vp, c_vp]),
    ("teal_batch_rope_cache", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_vp,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, c_vp]),
    ("teal_batch_silu_mul", ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    ("teal_batch_argmax", ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_vp, c_vp]),
    ("teal_stream_create", ctypes.c_int, [ctypes.POINTER(c_vp)]),
    ("teal_stream_destroy", ctypes.c_int, [c_vp]),
    ("teal_event_create", ctypes.c_int, [ctypes.POINTER(c_vp)]),
    ("teal_event_destroy", ctypes.c_int, [c_vp]),
    ("teal_stream_order", ctypes.c_int, [c_vp, c_vp, c_vp]),
    ("teal_residual_add", ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, ctypes.c_int, c_vp]),
    ("teal_step_ctas_per_sm", ctypes.c_int, [ctypes.c_int]),
    ("teal_gemv_batched_workspace", ctypes.c_int, [ctypes.POINTER(TealGemvBatchedArgs), ctypes.POINTER(ctypes.c_int),
                                                   ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    ("teal_gemv_batched", ctypes.c_int, [ctypes.POINTER(TealGemvBatchedArgs), c_vp]),
    ("teal_step_launch", ctypes.c_int, [c_vp, c_vp]),
]

EXPORTED = tuple(name for name, _, _ in _SIGNATURES)

_lib = None


class TealError(RuntimeError):
    """A CUDA-level failure reported by the TEAL library (status TEAL_ECUDA)."""


def lib():
    """Load the in-tree library (building it first if sources are newer)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists() or os.environ.get("TEAL_AUTOBUILD", "1") == "1":
            try:
                from . import build as _b
                if not LIB_PATH.exists() or _b._stale():
                    _b.build()
            except Exception as exc:  # no nvcc on this host: only a prebuilt lib will do
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"TEAL CUDA library {LIB_PATH} is missing and could not be built: {exc}") from exc
        L = ctypes.CDLL(str(LIB_PATH))
        for name, res, args in _SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    """Map a TEAL status to the reference's exception types."""
    if status == TEAL_OK:
        return
    msg = (lib().teal_last_error() or b"").decode(errors="replace")
    if status == TEAL_EINVAL:
        raise ValueError(msg)
    raise TealError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
