"""Device plumbing: CUDA requirement, current-stream handle, caller-owned
workspaces (split-K partials + self-resetting tickets) and launch plans.

PyTorch is used only for device memory, streams and graphs; every compute
step runs in the sm_100a library through :mod:`._clib`."""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np
import torch

from . import _clib as C

_ws_lock = threading.Lock()
_ws_cache: dict = {}
_ws_retired: list = []  # grown-out-of workspaces (CUDA graphs may still point at them)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("TEAL B200 path needs a CUDA device (sm_100a); there is no CPU fallback")
    C.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return C.TEAL_F32
    if dt == torch.bfloat16:
        return C.TEAL_BF16
    if dt == torch.int8:
        return C.TEAL_I8
    if dt == torch.float64:
        return C.TEAL_F64
    raise ValueError(f"unsupported dtype {dt}")


def workspace(nfloats: int, ntickets: int, device=None, stream: torch.cuda.Stream | None = None):
    """Grow-only (ws fp32, tickets int32 zeroed) pair, one per (device, stream).

    Tickets self-reset at the end of every launch, so the pair can be reused
    by any later stream-ordered launch (and inside CUDA graphs)."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), stream_handle(stream))
    with _ws_lock:
        ws, tk = _ws_cache.get(key, (None, None))
        # superseded buffers stay alive: a CUDA graph captured over an earlier
        # call keeps their raw pointers
        if ws is None or ws.numel() < nfloats:
            if ws is not None:
                _ws_retired.append(ws)
            ws = torch.empty(max(nfloats, 1 << 16), dtype=torch.float32, device=dev)
        if tk is None or tk.numel() < ntickets:
            if tk is not None:
                _ws_retired.append(tk)
            tk = torch.zeros(max(ntickets, 4096), dtype=torch.int32, device=dev)
        _ws_cache[key] = (ws, tk)
    return ws, tk


def gemv_workspace(args: C.TealGemvArgs) -> tuple[int, int, int]:
    """(ctas, ws floats, tickets) of the launch plan for ``args``."""
    g, ws, tk = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    C.call("teal_gemv_workspace", ctypes.byref(args), ctypes.byref(g), ctypes.byref(ws), ctypes.byref(tk))
    return g.value, ws.value, tk.value


def bind_workspace(args: C.TealGemvArgs, device=None, stream=None) -> None:
    """Attach the (device, stream) workspace sized for ``args``."""
    _, nws, ntk = gemv_workspace(args)
    ws, tk = workspace(nws, ntk, device, stream)
    args.ws, args.tickets = ws.data_ptr(), tk.data_ptr()


def single_gemv_args(wt: torch.Tensor, n: int, x: torch.Tensor, t32: float, y: torch.Tensor,
                     col_scale=None, kept=None) -> C.TealGemvArgs:
    """teal_gemv_args for one projection y = s_t(x) W^T over input-major ``wt``."""
    a = C.TealGemvArgs()
    a.w_dtype = dtype_code(wt.dtype)
    a.x_dtype = dtype_code(x.dtype)
    a.x = x.data_ptr()
    a.m = wt.shape[0]
    a.nseg = 1
    a.seg[0].w = wt.data_ptr()
    a.seg[0].ldw = wt.stride(0)
    a.seg[0].n = n
    a.seg[0].t32 = t32
    a.seg[0].y = y.data_ptr()
    a.seg[0].col_scale = ptr(col_scale)
    a.seg[0].kept = ptr(kept)
    a.prologue = C.PRO_PLAIN
    a.epilogue = C.EPI_STORE
    return a


def launch_gemv(args: C.TealGemvArgs, stream=None) -> None:
    C.check(C.lib().teal_fused_gemv(ctypes.byref(args), stream_handle(stream)))


def f32_round_nearest(t: float) -> float:
    """fl32(t), the threshold NumPy compares against in `sparsify`
    (sparsifier.py:121-125, weak-scalar promotion)."""
    with np.errstate(over="ignore"):
        return float(np.float32(t))


def f32_round_down(t: float) -> float:
    """Largest fp32 <= t: |x| <= t in fp64 (kernel.py:37, x fp32) holds iff
    |x| <= RD32(t), so an fp32 compare against RD32(t) is exact."""
    if math.isinf(t) or math.isnan(t):
        return t
    with np.errstate(over="ignore"):
        f = np.float32(t)
    if float(f) > t:
        f = np.nextafter(f, np.float32(-np.inf))
    return float(f)
