"""Sparse prefill: the prompt pass before decode.

TEAL sparsifies the prompt too, except its first positions (attention sinks,
PAPER.md:269-270, :439-446): rows t < ``sparse_from`` stay dense, later rows
are thresholded with decode's magnitude test.  Prefill is GEMM-shaped (T
tokens per weight read), so the product runs on the tcgen05 tensor cores
(``teal_prefill_gemm``, csrc/teal_prefill.cu) after one masking pass
(``teal_prefill_gate``) that also splits the kept fp32 activations into bf16
hi + lo operands, so the contraction is fp32-faithful against bf16 weights.

The per-row semantics are the reference's ``sparsify`` then ``matmul_dense``
(pkg/src/actsparse/sparsifier.py:120-134, tensor.py:130-140); the reference
itself has no prefill path.
"""

from __future__ import annotations

import torch

from . import _clib as C
from . import _runtime as RT

BK = 64    # the GEMM's K step (m must be a multiple)
BM = 128   # the GEMM's output tile (n must be a multiple)


def gate(x: torch.Tensor, t: float, sparse_from: int = 0, terms: int = 2, kept=None):
    """Masked bf16 operands of x [T, m] fp32: (hi, lo) with hi = rn(g), lo =
    rn(g - hi) (lo None when terms == 1), g = x where t < sparse_from or
    !(|x| <= fl32(t)), else 0.  ``kept`` (int64 cuda tensor, nullable) +=
    kept values among the thresholded rows."""
    if terms not in (1, 2):
        raise ValueError(f"terms must be 1 or 2, got {terms}")
    if not t >= 0.0:
        raise ValueError(f"threshold must be non-negative, got {t}")
    if sparse_from < 0:
        raise ValueError(f"sparse_from must be >= 0, got {sparse_from}")
    xd = x.float().contiguous()
    if xd.dim() != 2:
        raise ValueError(f"x must be [T, m], got shape {tuple(x.shape)}")
    T, m = xd.shape
    hi = torch.empty(T, m, dtype=torch.bfloat16, device=xd.device)
    lo = torch.empty_like(hi) if terms == 2 else None
    C.call("teal_prefill_gate", xd.data_ptr(), T, m, m, RT.f32_round_nearest(t), sparse_from, hi.data_ptr(),
           RT.ptr(lo), m, RT.ptr(kept), RT.stream_handle())
    return hi, lo


_WS: dict = {}  # device -> (float workspace, tickets), grown on demand


def _workspace(device, floats: int, tickets: int):
    ws, tk = _WS.get(device, (None, None))
    if ws is None or ws.numel() < floats:
        ws = torch.empty(max(floats, 1 << 20), device=device)
    if tk is None or tk.numel() < tickets:
        tk = torch.zeros(max(tickets, 1024), dtype=torch.int32, device=device)
    _WS[device] = (ws, tk)
    return ws, tk


def gemm(w: torch.Tensor, hi: torch.Tensor, lo=None, out=None, accumulate: bool = False,
         splits: int = 0) -> torch.Tensor:
    """y [T, n] (+)= (hi + lo) @ w on the tensor cores; w bf16 [m, n] input-major.
    ``splits``: K splits (0 = auto: fill the SMs; 1 = none)."""
    if w.dtype != torch.bfloat16 or hi.dtype != torch.bfloat16 or (lo is not None and lo.dtype != torch.bfloat16):
        raise ValueError("prefill gemm takes bf16 weights and bf16 operands")
    m, n = w.shape
    T = hi.shape[0]
    if hi.shape != (T, m) or (lo is not None and lo.shape != hi.shape):
        raise ValueError(f"operand shape {tuple(hi.shape)} does not match weights {tuple(w.shape)}")
    if w.stride(1) != 1 or hi.stride(1) != 1 or (lo is not None and (lo.stride(1) != 1 or lo.stride(0) != hi.stride(0))):
        raise ValueError("prefill gemm needs unit-stride rows")
    if out is None:
        if accumulate:
            raise ValueError("accumulate needs an output tensor")
        out = torch.empty(T, n, device=hi.device)
    elif out.dtype != torch.float32 or out.shape != (T, n) or out.stride(1) != 1:
        raise ValueError(f"out must be fp32 [{T}, {n}] with unit-stride rows")
    a = C.TealPrefillArgs(w=w.data_ptr(), m=m, n=n, ldw=w.stride(0), x_hi=hi.data_ptr(), x_lo=RT.ptr(lo), T=T,
                          ldx=hi.stride(0), y=out.data_ptr(), ldy=out.stride(0), accumulate=int(bool(accumulate)),
                          splits=int(splits))
    ns, wsf, tks = C.ctypes.c_int(0), C.c_i64(0), C.c_i64(0)
    C.call("teal_prefill_workspace", C.ctypes.byref(a), C.ctypes.byref(ns), C.ctypes.byref(wsf), C.ctypes.byref(tks))
    if ns.value > 1:
        ws, tk = _workspace(hi.device, wsf.value, tks.value)
        a.ws, a.tickets = ws.data_ptr(), tk.data_ptr()
    C.call("teal_prefill_gemm", C.ctypes.byref(a), RT.stream_handle())
    return out


def masked_gemm(x: torch.Tensor, w: torch.Tensor, t: float, sparse_from: int = 0, terms: int = 2, out=None,
                accumulate: bool = False, kept=None) -> torch.Tensor:
    """y (+)= g(x) @ w with TEAL's prefill mask (rows before ``sparse_from``
    dense): gate + tensor-core GEMM, two launches."""
    hi, lo = gate(x, t, sparse_from, terms, kept)
    return gemm(w, hi, lo, out, accumulate)
