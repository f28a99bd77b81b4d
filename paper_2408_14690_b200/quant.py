"""Weight quantisation for the sparse GEMV (BASELINE config 5) and the batched
shared-mask sparse GEMV entry point.

The reference keeps fp32 weights only (SPEC.md:506 puts quantised kernels
out of its scope; PAPER.md:365 reports TEAL composing with weight
quantisation).  Formats here (input-major, row i = the n outputs of input
channel i, the reference's COL_MAJOR storage, tensor.py:47-48):

* int8: symmetric per output column, W[i, j] = q[i, j] * s[j],
  s[j] = max_i |W[i, j]| / 127;
* int4: symmetric per (group of `group` input rows, output column),
  W[i, j] = q[i, j] * s[i // group, j], s = max |W| / 7 over the group,
  q in [-8, 7], two per byte along the output dimension (low nibble = even
  column).

Quantisation is offline weight preparation (torch ops on the device); the
product runs in ``teal_gemv_batched`` (csrc/teal_gemv_batched.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT


@dataclass
class QuantWeights:
    """Input-major quantised weights: data [m, n] (bf16 / int8) or [m, n/2]
    (int4, uint8 packed), scale per column (int8) or per (group, column)."""

    data: torch.Tensor
    dtype: int                      # TEAL_BF16 / TEAL_I8 / TEAL_I4
    m: int
    n: int
    scale: torch.Tensor | None = None
    group: int = 0

    def dequantize(self) -> torch.Tensor:
        """fp32 [m, n] values the kernel multiplies with (exact)."""
        if self.dtype == C.TEAL_BF16:
            return self.data.float()
        if self.dtype == C.TEAL_I8:
            return self.data.float() * self.scale[None, :]
        lo = (self.data & 0xF).to(torch.int16)
        hi = (self.data >> 4).to(torch.int16)
        q = torch.stack([lo, hi], dim=-1).reshape(self.m, self.n)
        q = torch.where(q >= 8, q - 16, q).float()
        g = torch.arange(self.m, device=q.device) // self.group
        return q * self.scale[g]


def as_bf16(w_in_major: torch.Tensor) -> QuantWeights:
    m, n = w_in_major.shape
    return QuantWeights(w_in_major.to(torch.bfloat16).contiguous(), C.TEAL_BF16, m, n)


def quantize_int8(w_in_major: torch.Tensor) -> QuantWeights:
    w = w_in_major.float()
    m, n = w.shape
    s = w.abs().amax(dim=0) / 127.0
    s = torch.where(s > 0, s, torch.ones_like(s))
    q = torch.clamp(torch.round(w / s[None, :]), -127, 127).to(torch.int8)
    return QuantWeights(q.contiguous(), C.TEAL_I8, m, n, s.contiguous())


def quantize_int4(w_in_major: torch.Tensor, group: int = 128) -> QuantWeights:
    w = w_in_major.float()
    m, n = w.shape
    if n % 2:
        raise ValueError("int4 rows need an even number of output columns")
    ng = -(-m // group)
    pad = ng * group - m
    wp = torch.cat([w, torch.zeros(pad, n, device=w.device)]) if pad else w
    s = wp.reshape(ng, group, n).abs().amax(dim=1) / 7.0
    s = torch.where(s > 0, s, torch.ones_like(s))
    g = torch.arange(m, device=w.device) // group
    q = torch.clamp(torch.round(w / s[g]), -8, 7).to(torch.int16)
    qu = (q & 0xF).to(torch.uint8).reshape(m, n // 2, 2)
    packed = (qu[..., 0] | (qu[..., 1] << 4)).contiguous()
    return QuantWeights(packed, C.TEAL_I4, m, n, s.contiguous(), group)


def sparse_gemv_batched(xs, t: float, w: QuantWeights, return_mask: bool = False, kept: torch.Tensor | None = None):
    """Y [B, n] = sparsify_batched(xs, t) @ W^T with each kept weight row read
    once for all B rows (sparsifier.py:136-155 mask: column i pruned iff
    mean_b |xs[b, i]| <= fl32(t)).  ``t = None`` or -inf: dense."""
    if t is not None and not t >= 0.0 and t != float("-inf"):
        raise ValueError(f"threshold must be non-negative, got {t}")
    host = not (isinstance(xs, torch.Tensor) and xs.is_cuda)
    x = (xs if not host else torch.from_numpy(np.ascontiguousarray(np.asarray(xs, np.float32))).to(RT.require_cuda()))
    x = x.float().contiguous()
    if x.dim() != 2 or not 1 <= x.shape[0] <= 16:
        raise ValueError(f"expected a [B, m] batch with 1 <= B <= 16, got shape {tuple(x.shape)}")
    B, m = x.shape
    if m != w.m:
        raise ValueError(f"dimension mismatch: x rows have length {m}, W has {w.m} input channels")
    dev = x.device
    t32 = float("-inf") if t is None or t == float("-inf") else RT.f32_round_nearest(float(t))
    if B == 1 and not return_mask and w.dtype in (C.TEAL_BF16, C.TEAL_I8) and w.data.dtype in (torch.bfloat16, torch.int8):
        # one row: mean_b |x| = |x| exactly, so the shared mask is sparsify's
        # fp32 `|x| <= fl32(t)` — the single-row split-K kernel (the fast B = 1
        # path) with that threshold gives the same mask and kept count
        y1 = torch.empty(w.n, device=dev)
        a1 = RT.single_gemv_args(w.data, w.n, x[0], t32, y1, w.scale if w.dtype == C.TEAL_I8 else None, kept)
        RT.bind_workspace(a1, dev)
        RT.launch_gemv(a1)
        y = y1.view(1, w.n)
        return y.cpu().numpy() if host else y
    y = torch.empty(B, w.n, device=dev)
    mask = torch.empty(m, dtype=torch.uint8, device=dev) if return_mask else None
    a = C.TealGemvBatchedArgs()
    a.w, a.scale, a.x, a.y = w.data.data_ptr(), RT.ptr(w.scale), x.data_ptr(), y.data_ptr()
    a.mask, a.kept = RT.ptr(mask), RT.ptr(kept)
    a.m, a.n, a.ldw = m, w.n, w.n
    a.w_dtype, a.group, a.B = w.dtype, w.group, B
    a.t32 = t32
    g, nws, ntk = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    C.call("teal_gemv_batched_workspace", ctypes.byref(a), ctypes.byref(g), ctypes.byref(nws), ctypes.byref(ntk))
    ws, tk = RT.workspace(nws.value, ntk.value, dev)
    a.ws, a.tickets = ws.data_ptr(), tk.data_ptr()
    C.check(C.lib().teal_gemv_batched(ctypes.byref(a), RT.stream_handle()))
    out = y.cpu().numpy() if host else y
    if return_mask:
        mk = mask.bool()
        return out, (mk.cpu().numpy() if host else mk)
    return out
