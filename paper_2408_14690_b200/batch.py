"""Small-batch TEAL decode (BASELINE config 5: Mistral-7B, B = 1..16, bf16 /
int8 / int4 weights at 50 %).

B sequences are decoded in lockstep.  Each projection input [B, m] is
sparsified with ONE shared column mask — column i pruned iff the batch mean
magnitude mean_b |h[b, i]| <= fl32(t) (``sparsify_batched``,
pkg/src/actsparse/sparsifier.py:136-155, paper §5.4.4) — so every kept weight
row is streamed from HBM once for all B rows (``teal_gemv_batched``: the
mask fused into the GEMV, mma.sync tensor-core contraction for B >= 4).
Thresholds must come from a separate histogram of batch-mean magnitudes per
batch size (pkg/tests/test_acceptance.py:223-239):
:func:`calibrate_batch_histograms` records exactly that statistic on the GPU
and :func:`batch_thresholds` inverts it, giving a [L][7] table for each B.

One step = embedding rows, per layer RMSNorm -> q / k / v (three shared-mask
GEMVs) -> RoPE + KV-cache append -> attention over each sequence's cache ->
o -> residual + RMSNorm -> gate / up -> SiLU * up -> down, then the final
norm, the dense LM head (the same batched kernel at t = -inf) and greedy
argmax per sequence — every launch one of this package's kernels, captured
in one CUDA graph.  (B = 1 is the persistent step engine's job,
:class:`.engine.StepDecoder`; this engine also runs it, as a baseline.)
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT
from . import quant as Q
from .decode import PROJ, PROJ_TAP, DecoderWeights, _t32

TAPS = ("pre_attn", "attn_out", "pre_mlp", "mlp_inter")
TAP_OF = {p: PROJ_TAP[p] for p in PROJ}
MAX_B = 16


def _quant(w: torch.Tensor, quant: str | None) -> Q.QuantWeights:
    if quant is None:
        return Q.as_bf16(w) if w.dtype == torch.bfloat16 else Q.QuantWeights(w.float().contiguous(), C.TEAL_F32,
                                                                             w.shape[0], w.shape[1])
    if quant == "int8":
        return Q.quantize_int8(w)
    if quant == "int4":
        return Q.quantize_int4(w)
    raise ValueError(f"unknown quantisation {quant!r} (None, 'int8', 'int4')")


class BatchDecoder:
    """TEAL decode of ``batch`` sequences in lockstep with shared masks.

    weights: :class:`.decode.DecoderWeights` (input-major, Llama / Mistral
    style with an embedding and LM head); thresholds: [n_layers][7] in the
    order q, k, v, o, gate, up, down (None = dense), calibrated for THIS batch
    size (:func:`batch_thresholds`); quant: None (weights' dtype), 'int8' or
    'int4'.  ``taps=True`` keeps, per layer, the projection inputs the kernels
    saw, the shared masks and a few intermediates (tests / calibration)."""

    def __init__(self, weights: DecoderWeights, thresholds, batch: int, quant: str | None = None,
                 kv_dtype=None, taps: bool = False, count_kept: bool = False, concurrent: bool = True):
        spec = self.spec = weights.spec
        if not spec.vocab:
            raise ValueError("BatchDecoder needs an embedding and LM head (vocab > 0)")
        if not 1 <= batch <= MAX_B:
            raise ValueError(f"batch must be in [1, {MAX_B}], got {batch}")
        self.w, self.B = weights, batch
        dev = self.device = RT.require_cuda()
        L, d, f, hd = spec.n_layers, spec.d_model, spec.d_ff, spec.head_dim
        nq, nkv, V = spec.n_q, spec.n_kv, spec.vocab
        thr = [[None] * 7 for _ in range(L)] if thresholds is None else [list(t) for t in thresholds]
        if len(thr) != L or any(len(t) != 7 for t in thr):
            raise ValueError(f"need {L} per-layer threshold lists of 7 (q,k,v,o,gate,up,down)")
        self.thresholds = thr
        self.quant = quant
        # weights per projection (input-major [m, n], contiguous)
        self.pw = []
        for lw in weights.layers:
            self.pw.append({"q": _quant(lw.wqkv[:, :nq], quant), "k": _quant(lw.wqkv[:, nq:nq + nkv], quant),
                            "v": _quant(lw.wqkv[:, nq + nkv:], quant), "o": _quant(lw.wo, quant),
                            "gate": _quant(lw.wgu[:, :f], quant), "up": _quant(lw.wgu[:, f:], quant),
                            "down": _quant(lw.wdown, quant)})
        self.lm = _quant(weights.lm_head, quant)
        self.kv_dtype = kv_dtype or torch.bfloat16
        B = batch
        f32 = dict(device=dev, dtype=torch.float32)
        self.x = torch.zeros(B, d, **f32)
        self.h = torch.zeros(B, d, **f32)
        self.q = torch.zeros(B, nq, **f32)
        self.k = torch.zeros(B, nkv, **f32)
        self.v = torch.zeros(B, nkv, **f32)
        self.ctx = torch.zeros(B, nq, **f32)
        self.o_out = torch.zeros(B, d, **f32)
        self.gate = torch.zeros(B, f, **f32)
        self.up = torch.zeros(B, f, **f32)
        self.inter = torch.zeros(B, f, **f32)
        self.down_out = torch.zeros(B, d, **f32)
        self.logits = torch.zeros(B, V, **f32)
        self.tokens = torch.zeros(B, device=dev, dtype=torch.int32)
        self.state = torch.zeros(2, device=dev, dtype=torch.int32)
        self.kcache = torch.zeros(L, B, spec.n_kv_heads, spec.max_seq, hd, device=dev, dtype=self.kv_dtype)
        self.vcache = torch.zeros_like(self.kcache)
        if spec.rope_theta is not None:
            inv = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
            ang = torch.arange(spec.max_seq, dtype=torch.float64)[:, None] * inv[None, :]
            self.rope_cos = torch.cos(ang).float().to(dev).contiguous()
            self.rope_sin = torch.sin(ang).float().to(dev).contiguous()
        else:
            self.rope_cos = self.rope_sin = None
        G = spec.n_heads // spec.n_kv_heads
        self.attn_nsplit = max(1, -(-spec.max_seq // 512))
        self.attn_ws = torch.zeros(B * spec.n_kv_heads * self.attn_nsplit * (G * hd + 2 * G), **f32)
        self.attn_tk = torch.zeros(B * spec.n_kv_heads, device=dev, dtype=torch.int32)
        self.kept = torch.zeros(L, 7, device=dev, dtype=torch.int64) if (count_kept or taps) else None
        self.taps = None
        if taps:
            dims = {"pre_attn": d, "attn_out": nq, "pre_mlp": d, "mlp_inter": f}
            self.taps = {t: torch.zeros(L, B, dims[t], **f32) for t in TAPS}
            self.tap_q = torch.zeros(L, B, nq, **f32)           # q after RoPE
            self.tap_o = torch.zeros(L, B, d, **f32)            # o projection output
            self.tap_down = torch.zeros(L, B, d, **f32)         # down projection output
            self.tap_final = torch.zeros(B, d, **f32)           # final-norm LM-head input
            self.masks = {p: torch.zeros(L, spec.proj_shapes()[p][1], device=dev, dtype=torch.uint8) for p in PROJ}
        # q / k / v (and gate / up) read the same input with their own masks:
        # with `concurrent` they run on three (two) streams at once, each launch
        # on its share of the SMs, so their fixed costs overlap
        self.concurrent = concurrent
        self._side, self._ev = [], []
        if concurrent:
            for lst, fn in ((self._side, "teal_stream_create"), (self._ev, "teal_event_create")):
                for _ in range(2 if lst is self._side else 3):
                    h = ctypes.c_void_p()
                    C.call(fn, ctypes.byref(h))
                    lst.append(h.value)
        self._build_args()
        self.graph = None
        self._pos = 0

    # -- launch descriptors ------------------------------------------------------
    def _gemv_args(self, w: Q.QuantWeights, x: torch.Tensor, y: torch.Tensor, t, mask=None, kept=None):
        a = C.TealGemvBatchedArgs()
        a.w, a.scale, a.x, a.y = w.data.data_ptr(), RT.ptr(w.scale), x.data_ptr(), y.data_ptr()
        a.mask, a.kept = RT.ptr(mask), RT.ptr(kept)
        a.m, a.n, a.ldw = w.m, w.n, w.n
        a.w_dtype, a.group, a.B = w.dtype, w.group, self.B
        a.t32 = _t32(t)
        g, nws, ntk = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        C.call("teal_gemv_batched_workspace", ctypes.byref(a), ctypes.byref(g), ctypes.byref(nws), ctypes.byref(ntk))
        self._ws_need = max(self._ws_need, nws.value)
        self._tk_need = max(self._tk_need, ntk.value)
        return a

    def _resize(self, a):
        g, nws, ntk = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        C.call("teal_gemv_batched_workspace", ctypes.byref(a), ctypes.byref(g), ctypes.byref(nws), ctypes.byref(ntk))
        self._ws_need = max(self._ws_need, nws.value)
        self._tk_need = max(self._tk_need, ntk.value)
        return a

    def _fork(self, sh: int, n: int) -> list:
        """Side streams that start after everything issued on `sh` so far."""
        for st in self._side[:n]:
            C.call("teal_stream_order", st, sh, self._ev[0])
        return self._side[:n]

    def _join(self, sh: int, n: int) -> None:
        for i, st in enumerate(self._side[:n]):
            C.call("teal_stream_order", sh, st, self._ev[1 + i])

    def __del__(self):
        try:
            for st in getattr(self, "_side", []):
                C.lib().teal_stream_destroy(st)
            for ev in getattr(self, "_ev", []):
                C.lib().teal_event_destroy(ev)
        except Exception:
            pass

    def _build_args(self):
        self._ws_need, self._tk_need = 1, 1
        L = self.spec.n_layers
        inputs = {"q": self.h, "k": self.h, "v": self.h, "o": self.ctx, "gate": self.h, "up": self.h,
                  "down": self.inter}
        outputs = {"q": self.q, "k": self.k, "v": self.v, "o": self.o_out, "gate": self.gate, "up": self.up,
                   "down": self.down_out}
        self.args = []
        for l in range(L):
            row = {}
            for i, p in enumerate(PROJ):
                mask = self.masks[p][l] if self.taps is not None else None
                kept = self.kept[l, i] if self.kept is not None else None
                row[p] = self._gemv_args(self.pw[l][p], inputs[p], outputs[p], self.thresholds[l][i], mask, kept)
            self.args.append(row)
        self.lm_args = self._gemv_args(self.lm, self.h, self.logits, None)
        if self.concurrent:  # SM shares of the concurrent launches (workspace sized after)
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            share = {"q": sms, "k": sms // 2, "v": sms // 2, "gate": 0, "up": 0}
            for l, row in enumerate(self.args):
                for p_, c in share.items():
                    row[p_].ctas = c
                    row[p_] = self._resize(row[p_])
        # concurrent launches need their own workspace: one per projection slot
        # (layers run in order, so the slots are reused across layers)
        self.ws = {p_: torch.zeros(self._ws_need, device=self.device) for p_ in PROJ}
        self.tk = {p_: torch.zeros(self._tk_need, device=self.device, dtype=torch.int32) for p_ in PROJ}
        for row in self.args:
            for p_, a in row.items():
                a.ws, a.tickets = self.ws[p_].data_ptr(), self.tk[p_].data_ptr()
        self.lm_args.ws, self.lm_args.tickets = self.ws["q"].data_ptr(), self.tk["q"].data_ptr()

    # -- step ---------------------------------------------------------------------
    def reset(self, start_pos: int = 0) -> None:
        self.state.copy_(torch.tensor([start_pos - 1, start_pos], dtype=torch.int32))
        self._pos = start_pos
        if start_pos == 0:
            self.kcache.zero_()
            self.vcache.zero_()

    def launches_per_step(self) -> int:
        return 1 + 13 * self.spec.n_layers + 3

    def _launch_step(self, sh: int) -> None:
        Lb = C.lib()
        sp, B = self.spec, self.B
        d, f, hd, H, KVH = sp.d_model, sp.d_ff, sp.head_dim, sp.n_heads, sp.n_kv_heads
        T = self.taps

        def gemv(a, stream=None):
            C.check(Lb.teal_gemv_batched(ctypes.byref(a), sh if stream is None else stream))

        C.check(Lb.teal_batch_embed(self.w.embedding.data_ptr(), RT.dtype_code(self.w.embedding.dtype),
                                    self.tokens.data_ptr(), B, d, self.x.data_ptr(), self.state.data_ptr(), sh))
        len_ptr = self.state.data_ptr() + 4
        for l, lw in enumerate(self.w.layers):
            A = self.args[l]
            delta = self.down_out.data_ptr() if l > 0 else None
            C.check(Lb.teal_batch_rmsnorm(self.x.data_ptr(), delta, lw.rms_attn.data_ptr(), sp.norm_eps, B, d,
                                          self.h.data_ptr(), sh))
            if T is not None:
                T["pre_attn"][l].copy_(self.h)
            if self.concurrent:
                s1, s2 = self._fork(sh, 2)
                gemv(A["k"], s1)
                gemv(A["v"], s2)
                gemv(A["q"])
                self._join(sh, 2)
            else:
                gemv(A["q"])
                gemv(A["k"])
                gemv(A["v"])
            C.check(Lb.teal_batch_rope_cache(self.q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(),
                                             self.kcache[l].data_ptr(), self.vcache[l].data_ptr(),
                                             RT.dtype_code(self.kv_dtype), RT.ptr(self.rope_cos),
                                             RT.ptr(self.rope_sin), self.state.data_ptr(), B, H, KVH, hd,
                                             sp.max_seq, sh))
            if T is not None:
                self.tap_q[l].copy_(self.q)
            C.check(Lb.teal_batch_attention(self.q.data_ptr(), self.kcache[l].data_ptr(), self.vcache[l].data_ptr(),
                                            RT.dtype_code(self.kv_dtype), B, H, KVH, hd, sp.max_seq, len_ptr,
                                            sp.max_seq, self.ctx.data_ptr(), self.attn_ws.data_ptr(),
                                            self.attn_tk.data_ptr(), self.attn_nsplit, sh))
            if T is not None:
                T["attn_out"][l].copy_(self.ctx)
            gemv(A["o"])
            if T is not None:
                self.tap_o[l].copy_(self.o_out)
            C.check(Lb.teal_batch_rmsnorm(self.x.data_ptr(), self.o_out.data_ptr(), lw.rms_mlp.data_ptr(),
                                          sp.norm_eps, B, d, self.h.data_ptr(), sh))
            if T is not None:
                T["pre_mlp"][l].copy_(self.h)
            if self.concurrent:
                (s1,) = self._fork(sh, 1)
                gemv(A["up"], s1)
                gemv(A["gate"])
                self._join(sh, 1)
            else:
                gemv(A["gate"])
                gemv(A["up"])
            C.check(Lb.teal_batch_silu_mul(self.gate.data_ptr(), self.up.data_ptr(), B * f, self.inter.data_ptr(), sh))
            if T is not None:
                T["mlp_inter"][l].copy_(self.inter)
            gemv(A["down"])
            if T is not None:
                self.tap_down[l].copy_(self.down_out)
        C.check(Lb.teal_batch_rmsnorm(self.x.data_ptr(), self.down_out.data_ptr(), self.w.final_norm.data_ptr(),
                                      sp.norm_eps, B, d, self.h.data_ptr(), sh))
        if T is not None:
            self.tap_final.copy_(self.h)
        gemv(self.lm_args)
        C.check(Lb.teal_batch_argmax(self.logits.data_ptr(), B, sp.vocab, self.tokens.data_ptr(), sh))

    def _advance(self) -> None:
        if self._pos >= self.spec.max_seq:
            raise ValueError(f"decode position {self._pos} would exceed max_seq {self.spec.max_seq}")
        self._pos += 1

    def step(self) -> torch.Tensor:
        """One decode step from self.tokens [B]; leaves the next tokens there."""
        self._advance()
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch_step(RT.stream_handle())
        return self.tokens

    def step_host(self, tok_in: torch.Tensor, tok_out: torch.Tensor) -> None:
        """End to end through pinned host buffers: H2D of the B input tokens,
        one step, D2H of the B next tokens (stream-ordered)."""
        self.tokens.copy_(tok_in, non_blocking=True)
        self.step()
        tok_out.copy_(self.tokens, non_blocking=True)

    def capture(self) -> torch.cuda.CUDAGraph:
        if self.taps is not None:
            raise ValueError("taps are for eager steps (tests / calibration)")
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._launch_step(s.cuda_stream)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        return g

    def replay(self) -> None:
        self._advance()
        self.graph.replay()

    def algorithmic_bytes(self, kept=None, steps: int = 1) -> float:
        """Bytes a step must touch (shared mask): kept rows x n x
        weight bytes (+ int8 column / int4 group scales of the kept rows) per
        projection, activation reads B x m x 4 and output writes B x n x 4,
        the dense LM head; K/V reads excluded (small at these contexts)."""
        sp = self.spec
        kept = (self.kept if kept is None else kept).double().cpu()
        bw = {C.TEAL_F32: 4.0, C.TEAL_BF16: 2.0, C.TEAL_I8: 1.0, C.TEAL_I4: 0.5}[self.lm.dtype]
        total = 0.0
        shapes = sp.proj_shapes()
        for i, p in enumerate(PROJ):
            n, m = shapes[p]
            k = float(kept[:, i].sum())
            total += k * n * bw
            if self.lm.dtype == C.TEAL_I4:
                total += k / 128.0 * n * 4  # group scales, proportional to touched groups
            total += steps * sp.n_layers * self.B * (m * 4 + n * 4)
            if self.lm.dtype == C.TEAL_I8:
                total += steps * sp.n_layers * n * 4
        total += steps * (sp.d_model * sp.vocab * bw + self.B * (sp.d_model * 4 + sp.vocab * 4))
        return total


def calibrate_batch_histograms(weights: DecoderWeights, batch: int, n_steps: int = 16, seed: int = 0,
                               bins: int | None = None, quant: str | None = None, thresholds=None):
    """Per-batch-size calibration (pkg/tests/test_acceptance.py:
    223-239): run ``n_steps`` dense lockstep decode steps of ``batch`` random
    token streams and bin, per (layer, tap), the batch-mean magnitude vector
    mean_b |h[b, :]| — the statistic the shared mask thresholds.  ``hi`` = 8 x
    the std of the first step's vector.  Returns
    {(layer, tap): ActivationHistogram}."""
    from .sparsifier import DEFAULT_BIN_COUNT, HI_STD_MULTIPLE, ActivationHistogram
    bins = bins or DEFAULT_BIN_COUNT
    spec = weights.spec
    dec = BatchDecoder(weights, thresholds, batch, quant=quant, taps=True)
    dec.reset()
    g = torch.Generator(device=dec.device).manual_seed(seed)
    hists = {}
    for _ in range(n_steps):
        dec.tokens.copy_(torch.randint(0, spec.vocab, (batch,), device=dec.device, generator=g, dtype=torch.int32))
        dec.step()
        for tap in TAPS:
            for l in range(spec.n_layers):
                mm = dec.taps[tap][l].abs().mean(dim=0)  # (calibration: plain torch mean over the batch)
                key = (l, tap)
                if key not in hists:
                    hi = HI_STD_MULTIPLE * float(mm.std(unbiased=False))
                    hists[key] = ActivationHistogram.empty(f"B{batch}.L{l}.{tap}", bins, hi if hi > 0 else 1.0)
                hists[key].record(mm)
    del dec
    torch.cuda.empty_cache()
    return hists


def calibrate_batch_thresholds(weights: DecoderWeights, batch: int, level: float, n_steps: int = 32,
                               seed: int = 0, passes: int = 2) -> list[list[float]]:
    """Batch-size-specific thresholds whose realized column sparsity matches
    ``level``.  The batch-mean statistic is concentrated (averaging B rows), so
    its quantiles move a lot when upstream projections are sparsified: pass 1
    calibrates on the dense decode (the reference's recipe), each further pass
    on the taps seen while decoding with the previous pass's thresholds."""
    thr = None
    for _ in range(max(1, passes)):
        hists = calibrate_batch_histograms(weights, batch, n_steps=n_steps, seed=seed, thresholds=thr)
        thr = batch_thresholds(hists, weights.spec.n_layers, level)
    return thr


def batch_thresholds(hists, n_layers: int, level: float) -> list[list[float]]:
    """[L][7] thresholds at a uniform level from batch-mean histograms."""
    from .decode import uniform_thresholds
    return uniform_thresholds(hists, n_layers, level)
