"""Batch-1 TEAL decode engine on the sm_100a kernels.

One decode step is the reference's `_forward` (pkg/src/actsparse/model.py:
158-198) evaluated for a single new position against a KV cache (the
reference has no cache; by causality a step equals row t of the full
forward, pkg/tests/test_model.py:171-178).  Per layer it launches

  1. qkv   : RMSNorm prologue -> 3 thresholds (q, k, v share the PRE_ATTN tap)
             -> sparse GEMV over the fused [d, n_q + 2 n_kv] input-major weight
             -> RoPE (Llama) + KV-cache write epilogue           (teal_fused_gemv)
  2. attention over the cache, GQA                            (teal_decode_attention)
  3. o     : threshold(ATTN_OUT) -> sparse GEMV -> residual add + sum-of-squares
  4. gate/up: RMSNorm prologue -> 2 thresholds -> sparse GEMV -> SiLU(gate)*up
  5. down  : threshold(MLP_INTER) -> sparse GEMV -> residual add + sum-of-squares

plus the residual load (embedding row or a given hidden row) and, for
Llama-style models, the final-norm dense LM head and greedy argmax.  Every
launch is stream-ordered, allocation-free and captured into one CUDA graph
per step; the step's position lives on the device, so the graph replays
token after token.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT

PROJ = ("q", "k", "v", "o", "gate", "up", "down")


@dataclass(frozen=True)
class DecoderSpec:
    """Shape of a decoder-only transformer (pre-norm, SiLU-gated MLP)."""

    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int
    n_layers: int
    vocab: int = 0                 # 0: no embedding / LM head (hidden rows in, hidden rows out)
    rope_theta: float | None = None  # None: no positional encoding (the reference toy block)
    norm_eps: float = 1e-6         # model.py:36
    max_seq: int = 2048
    head_dim_: int = 0             # 0: d_model // n_heads (set for tensor-parallel shards)

    @property
    def head_dim(self) -> int:
        return self.head_dim_ or self.d_model // self.n_heads

    @property
    def n_q(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def n_kv(self) -> int:
        return self.n_kv_heads * self.head_dim

    def proj_shapes(self) -> dict[str, tuple[int, int]]:
        """(n_out, m_in) of the seven projections."""
        d, f = self.d_model, self.d_ff
        return {"q": (self.n_q, d), "k": (self.n_kv, d), "v": (self.n_kv, d), "o": (d, self.n_q),
                "gate": (f, d), "up": (f, d), "down": (d, f)}

    def weight_bytes(self, elem_bytes: float) -> dict[str, float]:
        """Per-token weight bytes by projection (all layers) + LM head."""
        out = {k: n * m * elem_bytes * self.n_layers for k, (n, m) in self.proj_shapes().items()}
        out["lm_head"] = self.vocab * self.d_model * elem_bytes
        return out


LLAMA3_8B = DecoderSpec(4096, 32, 8, 14336, 32, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
LLAMA3_70B = DecoderSpec(8192, 64, 8, 28672, 80, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
MISTRAL_7B = DecoderSpec(4096, 32, 8, 14336, 32, vocab=32000, rope_theta=1000000.0, norm_eps=1e-5, max_seq=2048)


def toy_spec(d_model=512, n_heads=8, d_ff=1408, n_layers=2, max_seq=512) -> DecoderSpec:
    """The reference toy block (model.py:59-123): MHA, no RoPE, eps 1e-6."""
    return DecoderSpec(d_model, n_heads, n_heads, d_ff, n_layers, vocab=0, rope_theta=None,
                       norm_eps=1e-6, max_seq=max_seq)


@dataclass
class LayerWeights:
    wqkv: torch.Tensor      # [d, n_q + 2 n_kv]  input-major (q | k | v columns)
    wo: torch.Tensor        # [n_q, d]
    wgu: torch.Tensor       # [d, 2 d_ff]        (gate | up columns)
    wdown: torch.Tensor     # [d_ff, d]
    rms_attn: torch.Tensor  # [d] fp32
    rms_mlp: torch.Tensor   # [d] fp32


@dataclass
class DecoderWeights:
    spec: DecoderSpec
    layers: list[LayerWeights]
    embedding: torch.Tensor | None = None  # [vocab, d]
    final_norm: torch.Tensor | None = None  # [d] fp32
    lm_head: torch.Tensor | None = None     # [d, vocab] input-major

    @property
    def dtype(self) -> torch.dtype:
        return self.layers[0].wqkv.dtype


def random_weights(spec: DecoderSpec, dtype=torch.bfloat16, seed: int = 0, device=None) -> DecoderWeights:
    """Random-init weights of `spec` generated on the device: W ~ N(0, 1/d_in)
    (model.py:116-117), unit norm gains, embedding ~ N(0, 1)."""
    dev = device or RT.require_cuda()
    g = torch.Generator(device=dev).manual_seed(seed)

    def w(m_in, n_out):
        t = torch.empty(m_in, n_out, device=dev, dtype=dtype)
        # fill in chunks to bound the fp32 temporary
        rows = max(1, (1 << 27) // max(1, n_out))
        for r in range(0, m_in, rows):
            t[r:r + rows] = (torch.randn(min(rows, m_in - r), n_out, device=dev, generator=g)
                             * (1.0 / math.sqrt(m_in))).to(dtype)
        return t

    d, f = spec.d_model, spec.d_ff
    layers = []
    for _ in range(spec.n_layers):
        layers.append(LayerWeights(
            wqkv=w(d, spec.n_q + 2 * spec.n_kv), wo=w(spec.n_q, d), wgu=w(d, 2 * f), wdown=w(f, d),
            rms_attn=torch.ones(d, device=dev), rms_mlp=torch.ones(d, device=dev)))
    emb = fin = head = None
    if spec.vocab:
        emb = torch.empty(spec.vocab, d, device=dev, dtype=dtype)
        for r in range(0, spec.vocab, 8192):
            emb[r:r + 8192] = torch.randn(min(8192, spec.vocab - r), d, device=dev, generator=g).to(dtype)
        fin = torch.ones(d, device=dev)
        head = w(d, spec.vocab)
    return DecoderWeights(spec, layers, emb, fin, head)


def weights_from_blocks(blocks, n_heads: int, dtype=torch.float32, device=None, max_seq: int = 512) -> DecoderWeights:
    """Device weights for reference-style blocks given as dicts of logical
    [n_out, d_in] numpy matrices (model.py:60-123): (weights, rms_attn, rms_mlp)."""
    dev = device or RT.require_cuda()
    w0 = blocks[0][0]
    d = w0["q"].shape[1]
    f = w0["gate"].shape[0]
    spec = toy_spec(d, n_heads, f, len(blocks), max_seq)

    def im(a):  # logical [n_out, d_in] -> input-major [d_in, n_out]
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32).T)).to(dev, dtype)

    layers = []
    for wd, ra, rm in blocks:
        layers.append(LayerWeights(
            wqkv=torch.cat([im(wd["q"]), im(wd["k"]), im(wd["v"])], dim=1).contiguous(),
            wo=im(wd["o"]), wgu=torch.cat([im(wd["gate"]), im(wd["up"])], dim=1).contiguous(),
            wdown=im(wd["down"]),
            rms_attn=torch.from_numpy(np.asarray(ra, np.float32)).to(dev),
            rms_mlp=torch.from_numpy(np.asarray(rm, np.float32)).to(dev)))
    return DecoderWeights(spec, layers)


def _seg(a: C.TealGemvArgs, i: int, w: torch.Tensor, col0: int, n: int, t32: float, y=None):
    s = a.seg[i]
    s.w = w.data_ptr() + col0 * w.element_size()
    s.ldw = w.stride(0)
    s.n = n
    s.t32 = t32
    s.y = RT.ptr(y)
    s.col_scale = None
    s.dbg_bits = None
    s.kept = None


def _t32(t) -> float:
    """Model-path threshold: `sparsify` compares in fp32 after RN (sparsifier.py:121-125)."""
    if t is None:
        return float("-inf")
    return RT.f32_round_nearest(float(t))


@dataclass
class StepTaps:
    """Optional per-step debug outputs: the four tap vectors (model.py:171-193)
    and the keep bitmask of each of the seven projection inputs."""

    h: dict[str, torch.Tensor] = field(default_factory=dict)       # tap -> [n_layers, dim] fp32
    bits: dict[str, torch.Tensor] = field(default_factory=dict)    # proj -> [n_layers, words] int32
    kept: torch.Tensor | None = None                              # [n_layers, 7] int64


class SparseDecoder:
    """TEAL decode for one sequence (batch 1).

    thresholds: None (dense) or per-layer sequences of 7 floats in the
    order q, k, v, o, gate, up, down (BlockSparsityConfig.thresholds,
    model.py:226-244).  A threshold of None or -inf disables that
    projection's mask (dense GEMV through the same kernel)."""

    def __init__(self, weights: DecoderWeights, thresholds=None, kv_dtype=None, device=None,
                 attn_chunk: int = 64, taps: bool = False, lm_threshold: float | None = None):
        self.w = weights
        # optional LM-head input threshold (§8(f)#3): None = the dense LM head
        self.lm_threshold = lm_threshold
        spec = self.spec = weights.spec
        dev = self.device = device or RT.require_cuda()
        self.kv_dtype = kv_dtype or weights.dtype
        d, hd = spec.d_model, spec.head_dim
        L = spec.n_layers
        f32 = dict(device=dev, dtype=torch.float32)
        self.x = torch.zeros(d, **f32)
        self.x_in = torch.zeros(d, **f32)
        self.q = torch.zeros(spec.n_q, **f32)
        self.ctx = torch.zeros(spec.n_q, **f32)
        self.inter = torch.zeros(spec.d_ff, **f32)
        self.state = torch.zeros(2, device=dev, dtype=torch.int32)  # {pos, len}
        self.token = torch.zeros(1, device=dev, dtype=torch.int32)
        self.logits = torch.zeros(max(spec.vocab, 1), **f32)
        self.kcache = torch.zeros(L, spec.n_kv_heads, spec.max_seq, hd, device=dev, dtype=self.kv_dtype)
        self.vcache = torch.zeros_like(self.kcache)
        if spec.rope_theta is not None:
            inv = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
            ang = torch.arange(spec.max_seq, dtype=torch.float64)[:, None] * inv[None, :]
            self.rope_cos = torch.cos(ang).float().to(dev).contiguous()
            self.rope_sin = torch.sin(ang).float().to(dev).contiguous()
        else:
            self.rope_cos = self.rope_sin = None
        self.attn_nsplit = max(1, -(-spec.max_seq // attn_chunk))
        self.taps = StepTaps() if taps else None
        if taps:
            for tap, dim in (("pre_attn", d), ("attn_out", spec.n_q), ("pre_mlp", d), ("mlp_inter", spec.d_ff)):
                self.taps.h[tap] = torch.zeros(L, dim, **f32)
            for p, (_, m_in) in spec.proj_shapes().items():
                self.taps.bits[p] = torch.zeros(L, (m_in + 31) // 32, device=dev, dtype=torch.int32)
            self.taps.kept = torch.zeros(L, 7, device=dev, dtype=torch.int64)
        self._build(thresholds)
        self.graph = None
        self._pos = 0

    # -- launch descriptors ---------------------------------------------------
    def _build(self, thresholds):
        spec, W = self.spec, self.w
        d, f = spec.d_model, spec.d_ff
        nq, nkv = spec.n_q, spec.n_kv
        L = spec.n_layers
        thr = [[None] * 7 for _ in range(L)] if thresholds is None else [list(t) for t in thresholds]
        if len(thr) != L or any(len(t) != 7 for t in thr):
            raise ValueError(f"need {L} per-layer threshold lists of 7 (q,k,v,o,gate,up,down)")
        self.thresholds = thr
        wcode = RT.dtype_code(W.dtype)
        # the residual tiles (o / down outputs) fix the sum-of-squares partial layout
        probe = C.TealGemvArgs()
        probe.w_dtype, probe.nseg = wcode, 1
        _seg(probe, 0, W.layers[0].wo, 0, d, 0.0)
        self.res_tile = C.lib().teal_gemv_tile_width(ctypes.byref(probe))
        self.ss_count = -(-d // self.res_tile)
        self.ss = torch.zeros(max(self.ss_count, 1), device=self.device)
        self.layer_args = []
        max_ws, max_tk = 0, 0
        T = self.taps
        for l, (lw, t) in enumerate(zip(W.layers, thr)):
            kc = self.kcache[l]
            vc = self.vcache[l]
            # 1. q/k/v (RMSNorm prologue, QKV epilogue)
            a = C.TealGemvArgs()
            a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = wcode, C.TEAL_F32, self.x.data_ptr(), d, 3
            _seg(a, 0, lw.wqkv, 0, nq, _t32(t[0]))
            _seg(a, 1, lw.wqkv, nq, nkv, _t32(t[1]))
            _seg(a, 2, lw.wqkv, nq + nkv, nkv, _t32(t[2]))
            a.prologue, a.norm_scale, a.ss_part, a.ss_count, a.eps = (
                C.PRO_RMSNORM, lw.rms_attn.data_ptr(), self.ss.data_ptr(), self.ss_count, spec.norm_eps)
            a.epilogue, a.q_out, a.k_cache, a.v_cache = C.EPI_QKV, self.q.data_ptr(), kc.data_ptr(), vc.data_ptr()
            a.kv_dtype, a.max_seq, a.pos, a.head_dim = RT.dtype_code(self.kv_dtype), spec.max_seq, self.state.data_ptr(), spec.head_dim
            a.rope_cos, a.rope_sin = RT.ptr(self.rope_cos), RT.ptr(self.rope_sin)
            qkv = a
            # 3. o (plain prologue over ctx, residual epilogue)
            a = C.TealGemvArgs()
            a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = wcode, C.TEAL_F32, self.ctx.data_ptr(), nq, 1
            _seg(a, 0, lw.wo, 0, d, _t32(t[3]))
            a.prologue, a.epilogue, a.resid, a.ss_out = C.PRO_PLAIN, C.EPI_RESID, self.x.data_ptr(), self.ss.data_ptr()
            o = a
            # 4. gate/up (RMSNorm prologue, SiLU epilogue)
            a = C.TealGemvArgs()
            a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = wcode, C.TEAL_F32, self.x.data_ptr(), d, 2
            _seg(a, 0, lw.wgu, 0, f, _t32(t[4]))
            _seg(a, 1, lw.wgu, f, f, _t32(t[5]))
            a.prologue, a.norm_scale, a.ss_part, a.ss_count, a.eps = (
                C.PRO_RMSNORM, lw.rms_mlp.data_ptr(), self.ss.data_ptr(), self.ss_count, spec.norm_eps)
            a.epilogue, a.inter = C.EPI_SILU, self.inter.data_ptr()
            gu = a
            # 5. down (plain prologue over inter, residual epilogue)
            a = C.TealGemvArgs()
            a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = wcode, C.TEAL_F32, self.inter.data_ptr(), f, 1
            _seg(a, 0, lw.wdown, 0, d, _t32(t[6]))
            a.prologue, a.epilogue, a.resid, a.ss_out = C.PRO_PLAIN, C.EPI_RESID, self.x.data_ptr(), self.ss.data_ptr()
            dn = a
            if T is not None:
                qkv.dbg_h = T.h["pre_attn"][l].data_ptr()
                o.dbg_h = T.h["attn_out"][l].data_ptr()
                gu.dbg_h = T.h["pre_mlp"][l].data_ptr()
                dn.dbg_h = T.h["mlp_inter"][l].data_ptr()
                for args, names in ((qkv, ("q", "k", "v")), (o, ("o",)), (gu, ("gate", "up")), (dn, ("down",))):
                    for i, p in enumerate(names):
                        args.seg[i].dbg_bits = T.bits[p][l].data_ptr()
                        args.seg[i].kept = T.kept[l, PROJ.index(p)].data_ptr()
            for a in (qkv, o, gu, dn):
                _, nws, ntk = RT.gemv_workspace(a)
                max_ws, max_tk = max(max_ws, nws), max(max_tk, ntk)
            self.layer_args.append((qkv, o, gu, dn))
        self.lm_args = None
        if self.spec.vocab:
            a = C.TealGemvArgs()
            a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = wcode, C.TEAL_F32, self.x.data_ptr(), d, 1
            _seg(a, 0, W.lm_head, 0, spec.vocab, _t32(self.lm_threshold), self.logits)
            a.prologue, a.norm_scale, a.ss_part, a.ss_count, a.eps = (
                C.PRO_RMSNORM, W.final_norm.data_ptr(), self.ss.data_ptr(), self.ss_count, spec.norm_eps)
            a.epilogue = C.EPI_STORE
            _, nws, ntk = RT.gemv_workspace(a)
            max_ws, max_tk = max(max_ws, nws), max(max_tk, ntk)
            self.lm_args = a
        G = spec.n_heads // spec.n_kv_heads
        attn_ws = spec.n_kv_heads * self.attn_nsplit * (G * spec.head_dim + 2 * G)
        self.ws = torch.zeros(max(max_ws, attn_ws, 2 * 256), device=self.device)
        self.tickets = torch.zeros(max(max_tk, spec.n_kv_heads, 1) + 16, device=self.device, dtype=torch.int32)
        for group in self.layer_args:
            for a in group:
                a.ws, a.tickets = self.ws.data_ptr(), self.tickets.data_ptr()
        if self.lm_args is not None:
            self.lm_args.ws, self.lm_args.tickets = self.ws.data_ptr(), self.tickets.data_ptr()

    # -- step ---------------------------------------------------------------
    def reset(self, start_pos: int = 0) -> None:
        """Forget the cache; the next step writes position `start_pos`."""
        self.state.copy_(torch.tensor([start_pos - 1, start_pos], dtype=torch.int32))
        self._pos = start_pos
        if start_pos == 0:
            self.kcache.zero_()
            self.vcache.zero_()

    def _advance(self) -> None:
        """Host-side position guard: the step about to run writes K/V row
        `_pos`, which must lie inside the cache (the QKV epilogue also traps)."""
        if self._pos >= self.spec.max_seq:
            raise ValueError(f"decode position {self._pos} would exceed max_seq {self.spec.max_seq} "
                             f"(the KV cache holds positions [0, {self.spec.max_seq}))")
        self._pos += 1

    def launches_per_step(self) -> int:
        return 1 + 5 * self.spec.n_layers + (2 if self.lm_args is not None else 0)

    def _launch_step(self, stream_h: int, from_token: bool) -> None:
        L = C.lib()
        spec = self.spec
        if from_token:
            src, sdt, tok = self.w.embedding.data_ptr(), RT.dtype_code(self.w.embedding.dtype), self.token.data_ptr()
        else:
            src, sdt, tok = self.x_in.data_ptr(), C.TEAL_F32, None
        C.check(L.teal_load_residual(src, sdt, tok, spec.d_model, self.x.data_ptr(), self.ss.data_ptr(),
                                     self.res_tile, self.state.data_ptr(), stream_h))
        len_ptr = self.state.data_ptr() + 4
        for l, (qkv, o, gu, dn) in enumerate(self.layer_args):
            C.check(L.teal_fused_gemv(ctypes.byref(qkv), stream_h))
            C.check(L.teal_decode_attention(self.q.data_ptr(), self.kcache[l].data_ptr(), self.vcache[l].data_ptr(),
                                            RT.dtype_code(self.kv_dtype), spec.n_heads, spec.n_kv_heads,
                                            spec.head_dim, spec.max_seq, len_ptr, spec.max_seq,
                                            self.ctx.data_ptr(), self.ws.data_ptr(), self.tickets.data_ptr(),
                                            self.attn_nsplit, stream_h))
            C.check(L.teal_fused_gemv(ctypes.byref(o), stream_h))
            C.check(L.teal_fused_gemv(ctypes.byref(gu), stream_h))
            C.check(L.teal_fused_gemv(ctypes.byref(dn), stream_h))
        if self.lm_args is not None:
            C.check(L.teal_fused_gemv(ctypes.byref(self.lm_args), stream_h))
            C.check(L.teal_argmax(self.logits.data_ptr(), spec.vocab, self.token.data_ptr(), self.ws.data_ptr(),
                                  self.tickets.data_ptr(), stream_h))

    def step_hidden(self, x_row) -> torch.Tensor:
        """One step from a hidden row (no embedding): returns the new residual
        stream x (a view of the engine buffer)."""
        if isinstance(x_row, torch.Tensor):
            self.x_in.copy_(x_row.reshape(-1), non_blocking=True)
        else:
            self.x_in.copy_(torch.from_numpy(np.ascontiguousarray(x_row, dtype=np.float32)), non_blocking=True)
        self._advance()
        self._launch_step(RT.stream_handle(), from_token=False)
        return self.x

    def step_token(self) -> torch.Tensor:
        """One step from self.token (embedding lookup); leaves the argmax next
        token in self.token and returns it."""
        self._advance()
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch_step(RT.stream_handle(), from_token=True)
        return self.token

    def step_token_host(self, tok_in: torch.Tensor, tok_out: torch.Tensor) -> None:
        """End-to-end step through host buffers: H2D copy of the input token
        (pinned int32 [1]), one decode step, D2H copy of the argmax token into
        ``tok_out`` (pinned int32 [1]).  Stream-ordered, no host sync."""
        self.token.copy_(tok_in, non_blocking=True)
        self.step_token()
        tok_out.copy_(self.token, non_blocking=True)

    def capture(self, from_token: bool = True) -> torch.cuda.CUDAGraph:
        """Capture one step into a CUDA graph (replayed by step_token / replay())."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._launch_step(s.cuda_stream, from_token)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        return g

    def replay(self) -> None:
        self._advance()
        self.graph.replay()


# tap of each projection's input (model.py:39-56, MATRIX_TAP)
PROJ_TAP = {"q": "pre_attn", "k": "pre_attn", "v": "pre_attn", "o": "attn_out",
            "gate": "pre_mlp", "up": "pre_mlp", "down": "mlp_inter"}


def calibrate_histograms(weights, n_tokens: int = 16, seed: int = 0,
                         bins: int | None = None, hi_std_multiple: float | None = None, engine: str = "launch",
                         thresholds=None):
    """GPU-side calibration of the decode engine (model.py:268-294 restated for
    the KV-cache decode): run ``n_tokens`` dense decode steps on random tokens
    with the four taps captured, and bin each (layer, tap) vector on the GPU
    (``teal_hist_record``).  ``hi`` = HI_STD_MULTIPLE * std of the first
    step's tap, as the reference takes it from the first calibration sequence
    (model.py:286-291).  ``engine='step'`` runs the persistent engine (and
    accepts pre-tiled weights).  Returns {(layer, tap): ActivationHistogram}."""
    from .sparsifier import DEFAULT_BIN_COUNT, HI_STD_MULTIPLE, ActivationHistogram
    bins = bins or DEFAULT_BIN_COUNT
    mult = hi_std_multiple or HI_STD_MULTIPLE
    spec = weights.spec
    if not spec.vocab:
        raise ValueError("token calibration needs an embedding (vocab > 0)")
    if engine == "step":
        from .engine import StepDecoder
        dec = StepDecoder(weights, thresholds, taps=True)
    else:
        dec = SparseDecoder(weights, thresholds, taps=True)
    dec.reset()
    g = torch.Generator(device=dec.device).manual_seed(seed)
    toks = torch.randint(0, spec.vocab, (n_tokens,), device=dec.device, generator=g, dtype=torch.int32)
    hists = {}
    for i in range(n_tokens):
        dec.token.copy_(toks[i:i + 1])
        dec.step_token()
        for tap, h in dec.taps.h.items():
            for l in range(spec.n_layers):
                key = (l, tap)
                if key not in hists:
                    hi = mult * float(h[l].std(unbiased=False))
                    hists[key] = ActivationHistogram.empty(f"L{l}.{tap}", bins, hi if hi > 0 else 1.0)
                hists[key].record(h[l])
    del dec
    return hists


def calibrate_thresholds(weights, level: float, n_tokens: int = 128, seed: int = 0, passes: int = 2,
                         engine: str = "step") -> list[list[float]]:
    """Uniform-level thresholds whose REALIZED sparsity matches ``level``:
    pass 1 is the reference's calibration (tap histograms of the dense decode,
    model.py:268-294); every further pass re-records the taps while decoding
    with the previous pass's thresholds, so taps downstream of sparsified
    projections (attention output, SiLU*up) are calibrated on the
    activations they will actually see.  passes=1 is the reference's recipe."""
    thr = None
    for _ in range(max(1, passes)):
        hists = calibrate_histograms(weights, n_tokens=n_tokens, seed=seed, engine=engine, thresholds=thr)
        thr = uniform_thresholds(hists, weights.spec.n_layers, level)
    return thr


def uniform_thresholds(hists, n_layers: int, level: float) -> list[list[float]]:
    """Per-layer thresholds of a uniform config (greedy.py:130-134 with
    resolve_config, model.py:253-265): every projection at ``level``."""
    out = []
    cache = {}
    for l in range(n_layers):
        row = []
        for p in PROJ:
            key = (l, PROJ_TAP[p])
            if key not in cache:
                cache[key] = hists[key].threshold(level)
            row.append(cache[key])
        out.append(row)
    return out
