"""Persistent batch-1 decode engine: ONE cooperative sm_100a launch per token
(``teal_step_launch``, csrc/teal_step.cu).

Same decode-step semantics as :class:`.decode.SparseDecoder` (the
reference's ``_forward`` for one new position against a KV cache,
pkg/src/actsparse/model.py:158-198) but scheduled as a dependency-driven
work queue instead of 5 launches per layer, so the 148 SMs stream weights
without launch gaps or grid-wide barriers.

Weights are re-laid out once into the TILED input-major format the kernel
streams (``pack_tiled`` / ``pack_gate_up``): for a group with output columns
cut into tiles of TW = 256, tile t is the contiguous block ``[m][TW]`` so a
kept input channel reads one contiguous 512-byte (bf16) row chunk per tile.
The MLP tile interleaves 128 gate and 128 up columns so the SiLU(gate)*up
epilogue stays inside one tile.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT
from .decode import PROJ, DecoderWeights, StepTaps, _t32

TW = 256
TH = TW // 2
SEPI_STORE, SEPI_RESID, SEPI_SILU, SEPI_QKV, SEPI_LOGITS = 0, 1, 2, 3, 4

c_i64, c_vp, c_f, c_i = ctypes.c_int64, ctypes.c_void_p, ctypes.c_float, ctypes.c_int


class StepTile(ctypes.Structure):
    _fields_ = [("t_lo", c_f), ("t_hi", c_f), ("seg_lo", c_i), ("seg_hi", c_i),
                ("first_lo", c_i), ("first_hi", c_i), ("sig0", c_i), ("sig1", c_i)]


class StepGroup(ctypes.Structure):
    _fields_ = [("w", c_vp), ("col_scale", c_vp), ("tiles", c_vp), ("x", c_vp), ("gain", c_vp), ("ss", c_vp),
                ("partials", c_vp), ("tickets", c_vp), ("y", c_vp), ("resid", c_vp), ("ss_out", c_vp),
                ("inter", c_vp), ("q_out", c_vp), ("k_cache", c_vp), ("v_cache", c_vp), ("rope_cos", c_vp),
                ("rope_sin", c_vp), ("dbg_h", c_vp), ("dbg_bits", c_vp * 3), ("kept", c_vp * 3),
                ("max_seq", c_i64), ("m", c_i), ("n", c_i), ("ntiles", c_i), ("maxc", c_i),
                ("prologue", c_i), ("nss", c_i), ("eps", c_f), ("epilogue", c_i),
                ("nq", c_i), ("nkv", c_i), ("head_dim", c_i), ("kv_dtype", c_i), ("w_dtype", c_i),
                ("gscale", c_vp), ("group", c_i), ("t_all", c_f), ("tile_stride_b", c_i64), ("row_stride_b", c_i64),
                ("acc", c_vp), ("in_acc", c_vp), ("x_out", c_vp), ("ranges", c_vp), ("nranges", c_i),
                ("xsig", c_i), ("xwait", c_i), ("xwait_target", c_i), ("tp_sum", c_i)]


class StepAttn(ctypes.Structure):
    _fields_ = [("q", c_vp), ("k_cache", c_vp), ("v_cache", c_vp), ("ctx", c_vp), ("partials", c_vp),
                ("tickets", c_vp), ("max_seq", c_i64), ("H", c_i), ("KVH", c_i), ("hd", c_i), ("kv_dtype", c_i),
                ("chunk", c_i), ("nchunks", c_i), ("sig_base", c_i), ("dep_base", c_i), ("dep_target", c_vp),
                ("dbg", c_vp), ("qkv_acc", c_vp), ("rope_cos", c_vp), ("rope_sin", c_vp), ("nq", c_i), ("nkv", c_i),
                ("super_chunks", c_i), ("home", c_i)]


class StepPhase(ctypes.Structure):
    _fields_ = [("kind", c_i), ("group", c_i), ("dep_kind", c_i), ("dep", c_i), ("target", c_i), ("dep_rows", c_i)]


class StepPlan(ctypes.Structure):
    _fields_ = [("groups", c_vp), ("attns", c_vp), ("phases", c_vp), ("counters", c_vp), ("ctrl", c_vp),
                ("emb", c_vp), ("x_in", c_vp), ("token", c_vp), ("x", c_vp), ("ss", c_vp), ("state", c_vp),
                ("cand_v", c_vp), ("cand_i", c_vp), ("token_out", c_vp), ("lm_done", c_vp), ("timeline", c_vp),
                ("nphases", c_i), ("ncounters", c_i), ("prefetch_bytes", c_i), ("max_seq", c_i),
                ("d", c_i), ("emb_dtype", c_i), ("w_dtype", c_i), ("ctas", c_i),
                ("acc_zero", c_vp), ("acc_zero_n", c_i64), ("tp", c_vp), ("noncoop", c_i), ("long_ctx", c_i),
                ("phase_begin", c_i), ("phase_end", c_i)]


TP_MAX = 8


class StepTP(ctypes.Structure):
    _fields_ = [("acc", c_vp * TP_MAX), ("counters", c_vp * TP_MAX), ("epoch", c_vp * TP_MAX),
                ("token", c_vp * TP_MAX), ("cand_v", c_vp), ("cand_i", c_vp), ("lm_ticket", c_vp),
                ("world", c_i), ("rank", c_i), ("vocab_off", c_i), ("pad_", c_i)]


PHASE_LOAD, PHASE_GEMV, PHASE_ATTN, PHASE_RESID = 0, 1, 2, 3
PRO_RMS_ACC, PRO_SILU_ACC = 2, 3
CONTRIB = 1024  # TEAL_STEP_CONTRIB: counter units per finished tile of an ACC output
XS_MAX = 8192   # PRO_RMS_ACC staging limit on d
DEP_NONE, DEP_GLOBAL, DEP_ROWS = 0, 1, 2


def participants(ntiles: int, F: int, grid: int) -> int:
    """CTAs taking part in a GEMV phase (csrc/teal_step.cu participants())."""
    if F <= grid:
        return F
    aligned = ntiles * (grid // ntiles)
    if 2 * ntiles <= grid and 10 * aligned >= 9 * grid:
        return aligned
    return grid


def max_contributors(ntiles: int, m: int, G: int) -> int:
    """Most CTAs sharing one tile under the equal-range split of the
    flattened (tile, 32-row group) space (csrc/teal_step.cu owner_of)."""
    gpt = -(-m // 32)
    F = ntiles * gpt
    G = participants(ntiles, F, G)

    def owner(x):
        return ((x + 1) * G - 1) // F
    return max(owner((t + 1) * gpt - 1) - owner(t * gpt) + 1 for t in range(ntiles))


def weighted_ranges(ntiles: int, m: int, grid: int, penalty: int):
    """Work split of an ACC group whose equal ranges would cross tiles: CTA
    ranges of 32-row groups where a range spanning two tiles is charged
    `penalty` extra groups (its second compaction / reduction / ramp-up), so
    the two-tile CTAs, which gate half the tiles, finish with the rest.
    Returns [(g0, g1, w_first_tile, w_second_tile)] per CTA (counter weights:
    the first contributor of a tile adds CONTRIB - (contributors - 1), the
    others 1), or None when the equal split already keeps ranges in one tile."""
    gpt = -(-m // 32)
    F = ntiles * gpt
    if participants(ntiles, F, grid) != grid or F <= grid or penalty <= 0 or F > grid * gpt:
        return None
    if grid % ntiles == 0 or all((c * F // grid) // gpt == ((c + 1) * F // grid - 1) // gpt for c in range(grid)):
        return None

    def split(T):
        out, g = [], 0
        while g < F:
            t = g // gpt
            end1 = (t + 1) * gpt
            if end1 - g >= T:           # fits in this tile
                e = g + T
            elif end1 - g + penalty < T and end1 < F:  # spill into the next tile (never a third)
                e = min(F, end1 + gpt - 1, g + T - penalty)
            else:
                e = end1
            out.append((g, e))
            g = e
        return out

    lo, hi = 1, F
    while lo < hi:
        T = (lo + hi) // 2
        if len(split(T)) <= grid:
            hi = T
        else:
            lo = T + 1
    rs = split(lo)
    contrib = {}
    for i, (a, b) in enumerate(rs):
        for t in range(a // gpt, (b - 1) // gpt + 1):
            contrib.setdefault(t, []).append(i)
    res = []
    for i, (a, b) in enumerate(rs):
        ws = []
        for t in range(a // gpt, (b - 1) // gpt + 1):
            cs = contrib[t]
            ws.append(CONTRIB - (len(cs) - 1) if cs[0] == i else 1)
        ws += [0] * (2 - len(ws))
        res.append((a, b, ws[0], ws[1]))
    return res


_BOUND = False


def _bind():
    global _BOUND
    if not _BOUND:
        L = C.lib()
        L.teal_step_launch.restype = ctypes.c_int
        L.teal_step_launch.argtypes = [ctypes.POINTER(StepPlan), c_vp]
        L.teal_step_ctas_per_sm.restype = ctypes.c_int
        L.teal_step_ctas_per_sm.argtypes = [c_i]
        _BOUND = True
    return C.lib()


# ---- tiled weight layout --------------------------------------------------------

def pack_tiled(w_in_major: torch.Tensor, tw: int = TW) -> torch.Tensor:
    """[m, n] input-major -> [ceil(n/tw), m, tw] (zero-padded columns)."""
    m, n = w_in_major.shape
    nt = -(-n // tw)
    out = torch.zeros(nt, m, tw, dtype=w_in_major.dtype, device=w_in_major.device)
    for t in range(nt):
        c1 = min(n, (t + 1) * tw)
        out[t, :, : c1 - t * tw] = w_in_major[:, t * tw: c1]
    return out


def pack_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, tw: int = TW) -> torch.Tensor:
    """gate/up [m, f] each -> [ceil(f/(tw/2)), m, tw]: tile t = gate cols
    [t*tw/2, (t+1)*tw/2) | up cols of the same range."""
    m, f = w_gate.shape
    th = tw // 2
    nt = -(-f // th)
    out = torch.zeros(nt, m, tw, dtype=w_gate.dtype, device=w_gate.device)
    for t in range(nt):
        c1 = min(f, (t + 1) * th)
        out[t, :, : c1 - t * th] = w_gate[:, t * th: c1]
        out[t, :, th: th + c1 - t * th] = w_up[:, t * th: c1]
    return out


@dataclass
class TiledW:
    """One group's tiled weights: data [ntiles, m, TW] (fp32 / bf16 / int8)
    or [ntiles, m, TW/2] uint8 (int4 nibbles, low = even column); int8 carries
    a per-column scale [ntiles*TW], int4 a per (row group, column) scale
    [ceil(m/group), ntiles*TW]."""

    data: torch.Tensor
    col_scale: torch.Tensor | None = None
    gscale: torch.Tensor | None = None
    group: int = 0

    @property
    def ntiles(self) -> int:
        return self.data.shape[0]

    @property
    def dtype_code(self) -> int:
        if self.data.dtype == torch.uint8:
            return C.TEAL_I4
        return RT.dtype_code(self.data.dtype)

    def dequantize(self) -> torch.Tensor:
        """fp32 [ntiles, m, TW] values the kernel multiplies with."""
        d = self.data
        nt, m = d.shape[0], d.shape[1]
        if d.dtype == torch.int8:
            return d.float() * self.col_scale.view(nt, 1, TW)
        if d.dtype == torch.uint8:
            lo = (d & 0xF).to(torch.int16)
            hi = (d >> 4).to(torch.int16)
            q = torch.stack([lo, hi], dim=-1).reshape(nt, m, TW)
            q = torch.where(q >= 8, q - 16, q).float()
            gi = torch.arange(m, device=d.device) // self.group
            sc = self.gscale.view(-1, nt, TW)[gi]          # [m, nt, TW]
            return q * sc.permute(1, 0, 2)
        return d.float()


def quantize_tiles(t: torch.Tensor, quant: str | None, group: int = 128) -> TiledW:
    """Quantise tiled weights [ntiles, m, TW]: None keeps the dtype; 'int8'
    symmetric per output column; 'int4' symmetric per (row group, column)."""
    if quant == "int4" and (group < 128 or group & (group - 1)):
        raise ValueError("int4 row groups must be a power of two >= 128")
    if quant is None:
        return TiledW(t.contiguous())
    w = t.float()
    nt, m, tw = w.shape
    if quant == "int8":
        sc = w.abs().amax(dim=1) / 127.0                                   # [nt, TW]
        sc = torch.where(sc > 0, sc, torch.ones_like(sc))
        q = torch.clamp(torch.round(w / sc[:, None, :]), -127, 127).to(torch.int8)
        return TiledW(q.contiguous(), col_scale=sc.reshape(-1).contiguous())
    if quant == "int4":
        ng = -(-m // group)
        pad = ng * group - m
        wp = torch.cat([w, torch.zeros(nt, pad, tw, device=w.device)], dim=1) if pad else w
        sc = wp.view(nt, ng, group, tw).abs().amax(dim=2) / 7.0            # [nt, ng, TW]
        sc = torch.where(sc > 0, sc, torch.ones_like(sc))
        gi = torch.arange(m, device=w.device) // group
        q = torch.clamp(torch.round(w / sc[:, gi, :]), -8, 7).to(torch.int16)
        qu = (q & 0xF).to(torch.uint8).view(nt, m, tw // 2, 2)
        packed = (qu[..., 0] | (qu[..., 1] << 4)).contiguous()
        return TiledW(packed, gscale=sc.permute(1, 0, 2).reshape(ng, nt * tw).contiguous(), group=group)
    raise ValueError(f"unknown quantisation {quant!r} (None, 'int8', 'int4')")


def untile(t: torch.Tensor, n: int) -> torch.Tensor:
    """[ntiles, m, TW] -> input-major [m, n]."""
    nt, m, tw = t.shape
    return t.permute(1, 0, 2).reshape(m, nt * tw)[:, :n].contiguous()


def untile_gate_up(t: torch.Tensor, f: int) -> torch.Tensor:
    """Interleaved gate|up tiles -> input-major [m, 2f] (gate columns, then up)."""
    nt, m, tw = t.shape
    g = t[:, :, : tw // 2].permute(1, 0, 2).reshape(m, -1)[:, :f]
    u = t[:, :, tw // 2:].permute(1, 0, 2).reshape(m, -1)[:, :f]
    return torch.cat([g, u], dim=1).contiguous()


@dataclass
class TiledModel:
    """Decoder weights generated directly in the tiled layout (no untiled
    copy: Llama-3-70B bf16 fits one B200 only this way).  `layers[l]` holds
    the norm gains (rms_attn, rms_mlp), `tiles[l]` the TiledW groups."""

    spec: object
    layers: list
    tiles: list
    embedding: torch.Tensor | None
    final_norm: torch.Tensor | None
    lm: TiledW | None

    @property
    def dtype(self) -> torch.dtype:
        return self.embedding.dtype if self.embedding is not None else torch.bfloat16


def random_tiled_model(spec, dtype=torch.bfloat16, seed: int = 0, device=None, quant: str | None = None,
                       pool_gb: float = 2.0) -> TiledModel:
    """Random-init tiled weights W ~ N(0, 1/d_in) (model.py:116-117 scale).
    Values are copied out of one seeded pool of Gaussian samples at rotating
    offsets (HBM copy speed instead of RNG speed for 140 GB), which keeps
    every tile's rows distinct."""
    from types import SimpleNamespace
    dev = device or RT.require_cuda()
    g = torch.Generator(device=dev).manual_seed(seed)
    pool = torch.randn(int(pool_gb * (1 << 30)) // 2, device=dev, generator=g, dtype=torch.float32).to(dtype)
    state = {"off": 0}
    prime = 1000003

    def fill(nt, m, tw, scale):
        t = torch.empty(nt, m, tw, device=dev, dtype=dtype)
        flat = t.view(-1)
        pos = 0
        while pos < flat.numel():
            n = min(flat.numel() - pos, pool.numel() // 2)
            o = state["off"] % (pool.numel() - n)
            flat[pos:pos + n] = pool[o:o + n]
            state["off"] += prime * 7919 + n // 3
            pos += n
        t.mul_(scale)
        return quantize_tiles(t, quant)

    d, f = spec.d_model, spec.d_ff
    nq, nkv = spec.n_q, spec.n_kv
    layers, tiles = [], []
    for _ in range(spec.n_layers):
        layers.append(SimpleNamespace(rms_attn=torch.ones(d, device=dev), rms_mlp=torch.ones(d, device=dev)))
        tiles.append(dict(qkv=fill(-(-(nq + 2 * nkv) // TW), d, TW, d ** -0.5), o=fill(d // TW, nq, TW, nq ** -0.5),
                          gu=fill(f // TH, d, TW, d ** -0.5), down=fill(d // TW, f, TW, f ** -0.5)))
    emb = fin = lm = None
    if spec.vocab:
        emb = torch.empty(spec.vocab, d, device=dev, dtype=dtype)
        for r in range(0, spec.vocab, 8192):
            emb[r:r + 8192] = torch.randn(min(8192, spec.vocab - r), d, device=dev, generator=g).to(dtype)
        fin = torch.ones(d, device=dev)
        lm = fill(-(-spec.vocab // TW), d, TW, d ** -0.5)
    del pool
    torch.cuda.empty_cache()
    return TiledModel(spec, layers, tiles, emb, fin, lm)


class StepDecoder:
    """TEAL decode for one sequence with one persistent launch per token.

    Same constructor arguments and step API as :class:`.decode.SparseDecoder`
    (thresholds per layer in the order q,k,v,o,gate,up,down; None or -inf =
    dense for that projection)."""

    def __init__(self, weights, thresholds=None, kv_dtype=None, device=None,
                 taps: bool = False, attn_chunk: int = 0, ctas: int = 0,
                 count_kept: bool = False, attn_debug: bool = False, prefetch_kb: int = 0,
                 quant: str | None = None, long_context: int = 0, long_from: int = 2048,
                 lm_threshold: float | None = None):
        self.w = weights
        # optional LM-head input threshold (§8(f)#3): None = the dense LM head
        self.lm_threshold = lm_threshold
        spec = self.spec = weights.spec
        dev = self.device = device or RT.require_cuda()
        _bind()
        d, f, hd = spec.d_model, spec.d_ff, spec.head_dim
        nq, nkv, L = spec.n_q, spec.n_kv, spec.n_layers
        G = spec.n_heads // spec.n_kv_heads
        if d % TW or nq % TW or nkv % TH or (nq + 2 * nkv) % TW or TH % hd or f % TH:
            raise ValueError(f"StepDecoder needs d, n_q multiples of {TW}, n_kv of {TH}, head_dim | {TH}, "
                             f"d_ff multiple of {TH}")
        if d > XS_MAX:
            raise ValueError(f"StepDecoder needs d_model <= {XS_MAX}")
        if G > 8 or hd > 128 or G * hd > 1024:
            raise ValueError("StepDecoder attention supports <= 8 q heads per kv head and head_dim <= 128")
        kvb = torch.empty(0, dtype=kv_dtype or weights.dtype).element_size()
        stage_max = 16384 // (hd * kvb)  # positions whose K (and V) rows fit the kernel's staging buffer
        attn_chunk = attn_chunk or stage_max
        if not 1 <= attn_chunk <= min(256, stage_max):
            raise ValueError(f"attn_chunk must be in [1, {min(256, stage_max)}]")
        self.kv_dtype = kv_dtype or weights.dtype
        self.w_dtype = weights.dtype
        f32 = dict(device=dev, dtype=torch.float32)
        # tiled weights
        self.quant = quant
        if isinstance(weights, TiledModel):  # already tiled (and quantised): use as is
            self.tw = weights.tiles
            self.lm_t = weights.lm
        else:
            self.tw = []
            for lw in weights.layers:
                self.tw.append(dict(qkv=quantize_tiles(pack_tiled(lw.wqkv), quant),
                                    o=quantize_tiles(pack_tiled(lw.wo), quant),
                                    gu=quantize_tiles(pack_gate_up(lw.wgu[:, :f], lw.wgu[:, f:]), quant),
                                    down=quantize_tiles(pack_tiled(lw.wdown), quant)))
            self.lm_t = quantize_tiles(pack_tiled(weights.lm_head), quant) if spec.vocab else None
        self.w_code = (self.tw[0]["qkv"].dtype_code if self.tw else RT.dtype_code(weights.dtype))
        # activations / state
        # residual stream versions: xv[0] the loaded row, xv[2l+1] after layer
        # l's attention, xv[2l+2] after its MLP; x = xv[2L] the step's output
        self.xv = torch.zeros(2 * L + 1, d, **f32)
        self.x = self.xv[2 * L]
        self.x_in = torch.zeros(d, **f32)
        self.ss = torch.zeros(d // TW, **f32)
        self.q = torch.zeros(nq, **f32)
        self.ctx = torch.zeros(nq, **f32)
        self.inter = torch.zeros(f, **f32)
        self.state = torch.zeros(2, device=dev, dtype=torch.int32)
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
        self.attn_chunk = attn_chunk
        # long_context = S > 1: from position `long_from` on, steps run the kernel
        # variant whose attention units each walk S chunks with an online
        # softmax (fewer units and records; slower below ~2 K positions)
        self.super_chunks = int(long_context) if long_context and long_context > 1 else 1
        self.long_from = int(long_from)
        self._pos = 0
        self.last_long = False  # which kernel variant the latest step ran
        self.graph_long = None
        self.nchunks = -(-spec.max_seq // attn_chunk)
        self.taps = StepTaps() if taps else None
        if taps:
            for tap, dim in (("pre_attn", d), ("attn_out", nq), ("pre_mlp", d), ("mlp_inter", f)):
                self.taps.h[tap] = torch.zeros(L, dim, **f32)
            for p, (_, m_in) in spec.proj_shapes().items():
                self.taps.bits[p] = torch.zeros(L, (m_in + 31) // 32, device=dev, dtype=torch.int32)
            self.taps.kept = torch.zeros(L, 7, device=dev, dtype=torch.int64)
        # kept-channel counters accumulated over every step (for algorithmic bytes)
        self.kept = self.taps.kept if taps else (torch.zeros(L, 7, device=dev, dtype=torch.int64) if count_kept else None)
        self.ctas = ctas
        self.prefetch_bytes = max(0, int(prefetch_kb)) * 1024
        self.attn_dbg = torch.zeros(spec.n_kv_heads * self.nchunks, 6, device=dev, dtype=torch.int64) if attn_debug else None
        self._build(thresholds)
        self.graph = None

    # -- plan -----------------------------------------------------------------
    def _build(self, thresholds):
        spec, dev = self.spec, self.device
        d, f, hd, L = spec.d_model, spec.d_ff, spec.head_dim, spec.n_layers
        nq, nkv, KVH = spec.n_q, spec.n_kv, spec.n_kv_heads
        G = spec.n_heads // KVH
        thr = [[None] * 7 for _ in range(L)] if thresholds is None else [list(t) for t in thresholds]
        if len(thr) != L or any(len(t) != 7 for t in thr):
            raise ValueError(f"need {L} per-layer threshold lists of 7 (q,k,v,o,gate,up,down)")
        self.thresholds = thr
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        per = C.lib().teal_step_ctas_per_sm(self.w_code)
        if per < 1:
            raise RuntimeError("teal step kernel cannot be resident on this device")
        self.grid = min(self.ctas, per * sms) if self.ctas > 0 else per * sms
        Gc = self.grid
        nt_qkv, nt_o, nt_gu, nt_dn = (nq + 2 * nkv) // TW, d // TW, f // TH, d // TW
        # counters: 0 load; per layer: attn deps [KVH], ctx ready [KVH], o done, gate/up tiles [nt_gu], down done
        # + x-ready counters of the two residual versions the layer materialises
        per_layer = 2 * KVH + 1 + nt_gu + 1 + 2
        self.ncounters = 1 + per_layer * L

        def cbase(l):
            b = 1 + per_layer * l
            return dict(attn=b, odep=b + KVH, odone=b + 2 * KVH, gu=b + 2 * KVH + 1, down=b + 2 * KVH + 1 + nt_gu,
                        xq=b + 2 * KVH + 2 + nt_gu, xg=b + 2 * KVH + 3 + nt_gu)

        mc = {"qkv": max_contributors(nt_qkv, d, Gc), "o": max_contributors(nt_o, nq, Gc),
              "gu": max_contributors(nt_gu, d, Gc), "down": max_contributors(nt_dn, f, Gc)}
        nts = {"qkv": nt_qkv, "o": nt_o, "gu": nt_gu, "down": nt_dn}
        self.ws = {k: torch.zeros(nts[k] * mc[k] * TW, device=dev) for k in nts}
        self.tk = {k: torch.zeros(max(4096, nts.get(k, 0)), device=dev, dtype=torch.int32)
                   for k in ("qkv", "o", "gu", "down", "lm", "attn")}
        rec = G * hd + 2 * G
        self.ws["attn"] = torch.zeros(KVH * self.nchunks * rec, device=dev)
        # ACC accumulators per layer (int64 fixed point, zeroed by every step's
        # load phase): o and down deltas of the residual [d], gate/up [nt_gu*TW],
        # q|k|v [nt_qkv*TW]
        per_acc = 2 * d + nt_gu * TW + nt_qkv * TW
        self.acc = torch.zeros(L * per_acc, device=dev, dtype=torch.int64)

        def accs(l):
            b = self.acc[l * per_acc:(l + 1) * per_acc]
            return dict(o=b[:d], down=b[d:2 * d], gu=b[2 * d:2 * d + nt_gu * TW], qkv=b[2 * d + nt_gu * TW:])
        self.acc_views = [accs(l) for l in range(L)]
        K_ = CONTRIB

        groups, attns, phases, keep = [], [], [], []
        T, K = self.taps, self.kept

        def dev_bytes(arr):
            t = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(dev)
            keep.append(t)
            return t

        def tiles_tensor(meta):
            return dev_bytes((StepTile * len(meta))(*meta))

        phases.append(StepPhase(PHASE_LOAD, 0, DEP_NONE, 0, 0, 1))
        for l, t in enumerate(thr):
            cb = cbase(l)
            tw = self.tw[l]
            lw = self.w.layers[l]
            kc, vc = self.kcache[l], self.vcache[l]
            A = accs(l)
            if l == 0:  # the loaded row (sum-of-squares partials from the load phase)
                dep_in, qkv_in = (0, Gc), dict(x=self.xv[0], prologue=C.PRO_RMSNORM)
            else:       # x' = previous version + previous layer's down accumulator
                dep_in = (cbase(l - 1)["down"], nt_dn * K_)
                qkv_in = dict(x=self.xv[2 * l - 1], prologue=PRO_RMS_ACC, in_acc=accs(l - 1)["down"],
                              x_out=self.xv[2 * l])
            # --- qkv: RMSNorm(x) -> 3 thresholds -> q (RoPE), k (RoPE) -> cache, v -> cache
            meta, feeds = [], [0] * KVH
            for ti in range(nt_qkv):
                halves = []  # q / k / v segment per 128-column half (n_kv may be a multiple of 128)
                for hh in range(2):
                    c0 = ti * TW + hh * TH
                    c1 = c0 + TH - 1
                    seg = 0 if c0 < nq else (1 if c0 < nq + nkv else 2)
                    if seg == 0:
                        g0, g1 = (c0 // hd) // G, (c1 // hd) // G
                    else:
                        off = nq if seg == 1 else nq + nkv
                        g0, g1 = (c0 - off) // hd, (c1 - off) // hd
                    halves.append((seg, int(c0 in (0, nq, nq + nkv)), g0, g1))
                (sl, fl, a0, a1), (sh, fh, b0, b1) = halves
                g0, g1 = min(a0, b0), max(a1, b1)  # kv groups signalled by this tile
                for gg in range(g0, g1 + 1):
                    feeds[gg] += 1
                meta.append(StepTile(_t32(t[sl]), _t32(t[sh]), sl, sh, fl, fh, cb["attn"] + g0, cb["attn"] + g1))
            groups.append(self._group(tw["qkv"], tiles_tensor(meta), m=d, n=nq + 2 * nkv, maxc=mc["qkv"],
                                      gain=lw.rms_attn, ws="qkv", **qkv_in, acc=A["qkv"],
                                      epilogue=SEPI_QKV, q_out=self.q, k_cache=kc, v_cache=vc,
                                      dbg=(T.h["pre_attn"][l] if T else None,
                                           [T.bits[p][l] for p in ("q", "k", "v")] if T else None,
                                           [K[l, PROJ.index(p)] for p in ("q", "k", "v")] if K is not None else None)))
            phases.append(StepPhase(PHASE_GEMV, len(groups) - 1, DEP_GLOBAL, dep_in[0], dep_in[1], 1))
            # --- attention per (kv group, position chunk)
            tgt = torch.tensor([f_ * K_ for f_ in feeds], dtype=torch.int32, device=dev)
            keep.append(tgt)
            attns.append(StepAttn(self.q.data_ptr(), kc.data_ptr(), vc.data_ptr(), self.ctx.data_ptr(),
                                  self.ws["attn"].data_ptr(), self.tk["attn"].data_ptr(), spec.max_seq,
                                  spec.n_heads, KVH, hd, RT.dtype_code(self.kv_dtype), self.attn_chunk,
                                  self.nchunks, cb["odep"], cb["attn"], tgt.data_ptr(), RT.ptr(self.attn_dbg),
                                  A["qkv"].data_ptr(), RT.ptr(self.rope_cos), RT.ptr(self.rope_sin), nq, nkv,
                                  max(1, self.super_chunks), 0))
            phases.append(StepPhase(PHASE_ATTN, len(attns) - 1, DEP_GLOBAL, 0, Gc, 1))  # step state from the load
            # --- o: rows = context channels, each waits for its kv group's context
            tv = _t32(t[3])
            meta = [StepTile(tv, tv, 0, 0, int(ti == 0), int(ti == 0), cb["odone"], cb["odone"]) for ti in range(nt_o)]
            groups.append(self._group(tw["o"], tiles_tensor(meta), m=nq, n=d, maxc=mc["o"], x=self.ctx,
                                      prologue=C.PRO_PLAIN, ws="o", epilogue=SEPI_RESID, acc=A["o"],
                                      dbg=(T.h["attn_out"][l] if T else None, [T.bits["o"][l]] if T else None,
                                           [K[l, 3]] if K is not None else None)))
            phases.append(StepPhase(PHASE_GEMV, len(groups) - 1, DEP_ROWS, cb["odep"], 1, G * hd))
            # --- gate/up: RMSNorm(x) after every o tile -> SiLU(gate)*up
            tg, tu = _t32(t[4]), _t32(t[5])
            meta = [StepTile(tg, tu, 0, 1, int(ti == 0), int(ti == 0), cb["gu"] + ti, cb["gu"] + ti)
                    for ti in range(nt_gu)]
            groups.append(self._group(tw["gu"], tiles_tensor(meta), m=d, n=f, maxc=mc["gu"], x=self.xv[2 * l],
                                      gain=lw.rms_mlp, prologue=PRO_RMS_ACC, in_acc=A["o"], x_out=self.xv[2 * l + 1],
                                      ws="gu", epilogue=SEPI_SILU, acc=A["gu"],
                                      dbg=(T.h["pre_mlp"][l] if T else None,
                                           [T.bits["gate"][l], T.bits["up"][l]] if T else None,
                                           [K[l, 4], K[l, 5]] if K is not None else None)))
            phases.append(StepPhase(PHASE_GEMV, len(groups) - 1, DEP_GLOBAL, cb["odone"], nt_o * K_, 1))
            # --- down: rows = intermediate channels, each waits for its gate/up tile
            tv = _t32(t[6])
            meta = [StepTile(tv, tv, 0, 0, int(ti == 0), int(ti == 0), cb["down"], cb["down"]) for ti in range(nt_dn)]
            groups.append(self._group(tw["down"], tiles_tensor(meta), m=f, n=d, maxc=mc["down"], x=self.inter,
                                      prologue=PRO_SILU_ACC, in_acc=A["gu"], ws="down", epilogue=SEPI_RESID,
                                      acc=A["down"],
                                      dbg=(T.h["mlp_inter"][l] if T else None, [T.bits["down"][l]] if T else None,
                                           [K[l, 6]] if K is not None else None)))
            phases.append(StepPhase(PHASE_GEMV, len(groups) - 1, DEP_ROWS, cb["gu"], K_, TH))
        if spec.vocab:
            nt_lm = self.lm_t.ntiles
            mc_lm = max_contributors(nt_lm, d, Gc)
            self.ws["lm"] = torch.zeros(nt_lm * mc_lm * TW, device=dev)
            self.tk["lm"] = torch.zeros(max(4096, nt_lm), device=dev, dtype=torch.int32)
            t_lm = _t32(self.lm_threshold)
            meta = [StepTile(t_lm, t_lm, 0, 0, 0, 0, -1, -1) for _ in range(nt_lm)]
            groups.append(self._group(self.lm_t, tiles_tensor(meta), m=d, n=spec.vocab, maxc=mc_lm,
                                      x=self.xv[2 * L - 1], gain=self.w.final_norm, prologue=PRO_RMS_ACC,
                                      in_acc=accs(L - 1)["down"], x_out=self.xv[2 * L], ws="lm",
                                      epilogue=SEPI_LOGITS, y=self.logits))
            phases.append(StepPhase(PHASE_GEMV, len(groups) - 1, DEP_GLOBAL, cbase(L - 1)["down"], nt_dn * K_, 1))
            self.cand_v = torch.zeros(nt_lm, device=dev)
            self.cand_i = torch.zeros(nt_lm, device=dev, dtype=torch.int32)
        else:  # no LM head: materialise the output row x = xv[2L]
            g = StepGroup()
            g.x, g.in_acc, g.x_out, g.m = self.xv[2 * L - 1].data_ptr(), accs(L - 1)["down"].data_ptr(), \
                self.xv[2 * L].data_ptr(), d
            groups.append(g)
            phases.append(StepPhase(PHASE_RESID, len(groups) - 1, DEP_GLOBAL, cbase(L - 1)["down"], nt_dn * K_, 1))
            self.cand_v = torch.zeros(1, device=dev)
            self.cand_i = torch.zeros(1, device=dev, dtype=torch.int32)
        self.lm_done = torch.zeros(1, device=dev, dtype=torch.int32)
        # ACC groups whose equal split crosses tiles (gate/up): weighted ranges
        pen = 10  # groups charged for a second segment; measured: 0 -> 31.7 us, 10 -> 29.5 us gate/up
        self.range_tables = {}
        for gi, g in enumerate(groups):
            if not g.acc or g.m <= 0:
                continue
            key = (g.ntiles, g.m)
            if key not in self.range_tables:
                rs = weighted_ranges(g.ntiles, g.m, Gc, pen)
                self.range_tables[key] = None if rs is None else torch.tensor(rs, dtype=torch.int32, device=dev)
            tab = self.range_tables[key]
            if tab is not None:
                g.ranges, g.nranges = tab.data_ptr(), tab.shape[0]

        def ctas_of(g):  # CTAs taking part in a GEMV group (each writes one x_out share)
            return g.nranges if g.ranges else participants(g.ntiles, g.ntiles * (-(-g.m // 32)), Gc)

        # x-ready counters: an RMS_ACC phase stages the previous residual version
        # (complete once every CTA of its producer wrote its share) before waiting
        # for its own accumulator.  Groups per layer: qkv, o, gate/up, down; then LM.
        for l in range(L):
            gq, gg = groups[4 * l], groups[4 * l + 2]
            if l > 0:
                gq.xsig = cbase(l)["xq"]
                gq.xwait, gq.xwait_target = cbase(l - 1)["xg"], ctas_of(groups[4 * (l - 1) + 2])
            gg.xsig = cbase(l)["xg"]
            if l == 0:
                gg.xwait, gg.xwait_target = 0, Gc  # xv[0]: the load phase
            else:
                gg.xwait, gg.xwait_target = cbase(l)["xq"], ctas_of(gq)
        if spec.vocab:
            gl = groups[4 * L]
            gl.xwait, gl.xwait_target = cbase(L - 1)["xg"], ctas_of(groups[4 * (L - 1) + 2])
        # attention units on the CTAs the qkv phase leaves idle (when they fit)
        for l in range(L):
            pq = ctas_of(groups[4 * l])
            attns[l].home = pq if Gc - pq >= KVH else 0
        self._keep = keep
        self._groups_host = (StepGroup * len(groups))(*groups)
        self._phases_host = (StepPhase * len(phases))(*phases)
        self._groups = dev_bytes(self._groups_host)
        self._attns = dev_bytes((StepAttn * len(attns))(*attns))
        self._phases = dev_bytes(self._phases_host)
        self.nphases = len(phases)
        self.counters = torch.zeros(self.ncounters * 32, device=dev, dtype=torch.int32)
        self.ctrl = torch.zeros(4, device=dev, dtype=torch.int32)
        self.timeline = None
        p = StepPlan()
        p.groups, p.attns, p.phases = self._groups.data_ptr(), self._attns.data_ptr(), self._phases.data_ptr()
        p.counters, p.ctrl = self.counters.data_ptr(), self.ctrl.data_ptr()
        if spec.vocab:
            p.emb, p.emb_dtype = self.w.embedding.data_ptr(), RT.dtype_code(self.w.embedding.dtype)
        p.acc_zero, p.acc_zero_n = self.acc.data_ptr(), self.acc.numel()
        p.x_in, p.token, p.x, p.ss, p.state = (self.x_in.data_ptr(), self.token.data_ptr(), self.xv[0].data_ptr(),
                                               self.ss.data_ptr(), self.state.data_ptr())
        p.cand_v, p.cand_i, p.token_out, p.lm_done = (self.cand_v.data_ptr(), self.cand_i.data_ptr(),
                                                      self.token.data_ptr(), self.lm_done.data_ptr())
        p.nphases, p.ncounters, p.d = self.nphases, self.ncounters, d
        p.w_dtype, p.ctas = self.w_code, self.grid
        p.long_ctx = 0  # chosen per launch (_use_long)
        p.prefetch_bytes = self.prefetch_bytes
        p.max_seq = spec.max_seq
        self.plan = p

    def _upload_plan(self) -> None:
        """Re-upload the (host-edited) group and phase tables."""
        for t, h in ((self._groups, self._groups_host), (self._phases, self._phases_host)):
            t.copy_(torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8))

    def enable_timeline(self) -> torch.Tensor:
        """Debug: record %globaltimer at entry/exit of every phase of every CTA
        ([grid, nphases, 8] int64, overwritten by each launch): 0 start, 1 end;
        GEMV phases also 2 prologue done (first segment's rows ready), 3/5
        first/second segment streamed, 4 first segment finished, 6 global
        dependency met, 7 RMS prologue done (RMS_ACC phases).  Attention
        units (attn_debug): 0 entry, 1 q/k/v tiles ready, 2 q staged,
        3 scores, 4 context written, 5 signalled."""
        self.timeline = torch.zeros(self.grid, self.nphases, 8, device=self.device, dtype=torch.int64)
        self.plan.timeline = self.timeline.data_ptr()
        return self.timeline

    def _group(self, wt, tiles, m, n, maxc, x, prologue, ws, epilogue, gain=None, q_out=None, k_cache=None,
               v_cache=None, y=None, dbg=None, acc=None, in_acc=None, x_out=None):
        spec = self.spec
        g = StepGroup()
        g.w, g.tiles, g.x = wt.data.data_ptr(), tiles.data_ptr(), x.data_ptr()
        g.col_scale, g.gscale, g.group = RT.ptr(wt.col_scale), RT.ptr(wt.gscale), wt.group
        g.gain = gain.data_ptr() if gain is not None else None
        g.ss = self.ss.data_ptr()
        g.partials, g.tickets = self.ws[ws].data_ptr(), self.tk[ws].data_ptr()
        g.y = y.data_ptr() if y is not None else None
        g.resid, g.ss_out, g.inter = self.x.data_ptr(), self.ss.data_ptr(), self.inter.data_ptr()
        g.q_out = q_out.data_ptr() if q_out is not None else None
        g.k_cache = k_cache.data_ptr() if k_cache is not None else None
        g.v_cache = v_cache.data_ptr() if v_cache is not None else None
        g.rope_cos, g.rope_sin = RT.ptr(self.rope_cos), RT.ptr(self.rope_sin)
        if dbg is not None:
            h, bits, kept = dbg
            g.dbg_h = RT.ptr(h) if h is not None else None
            for i, b in enumerate(bits or []):
                g.dbg_bits[i] = b.data_ptr()
            for i, k in enumerate(kept or []):
                g.kept[i] = k.data_ptr()
        g.max_seq, g.m, g.n, g.ntiles, g.maxc = spec.max_seq, m, n, wt.ntiles, maxc
        g.prologue, g.nss, g.eps, g.epilogue = prologue, spec.d_model // TW, spec.norm_eps, epilogue
        g.nq, g.nkv, g.head_dim, g.kv_dtype = spec.n_q, spec.n_kv, spec.head_dim, RT.dtype_code(self.kv_dtype)
        g.w_dtype = wt.dtype_code
        g.acc, g.in_acc, g.x_out = RT.ptr(acc), RT.ptr(in_acc), RT.ptr(x_out)
        g.xsig, g.xwait, g.xwait_target = -1, -1, 0
        return g

    # -- step -----------------------------------------------------------------
    def reset(self, start_pos: int = 0) -> None:
        self.state.copy_(torch.tensor([start_pos - 1, start_pos], dtype=torch.int32))
        self._pos = start_pos
        if start_pos == 0:
            self.kcache.zero_()
            self.vcache.zero_()

    def launches_per_step(self) -> int:
        return 1

    def algorithmic_bytes(self, kept=None, steps: int = 1, positions: int = 0) -> float:
        """Bytes a step must touch: kept rows x n x bw for the
        seven projections of every layer (from `kept` [L,7] channel counts,
        e.g. self.kept accumulated over `steps` steps), + per step m x 4
        activation reads and n x 4 output writes per projection and the dense
        LM head, + K and V reads of `positions` attended positions (summed
        over the steps)."""
        spec = self.spec
        bw = {C.TEAL_F32: 4, C.TEAL_BF16: 2, C.TEAL_I8: 1, C.TEAL_I4: 0.5}[self.w_code]
        shapes = spec.proj_shapes()
        kept = (self.kept if kept is None else kept).double().cpu()
        total = 0.0
        for i, p in enumerate(PROJ):
            n, m = shapes[p]
            total += float(kept[:, i].sum()) * n * bw
        steps_proj_io = sum((m * 4 + n * 4) for (n, m) in shapes.values()) * spec.n_layers
        total += steps * steps_proj_io
        if spec.vocab:
            total += steps * (spec.d_model * spec.vocab * bw + spec.d_model * 4 + spec.vocab * 4)
        kvb = torch.empty(0, dtype=self.kv_dtype).element_size()
        total += positions * spec.n_layers * 2 * spec.n_kv * kvb
        return total

    def _use_long(self) -> bool:
        return self.super_chunks > 1 and self._pos >= self.long_from

    def _check_pos(self) -> None:
        if self._pos >= self.spec.max_seq:
            raise ValueError(f"decode position {self._pos} would exceed max_seq {self.spec.max_seq} "
                             f"(the KV cache holds positions [0, {self.spec.max_seq}))")

    def _launch(self, stream_h: int, from_token: bool, long_ctx: bool | None = None) -> None:
        p = self.plan
        p.long_ctx = int(self._use_long() if long_ctx is None else long_ctx)
        if from_token:
            p.emb = self.w.embedding.data_ptr()
        else:
            p.emb = None
        C.check(C.lib().teal_step_launch(ctypes.byref(p), stream_h))

    def step_hidden(self, x_row) -> torch.Tensor:
        if isinstance(x_row, torch.Tensor):
            self.x_in.copy_(x_row.reshape(-1), non_blocking=True)
        else:
            self.x_in.copy_(torch.from_numpy(np.ascontiguousarray(x_row, dtype=np.float32)), non_blocking=True)
        self._check_pos()
        self._launch(RT.stream_handle(), from_token=False)
        self.last_long = bool(self.plan.long_ctx)
        self._pos += 1
        return self.x

    def step_token(self) -> torch.Tensor:
        if self.graph is not None:
            self.replay()
        else:
            self._check_pos()
            self._launch(RT.stream_handle(), from_token=True)
            self.last_long = bool(self.plan.long_ctx)
            self._pos += 1
        return self.token

    def step_token_host(self, tok_in: torch.Tensor, tok_out: torch.Tensor) -> None:
        self.token.copy_(tok_in, non_blocking=True)
        self.step_token()
        tok_out.copy_(self.token, non_blocking=True)

    def capture(self, from_token: bool = True) -> torch.cuda.CUDAGraph:
        """One CUDA graph of the step launch (and, with long_context, a second
        one of the long-context variant; replay() picks by position)."""
        graphs = []
        for lc in ((False, True) if self.super_chunks > 1 else (False,)):
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._launch(s.cuda_stream, from_token, long_ctx=lc)
            torch.cuda.current_stream().wait_stream(s)
            graphs.append(g)
        self.graph = graphs[0]
        self.graph_long = graphs[1] if len(graphs) > 1 else None
        return self.graph

    def replay(self) -> None:
        self._check_pos()
        self.last_long = self._use_long() and self.graph_long is not None
        (self.graph_long if self.last_long else self.graph).replay()
        self._pos += 1
