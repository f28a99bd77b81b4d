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
    if not (t >= 0.0 or t == float("-inf")):
        raise ValueError(f"threshold must be non-negative (or -inf: dense), got {t}")
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


# ---- the prompt pass of a decoder ----------------------------------------------

PROJ = ("q", "k", "v", "o", "gate", "up", "down")


def _thr(t) -> float:
    return float("-inf") if t is None or t == float("-inf") else float(t)


class PrefillResult:
    """x: final residual rows [T, d]; logits: [T or 1, vocab] (None without an
    LM head); next_token: argmax of the last position (None without an LM
    head); kept: per-layer kept counts [L, 7] over the thresholded rows."""

    def __init__(self, x, logits, next_token, kept):
        self.x, self.logits, self.next_token, self.kept = x, logits, next_token, kept


class SparsePrefill:
    """TEAL's prompt pass for a ``DecoderWeights`` model (bf16 weights):
    every projection is ``masked_gemm`` (gate + tcgen05 GEMM) with the
    decoder's per-layer thresholds (q, k, v, o, gate, up, down) applied to
    prompt rows >= ``sparse_from`` — by default the second half of the
    prompt, the paper's recipe for log-likelihood evaluation (PAPER.md:269-270,
    :444) — and the first rows dense (attention sinks).  RMSNorm, SiLU*up and
    the LM-head argmax are this package's batch kernels; RoPE + K/V cache
    writes are ``teal_prefill_rope_cache``; causal attention over the cached
    K/V is torch's scaled_dot_product_attention (library attention, as
    cuBLAS is a library GEMM).

    With ``decoder`` (a SparseDecoder / StepDecoder over the same weights),
    the prompt's K/V land in that decoder's cache and the decoder continues
    at position T from the prompt's argmax token: prefill -> decode.
    """

    def __init__(self, weights, thresholds=None, terms: int = 2, kv_dtype=None, attention: str = "fp32"):
        W = weights
        if W.dtype != torch.bfloat16:
            raise ValueError("the prefill GEMM takes bf16 weights")
        if attention not in ("fp32", "bf16"):
            raise ValueError(f"attention must be 'fp32' or 'bf16', got {attention!r}")
        self.w, self.spec, self.terms, self.attention = W, W.spec, terms, attention
        L = self.spec.n_layers
        thr = [[None] * 7 for _ in range(L)] if thresholds is None else [list(t) for t in thresholds]
        if len(thr) != L or any(len(t) != 7 for t in thr):
            raise ValueError(f"need {L} per-layer threshold lists of 7 (q,k,v,o,gate,up,down)")
        self.thresholds = [[_thr(x) for x in t] for t in thr]
        self.kv_dtype = kv_dtype or W.dtype
        spec = self.spec
        hd = spec.head_dim
        if spec.rope_theta is not None:
            inv = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
            ang = torch.arange(spec.max_seq, dtype=torch.float64)[:, None] * inv[None, :]
            dev = W.layers[0].wqkv.device
            self.rope_cos = torch.cos(ang).float().to(dev).contiguous()
            self.rope_sin = torch.sin(ang).float().to(dev).contiguous()
        else:
            self.rope_cos = self.rope_sin = None

    def _attend(self, q, kc, vc, T, pos0=0):
        """Causal attention of the prompt rows (positions pos0 .. pos0+T-1) over
        the cached (kv-dtype) keys and values of positions 0 .. pos0+T-1: fp32
        (fused memory-efficient kernel; the decode engine's arithmetic: fp32 q,
        fp32 softmax) or bf16 (flash kernel, q rounded)."""
        from torch.nn.attention import SDPBackend, sdpa_kernel
        spec = self.spec
        G, hd = spec.n_heads // spec.n_kv_heads, spec.head_dim
        S = pos0 + T
        qh = q.view(T, spec.n_heads, hd).transpose(0, 1).unsqueeze(0)
        mask = None
        if pos0:  # key j visible to row t iff j <= pos0 + t
            mask = (torch.arange(S, device=q.device)[None, :] <= (pos0 + torch.arange(T, device=q.device))[:, None])
        kw = dict(is_causal=True) if mask is None else dict(attn_mask=mask)
        if self.attention == "fp32":
            kk = kc[:, :S].float().repeat_interleave(G, dim=0).unsqueeze(0)
            vv = vc[:, :S].float().repeat_interleave(G, dim=0).unsqueeze(0)
            with sdpa_kernel([SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH]):
                ctx = torch.nn.functional.scaled_dot_product_attention(qh, kk, vv, **kw)
        else:
            kk = kc[:, :S].to(torch.bfloat16).repeat_interleave(G, dim=0).unsqueeze(0)
            vv = vc[:, :S].to(torch.bfloat16).repeat_interleave(G, dim=0).unsqueeze(0)
            with sdpa_kernel([SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH]):
                ctx = torch.nn.functional.scaled_dot_product_attention(qh.to(torch.bfloat16), kk, vv, **kw)
        return ctx[0].transpose(0, 1).reshape(T, spec.n_q).float().contiguous()

    # one projection: y (+)= g(x) @ w[:, c0:c0+n]
    def _proj(self, x, w, t, sf, out=None, accumulate=False, kept=None):
        if t == float("-inf"):
            hi, lo = gate(x, float("-inf"), 0, self.terms)
        else:
            hi, lo = gate(x, t, sf, self.terms, kept)
        return gemm(w, hi, lo, out=out, accumulate=accumulate)

    def forward(self, tokens=None, hidden=None, sparse_from: int | None = None, decoder=None, logits: str = "last",
                kv_cache=None, start_pos: int = 0) -> PrefillResult:
        """Run the prompt (``tokens`` [T] int, or ``hidden`` rows [T, d]).
        ``sparse_from`` default T // 2 (rows of THIS call).  ``logits``:
        "last", "all" or "none".  ``kv_cache``: (k, v) tensors [L, KVH,
        max_seq, hd] to fill (default: the decoder's, else fresh ones).
        ``start_pos`` > 0: chunked prefill — the rows are positions start_pos ..
        start_pos+T-1 and attend to the cache's earlier positions (filled by a
        previous call on the same cache)."""
        spec, W = self.spec, self.w
        d, f, nq, nkv, hd = spec.d_model, spec.d_ff, spec.n_q, spec.n_kv, spec.head_dim
        dev = W.layers[0].wqkv.device
        L = C.lib()
        sh = RT.stream_handle()
        if (tokens is None) == (hidden is None):
            raise ValueError("pass exactly one of tokens / hidden")
        if tokens is not None:
            if W.embedding is None:
                raise ValueError("this model has no embedding: pass hidden rows")
            tok = torch.as_tensor(tokens, dtype=torch.int32).reshape(-1).to(dev).contiguous()
            T = tok.numel()
            x = torch.empty(T, d, device=dev)
            C.check(L.teal_batch_embed(W.embedding.data_ptr(), RT.dtype_code(W.embedding.dtype), tok.data_ptr(), T, d,
                                       x.data_ptr(), None, sh))
        else:
            h0 = hidden if isinstance(hidden, torch.Tensor) else torch.from_numpy(
                __import__("numpy").ascontiguousarray(hidden, dtype="float32"))
            x = h0.to(dev, torch.float32).reshape(-1, d).clone()
            T = x.shape[0]
        pos0 = int(start_pos)
        if T < 1 or pos0 < 0 or pos0 + T > spec.max_seq:
            raise ValueError(f"prompt positions [{pos0}, {pos0 + T}) outside [0, max_seq={spec.max_seq})")
        sf = T // 2 if sparse_from is None else int(sparse_from)
        if sf < 0:
            raise ValueError(f"sparse_from must be >= 0, got {sf}")
        if kv_cache is not None:
            kc_all, vc_all = kv_cache
        elif decoder is not None:
            kc_all, vc_all = decoder.kcache, decoder.vcache
        else:
            if pos0:
                raise ValueError("start_pos > 0 continues a cache: pass kv_cache or decoder")
            kc_all = torch.zeros(spec.n_layers, spec.n_kv_heads, spec.max_seq, hd, device=dev, dtype=self.kv_dtype)
            vc_all = torch.zeros_like(kc_all)
        kvc = RT.dtype_code(kc_all.dtype)
        kept = torch.zeros(spec.n_layers, 7, dtype=torch.int64, device=dev)
        h = torch.empty(T, d, device=dev)
        q = torch.empty(T, nq, device=dev)
        k = torch.empty(T, nkv, device=dev)
        v = torch.empty(T, nkv, device=dev)
        g = torch.empty(T, f, device=dev)
        u = torch.empty(T, f, device=dev)
        inter = torch.empty(T, f, device=dev)
        for l, lw in enumerate(W.layers):
            t = self.thresholds[l]
            C.check(L.teal_batch_rmsnorm(x.data_ptr(), None, lw.rms_attn.data_ptr(), spec.norm_eps, T, d,
                                         h.data_ptr(), sh))
            self._proj(h, lw.wqkv[:, :nq], t[0], sf, out=q, kept=kept[l, 0])
            self._proj(h, lw.wqkv[:, nq:nq + nkv], t[1], sf, out=k, kept=kept[l, 1])
            self._proj(h, lw.wqkv[:, nq + nkv:], t[2], sf, out=v, kept=kept[l, 2])
            kc, vc = kc_all[l], vc_all[l]
            C.check(L.teal_prefill_rope_cache(q.data_ptr(), nq, k.data_ptr(), nkv, v.data_ptr(), nkv, T,
                                              spec.n_heads, spec.n_kv_heads, hd, pos0, RT.ptr(self.rope_cos),
                                              RT.ptr(self.rope_sin), kc.data_ptr(), vc.data_ptr(), kvc,
                                              spec.max_seq, sh))
            ctx = self._attend(q, kc, vc, T, pos0)
            self._proj(ctx, lw.wo, t[3], sf, out=x, accumulate=True, kept=kept[l, 3])
            C.check(L.teal_batch_rmsnorm(x.data_ptr(), None, lw.rms_mlp.data_ptr(), spec.norm_eps, T, d,
                                         h.data_ptr(), sh))
            self._proj(h, lw.wgu[:, :f], t[4], sf, out=g, kept=kept[l, 4])
            self._proj(h, lw.wgu[:, f:], t[5], sf, out=u, kept=kept[l, 5])
            C.check(L.teal_batch_silu_mul(g.data_ptr(), u.data_ptr(), T * f, inter.data_ptr(), sh))
            self._proj(inter, lw.wdown, t[6], sf, out=x, accumulate=True, kept=kept[l, 6])
        lg = nxt = None
        if W.lm_head is not None and logits != "none":
            rows = x if logits == "all" else x[T - 1:]
            hn = torch.empty_like(rows)
            C.check(L.teal_batch_rmsnorm(rows.data_ptr(), None, W.final_norm.data_ptr(), spec.norm_eps, rows.shape[0],
                                         d, hn.data_ptr(), sh))
            lg = self._proj(hn, W.lm_head, float("-inf"), 0)
            toks = torch.empty(lg.shape[0], dtype=torch.int32, device=dev)
            C.check(L.teal_batch_argmax(lg.data_ptr(), lg.shape[0], lg.shape[1], toks.data_ptr(), sh))
            nxt = toks[-1:]
        if decoder is not None:
            decoder.reset(pos0 + T)
            if nxt is not None:
                decoder.token.copy_(nxt)
        return PrefillResult(x, lg, nxt, kept)

    def forward_batch(self, prompts, batch_decoder, sparse_from: int | None = None) -> list:
        """Prefill the B equal-length prompts of a small-batch decode: prompt b
        fills sequence b's slice of ``batch_decoder``'s cache (per-token masks,
        as in the prompt pass), then the batch decoder continues in lockstep at
        position T from each prompt's argmax token.  Returns the B results."""
        B = batch_decoder.B
        if len(prompts) != B or len({len(p_) for p_ in prompts}) != 1:
            raise ValueError(f"need {B} prompts of one length (the batch decodes in lockstep)")
        out = []
        for b, pr in enumerate(prompts):
            r = self.forward(tokens=pr, sparse_from=sparse_from,
                             kv_cache=(batch_decoder.kcache[:, b], batch_decoder.vcache[:, b]))
            out.append(r)
        T = len(prompts[0])
        batch_decoder.reset(T)
        if out[0].next_token is not None:
            batch_decoder.tokens.copy_(torch.cat([r.next_token for r in out]))
        return out


def generate(weights, thresholds, prompt, max_new_tokens: int, sparse_from: int | None = None, kv_dtype=None,
             prefill_thresholds="same") -> list:
    """Greedy generation: the prompt through ``SparsePrefill`` (``sparse_from``
    default: the second half; ``prefill_thresholds`` "same"
    or None for a dense prompt pass — the paper does not sparsify prefill on
    generation tasks), then ``max_new_tokens`` steps of the persistent decode
    engine (one CUDA-graph replay per token) continuing the same KV cache.
    Returns the generated token ids."""
    from . import engine as E
    dec = E.StepDecoder(weights, thresholds, kv_dtype=kv_dtype)
    dec.reset()
    pthr = thresholds if prefill_thresholds == "same" else prefill_thresholds
    r = SparsePrefill(weights, pthr, kv_dtype=dec.kv_dtype).forward(tokens=prompt, sparse_from=sparse_from,
                                                                   decoder=dec)
    out = [int(r.next_token)]
    if max_new_tokens > 1:
        dec.capture()
        for _ in range(max_new_tokens - 1):
            dec.step_token()
            out.append(int(dec.token))
    return out[:max_new_tokens]


def log_likelihood(weights, thresholds, tokens, sparse_from: int | None = None, kv_dtype=None):
    """Per-token log-likelihood of ``tokens`` under the sparse prompt pass —
    the evaluation TEAL sparsifies prefill for (the second
    half of the sequence thresholded by default, log-likelihood tasks and
    perplexity).  Returns (logp [T-1] fp32 on the device: log p(token[t+1] |
    tokens[..t]), perplexity = exp(-mean logp))."""
    tok = torch.as_tensor(tokens, dtype=torch.int64).reshape(-1)
    r = SparsePrefill(weights, thresholds, kv_dtype=kv_dtype).forward(tokens=tok, sparse_from=sparse_from,
                                                                     logits="all")
    lp = torch.log_softmax(r.logits[:-1].double(), dim=-1)
    tgt = tok[1:].to(lp.device)
    logp = lp.gather(1, tgt[:, None])[:, 0].float()
    return logp, float(torch.exp(-logp.double().mean()))
