"""GPU parity at the EXACT benchmarked configuration (BASELINE config 3/4).

The headline number runs ``step_kernel`` on Llama-3-8B shapes: d = 4096, 32
layers, 296 CTAs, qkv F = 3,072 (tile, 32-row group) units, gate/up on
weighted ranges, the 501-tile LM head — a regime the toy-shape tests never
reach (multi-group ranges, two-tile ranges, many-contributor int64
accumulation).  Here the bench's own model (``decode.random_weights(LLAMA3_8B,
bf16, seed=0)``) and calibration (``calibrate_histograms`` on 16 tokens,
``uniform_thresholds`` at 40 % and 50 %) drive ``engine.StepDecoder`` with
the kernel's debug taps on, and every step is checked:

* every layer x 7 projections: the keep bitmask the kernel wrote equals the
  oracle's ``keep_mask(h, t)`` (pkg/src/actsparse/sparsifier.py:120-125,
  kernel.py:36-38 predicate) of the kernel's own tap vector h, bit for bit,
  and the kept count equals its popcount;
* teacher-forced, layer by layer (LayerCheck): every tap vector, new K/V
  cache row, attention context, residual version and the logits within
  rel 1e-3 (north-star bar 1e-2; bf16 weights, fp32 accumulate) of a plain
  torch fp32 restatement of model.py:158-198 (GQA + RoPE + KV cache) fed the
  engine's own inputs to that operation;
* the greedy token equals the argmax of the reference logits (unless their
  top-2 gap is below numerical noise).

int8 / int4 rows: the same at 50 %, the reference multiplying with the
dequantised weights the kernel streams (parity unpinned).
Llama-3-70B tensor parallel: one TP-8 rank group at real shard shapes
(d = 8192, 8 q heads + 1 kv head, d_ff 3584 per rank; 2 layers) with the
exchange inside the kernel (tp.FusedTPGroup: all 8 ranks' launches on this
GPU, each adding into the others' accumulators) against the unsharded engine.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import actsparse_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

STEPS = 8
TAPS = {"q": "pre_attn", "k": "pre_attn", "v": "pre_attn", "o": "attn_out",
        "gate": "pre_mlp", "up": "pre_mlp", "down": "mlp_inter"}


@pytest.fixture(scope="module")
def llama8b():
    from paper_2408_14690_b200 import decode as D
    W = D.random_weights(D.LLAMA3_8B, torch.bfloat16, seed=0)          # bench.py: seed = rank
    hists = D.calibrate_histograms(W, n_tokens=16, seed=1000)           # bench.py calibration
    thr = {s: D.uniform_thresholds(hists, D.LLAMA3_8B.n_layers, s) for s in (0.4, 0.5)}
    return D, W, thr


class LayerCheck:
    """Teacher-forced fp32 torch restatement of one decode step, layer by
    layer, over the engine's own (tiled, possibly quantised) weights: every
    projection's input is the engine's tap vector and every layer's input its
    residual version, so each comparison is one operation deep.  (A
    free-running fp32 decode is not a usable oracle at 32 layers of random
    weights: a mask decision on an ulp tie perturbs the next layer's h, which
    flips more decisions, and the two runs drift apart — measured here: dense
    1.7e-3, 50 % 0.39 relative at layer 32 after one token.)"""

    def __init__(self, dec):
        self.dec, self.spec = dec, dec.spec
        hd = self.spec.head_dim
        self.inv = 1.0 / (self.spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64, device=dec.device) / hd))

    def _w(self, l):
        from paper_2408_14690_b200 import engine as E
        sp, tw = self.spec, self.dec.tw[l]
        return (E.untile(tw["qkv"].dequantize(), sp.n_q + 2 * sp.n_kv), E.untile(tw["o"].dequantize(), sp.d_model),
                E.untile_gate_up(tw["gu"].dequantize(), sp.d_ff), E.untile(tw["down"].dequantize(), sp.d_model))

    def _rope(self, x, pos):
        hd = self.spec.head_dim
        ang = pos * self.inv
        c, s = torch.cos(ang).float(), torch.sin(ang).float()
        x1, x2 = x[:, : hd // 2], x[:, hd // 2:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=1)

    def check_step(self, tok, thr, pos):
        """Returns {quantity: worst relative error over layers}."""
        from paper_2408_14690_b200 import engine as E
        sp, dec = self.spec, self.dec
        H, KVH, hd, nq, nkv, f = sp.n_heads, sp.n_kv_heads, sp.head_dim, sp.n_q, sp.n_kv, sp.d_ff
        G = H // KVH
        T = dec.taps.h
        worst = {}

        def rec(k, got, want):
            worst[k] = max(worst.get(k, 0.0), rel_err(got.cpu().numpy(), want.cpu().numpy()))

        def spz(a, t):
            return a if t is None else torch.where(a.abs() <= float(np.float32(t)), torch.zeros_like(a), a)

        def norm(x, w):
            return x / torch.sqrt((x * x).mean() + sp.norm_eps) * w

        rec("x_load", dec.xv[0], dec.w.embedding[tok].float())
        for l in range(sp.n_layers):
            t = thr[l]
            wqkv, wo, wgu, wdn = self._w(l)
            lw = dec.w.layers[l]
            rec("h_pre_attn", T["pre_attn"][l], norm(dec.xv[2 * l], lw.rms_attn))
            h = T["pre_attn"][l]
            q = self._rope((spz(h, t[0]) @ wqkv[:, :nq]).view(H, hd), pos)
            k = self._rope((spz(h, t[1]) @ wqkv[:, nq:nq + nkv]).view(KVH, hd), pos)
            v = (spz(h, t[2]) @ wqkv[:, nq + nkv:]).view(KVH, hd)
            rec("k_row", dec.kcache[l][:, pos].float(), k.to(dec.kv_dtype).float())
            rec("v_row", dec.vcache[l][:, pos].float(), v.to(dec.kv_dtype).float())
            Ks, Vs = dec.kcache[l][:, :pos + 1].float(), dec.vcache[l][:, :pos + 1].float()
            ctx = torch.cat([torch.softmax((Ks[hh // G] @ q[hh]) / math.sqrt(hd), 0) @ Vs[hh // G] for hh in range(H)])
            rec("ctx", T["attn_out"][l], ctx)
            rec("x_attn", dec.xv[2 * l + 1], dec.xv[2 * l] + spz(T["attn_out"][l], t[3]) @ wo)
            rec("h_pre_mlp", T["pre_mlp"][l], norm(dec.xv[2 * l + 1], lw.rms_mlp))
            hm = T["pre_mlp"][l]
            gate, up = spz(hm, t[4]) @ wgu[:, :f], spz(hm, t[5]) @ wgu[:, f:]
            rec("inter", T["mlp_inter"][l], gate / (1 + torch.exp(-gate)) * up)
            rec("x_mlp", dec.xv[2 * l + 2], dec.xv[2 * l + 1] + spz(T["mlp_inter"][l], t[6]) @ wdn)
            del wqkv, wo, wgu, wdn
        lg = norm(dec.xv[2 * sp.n_layers], dec.w.final_norm) @ E.untile(dec.lm_t.dequantize(), sp.vocab)
        rec("logits", dec.logits, lg)
        top2 = torch.topk(lg, 2).values
        if float(top2[0] - top2[1]) > 1e-4 * float(lg.abs().max()):
            assert int(dec.token.item()) == int(torch.argmax(lg).item()), pos
        return worst


def _check_masks(dec, thr, step):
    from paper_2408_14690_b200 import decode as D
    L = dec.spec.n_layers
    kept = dec.taps.kept.cpu().numpy()
    for l in range(L):
        taps = {tap: dec.taps.h[tap][l].cpu().numpy() for tap in set(TAPS.values())}
        for i, p in enumerate(D.PROJ):
            keep = R.keep_mask(taps[TAPS[p]], thr[l][i])
            got = dec.taps.bits[p][l].cpu().numpy().view(np.uint32)
            want = R.pack_bits(keep)
            if not np.array_equal(got, want):
                n = int(np.unpackbits((got ^ want).view(np.uint8)).sum())
                raise AssertionError(f"step {step} layer {l} {p}: {n} mask bits differ from keep_mask(h, t)")
            assert int(kept[l, i]) == int(keep.sum()), (step, l, p)


# every quantity is one fp32 operation deep from the engine's own inputs:
# measured ~1e-7 (fp32 weights) to ~1e-5; the north-star bar is 1e-2
TOL = 1e-3


def _run(dec, thr, tokens):
    chk = LayerCheck(dec)
    dec.reset()
    worst = {}
    for i, tok in enumerate(tokens):
        dec.taps.kept.zero_()
        dec.token.fill_(tok)
        dec.step_token()
        torch.cuda.synchronize()
        _check_masks(dec, thr, i)
        for k, v in chk.check_step(tok, thr, i).items():
            worst[k] = max(worst.get(k, 0.0), v)
    bad = {k: v for k, v in worst.items() if not v < TOL}
    assert not bad, bad
    return worst


def _tokens(n=STEPS, seed=77, vocab=128256):
    g = np.random.default_rng(seed)
    return [int(t) for t in g.integers(0, vocab, n)]


@pytest.mark.parametrize("level", [0.5, 0.4])
def test_llama3_8b_bf16_bench_config(llama8b, level):
    D, W, thr = llama8b
    from paper_2408_14690_b200 import engine as E
    dec = E.StepDecoder(W, thr[level], taps=True)
    assert dec.grid == 2 * torch.cuda.get_device_properties(0).multi_processor_count  # the bench's 296 CTAs
    worst = _run(dec, thr[level], _tokens())
    print(f"8B bf16 @{level}: worst rel", {k: f"{v:.1e}" for k, v in worst.items()})
    del dec
    torch.cuda.empty_cache()


@pytest.mark.parametrize("quant", ["int8", "int4"])
def test_llama3_8b_quantized_bench_config(llama8b, quant):
    D, W, thr = llama8b
    from paper_2408_14690_b200 import engine as E
    dec = E.StepDecoder(W, thr[0.5], taps=True, quant=quant)
    worst = _run(dec, thr[0.5], _tokens(seed=78))
    print(f"8B {quant} @0.5: worst rel", {k: f"{v:.1e}" for k, v in worst.items()})
    del dec
    torch.cuda.empty_cache()


def test_llama3_8b_graph_replay_equals_eager(llama8b):
    # the bench times CUDA-graph replays: same tokens, bit-identical residuals
    D, W, thr = llama8b
    from paper_2408_14690_b200 import engine as E
    dec = E.StepDecoder(W, thr[0.5])
    dec.reset()
    toks = _tokens(6, seed=79)
    eager = []
    for t in toks:
        dec.token.fill_(t)
        dec.step_token()
        eager.append(dec.x.clone())
    dec.reset()
    dec.capture()
    dec.reset()
    for t, e in zip(toks, eager):
        dec.token.fill_(t)
        dec.replay()
        torch.cuda.synchronize()
        assert torch.equal(dec.x, e)
    assert int(dec.counters.abs().sum()) == 0
    del dec
    torch.cuda.empty_cache()


def test_llama3_70b_tp8_shard_fused_exchange():
    # config 4 at real TP-8 shard shapes: every rank's launch on this GPU, the
    # row-parallel partials added into every rank's accumulators in-kernel
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200 import tp
    spec = D.DecoderSpec(8192, 64, 8, 28672, 2, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    ls = tp.shard_spec(spec, 8)
    assert (ls.d_model, ls.n_q, ls.n_kv, ls.d_ff) == (8192, 1024, 128, 3584)
    W = D.random_weights(spec, torch.bfloat16, seed=70)
    hists = D.calibrate_histograms(W, n_tokens=4, seed=71, engine="step")
    thr = D.uniform_thresholds(hists, spec.n_layers, 0.5)
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    grp = tp.FusedTPGroup([tp.shard_weights(W, r, 8) for r in range(8)], thr, kv_dtype=torch.float32)
    ref.reset()
    grp.reset()
    worst = 0.0
    for tok in _tokens(6, seed=72):
        ref.token.fill_(tok)
        ref.step_token()
        grp.set_token(tok)
        grp.step()
        torch.cuda.synchronize()
        x0 = grp.decs[0].x.clone()
        for d in grp.decs:
            assert torch.equal(d.x, x0)  # replicated residual identical on every rank
            assert int(d.token.item()) == int(ref.token.item())
        e = rel_err(x0.cpu().numpy(), ref.x.cpu().numpy())
        worst = max(worst, e)
        assert e < 1e-4, e
    print(f"70B TP8 shard fused: worst rel x {worst:.2e}")
