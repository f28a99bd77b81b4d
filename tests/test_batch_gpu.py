"""GPU: small-batch decode with shared masks (BASELINE config 5,
batch.BatchDecoder) against the reference semantics.

* masks: every projection's shared mask equals the oracle's
  sparsify_batched(h, t) mask (pkg/src/actsparse/sparsifier.py:136-155) of
  the [B, m] input the kernel saw — bit for bit;
* B = 1 reduces to the per-token engine (the reference's B = 1 reduction,
  pkg/tests/test_acceptance.py:216-221): BatchDecoder(B=1) == StepDecoder;
  B identical streams decode exactly like one stream;
* a 2-layer GQA + RoPE model decoded free-running against a plain torch fp32
  shared-mask decode (rel 1e-3, tokens equal);
* per-batch-size calibration (test_acceptance.py:223-239):
  thresholds from batch-mean histograms give ~50 % column sparsity on fresh
  streams at B = 2, 4, 8;
* config 5 at full Mistral-7B shape (32 layers, vocab 32000, B = 16,
  bf16 / int8 / int4 at 50 %): masks bit-exact and every projection output
  teacher-forced one operation deep within rel 1e-3 (north-star bar 1e-2).
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import actsparse_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

PROJ = ("q", "k", "v", "o", "gate", "up", "down")
TAP = {"q": "pre_attn", "k": "pre_attn", "v": "pre_attn", "o": "attn_out", "gate": "pre_mlp", "up": "pre_mlp",
       "down": "mlp_inter"}


def _small_spec():
    from paper_2408_14690_b200 import decode as D
    return D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)


def _check_masks(dec, thr):
    L = dec.spec.n_layers
    for l in range(L):
        for i, p in enumerate(PROJ):
            xs = dec.taps[TAP[p]][l].cpu().numpy()
            _, want = R.sparsify_batched(xs, thr[l][i]) if thr[l][i] is not None else (None, np.zeros(xs.shape[1], bool))
            got = dec.masks[p][l].cpu().numpy().astype(bool)
            assert np.array_equal(got, want), (l, p, int((got != want).sum()))
            assert int(dec.kept[l, i]) >= int((~want).sum())


def torch_batch_reference(W, thr, steps_tokens, spec, kv_dtype=torch.float32):
    """Plain torch fp32 lockstep decode with shared masks (mean_b |h| <= fl32(t))."""
    d, hd, H, KVH = spec.d_model, spec.head_dim, spec.n_heads, spec.n_kv_heads
    G = H // KVH
    emb = W.embedding.float()
    inv = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64, device=emb.device) / hd))

    def rope(x, pos):  # [B, heads, hd]
        ang = pos * inv
        c, s = torch.cos(ang).float(), torch.sin(ang).float()
        x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def sp(a, t):
        if t is None:
            return a
        m = a.abs().mean(dim=0) <= float(np.float32(t))
        return torch.where(m[None, :], torch.zeros_like(a), a)

    def norm(x, w):
        return x / torch.sqrt((x * x).mean(dim=1, keepdim=True) + spec.norm_eps) * w

    K = [[] for _ in W.layers]
    V = [[] for _ in W.layers]
    outs = []
    for pos, toks in enumerate(steps_tokens):
        B = len(toks)
        x = emb[torch.tensor(toks, device=emb.device)].clone()
        for l, lw in enumerate(W.layers):
            t = thr[l]
            h = norm(x, lw.rms_attn)
            wqkv = lw.wqkv.float()
            nq, nkv = spec.n_q, spec.n_kv
            q = rope((sp(h, t[0]) @ wqkv[:, :nq]).view(B, H, hd), pos)
            k = rope((sp(h, t[1]) @ wqkv[:, nq:nq + nkv]).view(B, KVH, hd), pos)
            v = (sp(h, t[2]) @ wqkv[:, nq + nkv:]).view(B, KVH, hd)
            K[l].append(k.to(kv_dtype).float())
            V[l].append(v.to(kv_dtype).float())
            Ks, Vs = torch.stack(K[l], 2), torch.stack(V[l], 2)  # [B, KVH, T, hd]
            ctx = torch.stack([torch.cat([torch.softmax((Ks[b, hh // G] @ q[b, hh]) / math.sqrt(hd), 0) @ Vs[b, hh // G]
                                          for hh in range(H)]) for b in range(B)])
            x = x + sp(ctx, t[3]) @ lw.wo.float()
            hm = norm(x, lw.rms_mlp)
            wgu = lw.wgu.float()
            f = spec.d_ff
            gate, up = sp(hm, t[4]) @ wgu[:, :f], sp(hm, t[5]) @ wgu[:, f:]
            x = x + sp(gate / (1 + torch.exp(-gate)) * up, t[6]) @ lw.wdown.float()
        outs.append((x.clone(), norm(x, W.final_norm) @ W.lm_head.float()))
    return outs


@pytest.mark.parametrize("B", [1, 3, 4, 16])
def test_small_model_against_torch_shared_mask_decode(B):
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    spec = _small_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=21)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    g = np.random.default_rng(22)
    steps = [g.integers(0, spec.vocab, B).tolist() for _ in range(6)]
    ref = torch_batch_reference(W, thr, steps, spec)
    dec = BT.BatchDecoder(W, thr, B, kv_dtype=torch.float32, taps=True)
    dec.reset()
    for i, toks in enumerate(steps):
        dec.tokens.copy_(torch.tensor(toks, dtype=torch.int32))
        dec.kept.zero_()
        dec.step()
        torch.cuda.synchronize()
        _check_masks(dec, thr)
        x_ref, lg_ref = ref[i]
        assert rel_err(dec.x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-3, i
        assert rel_err(dec.logits.cpu().numpy(), lg_ref.cpu().numpy()) < 1e-3, i
        assert dec.tokens.tolist() == torch.argmax(lg_ref, dim=1).tolist() or \
            rel_err(dec.logits.cpu().numpy(), lg_ref.cpu().numpy()) < 1e-5


def test_batch_one_equals_the_per_token_engine():
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    spec = _small_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=23)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    a = BT.BatchDecoder(W, thr, 1, kv_dtype=torch.float32)
    b = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    a.reset()
    b.reset()
    for tok in (5, 17, 999, 3, 250):
        a.tokens.fill_(tok)
        b.token.fill_(tok)
        a.step()
        b.step_token()
        torch.cuda.synchronize()
        assert rel_err(a.x[0].cpu().numpy(), b.x.cpu().numpy()) < 1e-5
        assert int(a.tokens[0]) == int(b.token)


def test_identical_streams_decode_like_one_stream():
    # mean_b |h| over B equal rows is |h|: the shared mask is the B = 1 mask
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    spec = _small_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=24)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    one = BT.BatchDecoder(W, thr, 1)
    four = BT.BatchDecoder(W, thr, 4)
    one.reset()
    four.reset()
    for tok in (5, 17, 999):
        one.tokens.fill_(tok)
        four.tokens.fill_(tok)
        one.step()
        four.step()
        torch.cuda.synchronize()
        for b in range(4):  # (B = 1 runs the FMA kernel, B = 4 the mma.sync one: fp32 rounding differs)
            assert rel_err(four.x[b].cpu().numpy(), one.x[0].cpu().numpy()) < 1e-5
            assert int(four.tokens[b]) == int(one.tokens[0])


def test_graph_replay_equals_eager():
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    spec = _small_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=25)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    dec = BT.BatchDecoder(W, thr, 8)
    toks = [np.random.default_rng(s).integers(0, 1000, 8).tolist() for s in range(4)]
    dec.reset()
    eager = []
    for t in toks:
        dec.tokens.copy_(torch.tensor(t, dtype=torch.int32))
        dec.step()
        eager.append(dec.x.clone())
    dec.reset()
    dec.capture()
    dec.reset()
    for t, e in zip(toks, eager):
        dec.tokens.copy_(torch.tensor(t, dtype=torch.int32))
        dec.replay()
        torch.cuda.synchronize()
        assert torch.equal(dec.x, e)


@pytest.mark.parametrize("B", [2, 4, 8])
def test_per_batch_size_calibration_realizes_target_column_sparsity(B):
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=128)
    W = D.random_weights(spec, torch.bfloat16, seed=26)
    hists = BT.calibrate_batch_histograms(W, B, n_steps=24, seed=27)
    thr = BT.batch_thresholds(hists, spec.n_layers, 0.5)
    dec = BT.BatchDecoder(W, thr, B, taps=True)
    dec.reset()
    g = torch.Generator(device="cuda").manual_seed(28)
    for _ in range(6):
        dec.tokens.copy_(torch.randint(0, spec.vocab, (B,), device="cuda", generator=g, dtype=torch.int32))
        dec.step()
    torch.cuda.synchronize()
    col = np.mean([float(dec.masks[p].float().mean()) for p in PROJ])
    assert abs(col - 0.5) <= 0.05, (B, col)


@pytest.fixture(scope="module")
def mistral():
    from paper_2408_14690_b200 import batch as BT
    from paper_2408_14690_b200 import decode as D
    W = D.random_weights(D.MISTRAL_7B, torch.bfloat16, seed=7)
    return W, BT.calibrate_batch_thresholds(W, 16, 0.5, n_steps=32, seed=8, passes=2)


def _teacher_forced(dec, thr, pos):
    """Each projection output one op deep from the engine's own inputs."""
    sp = dec.spec
    H, KVH, hd, nq, nkv = sp.n_heads, sp.n_kv_heads, sp.head_dim, sp.n_q, sp.n_kv
    G = H // KVH
    B = dec.B
    inv = 1.0 / (sp.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64, device="cuda") / hd))
    ang = pos * inv
    c, s = torch.cos(ang).float(), torch.sin(ang).float()

    def rope(x):
        x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def spz_p(a, proj, l):
        # the shared mask the kernel applied — checked bit-exact against the
        # oracle's sparsify_batched by _check_masks (a torch mean here could
        # round a tie the other way)
        m = dec.masks[proj][l].bool()
        return torch.where(m[None, :], torch.zeros_like(a), a)

    worst = {}

    def rec(k, got, want):
        worst[k] = max(worst.get(k, 0.0), rel_err(got.cpu().numpy(), want.cpu().numpy()))

    for l in range(sp.n_layers):
        t = thr[l]
        pw = dec.pw[l]
        W = {p: pw[p].dequantize() for p in PROJ}
        h = dec.taps["pre_attn"][l]
        rec("q", dec.tap_q[l], rope((spz_p(h, "q", l) @ W["q"]).view(B, H, hd)).view(B, nq))
        k = rope((spz_p(h, "k", l) @ W["k"]).view(B, KVH, hd))
        v = (spz_p(h, "v", l) @ W["v"]).view(B, KVH, hd)
        rec("k_row", dec.kcache[l][:, :, pos].float(), k.to(dec.kv_dtype).float())
        rec("v_row", dec.vcache[l][:, :, pos].float(), v.to(dec.kv_dtype).float())
        q = dec.tap_q[l].view(B, H, hd)
        Ks, Vs = dec.kcache[l][:, :, :pos + 1].float(), dec.vcache[l][:, :, :pos + 1].float()
        ctx = torch.stack([torch.cat([torch.softmax((Ks[b, hh // G] @ q[b, hh]) / math.sqrt(hd), 0) @ Vs[b, hh // G]
                                      for hh in range(H)]) for b in range(B)])
        rec("ctx", dec.taps["attn_out"][l], ctx)
        rec("o", dec.tap_o[l], spz_p(dec.taps["attn_out"][l], "o", l) @ W["o"])
        hm = dec.taps["pre_mlp"][l]
        gate, up = spz_p(hm, "gate", l) @ W["gate"], spz_p(hm, "up", l) @ W["up"]
        rec("inter", dec.taps["mlp_inter"][l], gate / (1 + torch.exp(-gate)) * up)
        rec("down", dec.tap_down[l], spz_p(dec.taps["mlp_inter"][l], "down", l) @ W["down"])
    lg = dec.tap_final @ dec.lm.dequantize()
    rec("logits", dec.logits, lg)
    assert dec.tokens.tolist() == torch.argmax(dec.logits, dim=1).tolist()
    return worst


@pytest.mark.parametrize("quant", [None, "int8", "int4"])
def test_mistral_7b_b16_config5(mistral, quant):
    from paper_2408_14690_b200 import batch as BT
    W, thr = mistral
    dec = BT.BatchDecoder(W, thr, 16, quant=quant, taps=True)
    dec.reset()
    g = np.random.default_rng(9)
    worst = {}
    cols = []
    for pos in range(3):
        dec.tokens.copy_(torch.tensor(g.integers(0, 32000, 16), dtype=torch.int32))
        dec.kept.zero_()
        dec.step()
        torch.cuda.synchronize()
        _check_masks(dec, thr)
        cols.append(np.mean([float(dec.masks[p].float().mean()) for p in PROJ]))
        for k, v in _teacher_forced(dec, thr, pos).items():
            worst[k] = max(worst.get(k, 0.0), v)
    per = {p: round(float(dec.masks[p].float().mean()), 3) for p in PROJ}
    print(f"Mistral-7B B=16 {quant}: column sparsity {np.mean(cols):.3f} (last step per projection {per}), "
          f"worst rel", {k: f"{v:.1e}" for k, v in worst.items()})
    bad = {k: v for k, v in worst.items() if not v < 1e-3}
    assert not bad, bad
    del dec
    torch.cuda.empty_cache()


def test_mistral_7b_b16_realized_column_sparsity(mistral):
    # thresholds from two-pass batch-mean calibration (B = 16, positions
    # 0..31): over the same span of positions the shared masks prune ~50 % of
    # the input columns of the projections
    from paper_2408_14690_b200 import batch as BT
    W, thr = mistral
    dec = BT.BatchDecoder(W, thr, 16, count_kept=True)
    dec.reset()
    g = torch.Generator(device="cuda").manual_seed(123)
    for _ in range(32):
        dec.tokens.copy_(torch.randint(0, 32000, (16,), device="cuda", generator=g, dtype=torch.int32))
        dec.step()
    torch.cuda.synchronize()
    shapes = dec.spec.proj_shapes()
    per = {p: 1.0 - float(dec.kept[:, i].sum()) / (32 * dec.spec.n_layers * shapes[p][1]) for i, p in enumerate(PROJ)}
    total = sum(m for (_, m) in shapes.values())
    overall = 1.0 - float(dec.kept.sum()) / (32 * dec.spec.n_layers * total)
    print("Mistral-7B B=16 realized column sparsity", round(overall, 3), {k: round(v, 3) for k, v in per.items()})
    # every projection whose input is position-independent lands on the
    # target; the attention output of a random-init model shrinks with the
    # position (softmax over random scores averages ~p value rows), so its
    # batch-mean mask ramps from 0 at position 0 to ~all pruned late in the
    # calibrated span — reported, not asserted
    assert all(abs(per[p] - 0.5) < 0.06 for p in PROJ if p != "o"), per
