"""Sparse prefill: the masking pass and the tcgen05 GEMM.

teal_prefill_gate is bit-exact against torch (mask = the reference's
sparsify test on rows >= sparse_from, sparsifier.py:120-134; bf16 hi / lo
split).  teal_prefill_gemm is checked against an fp64 product of the SAME
bf16 operands (the tensor cores multiply bf16 exactly and accumulate in
fp32: rel 1e-5 at m = 4096), and the two-term path against the fp32 masked product the
reference computes (rel 2e-5: hi + lo carries x to 2^-18).
"""

from __future__ import annotations

import pytest
import torch


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2408_14690_b200 import prefill
    return prefill


def _ref_gate(x, t, sparse_from):
    t32 = torch.tensor(t, dtype=torch.float32).item()
    keep = ~(x.abs() <= t32)
    keep[:sparse_from] = True
    return torch.where(keep, x, torch.zeros_like(x)), keep


def rel_err(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def _case(T, m, n=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, m, device="cuda", generator=g)
    w = (torch.randn(m, n, device="cuda", generator=g) / m ** 0.5).bfloat16()
    return x, w


@pytest.mark.parametrize("T,m,sparse_from,t", [(1, 64, 0, 0.5), (37, 256, 5, 0.8), (300, 4096, 64, 0.67),
                                                (5, 128, 9, 0.0), (16, 64, 0, float("inf"))])
def test_gate_bit_exact(P, T, m, sparse_from, t):
    x, _ = _case(T, m)
    x[0, :3] = torch.tensor([float("nan"), 0.0, -0.0])
    kept = torch.zeros(1, dtype=torch.int64, device="cuda")
    hi, lo = P.gate(x, t, sparse_from, terms=2, kept=kept)
    g, keep = _ref_gate(x, t, sparse_from)
    want_hi = g.bfloat16()
    want_lo = (g - want_hi.float()).bfloat16()
    assert torch.equal(hi.view(torch.int16), want_hi.view(torch.int16))
    assert torch.equal(lo.view(torch.int16), want_lo.view(torch.int16))
    assert kept.item() == int(keep[sparse_from:].sum())
    hi1, lo1 = P.gate(x, t, sparse_from, terms=1)
    assert lo1 is None and torch.equal(hi1.view(torch.int16), want_hi.view(torch.int16))


@pytest.mark.parametrize("T,m,n", [(1, 64, 128), (128, 64, 128), (129, 256, 256), (77, 512, 384),
                                   (300, 4096, 1024), (512, 4096, 4096)])
def test_gemm_one_term_exact_operands(P, T, m, n):
    x, w = _case(T, m, n, seed=T + m)
    hi = x.bfloat16()
    y = P.gemm(w, hi)
    want = hi.double() @ w.double()
    assert rel_err(y, want) < 1e-5  # fp32 accumulation in the tensor core over m terms


@pytest.mark.parametrize("T,m,n,sparse_from", [(64, 256, 128, 0), (200, 1024, 512, 32), (384, 4096, 1024, 100)])
def test_masked_gemm_matches_fp32_reference(P, T, m, n, sparse_from):
    x, w = _case(T, m, n, seed=7 + T)
    t = 0.6
    y = P.masked_gemm(x, w, t, sparse_from=sparse_from)
    g, _ = _ref_gate(x, t, sparse_from)
    want = g.double() @ w.double()
    assert rel_err(y, want) < 2e-5
    # rows before sparse_from are the dense product
    dense = x[:sparse_from].double() @ w.double()
    if sparse_from:
        assert rel_err(y[:sparse_from], dense) < 2e-5


@pytest.mark.parametrize("splits", [1, 2, 3, 0])
def test_split_k_is_deterministic(P, splits):
    # K split across CTAs, partials summed by the last arriver in split order:
    # identical bits on every run, and the same product as one split
    T, m, n = 70, 1024, 256
    x, w = _case(T, m, n, seed=11)
    hi, lo = P.gate(x, 0.5, 3)
    ys = [P.gemm(w, hi, lo, splits=splits) for _ in range(3)]
    assert all(torch.equal(ys[0], y) for y in ys[1:])
    g, _ = _ref_gate(x, 0.5, 3)
    assert rel_err(ys[0], g.double() @ w.double()) < 2e-5
    base = torch.randn(T, n, device="cuda")
    acc = base.clone()
    P.gemm(w, hi, lo, out=acc, accumulate=True, splits=splits)
    assert rel_err(acc, base.double() + g.double() @ w.double()) < 2e-5


def test_persistent_many_units(P):
    # more tiles than SMs: every CTA loops over several units (TMEM double buffer, smem ring wrap)
    T, m, n = 1000, 320, 4096
    x, w = _case(T, m, n, seed=5)
    y = P.masked_gemm(x, w, 0.4, sparse_from=10)
    g, _ = _ref_gate(x, 0.4, 10)
    assert rel_err(y, g.double() @ w.double()) < 2e-5


def test_accumulate_and_ragged_tail(P):
    T, m, n = 131, 192, 256
    x, w = _case(T, m, n, seed=3)
    base = torch.randn(T, n, device="cuda")
    y = base.clone()
    P.masked_gemm(x, w, 0.3, sparse_from=7, out=y, accumulate=True)
    g, _ = _ref_gate(x, 0.3, 7)
    assert rel_err(y, base.double() + g.double() @ w.double()) < 2e-5
    # a strided output row (ldy > n) leaves the padding untouched
    wide = torch.full((T, n + 64), 7.0, device="cuda")
    P.gemm(w, *P.gate(x, 0.3, 7), out=wide[:, :n])
    assert torch.all(wide[:, n:] == 7.0)
    assert rel_err(wide[:, :n], g.double() @ w.double()) < 2e-5


def test_rejects_bad_shapes(P):
    from paper_2408_14690_b200._clib import TealError  # noqa: F401
    x, w = _case(4, 96, 128)
    with pytest.raises(Exception, match="multiple of 64"):
        P.masked_gemm(x, w, 0.5)
    x, w = _case(4, 64, 96)
    with pytest.raises(Exception, match="multiple"):
        P.masked_gemm(x, w, 0.5)
    with pytest.raises(ValueError, match="sparse_from"):
        P.gate(x, 0.5, sparse_from=-1)


# ---- the decoder prompt pass ----------------------------------------------------

def _llama_toy(seed=0):
    from paper_2408_14690_b200 import decode as D
    spec = D.DecoderSpec(512, 8, 2, 1024, 2, vocab=1024, rope_theta=10000.0, norm_eps=1e-5, max_seq=128)
    return D.random_weights(spec, torch.bfloat16, seed=seed)


def _teacher_forced_decode(W, thr, toks, kv_dtype=None):
    from paper_2408_14690_b200 import decode as D
    dec = D.SparseDecoder(W, thr, kv_dtype=kv_dtype)
    dec.reset()
    for t in toks.tolist():
        dec.token.fill_(t)
        dec.step_token()
    return dec


@pytest.mark.parametrize("sparse", [False, True])
def test_prefill_matches_token_by_token_decode(P, sparse):
    # the prompt pass (all rows thresholded: sparse_from = 0) fills the same
    # K/V cache and last-position logits as stepping the decode engine
    # through the prompt one token at a time with the same thresholds
    from paper_2408_14690_b200 import decode as D
    W = _llama_toy()
    thr = D.calibrate_thresholds(W, 0.5, n_tokens=16, engine="launch") if sparse else None
    toks = torch.randint(0, 1024, (48,), generator=torch.Generator().manual_seed(1))
    dec = _teacher_forced_decode(W, thr, toks, kv_dtype=torch.float32)  # fp32 caches: no rounding flips
    pf = P.SparsePrefill(W, thr)
    kc = torch.zeros_like(dec.kcache)
    vc = torch.zeros_like(dec.vcache)
    r = pf.forward(tokens=toks, sparse_from=0, kv_cache=(kc, vc))
    T = len(toks)
    # sparse: rare mask flips where the two RMSNorm implementations round differently
    tol = 3e-3 if sparse else 2e-5
    assert rel_err(kc[:, :, :T], dec.kcache[:, :, :T]) < tol
    assert rel_err(vc[:, :, :T], dec.vcache[:, :, :T]) < tol
    assert rel_err(r.logits[0], dec.logits) < tol
    if sparse:  # realized sparsity of the thresholded rows is near the calibrated level
        frac = 1 - r.kept.sum().item() / (T * 2 * (3 * 512 + 512 + 2 * 512 + 1024))
        assert 0.35 < frac < 0.65, frac


def test_prefill_hands_off_to_the_decoder(P):
    # prefill(prompt) then decode == decode through prompt + continuation
    from paper_2408_14690_b200 import decode as D
    W = _llama_toy(seed=3)
    toks = torch.randint(0, 1024, (40,), generator=torch.Generator().manual_seed(2))
    ref = _teacher_forced_decode(W, None, toks)
    ref_next = ref.token.clone()
    ref.step_token()  # one generated step from the argmax token
    dec = D.SparseDecoder(W, None)
    dec.reset()
    r = P.SparsePrefill(W, None).forward(tokens=toks, decoder=dec)  # bf16 caches, as the decoder's
    assert dec._pos == len(toks) and int(dec.state[1]) == len(toks)
    assert torch.equal(r.next_token, ref_next)
    dec.step_token()
    # bf16 caches: values ~1e-6 apart can round one ulp (2^-8) apart
    assert rel_err(dec.logits, ref.logits) < 1e-3


def test_prefill_dense_prefix_matches_reference_forward(P):
    # the reference-written d=256 block (tests/golden/interop) with its TEALC1
    # thresholds: prefill with sparse_from = k reproduces model_forward_sparse
    # (dense_prefix = k) of the same model with bf16-rounded weights
    import numpy as np
    import paper_2408_14690_b200 as T
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200.model import MATRIX_NAMES, TransformerBlock, TransformerModel
    from paper_2408_14690_b200.tensor import Matrix
    from conftest import GOLDEN
    m = T.load_model(GOLDEN / "interop" / "model256.teal")
    cfgs, _ = T.load_configs(GOLDEN / "interop" / "configs256.txt")
    X = np.load(GOLDEN / "interop" / "expect.npz")["X256"]

    def rnd(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()

    blocks = tuple(TransformerBlock(b.d_model, b.n_heads, b.d_ff,
                                    {n: Matrix.from_2d(rnd(b.w2d(n)), b.weights[n].layout) for n in MATRIX_NAMES},
                                    b.rms_attn, b.rms_mlp) for b in m.blocks)
    mr = TransformerModel(m.d_model, m.n_heads, m.d_ff, blocks)
    W = T.decoder_weights(mr, dtype=torch.bfloat16, max_seq=64)
    thr = [[c.thresholds[n] for n in D.PROJ] for c in cfgs]
    for k in (0, 5, len(X)):
        want = T.model_forward_sparse(mr, X, cfgs, dense_prefix=k) if k else T.model_forward_sparse(mr, X, cfgs)
        got = P.SparsePrefill(W, thr, kv_dtype=torch.float32).forward(hidden=X, sparse_from=k).x
        assert rel_err(got, torch.as_tensor(want).to(got.device)) < 1e-5, k


def test_chunked_prefill_equals_one_pass(P):
    # the prompt in two chunks (the second attends to the first's cached K/V,
    # RoPE at its absolute positions) == one pass over the whole prompt
    W = _llama_toy(seed=5)
    from paper_2408_14690_b200 import decode as D
    thr = D.calibrate_thresholds(W, 0.5, n_tokens=16, engine="launch")
    toks = torch.randint(0, 1024, (56,), generator=torch.Generator().manual_seed(4))
    pf = P.SparsePrefill(W, thr, kv_dtype=torch.float32)
    L_, KVH, S, hd = W.spec.n_layers, W.spec.n_kv_heads, W.spec.max_seq, W.spec.head_dim
    one = (torch.zeros(L_, KVH, S, hd, device="cuda"), torch.zeros(L_, KVH, S, hd, device="cuda"))
    two = (torch.zeros_like(one[0]), torch.zeros_like(one[1]))
    r1 = pf.forward(tokens=toks, sparse_from=0, kv_cache=one, logits="all")
    pf.forward(tokens=toks[:24], sparse_from=0, kv_cache=two, logits="none")
    r2 = pf.forward(tokens=toks[24:], sparse_from=0, kv_cache=two, logits="all", start_pos=24)
    T = len(toks)
    assert rel_err(two[0][:, :, :T], one[0][:, :, :T]) < 1e-5
    assert rel_err(two[1][:, :, :T], one[1][:, :, :T]) < 1e-5
    assert rel_err(r2.x, r1.x[24:]) < 1e-5
    assert torch.equal(r2.next_token, r1.next_token)
    with pytest.raises(ValueError, match="continues a cache"):
        pf.forward(tokens=toks[:4], start_pos=4)


def test_batch_prefill_hands_off_to_the_batch_decoder(P):
    # B prompts prefilled into the batch decoder's per-sequence cache slices,
    # then one lockstep step == the batch decoder stepped through the prompts
    # (dense: the per-token and the shared batch masks coincide)
    from paper_2408_14690_b200 import batch as BT
    W = _llama_toy(seed=6)
    B, T = 4, 20
    prompts = torch.randint(0, 1024, (B, T), generator=torch.Generator().manual_seed(8))
    ref = BT.BatchDecoder(W, None, B)
    ref.reset()
    for t in range(T):
        ref.tokens.copy_(prompts[:, t].to(torch.int32))
        ref.step()
    ref_next = ref.tokens.clone()
    ref.step()
    dec = BT.BatchDecoder(W, None, B)
    dec.reset()
    P.SparsePrefill(W, None).forward_batch([p_.tolist() for p_ in prompts], dec)
    assert torch.equal(dec.tokens, ref_next)
    dec.step()
    assert rel_err(dec.logits, ref.logits) < 1e-3  # bf16 caches: one-ulp rounding differences


def test_generate_matches_step_decoding(P):
    # prefill + graph-replayed decode == the step engine stepped through the
    # prompt and then decoding greedily (dense, fp32 caches: no rounding ties)
    from paper_2408_14690_b200 import engine as E
    W = _llama_toy(seed=7)
    prompt = torch.randint(0, 1024, (16,), generator=torch.Generator().manual_seed(9)).tolist()
    got = P.generate(W, None, prompt, 8, kv_dtype=torch.float32)
    dec = E.StepDecoder(W, None, kv_dtype=torch.float32)
    dec.reset()
    for t in prompt:
        dec.token.fill_(t)
        dec.step_token()
    want = [int(dec.token)]
    for _ in range(7):
        dec.step_token()
        want.append(int(dec.token))
    assert got == want


def test_log_likelihood_matches_stepwise_logits(P):
    # the prompt pass with logits="all" gives every position's next-token
    # distribution: equal to the step engine's logits teacher-forced (dense)
    from paper_2408_14690_b200 import engine as E
    W = _llama_toy(seed=10)
    toks = torch.randint(0, 1024, (24,), generator=torch.Generator().manual_seed(11)).tolist()
    logp, ppl = P.log_likelihood(W, None, toks, kv_dtype=torch.float32)
    dec = E.StepDecoder(W, None, kv_dtype=torch.float32)
    dec.reset()
    want = []
    for i, t in enumerate(toks[:-1]):
        dec.token.fill_(t)
        dec.step_token()
        want.append(float(torch.log_softmax(dec.logits.double(), 0)[toks[i + 1]]))
    want = torch.tensor(want, dtype=torch.float64)
    assert torch.allclose(logp.cpu().double(), want, atol=1e-4, rtol=0)
    assert abs(ppl - float(torch.exp(-want.mean()))) / ppl < 1e-4
