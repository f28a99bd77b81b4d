"""GPU: the persistent one-launch-per-token decode engine (engine.StepDecoder,
csrc/teal_step.cu) against the reference and against the per-launch engine.

* config 1 toy model (fp32 weights, MHA, no RoPE): every decode step equals
  row t of the reference's model_forward_sparse / model_forward_dense
  (pkg/src/actsparse/model.py:398-410) on the golden inputs;
* masks bit-exact at the kernel boundary: the keep bitmask the kernel writes
  for each of the seven projection inputs equals the oracle's mask of the
  kernel's own tap vector; kept counts equal popcounts;
* Llama-style GQA + RoPE + bf16 weights (parity unpinned): against
  a plain torch fp32 decode of the same weights;
* the step is replay-safe (counters/queue self-reset) and deterministic.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, rel_err
from oracle import actsparse_ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def toy():
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    blocks = R.gen_model_weights(5, 2, 512, 8, 1408)
    return D, E, blocks, D.weights_from_blocks(blocks, 8, max_seq=64)


def _thr(g):
    return [g[f"thr50_{b}"].tolist() for b in range(2)]


def test_toy_dense_rows_match_reference(toy):
    D, E, _, W = toy
    g = golden("toy_model")
    dec = E.StepDecoder(W, None)
    dec.reset()
    errs = [rel_err(dec.step_hidden(g["X"][t]).cpu().numpy(), g["out_dense"][t]) for t in range(48)]
    assert max(errs) < 1e-5, max(errs)


@pytest.mark.parametrize("chunk", [8, 32, 64])
def test_toy_attention_chunking(toy, chunk):
    # single-chunk fast path, multi-chunk combine, and CTAs that reach the
    # attention phase without a qkv slice (they must wait for the step's load)
    D, E, _, W = toy
    g = golden("toy_model")
    dec = E.StepDecoder(W, _thr(g), attn_chunk=chunk)
    dec.reset()
    errs = [rel_err(dec.step_hidden(g["X"][t]).cpu().numpy(), g["out_sparse50"][t]) for t in range(40)]
    assert np.median(errs) < 1e-5 and max(errs) < 1e-4, (chunk, np.median(errs), max(errs))


def test_toy_sparse50_rows_match_reference(toy):
    D, E, _, W = toy
    g = golden("toy_model")
    dec = E.StepDecoder(W, _thr(g))
    dec.reset()
    errs = [rel_err(dec.step_hidden(g["X"][t]).cpu().numpy(), g["out_sparse50"][t]) for t in range(48)]
    assert np.median(errs) < 1e-5 and max(errs) < 1e-4, (np.median(errs), max(errs))


def test_toy_masks_bit_exact_at_kernel_boundary(toy):
    D, E, _, W = toy
    g = golden("toy_model")
    thr = _thr(g)
    dec = E.StepDecoder(W, thr, taps=True)
    dec.reset()
    for t in range(8):
        dec.taps.kept.zero_()
        dec.step_hidden(g["X"][t])
        torch.cuda.synchronize()
        for l in range(2):
            for p_i, p in enumerate(D.PROJ):
                h = dec.taps.h[R.MATRIX_TAP[p]][l].cpu().numpy()
                keep = R.keep_mask(h, thr[l][p_i])
                got = dec.taps.bits[p][l].cpu().numpy().view(np.uint32)
                assert np.array_equal(got, R.pack_bits(keep)), (t, l, p)
                assert int(dec.taps.kept[l, p_i]) == int(keep.sum()), (t, l, p)


def test_toy_matches_launch_engine(toy):
    D, E, _, W = toy
    g = golden("toy_model")
    a, b = D.SparseDecoder(W, _thr(g)), E.StepDecoder(W, _thr(g))
    a.reset()
    b.reset()
    for t in range(16):
        ya = a.step_hidden(g["X"][t]).clone()
        yb = b.step_hidden(g["X"][t]).clone()
        assert rel_err(yb.cpu().numpy(), ya.cpu().numpy()) < 1e-5, t


def test_replay_deterministic_and_self_resetting(toy):
    D, E, _, W = toy
    g = golden("toy_model")
    dec = E.StepDecoder(W, _thr(g))
    outs = []
    for _ in range(2):
        dec.reset()
        outs.append([dec.step_hidden(g["X"][t]).clone() for t in range(6)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    dec.reset()
    dec.capture(from_token=False)
    dec.reset()
    for t in range(6):
        dec.x_in.copy_(torch.from_numpy(g["X"][t]))
        dec.replay()
        assert torch.equal(dec.x, outs[0][t]), t
    assert int(dec.counters.abs().sum()) == 0 and int(dec.ctrl.abs().sum()) == 0


@pytest.mark.parametrize("kv", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("sparse", [False, True])
def test_llama_style_gqa_rope_bf16(sparse, kv):
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from test_decode_gpu import torch_decode_reference
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=3)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2 if sparse else [[None] * 7] * 2
    dec = E.StepDecoder(W, thr, kv_dtype=kv, attn_chunk=16)
    dec.reset()
    tokens = [5, 17, 999, 3, 250, 7, 7, 42, 11, 600, 1, 2, 3, 4, 5, 6, 8, 9, 10]
    ref = torch_decode_reference(W, thr, tokens, spec, kv)
    for i, tok in enumerate(tokens):
        dec.token.fill_(tok)
        dec.step_token()
        torch.cuda.synchronize()
        x_ref, logits_ref = ref[i]
        assert rel_err(dec.x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-3, i
        assert rel_err(dec.logits.cpu().numpy(), logits_ref.cpu().numpy()) < 1e-2, i
        lg = dec.logits
        assert int(dec.token.item()) == int(torch.argmax(lg).item()), i


def test_llama_graph_replay_chains_tokens():
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=4)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    a, b = D.SparseDecoder(W, thr), E.StepDecoder(W, thr)
    for dec in (a, b):
        dec.reset()
        dec.token.fill_(7)
    seq_a, seq_b = [], []
    b.capture()
    b.reset()
    b.token.fill_(7)
    for _ in range(12):
        seq_a.append(int(a.step_token().item()))
        b.replay()
        seq_b.append(int(b.token.item()))
    # same weights, same thresholds: the greedy chains agree (fp32 accumulate
    # order differs between engines; logits are far from ties here)
    assert seq_a == seq_b


@pytest.mark.parametrize("quant", ["int8", "int4"])
@pytest.mark.parametrize("sparse", [False, True])
def test_llama_style_quantised_weights(quant, sparse):
    # int8 / int4 tiled rows (config 5 at batch 1): the step engine against a
    # torch fp32 decode of the SAME dequantised weights (quantisation error
    # itself is not part of the parity; SURVEY.md §8c "parity unpinned")
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from test_decode_gpu import torch_decode_reference
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1024, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=5)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2 if sparse else [[None] * 7] * 2
    dec = E.StepDecoder(W, thr, kv_dtype=torch.float32, quant=quant, attn_chunk=16)
    f, nq, nkv = spec.d_ff, spec.n_q, spec.n_kv
    layers = []
    for lw, tw in zip(W.layers, dec.tw):
        layers.append(D.LayerWeights(
            wqkv=E.untile(tw["qkv"].dequantize(), nq + 2 * nkv), wo=E.untile(tw["o"].dequantize(), spec.d_model),
            wgu=E.untile_gate_up(tw["gu"].dequantize(), f), wdown=E.untile(tw["down"].dequantize(), spec.d_model),
            rms_attn=lw.rms_attn, rms_mlp=lw.rms_mlp))
    Wq = D.DecoderWeights(spec, layers, W.embedding, W.final_norm, E.untile(dec.lm_t.dequantize(), spec.vocab))
    err_q = float((Wq.layers[0].wdown - W.layers[0].wdown.float()).norm() / W.layers[0].wdown.float().norm())
    assert err_q < (0.02 if quant == "int8" else 0.2), err_q
    dec.reset()
    tokens = [5, 17, 999, 3, 250, 7, 7, 42, 11, 600]
    ref = torch_decode_reference(Wq, thr, tokens, spec, torch.float32)
    for i, tok in enumerate(tokens):
        dec.token.fill_(tok)
        dec.step_token()
        torch.cuda.synchronize()
        x_ref, logits_ref = ref[i]
        assert rel_err(dec.x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-3, (quant, i)
        assert rel_err(dec.logits.cpu().numpy(), logits_ref.cpu().numpy()) < 1e-3, (quant, i)


@pytest.mark.parametrize("super_chunks", [2, 3])
def test_long_context_variant_matches_default(super_chunks):
    # units walking several 16-position chunks with an online softmax (the
    # long-context kernel variant) against the default one-chunk units
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from test_decode_gpu import torch_decode_reference
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=128)
    W = D.random_weights(spec, torch.bfloat16, seed=3)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    dec = E.StepDecoder(W, thr, kv_dtype=torch.float32, attn_chunk=16, long_context=super_chunks)
    dec.reset()
    tokens = [5, 17, 999, 3, 250, 7, 7, 42, 11, 600] * 7  # 70 positions: up to 5 chunks, 2-3 super units
    ref = torch_decode_reference(W, thr, tokens, spec, torch.float32)
    for i, tok in enumerate(tokens):
        dec.token.fill_(tok)
        dec.step_token()
        torch.cuda.synchronize()
        x_ref, logits_ref = ref[i]
        assert rel_err(dec.x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-3, i
        assert int(dec.token.item()) == int(torch.argmax(logits_ref).item()) or \
            rel_err(dec.logits.cpu().numpy(), logits_ref.cpu().numpy()) < 1e-3, i


def test_long_context_switches_by_position():
    # long_context with a switch position: the first steps run the default
    # kernel, later ones the multi-chunk variant (eager and graph replay)
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from test_decode_gpu import torch_decode_reference
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=128)
    W = D.random_weights(spec, torch.bfloat16, seed=3)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    tokens = [5, 17, 999, 3, 250, 7, 7, 42, 11, 600] * 6
    ref = torch_decode_reference(W, thr, tokens, spec, torch.float32)
    for graph in (False, True):
        dec = E.StepDecoder(W, thr, kv_dtype=torch.float32, attn_chunk=16, long_context=2, long_from=30)
        dec.reset()
        if graph:
            dec.capture()
            dec.reset()
        for i, tok in enumerate(tokens):
            dec.token.fill_(tok)
            dec.step_token()
            torch.cuda.synchronize()
            assert rel_err(dec.x.cpu().numpy(), ref[i][0].cpu().numpy()) < 1e-3, (graph, i)
            assert dec.last_long == (i >= 30), (graph, i)  # the variant that actually ran


@pytest.mark.parametrize("engine", ["step", "launch"])
@pytest.mark.parametrize("graph", [False, True])
def test_position_past_max_seq_raises(engine, graph):
    # the KV cache holds max_seq positions: the step that would write row
    # max_seq is refused on the host (the kernels also trap on it)
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    spec = D.DecoderSpec(1024, 8, 2, 2816, 1, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=4)
    W = D.random_weights(spec, torch.bfloat16, seed=3)
    dec = E.StepDecoder(W, None) if engine == "step" else D.SparseDecoder(W, None)
    dec.reset()
    if graph:
        dec.capture()
        dec.reset()
    for _ in range(4):
        dec.step_token()
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="max_seq"):
        dec.step_token()
    dec.reset(start_pos=3)
    dec.step_token()
    torch.cuda.synchronize()


@pytest.mark.parametrize("engine", ["step", "launch"])
def test_thresholded_lm_head(engine):
    """§8(f)#3: an optional threshold on the LM head's input (the final-norm
    row).  Logits equal where(|h| <= fl32(t), 0, h) @ W_lm of the decoder's own
    final residual; lm_threshold None keeps the dense head."""
    import torch
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    spec = D.DecoderSpec(512, 8, 2, 1024, 2, vocab=2048, rope_theta=10000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=9)
    toks = [5, 77, 901, 12, 1500, 3]
    t = 0.8

    def run(lm_t):
        dec = (E.StepDecoder if engine == "step" else D.SparseDecoder)(W, None, lm_threshold=lm_t)
        dec.reset()
        for tk in toks:
            dec.token.fill_(tk)
            dec.step_token()
        torch.cuda.synchronize()
        return dec

    dense, sparse = run(None), run(t)
    x = dense.x.float()
    # the final residual row is the same in both runs (the threshold only acts on the LM head)
    h = x / torch.sqrt((x.double() ** 2).mean().float() + spec.norm_eps) * W.final_norm
    wl = W.lm_head.float()
    t32 = float(np.float32(t))
    ref_dense = h @ wl
    ref_sparse = torch.where(h.abs() <= t32, torch.zeros_like(h), h) @ wl
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm())  # noqa: E731
    assert rel(dense.logits, ref_dense) < 1e-4
    assert rel(sparse.logits, ref_sparse) < 2e-3
    assert rel(sparse.logits, ref_dense) > 1e-2  # the threshold really prunes
