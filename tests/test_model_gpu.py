"""Block / model forwards, calibration and greedy allocation against the
reference's golden outputs (tests/golden/make_golden.py).

Reference tests mirrored: pkg/tests/test_model.py:191-331 (sparse forward,
calibration), pkg/tests/test_greedy.py:57-127 (trace, invariants).  CPU-only
tests cover the host surface: seeded weights bit-identical to the reference
(SHA), file formats TEALM1 / TEALG1 / TEALC1 round trips, validation.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2408_14690_b200 as T
from conftest import golden, rel_err, sha
from oracle import actsparse_ref as R

TAPS = ("pre_attn", "attn_out", "pre_mlp", "mlp_inter")


@pytest.fixture(scope="module")
def toy_model():
    return T.gen_model(T.RngStream(5), 2, 512, 8, 1408)


@pytest.fixture(scope="module")
def greedy_block():
    return T.gen_block(T.RngStream(31), 64, 2, 176)


# ---------------------------------------------------------------- CPU ---------

def test_seeded_weights_match_reference(toy_model):
    g = golden("toy_model")
    for b, blk in enumerate(toy_model.blocks):
        for n in T.MATRIX_NAMES:
            assert sha(blk.weights[n].to_2d()) == str(g[f"w_sha_{b}_{n}"]), (b, n)
    blk0 = T.gen_block(T.RngStream(2024), 256, 4, 704)
    assert sha(blk0.weights["q"].to_2d()) == str(g["w_sha_default_q"])


def test_block_validation():
    blk = T.gen_block(T.RngStream(1), 8, 2, 16)
    with pytest.raises(ValueError, match="divisible"):
        T.TransformerBlock(8, 3, 16, blk.weights, blk.rms_attn, blk.rms_mlp)
    bad = dict(blk.weights)
    bad["q"] = T.Matrix.from_2d(np.zeros((4, 8), np.float32))
    with pytest.raises(ValueError, match="expected 8x8"):
        T.TransformerBlock(8, 2, 16, bad, blk.rms_attn, blk.rms_mlp)
    assert blk.footprints()["gate"] == 16 * 8
    assert T.tap_dim(blk, T.TapPosition.MLP_INTER) == 16


def test_config_validation():
    lv = {n: 0.5 for n in T.MATRIX_NAMES}
    th = {n: 0.1 for n in T.MATRIX_NAMES}
    cfg = T.BlockSparsityConfig(lv, th)
    assert cfg.as_row() == [0.1] * 7
    with pytest.raises(ValueError, match="outside"):
        T.BlockSparsityConfig({**lv, "q": 1.5}, th)
    with pytest.raises(ValueError, match="finite"):
        T.BlockSparsityConfig(lv, {**th, "k": float("inf")})
    with pytest.raises(ValueError, match="exactly"):
        T.BlockSparsityConfig({"q": 0.1}, th)


def test_model_file_round_trip(tmp_path, toy_model):
    p = tmp_path / "m.teal"
    T.save_model(p, toy_model)
    back = T.load_model(p)
    assert (back.d_model, back.n_heads, back.d_ff, len(back.blocks)) == (512, 8, 1408, 2)
    for a, b in zip(toy_model.blocks, back.blocks):
        for n in T.MATRIX_NAMES:
            assert np.array_equal(a.w2d(n), b.w2d(n))
        assert np.array_equal(a.rms_attn, b.rms_attn)
    head = p.read_bytes().split(b"\n", 1)[0]
    assert head == b"TEALM1 2 512 8 1408"


def test_trace_and_config_round_trip(tmp_path):
    steps = [T.GreedyStep(0.0, {n: 0.0 for n in T.MATRIX_NAMES}, None, 0.0),
             T.GreedyStep(0.05, {**{n: 0.0 for n in T.MATRIX_NAMES}, "down": 0.1 / 3}, "down", 0.123456789)]
    tr = T.GreedyTrace("block0", 0.05, steps)
    T.save_trace(tmp_path / "t", tr)
    back = T.load_trace(tmp_path / "t")
    assert back.block_id == "block0" and back.alpha == 0.05
    assert [s.chosen for s in back.steps] == [None, "down"]
    assert back.steps[1].levels["down"] == 0.1 / 3 and back.steps[1].error == 0.123456789
    cfg = T.BlockSparsityConfig({n: 0.3 for n in T.MATRIX_NAMES}, {n: 1 / 7 for n in T.MATRIX_NAMES})
    T.save_configs(tmp_path / "c", [cfg, cfg], 0.5)
    cfgs, tgt = T.load_configs(tmp_path / "c")
    assert tgt == 0.5 and cfgs[1].thresholds["q"] == 1 / 7  # %.17g round trip is exact
    assert (tmp_path / "c").read_text().splitlines()[0] == "TEALC1 2 0.5"


def test_cost_estimate_and_policy():
    assert T.cost_estimate(7, 0.05, 10) == 9800
    with pytest.raises(ValueError):
        T.StepPolicy(0.0)
    with pytest.raises(ValueError):
        T.cost_estimate(0, 0.1, 1)


def test_select_step():
    steps = [T.GreedyStep(p, {n: p for n in T.MATRIX_NAMES}, None if p == 0 else "q", 0.0) for p in (0.0, 0.3, 0.6, 1.0)]
    tr = T.GreedyTrace("b", 0.1, steps)
    assert T.select_step(tr, 0.5).block_sparsity == 0.6
    assert T.select_step(tr, 0.3).block_sparsity == 0.3
    T.validate_trace(tr, {n: 1 for n in T.MATRIX_NAMES})
    bad = T.GreedyTrace("b", 0.1, steps[:2] + [steps[1]])
    with pytest.raises(ValueError, match="strictly"):
        T.validate_trace(bad, {n: 1 for n in T.MATRIX_NAMES})


# ---------------------------------------------------------------- GPU ---------

@pytest.mark.gpu
class TestModelForwardGPU:
    def test_dense_and_sparse_forward_match_reference(self, toy_model):
        g = golden("toy_model")
        out = T.model_forward_dense(toy_model, g["X"])
        assert rel_err(out, g["out_dense"]) < 1e-5
        cfgs = [T.BlockSparsityConfig({n: 0.5 for n in T.MATRIX_NAMES},
                                      dict(zip(T.MATRIX_NAMES, g[f"thr50_{b}"].tolist()))) for b in range(2)]
        out = T.model_forward_sparse(toy_model, g["X"], cfgs)
        # fp32 on both sides; a channel within an ulp of its threshold may flip
        assert rel_err(out, g["out_sparse50"]) < 1e-4

    def test_zero_config_bit_identical_to_dense(self, toy_model):
        # test_model.py:192-197
        g = golden("toy_model")
        blk = toy_model.blocks[0]
        zero = T.BlockSparsityConfig({n: 0.0 for n in T.MATRIX_NAMES}, {n: 0.0 for n in T.MATRIX_NAMES})
        x = torch.from_numpy(g["X"][:16]).cuda()
        assert torch.equal(T.block_forward_sparse(blk, x, zero), T.block_forward_dense(blk, x))

    def test_full_config_residual_only(self, toy_model):
        # test_model.py:199-203: every input pruned -> output equals input
        blk = toy_model.blocks[0]
        big = T.BlockSparsityConfig({n: 1.0 for n in T.MATRIX_NAMES}, {n: 1e30 for n in T.MATRIX_NAMES})
        x = golden("toy_model")["X"][:8]
        assert np.array_equal(T.block_forward_sparse(blk, x, big), x)

    def test_nonfinite_raises(self, toy_model):
        x = golden("toy_model")["X"][:4].copy()
        x[1, 3] = np.inf
        with pytest.raises(FloatingPointError, match="pre_attn"):
            T.block_forward_dense(toy_model.blocks[0], x)

    def test_calibration_matches_reference(self, toy_model):
        g = golden("toy_model")
        cal = T.RngStream(6).next_generator().standard_normal((10, 128, 512), dtype=np.float32)
        per_block = T.calibrate_model(toy_model, cal)
        for b, taps in enumerate(per_block):
            for tap in TAPS:
                h = taps[T.TapPosition(tap)].histogram
                assert h.total == 10 * 128 * (1408 if tap == "mlp_inter" else 512)
                assert abs(h.hi - float(g[f"hist_{b}_{tap}_hi"])) <= 1e-6 * h.hi
                c, cref = h.counts, g[f"hist_{b}_{tap}_counts"]
                # GPU taps differ from numpy's by ulps; bins shift for a handful of values
                assert np.abs(c - cref).sum() <= 1e-3 * h.total, (b, tap)
            cfg = T.uniform_config(taps, 0.5)
            ref = g[f"thr50_{b}"]
            got = np.array(cfg.as_row())
            assert np.allclose(got, ref, rtol=1e-3), (b, got, ref)

    def test_calibration_counts_bit_exact_at_kernel_boundary(self, toy_model):
        # the same tap values binned by the GPU and by the oracle: identical
        blk = toy_model.blocks[0]
        cal = np.random.default_rng(3).standard_normal((3, 64, 512), dtype=np.float32)
        taps = T.calibrate_block(blk, cal)
        vals = T.tap_activations(blk, cal)
        for pos, tap in taps.items():
            h = tap.histogram
            c, ov = R.hist_record(np.zeros(h.bin_count, np.int64), 0, vals[pos], h.hi)
            assert np.array_equal(h.counts, c) and h.overflow_count == ov, pos
            assert h.hi == 8.0 * float(vals[pos][0].std())

    def test_calibrated_thresholds_realize_level(self, toy_model):
        # test_model.py:326-331: calibrated 50% realizes 0.5 +- 0.01 on the calibration taps
        blk = toy_model.blocks[0]
        cal = np.random.default_rng(4).standard_normal((4, 128, 512), dtype=np.float32)
        taps = T.calibrate_block(blk, cal)
        cfg = T.uniform_config(taps, 0.5)
        vals = T.tap_activations(blk, cal)
        for n in T.MATRIX_NAMES:
            s = T.realized_sparsity(vals[T.MATRIX_TAP[n]].ravel(), cfg.thresholds[n])
            assert abs(s - 0.5) <= 0.01, (n, s)


@pytest.mark.gpu
class TestGreedyGPU:
    def test_trace_matches_reference(self, greedy_block):
        g = golden("greedy")
        cal = np.random.default_rng(32).standard_normal((4, 32, 64), dtype=np.float32)
        taps = T.calibrate_block(greedy_block, cal)
        for tap in TAPS:
            assert abs(taps[T.TapPosition(tap)].histogram.hi - float(g[f"hist_{tap}_hi"])) <= 1e-6
        trace = T.greedy_optimize(greedy_block, taps, cal, T.StepPolicy(0.05))
        chosen = [s.chosen or "-" for s in trace.steps]
        assert chosen == g["chosen"].tolist()
        assert np.array_equal(np.array([s.block_sparsity for s in trace.steps]), g["P"])
        lv = np.array([[s.levels[n] for n in T.MATRIX_NAMES] for s in trace.steps])
        assert np.array_equal(lv, g["levels"])
        err = np.array([s.error for s in trace.steps])
        assert np.allclose(err, g["error"], rtol=1e-4, atol=0)
        T.validate_trace(trace, greedy_block.footprints())

    def test_candidate_sharing_equals_full_forward(self, greedy_block):
        cal = np.random.default_rng(32).standard_normal((4, 32, 64), dtype=np.float32)
        taps = T.calibrate_block(greedy_block, cal)
        trace = T.greedy_optimize(greedy_block, taps, cal, T.StepPolicy(0.2))
        dense = T.block_forward_dense(greedy_block, cal)
        for s in trace.steps[1:4]:
            cfg = T.resolve_config(taps, s.levels)
            err = float(np.sqrt(np.sum(np.square((dense - T.block_forward_sparse(greedy_block, cal, cfg)).astype(np.float64)))))
            assert err == pytest.approx(s.error, rel=1e-12)

    @staticmethod
    def _synthetic_taps():
        # test_greedy.py:34-42: unit-Gaussian histograms for degenerate blocks
        taps = {}
        for pos in T.TapPosition:
            h = T.ActivationHistogram.empty(pos.value, 1024, 8.0)
            h.record(T.sample_gaussian(T.RngStream(sum(map(ord, pos.value)) % 1000), 10**5, 1.0))
            taps[pos] = T.HiddenStateTap(pos, h)
        return taps

    @staticmethod
    def _zeroed(block, names):
        w = dict(block.weights)
        for n in names:
            w[n] = T.Matrix.from_2d(np.zeros((w[n].rows, w[n].cols), np.float32))
        return T.TransformerBlock(block.d_model, block.n_heads, block.d_ff, w, block.rms_attn, block.rms_mlp)

    def test_zero_value_matrix_sparsified_first(self, greedy_block):
        # test_greedy.py:65-79
        cal = np.random.default_rng(32).standard_normal((4, 32, 64), dtype=np.float32)
        trace = T.greedy_optimize(self._zeroed(greedy_block, ["q"]), self._synthetic_taps(), cal, T.StepPolicy(0.05))
        first_cap = next(i for i, s in enumerate(trace.steps) if s.levels["q"] >= 1.0)
        assert trace.steps[first_cap].error == 0.0
        for step in trace.steps[:first_cap + 1]:
            assert all(step.levels[n] == 0.0 for n in T.MATRIX_NAMES if n != "q")
            assert step.chosen in (None, "q")

    def test_tie_break_staircase_on_all_zero_block(self, greedy_block):
        # test_greedy.py:81-101
        cal = np.random.default_rng(32).standard_normal((4, 32, 64), dtype=np.float32)
        blk = self._zeroed(greedy_block, T.MATRIX_NAMES)
        policy = T.StepPolicy(0.05)
        trace = T.greedy_optimize(blk, self._synthetic_taps(), cal, policy)
        fp = blk.footprints()
        total = sum(fp.values())
        expected = []
        for n in T.MATRIX_NAMES:
            expected.extend([n] * int(np.ceil(1.0 / (policy.alpha * total / fp[n]))))
        assert [s.chosen for s in trace.steps[1:]] == expected


@pytest.mark.gpu
def test_sparse_prefill_dense_prefix(toy_model):
    # TEAL's prefill: positions before `dense_prefix` stay dense (attention
    # sinks).  Causality makes those rows identical to the dense forward; the
    # prefix 0 / full-length ends reproduce the sparse / dense forwards.
    g = golden("toy_model")
    thr = [g[f"thr50_{b}"].tolist() for b in range(2)]
    cfgs = [T.BlockSparsityConfig({n: 0.5 for n in T.MATRIX_NAMES}, dict(zip(T.MATRIX_NAMES, t))) for t in thr]
    X = torch.from_numpy(g["X"][:32]).cuda()
    dense = T.model_forward_dense(toy_model, X)
    sparse = T.model_forward_sparse(toy_model, X, cfgs)
    assert torch.equal(T.model_forward_sparse(toy_model, X, cfgs, dense_prefix=0), sparse)
    assert torch.equal(T.model_forward_sparse(toy_model, X, cfgs, dense_prefix=32), dense)
    mixed = T.model_forward_sparse(toy_model, X, cfgs, dense_prefix=12)
    assert torch.equal(mixed[:12], dense[:12])
    assert not torch.equal(mixed[12:], dense[12:]) and not torch.equal(mixed[12:], sparse[12:])
    with pytest.raises(ValueError, match="dense_prefix"):
        T.model_forward_sparse(toy_model, X, cfgs, dense_prefix=-1)


@pytest.mark.gpu
def test_greedy_on_the_gqa_decoder():
    # Algorithm 1 (greedy.py:76-127) on the Llama-style decoder the step
    # engine runs: block inputs from the engine's residual versions, all
    # candidates of a step in one batched forward (identical errors to one
    # forward per candidate), trace invariants, and the greedy 50% config
    # driving the persistent engine
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200 import greedy as G
    spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=41)
    hists = D.calibrate_histograms(W, n_tokens=16, seed=42, engine="step")
    toks = np.random.default_rng(43).integers(0, spec.vocab, 24).tolist()
    X = G.decoder_block_inputs(W, toks)
    pol = G.StepPolicy(0.1)
    tb = G.greedy_decoder_layer(W, 0, X[0], hists, pol, batched=True)
    ts = G.greedy_decoder_layer(W, 0, X[0], hists, pol, batched=False)
    assert [s.chosen for s in tb.steps] == [s.chosen for s in ts.steps]
    # same decisions; errors agree to cuBLAS reduction order (the stacked
    # [C, T, m] GEMM picks another split than the [1, T, m] one, which can
    # move a downstream tap value across its threshold)
    assert np.allclose([s.error for s in tb.steps], [s.error for s in ts.steps], rtol=1e-3)
    fp = {n: a * b for n, (a, b) in spec.proj_shapes().items()}
    G.validate_trace(tb, fp)
    assert tb.steps[-1].block_sparsity >= 1.0 - 1e-12
    # k / v jump 0 -> 1 in one step at GQA footprints (delta > 1, clamped)
    kv_steps = [s for s in tb.steps if s.chosen in ("k", "v")]
    assert all(s.levels[s.chosen] == 1.0 for s in kv_steps)
    traces = [tb, G.greedy_decoder_layer(W, 1, X[1], hists, pol)]
    thr = G.decoder_greedy_thresholds(traces, hists, 0.5)
    dec = E.StepDecoder(W, thr, count_kept=True)
    dec.reset()
    for t in toks[:4]:
        dec.token.fill_(t)
        dec.step_token()
    torch.cuda.synchronize()
    assert int(dec.kept.sum()) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("level", [0.0, 0.5, 0.9])
def test_cats_output_sparse_gemv(dtype, level):
    # CATS (model.py:331-341): out[j] = gate[j] * (x . W_up[j]) where |gate_j|
    # > fl32(t); only kept rows are read.  Mask bit-exact vs the oracle's
    # keep_mask of the gate, values vs torch (fp32 rows: 1e-5; bf16: same
    # bf16 weights on both sides)
    import paper_2408_14690_b200 as T
    from paper_2408_14690_b200.model import cats_gemv
    g = torch.Generator(device="cuda").manual_seed(5)
    n, m = 14336, 4096
    w = torch.randn(n, m, device="cuda", generator=g) / m ** 0.5
    if dtype == "bf16":
        w = w.to(torch.bfloat16)
    x = torch.randn(m, device="cuda", generator=g)
    gl = torch.randn(n, device="cuda", generator=g)
    gate = gl / (1 + torch.exp(-gl))
    t = float(torch.quantile(gate.abs(), level)) if level > 0 else 0.0
    bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    kept = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = cats_gemv(w, x, gate, t, kept=kept, keep_bits=bits)
    keep = R.keep_mask(gate.cpu().numpy(), t)
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), R.pack_bits(keep))
    assert int(kept.item()) == int(keep.sum())
    want = torch.where(torch.from_numpy(keep).cuda(), gate * (w.float() @ x), torch.zeros_like(gate))
    assert rel_err(out.cpu().numpy(), want.cpu().numpy()) < 1e-5


@pytest.mark.gpu
def test_cats_mlp_decode_matches_reference_semantics():
    from paper_2408_14690_b200.model import cats_mlp_decode
    g = torch.Generator(device="cuda").manual_seed(6)
    d, f = 1024, 2816
    wg = torch.randn(d, f, device="cuda", generator=g) / d ** 0.5
    wu = torch.randn(f, d, device="cuda", generator=g) / d ** 0.5   # row-major W_up
    wd = torch.randn(f, d, device="cuda", generator=g) / f ** 0.5   # input-major W_down
    h = torch.randn(d, device="cuda", generator=g)
    gate = (h @ wg) / (1 + torch.exp(-(h @ wg)))
    t = float(torch.quantile(gate.abs(), 0.5))
    out = cats_mlp_decode(wg, wu, wd, h, t)
    assert not torch.backends.cuda.matmul.allow_tf32  # true fp32 reference GEMVs
    masked = torch.where(gate.abs() <= float(np.float32(t)), torch.zeros_like(gate), gate)
    want = (masked * (wu @ h)) @ wd
    assert rel_err(out.cpu().numpy(), want.cpu().numpy()) < 1e-4
