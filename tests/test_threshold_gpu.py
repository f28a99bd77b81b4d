"""GPU parity of thresholding, batched shared masks and histogram calibration
against the reference's golden vectors (bit-exact).  Mirrors
pkg/tests/test_sparsifier.py:32-225 and test_acceptance.py:215-248."""

from __future__ import annotations

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.extra import numpy as hnp

from conftest import golden, sha
from oracle import actsparse_ref as R

pytestmark = pytest.mark.gpu
finite_f32 = st.floats(-100.0, 100.0, allow_nan=False, width=32)


@pytest.fixture(scope="module")
def T():
    import paper_2408_14690_b200 as T
    return T


class TestSparsify:
    def test_reference_digests(self, T):
        g = golden("sparsify")
        for r in range(g["x"].shape[0]):
            for k, t in enumerate(g["t"]):
                assert sha(T.sparsify(g["x"][r], float(t))) == g["sparsify_sha"][r, k]
                assert T.realized_sparsity(g["x"][r], float(t)) == g["realized"][r, k]

    def test_direct_definition(self, T):
        x = np.array([0.1, -0.5, 2.0, -0.05], dtype=np.float32)
        assert T.sparsify(x, 0.2).tolist() == [0.0, -0.5, 2.0, 0.0]
        z = np.array([0.1, -0.5, 0.0], np.float32)
        assert T.sparsify(z, 0.0).tobytes() == z.tobytes()

    def test_tie_prunes_at_fl32_threshold(self, T):
        g = golden("sparsify")
        assert T.sparsify(g["tie_x"], 0.3).tobytes() == g["tie_sparsify"].tobytes()

    def test_nan_kept_neg_zero_positive(self, T):
        out = T.sparsify(np.array([np.nan, -0.0, -0.1, 4.0], np.float32), 0.5)
        assert np.isnan(out[0]) and out.view(np.uint32)[1:3].tolist() == [0, 0] and out[3] == 4.0

    def test_realized_boundary_and_empty(self, T):
        assert T.realized_sparsity([1.0, 2.0, 3.0], 3.0) == 1.0
        # the reference does not validate t: a negative or NaN t prunes nothing
        for t in (-0.5, float("nan")):
            assert T.realized_sparsity([0.0, -0.5, 2.0], t) == R.realized_sparsity([0.0, -0.5, 2.0], t) == 0.0
        assert T.realized_sparsity([0.1, -0.5, 2.0, -0.05], 0.2) == 0.5
        with pytest.raises(ValueError):
            T.realized_sparsity([], 0.1)

    def test_negative_threshold_rejected(self, T):
        with pytest.raises(ValueError):
            T.sparsify(np.ones(3, np.float32), -1.0)

    @given(hnp.arrays(np.float32, st.integers(1, 300), elements=finite_f32), st.floats(0.0, 10.0))
    @settings(max_examples=60, deadline=None)
    def test_matches_oracle_and_idempotent(self, T, x, t):
        once = T.sparsify(x, t)
        assert once.tobytes() == R.sparsify(x, t).tobytes()
        assert T.sparsify(once, t).tobytes() == once.tobytes()

    def test_bitmask_and_bf16(self, T, cuda_device):
        rng = np.random.default_rng(3)
        x = rng.standard_normal(10_007, dtype=np.float32)
        for t in (0.0, 0.3, 0.6744897501960817, 2.0):
            bits, pruned = T.threshold_bits(torch.from_numpy(x).to(cuda_device), t)
            assert np.array_equal(bits.cpu().numpy().view(np.uint32), R.pack_bits(R.keep_mask(x, t)))
            assert int(pruned.item()) == int((~R.keep_mask(x, t)).sum())
        xb = torch.from_numpy(x).to(torch.bfloat16)
        out = T.sparsify(xb.to(cuda_device), 0.5)
        assert out.dtype == torch.bfloat16
        assert np.array_equal(out.float().cpu().numpy(), R.sparsify(xb.float().numpy(), 0.5))


class TestBatched:
    def test_reference_masks(self, T):
        g = golden("sparsify")
        for seed in range(20):
            gg = np.random.default_rng(40_000 + seed)
            B = 1 + seed % 7
            xb = gg.standard_normal((B, 300), dtype=np.float32)
            t = float(gg.uniform(0.0, 1.5))
            out, mask = T.sparsify_batched(xb, t)
            assert np.array_equal(np.packbits(mask), g["batched_maskbits"][seed])
            assert sha(out) == g["batched_sha"][seed]

    def test_b1_reduces_to_sparsify_1000_cases(self, T):
        for seed in range(0, 1000, 10):
            g = np.random.default_rng(40_000 + seed)
            x = g.standard_normal(64, dtype=np.float32)
            t = float(g.uniform(0.0, 1.5))
            batched, _ = T.sparsify_batched(x[None, :], t)
            assert batched[0].tobytes() == R.sparsify(x, t).tobytes()

    def test_mean_magnitude_mask_and_ragged(self, T):
        b, mask = T.sparsify_batched(np.array([[1.0, 0.1], [-1.0, 0.1]], np.float32), 0.5)
        assert mask.tolist() == [False, True] and b[:, 1].tolist() == [0.0, 0.0]
        with pytest.raises(ValueError, match="ragged|length"):
            T.sparsify_batched([[1.0, 2.0], [1.0]], 0.5)

    def test_calibrated_column_sparsity(self, T):
        # test_acceptance.py:223-239 on the GPU histogram + batched mask
        m = 4096
        for bsz in (2, 4, 8):
            hist = T.ActivationHistogram.empty(f"braw{bsz}", 4096, 4.0)
            cal = T.RngStream(42_000 + bsz)
            for _ in range(64):
                xs = T.sample_gaussian(cal, bsz * m, 1.0).reshape(bsz, m)
                hist.record(np.abs(xs).mean(axis=0))
            t = hist.threshold(0.5)
            fresh = T.sample_gaussian(T.RngStream(43_000 + bsz), bsz * m, 1.0).reshape(bsz, m)
            _, mask = T.sparsify_batched(fresh, t)
            assert abs(float(mask.mean()) - 0.5) <= 0.05


class TestHistogram:
    @pytest.mark.parametrize("seed,n", [(0, 10**6), (1, 10**6), (15, 10**5)])
    def test_counts_and_thresholds_bit_exact(self, T, seed, n):
        g = golden("histogram")
        h = T.ActivationHistogram.empty("g", 4096, 8.0)
        h.record(T.sample_gaussian(T.RngStream(seed), n, 1.0))
        assert np.array_equal(h.counts, g[f"counts_{seed}"])
        assert h.overflow_count == int(g[f"overflow_{seed}"]) and h.total == n
        assert h.thresholds(g["p_grid"]) == g[f"thr_{seed}"].tolist()

    def test_odd_binning_boundaries(self, T):
        g = golden("histogram")
        h = T.ActivationHistogram.empty("odd", 777, 1.25)
        h.record(g["odd_vals"])
        assert np.array_equal(h.counts, g["odd_counts"]) and h.overflow_count == int(g["odd_overflow"])
        assert h.thresholds(np.linspace(0, 1, 41)) == g["odd_thr"].tolist()

    def test_direct_binning_and_overflow(self, T):
        h = T.ActivationHistogram.empty("t", 2, 1.0)
        h.record(np.array([0.5, -0.5], dtype=np.float32))
        assert h.counts.tolist() == [0, 2] and h.total == 2 and h.overflow_count == 0
        h = T.ActivationHistogram.empty("t", 4, 1.0)
        h.record(np.array([0.5, 2.0, 1.0], dtype=np.float32))
        assert h.overflow_count == 1 and h.total == 3 and h.counts.sum() == 2

    def test_float64_input_binned_unrounded(self, T):
        # values within fp32 rounding of bin edges and of hi: the reference
        # bins np.asarray(x, float64) (sparsifier.py:75-80) — an fp32 upload
        # would move them across edges
        bins, hi = 1000, 1.0
        edges = np.arange(1, bins, dtype=np.float64) / bins
        xs = np.concatenate([edges - 1e-12, edges + 1e-12, [hi, hi + 1e-12, hi - 1e-12], -edges[:50] - 1e-13])
        h = T.ActivationHistogram.empty("f64", bins, hi)
        h.record(xs)
        cnt, ov = np.zeros(bins, np.int64), 0
        cnt, ov = R.hist_record(cnt, ov, xs, hi)
        assert np.array_equal(h.counts, cnt) and h.overflow_count == ov and h.total == xs.size
        import torch
        h2 = T.ActivationHistogram.empty("f64d", bins, hi)
        h2.record(torch.from_numpy(xs).cuda())
        assert np.array_equal(h2.counts, cnt) and h2.overflow_count == ov

    def test_nan_rejected_without_mutation(self, T):
        h = T.ActivationHistogram.empty("t", 4, 1.0)
        h.record(np.array([0.1], np.float32))
        with pytest.raises(ValueError, match="NaN"):
            h.record(np.array([0.1, np.nan], dtype=np.float32))
        assert h.total == 1 and h.counts.sum() == 1

    def test_empty_and_bounds(self, T):
        h = T.ActivationHistogram.empty("t", 4, 1.0)
        h.record(np.array([], np.float32))
        assert h.total == 0
        with pytest.raises(ValueError, match="empty"):
            h.threshold(0.5)
        h.record(np.ones(3, np.float32))
        assert h.threshold(0.0) == 0.0 and h.threshold(1.0) == 1.0

    def test_merge(self, T):
        a = T.ActivationHistogram.empty("a", 4096, 8.0).record(T.sample_gaussian(T.RngStream(12), 10**4, 1.0))
        b = T.ActivationHistogram.empty("b", 4096, 8.0).record(T.sample_gaussian(T.RngStream(13), 10**4, 1.0))
        ca = a.counts
        a.merge(b)
        assert a.total == 2 * 10**4 and np.array_equal(a.counts, ca + b.counts)
        with pytest.raises(ValueError, match="binning"):
            a.merge(T.ActivationHistogram.empty("t", 4096, 4.0))

    def test_bf16_record(self, T, cuda_device):
        x = torch.randn(100_000, generator=torch.Generator().manual_seed(0)).to(torch.bfloat16)
        h = T.ActivationHistogram.empty("b", 512, 5.0)
        h.record(x.to(cuda_device))
        counts, ov = R.hist_record(np.zeros(512, np.int64), 0, x.float().numpy(), 5.0)
        assert np.array_equal(h.counts, counts) and h.overflow_count == ov
