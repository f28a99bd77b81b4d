"""GPU: batched shared-mask sparse GEMV over bf16 / int8 / int4 rows
(BASELINE config 5; quant.sparse_gemv_batched -> teal_gemv_batched).

Pinned to the reference's `sparsify_batched` (sparsifier.py:136-155): the
shared column mask is bit-exact against the oracle and the golden batched
fixtures; outputs equal the oracle's sparsify_batched(X, t) @ W_deq^T on the
kernel's own dequantised weights within fp32 rounding (rel 1e-5; the int4 /
int8 / bf16 values are exact fp32 numbers, only summation order differs).
Quantisation error itself is reported, not bounded (parity unpinned for
quantised weights).
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden, rel_err
from oracle import actsparse_ref as R

pytestmark = pytest.mark.gpu


def _case(seed, B, m, n):
    g = np.random.default_rng(seed)
    return g.standard_normal((B, m), dtype=np.float32), g.standard_normal((m, n), dtype=np.float32) / np.sqrt(m)


@pytest.mark.parametrize("kind", ["bf16", "int8", "int4"])
@pytest.mark.parametrize("B", [1, 2, 3, 4, 8, 13, 16])
def test_matches_oracle(kind, B):
    from paper_2408_14690_b200 import quant as Q
    m, n = 1024, 768
    xs, w = _case(100 + B, B, m, n)
    wt = torch.from_numpy(w).cuda()
    qw = {"bf16": Q.as_bf16, "int8": Q.quantize_int8, "int4": lambda a: Q.quantize_int4(a, 128)}[kind](wt)
    wd = qw.dequantize().cpu().numpy()
    for t in (0.0, 0.3, 0.6745, 1.2):
        y, mask = Q.sparse_gemv_batched(xs, t, qw, return_mask=True)
        xs_s, mref = R.sparsify_batched(xs, t)
        assert np.array_equal(mask, mref), (kind, B, t)
        ref = xs_s.astype(np.float64) @ wd.astype(np.float64)
        assert rel_err(y, ref) < 1e-5, (kind, B, t, rel_err(y, ref))


@pytest.mark.parametrize("kind", ["bf16", "int8", "int4"])
@pytest.mark.parametrize("B", [4, 13, 16])
def test_mma_path_wide_ragged(kind, B):
    """The tensor-core variant (bf16 / int8 / int4-group-128 rows, B >= 4):
    ragged m (partial 128-row chunk, 32-row group and int4 scale group) and
    a partial last 256-column tile (n = 4112; 4128 for int4, whose MMA path
    needs n % 32 == 0), against the float64 product of the kernel's own
    dequantised weights at the fp32 bar (rel 1e-5)."""
    from paper_2408_14690_b200 import quant as Q
    m, n = 1000, (4128 if kind == "int4" else 4112)
    xs, w = _case(700 + B, B, m, n)
    qw = {"bf16": Q.as_bf16, "int8": Q.quantize_int8,
          "int4": lambda a: Q.quantize_int4(a, 128)}[kind](torch.from_numpy(w).cuda())
    wd = qw.dequantize().cpu().numpy().astype(np.float64)
    for t in (0.0, 0.6745, 1.5):
        y, mask = Q.sparse_gemv_batched(xs, t, qw, return_mask=True)
        xs_s, mref = R.sparsify_batched(xs, t)
        assert np.array_equal(mask, mref), (kind, B, t)
        assert rel_err(y, xs_s.astype(np.float64) @ wd) < 1e-5, (kind, B, t)


@pytest.mark.parametrize("kind", ["bf16", "int8", "int4"])
def test_config5_full_shape(kind):
    """BASELINE config 5 at its real size: Mistral-7B gate 4096 x 14336,
    B = 16, threshold at the 50 % quantile of the batch-mean magnitude.
    Mask bit-exact against the oracle's sparsify_batched; product against a
    float64 product of the dequantised weights (on the device) at rel 1e-5."""
    from paper_2408_14690_b200 import quant as Q
    m, n, B = 4096, 14336, 16
    g = torch.Generator(device="cuda").manual_seed(55)
    x = torch.randn(B, m, device="cuda", generator=g)
    w = torch.randn(m, n, device="cuda", generator=g) / math.sqrt(m)
    qw = {"bf16": Q.as_bf16, "int8": Q.quantize_int8, "int4": lambda a: Q.quantize_int4(a, 128)}[kind](w)
    t = float(torch.quantile(x.abs().mean(0), 0.5))
    y, mask = Q.sparse_gemv_batched(x, t, qw, return_mask=True)
    xs_s, mref = R.sparsify_batched(x.cpu().numpy(), t)
    assert np.array_equal(mask.cpu().numpy(), mref)
    assert 0.45 < float(mref.mean()) < 0.55
    ref = torch.from_numpy(xs_s).cuda().double() @ qw.dequantize().double()
    assert rel_err(y.cpu().numpy(), ref.cpu().numpy()) < 1e-5, kind


def test_dense_and_all_pruned():
    from paper_2408_14690_b200 import quant as Q
    xs, w = _case(7, 4, 512, 256)
    qw = Q.quantize_int8(torch.from_numpy(w).cuda())
    y = Q.sparse_gemv_batched(xs, None, qw)
    assert rel_err(y, xs.astype(np.float64) @ qw.dequantize().cpu().numpy()) < 1e-5
    y = Q.sparse_gemv_batched(xs, 1e9, qw)
    assert np.all(y == 0)


def test_batch1_equals_single_row_sparsify():
    # B = 1 shared mask == sparsify (test_acceptance.py:216-221)
    from paper_2408_14690_b200 import quant as Q
    xs, w = _case(9, 1, 2048, 512)
    qw = Q.as_bf16(torch.from_numpy(w).cuda())
    y, mask = Q.sparse_gemv_batched(xs, 0.5, qw, return_mask=True)
    assert np.array_equal(~mask, R.keep_mask(xs[0], 0.5))


@pytest.mark.parametrize("kind", ["bf16", "int8"])
def test_batch1_single_row_route(kind):
    """B = 1 without a mask request runs the single-row kernel: same kept
    count as the batched kernel (mask identical by construction) and the
    same product at the fp32 bar."""
    from paper_2408_14690_b200 import quant as Q
    xs, w = _case(31, 1, 1536, 1280)
    qw = {"bf16": Q.as_bf16, "int8": Q.quantize_int8}[kind](torch.from_numpy(w).cuda())
    wd = qw.dequantize().cpu().numpy().astype(np.float64)
    for t in (0.0, 0.6745, 2.0):
        k1 = torch.zeros(1, dtype=torch.int64, device="cuda")
        y = Q.sparse_gemv_batched(xs, t, qw, kept=k1)
        yb, mask = Q.sparse_gemv_batched(xs, t, qw, return_mask=True)
        xs_s, mref = R.sparsify_batched(xs, t)
        assert int(k1.item()) == int((~mref).sum()), (kind, t)
        assert rel_err(y, xs_s.astype(np.float64) @ wd) < 1e-5, (kind, t)
        assert rel_err(y, yb) < 1e-5, (kind, t)


def test_golden_batched_masks():
    # masks of the real reference's sparsify_batched on seeds 40000+s
    from paper_2408_14690_b200 import quant as Q
    g = golden("sparsify")
    for seed in range(20):
        gg = np.random.default_rng(40_000 + seed)
        B = 1 + seed % 7
        xb = gg.standard_normal((B, 300), dtype=np.float32)
        t = float(gg.uniform(0.0, 1.5))
        qw = Q.as_bf16(torch.randn(300, 64, device="cuda"))
        _, mask = Q.sparse_gemv_batched(xb, t, qw, return_mask=True)
        assert np.array_equal(np.packbits(mask), g["batched_maskbits"][seed]), seed


def test_kept_count_and_validation():
    from paper_2408_14690_b200 import quant as Q
    xs, w = _case(11, 2, 640, 128)
    qw = Q.quantize_int4(torch.from_numpy(w).cuda(), 64)
    kept = torch.zeros(1, dtype=torch.int64, device="cuda")
    _, mask = Q.sparse_gemv_batched(xs, 0.4, qw, return_mask=True, kept=kept)
    assert int(kept.item()) == int((~mask).sum())
    with pytest.raises(ValueError, match="mismatch"):
        Q.sparse_gemv_batched(xs[:, :320], 0.4, qw)
    with pytest.raises(ValueError, match="B <= 16"):
        Q.sparse_gemv_batched(np.zeros((17, 640), np.float32), 0.4, qw)


def test_quantisation_roundtrip_error_small():
    from paper_2408_14690_b200 import quant as Q
    w = torch.randn(1024, 512, device="cuda")
    for q, tol in ((Q.quantize_int8(w), 0.01), (Q.quantize_int4(w, 128), 0.12)):
        err = (q.dequantize() - w).norm() / w.norm()
        assert float(err) < tol


@pytest.mark.parametrize("B", [4, 7, 13, 16])
def test_tcgen05_path_ragged(B):
    """The tcgen05 route (bf16, B >= 4, n >= 64 * 128): compaction of a ragged
    m (a partial 1024-column chunk), padded K blocks, deterministic split K,
    dense (t None) and all-pruned thresholds; mask bit-exact, product at the
    fp32 bar (bf16 hi + lo activations: rel 1e-5) against float64, kept count
    = the oracle's, and identical bits on a repeat."""
    from paper_2408_14690_b200 import quant as Q
    m, n = 3000, 8192
    xs, w = _case(900 + B, B, m, n)
    qw = Q.as_bf16(torch.from_numpy(w).cuda())
    wd = qw.dequantize().cpu().numpy().astype(np.float64)
    for t in (None, 0.0, 0.6745, 1.5, 1e9):
        kept = torch.zeros(1, dtype=torch.int64, device="cuda")
        y, mask = Q.sparse_gemv_batched(xs, t, qw, return_mask=True, kept=kept)
        y2 = Q.sparse_gemv_batched(xs, t, qw)
        assert np.array_equal(np.asarray(y), np.asarray(y2)), (B, t)
        xs_s, mref = (xs, np.zeros(m, np.uint8)) if t is None else R.sparsify_batched(xs, t)
        assert np.array_equal(mask, mref), (B, t)
        assert int(kept.item()) == int((~mref.astype(bool)).sum()), (B, t)
        ref = xs_s.astype(np.float64) @ wd
        if t == 1e9:
            assert np.all(np.asarray(y) == 0)
        else:
            assert rel_err(y, ref) < 1e-5, (B, t, rel_err(y, ref))
