"""Generate the golden fixtures that pin the oracle (and, through it, the GPU
path) to the REAL reference implementation.

Run in the build container, where the reference is available:

    python tests/golden/make_golden.py

It imports ``actsparse`` 0.1.0 from a scratch copy of
``/root/reference/pkg/src`` (numba's on-disk cache would otherwise write into
the read-only reference tree) and records the reference's outputs on seeded
inputs that the tests regenerate with ``np.random.default_rng(seed)`` — so
only small outputs (or SHA-256 digests of exact outputs) are committed.
Inputs/seeds follow the reference's own tests:
  pkg/tests/test_kernel.py:35-91, pkg/tests/test_acceptance.py:173-248,
  pkg/tests/test_sparsifier.py:32-225, pkg/tests/test_model.py:191-331,
  pkg/tests/test_greedy.py:57-127.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")


def _import_reference():
    scratch = Path(tempfile.mkdtemp(prefix="actsparse_ref_"))
    shutil.copytree(REF_SRC / "actsparse", scratch / "actsparse")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(scratch / "numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(scratch))
    import actsparse  # noqa: E402
    return actsparse


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    A = _import_reference()
    from actsparse import model as M

    meta = {"reference": "actsparse " + A.__version__, "numpy": np.__version__}

    # --- kernel: test_kernel.py:47-56 oracle-equivalence grid (25 seeds, 64x96)
    kern = {}
    ys, macs, ts = [], [], []
    for seed in range(25):
        g = np.random.default_rng(1000 + seed)
        x = g.standard_normal(96, dtype=np.float32)
        arr = g.standard_normal((64, 96), dtype=np.float32)
        t = float(g.uniform(0.0, 2.0))
        w = A.Matrix.from_2d(arr, A.Layout.COL_MAJOR)
        y, mc = A.sparse_gemv(x, t, w, count_macs=True)
        ys.append(y)
        macs.append(mc)
        ts.append(t)
    kern["grid25_y"] = np.stack(ys)
    kern["grid25_macs"] = np.array(macs, dtype=np.int64)
    kern["grid25_t"] = np.array(ts)

    # --- acceptance criterion 6 (test_acceptance.py:173-192): exact digests
    def crit6(seed, n, m):
        g = np.random.default_rng(seed)
        x = g.standard_normal(m, dtype=np.float32)
        w = A.Matrix(n, m, A.Layout.COL_MAJOR, g.standard_normal(n * m, dtype=np.float32))
        t = float(g.uniform(0.0, 1.5))
        y, mc = A.sparse_gemv(x, t, w, count_macs=True)
        ref = A.matmul_dense(A.sparsify(x, t), w)
        return sha(y), sha(ref), mc, t, float(np.sum(y, dtype=np.float64))

    c6 = {"small": [], "large": []}
    for seed in range(1000):
        c6["small"].append(crit6(seed, 256, 256))
    for seed in range(100):
        c6["large"].append(crit6(10_000 + seed, 1024, 4096))

    # --- sparsify / realized / batched KATs
    sp = {}
    g = np.random.default_rng(7)
    xs = g.standard_normal((16, 257), dtype=np.float32) * 2
    xs[0, :4] = [0.1, -0.5, 2.0, -0.05]
    t_grid = [0.0, 0.2, 0.3, 0.5, 0.6744897501960817, 1.0, 1.5, 3.0]
    sp["x"] = xs
    sp["t"] = np.array(t_grid)
    sp["sparsify_sha"] = np.array([[sha(A.sparsify(xs[r], t)) for t in t_grid] for r in range(16)])
    sp["realized"] = np.array([[A.realized_sparsity(xs[r], t) for t in t_grid] for r in range(16)])
    # tie exactly at fl32(0.3): sparsify prunes, sparse_gemv (fp64 compare) keeps
    tie = np.array([np.float32(0.3), 0.1, -np.float32(0.3), 2.0], dtype=np.float32)
    sp["tie_x"] = tie
    sp["tie_sparsify"] = A.sparsify(tie, 0.3)
    _, tie_macs = A.sparse_gemv(tie, 0.3, A.Matrix.from_2d(np.ones((3, 4), np.float32), A.Layout.COL_MAJOR), count_macs=True)
    sp["tie_gemv_macs"] = np.int64(tie_macs)
    bm, bsha = [], []
    for seed in range(20):
        gg = np.random.default_rng(40_000 + seed)
        B = 1 + seed % 7
        xb = gg.standard_normal((B, 300), dtype=np.float32)
        t = float(gg.uniform(0.0, 1.5))
        out, mask = A.sparsify_batched(xb, t)
        bm.append(np.packbits(mask))
        bsha.append(sha(out))
    sp["batched_maskbits"] = np.stack(bm)
    sp["batched_sha"] = np.array(bsha)

    # --- histogram (test_sparsifier.py:26-30 gaussian_hist) + thresholds
    hist = {}
    for seed, n in ((0, 10**6), (1, 10**6), (15, 10**5)):
        h = A.ActivationHistogram.empty("g", 4096, 8.0)
        h.record(A.sample_gaussian(A.RngStream(seed), n, 1.0))
        hist[f"counts_{seed}"] = h.counts.copy()
        hist[f"overflow_{seed}"] = np.int64(h.overflow_count)
        grid = np.linspace(0.0, 1.0, 41)
        hist[f"thr_{seed}"] = np.array([h.threshold(float(p)) for p in grid])
    hist["p_grid"] = np.linspace(0.0, 1.0, 41)
    # odd hi / bins / overflow and boundary values
    gg = np.random.default_rng(99)
    vals = (gg.standard_normal(50_000) * 1.7).astype(np.float32)
    vals[:5] = [0.0, 1.25, -1.25, 2.5, 2.5000002]
    h = A.ActivationHistogram.empty("odd", 777, 1.25)
    h.record(vals)
    hist["odd_vals"] = vals
    hist["odd_counts"] = h.counts.copy()
    hist["odd_overflow"] = np.int64(h.overflow_count)
    hist["odd_thr"] = np.array([h.threshold(float(p)) for p in np.linspace(0, 1, 41)])

    # --- theory
    th = {"p": np.array([0.0, 0.1, 0.25, 0.4, 0.5, 0.65, 0.9, 0.99]),}
    th["t"] = np.array([A.gaussian_threshold(float(p)) for p in th["p"]])

    # --- toy model config 1 (d=512, ffn=1408, 8 heads, 2 blocks) + default blocks
    model = A.gen_model(A.RngStream(5), 2, 512, 8, 1408)
    toy = {}
    for b, blk in enumerate(model.blocks):
        for n in M.MATRIX_NAMES:
            toy[f"w_sha_{b}_{n}"] = np.array(sha(blk.weights[n].to_2d()))
    cal = A.RngStream(6).next_generator().standard_normal((10, 128, 512), dtype=np.float32)
    per_block = A.calibrate_model(model, cal)
    cfgs = [A.uniform_config(taps, 0.5) for taps in per_block]
    for b, taps in enumerate(per_block):
        for pos, tap in taps.items():
            toy[f"hist_{b}_{pos.value}_counts"] = tap.histogram.counts.copy()
            toy[f"hist_{b}_{pos.value}_hi"] = np.float64(tap.histogram.hi)
            toy[f"hist_{b}_{pos.value}_overflow"] = np.int64(tap.histogram.overflow_count)
        toy[f"thr50_{b}"] = np.array([cfgs[b].thresholds[n] for n in M.MATRIX_NAMES])
    X = A.RngStream(7).next_generator().standard_normal((48, 512), dtype=np.float32)
    toy["X"] = X
    toy["out_sparse50"] = A.model_forward_sparse(model, X, cfgs)
    toy["out_dense"] = A.model_forward_dense(model, X)
    blk0 = A.gen_block(A.RngStream(2024), 256, 4, 704)
    toy["w_sha_default_q"] = np.array(sha(blk0.weights["q"].to_2d()))

    # --- greedy trace (test_greedy.py:57-62 small_setup, alpha 0.05)
    block = A.gen_block(A.RngStream(31), 64, 2, 176)
    calg = np.random.default_rng(32).standard_normal((4, 32, 64), dtype=np.float32)
    taps = A.calibrate_block(block, calg)
    trace = A.greedy_optimize(block, taps, calg, A.StepPolicy(0.05))
    gr = {
        "P": np.array([s.block_sparsity for s in trace.steps]),
        "levels": np.array([[s.levels[n] for n in M.MATRIX_NAMES] for s in trace.steps]),
        "chosen": np.array([s.chosen or "-" for s in trace.steps]),
        "error": np.array([s.error for s in trace.steps]),
    }
    for pos, tap in taps.items():
        gr[f"hist_{pos.value}_counts"] = tap.histogram.counts.copy()
        gr[f"hist_{pos.value}_hi"] = np.float64(tap.histogram.hi)

    np.savez_compressed(OUT / "kernel.npz", **kern)
    np.savez_compressed(OUT / "sparsify.npz", **sp)
    np.savez_compressed(OUT / "histogram.npz", **hist)
    np.savez_compressed(OUT / "theory.npz", **th)
    np.savez_compressed(OUT / "toy_model.npz", **toy)
    np.savez_compressed(OUT / "greedy.npz", **gr)
    (OUT / "crit6.json").write_text(json.dumps(c6))
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
