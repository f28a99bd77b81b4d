"""Write the reference's own wire-format files as fixtures.

Run in the build container, where the reference is importable:

    python tests/golden/make_interop.py

The REAL reference (``actsparse`` 0.1.0, imported from a scratch copy of
/root/reference/pkg/src exactly as make_golden.py does) generates a small
model, calibrates it, runs its greedy search and writes every file format
the CLI exchanges — through its own writers:

  model.teal     TEALM1  model.save_model        (pkg/src/actsparse/model.py:436-474)
  matrix.teal    TEALW1  tensor.save_matrix      (tensor.py:197-235)
  hist_*.txt     TEALH1  sparsifier.save_histogram (sparsifier.py:189-219)
  trace.txt      TEALG1  greedy.save_trace       (greedy.py:200-237)
  configs.txt    TEALC1  greedy.save_configs     (greedy.py:239-271)

plus ``expect.npz``: what the reference computes from those files (the
thresholds of every loaded histogram on a p grid, the uniform / greedy
configs' thresholds, and model_forward_sparse rows of the loaded model under
the loaded configs), so the tests can load the reference-written files into
this package, re-write them byte for byte, and drive the GPU path with them.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "interop"
sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import _import_reference  # noqa: E402


def main() -> None:
    A = _import_reference()
    from actsparse import greedy as G
    from actsparse import model as M
    from actsparse import sparsifier as S
    from actsparse import tensor as TT

    OUT.mkdir(exist_ok=True)
    exp = {}
    # a small model (2 blocks, d 64, 4 heads, d_ff 176), its files and forward
    model = A.gen_model(A.RngStream(11), 2, 64, 4, 176)
    M.save_model(OUT / "model.teal", model)
    w = TT.Matrix.from_2d(np.random.default_rng(12).standard_normal((5, 7), dtype=np.float32), TT.Layout.COL_MAJOR)
    TT.save_matrix(OUT / "matrix.teal", w)
    exp["matrix"] = w.to_2d()
    cal = A.RngStream(13).next_generator().standard_normal((4, 32, 64), dtype=np.float32)
    per_block = A.calibrate_model(model, cal)
    grid = np.linspace(0.0, 1.0, 21)
    names = []
    for b, taps in enumerate(per_block):
        for pos, tap in taps.items():
            fn = f"hist_{b}_{pos.value}.txt"
            S.save_histogram(OUT / fn, tap.histogram)
            names.append(fn)
            exp[f"thr_{fn}"] = np.array([tap.histogram.threshold(float(p)) for p in grid])
    exp["p_grid"] = grid
    # greedy on block 0 (alpha 0.1), the 50% greedy config of block 0 and a
    # uniform 40% config of block 1 -> one TEALC1 file
    trace = A.greedy_optimize(model.blocks[0], per_block[0], cal, A.StepPolicy(0.1))
    G.save_trace(OUT / "trace.txt", trace)
    cfg0 = A.select_config(trace, 0.5, per_block[0])
    cfg1 = A.uniform_config(per_block[1], 0.4)
    G.save_configs(OUT / "configs.txt", [cfg0, cfg1], 0.5)
    exp["cfg_thresholds"] = np.array([[c.thresholds[n] for n in M.MATRIX_NAMES] for c in (cfg0, cfg1)])
    exp["cfg_levels"] = np.array([[c.levels[n] for n in M.MATRIX_NAMES] for c in (cfg0, cfg1)])
    X = A.RngStream(14).next_generator().standard_normal((12, 64), dtype=np.float32)
    exp["X"] = X
    exp["out_sparse"] = A.model_forward_sparse(model, X, [cfg0, cfg1])
    exp["out_dense"] = A.model_forward_dense(model, X)
    exp["trace_P"] = np.array([s.block_sparsity for s in trace.steps])
    # a one-block model whose shapes the persistent step engine tiles (d and
    # n_q multiples of 256, head_dim 64 | 128, d_ff multiple of 128), with its
    # own calibration and configs file, for driving the step engine
    m2 = A.gen_model(A.RngStream(21), 1, 256, 4, 256)
    M.save_model(OUT / "model256.teal", m2)
    cal2 = A.RngStream(22).next_generator().standard_normal((4, 32, 256), dtype=np.float32)
    taps2 = A.calibrate_model(m2, cal2)[0]
    c2 = A.uniform_config(taps2, 0.5)
    G.save_configs(OUT / "configs256.txt", [c2], 0.5)
    X2 = A.RngStream(23).next_generator().standard_normal((12, 256), dtype=np.float32)
    exp["X256"] = X2
    exp["out256_sparse"] = A.model_forward_sparse(m2, X2, [c2])
    np.savez_compressed(OUT / "expect.npz", **exp)
    (OUT / "manifest.json").write_text(json.dumps(
        {"reference": "actsparse " + A.__version__, "histograms": names,
         "files": ["model.teal", "matrix.teal", "trace.txt", "configs.txt", "model256.teal", "configs256.txt"]
         + names}, indent=1) + "\n")
    print("interop fixtures written to", OUT)


if __name__ == "__main__":
    main()
