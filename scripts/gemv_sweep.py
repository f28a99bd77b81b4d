"""Sparse-GEMV sweep over the Llama-3-8B projection shapes (BASELINE config 2).

Times teal_sparse_gemv with CUDA events on the launching stream over a
rotating pool of weight copies larger than 3x L2 (so every launch streams
from HBM), at the given sparsities; reports achieved GB/s on algorithmic
(touched) bytes = nnz*n*2 + m*4 + n*4 and the fraction of measured HBM peak.

    python scripts/gemv_sweep.py [--sparsities 0,0.25,0.4,0.5,0.65] [--reps 50]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2408_14690_b200 as T  # noqa: E402
from paper_2408_14690_b200 import _runtime as RT  # noqa: E402

SHAPES = {"q": (4096, 4096), "k": (1024, 4096), "v": (1024, 4096), "o": (4096, 4096),
          "gate": (14336, 4096), "up": (14336, 4096), "down": (4096, 14336)}


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def sweep(sparsities, reps=50, warmup=5, dtype=torch.bfloat16, shapes=SHAPES):
    dev = RT.require_cuda()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    peak, src = peak_gbs()
    gen = torch.Generator(device=dev).manual_seed(0)
    rows = []
    for name, (n, m) in shapes.items():
        esz = torch.finfo(dtype).bits // 8
        nbytes = n * m * esz
        copies = max(2, math.ceil(3 * l2 / nbytes))
        pool = [T.Matrix.from_device(torch.randn(m, n, device=dev, generator=gen).to(dtype)) for _ in range(copies)]
        x = torch.randn(m, device=dev, generator=gen)
        out = torch.empty(n, device=dev)
        from paper_2408_14690_b200.tensor import _gemv
        for s in sparsities:
            t = T.gaussian_threshold(s)
            t32 = RT.f32_round_down(t) if s > 0 else float("-inf")
            kept = int((~(x.abs().double() <= t)).sum().item()) if s > 0 else m
            # capture `inner` back-to-back launches (rotating weights) in one
            # CUDA graph so host launch overhead is off the device timeline;
            # time each replay with events and divide by `inner`.
            inner = max(copies, 8)
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                for i in range(warmup):
                    _gemv(pool[i % copies], x, t32, out=out)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(inner):
                        _gemv(pool[i % copies], x, t32, out=out)
            torch.cuda.current_stream().wait_stream(st)
            for _ in range(2):
                g.replay()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            torch.cuda.synchronize()
            for a, b in evs:
                a.record()
                g.replay()
                b.record()
            torch.cuda.synchronize()
            us = sorted(a.elapsed_time(b) * 1e3 / inner for a, b in evs)
            med = us[len(us) // 2]
            algo = kept * n * esz + m * 4 + n * 4
            gbs = algo / (med * 1e-6) / 1e9
            rows.append({"proj": name, "n": n, "m": m, "s": s, "kept": kept, "median_us": round(med, 3),
                         "min_us": round(us[0], 3), "algo_bytes": algo, "gbs": round(gbs, 1),
                         "frac": round(gbs / peak, 4), "copies": copies})
            print(json.dumps(rows[-1]), flush=True)
        del pool
        torch.cuda.empty_cache()
    return rows, peak, src


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sparsities", default="0,0.25,0.4,0.5,0.65")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--out")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    shapes = {k: v for k, v in SHAPES.items() if not a.only or k in a.only.split(",")}
    rows, peak, src = sweep([float(s) for s in a.sparsities.split(",")], reps=a.reps,
                            dtype=torch.float32 if a.f32 else torch.bfloat16, shapes=shapes)
    if a.out:
        Path(a.out).write_text(json.dumps({"peak_gbs": peak, "peak_src": src, "rows": rows,
                                           "ctas_per_sm": os.environ.get("TEAL_CTAS_PER_SM", "4")}, indent=1))
