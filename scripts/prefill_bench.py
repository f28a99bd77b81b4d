"""Sparse-prefill GEMM throughput on B200.

For Llama-3-8B's projection shapes and prompt lengths T, times (CUDA events,
L2 flushed before every timed launch, median of --reps):
  gate    teal_prefill_gate (mask + bf16 hi/lo split, HBM-bound)
  tc1     teal_prefill_gemm, one bf16 term (tcgen05)
  tc2     teal_prefill_gemm, hi + lo terms (fp32-faithful activations)
  cublas  torch.matmul bf16 x bf16 -> bf16 (cuBLAS, the library bar)
and prints one JSON line per (shape, T) with TFLOP/s (2*T*m*n per term-pass).

    python scripts/prefill_bench.py [--T 128,512,2048] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import prefill as P  # noqa: E402

SHAPES = {"q/o": (4096, 4096), "k/v": (4096, 1024), "gate/up": (4096, 14336), "down": (14336, 4096)}


def timed(fn, reps, flush):
    out = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) * 1e3)
    return statistics.median(out)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="128,512,2048")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", default=",".join(SHAPES))
    args = ap.parse_args()
    torch.manual_seed(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in args.shapes.split(","):
        m, n = SHAPES[name]
        w = (torch.randn(m, n, device="cuda") / m ** 0.5).bfloat16()
        for T in [int(t) for t in args.T.split(",")]:
            x = torch.randn(T, m, device="cuda")
            hi, lo = P.gate(x, 0.67, sparse_from=min(T, 64))
            y = torch.empty(T, n, device="cuda")
            for _ in range(3):
                P.gemm(w, hi, lo, out=y)
                P.gemm(w, hi, None, out=y)
                torch.matmul(hi, w)
            torch.cuda.synchronize()
            us = {
                "gate": timed(lambda: P.gate(x, 0.67, sparse_from=min(T, 64)), args.reps, flush),
                "tc1": timed(lambda: P.gemm(w, hi, None, out=y), args.reps, flush),
                "tc2": timed(lambda: P.gemm(w, hi, lo, out=y), args.reps, flush),
                "cublas": timed(lambda: torch.matmul(hi, w), args.reps, flush),
            }
            fl = 2.0 * T * m * n
            rec = {"shape": name, "m": m, "n": n, "T": T, "us": {k: round(v, 2) for k, v in us.items()},
                   "tflops": {"tc1": round(fl / us["tc1"] / 1e6, 1), "tc2": round(2 * fl / us["tc2"] / 1e6, 1),
                              "cublas": round(fl / us["cublas"] / 1e6, 1)},
                   "gate_gbs": round(T * m * (4 + 4) / us["gate"] / 1e3, 1)}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
