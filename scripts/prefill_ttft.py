"""Time to first token of TEAL's sparse prefill on Llama-3-8B (random init, bf16).

For each prompt length T: the whole prompt pass (embedding, 32 layers, LM head
of the last position) of ``prefill.SparsePrefill`` timed with CUDA events
(median of --reps), for
  dense            every row dense (thresholds None; fp32-faithful hi+lo GEMMs,
                   fp32 attention)
  sparse_half      the paper's recipe: rows >= T/2 thresholded at --level
                   (two-pass calibrated thresholds), hi+lo GEMMs
  sparse_half_fast the same with one bf16 activation term and bf16 (flash) attention
plus the tensor-core share: the summed device time of the 7 GEMMs of one layer
(prefill_gemm) times the layer count, over the whole pass.

    python scripts/prefill_ttft.py [--T 512,2048] [--level 0.5] [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _time(fn, reps):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def run(W, thr, lengths=(512, 2048), reps: int = 3) -> dict:
    from paper_2408_14690_b200 import prefill as P
    spec = W.spec
    out = {}
    for T in lengths:
        toks = torch.randint(0, spec.vocab, (T,), generator=torch.Generator().manual_seed(T))
        kc = torch.zeros(spec.n_layers, spec.n_kv_heads, spec.max_seq, spec.head_dim, device="cuda",
                         dtype=torch.bfloat16)
        vc = torch.zeros_like(kc)
        row = {}
        for name, th, terms, att in (("dense", None, 2, "fp32"), ("sparse_half", thr, 2, "fp32"),
                                     ("sparse_half_fast", thr, 1, "bf16")):
            pf = P.SparsePrefill(W, th, terms=terms, attention=att)
            r = pf.forward(tokens=toks, kv_cache=(kc, vc))
            torch.cuda.synchronize()
            ms = _time(lambda: pf.forward(tokens=toks, kv_cache=(kc, vc)), reps)
            rec = {"ttft_ms": round(ms, 2), "prompt_tok_s": round(T / ms * 1e3, 1)}
            if th is not None:
                rows = T - T // 2
                per_row = sum(m for (_, m) in spec.proj_shapes().values())
                rec["realized_sparsity_2nd_half"] = round(1 - float(r.kept.sum()) / (rows * per_row * spec.n_layers), 4)
            row[name] = rec
        # tensor-core share: one layer's 7 GEMMs (2 terms), device time, x layers
        lw = W.layers[0]
        d, f, nq, nkv = spec.d_model, spec.d_ff, spec.n_q, spec.n_kv
        x = torch.randn(T, d, device="cuda")
        xf = torch.randn(T, f, device="cuda")
        hd = P.gate(x, 0.0)
        hf = P.gate(xf, 0.0)
        outs = {n: torch.empty(T, c, device="cuda") for n, c in (("q", nq), ("kv", nkv), ("d", d), ("f", f))}

        def layer_gemms():
            P.gemm(lw.wqkv[:, :nq], *hd, out=outs["q"])
            P.gemm(lw.wqkv[:, nq:nq + nkv], *hd, out=outs["kv"])
            P.gemm(lw.wqkv[:, nq + nkv:], *hd, out=outs["kv"])
            P.gemm(lw.wo, *hd, out=outs["d"])
            P.gemm(lw.wgu[:, :f], *hd, out=outs["f"])
            P.gemm(lw.wgu[:, f:], *hd, out=outs["f"])
            P.gemm(lw.wdown, *hf, out=outs["d"])
        layer_gemms()
        gms = _time(layer_gemms, reps) * spec.n_layers
        flops = 2 * 2 * T * spec.n_layers * sum(n * m for (n, m) in spec.proj_shapes().values())
        row["gemm_ms_32_layers"] = round(gms, 2)
        row["gemm_share_of_dense"] = round(gms / row["dense"]["ttft_ms"], 3)
        row["gemm_tflops_2terms"] = round(flops / (gms * 1e-3) / 1e12, 1)
        out[str(T)] = row
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="512,2048")
    ap.add_argument("--level", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from paper_2408_14690_b200 import decode as D
    W = D.random_weights(D.LLAMA3_8B, torch.bfloat16, seed=0)
    thr = D.calibrate_thresholds(W, args.level, n_tokens=64, seed=1000, passes=2, engine="step")
    print(json.dumps(run(W, thr, tuple(int(t) for t in args.T.split(",")), args.reps)))


if __name__ == "__main__":
    main()
