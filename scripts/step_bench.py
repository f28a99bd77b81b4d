"""Quick A/B of the decode engines on Llama-3-8B shapes (random bf16 weights):
per-launch SparseDecoder vs persistent StepDecoder, dense and uniform
Gaussian-quantile thresholds (no calibration; for engine comparison only).

    python scripts/step_bench.py [--steps 50] [--rows 512]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--timeline", action="store_true")
ap.add_argument("--quant", default="none")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--engines", default="launch,step")
a = ap.parse_args()
spec = D.LLAMA3_8B if a.layers == 32 else D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=128256,
                                                         rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = D.random_weights(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8)
for s in (None, 0.5):
    thr = None if s is None else D.uniform_thresholds(hists, spec.n_layers, s)
    for eng in a.engines.split(","):
        dec = (E.StepDecoder(W, thr, ctas=a.ctas, count_kept=True, quant=None if a.quant == "none" else a.quant) if eng == "step"
               else D.SparseDecoder(W, thr))
        dec.reset()
        dec.capture()
        dec.reset()
        for _ in range(3):
            dec.replay()
        torch.cuda.synchronize()
        if eng == "step":
            dec.kept.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            dec.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        extra = ""
        if eng == "step":
            byts = dec.algorithmic_bytes(dec.kept, steps=a.steps) / a.steps
            extra = f" algo {byts / 1e9:.3f} GB/step -> {byts / (ms * 1e-3) / 1e9:.0f} GB/s"
        print(f"{eng:6s} {a.quant:4s} s={s}: {ms:.3f} ms/token  {1e3 / ms:.1f} tok/s{extra}", flush=True)
        if eng == "step" and a.timeline:
            tl = dec.enable_timeline()
            dec.capture()
            dec.replay()
            dec.replay()
            torch.cuda.synchronize()
            t = tl.cpu().double()
            t0 = t[:, 0, 0].min()
            t = (t - t0) / 1e3  # us
            names = ["load"] + ["qkv", "attn", "o", "gu", "down"] * spec.n_layers + (["lm"] if spec.vocab else [])
            for p_ in list(range(0, 11)) + list(range(len(names) - 6, len(names))):
                st, en = t[:, p_, 0], t[:, p_, 1]
                print(f"   phase {p_:3d} {names[p_]:5s} start min {st.min():8.1f} med {st.median():8.1f} max {st.max():8.1f}"
                      f" | end min {en.min():8.1f} med {en.median():8.1f} max {en.max():8.1f}")
        del dec
        torch.cuda.empty_cache()
