"""Per-phase critical-path breakdown of the persistent step on a Llama-3-8B
shaped model: for every phase, (latest CTA end) - (latest CTA end of the
previous phase), averaged over layers and steps.
python scripts/step_phases.py [--s 0.5] [--layers 32] [--steps 10]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=float, default=0.5)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warm", type=int, default=30)
a = ap.parse_args()
spec = D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = E.random_tiled_model(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8, engine="step")
thr = D.uniform_thresholds(hists, spec.n_layers, a.s) if a.s > 0 else None
dec = E.StepDecoder(W, thr)
dec.reset()
for _ in range(a.warm):
    dec.step_token()
tl = dec.enable_timeline()
names = ["load"] + ["qkv", "attn", "o", "gu", "down"] * spec.n_layers + ["lm"]
acc = {}
tot = []
for _ in range(a.steps):
    dec.step_token()
    torch.cuda.synchronize()
    t = tl.cpu().double()
    t0 = t[:, 0, 0].min()
    ends = (t[:, :, 1].max(dim=0).values - t0) / 1e3
    prev = 0.0
    for p, nm in enumerate(names):
        acc.setdefault(nm, []).append(float(ends[p]) - prev)
        prev = float(ends[p])
    tot.append(prev)
print(f"s={a.s} layers={spec.n_layers} step (timeline clock) {sum(tot) / len(tot):.1f} us")
for nm in ["load", "qkv", "attn", "o", "gu", "down", "lm"]:
    v = acc[nm]
    n = len(v) // a.steps
    print(f"  {nm:5s} {sum(v) / len(v):7.2f} us/phase x {n:3d} = {sum(v) / a.steps:8.1f} us/step")
