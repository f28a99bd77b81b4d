"""Debug: per-CTA phase timeline of the persistent step (StepDecoder) on
Llama-3-8B shapes; prints the slowest CTAs of a chosen phase with the
attention units they own.  python scripts/step_timeline.py [--layers 4] [--phase 2]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--phase", type=int, default=7)
ap.add_argument("--s", type=float, default=0.5)
ap.add_argument("--steps", type=int, default=40)
a = ap.parse_args()
spec = D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = D.random_weights(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8)
thr = D.uniform_thresholds(hists, spec.n_layers, a.s)
dec = E.StepDecoder(W, thr, attn_debug=True)
dec.reset()
for _ in range(a.steps):
    dec.step_token()
tl = dec.enable_timeline()
dec.step_token()
torch.cuda.synchronize()
t = tl.cpu().double()
t = (t - t[:, 0, 0].min()) / 1e3
G = dec.grid
nu = spec.n_kv_heads * dec.nchunks
p = a.phase
dur = t[:, p, 1] - t[:, p, 0]
order = torch.argsort(t[:, p, 1], descending=True)[:12]
print(f"grid {G}, attention units {nu}, chunk {dec.attn_chunk}")
for c in order.tolist():
    units = [u for u in range(nu) if (u * G) // nu == c]
    print(f"cta {c:4d}: start {t[c, p, 0]:7.1f} end {t[c, p, 1]:7.1f} dur {dur[c]:6.1f} prev-phase end {t[c, p - 1, 1]:7.1f} units {[(u // dec.nchunks, u % dec.nchunks) for u in units]}")
dbg = dec.attn_dbg.cpu().double()
base = t0 = None
raw = tl.cpu().double()
t0 = raw[:, 0, 0].min()
for u in range(0, nu, dec.nchunks):
    row = (dbg[u] - t0) / 1e3
    print(f"group {u // dec.nchunks} chunk 0 stamps (us): " + " ".join(f"{v:7.1f}" for v in row.tolist()))
row = (dbg[1] - t0) / 1e3
print("group 0 chunk 1 stamps: " + " ".join(f"{v:7.1f}" for v in row.tolist()))
