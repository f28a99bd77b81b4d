"""Minimal driver for an ncu capture of the persistent step kernel on
Llama-3-8B layer shapes (reduced layer count, small vocab).
    ncu --set full -k regex:step_kernel -s 3 -c 1 python scripts/prof_step.py"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--s", type=float, default=0.5)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--vocab", type=int, default=128256)
a = ap.parse_args()
spec = D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=a.vocab, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = D.random_weights(spec, torch.bfloat16, seed=0)
if a.s > 0:  # the bench's calibration recipe (two passes; launch engine, so no step_kernel launches here)
    thr = D.calibrate_thresholds(W, a.s, n_tokens=32, passes=2, engine="launch")
else:
    thr = None
dec = E.StepDecoder(W, thr)
dec.reset()
for _ in range(a.steps):
    dec.step_token()
torch.cuda.synchronize()
print("done")
