"""Minimal driver for ncu captures of the fused decode launches at Llama-3-8B
layer shapes (one layer, no embedding): per step the engine issues
load_residual, qkv gemv, attention, o gemv, gate/up gemv, down gemv — so
`ncu -k regex:gemv_tma -s 6 -c 1` captures step 1's gate/up launch.

    python scripts/prof_gateup.py [--steps 4] [--s 0.5]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200.theory import gaussian_threshold  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--s", type=float, default=0.5)
ap.add_argument("--layers", type=int, default=1)
a = ap.parse_args()
spec = D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=0, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
W = D.random_weights(spec, torch.bfloat16, seed=0)
t = gaussian_threshold(a.s) if a.s > 0 else None
# post-RMSNorm taps ~ N(0,1): Gaussian quantile; attn_out / mlp_inter: small magnitudes -> scaled
thr = [[t, t, t, None if t is None else 0.02 * t, t, t, None if t is None else 0.05 * t]] * a.layers
dec = D.SparseDecoder(W, thr)
dec.reset()
x = torch.from_numpy(np.random.default_rng(0).standard_normal(4096).astype(np.float32)).cuda()
for _ in range(a.steps):
    dec.step_hidden(x)
torch.cuda.synchronize()
print("done")
