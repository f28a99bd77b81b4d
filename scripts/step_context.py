"""Decode tok/s of the persistent step engine vs context length (Llama-3-8B
shapes, 50 % sparsity): positions before the start hold zero K/V (timing
only).  python scripts/step_context.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

spec = D.DecoderSpec(4096, 32, 8, 14336, 32, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=8192)
W = E.random_tiled_model(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8, engine="step")
thr = D.uniform_thresholds(hists, spec.n_layers, 0.5)
dec = E.StepDecoder(W, thr)
for pos in (64, 512, 1024, 2048, 4096, 8000):
    dec.reset(pos)
    dec.token.fill_(1)
    dec.capture()
    dec.reset(pos)
    for _ in range(3):
        dec.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dec.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"context ~{pos + 13:5d}: {ms:.3f} ms/token  {1e3 / ms:.1f} tok/s", flush=True)

# the long-context kernel variant: units walk 4 chunks with an online softmax
del dec
torch.cuda.empty_cache()
dec = E.StepDecoder(W, thr, long_context=4)
for pos in (64, 512, 1024, 2048, 4096, 8000):
    dec.reset(pos)
    dec.token.fill_(1)
    dec.capture()
    dec.reset(pos)
    for _ in range(3):
        dec.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dec.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"long_context=4 context ~{pos + 13:5d}: {ms:.3f} ms/token  {1e3 / ms:.1f} tok/s", flush=True)
