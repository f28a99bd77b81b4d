"""Fused tensor parallelism on ONE GPU (the validation harness): Llama-3-8B
shards of TP degree 1/2/4 whose launches run concurrently on this device and
exchange through each other's memory inside the kernel.  Total bytes per
token equal the single-GPU engine's, so tok/s here measures the protocol's
cost (cross-rank barriers, peer adds, 1/world of the CTAs per rank), next to
the single persistent launch and the launch-split TP (collectives between
launches).  python scripts/tp_fused_bench.py [--steps 30]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402
from paper_2408_14690_b200 import tp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--s", type=float, default=0.5)
a = ap.parse_args()
spec = D.LLAMA3_8B
W = D.random_weights(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8, engine="step")
thr = D.uniform_thresholds(hists, spec.n_layers, a.s)


def timeit(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ref = E.StepDecoder(W, thr)
ref.reset()
ref.token.fill_(1)
ms = timeit(ref.step_token, a.steps)
print(f"single persistent launch      : {ms:.3f} ms/token  {1e3 / ms:.1f} tok/s", flush=True)
del ref
torch.cuda.empty_cache()
for world in (1, 2, 4):
    grp = tp.FusedTPGroup([tp.shard_weights(W, r, world) for r in range(world)], thr)
    grp.reset()
    grp.set_token(1)
    ms = timeit(grp.step, a.steps)
    print(f"fused TP {world} ranks on one GPU   : {ms:.3f} ms/token  {1e3 / ms:.1f} tok/s", flush=True)
    del grp
    torch.cuda.empty_cache()
