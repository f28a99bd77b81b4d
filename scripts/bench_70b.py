"""Config 4 on ONE B200: Llama-3-70B random-init bf16 (141 GB, tiled in HBM)
batch-1 decode with the persistent step engine at dense / 40% / 50% uniform
calibrated sparsity (tensor parallelism degree 1 — this run has one GPU).
Prints one JSON line per level."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--layers", type=int, default=80)
ap.add_argument("--quant", default="none")
a = ap.parse_args()
spec = D.LLAMA3_70B if a.layers == 80 else D.DecoderSpec(8192, 64, 8, 28672, a.layers, vocab=128256,
                                                         rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
q = None if a.quant == "none" else a.quant
Wt = E.random_tiled_model(spec, torch.bfloat16, seed=0, quant=q)
torch.cuda.synchronize()
print("weights ready", torch.cuda.memory_allocated() / 1e9, "GB", flush=True)
hists = D.calibrate_histograms(Wt, n_tokens=8, engine="step")
for s in (None, 0.4, 0.5):
    thr = None if s is None else D.uniform_thresholds(hists, spec.n_layers, s)
    dec = E.StepDecoder(Wt, thr, count_kept=True)
    dec.reset()
    dec.capture()
    dec.reset()
    for _ in range(3):
        dec.replay()
    torch.cuda.synchronize()
    dec.kept.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        dec.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    algo = dec.algorithmic_bytes(dec.kept, steps=a.steps) / a.steps
    print(json.dumps({"model": "llama3-70b", "tp": 1, "quant": a.quant, "sparsity": s, "ms_per_token": round(ms, 3),
                      "tok_s": round(1e3 / ms, 2), "algo_gb_per_token": round(algo / 1e9, 3),
                      "algo_gbs": round(algo / (ms * 1e-3) / 1e9, 1)}), flush=True)
    del dec
    torch.cuda.empty_cache()
