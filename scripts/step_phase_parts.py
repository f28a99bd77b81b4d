"""Median-CTA composition of each GEMV phase of the persistent step (layers
1-5 of an 8-layer Llama-3-8B-shaped model at s=0.5, 10 steps): ready = from the
CTA's phase start to its first segment's rows being ready (dependency wait +
RMS prologue / row dependencies), stream1 = compaction + streaming of the
first segment, tail = reduction and signals; end_spread = latest minus
median CTA end; start_to_prevmax = how long before the previous phase's
last CTA the median CTA entered this phase."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D
from paper_2408_14690_b200 import engine as E
spec = D.DecoderSpec(4096, 32, 8, 14336, 8, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = E.random_tiled_model(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=8, engine="step")
thr = D.uniform_thresholds(hists, spec.n_layers, 0.5)
dec = E.StepDecoder(W, thr)
dec.reset()
for _ in range(20):
    dec.step_token()
tl = dec.enable_timeline()
names = ["load"] + ["qkv", "attn", "o", "gu", "down"] * spec.n_layers + ["lm"]
acc = {}
for _ in range(10):
    dec.step_token(); torch.cuda.synchronize()
    t = tl.cpu().double()
    for p in range(6, 6 + 5 * 6):
        nm = names[p]
        if nm == "attn": continue
        ok = t[:, p, 2] > 0
        st = t[ok, p, 0]; s2 = t[ok, p, 2]; s3 = t[ok, p, 3]; en = t[ok, p, 1]
        prev_end_max = t[:, p - 1, 1].max()
        d = acc.setdefault(nm, {k: [] for k in ("ready", "stream1", "tail", "end_spread", "start_to_prevmax")})
        d["ready"].append(float((s2 - st).median()) / 1e3)
        d["stream1"].append(float((s3 - s2).median()) / 1e3)
        d["tail"].append(float((en - s3).median()) / 1e3)
        d["end_spread"].append(float(en.max() - en.median()) / 1e3)
        d["start_to_prevmax"].append(float(prev_end_max - st.median()) / 1e3)
for nm, d in acc.items():
    print(nm.ljust(5), " ".join(f"{k} {sum(v)/len(v):5.2f}" for k, v in d.items()))
