"""Per-CTA anatomy of every phase of the persistent step (Llama-3-8B shapes).

For each phase kind (qkv, attn, o, gu, down) and layers in [--l0, --l1), all
times relative to T0 = the latest CTA end of the previous phase (the moment
the previous phase is complete):
  start   CTA entered the phase (negative: it was waiting early)
  ready   first segment's rows ready (dependency met + prologue done)
  strm    first segment streamed (compaction + weight stream)
  end     CTA left the phase
Quantiles over CTAs (p10 / p50 / p90 / max), averaged over layers x steps.
`len` = the phase's latest end - T0 (its contribution to the step).

    python scripts/step_anatomy.py [--s 0.5] [--layers 32] [--steps 5]
"""
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
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warm", type=int, default=20)
ap.add_argument("--l0", type=int, default=2)
ap.add_argument("--l1", type=int, default=30)
ap.add_argument("--quant", default="none")
a = ap.parse_args()
spec = D.DecoderSpec(4096, 32, 8, 14336, a.layers, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
q = None if a.quant == "none" else a.quant
W = E.random_tiled_model(spec, torch.bfloat16, seed=0, quant=q)
hists = D.calibrate_histograms(W, n_tokens=8, engine="step")
thr = D.uniform_thresholds(hists, spec.n_layers, a.s) if a.s > 0 else None
dec = E.StepDecoder(W, thr)
dec.reset()
for _ in range(a.warm):
    dec.step_token()
tl = dec.enable_timeline()
names = ["load"] + ["qkv", "attn", "o", "gu", "down"] * spec.n_layers + ["lm"]
qs = torch.tensor([0.1, 0.5, 0.9, 1.0], dtype=torch.float64)
rows = {}
lens = {}
for _ in range(a.steps):
    dec.step_token()
    torch.cuda.synchronize()
    t = tl.cpu().double()
    for p in range(1 + 5 * a.l0, 1 + 5 * a.l1):
        nm = names[p]
        T0 = t[:, p - 1, 1].max()
        ok = t[:, p, 1] > 0
        st, en = t[ok, p, 0] - T0, t[ok, p, 1] - T0
        lens.setdefault(nm, []).append(float(en.max()) / 1e3)
        d = rows.setdefault(nm, {})
        d.setdefault("start", []).append(torch.quantile(st, qs) / 1e3)
        if nm != "attn":
            act = ok & (t[:, p, 2] > 0)
            rd = t[act, p, 2] - T0
            s3 = t[act, p, 3] - T0
            d.setdefault("ready", []).append(torch.quantile(rd, qs) / 1e3)
            d.setdefault("strm", []).append(torch.quantile(s3, qs) / 1e3)
            d.setdefault("strm_dur", []).append(torch.quantile(s3 - rd, qs) / 1e3)
            if nm in ("qkv", "gu"):
                d.setdefault("dep_met", []).append(torch.quantile(t[act, p, 6] - T0, qs) / 1e3)
                d.setdefault("rms_done", []).append(torch.quantile(t[act, p, 7] - T0, qs) / 1e3)
        d.setdefault("end", []).append(torch.quantile(en, qs) / 1e3)
print(f"s={a.s} layers {a.l0}..{a.l1 - 1} of {spec.n_layers}, {a.steps} steps; us relative to previous phase's last end")
print(f"{'':12s} {'p10':>7s} {'p50':>7s} {'p90':>7s} {'max':>7s}")
for nm in ("qkv", "attn", "o", "gu", "down"):
    print(f"{nm}: len {sum(lens[nm]) / len(lens[nm]):.2f} us")
    for k, v in rows[nm].items():
        m = torch.stack(v).mean(0)
        print(f"  {k:10s} " + " ".join(f"{float(x):7.2f}" for x in m))

# attention units: internal stamps (attn_debug) of the LAST layer relative to
# its qkv phase's last end, averaged over steps
dec2 = E.StepDecoder(W, thr, attn_debug=True)
dec2.reset()
for _ in range(a.warm):
    dec2.step_token()
tl2 = dec2.enable_timeline()
p_qkv = 1 + 5 * (spec.n_layers - 1)
acc = []
for _ in range(a.steps):
    dec2.step_token()
    torch.cuda.synchronize()
    t = tl2.cpu().double()
    ad = dec2.attn_dbg.cpu().double()
    T0 = t[:, p_qkv, 1].max()
    act = ad[:, 0] > 0
    r = ad[act].clone()
    r[:, :2] = (r[:, :2] - T0) / 1e3          # us vs the qkv phase's last end
    r[:, 2:] = r[:, 2:] / 1965.0               # SM cycles since 'tiles ready' -> us at 1965 MHz
    acc.append(r)
m = torch.stack(acc).mean(0)
print("attention units, last layer: entry / tiles ready (us vs qkv last end); then us after tiles ready: "
      "q staged, scores, ctx, signalled")
for u in range(m.shape[0]):
    print("  unit", u, " ".join(f"{k}:{float(m[u, k]):6.2f}" for k in range(6)))
