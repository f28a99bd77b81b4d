"""Debug: detailed per-CTA slice timeline of the persistent step (layer 1 of a
4-layer Llama-3-8B-shaped model at s=0.5)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402

s_ = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
spec = D.DecoderSpec(4096, 32, 8, 14336, 4, vocab=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq=2048)
W = D.random_weights(spec, torch.bfloat16, seed=0)
hists = D.calibrate_histograms(W, n_tokens=4)
thr = D.uniform_thresholds(hists, spec.n_layers, s_) if s_ > 0 else None
dec = E.StepDecoder(W, thr)
dec.reset()
for _ in range(20):
    dec.step_token()
tl = dec.enable_timeline()
dec.step_token()
torch.cuda.synchronize()
t = tl.cpu().double()
t0 = t[:, 0, 0].min()
names = ["load"] + ["qkv", "attn", "o", "gu", "down"] * 4 + ["lm"]
for p in range(6, 12):
    st, en = (t[:, p, 0] - t0) / 1e3, (t[:, p, 1] - t0) / 1e3
    line = f"{names[p]:5s} start med {st.median():7.1f} max {st.max():7.1f} | end min {en.min():7.1f} med {en.median():7.1f} max {en.max():7.1f}"
    if names[p] not in ("attn",):
        dep = (t[:, p, 2] - t[:, p, 0]) / 1e3
        s1 = (t[:, p, 3] - t[:, p, 2]) / 1e3
        f1 = (t[:, p, 4] - t[:, p, 3]) / 1e3
        seg = t[:, p, 6]
        two = seg > 1
        s2 = (t[:, p, 5] - t[:, p, 4]) / 1e3
        tail = (t[:, p, 1] - torch.where(two, t[:, p, 5], t[:, p, 3])) / 1e3
        ok = t[:, p, 2] > 0
        line += (f"\n      dep wait med {dep[ok].median():6.1f} max {dep[ok].max():6.1f} | seg1 stream med {s1[ok].median():6.1f} max {s1[ok].max():6.1f}"
                 f" | seg1 fin med {f1[ok].median():6.1f} max {f1[ok].max():6.1f} | 2-seg CTAs {int(two.sum())} seg2 med {s2[two].median() if two.any() else 0:6.1f}"
                 f" | tail (last stream->end) med {tail[ok].median():6.1f} max {tail[ok].max():6.1f}")
        # the slowest CTA
        c = int(torch.argmax(t[:, p, 1]))
        row = ((t[c, p, :6] - t0) / 1e3).tolist()
        line += f"\n      slowest cta {c}: " + " ".join(f"{v:7.1f}" for v in row) + f" segs {int(t[c, p, 6])} fin {int(t[c, p, 7])}"
    print(line)
