"""Debug: one Llama-style step, GPU taps vs a torch fp32 recompute."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import decode as D  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


spec = D.DecoderSpec(1024, 8, 2, 2816, 1, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
W = D.random_weights(spec, torch.bfloat16, seed=3)
thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]]
if len(sys.argv) > 1:
    thr = [[None if v == "x" else float(v) for v in sys.argv[1].split(",")]]
dec = D.SparseDecoder(W, thr, taps=True, kv_dtype=torch.float32)
dec.reset()
dec.token.fill_(5)
dec.step_token()
torch.cuda.synchronize()
lw = W.layers[0]
t = thr[0]


def sp(a, tt):
    return a if tt is None else torch.where(a.abs() <= float(np.float32(tt)), torch.zeros_like(a), a)


x = W.embedding[5].float()
h = x / torch.sqrt((x * x).mean() + spec.norm_eps) * lw.rms_attn
print("pre_attn", rel(dec.taps.h["pre_attn"][0], h))
wqkv = lw.wqkv.float()
nq, nkv = spec.n_q, spec.n_kv
v = sp(h, t[2]) @ wqkv[:, nq + nkv:]
ctx = v.view(2, 128).repeat_interleave(4, 0).reshape(-1)
print("attn_out", rel(dec.taps.h["attn_out"][0], ctx))
print("vcache", rel(dec.vcache[0, :, 0, :].reshape(-1).float(), v))
y = x + sp(ctx, t[3]) @ lw.wo.float()
hm = y / torch.sqrt((y * y).mean() + spec.norm_eps) * lw.rms_mlp
print("pre_mlp", rel(dec.taps.h["pre_mlp"][0], hm))
f = spec.d_ff
gate = sp(hm, t[4]) @ lw.wgu.float()[:, :f]
up = sp(hm, t[5]) @ lw.wgu.float()[:, f:]
inter = gate / (1 + torch.exp(-gate)) * up
print("mlp_inter", rel(dec.taps.h["mlp_inter"][0], inter))
out = y + sp(inter, t[6]) @ lw.wdown.float()
print("x_out", rel(dec.x, out))
for p_i, p in enumerate(D.PROJ):
    print(p, "kept", int(dec.taps.kept[0, p_i]))
