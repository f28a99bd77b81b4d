import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_2408_14690_b200 import decode as D
from test_decode_gpu import torch_decode_reference
for L in (1, 2):
  for kv in (torch.float32, torch.bfloat16):
    spec = D.DecoderSpec(1024, 8, 2, 2816, L, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=3)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * L
    dec = D.SparseDecoder(W, thr, kv_dtype=kv, taps=True)
    dec.reset()
    ref = torch_decode_reference(W, thr, [5, 17, 999], spec)
    for i, tok in enumerate([5, 17, 999]):
        dec.token.fill_(tok); dec.taps.kept.zero_(); dec.step_token(); torch.cuda.synchronize()
        x_ref, lg = ref[i]
        e = float((dec.x - x_ref).norm() / x_ref.norm())
        print(L, kv, i, "x rel", e, "kept", dec.taps.kept.tolist())
