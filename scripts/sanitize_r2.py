"""compute-sanitizer workload for the round-2 kernels (one small invocation
each): the sparse-prefill gate / tcgen05 GEMM (one and two terms, split K,
several units per persistent CTA) / RoPE-cache kernels and a SparsePrefill
prompt pass, the tcgen05 batched GEMV with its compaction (B = 4 / 16, ragged
m, dense and all-pruned), the CATS output-sparse GEMV, and one step of the
small-batch decoder (embed, RMSNorm, RoPE + cache, attention, SiLU*up,
argmax kernels).

    compute-sanitizer --tool memcheck --kernel-name kns=4teal python scripts/sanitize_r2.py
"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import batch as BT  # noqa: E402
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import prefill as P  # noqa: E402
from paper_2408_14690_b200 import quant as Q  # noqa: E402
from paper_2408_14690_b200.model import cats_gemv  # noqa: E402


def step(msg):
    torch.cuda.synchronize()
    print("ok:", msg, flush=True)


g = torch.Generator(device="cuda").manual_seed(0)
# prefill: gate + GEMM, ragged T, split K, persistent multi-unit, accumulate
for T, m, n, splits in ((5, 128, 256, 0), (70, 1024, 256, 3), (300, 320, 4096, 1)):
    x = torch.randn(T, m, device="cuda", generator=g)
    w = (torch.randn(m, n, device="cuda", generator=g) / math.sqrt(m)).bfloat16()
    kept = torch.zeros(1, dtype=torch.int64, device="cuda")
    hi, lo = P.gate(x, 0.5, sparse_from=2, kept=kept)
    y = P.gemm(w, hi, lo, splits=splits)
    P.gemm(w, hi, None, out=y, accumulate=True, splits=splits)
step("prefill gate + tcgen05 GEMM")
spec = D.DecoderSpec(256, 4, 2, 256, 1, vocab=512, rope_theta=10000.0, norm_eps=1e-5, max_seq=32)
W = D.random_weights(spec, torch.bfloat16, seed=1)
dec = D.SparseDecoder(W, None)
dec.reset()
P.SparsePrefill(W, [[0.3] * 7]).forward(tokens=list(range(9)), decoder=dec)
step("SparsePrefill prompt pass (RoPE + cache, batch RMSNorm / SiLU / argmax)")
# tcgen05 batched GEMV + compaction
wq = Q.as_bf16(torch.randn(3000, 8192, device="cuda", generator=g) / 50.0)
for B in (4, 16):
    xs = torch.randn(B, 3000, device="cuda", generator=g)
    for t in (None, 0.6, 1e9):
        Q.sparse_gemv_batched(xs, t, wq, return_mask=True)
step("tcgen05 batched GEMV")
# CATS
wr = (torch.randn(1024, 512, device="cuda", generator=g) / 20.0).bfloat16()
cats_gemv(wr, torch.randn(512, device="cuda", generator=g), torch.randn(1024, device="cuda", generator=g), 0.4)
step("CATS output-sparse GEMV")
# small-batch decoder step (batch kernels + batched GEMVs incl. the tcgen05 LM head: vocab 8192)
spec2 = D.DecoderSpec(256, 4, 2, 256, 1, vocab=8192, rope_theta=10000.0, norm_eps=1e-5, max_seq=16)
W2 = D.random_weights(spec2, torch.bfloat16, seed=2)
bd = BT.BatchDecoder(W2, [[0.3] * 7], 4)
bd.reset()
bd.tokens.copy_(torch.tensor([1, 2, 3, 4], dtype=torch.int32))
bd.step()
bd.step()
step("batch decoder steps")
print("sanitize workload done", flush=True)
