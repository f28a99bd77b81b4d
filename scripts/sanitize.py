"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one small invocation of every kernel family of the library.

    compute-sanitizer --tool memcheck python scripts/sanitize.py
    compute-sanitizer --tool racecheck python scripts/sanitize.py

Covered: teal_threshold / _batched, teal_hist_record / _threshold, the single
sparse GEMV (gemv_one_kernel: fp32 / bf16 / int8), the fused GEMV kernels
(RMSNorm / SiLU / QKV epilogues through the per-launch decode engine) with
attention, load_residual and argmax, the batched shared-mask GEMV (FMA and
mma.sync variants: bf16 / int8 / int4, B = 1 / 4 / 16), and the persistent
step kernel (toy MHA block, 2-layer Llama-style GQA + RoPE with LM head, the
long-context variant, and tensor-parallel launch-split ranks).  The fused
in-kernel TP exchange (FusedTPGroup) is NOT run here: its ranks' launches
must run concurrently, and the sanitizer serialises kernel launches.
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2408_14690_b200 as T  # noqa: E402
from paper_2408_14690_b200 import decode as D  # noqa: E402
from paper_2408_14690_b200 import engine as E  # noqa: E402
from paper_2408_14690_b200 import quant as Q  # noqa: E402
from paper_2408_14690_b200 import tp  # noqa: E402


def step(msg):
    torch.cuda.synchronize()
    print("ok:", msg, flush=True)


QUICK = "--quick" in sys.argv  # stop after the per-launch decode engine
TINY = "--tiny" in sys.argv    # threshold, single GEMVs and the toy step kernel only (initcheck)
g = np.random.default_rng(0)
# threshold / batched threshold / histogram
x = torch.randn(5000, device="cuda")
T.sparsify(x, 0.5)
T.realized_sparsity(x, 0.5)
T.threshold_bits(x, 0.3)
T.sparsify_batched(torch.randn(4, 3000, device="cuda"), 0.4)
h = T.ActivationHistogram.empty("h", 4096, 4.0)
h.record(x)
h.thresholds([0.1, 0.5, 0.9])
step("threshold, batched threshold, histogram")
# single sparse GEMV: fp32 / bf16 / int8 rows, ragged shapes
for n, m in ((200, 333), (1024, 4096)):
    w = T.Matrix.from_2d(g.standard_normal((n, m), dtype=np.float32))
    w = T.to_layout(w, T.Layout.COL_MAJOR)
    xv = g.standard_normal(m, dtype=np.float32)
    T.sparse_gemv(xv, 0.5, w, count_macs=True)
    T.matmul_dense(xv, w)
    wd = torch.randn(m, n, device="cuda").to(torch.bfloat16)
    T.sparse_gemv(torch.from_numpy(xv).cuda(), 0.5, T.Matrix.from_device(wd))
step("single sparse / dense GEMV")
if TINY:
    from oracle import actsparse_ref as R  # noqa: E402  (weights of the toy block only)
    blocks = R.gen_model_weights(5, 1, 256, 4, 768)
    Wt = D.weights_from_blocks(blocks, 4, max_seq=8)
    dt = E.StepDecoder(Wt, [[0.3, 0.3, 0.3, 0.01, 0.4, 0.4, 0.02]])
    dt.reset()
    dt.step_hidden(np.random.default_rng(0).standard_normal(256).astype(np.float32))
    step("step kernel, toy block")
    print("sanitize workload done (tiny)")
    sys.exit(0)
# batched shared-mask GEMV (FMA and MMA kernels)
for kind in ("bf16", "int8", "int4"):
    for B in (1, 4, 16):
        Wm = torch.randn(1024, 896, device="cuda") / 32  # input-major [m, n]
        qw = {"bf16": Q.as_bf16, "int8": Q.quantize_int8, "int4": Q.quantize_int4}[kind](Wm)
        X = torch.randn(B, 1024, device="cuda")
        Q.sparse_gemv_batched(X, 0.5, qw, return_mask=True)
step("batched GEMV")
# per-launch decode engine (fused GEMV epilogues, attention, load, argmax)
spec = D.DecoderSpec(1024, 8, 2, 2816, 2, vocab=1000, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
W = D.random_weights(spec, torch.bfloat16, seed=3)
thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
dec = D.SparseDecoder(W, thr)
dec.reset()
for tok in (5, 17, 999):
    dec.token.fill_(tok)
    dec.step_token()
step("per-launch decode engine")
if QUICK:
    print("sanitize workload done (quick)")
    sys.exit(0)
# persistent step kernel: toy MHA block (fp32), Llama-style GQA, long-context variant
from oracle import actsparse_ref as R  # noqa: E402  (weights of the toy block only)
blocks = R.gen_model_weights(5, 1, 256, 4, 768)
Wt = D.weights_from_blocks(blocks, 4, max_seq=8)
dt = E.StepDecoder(Wt, [[0.3, 0.3, 0.3, 0.01, 0.4, 0.4, 0.02]])
dt.reset()
for r in range(3):
    dt.step_hidden(np.random.default_rng(r).standard_normal(256).astype(np.float32))
step("step kernel, toy block")
ds = E.StepDecoder(W, thr, taps=True, count_kept=True)
ds.reset()
for tok in (5, 17, 999, 3):
    ds.token.fill_(tok)
    ds.step_token()
step("step kernel, GQA + RoPE + LM head")
dl = E.StepDecoder(W, thr, kv_dtype=torch.float32, attn_chunk=16, long_context=2)
dl.reset()
for i in range(40):
    dl.token.fill_(i * 7 % 1000)
    dl.step_token()
step("step kernel, long-context variant (40 positions, 3 chunks)")
for q in ("int8", "int4"):
    dqq = E.StepDecoder(W, thr, quant=q)
    dqq.reset()
    dqq.step_token()
step("step kernel, int8 / int4 rows")
ranks = [tp.TPStepDecoder(tp.shard_weights(W, r, 2), thr, rank=r, world=2) for r in range(2)]
for d in ranks:
    d.reset()
    d.token.fill_(5)
tp.run_lockstep_step(ranks)
step("step kernel, launch-split tensor parallel ranks (lockstep)")
print("sanitize workload done")
