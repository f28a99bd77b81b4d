"""One shared-mask batched GEMV (Mistral-7B gate shape, bf16, B=16, 50%) for
ncu: python scripts/prof_batched2.py [B] [n] [m]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import quant as Q  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 14336
m = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
w = Q.as_bf16(torch.randn(m, n, device="cuda") / m ** 0.5)
x = torch.randn(B, m, device="cuda")
t = float(torch.quantile(x.abs().mean(0), 0.5))
for _ in range(4):
    Q.sparse_gemv_batched(x, t, w)
torch.cuda.synchronize()
print("done")
