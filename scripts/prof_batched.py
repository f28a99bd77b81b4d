"""Driver for an ncu capture of the batched sparse GEMV (gate shape, B=16, 50%):
    ncu --set full -k regex:gemv_batched -s 3 -c 1 python scripts/prof_batched.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import quant as Q  # noqa: E402
from paper_2408_14690_b200.theory import gaussian_threshold  # noqa: E402

B, n, m = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 14336, 4096
w = torch.randn(m, n, device="cuda").to(torch.bfloat16)
qw = Q.as_bf16(w)
x = torch.randn(B, m, device="cuda")
t = gaussian_threshold(0.5) * 0.8
for _ in range(6):
    y = Q.sparse_gemv_batched(x, t, qw)
torch.cuda.synchronize()
print("ok", tuple(y.shape))
