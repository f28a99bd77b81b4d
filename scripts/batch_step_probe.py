"""Two lockstep decode steps of Mistral-7B at B = 16 (bf16, 50 %, per-batch
calibrated) through batch.BatchDecoder — the launch list of one step for
`ncu --metrics gpu__time_duration.sum` (which kernels take the step's time)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import batch as BT  # noqa: E402
from paper_2408_14690_b200 import decode as D  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
W = D.random_weights(D.MISTRAL_7B, torch.bfloat16, seed=7)
thr = BT.calibrate_batch_thresholds(W, B, 0.5, n_steps=8, seed=8, passes=1)
dec = BT.BatchDecoder(W, thr, B)
dec.reset()
for _ in range(2):
    dec.tokens.copy_(torch.randint(0, 32000, (B,), device="cuda", dtype=torch.int32))
    dec.step()
torch.cuda.synchronize()
print("done")
