"""Config 5 sweep: batched (B = 1..16) shared-mask sparse GEMV over bf16 /
int8 / int4 rows at Mistral-7B projection shapes, 50% sparsity (threshold =
Gaussian quantile of mean |x| over the batch, calibrated per B on the input).
Reports per-launch time and GB/s on touched weight bytes (kept rows x n x
bytes-per-element + touched scales).  Rotating weight pool > 2x L2; reps launches captured in one CUDA graph
(device time, CUDA events around the replay)."""
import argparse
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_14690_b200 import quant as Q  # noqa: E402

SHAPES = {"q": (4096, 4096), "kv": (1024, 4096), "o": (4096, 4096), "gate": (14336, 4096), "down": (4096, 14336)}


def run(batches=(1, 2, 4, 8, 16), kinds=("bf16", "int8", "int4"), s=0.5, reps=20, shapes=SHAPES, quiet=False):
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    out = []
    for name, (n, m) in shapes.items():
        w = torch.randn(m, n, device=dev) / math.sqrt(m)
        for kind in kinds:
            mk = {"bf16": Q.as_bf16, "int8": Q.quantize_int8, "int4": lambda a: Q.quantize_int4(a, 128)}[kind]
            q0 = mk(w)
            nbytes = q0.data.numel() * q0.data.element_size()
            copies = max(2, math.ceil(2 * l2 / nbytes))
            pool = [q0] + [Q.QuantWeights(q0.data.clone(), q0.dtype, q0.m, q0.n,
                                          None if q0.scale is None else q0.scale.clone(), q0.group)
                           for _ in range(copies - 1)]
            for B in batches:
                x = torch.randn(B, m, device=dev)
                t = float(torch.quantile(x.abs().mean(0), s))
                kept = torch.zeros(1, dtype=torch.int64, device=dev)
                Q.sparse_gemv_batched(x, t, pool[0], kept=kept)
                torch.cuda.synchronize()
                k = int(kept.item())
                for i in range(3):
                    Q.sparse_gemv_batched(x, t, pool[i % copies])
                torch.cuda.synchronize()
                # device time: the reps launches captured in one CUDA graph (the
                # ctypes wrapper's host cost per call would otherwise dominate)
                st = torch.cuda.Stream()
                st.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(reps):
                        Q.sparse_gemv_batched(x, t, pool[i % copies])
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / reps
                del g
                bpe = {"bf16": 2, "int8": 1, "int4": 0.5}[kind]
                sc = n * 4 if kind == "int8" else (math.ceil(m / 128) * n * 4 if kind == "int4" else 0)
                touched = k * n * bpe + sc
                row = {"proj": name, "kind": kind, "B": B, "n": n, "m": m, "kept": k, "us": round(us, 2),
                       "gbs": round(touched / (us * 1e-6) / 1e9, 1),
                       "gflops": round(2 * B * k * n / (us * 1e-6) / 1e9, 1)}
                out.append(row)
                if not quiet:
                    print(json.dumps(row), flush=True)
            del pool
        del w
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    sh = {k: v for k, v in SHAPES.items() if not a.only or k in a.only.split(",")}
    run(shapes=sh)
