"""Per-CTA phase timeline of one teal_fused_gemv launch (TEAL_TIMELINE=1).

Phases: 0 entry, 1 first bulk copy issued, 2 streaming done, 3 exit.
    TEAL_TIMELINE=1 python scripts/timeline.py --proj gate --s 0.5
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("TEAL_TIMELINE", "1")
import paper_2408_14690_b200 as T  # noqa: E402
from paper_2408_14690_b200 import _clib as C, _runtime as RT  # noqa: E402
from paper_2408_14690_b200.tensor import _gemv  # noqa: E402

SHAPES = {"q": (4096, 4096), "k": (1024, 4096), "o": (4096, 4096), "gate": (14336, 4096), "down": (4096, 14336),
          "gateup": (28672, 4096)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--proj", default="gate")
    ap.add_argument("--s", type=float, default=0.5)
    ap.add_argument("--graph", type=int, default=4)
    a = ap.parse_args()
    n, m = SHAPES[a.proj]
    dev = RT.require_cuda()
    ws = [T.Matrix.from_device(torch.randn(m, n, device=dev).to(torch.bfloat16)) for _ in range(a.graph)]
    x = torch.randn(m, device=dev)
    t32 = RT.f32_round_down(T.gaussian_threshold(a.s)) if a.s > 0 else float("-inf")
    out = torch.empty(n, device=dev)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for w in ws:
            _gemv(w, x, t32, out=out)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for w in ws:
                _gemv(w, x, t32, out=out)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e3 / a.graph
    buf = (ctypes.c_ulonglong * (4 * 4096))()
    C.call("teal_debug_timeline", ctypes.cast(buf, ctypes.c_void_p), 4 * 4096)
    tl = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 4).astype(np.int64)
    tl = tl[tl[:, 0] > 0]
    t0 = tl[:, 0].min()
    rel = (tl - t0) / 1e3
    print(f"{a.proj} s={a.s}: graph per-launch {per:.2f} us; CTAs {len(tl)}")
    for k, name in enumerate(["entry", "first copy", "stream done", "exit"]):
        v = rel[:, k]
        print(f"  {name:12s} min {v.min():7.2f}  p50 {np.median(v):7.2f}  p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f} us")
    d = rel[:, 2] - rel[:, 1]
    print(f"  stream dur   min {d.min():7.2f}  p50 {np.median(d):7.2f}  max {d.max():7.2f} us")
    print(f"  epi dur      p50 {np.median(rel[:, 3] - rel[:, 2]):7.2f}  max {(rel[:, 3] - rel[:, 2]).max():7.2f} us")


if __name__ == "__main__":
    main()
