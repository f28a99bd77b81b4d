"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly the
entry points include/teal_b200.h declares; host-side logic that needs no GPU."""

from __future__ import annotations

import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "teal_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(teal_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2408_14690_b200 import _clib as C
    L = C.lib()
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert sorted(C.EXPORTED) == declared
    for name in declared:
        assert hasattr(L, name), name
    assert L.teal_abi_version() == 1


def test_library_is_sm100a():
    from paper_2408_14690_b200 import _clib as C
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "--list-elf", str(C.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_args_raise_valueerror_without_gpu():
    from paper_2408_14690_b200 import _clib as C
    # argument validation happens before any CUDA call
    with pytest.raises(ValueError, match="nseg"):
        a = C.TealGemvArgs()
        a.nseg = 0
        import ctypes
        C.check(C.lib().teal_fused_gemv(ctypes.byref(a), None))
    with pytest.raises(ValueError, match="non-negative"):
        C.call("teal_threshold", None, 0, 10, -1.0, None, None, None, None)


def test_threshold_rounding_modes():
    from paper_2408_14690_b200 import _runtime as RT
    t = 0.3
    rn, rd = RT.f32_round_nearest(t), RT.f32_round_down(t)
    assert rn == float(np.float32(0.3)) and rn > t          # fl32(0.3) > 0.3
    assert rd < t and np.float32(rd) == np.nextafter(np.float32(rn), np.float32(0))
    assert RT.f32_round_down(0.5) == 0.5 and RT.f32_round_down(float("inf")) == float("inf")
    # the fp64 compare |x| <= t of _skip_gemv equals the fp32 compare against RD32(t)
    xs = np.array([np.float32(0.3), np.nextafter(np.float32(0.3), 0), 0.29999998], np.float32)
    assert [abs(float(v)) <= t for v in xs] == [bool(abs(v) <= np.float32(rd)) for v in xs]


def test_gemv_workspace_plan():
    import torch
    from paper_2408_14690_b200 import _runtime as RT
    for m, n, dt in [(4096, 14336, torch.bfloat16), (14336, 4096, torch.bfloat16), (4096, 128256, torch.bfloat16),
                     (512, 1408, torch.float32), (1, 1, torch.float32), (28672, 8192, torch.bfloat16)]:
        wt = torch.empty(m, n, dtype=dt)
        a = RT.single_gemv_args(wt, n, torch.empty(m), 0.5, torch.empty(n))
        g, nws, ntk = RT.gemv_workspace(a)
        tile = 512 if (dt == torch.bfloat16 and n % 16 == 0) else 256
        tiles = -(-n // tile)
        groups = tiles * (-(-m // 32))
        # the workspace covers both the fused kernel and the single-GEMV step path
        assert 1 <= g <= groups and ntk >= tiles and nws >= tiles * tile


def test_traffic_model_matches_reference():
    import paper_2408_14690_b200 as T
    r = T.traffic_model(4096, 14336, 0.5)
    assert r.weight_bytes_sparse == 117_440_512 and r.activation_bytes == 14336 * 4
    assert T.traffic_model(8, 8, 0.0).weight_bytes_dense == 256
    assert T.traffic_model(16, 16, 1.0).weight_bytes_sparse == 0.0
    assert T.traffic_model(4096, 4096, 0.5, 0.5).weight_bytes_sparse == 4096 * 4096 * 0.25
    with pytest.raises(ValueError):
        T.traffic_model(0, 8, 0.5)
    with pytest.raises(ValueError):
        T.traffic_model(8, 8, 1.5)


def test_gaussian_threshold_kat():
    import paper_2408_14690_b200 as T
    from conftest import golden
    g = golden("theory")
    for p, t in zip(g["p"], g["t"]):
        assert T.gaussian_threshold(float(p)) == t


def test_rng_stream_reproduces_reference_draws():
    import paper_2408_14690_b200 as T
    from oracle import actsparse_ref as R
    a = T.sample_gaussian(T.RngStream(202), 1000, 1.0)
    b = R.philox_generator(202, 0).standard_normal(1000, dtype=np.float32)
    assert a.tobytes() == b.tobytes()
    assert T.RngStream(5).child(1).seed == R.child_seed(5, 1)


def test_cli_bench_parser_and_errors():
    # the reference CLI's bench flags parse; invalid arguments exit 2 before any GPU work
    from paper_2408_14690_b200 import cli
    a = cli.build_parser().parse_args(["bench", "--rows", "64", "--cols", "96", "--sparsities", "0,0.5"])
    assert (a.rows, a.cols, a.reps, a.warmup, a.dtype) == (64, 96, 100, 10, "f32")
    assert cli.main(["bench", "--sparsities", "0,x"]) == cli.EXIT_INVALID
    assert cli._fmt_cell(0.1 + 0.2) == "0.3" and cli._fmt_cell(7) == "7"


@pytest.mark.gpu
def test_cli_bench_tsv(tmp_path):
    from paper_2408_14690_b200 import cli
    out = tmp_path / "bench.tsv"
    assert cli.main(["bench", "--rows", "256", "--cols", "512", "--sparsities", "0,0.5", "--reps", "10",
                     "--warmup", "3", "--out", str(out)]) == cli.EXIT_OK
    lines = out.read_text().splitlines()
    assert lines[0].split("\t") == ["sparsity", "median_ns", "min_ns", "dense_median_ns", "speedup", "weight_bytes"]
    assert len(lines) == 3 and (tmp_path / "bench.tsv.manifest.json").exists()


def test_prefill_workspace_plan_and_validation():
    """teal_prefill_workspace (host planning, no GPU): K splits only below the
    SM count, ws = splits * T * n floats, two tickets per output tile; shape
    checks raise the reference's ValueError."""
    import ctypes
    from paper_2408_14690_b200 import _clib as C

    def plan(T, m, n, splits=0):
        a = C.TealPrefillArgs(m=m, n=n, ldw=n, T=T, ldx=m, ldy=n, splits=splits)
        ns, wsf, tks = ctypes.c_int(0), C.c_i64(0), C.c_i64(0)
        C.call("teal_prefill_workspace", ctypes.byref(a), ctypes.byref(ns), ctypes.byref(wsf), ctypes.byref(tks))
        return ns.value, wsf.value, tks.value

    s, ws, tk = plan(2048, 4096, 14336)          # 112 x 8 tiles >= SMs: no split
    assert s == 1 and ws == 0 and tk == 0
    s, ws, tk = plan(128, 4096, 1024)            # 8 tiles: split K
    assert s > 1 and ws == s * 128 * 1024 and tk == 2 * 8
    assert plan(128, 4096, 1024, splits=1)[0] == 1
    assert plan(100, 4096, 4096, splits=3)[0] == 3
    with pytest.raises(ValueError, match="multiple of 64"):
        plan(16, 96, 128)
    from paper_2408_14690_b200 import prefill as P
    import torch
    with pytest.raises(ValueError, match="non-negative"):
        P.gate(torch.zeros(2, 64), -0.5)
    with pytest.raises(ValueError, match="sparse_from"):
        P.gate(torch.zeros(2, 64), 0.5, sparse_from=-1)
    with pytest.raises(ValueError, match="terms"):
        P.gate(torch.zeros(2, 64), 0.5, terms=3)


def test_batched_route_plan():
    """teal_gemv_batched_workspace picks the tcgen05 route (ctas reported 0,
    compaction + operand workspace) for bf16, B >= 4, n >= 8192, and the
    mma.sync / FMA kernels otherwise."""
    import ctypes
    from paper_2408_14690_b200 import _clib as C

    def route(B, m, n, wdt=C.TEAL_BF16):
        a = C.TealGemvBatchedArgs(m=m, n=n, ldw=n, w_dtype=wdt, B=B, group=128, t32=0.5)
        a.w, a.x, a.y, a.scale = 16, 16, 16, 16   # validation needs non-null pointers; nothing is launched
        g, nws, ntk = ctypes.c_int(-1), ctypes.c_int64(0), ctypes.c_int64(0)
        C.call("teal_gemv_batched_workspace", ctypes.byref(a), ctypes.byref(g), ctypes.byref(nws), ctypes.byref(ntk))
        return g.value, nws.value, ntk.value

    g, nws, ntk = route(16, 4096, 14336)
    assert g == 0 and nws > 16 * 4096 and ntk == 14336 // 128      # tcgen05: operand tiles, kept lists, counts
    assert route(16, 4096, 4096)[0] > 0                              # narrow: mma.sync
    assert route(2, 4096, 14336)[0] > 0                              # B < 4: FMA kernel
    assert route(16, 4096, 14336, C.TEAL_I8)[0] > 0                  # int8: mma.sync
