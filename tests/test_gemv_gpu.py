"""GPU parity of the sparse GEMV (teal_sparse_gemv / teal_fused_gemv) against
the oracle and the reference's golden vectors.  Mirrors
pkg/tests/test_kernel.py:35-91 and test_acceptance.py:173-192."""

from __future__ import annotations

import ctypes
import zlib

import numpy as np
import pytest
import torch

from conftest import golden, golden_json, rel_err, seeded_case, sha
from oracle import actsparse_ref as R
from oracle import cpu as OC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_2408_14690_b200 as T
    return T


def colmajor(T, arr):
    return T.Matrix.from_2d(arr, T.Layout.COL_MAJOR)


class TestSparseGemv:
    def test_zero_threshold_matches_dense(self, T):
        x, arr = seeded_case(0, 48, 96)
        w = colmajor(T, arr)
        assert rel_err(T.sparse_gemv(x, 0.0, w), T.matmul_dense(x, w)) <= 1e-5
        assert rel_err(T.matmul_dense(x, w), OC.gemv_dense(x, np.ascontiguousarray(arr.T))) <= 1e-6

    def test_all_pruned_zero_output_zero_work(self, T):
        x, arr = seeded_case(1, 16, 32)
        t = float(np.abs(x).max())
        y, macs = T.sparse_gemv(x, t, colmajor(T, arr), count_macs=True)
        assert np.array_equal(y, np.zeros(16, dtype=np.float32)) and macs == 0

    @pytest.mark.parametrize("seed", range(25))
    def test_reference_golden_grid(self, T, seed):
        g = golden("kernel")
        rng = np.random.default_rng(1000 + seed)
        x = rng.standard_normal(96, dtype=np.float32)
        arr = rng.standard_normal((64, 96), dtype=np.float32)
        t = float(rng.uniform(0.0, 2.0))
        y, macs = T.sparse_gemv(x, t, colmajor(T, arr), count_macs=True)
        assert rel_err(y, g["grid25_y"][seed]) <= 1e-5
        assert macs == int(g["grid25_macs"][seed])

    def test_mac_counter_proportional_to_kept_columns(self, T):
        x, arr = seeded_case(3, 64, 128)
        w = colmajor(T, arr)
        for t in (0.0, 0.3, 0.7, 1.5):
            _, macs = T.sparse_gemv(x, t, w, count_macs=True)
            assert macs == (128 - int(np.count_nonzero(np.abs(x) <= t))) * 64

    def test_row_major_rejected(self, T):
        x, arr = seeded_case(4, 8, 8)
        with pytest.raises(ValueError, match="column-major"):
            T.sparse_gemv(x, 0.5, T.Matrix.from_2d(arr, T.Layout.ROW_MAJOR))

    def test_negative_and_nan_threshold_rejected(self, T):
        x, arr = seeded_case(5, 8, 8)
        for t in (-0.1, float("nan")):
            with pytest.raises(ValueError):
                T.sparse_gemv(x, t, colmajor(T, arr))

    def test_dimension_mismatch_rejected(self, T):
        _, arr = seeded_case(6, 8, 8)
        with pytest.raises(ValueError, match="mismatch"):
            T.sparse_gemv(np.zeros(9, np.float32), 0.0, colmajor(T, arr))

    def test_infinite_threshold_skips_everything(self, T):
        x, arr = seeded_case(7, 8, 8)
        y, macs = T.sparse_gemv(x, float("inf"), colmajor(T, arr), count_macs=True)
        assert macs == 0 and not y.any()

    def test_fp64_tie_semantics_of_skip_gemv(self, T):
        g = golden("sparsify")
        w = colmajor(T, np.ones((3, 4), np.float32))
        _, macs = T.sparse_gemv(g["tie_x"], 0.3, w, count_macs=True)
        assert macs == int(g["tie_gemv_macs"])

    def test_nan_input_kept(self, T):
        x = np.array([np.nan, 0.1, 3.0, -0.01], np.float32)
        _, macs = T.sparse_gemv(x, 0.5, colmajor(T, np.ones((2, 4), np.float32)), count_macs=True)
        assert macs == 2 * 2


class TestAcceptanceCriterion6:
    def test_1000_small_cases(self, T):
        c6 = golden_json("crit6")["small"]
        for seed in range(1000):
            rng = np.random.default_rng(seed)
            x = rng.standard_normal(256, dtype=np.float32)
            data = rng.standard_normal(256 * 256, dtype=np.float32)
            t = float(rng.uniform(0.0, 1.5))
            w = T.Matrix(256, 256, T.Layout.COL_MAJOR, data)
            y, macs = T.sparse_gemv(x, t, w, count_macs=True)
            ref, _ = OC.skip_gemv(x, data.reshape(256, 256), t)
            assert rel_err(y, ref) <= 1e-5, seed
            assert macs == c6[seed][2], seed

    def test_100_large_cases(self, T):
        c6 = golden_json("crit6")["large"]
        for k in range(100):
            rng = np.random.default_rng(10_000 + k)
            x = rng.standard_normal(4096, dtype=np.float32)
            data = rng.standard_normal(1024 * 4096, dtype=np.float32)
            t = float(rng.uniform(0.0, 1.5))
            w = T.Matrix(1024, 4096, T.Layout.COL_MAJOR, data)
            y, macs = T.sparse_gemv(x, t, w, count_macs=True)
            ref, _ = OC.skip_gemv(x, data.reshape(4096, 1024), t, threads=8)
            assert sha(ref) == c6[k][0]
            assert rel_err(y, ref) <= 1e-5 and macs == c6[k][2]


LLAMA8B = {"q": (4096, 4096), "k": (1024, 4096), "v": (1024, 4096), "o": (4096, 4096),
           "gate": (14336, 4096), "up": (14336, 4096), "down": (4096, 14336)}


def _bits_and_y(T, wt, x, t32, kept=True):
    """Run teal_fused_gemv with the debug keep-bitmask enabled."""
    from paper_2408_14690_b200 import _clib as C, _runtime as RT
    dev = wt.device
    m, n = wt.shape
    y = torch.empty(n, device=dev)
    bits = torch.zeros((m + 31) // 32, dtype=torch.int32, device=dev)
    kc = torch.zeros(1, dtype=torch.int64, device=dev)
    a = C.TealGemvArgs()
    a.w_dtype = RT.dtype_code(wt.dtype)
    a.x_dtype = RT.dtype_code(x.dtype)
    a.x = x.data_ptr()
    a.m = m
    a.nseg = 1
    a.seg[0].w = wt.data_ptr()
    a.seg[0].ldw = n
    a.seg[0].n = n
    a.seg[0].t32 = t32
    a.seg[0].y = y.data_ptr()
    a.seg[0].dbg_bits = bits.data_ptr()
    a.seg[0].kept = kc.data_ptr()
    RT.bind_workspace(a, dev)
    C.check(C.lib().teal_fused_gemv(ctypes.byref(a), RT.stream_handle()))
    return y, bits, int(kc.item())


class TestLlamaShapesBf16:
    @pytest.mark.parametrize("proj", list(LLAMA8B))
    @pytest.mark.parametrize("s", [0.0, 0.25, 0.4, 0.5, 0.65])
    def test_projection_parity(self, T, proj, s, cuda_device):
        n, m = LLAMA8B[proj]
        rng = np.random.default_rng(zlib.crc32(f"{proj}{s}".encode()))
        x = rng.standard_normal(m, dtype=np.float32)
        wt = torch.randn(m, n, generator=torch.Generator().manual_seed(5), dtype=torch.float32).to(torch.bfloat16)
        t = T.gaussian_threshold(s)
        from paper_2408_14690_b200 import _runtime as RT
        t32 = RT.f32_round_down(t)
        y, bits, kept = _bits_and_y(T, wt.to(cuda_device), torch.from_numpy(x).to(cuda_device), t32)
        keep = ~(np.abs(x).astype(np.float64) <= t)
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), R.pack_bits(keep))
        assert kept == int(keep.sum())
        ref, used = OC.skip_gemv_bf16(x, wt.view(torch.int16).numpy().view(np.uint16), t, threads=8)
        assert used == kept
        assert rel_err(y.cpu().numpy(), ref) <= 1e-2
        assert rel_err(y.cpu().numpy(), ref) <= 1e-5  # fp32 accumulate: far inside the bf16 bar


class TestShapesAndDtypes:
    @pytest.mark.parametrize("n,m", [(1, 1), (3, 5), (17, 33), (100, 1000), (1408, 512), (512, 1408),
                                     (24, 40), (4096, 2049), (257, 4100)])
    @pytest.mark.parametrize("wdt", [torch.float32, torch.bfloat16])
    def test_odd_shapes(self, T, n, m, wdt, cuda_device):
        rng = np.random.default_rng(n * 7919 + m)
        x = rng.standard_normal(m, dtype=np.float32)
        arr = rng.standard_normal((n, m), dtype=np.float32)
        wt = torch.from_numpy(np.ascontiguousarray(arr.T)).to(wdt)
        w = T.Matrix.from_device(wt.to(cuda_device))
        for t in (0.0, 0.5, 1.2):
            y, macs = T.sparse_gemv(x, t, w, count_macs=True)
            wref = wt.float().numpy()
            ref, used = OC.skip_gemv(x, wref, t)
            assert rel_err(y, ref) <= 1e-5 and macs == used * n

    def test_bf16_activation_input(self, T, cuda_device):
        rng = np.random.default_rng(11)
        xb = torch.from_numpy(rng.standard_normal(4096, dtype=np.float32)).to(torch.bfloat16)
        arr = rng.standard_normal((1024, 4096), dtype=np.float32)
        w = T.Matrix.from_2d(arr, T.Layout.COL_MAJOR)
        y = T.sparse_gemv(xb.to(cuda_device), 0.7, w)
        ref, _ = OC.skip_gemv(xb.float().numpy(), np.ascontiguousarray(arr.T), 0.7)
        assert rel_err(y.cpu().numpy(), ref) <= 1e-5

    def test_int8_rows_with_column_scale(self, T, cuda_device):
        rng = np.random.default_rng(12)
        m, n = 4096, 2048
        q = rng.integers(-127, 128, size=(m, n), dtype=np.int8)
        scale = (rng.random(n, dtype=np.float32) * 0.02 + 0.001).astype(np.float32)
        x = rng.standard_normal(m, dtype=np.float32)
        w = T.Matrix.from_device(torch.from_numpy(q).to(cuda_device), torch.from_numpy(scale).to(cuda_device))
        t = T.gaussian_threshold(0.5)
        y, macs = T.sparse_gemv(x, t, w, count_macs=True)
        ref, used = OC.skip_gemv(x, q.astype(np.float32), t)
        assert rel_err(y, ref * scale) <= 1e-5 and macs == used * n

    def test_deterministic_and_graph_capturable(self, T, cuda_device):
        rng = np.random.default_rng(13)
        x = torch.from_numpy(rng.standard_normal(14336, dtype=np.float32)).to(cuda_device)
        wt = torch.randn(14336, 4096, device=cuda_device).to(torch.bfloat16)
        w = T.Matrix.from_device(wt)
        a = T.sparse_gemv(x, 0.6, w).clone()
        b = T.sparse_gemv(x, 0.6, w).clone()
        assert torch.equal(a, b)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            T.sparse_gemv(x, 0.6, w)  # warm workspace on this stream
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                y = T.sparse_gemv(x, 0.6, w)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, a)


class TestFusedSegments:
    """Multi-projection launches: each segment carries its own threshold."""

    def _run(self, cuda_device, n_list, m, thr, dtype, epi="store", seed=0):
        from paper_2408_14690_b200 import _clib as C, _runtime as RT
        rng = np.random.default_rng(seed)
        x = rng.standard_normal(m, dtype=np.float32)
        w = rng.standard_normal((m, sum(n_list)), dtype=np.float32)
        wt = torch.from_numpy(w).to(dtype).to(cuda_device)
        xd = torch.from_numpy(x).to(cuda_device)
        ys = [torch.zeros(n, device=cuda_device) for n in n_list]
        a = C.TealGemvArgs()
        a.w_dtype, a.x_dtype, a.x, a.m, a.nseg = RT.dtype_code(dtype), C.TEAL_F32, xd.data_ptr(), m, len(n_list)
        col = 0
        for i, n in enumerate(n_list):
            s = a.seg[i]
            s.w, s.ldw, s.n, s.t32, s.y = wt.data_ptr() + col * wt.element_size(), wt.stride(0), n, RT.f32_round_down(thr[i]), ys[i].data_ptr()
            col += n
        inter = torch.zeros(n_list[0], device=cuda_device)
        if epi == "silu":
            a.epilogue, a.inter = C.EPI_SILU, inter.data_ptr()
        RT.bind_workspace(a, cuda_device)
        RT.launch_gemv(a)
        torch.cuda.synchronize()
        wf = wt.float().cpu().numpy()
        refs, col = [], 0
        for i, n in enumerate(n_list):
            refs.append(OC.skip_gemv(x, np.ascontiguousarray(wf[:, col:col + n]), thr[i])[0])
            col += n
        return ys, refs, inter

    @pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
    def test_three_segments_distinct_thresholds(self, cuda_device, dtype):
        ys, refs, _ = self._run(cuda_device, [1024, 256, 256], 1024, [0.3, 0.9, 1.5], dtype)
        for y, r in zip(ys, refs):
            assert rel_err(y.cpu().numpy(), r) <= 1e-5

    @pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
    def test_silu_pair_distinct_thresholds(self, cuda_device, dtype):
        _, (g, u), inter = self._run(cuda_device, [2816, 2816], 1024, [0.6, 0.7], dtype, epi="silu")
        want = g / (1 + np.exp(-g)) * u
        assert rel_err(inter.cpu().numpy(), want) <= 1e-5


@pytest.mark.parametrize("bpe", [4, 2])
def test_bench_gemv_checks_against_an_independent_product(bpe):
    # kernel.bench_gemv (kernel.py:133-209): every rep checked after timing
    # against cuBLAS fp64 of the fp64-masked input (not this package's
    # kernels), realized sparsity near the Gaussian quantile, MAC-free
    # traffic model (kernel.py:68-91)
    import paper_2408_14690_b200 as T
    r = T.bench_gemv(1024, 4096, [0.0, 0.25, 0.5, 0.65], reps=10, warmup=3, rng=T.RngStream(5),
                     bytes_per_element=bpe)
    assert r.rows == 1024 and r.cols == 4096 and len(r.points) == 4
    for p in r.points:
        assert p.checksum_ok
        assert abs(p.realized_sparsity - p.sparsity) < 0.05
        assert abs(p.traffic.weight_bytes_sparse - (1 - p.realized_sparsity) * 1024 * 4096 * bpe) <= 1
        assert p.median_ns > 0 and p.min_ns <= p.median_ns
