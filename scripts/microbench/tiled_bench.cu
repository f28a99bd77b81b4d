// Design probe (not product code): HBM read ceilings on B200 for the sparse
// GEMV streaming core.
//
//  A. contiguous read of a large buffer (grid-stride, V independent 16-byte
//     loads per thread per iteration) -> practical read ceiling
//  B. gather of kept rows from a TILED input-major weight ([tile][m][W] bf16):
//     each CTA owns a contiguous range of the flattened (tile, row) space,
//     rows kept with probability (1 - s) from a fixed random mask; warps take
//     kept rows round-robin and issue one 16-byte load per lane per row
//     chunk, U rows in flight per warp; FMA into fp32 accumulators.
//  C. the same gather over the UNTILED layout (row stride = n) for contrast.
//
// Every configuration runs 20 back-to-back launches between two events (the
// GPU queue stays full, so launch latency is hidden like in a CUDA graph).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float bflo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bfhi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

template <int V>
__global__ void k_contig(const uint4* __restrict__ p, long n16, float* out) {
    float acc = 0.f;
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * V) {
        uint4 d[V];
#pragma unroll
        for (int v = 0; v < V; ++v) d[v] = (i + v * stride < n16) ? ldg_stream(p + i + v * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int v = 0; v < V; ++v) acc += __uint_as_float(d[v].x) + __uint_as_float(d[v].w);
    }
    if (acc == 1234.5f) out[0] = acc;
}

// W = columns per tile (bf16), C16 = W*2/16 vectors per row chunk (<= 32, power of 2)
// rows per warp instruction R = 32 / C16.
template <int C16, int U>
__global__ void __launch_bounds__(256) k_gather(const uint16_t* __restrict__ w, long tile_stride, long ldw,
                                                 int m, int ntiles, const uint8_t* __restrict__ keep,
                                                 float* __restrict__ out) {
    constexpr int R = 32 / C16;
    constexpr int NW = 8;
    __shared__ int s_idx[4096 * 2];
    __shared__ int s_cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long F = (long)ntiles * m;
    const long g0 = (long)blockIdx.x * F / gridDim.x, g1 = (long)(blockIdx.x + 1) * F / gridDim.x;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    // walk the range tile by tile
    for (long gs = g0; gs < g1;) {
        const int tile = (int)(gs / m);
        const long ge = (long)(tile + 1) * m < g1 ? (long)(tile + 1) * m : g1;
        const int r0 = (int)(gs - (long)tile * m), r1 = (int)(ge - (long)tile * m);
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        // compaction (ordered): warp-ballot per 32 rows, sequential per block for simplicity
        for (int base = r0; base < r1; base += 256) {
            const int r = base + threadIdx.x;
            const bool k = r < r1 && keep[r];
            const unsigned b = __ballot_sync(0xffffffffu, k);
            __shared__ int s_wc[8];
            if (lane == 0) s_wc[warp] = __popc(b);
            __syncthreads();
            int off = s_cnt;
            for (int q = 0; q < warp; ++q) off += s_wc[q];
            if (k) s_idx[off + __popc(b & ((1u << lane) - 1))] = r;
            __syncthreads();
            if (threadIdx.x == 0) { int t = 0; for (int q = 0; q < 8; ++q) t += s_wc[q]; s_cnt += t; }
            __syncthreads();
        }
        const int cnt = s_cnt;
        const uint16_t* tb = w + (long)tile * tile_stride;
        const int sub = lane / C16, vec = lane % C16;
        for (int e = warp * R * U; e < cnt; e += NW * R * U) {
            uint4 d[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int ei = e + u * R + sub;
                d[u] = ei < cnt ? ldg_stream(tb + (long)s_idx[ei] * ldw + vec * 8) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float h = 0.5f;
                acc[0] = fmaf(h, bflo(d[u].x), acc[0]); acc[1] = fmaf(h, bfhi(d[u].x), acc[1]);
                acc[2] = fmaf(h, bflo(d[u].y), acc[2]); acc[3] = fmaf(h, bfhi(d[u].y), acc[3]);
                acc[4] = fmaf(h, bflo(d[u].z), acc[4]); acc[5] = fmaf(h, bfhi(d[u].z), acc[5]);
                acc[6] = fmaf(h, bflo(d[u].w), acc[6]); acc[7] = fmaf(h, bfhi(d[u].w), acc[7]);
            }
        }
        __syncthreads();
        gs = ge;
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = (size_t)2 << 30;  // 2 GiB pool
    char* base;
    float* out;
    CK(cudaMalloc(&base, big));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(base, 0x11, big));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 20;
    auto run = [&](auto launch) {
        for (int i = 0; i < 3; ++i) launch(i);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) launch(i);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms * 1e3 / reps;  // us per launch
    };
    // A. contiguous read
    for (size_t bytes : {(size_t)117 << 20, (size_t)1 << 30}) {
        const long n16 = bytes / 16;
        for (int per : {1, 2, 4, 8}) {
            for (int V : {4, 8}) {
                const int G = per * sms;
                float us = run([&](int i) {
                    const uint4* p = (const uint4*)(base + (size_t)(i % 2) * (big / 2));
                    if (V == 4) k_contig<4><<<G, 512>>>(p, n16, out);
                    else k_contig<8><<<G, 512>>>(p, n16, out);
                });
                printf("A contig %5zu MB G=%4d V=%d : %7.2f us  %7.1f GB/s\n", bytes >> 20, G, V, us, bytes / (us * 1e-6) / 1e9);
            }
        }
    }
    // B/C. gather, Llama gate|up shape: n = 28672 cols, m = 4096 rows, bf16
    const int m = 4096;
    std::mt19937 rng(1);
    for (double s : {0.0, 0.5}) {
        std::vector<uint8_t> hk(m);
        for (int i = 0; i < m; ++i) hk[i] = (s == 0.0) ? 1 : ((rng() & 1) ? 1 : 0);
        long kept = 0;
        for (int i = 0; i < m; ++i) kept += hk[i];
        uint8_t* keep;
        CK(cudaMalloc(&keep, m));
        CK(cudaMemcpy(keep, hk.data(), m, cudaMemcpyHostToDevice));
        for (int W : {128, 256}) {
            const int n = 28672;
            const int ntiles = n / W;
            const double bytes = (double)kept * n * 2;
            for (int tiled = 1; tiled >= 0; --tiled) {
                const long tile_stride = tiled ? (long)m * W : W;
                const long ldw = tiled ? W : n;
                for (int per : {1, 2, 3, 4}) {
                    const int G = per * sms;
                    for (int U : {4, 8}) {
                        float us = run([&](int i) {
                            const uint16_t* wp = (const uint16_t*)(base + (size_t)(i % 4) * ((size_t)m * n * 2));
                            if (W == 128) {
                                if (U == 4) k_gather<16, 4><<<G, 256>>>(wp, tile_stride, ldw, m, ntiles, keep, out);
                                else k_gather<16, 8><<<G, 256>>>(wp, tile_stride, ldw, m, ntiles, keep, out);
                            } else {
                                if (U == 4) k_gather<32, 4><<<G, 256>>>(wp, tile_stride, ldw, m, ntiles, keep, out);
                                else k_gather<32, 8><<<G, 256>>>(wp, tile_stride, ldw, m, ntiles, keep, out);
                            }
                        });
                        printf("%s gather s=%.1f W=%3d G=%4d U=%d : %7.2f us  %7.1f GB/s (touched %.1f MB)\n",
                               tiled ? "B tiled  " : "C untiled", s, W, G, U, us, bytes / (us * 1e-6) / 1e9, bytes / 1e6);
                    }
                }
            }
        }
        cudaFree(keep);
    }
    return 0;
}
