// Design probe (not product code): DRAM efficiency of the sparse row gather vs
// the row-chunk width of the tiled layout.  Weight block [tile][m][W] bf16 for
// the Llama-3-8B gate|up shape (m = 4096, 28672 columns), 50% random rows,
// equal contiguous (tile,row) ranges per CTA, pipelined 16-byte LDG with
// V = W*2/512 vectors per lane per row.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint4 ldg(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float bflo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bfhi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
constexpr int NT = 256, NW = 8;
template <int V, int U>  // V vectors (16 B) per lane per row; U rows per stage
__global__ void __launch_bounds__(NT, 2) k(const unsigned char* w, int m, int ntiles, const uint8_t* keep, float* out) {
    constexpr int ROWB = V * 512;
    __shared__ int idx[4096];
    __shared__ int s_cnt, s_wc[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long gpt = m / 32, F = (long)ntiles * gpt;
    const long g0 = (long)blockIdx.x * F / gridDim.x, g1 = (long)(blockIdx.x + 1) * F / gridDim.x;
    float acc[8 * V];
    for (int j = 0; j < 8 * V; ++j) acc[j] = 0.f;
    for (long gs = g0; gs < g1;) {
        const int tile = (int)(gs / gpt);
        const long ge = min(g1, (long)(tile + 1) * gpt);
        const int r0 = (int)(gs - tile * gpt) * 32, r1 = (int)(ge - tile * gpt) * 32;
        gs = ge;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int i0 = r0; i0 < r1; i0 += NT) {
            const int i = i0 + threadIdx.x;
            const bool kk = i < r1 && keep[i];
            const unsigned b = __ballot_sync(~0u, kk);
            if (lane == 0) s_wc[warp] = __popc(b);
            __syncthreads();
            int off = s_cnt;
            for (int q = 0; q < warp; ++q) off += s_wc[q];
            if (kk) idx[off + __popc(b & ((1u << lane) - 1))] = i - r0;
            __syncthreads();
            if (threadIdx.x == 0) { int t = 0; for (int q = 0; q < NW; ++q) t += s_wc[q]; s_cnt += t; }
            __syncthreads();
        }
        const int cnt = s_cnt;
        const unsigned char* tb = w + ((long)tile * m + r0) * ROWB + lane * 16;
        uint4 a[U][V], bb[U][V];
        auto fetch = [&](int e0, uint4 (&d)[U][V]) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v)
                    d[u][v] = e0 + u < cnt ? ldg(tb + (long)idx[e0 + u] * ROWB + v * 512) : make_uint4(0, 0, 0, 0);
        };
        auto consume = [&](const uint4 (&d)[U][V]) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    acc[8 * v + 0] = fmaf(0.5f, bflo(d[u][v].x), acc[8 * v + 0]); acc[8 * v + 1] = fmaf(0.5f, bfhi(d[u][v].x), acc[8 * v + 1]);
                    acc[8 * v + 2] = fmaf(0.5f, bflo(d[u][v].y), acc[8 * v + 2]); acc[8 * v + 3] = fmaf(0.5f, bfhi(d[u][v].y), acc[8 * v + 3]);
                    acc[8 * v + 4] = fmaf(0.5f, bflo(d[u][v].z), acc[8 * v + 4]); acc[8 * v + 5] = fmaf(0.5f, bfhi(d[u][v].z), acc[8 * v + 5]);
                    acc[8 * v + 6] = fmaf(0.5f, bflo(d[u][v].w), acc[8 * v + 6]); acc[8 * v + 7] = fmaf(0.5f, bfhi(d[u][v].w), acc[8 * v + 7]);
                }
        };
        int e0 = warp * U;
        if (e0 < cnt) {
            fetch(e0, a);
            for (;;) {
                const int en = e0 + NW * U;
                if (en < cnt) fetch(en, bb);
                consume(a);
                if (en >= cnt) break;
                e0 = en;
                if (e0 + NW * U < cnt) fetch(e0 + NW * U, a);
                consume(bb);
                if (e0 + NW * U >= cnt) break;
                e0 += NW * U;
            }
        }
        __syncthreads();
    }
    float s = 0;
    for (int j = 0; j < 8 * V; ++j) s += acc[j];
    if (s == 1234.5f) out[0] = s;
}
int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int m = 4096, cols = 28672;
    const size_t wbytes = (size_t)m * cols * 2;
    const int pool = 4;
    unsigned char* w; float* out;
    CK(cudaMalloc(&w, wbytes * pool)); CK(cudaMalloc(&out, 64)); CK(cudaMemset(w, 0x11, wbytes * pool));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (double s : {0.0, 0.5}) {
        std::mt19937 rng(1);
        std::vector<uint8_t> hk(m); long kept = 0;
        for (int i = 0; i < m; ++i) { hk[i] = s == 0 ? 1 : (rng() & 1); kept += hk[i]; }
        uint8_t* keep; CK(cudaMalloc(&keep, m)); CK(cudaMemcpy(keep, hk.data(), m, cudaMemcpyHostToDevice));
        const double bytes = (double)kept * cols * 2;
        auto run = [&](const char* name, auto kern, int ntiles, int G) {
            for (int i = 0; i < 3; ++i) kern<<<G, NT>>>(w + (i % pool) * wbytes, m, ntiles, keep, out);
            CK(cudaDeviceSynchronize());
            const int reps = 20;
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i) kern<<<G, NT>>>(w + (i % pool) * wbytes, m, ntiles, keep, out);
            cudaEventRecord(b); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double us = ms * 1e3 / reps;
            printf("s=%.1f %-22s tiles=%4d G=%4d: %7.2f us  %7.1f GB/s\n", s, name, ntiles, G, us, bytes / (us * 1e-6) / 1e9);
        };
        for (int G : {2 * sms, 224, 280}) {
            run("W=256  (512B) U=8", k<1, 8>, cols / 256, G);
            run("W=512  (1KB)  U=4", k<2, 4>, cols / 512, G);
            run("W=1024 (2KB)  U=2", k<4, 2>, cols / 1024, G);
            run("W=2048 (4KB)  U=1", k<8, 1>, cols / 2048, G);
        }
        cudaFree(keep);
    }
    return 0;
}
