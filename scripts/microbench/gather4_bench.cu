// Design probe (not product code): sparse row gather on B200 with TMA
// gather4 (UTMALDG.2D.GATHER4: 4 arbitrary rows x 512 B per op) into a
// shared-memory ring, vs pipelined LDG, on the TILED layout ([tile][m][256]
// bf16) at 0% / 50% row sparsity; equal contiguous (tile,row) ranges per CTA.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float bflo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bfhi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
__device__ __forceinline__ void fma8(float* a, uint4 d, float h) {
    a[0] = fmaf(h, bflo(d.x), a[0]); a[1] = fmaf(h, bfhi(d.x), a[1]); a[2] = fmaf(h, bflo(d.y), a[2]); a[3] = fmaf(h, bfhi(d.y), a[3]);
    a[4] = fmaf(h, bflo(d.z), a[4]); a[5] = fmaf(h, bfhi(d.z), a[5]); a[6] = fmaf(h, bflo(d.w), a[6]); a[7] = fmaf(h, bfhi(d.w), a[7]);
}
__device__ __forceinline__ void mwait(uint32_t bar, uint32_t par) {
    uint32_t done = 0;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(bar), "r"(par) : "memory"); } while (!done);
}

constexpr int NC = 8;  // consumer warps
template <int S>
__global__ void __launch_bounds__(NC * 32 + 32) k_g4(const __grid_constant__ CUtensorMap tm, int m, int ntiles,
                                                     const uint8_t* keep, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = sm;                              // [S][2048]
    uint64_t* full = (uint64_t*)(sm + S * 2048);
    uint64_t* empty = full + S;
    int* idx = (int*)(empty + S);                          // [4096]
    __shared__ int s_cnt, s_wc[NC + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < S) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[threadIdx.x])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[threadIdx.x])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const long gpt = m / 32, F = (long)ntiles * gpt;
    const long g0 = (long)blockIdx.x * F / gridDim.x, g1 = (long)(blockIdx.x + 1) * F / gridDim.x;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t J = 0;  // groups issued/consumed so far (ring position)
    for (long gs = g0; gs < g1;) {
        const int tile = (int)(gs / gpt);
        const long ge = min(g1, (long)(tile + 1) * gpt);
        const int r0 = (int)(gs - tile * gpt) * 32, r1 = (int)(ge - tile * gpt) * 32;
        gs = ge;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int i0 = r0; i0 < r1; i0 += blockDim.x) {
            const int i = i0 + threadIdx.x;
            const bool kk = i < r1 && keep[i];
            const unsigned b = __ballot_sync(~0u, kk);
            if (lane == 0) s_wc[warp] = __popc(b);
            __syncthreads();
            int off = s_cnt;
            for (int q = 0; q < warp; ++q) off += s_wc[q];
            if (kk) idx[off + __popc(b & ((1u << lane) - 1))] = tile * m + i;
            __syncthreads();
            if (threadIdx.x == 0) { int t = 0; for (int q = 0; q <= NC; ++q) t += s_wc[q]; s_cnt += t; }
            __syncthreads();
        }
        const int cnt = s_cnt;
        const int ng = (cnt + 3) / 4;
        if (warp == NC) {  // producer
            if (lane == 0) {
                for (int j = 0; j < ng; ++j) {
                    const uint32_t jj = J + j, slot = jj % S;
                    if (jj >= S) mwait(su(&empty[slot]), ((jj / S) - 1) & 1);
                    int r[4];
                    for (int q = 0; q < 4; ++q) r[q] = idx[min(4 * j + q, cnt - 1)];
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[slot])), "r"(2048) : "memory");
                    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                                 ::"r"(su(ring + slot * 2048)), "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[slot])) : "memory");
                }
            }
        } else {
            for (int j = warp; j < ng; j += NC) {
                const uint32_t jj = J + j, slot = jj % S;
                mwait(su(&full[slot]), (jj / S) & 1);
                const unsigned char* p = ring + slot * 2048 + lane * 16;
                for (int q = 0; q < 4; ++q) {
                    const float h = (4 * j + q < cnt) ? 0.5f : 0.f;
                    fma8(acc, *(const uint4*)(p + q * 512), h);
                }
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[slot])) : "memory");
            }
        }
        J += ng;
        __syncthreads();
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j];
    if (s == 1234.5f) out[0] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    const int m = 4096, ntiles = 112;
    const size_t wbytes = (size_t)ntiles * m * 512;
    const int pool = 4;
    unsigned char* w;
    float* out;
    CK(cudaMalloc(&w, wbytes * pool));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(w, 0x11, wbytes * pool));
    std::vector<CUtensorMap> maps(pool);
    for (int i = 0; i < pool; ++i) {
        cuuint64_t dims[2] = {256, (cuuint64_t)ntiles * m};
        cuuint64_t strides[1] = {512};
        cuuint32_t box[2] = {256, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w + i * wbytes, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (double s : {0.0, 0.5}) {
        std::mt19937 rng(1);
        std::vector<uint8_t> hk(m);
        long kept = 0;
        for (int i = 0; i < m; ++i) { hk[i] = s == 0 ? 1 : (rng() & 1); kept += hk[i]; }
        uint8_t* keep;
        CK(cudaMalloc(&keep, m));
        CK(cudaMemcpy(keep, hk.data(), m, cudaMemcpyHostToDevice));
        const double bytes = (double)kept * ntiles * 512;
        auto run = [&](const char* name, auto kern, size_t smem, int per) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int G = per * sms;
            for (int i = 0; i < 3; ++i) kern<<<G, NC * 32 + 32, smem>>>(maps[i % pool], m, ntiles, keep, out);
            CK(cudaDeviceSynchronize());
            const int reps = 20;
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i) kern<<<G, NC * 32 + 32, smem>>>(maps[i % pool], m, ntiles, keep, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double us = ms * 1e3 / reps;
            printf("s=%.1f %-24s G=%4d: %7.2f us  %7.1f GB/s\n", s, name, G, us, bytes / (us * 1e-6) / 1e9);
        };
        for (int per : {1, 2, 3}) {
            run("gather4 ring S=16", k_g4<16>, 16 * 2048 + 16 * 16 + 4096 * 4 + 1024, per);
            run("gather4 ring S=32", k_g4<32>, 32 * 2048 + 32 * 16 + 4096 * 4 + 1024, per);
            if (per <= 2) run("gather4 ring S=48", k_g4<48>, 48 * 2048 + 48 * 16 + 4096 * 4 + 1024, per);
        }
        cudaFree(keep);
    }
    return 0;
}
