// Microbenchmark: how fast can one wave of CTAs gather 1-4 KB row segments
// from HBM on B200?  (design probe for the sparse-GEMV streaming core; not
// part of the product library)
//
//   mode 0: LDG.256, U rows per warp per synchronous round
//   mode 1: LDG.256, register double-buffered (prefetch next round)
//   mode 2: cp.async.bulk ring (1 producer warp, 8 consumer warps)
//
// Every mode reads `rows` row segments of `seg` bytes, row i at base + i*stride
// (stride = 28 KB like a gate row), split evenly over G CTAs, and sums them.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct alignas(32) U8 { uint32_t v[8]; };
__device__ __forceinline__ U8 ldg256(const void* p) {
    U8 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
    return r;
}

template <int U, int SEGV>  // SEGV = 32-byte vectors per lane per row segment (seg = SEGV*1KB)
__global__ void __launch_bounds__(256) k_ldg(const char* base, long rows, long stride, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long r0 = (long)blockIdx.x * rows / gridDim.x, r1 = (long)(blockIdx.x + 1) * rows / gridDim.x;
    float acc = 0.f;
    for (long r = r0 + warp * U; r < r1; r += 8 * U) {
        U8 d[U][SEGV];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < SEGV; ++v) {
                if (r + u < r1) d[u][v] = ldg256(base + (r + u) * stride + v * 1024 + lane * 32);
                else for (int k = 0; k < 8; ++k) d[u][v].v[k] = 0;
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < SEGV; ++v)
#pragma unroll
                for (int k = 0; k < 8; ++k) acc += __uint_as_float(d[u][v].v[k]);
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg_db(const char* base, long rows, long stride, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long r0 = (long)blockIdx.x * rows / gridDim.x, r1 = (long)(blockIdx.x + 1) * rows / gridDim.x;
    float acc = 0.f;
    U8 a[U], b[U];
    long r = r0 + warp * U;
#pragma unroll
    for (int u = 0; u < U; ++u) if (r + u < r1) a[u] = ldg256(base + (r + u) * stride + lane * 32); else for (int k = 0; k < 8; ++k) a[u].v[k] = 0;
    for (; r < r1; r += 8 * U) {
        const long rn = r + 8 * U;
#pragma unroll
        for (int u = 0; u < U; ++u) if (rn + u < r1) b[u] = ldg256(base + (rn + u) * stride + lane * 32); else for (int k = 0; k < 8; ++k) b[u].v[k] = 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += __uint_as_float(a[u].v[k]);
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = b[u];
    }
    if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SEG>
__global__ void __launch_bounds__(288) k_bulk(const char* base, long rows, long stride, float* out, int ns) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* ring = sm;
    uint64_t* full = (uint64_t*)(ring + (size_t)ns * SEG);
    uint64_t* empty = full + ns;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    const long r0 = (long)blockIdx.x * rows / gridDim.x, r1 = (long)(blockIdx.x + 1) * rows / gridDim.x;
    const int cnt = (int)(r1 - r0);
    if (warp == 8) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int e = lane; e < cnt + 8; e += 32) {
            const int s = e % ns, use = e / ns;
            if (use > 0) {
                uint32_t done = 0;
                do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(&empty[s])), "r"((use - 1) & 1) : "memory"); } while (!done);
            }
            if (e < cnt) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(SEG) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                             ::"r"(su32(ring + (size_t)s * SEG)), "l"(base + (r0 + e) * stride), "r"(SEG), "r"(su32(&full[s])), "l"(pol) : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            }
        }
    } else {
        float acc = 0.f;
        for (int e = warp; e < cnt; e += 8) {
            const int s = e % ns;
            uint32_t done = 0;
            do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(&full[s])), "r"((e / ns) & 1) : "memory"); } while (!done);
            const unsigned char* row = ring + (size_t)s * SEG;
#pragma unroll
            for (int off = lane * 16; off < SEG; off += 512) {
                uint4 v = *(const uint4*)(row + off);
                acc += __uint_as_float(v.x) + __uint_as_float(v.w);
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
        if (acc == 1234.5f) out[0] = acc;
    }
}

int main(int argc, char** argv) {
    const long stride = 28672;          // bytes between consecutive rows (gate row, bf16)
    const long rows_total = 4096 * 14;  // rows available in the pool
    const long pool = stride * rows_total + (1 << 20);
    char* base;
    float* out;
    CK(cudaMalloc(&base, pool));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(base, 1, pool));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto bench = [&](const char* name, auto launch, long rows, long seg) {
        for (int i = 0; i < 3; ++i) launch(rows);
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            cudaEventRecord(a);
            launch(rows);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        CK(cudaGetLastError());
        const double bytes = (double)rows * seg;
        printf("%-34s rows=%6ld seg=%5ld  %8.2f us  %7.1f GB/s\n", name, rows, seg, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    for (long rows : {28672L, 57344L}) {  // 28 / 58 MB of 1 KB segments
        for (int G : {sms, 2 * sms, 4 * sms}) {
            char nm[64];
            snprintf(nm, 64, "ldg U=4 G=%d", G);
            bench(nm, [&](long r) { k_ldg<4, 1><<<G, 256>>>(base, r, stride, out); }, rows, 1024);
            snprintf(nm, 64, "ldg U=8 G=%d", G);
            bench(nm, [&](long r) { k_ldg<8, 1><<<G, 256>>>(base, r, stride, out); }, rows, 1024);
            snprintf(nm, 64, "ldg U=16 G=%d", G);
            bench(nm, [&](long r) { k_ldg<16, 1><<<G, 256>>>(base, r, stride, out); }, rows, 1024);
            snprintf(nm, 64, "ldg dbuf U=4 G=%d", G);
            bench(nm, [&](long r) { k_ldg_db<4><<<G, 256>>>(base, r, stride, out); }, rows, 1024);
            snprintf(nm, 64, "ldg dbuf U=8 G=%d", G);
            bench(nm, [&](long r) { k_ldg_db<8><<<G, 256>>>(base, r, stride, out); }, rows, 1024);
        }
        for (int G : {sms, 2 * sms}) {
            for (int ns : {32, 64, 96}) {
                if (G == 2 * sms && ns > 96) continue;
                char nm[64];
                snprintf(nm, 64, "bulk 1KB ns=%d G=%d", ns, G);
                size_t smem = (size_t)ns * 1024 + ns * 16;
                cudaFuncSetAttribute(k_bulk<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                bench(nm, [&](long r) { k_bulk<1024><<<G, 288, smem>>>(base, r, stride, out, ns); }, rows, 1024);
            }
        }
    }
    // bigger segments
    for (int G : {sms, 2 * sms}) {
        char nm[64];
        snprintf(nm, 64, "ldg 2KB U=4 G=%d", G);
        bench(nm, [&](long r) { k_ldg<4, 2><<<G, 256>>>(base, r, stride, out); }, 28672, 2048);
        snprintf(nm, 64, "ldg 4KB U=4 G=%d", G);
        bench(nm, [&](long r) { k_ldg<4, 4><<<G, 256>>>(base, r, stride, out); }, 14336, 4096);
        if (G == sms) {
            snprintf(nm, 64, "bulk 4KB ns=40 G=%d", G);
            size_t smem = 40 * 4096 + 40 * 16;
            cudaFuncSetAttribute(k_bulk<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            bench(nm, [&](long r) { k_bulk<4096><<<G, 288, smem>>>(base, r, stride, out, 40); }, 14336, 4096);
        }
    }
    // back-to-back launches (GPU queue kept full): per-kernel time incl. gaps
    for (long rows : {4096L, 28672L, 57344L}) {
        for (int G : {sms, 2 * sms}) {
            for (int i = 0; i < 3; ++i) k_ldg_db<8><<<G, 256>>>(base, rows, stride, out);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int i = 0; i < 20; ++i) k_ldg_db<8><<<G, 256>>>(base + (i % 2) * 64, rows, stride, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("b2b ldg dbuf U=8 G=%d rows=%ld: %.2f us/kernel  %.1f GB/s\n", G, rows, ms * 1e3 / 20, rows * 1024.0 / (ms * 1e-3 / 20) / 1e9);
        }
    }
    // contiguous streaming reference: copy-like read of 117 MB
    {
        long rows = 114688;  // 1 KB rows, stride 1 KB -> contiguous
        for (int G : {sms, 2 * sms, 4 * sms}) {
            char nm[64];
            snprintf(nm, 64, "contig ldg U=8 G=%d", G);
            bench(nm, [&](long r) { k_ldg<8, 1><<<G, 256>>>(base, r, 1024, out); }, rows, 1024);
        }
    }
    return 0;
}
