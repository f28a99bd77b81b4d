// Design probe: latency of one round of 8 independent loads per thread (256
// threads, 1 CTA) for load flavours: ld.global.cg (__ldcg, SASS
// LDG.STRONG.GPU), ld.relaxed.gpu, weak ld.global, ld.global.nc, with the
// buffer L2-resident (warm) or just evicted (cold).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ float ld(const float* p) {
    float v;
    if (MODE == 0) v = __ldcg(p);
    else if (MODE == 1) asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    else if (MODE == 2) asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if (MODE == 3) v = __ldg(p);
    else asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
template <int MODE>
__global__ void k(const float* buf, int rounds, long stride, float* out, unsigned long long* t) {
    float acc = 0.f;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    long off = threadIdx.x;
    for (int r = 0; r < rounds; ++r) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = ld<MODE>(buf + ((off + (long)q * stride + (long)r * 8 * stride) & ((1L << 26) - 1)));
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
        off += (long)(acc == 12345.f);
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) *t = t1 - t0;
    if (acc == 1.f) out[0] = acc;
}
int main() {
    float* buf; float* out; unsigned long long* t; float* flush;
    cudaMalloc(&buf, (1L << 26) * 4); cudaMalloc(&out, 64); cudaMalloc(&t, 8); cudaMalloc(&flush, 512L << 20);
    cudaMemset(buf, 0, (1L << 26) * 4);
    const char* names[] = {"ldcg", "relaxed.gpu", "weak", "nc", "weak.L1noalloc"};
    for (int cold = 0; cold < 2; ++cold) {
        for (int mode = 0; mode < 5; ++mode) {
            const int rounds = 20;
            for (int rep = 0; rep < 2; ++rep) {
                if (cold) cudaMemset(flush, rep, 512L << 20);  // evict L2
                else { // warm: touch the lines
                    auto kk = k<3>; kk<<<1, 256>>>(buf, rounds, 4096, out, t);
                }
                switch (mode) {
                    case 0: k<0><<<1, 256>>>(buf, rounds, 4096, out, t); break;
                    case 1: k<1><<<1, 256>>>(buf, rounds, 4096, out, t); break;
                    case 2: k<2><<<1, 256>>>(buf, rounds, 4096, out, t); break;
                    case 3: k<3><<<1, 256>>>(buf, rounds, 4096, out, t); break;
                    case 4: k<4><<<1, 256>>>(buf, rounds, 4096, out, t); break;
                }
                cudaDeviceSynchronize();
            }
            unsigned long long ns;
            cudaMemcpy(&ns, t, 8, cudaMemcpyDeviceToHost);
            printf("%s %-16s %6.0f ns per round of 8 loads\n", cold ? "cold" : "warm", names[mode], ns / (double)rounds);
        }
    }
    return 0;
}
