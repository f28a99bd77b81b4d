// Sparse prefill (sm_100a, tcgen05 + TMA): the masked GEMM of TEAL's prompt
// pass — PAPER.md:269-270, :439-446: the first `sparse_from` prompt positions
// stay dense (attention sinks), every later position's activations are
// thresholded with the same magnitude test as decode, then multiplied by the
// projection.  The reference has no prefill; the semantics per
// row are the reference's `sparsify` followed by `matmul_dense`
// (pkg/src/actsparse/sparsifier.py:120-134, tensor.py:130-140):
//
//   Y[t, :] (+)= g(X[t, :]) @ W,   g(x)_i = x_i if t < sparse_from or !(|x_i| <= thr) else 0
//
// Two kernels:
//
//  * prefill_gate_kernel — one pass over X (fp32 [T][m]): applies the mask
//    and splits every kept value into bf16 hi + lo (hi = rn(x), lo = rn(x -
//    hi); |x - hi - lo| <= 2^-18 |x|), written as the tensor-core operands.
//    This is the only place the mask is evaluated, so the GEMM never
//    re-thresholds a row per output tile (X is read once, not n/128 times).
//
//  * prefill_gemm_kernel — Y^T tile [128 output columns x BN tokens] =
//    W^T[128 x m] . G^T[m x BN] on the 5th-generation tensor cores:
//      - A = the weights in the decode engines' input-major layout
//        (W[i][j], row i = the n outputs of input i): an MN-major operand,
//        staged by TMA (2D tensor map, 128-byte swizzle, boxes of 64 outputs
//        x 64 input rows);
//      - B = the gated activations G[t][i] (K-major), TMA-staged the same
//        way, hi and lo terms as two MMAs into one accumulator;
//      - the fp32 accumulator lives in TMEM (BN columns x 128 lanes); one
//        elected thread issues tcgen05.mma (M = 128, N = BN, K = 16) and
//        tcgen05.commit frees each smem stage back to the TMA producer;
//      - 4 epilogue warps tcgen05.ld their 32 TMEM lanes (= 32 output
//        columns) and write Y rows coalesced (optionally accumulating into Y,
//        the residual add of o / down).
//    Warp roles: 0 = TMA producer, 1 = MMA issuer, 2 = TMEM allocator,
//    4..7 = epilogue.  A STAGES-deep smem ring (full / empty mbarriers).
//
// The per-token masks differ, so no K block is shared-zero across a token
// tile (at 50% sparsity a 128 x 64 block is all-zero with probability
// 2^-8192): the contraction is dense on the tensor cores, and sparsity in
// prefill is an accuracy recipe, not a speed one (the decode GEMVs are where
// TEAL saves bytes).
#include "teal_common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>

namespace teal {
namespace prefill {

constexpr int NT = 256;
constexpr int BM = 128;  // output columns per CTA (UMMA M)
constexpr int BK = 64;   // input rows per stage (one 128-byte swizzle row of bf16 activations)
constexpr int UK = 16;   // UMMA K for kind::f16

#ifndef PF_A_LBO
#define PF_A_LBO 8192    // A (MN-major, SW128): byte stride between the two 64-output halves
#endif
#ifndef PF_A_SBO
#define PF_A_SBO 1024    // A: byte stride between 8-input-row groups
#endif

template <int BN, int STAGES, int NBT = 1>
struct Cfg {
    static constexpr int A_BYTES = BK * BM * 2;  // 16 KB: 64 input rows x 128 outputs
    static constexpr int B_BYTES = BN * BK * 2;  // BN tokens x 64 inputs
    static constexpr int STAGE_BYTES = A_BYTES + NBT * B_BYTES;  // NBT activation tiles share the weight tile
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr uint32_t TMEM_COLS = 2u * BN;  // double-buffered accumulator (power of 2)
    // kind::f16 instruction descriptor: D f32, A / B bf16, A MN-major, B K-major, N, M
    static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                                      ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

// shared-memory matrix descriptor, 128-byte swizzle (layout type 2), sm_100 version bit
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Shape {
    int64_t T, n, ldy;
    int n_tiles, t_tiles, splits, kps, m_blocks, accumulate;
};

// persistent: CTA c runs units c, c + G, ...; unit = (output tile i, token tile j, K split sp).
// SHARE: one stage holds the weight tile and every term's activation tile (the weight
// tile is staged once per K block); otherwise each term is its own stage.
template <int BN, int TERMS, int STAGES, bool SHARE = false>
__global__ void __launch_bounds__(NT, 1)
prefill_gemm_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap txh,
                    const __grid_constant__ CUtensorMap txl, const Shape sh, float* __restrict__ y,
                    float* __restrict__ ws, uint32_t* __restrict__ tickets) {
    using C = Cfg<BN, STAGES, SHARE ? TERMS : 1>;
    constexpr int NV = SHARE ? 1 : TERMS;   // stages per K block
    constexpr int NBT = SHARE ? TERMS : 1;  // activation tiles per stage
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;   // [2]
    uint64_t* acc_empty = acc_full + 2;    // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = sh.n_tiles * sh.t_tiles * sh.splits;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&txh)) : "memory");
        if (TERMS == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&txl)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);  // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            uint32_t it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int sp = u % sh.splits, tile = u / sh.splits;
                const int j = tile % sh.t_tiles, i = tile / sh.t_tiles;
                const int kb0 = sp * sh.kps, kb1 = min(sh.m_blocks, kb0 + sh.kps);
                for (int kb = kb0; kb < kb1; ++kb) {
#pragma unroll
                    for (int v = 0; v < NV; ++v, ++it) {
                        const uint32_t s = it % STAGES;
                        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                        uint8_t* st = smem + s * C::STAGE_BYTES;
                        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                        tma_2d(st, &tw, i * BM, kb * BK, &full[s]);
                        tma_2d(st + C::A_BYTES / 2, &tw, i * BM + BM / 2, kb * BK, &full[s]);
#pragma unroll
                        for (int b = 0; b < NBT; ++b)
                            tma_2d(st + C::A_BYTES + b * C::B_BYTES, (v + b) ? &txl : &txh, kb * BK, j * BN, &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            uint32_t it = 0, lu = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
                const int sp = u % sh.splits;
                const int kb0 = sp * sh.kps, kb1 = min(sh.m_blocks, kb0 + sh.kps);
                const uint32_t a = lu & 1;
                if (lu >= 2) mbar_wait(&acc_empty[a], ((lu >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN;
                uint32_t acc = 0;
                for (int kb = kb0; kb < kb1; ++kb) {
#pragma unroll
                    for (int v = 0; v < NV; ++v, ++it) {
                        const uint32_t s = it % STAGES;
                        mbar_wait(&full[s], (it / STAGES) & 1);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(smem + s * C::STAGE_BYTES);
                        const uint32_t b0 = a0 + C::A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / UK; ++kk) {
                            // A: 16 input rows = 2 swizzle atoms of 8 rows x 128 B; B: 16 bf16 = 32 B along the swizzled row
                            const uint64_t ad = sw128_desc(a0 + kk * UK * 128, PF_A_LBO, PF_A_SBO);
#pragma unroll
                            for (int b = 0; b < NBT; ++b) {
                                tc_mma(d, ad, sw128_desc(b0 + b * C::B_BYTES + kk * UK * 2, 16, 1024), C::IDESC, acc);
                                acc = 1u;
                            }
                        }
                        tc_commit(&empty[s]);  // the stage is free once these MMAs have read it
                    }
                }
                tc_commit(&acc_full[a]);
            }
        }
    } else if (warp >= 4) {  // ---- epilogue: TMEM lanes 32*(warp-4) .. +31 = output columns
        const int q4 = warp - 4;
        uint32_t lu = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
            const int sp = u % sh.splits, tile = u / sh.splits;
            const int j = tile % sh.t_tiles, i = tile / sh.t_tiles;
            const uint32_t a = lu & 1;
            mbar_wait(&acc_full[a], (lu >> 1) & 1);
            tc_fence_after();
            const int64_t col = (int64_t)i * BM + 32 * q4 + lane;
            const int64_t t0 = (int64_t)j * BN;
            float* dst = sh.splits == 1 ? y : ws + (int64_t)sp * sh.T * sh.n;
            const int64_t ld = sh.splits == 1 ? sh.ldy : sh.n;
            const bool acc = sh.splits == 1 && sh.accumulate;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + a * BN + (uint32_t)(c * 32), r);
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int64_t t = t0 + c * 32 + q;
                    if (t < sh.T) {
                        float* p = dst + t * ld + col;
                        const float v = __uint_as_float(r[q]);
                        *p = acc ? *p + v : v;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);  // TMEM buffer a may take the next unit
            if (sh.splits > 1) {
                // split K (one unit per CTA, all co-resident: cooperative launch).  Every
                // split publishes its partial, waits for the tile's other splits, then sums
                // ITS slice of the tile's rows over all partials in ascending split order
                // (deterministic); the last to finish resets the tile's two counters.
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 128) {
                    atomicAdd(&tickets[2 * tile], 1u);
                    uint32_t seen;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&tickets[2 * tile]) : "memory");
                    } while (seen < (uint32_t)sh.splits);
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const int rows = (BN + sh.splits - 1) / sh.splits;
                const int64_t r0 = t0 + (int64_t)sp * rows, r1 = min64(min64(r0 + rows, t0 + BN), sh.T);
                const float* __restrict__ src = ws + col;
                for (int64_t tb = r0; tb < r1; tb += 16) {  // 16 rows' partial loads in flight per split
                    float v[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = 0.f;
                    for (int k = 0; k < sh.splits; ++k) {
#pragma unroll
                        for (int q = 0; q < 16; ++q)
                            if (tb + q < r1) v[q] += __ldcg(src + ((int64_t)k * sh.T + tb + q) * sh.n);
                    }
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (tb + q < r1) {
                            float* p = y + (tb + q) * sh.ldy + col;
                            *p = sh.accumulate ? *p + v[q] : v[q];
                        }
                    }
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 128 && atomicAdd(&tickets[2 * tile + 1], 1u) == (uint32_t)(sh.splits - 1)) {
                    tickets[2 * tile] = 0u;  // every split has passed its wait
                    tickets[2 * tile + 1] = 0u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS)
                     : "memory");
    }
}

// mask + bf16 hi/lo split, 4 elements per thread-step
__global__ void __launch_bounds__(256) prefill_gate_kernel(const float* __restrict__ x, int64_t T, int64_t m,
                                                           int64_t ldx, float t32, int64_t sparse_from,
                                                           uint16_t* __restrict__ hi, uint16_t* __restrict__ lo,
                                                           int64_t ldo, unsigned long long* __restrict__ kept) {
    const int64_t q4 = m >> 2;
    const int64_t total = T * q4;
    unsigned long long nk = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / q4, i = (e - t * q4) * 4;
        const float4 v = *reinterpret_cast<const float4*>(x + t * ldx + i);
        const bool dense = t < sparse_from;
        float g[4] = {v.x, v.y, v.z, v.w};
        uint16_t h[4], l[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool keep = dense || !(fabsf(g[k]) <= t32);
            if (!keep) g[k] = 0.f;
            nk += (!dense && keep) ? 1ull : 0ull;
            h[k] = f32_to_bf16_rn(g[k]);
            l[k] = f32_to_bf16_rn(g[k] - bf16_to_f32(h[k]));
        }
        *reinterpret_cast<uint2*>(hi + t * ldo + i) =
            make_uint2((uint32_t)h[0] | ((uint32_t)h[1] << 16), (uint32_t)h[2] | ((uint32_t)h[3] << 16));
        if (lo)
            *reinterpret_cast<uint2*>(lo + t * ldo + i) =
                make_uint2((uint32_t)l[0] | ((uint32_t)l[1] << 16), (uint32_t)l[2] | ((uint32_t)l[3] << 16));
    }
    if (kept) {
#pragma unroll
        for (int o = 16; o; o >>= 1) nk += __shfl_xor_sync(0xffffffffu, nk, o);
        if ((threadIdx.x & 31) == 0 && nk) atomicAdd(kept, nk);
    }
}

// RoPE (rotate-half, as teal_batch_rope_cache) of the prompt's q rows in place
// and k rows into the cache, v rows copied; prompt row t is position pos0 + t
template <typename KT>
__global__ void __launch_bounds__(128) prefill_rope_cache_kernel(float* __restrict__ q, int64_t ldq,
                                                                 const float* __restrict__ k, int64_t ldk,
                                                                 const float* __restrict__ v, int64_t ldv, int H,
                                                                 int KVH, int hd, int64_t pos0,
                                                                 const float* __restrict__ cosv,
                                                                 const float* __restrict__ sinv, KT* __restrict__ kc,
                                                                 KT* __restrict__ vc, int64_t max_seq) {
    const int head = blockIdx.y, half = hd >> 1;
    const int64_t t = blockIdx.x, pos = pos0 + t;
    for (int dd = threadIdx.x; dd < half; dd += blockDim.x) {
        const float cs = cosv ? cosv[pos * half + dd] : 1.f;
        const float sn = sinv ? sinv[pos * half + dd] : 0.f;
        if (head < H) {
            float* r = q + t * ldq + (int64_t)head * hd;
            const float x0 = r[dd], x1 = r[dd + half];
            r[dd] = fmaf(-x1, sn, x0 * cs);
            r[dd + half] = fmaf(x0, sn, x1 * cs);
        } else {
            const int kh = head - H;
            const float* r = k + t * ldk + (int64_t)kh * hd;
            const float x0 = r[dd], x1 = r[dd + half];
            const float k0 = fmaf(-x1, sn, x0 * cs), k1 = fmaf(x0, sn, x1 * cs);
            const float* vr = v + t * ldv + (int64_t)kh * hd;
            const int64_t off = ((int64_t)kh * max_seq + pos) * hd;
            if constexpr (sizeof(KT) == 2) {
                kc[off + dd] = f32_to_bf16_rn(k0);
                kc[off + dd + half] = f32_to_bf16_rn(k1);
                vc[off + dd] = f32_to_bf16_rn(vr[dd]);
                vc[off + dd + half] = f32_to_bf16_rn(vr[dd + half]);
            } else {
                kc[off + dd] = k0;
                kc[off + dd + half] = k1;
                vc[off + dd] = vr[dd];
                vc[off + dd + half] = vr[dd + half];
            }
        }
    }
}

// ---- host side -------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2D bf16 tensor map over rows of `inner` elements (row stride ld), box {64, rows}, 128-byte swizzle
int make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld, int box_rows) {
    auto fn = encode_fn();
    TEAL_REQUIRE(fn, "teal_prefill_gemm: cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1u, 1u};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    TEAL_REQUIRE(r == CUDA_SUCCESS, "teal_prefill_gemm: tensor map encode failed (%d)", (int)r);
    return TEAL_OK;
}


int sm_count() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

// token tile: 256 (half the A traffic per flop) unless that leaves the SMs idle
int bn_for(int64_t T, int64_t n) {
    // 256 when that still gives half the SMs a tile; else 128 (split K below the SM count)
    return (n / BM) * ((T + 255) / 256) * 2 >= sm_count() ? 256 : 128;
}

// K splits: spread a grid smaller than the SM count over K (>= 4 blocks of 64 inputs per split)
Shape plan(const teal_prefill_args* a) {
    Shape sh{};
    const int bn = bn_for(a->T, a->n);
    sh.T = a->T;
    sh.n = a->n;
    sh.ldy = a->ldy;
    sh.accumulate = a->accumulate;
    sh.n_tiles = (int)(a->n / BM);
    sh.t_tiles = (int)((a->T + bn - 1) / bn);
    sh.m_blocks = (int)(a->m / BK);
    const int tiles = sh.n_tiles * sh.t_tiles, sms = sm_count();
    // a split grid runs one unit per CTA (the splits of a tile wait for each other)
    int splits = a->splits > 0 ? a->splits : (tiles >= sms ? 1 : sms / tiles);
    if (a->splits <= 0) splits = (int)min64(splits, max64(1, sh.m_blocks / 4));
    splits = (int)max64(1, min64(min64(splits, sh.m_blocks), tiles <= sms ? sms / tiles : 1));
    sh.kps = (sh.m_blocks + splits - 1) / splits;
    sh.splits = (sh.m_blocks + sh.kps - 1) / sh.kps;
    return sh;
}

template <int BN, int TERMS, int STAGES, bool SHARE = false>
int launch(const teal_prefill_args* a, const Shape& sh, cudaStream_t stream) {
    using C = Cfg<BN, STAGES, SHARE ? TERMS : 1>;
    CUtensorMap tw, txh, txl;
    int rc = make_map(&tw, a->w, a->n, a->m, a->ldw, BK);
    if (rc) return rc;
    if ((rc = make_map(&txh, a->x_hi, a->m, a->T, a->ldx, BN))) return rc;
    if (TERMS == 2) {
        if ((rc = make_map(&txl, a->x_lo, a->m, a->T, a->ldx, BN))) return rc;
    } else {
        txl = txh;
    }
    static unsigned long long attr = 0ull;  // dynamic shared-memory opt-in, per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("teal_prefill_gemm (device)");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&attr, __ATOMIC_ACQUIRE) & bit)) {
        cudaFuncSetAttribute(prefill_gemm_kernel<BN, TERMS, STAGES, SHARE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM);
        __atomic_fetch_or(&attr, bit, __ATOMIC_RELEASE);
    }
    const int units = sh.n_tiles * sh.t_tiles * sh.splits;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)min64(units, sm_count()));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // split K waits on its sibling splits
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = sh.splits > 1 ? 1 : 0;
    cudaLaunchKernelEx(&cfg, prefill_gemm_kernel<BN, TERMS, STAGES, SHARE>, tw, txh, txl, sh, a->y, a->ws, a->tickets);
    return check_launch("teal_prefill_gemm");
}

}  // namespace prefill
}  // namespace teal

using namespace teal;
using namespace teal::prefill;

extern "C" {

int teal_prefill_gate(const float* x, int64_t T, int64_t m, int64_t ldx, float t32, int64_t sparse_from,
                      void* x_hi, void* x_lo, int64_t ldo, unsigned long long* kept, cudaStream_t stream) {
    TEAL_REQUIRE(x && x_hi, "teal_prefill_gate: null pointer");
    TEAL_REQUIRE(T >= 0 && m >= 4 && m % 4 == 0 && ldx >= m && ldo >= m && ldx % 4 == 0 && ldo % 4 == 0,
                 "teal_prefill_gate: bad shape T=%lld m=%lld ldx=%lld ldo=%lld (m, ldx, ldo multiples of 4)",
                 (long long)T, (long long)m, (long long)ldx, (long long)ldo);
    TEAL_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(x_hi) & 7) == 0 &&
                     (reinterpret_cast<uintptr_t>(x_lo) & 7) == 0,
                 "teal_prefill_gate: x must be 16-byte and outputs 8-byte aligned");
    TEAL_REQUIRE(t32 == t32 && (t32 >= 0.f || t32 == -INFINITY), "threshold must be non-negative, got %g", (double)t32);
    TEAL_REQUIRE(sparse_from >= 0, "teal_prefill_gate: sparse_from must be >= 0, got %lld", (long long)sparse_from);
    if (T == 0) return TEAL_OK;
    const int64_t total = T * (m / 4);
    const int grid = (int)min64((total + 255) / 256, (int64_t)148 * 8);
    prefill_gate_kernel<<<grid, 256, 0, stream>>>(x, T, m, ldx, t32, sparse_from, (uint16_t*)x_hi, (uint16_t*)x_lo,
                                                  ldo, kept);
    return check_launch("teal_prefill_gate");
}

int teal_prefill_workspace(const teal_prefill_args* a, int* splits, int64_t* ws_floats, int64_t* tickets) {
    TEAL_REQUIRE(a, "teal_prefill_workspace: null args");
    TEAL_REQUIRE(a->m >= BK && a->m % BK == 0 && a->n >= BM && a->n % BM == 0 && a->T >= 0,
                 "teal_prefill_workspace: m must be a multiple of %d and n of %d (got m=%lld n=%lld)", BK, BM,
                 (long long)a->m, (long long)a->n);
    const Shape sh = plan(a);
    if (splits) *splits = sh.splits;
    if (ws_floats) *ws_floats = sh.splits > 1 ? (int64_t)sh.splits * a->T * a->n : 0;
    if (tickets) *tickets = sh.splits > 1 ? 2 * (int64_t)sh.n_tiles * sh.t_tiles : 0;
    return TEAL_OK;
}

int teal_prefill_gemm(const teal_prefill_args* a, cudaStream_t stream) {
    TEAL_REQUIRE(a && a->w && a->x_hi && a->y, "teal_prefill_gemm: null pointer");
    TEAL_REQUIRE(a->m >= BK && a->m % BK == 0 && a->n >= BM && a->n % BM == 0 && a->T >= 0,
                 "teal_prefill_gemm: m must be a multiple of %d and n of %d (got m=%lld n=%lld)", BK, BM,
                 (long long)a->m, (long long)a->n);
    TEAL_REQUIRE(a->ldw >= a->n && a->ldx >= a->m && a->ldy >= a->n && a->ldw % 8 == 0 && a->ldx % 8 == 0,
                 "teal_prefill_gemm: bad strides (ldw, ldx multiples of 8 elements)");
    TEAL_REQUIRE((reinterpret_cast<uintptr_t>(a->w) & 15) == 0 && (reinterpret_cast<uintptr_t>(a->x_hi) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(a->x_lo) & 15) == 0,
                 "teal_prefill_gemm: operands must be 16-byte aligned");
    TEAL_REQUIRE(a->T <= INT32_MAX && a->m <= INT32_MAX && a->n <= INT32_MAX, "teal_prefill_gemm: shape too large");
    if (a->T == 0) return TEAL_OK;
    Shape sh = plan(a);
    if (sh.splits > 1 && !(a->ws && a->tickets)) {  // no workspace: one split
        teal_prefill_args one = *a;
        one.splits = 1;
        sh = plan(&one);
    }
    const bool two = a->x_lo != nullptr;
    // two terms: at BN = 128 one stage carries the weight tile and both activation
    // tiles (4 stages; the weight tile staged once: q/o T = 512 43.9 -> 37.4 us); at
    // BN = 256 that leaves 2 stages, too shallow (gate/up T = 2048 341 -> 409 us),
    // so each term keeps its own stage there
    if (bn_for(a->T, a->n) == 128)
        return two ? launch<128, 2, 4, true>(a, sh, stream) : launch<128, 1, 6>(a, sh, stream);
    return two ? launch<256, 2, 4>(a, sh, stream) : launch<256, 1, 4>(a, sh, stream);
}

int teal_prefill_rope_cache(float* q, int64_t ldq, const float* k, int64_t ldk, const float* v, int64_t ldv, int T,
                            int H, int KVH, int hd, int64_t pos0, const float* rope_cos, const float* rope_sin,
                            void* k_cache, void* v_cache, int kv_dtype, int64_t max_seq, cudaStream_t stream) {
    TEAL_REQUIRE(q && k && v && k_cache && v_cache, "teal_prefill_rope_cache: null pointer");
    TEAL_REQUIRE(T >= 0 && H >= 1 && KVH >= 1 && H % KVH == 0 && hd >= 2 && hd % 2 == 0,
                 "teal_prefill_rope_cache: bad shape T=%d H=%d KVH=%d hd=%d", T, H, KVH, hd);
    TEAL_REQUIRE(ldq >= (int64_t)H * hd && ldk >= (int64_t)KVH * hd && ldv >= (int64_t)KVH * hd,
                 "teal_prefill_rope_cache: bad row strides");
    TEAL_REQUIRE(pos0 >= 0 && pos0 + T <= max_seq,
                 "teal_prefill_rope_cache: positions [%lld, %lld) exceed the cache (max_seq %lld)", (long long)pos0,
                 (long long)(pos0 + T), (long long)max_seq);
    if (T == 0) return TEAL_OK;
    const dim3 grid((unsigned)T, (unsigned)(H + KVH));
    const int nt = hd / 2 >= 128 ? 128 : (hd / 2 + 31) / 32 * 32;
    if (kv_dtype == TEAL_BF16)
        prefill_rope_cache_kernel<uint16_t><<<grid, nt, 0, stream>>>(q, ldq, k, ldk, v, ldv, H, KVH, hd, pos0, rope_cos,
                                                                     rope_sin, (uint16_t*)k_cache, (uint16_t*)v_cache,
                                                                     max_seq);
    else if (kv_dtype == TEAL_F32)
        prefill_rope_cache_kernel<float><<<grid, nt, 0, stream>>>(q, ldq, k, ldk, v, ldv, H, KVH, hd, pos0, rope_cos,
                                                                  rope_sin, (float*)k_cache, (float*)v_cache, max_seq);
    else
        TEAL_REQUIRE(false, "teal_prefill_rope_cache: unsupported kv dtype %d", kv_dtype);
    return check_launch("teal_prefill_rope_cache");
}

}  // extern "C"
