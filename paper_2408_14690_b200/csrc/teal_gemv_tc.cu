// Small-batch shared-mask sparse GEMV on the 5th-generation tensor cores
// (sm_100a, tcgen05 + TMEM) — BASELINE config 5, bf16 weights, 4 <= B <= 16.
//
// Semantics = teal_gemv_batched (the reference's sparsify_batched followed by
// the dense product, pkg/src/actsparse/sparsifier.py:136-155 and
// tensor.py:130-140): column i of X [B][m] is pruned in every row iff
// mean_b |X[b,i]| <= t (fp32 sum in ascending b, fp64 quotient rounded to
// fp32), Y[b] = sum over kept i of X[b,i] * W[i,:].
//
// Two launches:
//
//  * tc_compact_kernel — one CTA per 1024-column chunk: the shared mask, an
//    ORDERED compaction of the chunk's kept columns (idx), and the batch's
//    kept activations gathered into the tensor-core operand layout
//    Xg[chunk][16 rows][1024] as bf16 hi + lo (hi = rn(x), lo = rn(x - hi):
//    fp32-faithful against bf16 weights), rows b >= B and the tail up to a
//    multiple of 64 zero.
//
//  * tc_gemv_kernel — persistent; unit = (128-column output tile, K split).
//    D[128 outputs x 16] (TMEM, fp32, double-buffered) += W_kept^T . Xg^T:
//      - A = the kept weight rows, GATHERED: four producer warps cp.async
//        each kept row's 256-byte segment into the 128-byte-swizzled
//        MN-major layout tcgen05 reads (the layout a TMA SWIZZLE_128B box
//        produces; one warp instruction = two whole row segments, every L2
//        sector used in full), completion signalled by
//        cp.async.mbarrier.arrive — measured faster than TMA tile::gather4
//        (4 x 128 B per instruction) and than register loads + st.shared;
//      - B = Xg hi and lo, TMA 2D boxes {64, 16};
//      - one thread issues tcgen05.mma.cta_group::1.kind::f16 (M = 128,
//        N = 16, K = 16), tcgen05.commit frees each stage;
//      - four epilogue warps tcgen05.ld their 32 TMEM lanes; a grid smaller
//        than the SM count splits the kept-row list, the last-arriving split
//        of a tile summing the partials in ascending split order
//        (deterministic).
//    The weight bytes streamed are kept * 128 * 2 per tile: only kept rows.
//    Two CTAs per SM.  Routed for n >= 64 * 128 (gate / up / LM head); the
//    narrower projections stay on the mma.sync kernel, which is as fast there
//    (profiles/r02_config5_tcgen05.md: the first kept rows arrive ~3.5 us
//    after launch, a fixed cost the 8-32 K blocks of a narrow tile cannot
//    amortise).
#include "teal_common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>

namespace teal {
namespace prefill {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
}
namespace gemvtc {

constexpr int CH = 1024;  // columns per compaction chunk
constexpr int CT = 1024;  // compaction threads (one per column)
constexpr int MAXCH = 64; // m <= 65536
constexpr int BM = 128, BK = 64, UK = 16, BN = 16;
// warps 0-3 epilogue, 4 idle, 5 MMA issuer + TMEM owner, 6-9 cp.async producers
constexpr int NTH = 320;
constexpr int MT = 1;       // 128-column M tiles per CTA (2 and 4, 512 / 1024-byte row reads, measured slower)
constexpr int TILE = BM * MT;
constexpr int OCC = 2;      // CTAs per SM (two CTAs' cp.async streams in flight)
constexpr int STAGES = (MT == 4 ? 3 : MT == 2 ? 6 : 8) / OCC;
constexpr int PF = 8;     // producer: kept-row indices prefetched one group of PF K blocks ahead
constexpr int A_BYTES = BK * BM * 2 * MT;     // 16 KB per M tile
constexpr int B_BYTES = BN * BK * 2;          // 2 KB per term
constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512 + (MAXCH + 1) * 4;
constexpr uint32_t TMEM_COLS = 32 * MT;       // 2 buffers x MT x 16 fp32 columns
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

struct Shape {
    int64_t m, n, ldw;
    int n_tiles, splits, n_chunks, B;
};

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
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d), "l"(ad), "l"(bd), "r"(IDESC), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}

// ---- compaction -----------------------------------------------------------------
// one thread per column: all B loads in flight at once, kept values stay in registers
__global__ void __launch_bounds__(CT) tc_compact_kernel(const float* __restrict__ x, int B, int64_t m, float t32,
                                                        uint16_t* __restrict__ xh, uint16_t* __restrict__ xl,
                                                        int* __restrict__ idx, int* __restrict__ kcnt,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ kept) {
    __shared__ int s_w[CT / 32];
    const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t c0 = (int64_t)c * CH;
    const int64_t i = c0 + tid;
    float v[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = (b < B && i < m) ? __ldg(x + (int64_t)b * m + i) : 0.f;
    bool keep = false;
    if (i < m) {
        float s = 0.f;
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (b < B) s = __fadd_rn(s, fabsf(v[b]));
        keep = !((float)__ddiv_rn((double)s, (double)B) <= t32);
        if (mask) mask[i] = keep ? 0 : 1;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < CT / 32; ++w) {
        const int t = s_w[w];
        off += w < warp ? t : 0;
        tot += t;
    }
    uint16_t* hrow = xh + (int64_t)c * 16 * CH;
    uint16_t* lrow = xl + (int64_t)c * 16 * CH;
    if (keep) {
        const int pos = off + __popc(bal & ((1u << lane) - 1u));
        idx[c0 + pos] = (int)i;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const uint16_t h = f32_to_bf16_rn(v[b]);
            hrow[(int64_t)b * CH + pos] = h;
            lrow[(int64_t)b * CH + pos] = f32_to_bf16_rn(v[b] - bf16_to_f32(h));
        }
    }
    const int padded = (tot + BK - 1) & ~(BK - 1);
    if (tid >= tot && tid < padded) {  // padding rows: a valid row index, zero activations
        idx[c0 + tid] = (int)c0;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            hrow[(int64_t)b * CH + tid] = 0;
            lrow[(int64_t)b * CH + tid] = 0;
        }
    }
    if (tid == 0) {
        kcnt[c] = tot;
        if (kept && tot) atomicAdd(kept, (unsigned long long)tot);
    }
}

// ---- contraction -------------------------------------------------------------------
// the CTA's it-th (unit, K block) pair -> global K block index, or -1 past the end
__device__ __forceinline__ int kb_range(const Shape& sh, int total, int u, int* kb1) {
    const int sp = u % sh.splits;
    *kb1 = (int)((int64_t)total * (sp + 1) / sh.splits);
    return (int)((int64_t)total * sp / sh.splits);
}

__global__ void __launch_bounds__(NTH, OCC)
tc_gemv_kernel(const __grid_constant__ CUtensorMap txh, const __grid_constant__ CUtensorMap txl,
               const uint16_t* __restrict__ w, const int* __restrict__ idx, const int* __restrict__ kcnt,
               const Shape sh, float* __restrict__ y, float* __restrict__ part, uint32_t* __restrict__ tickets) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + 2);
    int* s_last = reinterpret_cast<int*>(s_tmem + 1);
    int* s_pre = reinterpret_cast<int*>(smem + STAGES * STAGE_BYTES + 512);  // [n_chunks + 1] K-block prefix

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int units = sh.n_tiles * sh.splits;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 128 + 1);  // the producer threads' cp.async arrivals + the expect_tx arrival
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);
        }
        fence_mbar_init();
        int acc = 0;
        s_pre[0] = 0;
        for (int c = 0; c < sh.n_chunks; ++c) {
            acc += (kcnt[c] + BK - 1) / BK;
            s_pre[c + 1] = acc;
        }
    }
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&txh)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&txl)) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const int total = s_pre[sh.n_chunks];

    if (warp >= 6) {  // ---- producers: gather kept weight rows with cp.async, stage activations
        // warp pw stages rows 16*pw .. 16*pw+15 of each 64-row K block; one cp.async
        // instruction moves two whole 256-byte row segments (lanes 0-15 / 16-31: the
        // 16-byte chunks of rows 2k / 2k+1), so every L2 sector fetched is used in full
        const int pt = tid - 192, pw = pt >> 5, half_lane = lane >> 4, q = lane & 15;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        uint32_t it = 0;
        auto slice = [&](int kb) -> int64_t {
            int c = 0;
            while (s_pre[c + 1] <= kb) ++c;
            return (int64_t)c * CH + (int64_t)(kb - s_pre[c]) * BK;
        };
        const int my_row = 16 * pw + q;  // the row whose index this lane loads
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int i = u / sh.splits;
            int kb1;
            const int kb0 = kb_range(sh, total, u, &kb1);
            int cur[PF], nxt[PF];
#pragma unroll
            for (int g = 0; g < PF; ++g) cur[g] = kb0 + g < kb1 ? __ldg(idx + slice(kb0 + g) + my_row) : 0;
            for (int g0 = kb0; g0 < kb1; g0 += PF) {
#pragma unroll
                for (int g = 0; g < PF; ++g) nxt[g] = g0 + PF + g < kb1 ? __ldg(idx + slice(g0 + PF + g) + my_row) : 0;
#pragma unroll
                for (int g = 0; g < PF; ++g) {
                    const int kb = g0 + g;
                    if (kb < kb1) {
                        const uint32_t s = it % STAGES;
                        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                        uint8_t* st = smem + s * STAGE_BYTES;
                        const uint32_t sbase = smem_u32(st);
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int rl = 2 * k + half_lane;
                            const int r = 16 * pw + rl;
                            const int wr = __shfl_sync(0xffffffffu, cur[g], rl);
                            const uint16_t* src = w + (int64_t)wr * sh.ldw + (int64_t)i * TILE + q * 8;
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt)
                                cp_async16(sbase + mt * 16384 + (q >> 3) * 8192 + r * 128 + (((q & 7) ^ (r & 7)) << 4),
                                           src + mt * BM, pol);
                        }
                        if (pt == 0) {
                            int c = 0;
                            while (s_pre[c + 1] <= kb) ++c;
                            mbar_arrive_expect_tx(&full[s], 2 * B_BYTES);
                            tma_2d(st + A_BYTES, &txh, (kb - s_pre[c]) * BK, c * 16, &full[s]);
                            tma_2d(st + A_BYTES + B_BYTES, &txl, (kb - s_pre[c]) * BK, c * 16, &full[s]);
                        }
                        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s]))
                                     : "memory");
                        ++it;
                    }
                }
#pragma unroll
                for (int g = 0; g < PF; ++g) cur[g] = nxt[g];
            }
        }
    } else if (warp == 5) {  // ---- MMA issuer
        if (lane == 0) {
            uint32_t it = 0, lu = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
                int kb1;
                const int kb0 = kb_range(sh, total, u, &kb1);
                const uint32_t a = lu & 1;
                if (lu >= 2) mbar_wait(&acc_empty[a], ((lu >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN * MT;
                uint32_t acc = 0;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk) {
                        const uint64_t bh = sw128_desc(b0 + kk * UK * 2, 16, 1024);
                        const uint64_t bl = sw128_desc(b0 + B_BYTES + kk * UK * 2, 16, 1024);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint64_t ad = sw128_desc(a0 + mt * 16384 + kk * UK * 128, 8192, 1024);
                            tc_mma(d + mt * BN, ad, bh, acc);
                            tc_mma(d + mt * BN, ad, bl, 1u);
                        }
                        acc = 1u;
                    }
                    tc_commit(&empty[s]);
                }
                tc_commit(&acc_full[a]);
            }
        }
    } else if (warp < 4) {  // ---- epilogue: warp q4 reads TMEM lanes 32*q4 .. +31 = output columns
        const int q4 = warp;
        uint32_t lu = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
            const int i = u / sh.splits, sp = u % sh.splits;
            int kb1;
            const int kb0 = kb_range(sh, total, u, &kb1);
            const uint32_t a = lu & 1;
            mbar_wait(&acc_full[a], (lu >> 1) & 1);
            tc_fence_after();
            float v[MT][16];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                if (kb1 > kb0) {
                    tmem_ld16(tmem + ((uint32_t)(32 * q4) << 16) + (a * MT + mt) * BN, v[mt]);
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[mt][q] = 0.f;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
            const int64_t j0 = (int64_t)i * TILE + 32 * q4 + lane;
            if (sh.splits == 1) {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        if (b < sh.B) y[b * sh.n + j0 + mt * BM] = v[mt][b];
            } else {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        if (b < sh.B) part[((int64_t)sp * 16 + b) * sh.n + j0 + mt * BM] = v[mt][b];
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tid == 0) *s_last = atomicAdd(&tickets[i], 1u) == (uint32_t)(sh.splits - 1);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (*s_last) {  // the tile's last split: partials summed in ascending split order
                    __threadfence();
#pragma unroll 1
                    for (int mt = 0; mt < MT; ++mt) {
                        const int64_t j = j0 + mt * BM;
                        float acc[16];
#pragma unroll
                        for (int b = 0; b < 16; ++b) acc[b] = 0.f;
                        for (int k = 0; k < sh.splits; ++k) {
                            float pv[16];
#pragma unroll
                            for (int b = 0; b < 16; ++b)
                                pv[b] = b < sh.B ? __ldcg(part + ((int64_t)k * 16 + b) * sh.n + j) : 0.f;
#pragma unroll
                            for (int b = 0; b < 16; ++b) acc[b] += pv[b];
                        }
#pragma unroll
                        for (int b = 0; b < 16; ++b)
                            if (b < sh.B) y[b * sh.n + j] = acc[b];
                    }
                    if (tid == 0) tickets[i] = 0u;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
}

// ---- host -----------------------------------------------------------------------

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms = v > 0 ? v : 148;
    }
    return sms;
}

struct Plan {
    Shape sh;
    int64_t off_xl, off_idx, off_kcnt, off_part, bytes;  // workspace byte offsets (xh at 0)
};

constexpr int TC_MINKB = 2;       // K blocks per split at full density, at least
constexpr int TC_MIN_CTAS = 296;  // streaming CTAs wanted (2 per SM)

int64_t al256(int64_t b) { return (b + 255) & ~int64_t(255); }

Plan plan(const teal_gemv_batched_args* a) {
    Plan p;
    memset(&p, 0, sizeof(p));
    p.sh.m = a->m;
    p.sh.n = a->n;
    p.sh.ldw = a->ldw;
    p.sh.B = a->B;
    p.sh.n_tiles = (int)(a->n / TILE);
    p.sh.n_chunks = (int)((a->m + CH - 1) / CH);
    const int sms = sm_count();
    // splits: enough streaming CTAs for HBM (~64), at most one round; at least two K blocks per split
    int s = p.sh.n_tiles >= TC_MIN_CTAS ? 1 : (TC_MIN_CTAS + p.sh.n_tiles - 1) / p.sh.n_tiles;
    if (s * p.sh.n_tiles > sms * OCC) s = sms * OCC / p.sh.n_tiles > 0 ? sms * OCC / p.sh.n_tiles : 1;
    const int max_kb = (int)((a->m + BK - 1) / BK);
    if (s > max_kb / TC_MINKB) s = max_kb / TC_MINKB > 0 ? max_kb / TC_MINKB : 1;
    p.sh.splits = s;
    const int64_t xg = al256((int64_t)p.sh.n_chunks * 16 * CH * 2);
    p.off_xl = xg;
    p.off_idx = 2 * xg;
    p.off_kcnt = p.off_idx + al256((int64_t)p.sh.n_chunks * CH * 4);
    p.off_part = p.off_kcnt + al256(MAXCH * 4);
    p.bytes = p.off_part + (s > 1 ? al256((int64_t)s * 16 * a->n * 4) : 0);
    return p;
}

int make_map(CUtensorMap* map, const void* base, int n_chunks) {
    auto fn = prefill::encode_fn();
    TEAL_REQUIRE(fn, "teal_gemv_batched: cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[2] = {(cuuint64_t)CH, (cuuint64_t)n_chunks * 16};
    const cuuint64_t strides[1] = {(cuuint64_t)CH * 2};
    const cuuint32_t box[2] = {64u, 16u};
    const cuuint32_t es[2] = {1u, 1u};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    TEAL_REQUIRE(r == CUDA_SUCCESS, "teal_gemv_batched: tensor map encode failed (%d)", (int)r);
    return TEAL_OK;
}

}  // namespace gemvtc

// entry points used by teal_gemv_batched.cu
bool gemv_tc_eligible(const teal_gemv_batched_args* a) {
    using namespace gemvtc;
    // wide outputs only (gate / up / LM head): below 64 column tiles the mma.sync kernel of
    // teal_gemv_batched.cu is as fast (profiles/r02_config5_tcgen05.md)
    return a->w_dtype == TEAL_BF16 && a->B >= 4 && a->B <= 16 && a->n % TILE == 0 && a->n / TILE >= 64 &&
           a->ldw % 8 == 0 &&
           a->m <= (int64_t)MAXCH * CH && (reinterpret_cast<uintptr_t>(a->w) & 15) == 0;
}

int64_t gemv_tc_workspace_floats(const teal_gemv_batched_args* a, int64_t* tickets) {
    using namespace gemvtc;
    const Plan p = plan(a);
    if (tickets) *tickets = p.sh.n_tiles;
    return (p.bytes + 3) / 4;
}

int gemv_tc_launch(const teal_gemv_batched_args* a, cudaStream_t stream) {
    using namespace gemvtc;
    const Plan p = plan(a);
    TEAL_REQUIRE(a->ws && a->tickets, "teal_gemv_batched: ws and tickets are required");
    uint8_t* ws = reinterpret_cast<uint8_t*>(a->ws);
    TEAL_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 255) == 0, "teal_gemv_batched: ws must be 256-byte aligned");
    uint16_t* xh = reinterpret_cast<uint16_t*>(ws);
    uint16_t* xl = reinterpret_cast<uint16_t*>(ws + p.off_xl);
    int* idx = reinterpret_cast<int*>(ws + p.off_idx);
    int* kcnt = reinterpret_cast<int*>(ws + p.off_kcnt);
    float* part = reinterpret_cast<float*>(ws + p.off_part);
    tc_compact_kernel<<<p.sh.n_chunks, CT, 0, stream>>>(a->x, a->B, a->m, a->t32, xh, xl, idx, kcnt, a->mask, a->kept);
    int rc = check_launch("teal_gemv_batched (compact)");
    if (rc) return rc;
    CUtensorMap mh, ml;
    if ((rc = make_map(&mh, xh, p.sh.n_chunks))) return rc;
    if ((rc = make_map(&ml, xl, p.sh.n_chunks))) return rc;
    static unsigned long long attr = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("teal_gemv_batched (device)");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&attr, __ATOMIC_ACQUIRE) & bit)) {
        cudaFuncSetAttribute(tc_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        __atomic_fetch_or(&attr, bit, __ATOMIC_RELEASE);
    }
    const int units = p.sh.n_tiles * p.sh.splits;
    const int grid = units < sm_count() * OCC ? units : sm_count() * OCC;
    tc_gemv_kernel<<<grid, NTH, SMEM, stream>>>(mh, ml, (const uint16_t*)a->w, idx, kcnt, p.sh, a->y, part,
                                                a->tickets);
    return check_launch("teal_gemv_batched (tcgen05)");
}

}  // namespace teal
