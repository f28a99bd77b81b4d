// Fused threshold + sparse GEMV over input-channel-major weights (sm_100a).
//
// Replaces the reference's column-skipping numba GEMV
// (pkg/src/actsparse/kernel.py:30-44, `_skip_gemv`) and the seven masked
// `gated(name, a) @ W.T` products of model._forward (model.py:166-198).
//
// Work decomposition (one launch = one fused projection group, one wave):
//   The work space is (column tile, 32-channel group) over all segments,
//   flattened tile-major: F = ntiles * ceil(m/32) groups.  CTA c of G owns the
//   contiguous group range [c*F/G, (c+1)*F/G) — every SM gets the same number
//   of input channels to threshold and (in expectation) the same number of
//   surviving rows to stream, and a range spans at most `ntmax` tiles.
// Each CTA
//   1. loads its x slice (+ RMSNorm from fixed-order sum-of-squares partials),
//   2. thresholds keep_i = !(|h_i| <= t_seg) and compacts surviving channel
//      indices CTA-locally with warp ballot/popc (ascending order preserved),
//   3. streams only the surviving rows' TILE-column segments (1 KB for bf16 /
//      fp32, 512 B for int8): a producer warp issues one cp.async.bulk (TMA
//      engine, L2 evict-first) per surviving row into a shared-memory ring
//      guarded by full/empty mbarriers, and 8 consumer warps FMA the segments
//      into fp32 register accumulators — in-flight depth is the ring, not the
//      register file (odd shapes use a register-streaming variant),
//   4. reduces its warps per tile in fixed order; a tile shared by several CTAs
//      is finished by the last-arriving CTA (ticket counter) which sums the
//      contributors' fp32 partials in ascending CTA order — a deterministic
//      two-phase reduction — and runs the fused epilogue (store /
//      residual+sum-of-squares / SiLU(gate)*up / RoPE + KV-cache write).
// No tensor cores: a batch-1 matvec is ~1 flop/byte, far below the ridge.
#include "teal_common.cuh"
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

namespace teal {

int step_gemv_eligible(const teal_gemv_args* a, int64_t* ws_floats, int64_t* tickets, int* grid_out);
int step_gemv_single(const teal_gemv_args* a, cudaStream_t stream);

constexpr int NT_MAX = 4;  // max column tiles one CTA's range may span

struct KParams {
    teal_gemv_args a;
    int tile;       // TILE columns per tile
    int ntiles;     // tiles over all segments
    int tile0[4];   // first tile of each segment (+ sentinel)
    int gpt;        // 32-channel groups per tile = ceil(m / 32)
    int64_t F;      // total groups = ntiles * gpt
    int G;          // CTAs
    int maxc;       // partial slots per tile in ws
    int ns;         // bulk-copy ring slots (TMA path)
    int emax;       // smem entry-list capacity per CTA
    int ntmax;      // max tiles per CTA range
    int timeline;   // debug builds: record per-CTA phase timestamps
};

// Phase timeline probe (debug): g_teal_tl[cta*4 + k] = %globaltimer at
// k=0 entry, 1 first bulk copy issued, 2 streaming done, 3 exit.
__device__ unsigned long long g_teal_tl[4 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TEAL_TL(k)                                                           \
    do {                                                                     \
        if (P.timeline && blockIdx.x < 4096) g_teal_tl[blockIdx.x * 4 + (k)] = gtimer(); \
    } while (0)

__device__ __forceinline__ float silu(float z) { return z / (1.0f + expf(-z)); }

template <typename XT>
__device__ __forceinline__ float load_x(const void* x, int64_t i) {
    return to_f32<XT>(reinterpret_cast<const XT*>(x)[i]);
}

// CTA owning flattened group g under the equal-range split.
// (host guarantees (F + 1) * G < 2^32, so 32-bit unsigned arithmetic is exact)
__device__ __forceinline__ int owner_of(int64_t g, int64_t F, int G) {
    return (int)(((uint32_t)(g + 1) * (uint32_t)G - 1u) / (uint32_t)F);
}
__device__ __forceinline__ int range_begin(int c, int64_t F, int G) { return (int)((uint32_t)c * (uint32_t)F / (uint32_t)G); }

// Programmatic dependent launch: wait until the previous kernel in the stream
// has completed (and its writes are visible); let the next one start early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int seg_of_tile(const KParams& P, int t) {
    return (t >= P.tile0[1]) ? ((t >= P.tile0[2]) ? 2 : 1) : 0;
}

// Fused epilogue for one finished column tile (all threads of the CTA).
template <int TILE, int QN>
__device__ __forceinline__ void run_epilogue(const KParams& P, int seg, int tis, const float* tot,
                                             const float* tot_up, float* s_tile, float* s_scr) {
    const teal_gemv_args& A = P.a;
    const teal_seg& S = A.seg[seg];
    const int tid = threadIdx.x;
    const bool ct = tid < kThreads;  // column threads (a producer warp may follow)
    const int64_t c0 = (int64_t)tis * TILE;
    const int ncols = (int)min64(TILE, S.n - c0);
    const int epi = A.epilogue;
    if (epi == TEAL_EPI_STORE) {
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (ct && c < ncols) {
                float v = tot[q];
                if (S.col_scale) v *= S.col_scale[c0 + c];
                S.y[c0 + c] = v;
            }
        }
    } else if (epi == TEAL_EPI_RESID) {
        float sq = 0.f;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (ct && c < ncols) {
                float v = tot[q];
                if (S.col_scale) v *= S.col_scale[c0 + c];
                const float xn = A.resid[c0 + c] + v;
                A.resid[c0 + c] = xn;
                sq += xn * xn;
            }
        }
        const float ssum = block_sum(sq, s_scr);
        if (tid == 0 && A.ss_out) A.ss_out[tis] = ssum;
    } else if (epi == TEAL_EPI_SILU) {
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (ct && c < ncols) {
                float g = tot[q], u = tot_up[q];
                if (A.seg[0].col_scale) g *= A.seg[0].col_scale[c0 + c];
                if (A.seg[1].col_scale) u *= A.seg[1].col_scale[c0 + c];
                A.inter[c0 + c] = silu(g) * u;
            }
        }
    } else {  // TEAL_EPI_QKV: seg 0 = q, 1 = k, 2 = v
        __syncthreads();
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (ct && c < TILE) {
                float v = (c < ncols) ? tot[q] : 0.f;
                if (c < ncols && S.col_scale) v *= S.col_scale[c0 + c];
                s_tile[c] = v;
            }
        }
        __syncthreads();
        const int hd = A.head_dim, half = hd >> 1;
        const int pos = *A.pos;
        // a position past the cache would write into the next head's / layer's
        // slice (and read RoPE tables out of bounds): fail loudly instead
        if (pos < 0 || pos >= A.max_seq) asm volatile("trap;");
        const bool rope = (A.rope_cos != nullptr) && (seg < 2);
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (ct && c < ncols) {
                const int64_t col = c0 + c;
                const int d = (int)(col % hd);
                float v = s_tile[c];
                if (rope) {
                    const int dd = (d < half) ? d : d - half;
                    const float cs = A.rope_cos[(int64_t)pos * half + dd];
                    const float sn = A.rope_sin[(int64_t)pos * half + dd];
                    v = (d < half) ? (v * cs - s_tile[c + half] * sn) : (v * cs + s_tile[c - half] * sn);
                }
                if (seg == 0) {
                    A.q_out[col] = v;
                } else {
                    const int64_t kvh = col / hd;
                    const int64_t off = (kvh * A.max_seq + pos) * hd + d;
                    void* cache = (seg == 1) ? A.k_cache : A.v_cache;
                    if (A.kv_dtype == TEAL_BF16) reinterpret_cast<uint16_t*>(cache)[off] = f32_to_bf16_rn(v);
                    else reinterpret_cast<float*>(cache)[off] = v;
                }
            }
        }
        __syncthreads();
    }
}


// ---- step 4 (both kernels): per-tile warp reduction, split-K combine, epilogue
// Column work is done by threads [0, kThreads); every thread of the block
// reaches the barriers.  A tile shared by several CTAs: each contributor
// stores its fp32 partial into the tile's contiguous ws block; the last to
// arrive (ticket) stages the whole block into shared memory with coalesced
// 16-byte loads (one L2 round trip per `stage_cap` partials) and sums it per
// column in ascending-contributor order.
template <int TILE>
__device__ __forceinline__ void finish_tiles(const KParams& P, int c, int tfirst, int nt, float* s_red,
                                             const unsigned* s_wmask, const int* s_ncols, float* s_scr,
                                             int* s_last, float* stage, int stage_cap) {
    constexpr int QN = (TILE + kThreads - 1) / kThreads;
    const teal_gemv_args& A = P.a;
    const int tid = threadIdx.x;
    const bool ct = tid < kThreads;
    const int epi = A.epilogue;
    for (int k = 0; k < nt; ++k) {
        const int t = tfirst + k;
        const int sg = seg_of_tile(P, t);
        const int tis = t - P.tile0[sg];
        const unsigned wm = s_wmask[k];
        float tot[QN], tot_up[QN];
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int cc = tid + q * kThreads;
            float s = 0.f;
            if (ct && cc < TILE) {
#pragma unroll
                for (int w = 0; w < kWarps; ++w)
                    if (wm & (1u << w)) s += s_red[((size_t)k * kWarps + w) * TILE + cc];
            }
            tot[q] = s;
            tot_up[q] = 0.f;
        }
        const int cf = owner_of((int64_t)t * P.gpt, P.F, P.G);
        const int cn = owner_of((int64_t)(t + 1) * P.gpt - 1, P.F, P.G) - cf + 1;
        const bool direct = (cn == 1) && (epi != TEAL_EPI_SILU);
        if (!direct) {
            float* slot = A.ws + ((size_t)t * P.maxc + (c - cf)) * TILE;
#pragma unroll
            for (int q = 0; q < QN; ++q) {
                const int cc = tid + q * kThreads;
                if (ct && cc < TILE) __stcg(slot + cc, tot[q]);  // full tile: the block stays float4-loadable
            }
            __threadfence();
            __syncthreads();
            int gt = t, ut = -1, un = 0;
            if (epi == TEAL_EPI_SILU) {
                gt = P.tile0[0] + tis;
                ut = P.tile0[1] + tis;
                const int ucf = owner_of((int64_t)ut * P.gpt, P.F, P.G);
                un = owner_of((int64_t)(ut + 1) * P.gpt - 1, P.F, P.G) - ucf + 1;
            }
            const int gcf = owner_of((int64_t)gt * P.gpt, P.F, P.G);
            const int gn = owner_of((int64_t)(gt + 1) * P.gpt - 1, P.F, P.G) - gcf + 1;
            if (tid == 0) {
                const int tk = (epi == TEAL_EPI_SILU) ? tis : t;
                const unsigned expected = (unsigned)(gn + un);
                const unsigned prev = atomicAdd(&A.tickets[tk], 1u);
                const int last = (prev == expected - 1u);
                if (last) A.tickets[tk] = 0u;  // self-reset for the next launch
                *s_last = last;
            }
            __syncthreads();
            if (!*s_last) continue;
            __threadfence();
            // staged, coalesced combine of the gate (or only) block, then the up block
#pragma unroll
            for (int q = 0; q < QN; ++q) tot[q] = 0.f;
            for (int pass = 0; pass < 2; ++pass) {
                const int np = pass == 0 ? gn : un;
                if (np == 0) continue;
                const float4* blk = reinterpret_cast<const float4*>(A.ws + (size_t)(pass == 0 ? gt : ut) * P.maxc * TILE);
                for (int jb = 0; jb < np; jb += stage_cap) {
                    const int nb = min(stage_cap, np - jb);
                    const int n4 = nb * TILE / 4;
                    for (int i = tid; i < n4; i += blockDim.x)
                        reinterpret_cast<float4*>(stage)[i] = __ldcg(blk + (size_t)jb * (TILE / 4) + i);
                    __syncthreads();
#pragma unroll
                    for (int q = 0; q < QN; ++q) {
                        const int cc = tid + q * kThreads;
                        if (ct && cc < TILE) {
                            float s = (pass == 0) ? tot[q] : tot_up[q];
                            for (int j = 0; j < nb; ++j) s += stage[j * TILE + cc];
                            if (pass == 0) tot[q] = s;
                            else tot_up[q] = s;
                        }
                    }
                    __syncthreads();
                }
            }
        }
        run_epilogue<TILE, QN>(P, (epi == TEAL_EPI_SILU) ? 0 : sg, tis, tot, tot_up, s_red, s_scr);
        __syncthreads();
    }
}

// Per-CTA tile-slot table: weight base (column tile applied), row stride,
// valid columns.
template <typename WT, int TILE>
__device__ __forceinline__ void setup_slots(const KParams& P, int tfirst, int nt, const WT** s_wptr, int64_t* s_ldw,
                                            int* s_ncols, unsigned* s_wmask) {
    const int tid = threadIdx.x;
    if (tid < NT_MAX) {
        s_wmask[tid] = 0u;
        if (tid < nt) {
            const int t = tfirst + tid;
            const int sg = seg_of_tile(P, t);
            const int64_t col0 = (int64_t)(t - P.tile0[sg]) * TILE;
            const teal_seg& S = P.a.seg[sg];
            s_wptr[tid] = reinterpret_cast<const WT*>(S.w) + col0;
            s_ldw[tid] = S.ldw;
            s_ncols[tid] = (int)min64(TILE, S.n - col0);
        }
    }
}

// ============================================================================
// TMA-bulk kernel (wide rows): 8 consumer warps + 1 producer warp.
//   The producer warp thresholds its range 32 channels at a time (ballot) and
//   for every surviving channel issues one cp.async.bulk of the row segment
//   (TILE columns, SLOT bytes) into a ring of NS shared-memory slots, each
//   with a full/empty mbarrier pair; per-slot metadata carries h and the tile
//   slot.  Consumer warp w drains entries w, w+8, ... in order: wait full,
//   FMA the row segment (16 B chunks per lane) into fp32 register
//   accumulators, release the slot.  In-flight depth is the ring,
//   independent of registers, and the first copy is issued one L2 round trip
//   after launch.  Eight END entries terminate the consumers.
// ============================================================================
constexpr int kThreadsTMA = kThreads + 32;

// KB = row-segment kilobytes (1 or 2) for 2-4 byte weights (int8: half).
template <typename WT, int KB> struct TmaCfg {
    static constexpr int ESZ = (int)sizeof(WT);
    static constexpr int NCH = (ESZ == 1) ? KB : 2 * KB;  // 16-byte chunks per lane per row segment
    static constexpr int E16 = 16 / ESZ;                   // elements per chunk
    static constexpr int SLOT = NCH * 512;                 // bytes per row segment
    static constexpr int TILE = SLOT / ESZ;                // columns per tile
    static constexpr int NS = 64 / KB;                     // ring slots (power of two, >= 32)
};

template <typename WT, typename XT, int KB>
__global__ void __launch_bounds__(kThreadsTMA, 2) gemv_tma_kernel(const __grid_constant__ KParams P) {
    using Cfg = TmaCfg<WT, KB>;
    constexpr int ESZ = Cfg::ESZ, NCH = Cfg::NCH, E16 = Cfg::E16, SLOT = Cfg::SLOT, TILE = Cfg::TILE;
    constexpr int NS = Cfg::NS;
    constexpr int GB = 16;  // groups whose x is preloaded together

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* ring = smem_raw;                                                        // [NS][SLOT]
    float* s_red = reinterpret_cast<float*>(ring + (size_t)NS * SLOT);                     // [ntmax][8][TILE]
    float2* s_meta = reinterpret_cast<float2*>(s_red + (size_t)P.ntmax * kWarps * TILE);  // [NS] {h, slot}
    uint64_t* s_full = reinterpret_cast<uint64_t*>(s_meta + NS);                           // [NS]
    uint64_t* s_empty = s_full + NS;                                                       // [NS]
    __shared__ unsigned s_wmask[NT_MAX];
    __shared__ const WT* s_wptr[NT_MAX];
    __shared__ int64_t s_ldw[NT_MAX];
    __shared__ int s_ncols[NT_MAX];
    __shared__ float s_scr[kThreadsTMA / 32 + 1];
    __shared__ int s_last;

    const teal_gemv_args& A = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t g0 = range_begin(c, P.F, P.G);
    const int64_t g1 = range_begin(c + 1, P.F, P.G);
    const int ngroups = (int)(g1 - g0);
    const int tfirst = (int)((uint32_t)g0 / (uint32_t)P.gpt);
    const int nt = (int)((uint32_t)(g1 - 1) / (uint32_t)P.gpt) - tfirst + 1;

    if (tid == 0) TEAL_TL(0);
    setup_slots<WT, TILE>(P, tfirst, nt, s_wptr, s_ldw, s_ncols, s_wmask);
    if (tid < NS) {
        mbar_init(&s_full[tid], 1);
        mbar_init(&s_empty[tid], 1);
    }
    fence_mbar_init();
    pdl_trigger();
    pdl_wait();  // x, ss_part, ws/tickets and outputs belong to the previous kernel until here
    __syncthreads();

    if (warp == kWarps) {
        // ===================== producer warp =====================
        const bool rms = (A.prologue == TEAL_PRO_RMSNORM);
        const uint64_t pol = l2_evict_first_policy();
        const int gpt = P.gpt;
        const int64_t m = A.m;
        // (tile, group-in-tile) of the first group; advanced incrementally
        int tile_b = tfirst, gin_b = (int)(g0 - (int64_t)tfirst * gpt);
        float xv[GB], nv[GB];
        auto preload = [&](int jb) {
            int tl = tile_b, gn = gin_b;
#pragma unroll
            for (int q = 0; q < GB; ++q) {
                xv[q] = 0.f;
                nv[q] = 1.f;
                if (jb + q < ngroups) {
                    const int64_t ch = (int64_t)gn * 32 + lane;
                    if (ch < m) {
                        xv[q] = load_x<XT>(A.x, ch);
                        if (rms) nv[q] = A.norm_scale[ch];
                    }
                }
                if (++gn == gpt) { gn = 0; ++tl; }
            }
            (void)tl;
        };
        preload(0);
        float rden = 1.f;
        if (rms) {
            float s = 0.f;
            if (lane == 0) {
                for (int p = 0; p < A.ss_count; ++p) s += A.ss_part[p];
                s = sqrtf(s / (float)A.m + A.eps);
            }
            rden = __shfl_sync(0xffffffffu, s, 0);
        }
        unsigned kcnt0 = 0, kcnt1 = 0, kcnt2 = 0;
        int e = 0;  // next entry index (warp-uniform)
        for (int jb = 0; jb < ngroups; jb += GB) {
            if (jb) preload(jb);
#pragma unroll
            for (int q = 0; q < GB; ++q) {
                if (jb + q >= ngroups) break;
                const int tile = tile_b;
                const int64_t ch = (int64_t)gin_b * 32 + lane;
                if (++gin_b == gpt) { gin_b = 0; ++tile_b; }
                const int sg = seg_of_tile(P, tile);
                const bool chv = ch < m;
                const float h = rms ? (xv[q] / rden * nv[q]) : xv[q];
                const bool keep = chv && !(fabsf(h) <= A.seg[sg].t32);
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (tile == P.tile0[sg]) {  // first tile of its segment: bookkeeping once per channel
                    uint32_t* bits = A.seg[sg].dbg_bits;
                    if (bits && lane == 0) bits[(ch - lane) >> 5] = bal;
                    if (sg == 0 && A.dbg_h && chv) A.dbg_h[ch] = h;
                    const unsigned pc = __popc(bal);
                    kcnt0 += (sg == 0) ? pc : 0u;
                    kcnt1 += (sg == 1) ? pc : 0u;
                    kcnt2 += (sg == 2) ? pc : 0u;
                }
                if (keep) {
                    const int k = tile - tfirst;
                    const int me = e + __popc(bal & ((1u << lane) - 1u));
                    const int s = me & (NS - 1);
                    const int use = me / NS;
                    if (use > 0) mbar_wait(&s_empty[s], (uint32_t)((use - 1) & 1));
                    s_meta[s] = make_float2(h, __int_as_float(k));
                    const uint32_t bytes = (uint32_t)(s_ncols[k] * ESZ);
                    mbar_arrive_expect_tx(&s_full[s], bytes);
                    bulk_g2s(ring + (size_t)s * SLOT, s_wptr[k] + ch * s_ldw[k], bytes, &s_full[s], pol);
                    if (me == 0) TEAL_TL(1);
                }
                e += __popc(bal);
            }
        }
        // END markers: entry e + w belongs to consumer warp (e + w) % 8
        if (lane < kWarps) {
            const int me = e + lane;
            const int s = me & (NS - 1);
            const int use = me / NS;
            if (use > 0) mbar_wait(&s_empty[s], (uint32_t)((use - 1) & 1));
            s_meta[s] = make_float2(0.f, __int_as_float(-1));
            mbar_arrive_expect_tx(&s_full[s], 0u);  // (the same release-arrive as a data entry, no bytes)
        }
        if (lane == 0) {
            if (kcnt0 && A.seg[0].kept) atomicAdd(A.seg[0].kept, (unsigned long long)kcnt0);
            if (kcnt1 && A.seg[1].kept) atomicAdd(A.seg[1].kept, (unsigned long long)kcnt1);
            if (kcnt2 && A.seg[2].kept) atomicAdd(A.seg[2].kept, (unsigned long long)kcnt2);
        }
    } else {
        // ===================== consumer warps =====================
        float acc[NCH * E16];
#pragma unroll
        for (int i = 0; i < NCH * E16; ++i) acc[i] = 0.f;
        int cur = -1;
        auto flush = [&]() {
            if (cur < 0) return;
            float* dst = s_red + ((size_t)cur * kWarps + warp) * TILE;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const int col = (ch * 512 + lane * 16) / ESZ;
#pragma unroll
                for (int i = 0; i < E16; i += 4)
                    *reinterpret_cast<float4*>(dst + col + i) =
                        make_float4(acc[ch * E16 + i], acc[ch * E16 + i + 1], acc[ch * E16 + i + 2], acc[ch * E16 + i + 3]);
            }
#pragma unroll
            for (int i = 0; i < NCH * E16; ++i) acc[i] = 0.f;
            if (lane == 0) atomicOr(&s_wmask[cur], 1u << warp);
        };
        for (int e = warp;; e += kWarps) {
            const int s = e & (NS - 1);
            mbar_wait(&s_full[s], (uint32_t)((e / NS) & 1));
            const float2 meta = s_meta[s];
            const int k = __float_as_int(meta.y);
            if (k < 0) break;
            if (k != cur) {
                flush();
                cur = k;
            }
            const int nbytes = s_ncols[k] * ESZ;
            const unsigned char* row = ring + (size_t)s * SLOT;
            uint4 d[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const int off = ch * 512 + lane * 16;
                d[ch] = (off < nbytes) ? *reinterpret_cast<const uint4*>(row + off) : make_uint4(0u, 0u, 0u, 0u);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[s]);
            const float hx = meta.x;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const uint32_t w4[4] = {d[ch].x, d[ch].y, d[ch].z, d[ch].w};
                float* a = acc + ch * E16;
                if constexpr (ESZ == 2) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        a[2 * i] = fmaf(hx, bf16_lo(w4[i]), a[2 * i]);
                        a[2 * i + 1] = fmaf(hx, bf16_hi(w4[i]), a[2 * i + 1]);
                    }
                } else if constexpr (ESZ == 4) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = fmaf(hx, __uint_as_float(w4[i]), a[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            a[4 * i + b] = fmaf(hx, (float)(int8_t)((w4[i] >> (8 * b)) & 0xffu), a[4 * i + b]);
                }
            }
        }
        flush();
    }
    __syncthreads();
    if (tid == 0) TEAL_TL(2);
    // the ring is idle now: reuse it to stage split-K partials
    finish_tiles<TILE>(P, c, tfirst, nt, s_red, s_wmask, s_ncols, s_scr, &s_last,
                       reinterpret_cast<float*>(ring), (NS * SLOT) / (TILE * 4));
    if (tid == 0) TEAL_TL(3);
}

// ============================================================================
// Register-streaming kernel (scalar rows: any n / ldw / alignment).
// ============================================================================
template <typename WT, typename XT>
__global__ void __launch_bounds__(kThreads, 2) gemv_simple_kernel(const __grid_constant__ KParams P) {
    constexpr int NV = 8;
    constexpr int TILE = 32 * NV;
    constexpr int U = 8;  // rows in flight per warp

    extern __shared__ __align__(32) unsigned char smem_raw[];
    float* s_red = reinterpret_cast<float*>(smem_raw);                              // [ntmax][kWarps][TILE]
    int* s_idx = reinterpret_cast<int*>(s_red + (size_t)P.ntmax * kWarps * TILE);  // [emax]
    float* s_val = reinterpret_cast<float*>(s_idx + P.emax);                        // [emax]
    __shared__ int s_wcnt[kWarps];
    __shared__ int s_tbeg[NT_MAX + 1];
    __shared__ unsigned s_wmask[NT_MAX];
    __shared__ const WT* s_wptr[NT_MAX];
    __shared__ int64_t s_ldw[NT_MAX];
    __shared__ int s_ncols[NT_MAX];
    __shared__ float s_scr[kWarps + 1];
    __shared__ float s_rden;
    __shared__ int s_last;
    __shared__ __align__(16) float s_stage[4 * TILE];

    const teal_gemv_args& A = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t g0 = range_begin(c, P.F, P.G);
    const int64_t g1 = range_begin(c + 1, P.F, P.G);
    const int64_t ngroups = g1 - g0;
    const int tfirst = (int)((uint32_t)g0 / (uint32_t)P.gpt);
    const int nt = (int)((uint32_t)(g1 - 1) / (uint32_t)P.gpt) - tfirst + 1;
    const bool rms = (A.prologue == TEAL_PRO_RMSNORM);

    setup_slots<WT, TILE>(P, tfirst, nt, s_wptr, s_ldw, s_ncols, s_wmask);
    pdl_trigger();
    pdl_wait();
    if (rms && tid == 0) {
        float s = 0.f;
        for (int p = 0; p < A.ss_count; ++p) s += A.ss_part[p];
        s_rden = sqrtf(s / (float)A.m + A.eps);
    }
    __syncthreads();
    const float rden = rms ? s_rden : 1.f;

    // threshold + CTA-local compaction, 8 groups (one per warp) per round
    int base = 0;
    unsigned kcnt0 = 0, kcnt1 = 0, kcnt2 = 0;
    const int64_t rounds = (ngroups + kWarps - 1) / kWarps;
    for (int64_t j = 0; j < rounds; ++j) {
        const int64_t gi = g0 + j * kWarps + warp;
        const bool valid = gi < g1;
        int tile = 0, sg = 0;
        int64_t ch = 0;
        bool chv = false;
        float h = 0.f;
        if (valid) {
            tile = (int)(gi / P.gpt);
            ch = (gi - (int64_t)tile * P.gpt) * 32 + lane;
            sg = seg_of_tile(P, tile);
            chv = ch < A.m;
            if (chv) {
                h = load_x<XT>(A.x, ch);
                if (rms) h = h / rden * A.norm_scale[ch];
            }
        }
        const bool keep = chv && !(fabsf(h) <= A.seg[sg].t32);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        if (valid && tile == P.tile0[sg]) {
            uint32_t* bits = A.seg[sg].dbg_bits;
            if (bits && lane == 0) bits[(ch - lane) >> 5] = bal;
            if (sg == 0 && A.dbg_h && chv) A.dbg_h[ch] = h;
            const unsigned pc = __popc(bal);
            kcnt0 += (sg == 0) ? pc : 0u;
            kcnt1 += (sg == 1) ? pc : 0u;
            kcnt2 += (sg == 2) ? pc : 0u;
        }
        __syncthreads();
        int off = base, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int cw = s_wcnt[w];
            off += (w < warp) ? cw : 0;
            tot += cw;
        }
        if (valid && lane == 0 && (gi == g0 || (gi % P.gpt) == 0)) s_tbeg[tile - tfirst] = off;
        if (keep) {
            const int pos = off + __popc(bal & ((1u << lane) - 1u));
            s_idx[pos] = (int)ch;
            s_val[pos] = h;
        }
        base += tot;
        __syncthreads();
    }
    if (lane == 0) {
        if (kcnt0 && A.seg[0].kept) atomicAdd(A.seg[0].kept, (unsigned long long)kcnt0);
        if (kcnt1 && A.seg[1].kept) atomicAdd(A.seg[1].kept, (unsigned long long)kcnt1);
        if (kcnt2 && A.seg[2].kept) atomicAdd(A.seg[2].kept, (unsigned long long)kcnt2);
    }
    if (tid == 0) s_tbeg[nt] = base;
    __syncthreads();
    const int count = base;

    float acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.f;
    int cur = -1;
    auto flush = [&]() {
        if (cur < 0) return;
        float* dst = s_red + ((size_t)cur * kWarps + warp) * TILE;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            dst[v * 32 + lane] = acc[v];
            acc[v] = 0.f;
        }
        if (lane == 0) atomicOr(&s_wmask[cur], 1u << warp);
    };
    for (int r = warp * U; r < count; r += kWarps * U) {
        WT raw[U][NV];
        float xv[U];
        int ks[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int rr = r + u;
            ks[u] = -1;
            xv[u] = 0.f;
#pragma unroll
            for (int v = 0; v < NV; ++v) raw[u][v] = WT(0);
            if (rr < count) {
                int k = 0;
#pragma unroll
                for (int s = 1; s < NT_MAX; ++s) k += (s < nt && rr >= s_tbeg[s]) ? 1 : 0;
                ks[u] = k;
                const WT* row = s_wptr[k] + (int64_t)s_idx[rr] * s_ldw[k];
                const int ncols = s_ncols[k];
                xv[u] = s_val[rr];
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    if (v * 32 + lane < ncols) raw[u][v] = __ldg(row + v * 32 + lane);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (ks[u] >= 0) {
                if (ks[u] != cur) {
                    flush();
                    cur = ks[u];
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) acc[v] = fmaf(xv[u], to_f32<WT>(raw[u][v]), acc[v]);
            }
        }
    }
    flush();
    __syncthreads();
    finish_tiles<TILE>(P, c, tfirst, nt, s_red, s_wmask, s_ncols, s_scr, &s_last, s_stage, 4);
}

// ---- host side ---------------------------------------------------------------
static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return TEAL_ECUDA;
    }
    return TEAL_OK;
}

static int esz_of(int dt) { return dt == TEAL_F32 ? 4 : dt == TEAL_BF16 ? 2 : 1; }

// Bulk copies need 16-byte aligned row segments of a multiple of 16 bytes.
static bool seg_wide_ok(const teal_gemv_args* a) {
    const int ve = 16 / esz_of(a->w_dtype);
    for (int s = 0; s < a->nseg; ++s) {
        const teal_seg& g = a->seg[s];
        if (g.n % ve) return false;
        if (g.ldw % ve) return false;
        if (reinterpret_cast<uintptr_t>(g.w) % 16) return false;
    }
    return true;
}

// Programmatic dependent launch between consecutive GEMV launches (the next
// launch's prologue overlaps this one's tail): always on.
int pdl_enabled() { return 1; }

// 1 KB bulk-copy slots per row segment (TmaCfg::NS = 64 slots)
static int slot_kb() { return 1; }

static int tile_width(const teal_gemv_args* a) {
    const int esz = esz_of(a->w_dtype);
    if (seg_wide_ok(a)) return (esz == 1 ? 512 : 1024) * slot_kb() / esz;  // one bulk slot per row segment
    return 32 * 8;                                                        // register path: 8 columns per lane
}

static int sm_count_cached() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        cudaGetLastError();
    }
    return sms;
}

// Resolve the decomposition for `a` (ctas <= 0: auto).
static int plan(const teal_gemv_args* a, KParams* P) {
    const int tile = tile_width(a);
    int t = 0;
    for (int s = 0; s < a->nseg; ++s) {
        P->tile0[s] = t;
        t += (int)((a->seg[s].n + tile - 1) / tile);
    }
    for (int s = a->nseg; s < 4; ++s) P->tile0[s] = t;
    P->tile = tile;
    P->ntiles = t;
    P->gpt = (int)((a->m + 31) / 32);
    P->F = (int64_t)t * P->gpt;
    int64_t G = a->ctas;
    if (G <= 0) G = (int64_t)sm_count_cached() * 2;  // 2 resident CTAs per SM
    if (G > P->F) G = P->F;
    if ((P->F + 1) * G >= (int64_t)1 << 32) G = ((int64_t)1 << 32) / (P->F + 1) - 1;  // keep index math 32-bit
    // a range must not span more than NT_MAX tiles
    const int64_t min_g = (P->F + (int64_t)(NT_MAX - 1) * P->gpt - 1) / ((int64_t)(NT_MAX - 1) * P->gpt);
    if (G < min_g) G = min_g;
    P->G = (int)G;
    const int64_t per = (P->F + G - 1) / G;  // max groups per CTA
    P->ntmax = (int)min64((per + P->gpt - 1) / P->gpt + 1, (int64_t)t);
    if (P->ntmax > NT_MAX) P->ntmax = NT_MAX;
    P->emax = (int)(per * 32);
    P->maxc = (int)((P->gpt * G + P->F - 1) / P->F + 1);
    P->ns = 64 / slot_kb();  // TMA ring slots (TmaCfg::NS)
    P->timeline = 0;  // (debug probe: set to 1 in a build to record phase stamps)
    return TEAL_OK;
}

static bool use_tma(const teal_gemv_args* a) { return seg_wide_ok(a); }

static size_t smem_bytes(const KParams& P, bool tma) {
    if (tma) {
        const size_t slot = (size_t)P.tile * esz_of(P.a.w_dtype);
        return (size_t)P.ns * slot + (size_t)P.ntmax * kWarps * P.tile * 4 + (size_t)P.ns * (8 + 16);
    }
    return (size_t)P.ntmax * kWarps * P.tile * 4 + (size_t)P.emax * 8;
}

template <typename K>
static int launch_kernel(K kernel, const KParams& P, int threads, size_t smem, cudaStream_t st) {
    if (smem > 227 * 1024) {
        set_error("teal_fused_gemv: %zu bytes of shared memory needed; raise ctas", smem);
        return TEAL_EINVAL;
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, P);
    return check_launch("teal_fused_gemv");
}

template <typename WT, typename XT>
static int launch(const KParams& P, cudaStream_t st) {
    if (use_tma(&P.a)) {
        if (slot_kb() == 2) return launch_kernel(gemv_tma_kernel<WT, XT, 2>, P, kThreadsTMA, smem_bytes(P, true), st);
        return launch_kernel(gemv_tma_kernel<WT, XT, 1>, P, kThreadsTMA, smem_bytes(P, true), st);
    }
    return launch_kernel(gemv_simple_kernel<WT, XT>, P, kThreads, smem_bytes(P, false), st);
}

static int validate(const teal_gemv_args* a) {
    TEAL_REQUIRE(a, "teal_fused_gemv: null args");
    TEAL_REQUIRE(a->nseg >= 1 && a->nseg <= 3, "teal_fused_gemv: nseg must be 1..3, got %d", a->nseg);
    TEAL_REQUIRE(a->m >= 1, "teal_fused_gemv: m must be >= 1");
    TEAL_REQUIRE(a->w_dtype == TEAL_F32 || a->w_dtype == TEAL_BF16 || a->w_dtype == TEAL_I8,
                 "teal_fused_gemv: unsupported weight dtype %d", a->w_dtype);
    TEAL_REQUIRE(a->x_dtype == TEAL_F32 || a->x_dtype == TEAL_BF16, "teal_fused_gemv: unsupported x dtype %d",
                 a->x_dtype);
    for (int s = 0; s < a->nseg; ++s) {
        const teal_seg& g = a->seg[s];
        TEAL_REQUIRE(g.w && g.n >= 1 && g.ldw >= g.n, "teal_fused_gemv: bad segment %d (n=%lld ldw=%lld)", s,
                     (long long)g.n, (long long)g.ldw);
        TEAL_REQUIRE(g.t32 == g.t32 && (!(g.t32 < 0.f) || g.t32 == -INFINITY),
                     "teal_fused_gemv: threshold must be >= 0 (or -inf for dense), got %g", (double)g.t32);
        TEAL_REQUIRE(a->w_dtype != TEAL_I8 || g.col_scale, "teal_fused_gemv: int8 weights need col_scale");
        if (a->epilogue == TEAL_EPI_STORE) TEAL_REQUIRE(g.y, "teal_fused_gemv: STORE epilogue needs seg[%d].y", s);
    }
    TEAL_REQUIRE(a->w_dtype != TEAL_I8 || seg_wide_ok(a),
                 "teal_fused_gemv: int8 rows need n%%16==0, ldw%%16==0 and 16-byte alignment");
    return TEAL_OK;
}

}  // namespace teal

using namespace teal;

extern "C" {

const char* teal_last_error(void) { return g_err; }
int teal_abi_version(void) { return TEAL_ABI_VERSION; }
int teal_device_sm_count(int device) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return sms;
}

int teal_gemv_tile_width(const teal_gemv_args* a) { return a ? tile_width(a) : -1; }

int teal_debug_timeline(unsigned long long* host_dst, int n) {
    TEAL_REQUIRE(host_dst && n >= 0 && n <= 4 * 4096, "teal_debug_timeline: bad arguments");
    cudaError_t e = cudaMemcpyFromSymbol(host_dst, g_teal_tl, (size_t)n * 8);
    if (e != cudaSuccess) {
        set_error("teal_debug_timeline: %s", cudaGetErrorString(e));
        return TEAL_ECUDA;
    }
    return TEAL_OK;
}

int teal_gemv_workspace(const teal_gemv_args* a, int* ctas, int64_t* ws_floats, int64_t* tickets) {
    int st = validate(a);
    if (st) return st;
    KParams P;
    memset(&P, 0, sizeof(P));
    plan(a, &P);
    int64_t wsf = (int64_t)P.ntiles * P.maxc * P.tile, ntk = P.ntiles;
    int64_t wsf2 = 0, ntk2 = 0;
    int g2 = 0;
    if (teal::step_gemv_eligible(a, &wsf2, &ntk2, &g2) == 0) {  // single-GEMV path sizes
        if (wsf2 > wsf) wsf = wsf2;
        if (ntk2 > ntk) ntk = ntk2;
    }
    if (ctas) *ctas = P.G;
    if (ws_floats) *ws_floats = wsf;
    if (tickets) *tickets = ntk;
    return TEAL_OK;
}

int teal_fused_gemv(const teal_gemv_args* a, cudaStream_t stream) {
    int st = validate(a);
    if (st) return st;
    if (a->prologue == TEAL_PRO_RMSNORM) {
        TEAL_REQUIRE(a->x_dtype == TEAL_F32 && a->norm_scale && a->ss_part && a->ss_count >= 1,
                     "teal_fused_gemv: RMSNORM prologue needs fp32 x, norm_scale and ss_part");
    } else {
        TEAL_REQUIRE(a->prologue == TEAL_PRO_PLAIN, "teal_fused_gemv: unknown prologue %d", a->prologue);
    }
    switch (a->epilogue) {
        case TEAL_EPI_STORE:
            break;
        case TEAL_EPI_RESID:
            TEAL_REQUIRE(a->nseg == 1 && a->resid, "teal_fused_gemv: RESID epilogue needs one segment and resid");
            break;
        case TEAL_EPI_SILU:
            TEAL_REQUIRE(a->nseg == 2 && a->seg[0].n == a->seg[1].n && a->inter,
                         "teal_fused_gemv: SILU epilogue needs two equal segments (gate, up) and inter");
            break;
        case TEAL_EPI_QKV:
            TEAL_REQUIRE(a->nseg == 3 && a->q_out && a->k_cache && a->v_cache && a->pos && a->head_dim > 0,
                         "teal_fused_gemv: QKV epilogue needs q_out, k/v caches, pos, head_dim");
            break;
        default:
            TEAL_REQUIRE(false, "teal_fused_gemv: unknown epilogue %d", a->epilogue);
    }
    KParams P;
    memset(&P, 0, sizeof(P));
    P.a = *a;
    plan(a, &P);
    if (a->epilogue == TEAL_EPI_QKV)
        TEAL_REQUIRE(P.tile % a->head_dim == 0 && a->seg[0].n % a->head_dim == 0 && a->seg[1].n % a->head_dim == 0,
                     "teal_fused_gemv: QKV epilogue needs head_dim | tile (%d) and head_dim | n", P.tile);
    TEAL_REQUIRE(a->ws && a->tickets, "teal_fused_gemv: ws and tickets are required");
    // Plain single-projection calls (one segment, PLAIN prologue, STORE
    // epilogue, fp32 x, bf16/fp32/int8 rows) run on the persistent step
    // kernel's streaming core (gemv_one_kernel, teal_step.cu), documented in
    // include/teal_b200.h; the fused prologue/epilogue variants run here.
    if (teal::step_gemv_eligible(a, nullptr, nullptr, nullptr) == 0)
        return teal::step_gemv_single(a, stream);
    const bool xb = (a->x_dtype == TEAL_BF16);
    if (a->w_dtype == TEAL_BF16) return xb ? launch<uint16_t, uint16_t>(P, stream) : launch<uint16_t, float>(P, stream);
    if (a->w_dtype == TEAL_F32) return xb ? launch<float, uint16_t>(P, stream) : launch<float, float>(P, stream);
    return xb ? launch<int8_t, uint16_t>(P, stream) : launch<int8_t, float>(P, stream);
}

int teal_sparse_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw, const void* x, int x_dtype,
                     float t32, float* y, const float* col_scale, float* ws, uint32_t* tickets, int ctas,
                     unsigned long long* kept, cudaStream_t stream) {
    teal_gemv_args a;
    memset(&a, 0, sizeof(a));
    a.w_dtype = w_dtype;
    a.x_dtype = x_dtype;
    a.x = x;
    a.m = m;
    a.nseg = 1;
    a.seg[0].w = w;
    a.seg[0].ldw = ldw;
    a.seg[0].n = n;
    a.seg[0].t32 = t32;
    a.seg[0].y = y;
    a.seg[0].col_scale = col_scale;
    a.seg[0].kept = kept;
    a.prologue = TEAL_PRO_PLAIN;
    a.epilogue = TEAL_EPI_STORE;
    a.ctas = ctas;
    a.ws = ws;
    a.tickets = tickets;
    return teal_fused_gemv(&a, stream);
}

int teal_dense_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw, const void* x, int x_dtype,
                    float* y, const float* col_scale, float* ws, uint32_t* tickets, int ctas, cudaStream_t stream) {
    return teal_sparse_gemv(w, w_dtype, m, n, ldw, x, x_dtype, -INFINITY, y, col_scale, ws, tickets, ctas, nullptr,
                            stream);
}

}  // extern "C"
