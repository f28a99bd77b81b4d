// Persistent decode-step kernel (sm_100a): one cooperative launch per token.
//
// Replaces the per-projection launch sequence of a decode step — the seven
// `gated(name, a) @ W.T` products of model._forward
// (pkg/src/actsparse/model.py:158-198) with their RMSNorm / SiLU*up /
// residual epilogues, causal attention (model.py:135-150, one query row over
// a KV cache), the dense LM head and greedy argmax.
//
// Execution model
//   * grid = resident CTAs (cooperative launch); every CTA walks the plan's
//     phase list (per layer: qkv, attention, o, gate/up, down; then LM head).
//   * GEMV phase: the flattened (column tile, 32-channel group) space is cut
//     into G equal contiguous ranges, CTA c owning [c*F/G, (c+1)*F/G) — equal
//     input channels to threshold and, in expectation, equal kept rows to
//     stream, so CTAs finish a phase together.  A range spans one or two
//     tiles; layer outputs are int64 fixed-point accumulators every
//     contributor adds into (the consumer applies the epilogue while loading
//     its input); the LM head's split tiles are finished by the last-arriving
//     contributor (ticket), summing fp32 partials in contributor order.
//   * Dependencies are counters bumped (release) by tile epilogues and
//     polled (acquire) before a slice reads its input rows: o waits only for
//     the attention groups its rows come from, down only for the gate/up
//     tiles its rows come from, attention for kv-group g only for the q/k/v
//     tiles of g.  The RMSNorm inputs (residual + sum of squares) are the
//     only global joins.  Every wait targets an earlier phase and all CTAs
//     are resident, so the schedule cannot deadlock; the last CTA to leave
//     resets the counters, so a CUDA graph of the launch replays per token.
//
// Streaming core (per CTA slice segment = one tile x a row range):
//   1. h_i = x_i or RMSNorm(x)_i (x / sqrt(sum(ss)/m + eps) * g, fixed-order
//      sum of sum-of-squares partials); keep_lo/hi = !(|h_i| <= t_lo/hi)
//      (closed prune boundary, NaN kept); ordered CTA-local compaction with
//      warp ballot/popc;
//   2. warp w takes kept rows w*U.., w*U + NW*U.., register-streamed: each
//      lane issues 16-byte (bf16/fp32), 8-byte (int8) or 4-byte (int4)
//      ld.global.nc.L1::no_allocate loads with an L2 evict-first policy, the
//      next U rows' loads in flight before the current U are consumed; only
//      the kept half of a row is loaded; fp32 FMA into per-lane registers;
//   3. fixed-order cross-warp reduction -> TW column sums, then either an
//      int64 fixed-point red.add into the tile's accumulator (ACC outputs:
//      order-independent, so deterministic, and nobody waits) or, for the
//      LM head, fp32 partials summed in contributor order by the tile's last
//      arriving contributor (ticket).
// No tensor cores: a batch-1 matvec is ~1 flop/byte.
#include "teal_common.cuh"
#include <string.h>
#include <stdlib.h>

namespace teal {
namespace step {

constexpr int TW = TEAL_STEP_TW;  // columns per tile
constexpr int TH = TW / 2;        // columns per half
constexpr int NT = 256;           // threads per CTA (== TW: one column per thread in epilogues)
constexpr int NW = NT / 32;
constexpr int MAXR = 1024;        // rows per compaction chunk
constexpr int GSC_MAX = 9;        // int4 row groups one chunk can touch (group >= 128)
constexpr int ATT_MAXG = 8;
constexpr int ATT_MAXHD = 128;
constexpr int ATT_MAXCHUNK = 256;
constexpr int ATT_STAGE = 16384;  // bytes of K (and of V) staged per attention unit
                                  // (engine: chunk <= 16384 / (hd * kv bytes))
constexpr int XS_MAX = 8192;      // PRO_RMS_ACC: the CTA's copy of x' (m <= XS_MAX)
constexpr int CONTRIB = TEAL_STEP_CONTRIB;
static_assert(NT == TW, "epilogues map one thread per tile column");

struct Smem {
    union {
        struct {
            int idx[MAXR];    // row - r0 | keep_lo << 30 | keep_hi << 31
            float h[MAXR];
            float gsc[GSC_MAX * TW];  // int4: scales of the chunk's row groups
            float xs[XS_MAX];         // PRO_RMS_ACC: x' = x + fx(in_acc), all m channels
        } g;
        struct {
            float q[ATT_MAXG * ATT_MAXHD];
            float sc[ATT_MAXG * ATT_MAXCHUNK];
            uint4 k[ATT_STAGE / 16 + ATT_MAXCHUNK];  // K rows (cache dtype), each padded by 16 B
            uint4 v[ATT_STAGE / 16];                 // V rows of the chunk
        } a;
    } u;
    float red[NW * TW];
    float col[TW];
    float am[ATT_MAXG], al[ATT_MAXG];
    float scr[NW + 1];
    int wcnt[NW];
    float rden;
    int last;
};
constexpr size_t kSmemBytes = sizeof(Smem);
// The CTA's shared memory seen through its declared address space: noinline
// functions must not take Smem& parameters (the pointer would be generic and
// every access a generic LD/ST instead of LDS/STS).
__device__ __forceinline__ Smem& smem() {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    return *reinterpret_cast<Smem*>(smem_raw);
}

__device__ __forceinline__ unsigned long long gtimer_() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Each counter lives in its own 128-byte line (index * CSTRIDE) so hundreds
// of pollers of one counter do not contend with the other counters' updates.
constexpr int CSTRIDE = 32;
#ifndef TEAL_POLL_NS
#define TEAL_POLL_NS 128
#endif

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys(int* p, int v) {
    asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Counters signalled by other GPUs (fused tensor parallel): system-scope
// acquire, and a watchdog — a wait that cannot complete (a peer that never
// launched) traps after ~10 s instead of hanging the device.
__device__ __forceinline__ void wait_range_sys(const int* counters, int c0, int c1, int target) {
    if (threadIdx.x == 0) {
        for (int c = c0; c <= c1; ++c) {
            if (ld_acquire_sys(counters + (int64_t)c * CSTRIDE) >= target) continue;
            const unsigned long long t0 = gtimer_();
            unsigned ns = 32;
            while (ld_acquire_sys(counters + (int64_t)c * CSTRIDE) < target) {
                __nanosleep(ns);
                ns = ns < TEAL_POLL_NS ? ns * 2 : TEAL_POLL_NS;
                if (gtimer_() - t0 > 10000000000ull) asm volatile("trap;");
            }
        }
    }
    __syncthreads();
}

#ifndef TEAL_PAR_WAIT
#define TEAL_PAR_WAIT 1
#endif
// warp 0 polls up to 32 counters at once (one L2 round trip for a row range
// spanning several producer tiles, not one per counter), with backoff; the
// barrier publishes the result to the CTA
__device__ __forceinline__ void wait_range(const int* counters, int c0, int c1, int target) {
#if TEAL_PAR_WAIT
    if (threadIdx.x < 32) {
        for (int b = c0; b <= c1; b += 32) {
            const int c = b + (int)threadIdx.x;
            const int* p = counters + (int64_t)c * CSTRIDE;
            bool done = c > c1 || ld_acquire(p) >= target;
            unsigned ns = 32;
            while (!__all_sync(0xffffffffu, done)) {
                __nanosleep(ns);
                ns = ns < TEAL_POLL_NS ? ns * 2 : TEAL_POLL_NS;
                if (!done) done = ld_acquire(p) >= target;
            }
        }
    }
#else
    if (threadIdx.x == 0) {
        for (int c = c0; c <= c1; ++c) {
            unsigned ns = 32;
            while (ld_acquire(counters + (int64_t)c * CSTRIDE) < target) {
                __nanosleep(ns);
                ns = ns < TEAL_POLL_NS ? ns * 2 : TEAL_POLL_NS;
            }
        }
    }
#endif
    __syncthreads();
}

// Publish the CTA's prior global writes, then bump the counters: the barrier
// orders every thread's writes before thread 0, whose gpu-scope fence makes
// them (cumulatively) visible before its atomics — the cooperative-groups
// grid-sync pattern, one fence per CTA instead of one per thread.
// The barrier orders the CTA's writes before thread 0 (CTA scope); thread
// 0's gpu-scope RELEASE reduction is cumulative over them, so no separate
// sequentially-consistent fence (and L1 invalidation) is needed.
__device__ __forceinline__ void red_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acq_rel_add(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void signal(int* counters, int c0, int c1, int w = 1) {
    __syncthreads();
    if (threadIdx.x == 0 && c0 >= 0)
        for (int c = c0; c <= c1; ++c) red_release(counters + (int64_t)c * CSTRIDE, w);
}

// ---- fixed-point accumulators (ACC outputs) ---------------------------------
// Split-K contributors add int64 multiples of 2^-32 instead of handing fp32
// partials to a last arriver: integer addition is associative, so the sum is
// the same whatever order the contributors arrive in (deterministic), and no
// contributor waits for another — the reduction leaves the critical path.
__device__ __forceinline__ long long to_fx(float v) { return __float2ll_rn(v * 4294967296.0f); }
__device__ __forceinline__ float from_fx(long long a) { return __ll2float_rn(a) * 2.3283064365386963e-10f; }
__device__ __forceinline__ void red_add_s64(long long* p, long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Take a split-K ticket after storing this CTA's partial: returns (to every
// thread) whether this CTA arrived last; the last arriver's thread 0 fences
// again (acquire side) before the barrier that precedes the partial reads.
// (acq_rel: releases this CTA's partial, and the last arriver acquires every
// other contributor's before the barrier that precedes its partial reads)
__device__ __forceinline__ bool take_ticket(unsigned* ticket, unsigned expected_prev, int& s_last) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atom_acq_rel_add(ticket, 1u);
        const int last = prev == expected_prev;
        if (last) *ticket = 0u;
        s_last = last;
    }
    __syncthreads();
    return s_last != 0;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float silu(float z) { return z / (1.0f + expf(-z)); }

__device__ __forceinline__ float block_sum_nt(float v, Smem& s) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) s.scr[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < NW; ++w) t += s.scr[w];
        s.scr[NW] = t;
    }
    __syncthreads();
    const float r = s.scr[NW];
    __syncthreads();
    return r;
}

template <typename T>
__device__ __forceinline__ float ld_kv(const void* base, int64_t off);
template <>
__device__ __forceinline__ float ld_kv<float>(const void* base, int64_t off) {
    return __ldcg(reinterpret_cast<const float*>(base) + off);
}
template <>
__device__ __forceinline__ float ld_kv<uint16_t>(const void* base, int64_t off) {
    return bf16_to_f32(__ldcg(reinterpret_cast<const unsigned short*>(base) + off));
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Tile thresholds / signals: the plan's per-tile table, or (tiles == NULL,
// single-GEMV launches) one threshold for every tile and no signals.
__device__ __forceinline__ teal_step_tile tile_meta(const teal_step_group& g, int tile) {
    if (g.tiles) return g.tiles[tile];
    teal_step_tile t;
    t.t_lo = t.t_hi = g.t_all;
    t.seg_lo = t.seg_hi = 0;
    t.first_lo = t.first_hi = tile == 0;
    t.sig0 = t.sig1 = -1;
    return t;
}

// ---- epilogue of one finished column tile (thread c = column c) --------------
// `pre`: the residual value of this column, loaded by the caller together
// with the split-K partials (RESID epilogue).
__device__ __noinline__ void finalize(const teal_step_plan& P, const teal_step_group& g, int tile, float v, float pre) {
    Smem& s = smem();
    const int c = threadIdx.x;
    const int64_t col = (int64_t)tile * TW + c;
    const teal_step_tile tm = tile_meta(g, tile);
    switch (g.epilogue) {
        case TEAL_SEPI_STORE: {
            if (col < g.n) g.y[col] = v;
            break;
        }
        case TEAL_SEPI_RESID: {
            float xn = 0.f;
            if (col < g.n) {
                xn = pre + v;
                g.resid[col] = xn;
            }
            const float ss = block_sum_nt(xn * xn, s);
            if (c == 0) g.ss_out[tile] = ss;
            break;
        }
        case TEAL_SEPI_SILU: {
            s.col[c] = v;
            __syncthreads();
            if (c < TH) {
                const int64_t ic = (int64_t)tile * TH + c;
                if (ic < g.n) g.inter[ic] = silu(s.col[c]) * s.col[TH + c];
            }
            break;
        }
        case TEAL_SEPI_QKV: {
            s.col[c] = v;
            __syncthreads();
            if (col < g.n) {
                const int hd = g.head_dim, half = hd >> 1;
                const int d = (int)(col % hd);
                const int pos = __ldcg(P.state);
                float val = v;
                const bool is_q = col < g.nq;
                const bool is_k = !is_q && col < g.nq + g.nkv;
                if (g.rope_cos && (is_q || is_k)) {
                    const int dd = d < half ? d : d - half;
                    const float cs = g.rope_cos[(int64_t)pos * half + dd];
                    const float sn = g.rope_sin[(int64_t)pos * half + dd];
                    val = d < half ? (v * cs - s.col[c + half] * sn) : (v * cs + s.col[c - half] * sn);
                }
                if (is_q) {
                    g.q_out[col] = val;
                } else {
                    const int64_t kc = is_k ? col - g.nq : col - g.nq - g.nkv;
                    const int64_t off = ((kc / hd) * g.max_seq + pos) * hd + d;
                    void* cache = is_k ? g.k_cache : g.v_cache;
                    if (g.kv_dtype == TEAL_BF16) reinterpret_cast<uint16_t*>(cache)[off] = f32_to_bf16_rn(val);
                    else reinterpret_cast<float*>(cache)[off] = val;
                }
            }
            break;
        }
        case TEAL_SEPI_LOGITS: {
            const bool ok = col < g.n && v == v;
            if (col < g.n) g.y[col] = v;
            // tile argmax: largest value, lowest index on ties, NaN ignored
            float bv = ok ? v : -INFINITY;
            int bi = ok ? (int)col : 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            if ((c & 31) == 0) { s.scr[c >> 5] = bv; s.wcnt[c >> 5] = bi; }
            __syncthreads();
            if (c == 0) {
                float tv = s.scr[0];
                int ti = s.wcnt[0];
                for (int w = 1; w < NW; ++w)
                    if (s.scr[w] > tv || (s.scr[w] == tv && s.wcnt[w] < ti)) { tv = s.scr[w]; ti = s.wcnt[w]; }
                P.cand_v[tile] = tv;
                P.cand_i[tile] = ti;
                if (P.tp) {  // vocabulary-parallel: candidates and ticket on rank 0, global indices
                    const teal_step_tp& T = *P.tp;
                    const int slot = T.rank * g.ntiles + tile;
                    T.cand_v[slot] = tv;
                    T.cand_i[slot] = ti == 0x7fffffff ? ti : ti + T.vocab_off;
                    __threadfence_system();
                    unsigned prev;
                    asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(T.lm_ticket) : "memory");
                    s.last = prev == (unsigned)(T.world * g.ntiles) - 1u;
                    if (s.last) *T.lm_ticket = 0u;
                } else {
                    __threadfence();
                    const unsigned prev = atomicAdd(P.lm_done, 1u);
                    s.last = prev == (unsigned)g.ntiles - 1u;
                    if (s.last) {
                        *P.lm_done = 0u;
                        __threadfence();
                    }
                }
            }
            __syncthreads();
            if (s.last) {  // the last tile: argmax over the per-tile candidates, whole CTA
                float gv = -INFINITY;
                int gi = 0x7fffffff;
                const float* cvs = P.tp ? P.tp->cand_v : P.cand_v;
                const int* cis = P.tp ? P.tp->cand_i : P.cand_i;
                const int ncand = P.tp ? P.tp->world * g.ntiles : g.ntiles;
                for (int t = c; t < ncand; t += NT) {
                    const float cv = __ldcg(cvs + t);
                    const int ci = __ldcg(cis + t);
                    if (cv > gv || (cv == gv && ci < gi)) { gv = cv; gi = ci; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, gv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
                    if (ov > gv || (ov == gv && oi < gi)) { gv = ov; gi = oi; }
                }
                __syncthreads();
                if ((c & 31) == 0) { s.scr[c >> 5] = gv; s.wcnt[c >> 5] = gi; }
                __syncthreads();
                if (c == 0) {
                    for (int w = 1; w < NW; ++w)
                        if (s.scr[w] > s.scr[0] || (s.scr[w] == s.scr[0] && s.wcnt[w] < s.wcnt[0])) {
                            s.scr[0] = s.scr[w];
                            s.wcnt[0] = s.wcnt[w];
                        }
                    const int tok = s.wcnt[0] == 0x7fffffff ? 0 : s.wcnt[0];
                    if (P.tp)
                        for (int j = 0; j < P.tp->world; ++j) *P.tp->token[j] = tok;
                    else
                        *P.token_out = tok;
                }
            }
            __syncthreads();
            break;
        }
        default:
            break;
    }
    signal(P.counters, tm.sig0, tm.sig1);
}

// Weight element formats of a tile row chunk (TW columns):
//   fp32 1 KB, bf16 512 B, int8 256 B (per-column scale applied after the
//   reduction), int4 128 B (two's-complement nibbles, low nibble = even
//   column; fp32 scale per (row group, column)).
// Per-lane accumulator columns: bf16 / int8 / int4 lane l owns [8l, 8l+8)
// (lanes 16..31 = hi half); fp32 lane l owns [4l, 4l+4) (lo) and
// [128+4l, 128+4l+4) (hi).
template <int WT> struct WFmt;
template <> struct WFmt<TEAL_F32> { static constexpr int ROWB = TW * 4; static constexpr int LB = 16; };
template <> struct WFmt<TEAL_BF16> { static constexpr int ROWB = TW * 2; static constexpr int LB = 16; };
template <> struct WFmt<TEAL_I8> { static constexpr int ROWB = TW; static constexpr int LB = 8; };
template <> struct WFmt<TEAL_I4> { static constexpr int ROWB = TW / 2; static constexpr int LB = 4; };

template <int WT>
__device__ __forceinline__ int acc_col(int lane, int j) {
    if constexpr (WT != TEAL_F32) return lane * 8 + j;
    else return j < 4 ? lane * 4 + j : TH + lane * 4 + (j - 4);
}

// one lane's raw weights of a row chunk: 8 words (fp32), 4 (bf16), 2 (int8), 1 (int4)
template <int WT> struct LaneW { static constexpr int N = WT == TEAL_F32 ? 8 : (WT == TEAL_BF16 ? 4 : (WT == TEAL_I8 ? 2 : 1)); uint32_t u[N]; };

// lane's 8 weights of one row chunk (unscaled for int8 / int4)
template <int WT>
__device__ __forceinline__ void unpack8(const LaneW<WT>& d, float w[8]) {
    if constexpr (WT == TEAL_BF16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) { w[2 * q] = bf16_lo(d.u[q]); w[2 * q + 1] = bf16_hi(d.u[q]); }
    } else if constexpr (WT == TEAL_F32) {
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = __uint_as_float(d.u[q]);
    } else if constexpr (WT == TEAL_I8) {
        // magic-number conversion (no I2F, a quarter-rate op): b ^ 0x80 = b + 128
        // placed in the mantissa of 2^23 (one PRMT), minus 2^23 + 128 (one FADD)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t x = d.u[q] ^ 0x80808080u;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                w[4 * q + k] = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7540u | k)) - 8388736.0f;
        }
    } else {
        // nibble n (two's complement) ^ 8 = n + 8 into the mantissa of 2^23
        // (shift + LOP3), minus 2^23 + 8
        const uint32_t x = d.u[0] ^ 0x88888888u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            w[k] = __uint_as_float(((x >> (4 * k)) & 0xfu) | 0x4B000000u) - 8388616.0f;
    }
}

// streaming load of 16 / 8 / 4 bytes (L2 evict-first policy), by value
__device__ __forceinline__ uint4 ldw16(const unsigned char* p, uint64_t pol) { return ldg128_stream_pol(p, pol); }
__device__ __forceinline__ uint2 ldw8(const unsigned char* p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ldw4(const unsigned char* p, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

// sqrt(sum(ss)/m + eps) with the partials summed in ascending order: one
// warp loads them in parallel (one L2 round trip), lane 0 adds in order.
__device__ __forceinline__ float rms_den(const teal_step_group& g, int lane) {
    float a = 0.f;
    for (int p0 = 0; p0 < g.nss; p0 += 32) {
        const float v = (p0 + lane < g.nss) ? __ldcg(g.ss + p0 + lane) : 0.f;
        const int n = min(32, g.nss - p0);
        for (int q = 0; q < n; ++q) a += __shfl_sync(0xffffffffu, v, q);
    }
    return sqrtf(a / (float)g.m + g.eps);
}

// PRO_RMS_ACC, in two parts.  rms_stage_x: the previous residual version x
// (final since an earlier phase) -> s.u.g.xs, issued while the phase still
// waits for its accumulator.  rms_acc_finish: x' = x + fx(in_acc) over all m
// channels (every load in flight at once), CTA c of G writes its share
// [c*m/G, (c+1)*m/G) of x' to x_out (the next residual version), and the
// RMSNorm denominator is returned.  Every CTA computes the same sum in the
// same order, so all tiles threshold the same h.
__device__ void rms_stage_x(const teal_step_group& g, Smem& s) {
    const int tid = threadIdx.x, m = g.m;
#pragma unroll 1
    for (int i0 = 0; i0 < m; i0 += 16 * NT) {
        float xb[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = i0 + q * NT + tid;
            xb[q] = __ldcg(g.x + (i < m ? i : 0));  // straight-line (unused past m)
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = i0 + q * NT + tid;
            if (i < m) s.u.g.xs[i] = xb[q];
        }
    }
}

__device__ float rms_acc_finish(const teal_step_group& g, int c, int G, Smem& s) {
    const int tid = threadIdx.x, m = g.m;
    const int p0 = c * m / G, p1 = (c + 1) * m / G;  // m <= XS_MAX: 32-bit
    float ss = 0.f;
#pragma unroll 1
    for (int i0 = 0; i0 < m; i0 += 16 * NT) {
        long long xa[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = i0 + q * NT + tid;
            xa[q] = __ldcg(g.in_acc + (i < m ? i : 0));
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = i0 + q * NT + tid;
            if (i < m) {
                const float xn = s.u.g.xs[i] + from_fx(xa[q]);  // own thread's staged x: no barrier needed
                s.u.g.xs[i] = xn;
                ss = fmaf(xn, xn, ss);
                if (i >= p0 && i < p1) g.x_out[i] = xn;
            }
        }
    }
    return sqrtf(block_sum_nt(ss, s) / (float)m + g.eps);
}

// CTAs taking part in a GEMV phase: never more than the 32-row groups (every
// range non-empty) and, when the phase has at most half as many tiles as the
// grid has CTAs, a multiple of the tile count so that every range lies inside
// one tile (no CTA pays the fixed cost of a second segment; each tile has the
// same number of contributors).  Mirrored by engine.participants().
__device__ __forceinline__ int participants(int ntiles, int64_t F) {
    const int grid = gridDim.x;
    if (F <= grid) return (int)F;
    const int aligned = ntiles * (grid / ntiles);
    if (2 * ntiles <= grid && 10 * aligned >= 9 * grid) return aligned;  // keep >= 90% of the grid busy
    return grid;
}

// a * b / c for non-negative operands; 32-bit division when the product fits
// (every step-plan group), 64-bit (a software routine) only for huge
// single-GEMV launches
__device__ __forceinline__ int64_t muldiv(int64_t a, int64_t b, int64_t c) {
    const int64_t p = a * b;
    if (p <= 0x7fffffff && c <= 0x7fffffff) return (int64_t)((unsigned)p / (unsigned)c);
    return p / c;
}

__device__ __forceinline__ int owner_of(int64_t gidx, int64_t F, int G) {
    const int64_t p = (gidx + 1) * (int64_t)G - 1;
    return (int)((p <= 0x7fffffff && F <= 0x7fffffff) ? (int64_t)((unsigned)p / (unsigned)F) : p / F);
}
__device__ __forceinline__ int tile_of(int64_t gidx, int gpt) {
    return gidx <= 0x7fffffff ? (int)((unsigned)gidx / (unsigned)gpt) : (int)(gidx / gpt);
}

// Threshold + compact rows [r0, r1) of one tile into s.u.g (ordered).
// `rden` < 0: compute the RMSNorm denominator here (warp 0), its
// sum-of-squares loads in flight together with every thread's x / gain loads.
__device__ int compact_rows(const teal_step_group& g, const teal_step_tile& tm, int tile, int r0, int r1,
                            float& rden, bool rms, Smem& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool two = tm.seg_hi != tm.seg_lo;
    constexpr int RPT = MAXR / NT;  // rows per thread
    float hx[RPT], gx[RPT];
    // Loads are straight-line (rows past r1 read row r0 and are ignored by
    // the compaction): a branch per row would make the compiler wait on each
    // load at the reconvergence point instead of keeping them all in flight.
    if (g.prologue == TEAL_PRO_SILU_ACC) {  // h = silu(gate) * up from the gate/up accumulator
        long long ga[RPT], ua[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int i = r0 + q * NT + tid;
            const int ic = i < r1 ? i : r0;
            const int64_t b = (int64_t)(ic / TH) * TW + (ic % TH);
            ga[q] = __ldcg(g.in_acc + b);
            ua[q] = __ldcg(g.in_acc + b + TH);
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            hx[q] = silu(from_fx(ga[q])) * from_fx(ua[q]);
            gx[q] = 1.f;
        }
    } else {
        if (g.prologue == TEAL_PRO_RMS_ACC) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int i = r0 + q * NT + tid;
                hx[q] = s.u.g.xs[i < r1 ? i : r0];
            }
        } else {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {  // all x loads in flight at once
                const int i = r0 + q * NT + tid;
                hx[q] = __ldcg(g.x + (i < r1 ? i : r0));
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int i = r0 + q * NT + tid;
            gx[q] = rms ? __ldg(g.gain + (i < r1 ? i : r0)) : 1.f;
        }
    }
    if (rms) {
        if (rden < 0.f) {
            if (warp == 0) s.rden = rms_den(g, lane);
            __syncthreads();
            rden = s.rden;
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) hx[q] = (hx[q] / rden) * gx[q];
    }
    int base = 0;
#pragma unroll 1
    for (int q = 0; q < RPT; ++q) {
        const int i0 = r0 + q * NT;
        if (i0 >= r1) break;
        const int i = i0 + tid;
        const bool v = i < r1;
        const float h = hx[q];
        const bool klo = v && !(fabsf(h) <= tm.t_lo);
        const bool khi = v && !(fabsf(h) <= tm.t_hi);
        const bool k = klo || khi;
        const unsigned bk = __ballot_sync(0xffffffffu, k);
        const bool wv = (i - lane) < r1;
        if (g.dbg_h && tile == 0 && v) g.dbg_h[i] = h;
        if (tm.first_lo && wv) {
            const unsigned bl = __ballot_sync(0xffffffffu, klo);
            if (lane == 0) {
                if (g.dbg_bits[tm.seg_lo]) g.dbg_bits[tm.seg_lo][(i - lane) >> 5] = bl;
                if (g.kept[tm.seg_lo] && bl) atomicAdd(g.kept[tm.seg_lo], (unsigned long long)__popc(bl));
            }
        }
        if (tm.first_hi && two && wv) {
            const unsigned bh = __ballot_sync(0xffffffffu, khi);
            if (lane == 0) {
                if (g.dbg_bits[tm.seg_hi]) g.dbg_bits[tm.seg_hi][(i - lane) >> 5] = bh;
                if (g.kept[tm.seg_hi] && bh) atomicAdd(g.kept[tm.seg_hi], (unsigned long long)__popc(bh));
            }
        }
        if (lane == 0) s.wcnt[warp] = __popc(bk);
        __syncthreads();
        int off = base, tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int cw = s.wcnt[w];
            off += (w < warp) ? cw : 0;
            tot += cw;
        }
        if (k) {
            const int pos = off + __popc(bk & ((1u << lane) - 1u));
            s.u.g.idx[pos] = (i - r0) | (klo ? (1 << 30) : 0) | (khi ? (int)(1u << 31) : 0);
            s.u.g.h[pos] = h;
        }
        base += tot;
        __syncthreads();
    }
    return base;
}

// Stream the `cnt` compacted rows: warp w takes rows w*U.., w*U+NW*U.., with
// the next batch of U rows' loads issued before the current batch is consumed
// (software pipeline: 2U row chunks in flight per warp).  Only the kept half
// of a row is loaded (bf16 / int8 / int4: lanes 0-15 = lo, 16-31 = hi; fp32:
// every lane loads 16 B of each kept half).  int4 rows accumulate per row
// group and are scaled when the group changes (scales staged in s.u.g.gsc).
template <int WT, int UB>
__device__ __forceinline__ void stream_rows(const unsigned char* tb, int64_t rsb, int cnt, const Smem& s, float acc[8],
                                            uint64_t pol, int gbase, int group, bool ok_lo, bool ok_hi) {
    const int gsh = __ffs(group) - 1;  // int4 row groups: a power of two (host-checked)
    constexpr int ROWB = WFmt<WT>::ROWB;
    constexpr int LB = WFmt<WT>::LB;
    constexpr int HB = ROWB / 2;
    // rows per pipeline stage (int8 / int4 rows are narrower; measured: more
    // rows per stage does not help them — their unpack is issue-bound)
    // (narrow int8 / int4 rows: more of them per stage keep the bytes in
    // flight per warp closer to bf16's, at similar register cost)
    constexpr int U = WT == TEAL_F32 ? UB / 2 : (WT == TEAL_I8 ? UB + UB / 2 : (WT == TEAL_I4 ? 2 * UB : UB));
    constexpr int NW_ = LaneW<WT>::N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int myhalf = lane < 16 ? 30 : 31;
    // the lane's h values ride in registers with the loads (0 where this
    // lane's half of the row is pruned)
    constexpr int HN = U * (WT == TEAL_F32 ? 2 : 1);
    LaneW<WT> a[U], b[U];
    float ha[HN], hb[HN];
    float accg[8];
    int curg = -1;
#pragma unroll
    for (int j = 0; j < 8; ++j) accg[j] = 0.f;
    // loads only: the kept bits and h are re-read from shared memory when consumed
    auto fetch = [&](int e0, LaneW<WT> (&d)[U], float (&hh)[HN]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u;
#pragma unroll
            for (int k = 0; k < NW_; ++k) d[u].u[k] = 0u;
            hh[u * (HN / U)] = 0.f;
            if constexpr (WT == TEAL_F32) hh[2 * u + 1] = 0.f;
            if (e < cnt) {
                const unsigned pk = (unsigned)s.u.g.idx[e];
                const unsigned char* rp = tb + (int64_t)(pk & 0x3fffffffu) * rsb;
                if constexpr (WT == TEAL_F32) {
                    const float hv = s.u.g.h[e];
                    if (((pk >> 30) & 1u) && ok_lo) {
                        const uint4 r = ldw16(rp + lane * 16, pol);
                        d[u].u[0] = r.x; d[u].u[1] = r.y; d[u].u[2] = r.z; d[u].u[3] = r.w;
                        hh[2 * u] = hv;
                    }
                    if (((pk >> 31) & 1u) && ok_hi) {
                        const uint4 r = ldw16(rp + HB + lane * 16, pol);
                        d[u].u[4] = r.x; d[u].u[5] = r.y; d[u].u[6] = r.z; d[u].u[7] = r.w;
                        hh[2 * u + 1] = hv;
                    }
                } else if (((pk >> myhalf) & 1u) && ok_lo) {
                    hh[u] = s.u.g.h[e];
                    if constexpr (LB == 16) {
                        const uint4 r = ldw16(rp + lane * 16, pol);
                        d[u].u[0] = r.x; d[u].u[1] = r.y; d[u].u[2] = r.z; d[u].u[3] = r.w;
                    } else if constexpr (LB == 8) {
                        const uint2 r = ldw8(rp + lane * 8, pol);
                        d[u].u[0] = r.x; d[u].u[1] = r.y;
                    } else {
                        d[u].u[0] = ldw4(rp + lane * 4, pol);
                    }
                }
            }
        }
    };
    auto flush_group = [&]() {  // int4: acc += accg * scale(group, column)
        if (curg >= 0) {
            const float* sc = s.u.g.gsc + (curg - (gbase >> gsh)) * TW + lane * 8;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                acc[j] = fmaf(accg[j], sc[j], acc[j]);
                accg[j] = 0.f;
            }
        }
    };
    auto consume = [&](int e0, const LaneW<WT> (&d)[U], const float (&hh)[HN]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float w[8];
            unpack8<WT>(d[u], w);
            if constexpr (WT == TEAL_F32) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[k] = fmaf(hh[2 * u], w[k], acc[k]);
#pragma unroll
                for (int k = 4; k < 8; ++k) acc[k] = fmaf(hh[2 * u + 1], w[k], acc[k]);
            } else if constexpr (WT == TEAL_I4) {
                const int e = e0 + u;
                if (e < cnt) {
                    const int gr = (gbase + (int)((unsigned)s.u.g.idx[e] & 0x3fffffffu)) >> gsh;
                    if (gr != curg) {
                        flush_group();
                        curg = gr;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) accg[k] = fmaf(hh[u], w[k], accg[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = fmaf(hh[u], w[k], acc[k]);
            }
        }
    };
    int e0 = warp * U;
    if (e0 < cnt) {
        fetch(e0, a, ha);
        for (;;) {
            const int en = e0 + NW * U;
            if (en < cnt) fetch(en, b, hb);
            consume(e0, a, ha);
            if (en >= cnt) break;
            e0 = en;
            if (e0 + NW * U < cnt) fetch(e0 + NW * U, a, ha);
            consume(e0, b, hb);
            if (e0 + NW * U >= cnt) break;
            e0 += NW * U;
        }
    }
    if constexpr (WT == TEAL_I4) flush_group();
}

// Fused tensor-parallel row-parallel output: this CTA's column partial goes
// into every rank's accumulator (peer memory) and every rank's counters are
// bumped (system-scope release after the CTA's adds).  Integer adds: the
// sum is the same on every rank whatever the arrival order.
__device__ __noinline__ void tp_accumulate(const teal_step_plan& P, const teal_step_group& g, int tile, long long fx,
                                           int sig0, int sig1, int w) {
    const teal_step_tp& T = *P.tp;
    const int64_t off = (g.acc - T.acc[T.rank]) + (int64_t)tile * TW + threadIdx.x;
    for (int j = 0; j < T.world; ++j) red_add_s64(T.acc[j] + off, fx);
    __syncthreads();
    if (threadIdx.x == 0 && sig0 >= 0) {  // (release: cumulative over the CTA's adds ordered by the barrier)
        for (int j = 0; j < T.world; ++j)
            for (int c = sig0; c <= sig1; ++c) red_release_sys(T.counters[j] + (int64_t)c * CSTRIDE, w);
    }
}

template <int WT, int UB>
__device__ void gemv_slice_t(const teal_step_plan& P, const teal_step_phase& ph, const teal_step_group& g, Smem& s,
                             uint64_t pol, unsigned long long* tl) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gpt = (g.m + 31) / 32;
    const int64_t F = (int64_t)g.ntiles * gpt;
    const int c = blockIdx.x;
    const int G = g.ranges ? g.nranges : participants(g.ntiles, F);
    if (c >= G) return;
    int4 rg = make_int4(0, 0, 0, 0);
    if (g.ranges) rg = g.ranges[c];
    const int64_t g0 = g.ranges ? (int64_t)rg.x : muldiv(c, F, G);
    const int64_t g1 = g.ranges ? (int64_t)rg.y : muldiv(c + 1, F, G);
    const bool rms = g.prologue == TEAL_PRO_RMSNORM || g.prologue == TEAL_PRO_RMS_ACC;
    // While this slice waits for its inputs, pull the head of its weight range
    // into L2 (one bulk prefetch of contiguous tiled rows): the wait is tail
    // time of the previous phase, when HBM is mostly idle.  Rows that turn out
    // pruned cost idle bandwidth only; kept rows then stream from L2.
    const int pf_bytes = P.prefetch_bytes;
    if (tid == 0 && pf_bytes > 0) {
        const int tile = tile_of(g0, gpt);
        const int r0 = (int)(g0 - (int64_t)tile * gpt) * 32;
        const int r1 = min(g.m, (int)(min64(g1, (int64_t)(tile + 1) * gpt) - (int64_t)tile * gpt) * 32);
        const int64_t rowb = WFmt<WT>::ROWB;
        const int64_t bytes = min64((int64_t)(r1 - r0) * rowb, (int64_t)pf_bytes) & ~(int64_t)15;
        if (bytes > 0) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(g.w) + ((int64_t)tile * g.m + r0) * rowb;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((uint32_t)bytes) : "memory");
        }
    }
    const bool racc = g.prologue == TEAL_PRO_RMS_ACC;
    if (racc && g.xwait >= 0) {  // stage x before the wait (off the critical path)
        wait_range(P.counters, g.xwait, g.xwait, g.xwait_target);
        rms_stage_x(g, s);
    }
    if (ph.dep_kind == TEAL_DEP_GLOBAL) {
        if (P.tp) wait_range_sys(P.counters, ph.dep, ph.dep, ph.target);
        else wait_range(P.counters, ph.dep, ph.dep, ph.target);
    }
    if (tl && tid == 0) tl[6] = gtimer();  // global dependency met
    // PRO_RMSNORM: rden computed by the first compaction, overlapped with its x loads
    float rden = rms ? -1.f : 1.f;
    if (racc) {
        if (g.xwait < 0) rms_stage_x(g, s);
        rden = rms_acc_finish(g, c, G, s);
        if (tl && tid == 0) tl[7] = gtimer();  // RMS prologue done
        if (g.xsig >= 0) signal(P.counters, g.xsig, g.xsig);  // x_out share written
    }
    constexpr int ROWB = WFmt<WT>::ROWB;
    int segi = 0, lasts = 0;
#define SL_STAMP(k, v) do { if (tl && tid == 0) tl[k] = (v); } while (0)
    for (int64_t gs = g0; gs < g1; ++segi) {
        const int tile = tile_of(gs, gpt);
        const int64_t ge = min64(g1, (int64_t)(tile + 1) * gpt);
        const int r0 = (int)(gs - (int64_t)tile * gpt) * 32;
        const int r1 = min(g.m, (int)(ge - (int64_t)tile * gpt) * 32);
        gs = ge;
        if (ph.dep_kind == TEAL_DEP_ROWS)
            wait_range(P.counters, ph.dep + r0 / ph.dep_rows, ph.dep + (r1 - 1) / ph.dep_rows, ph.target);
        if (segi == 0) SL_STAMP(2, gtimer());
        const teal_step_tile tm = tile_meta(g, tile);
        // tiled: tile t = block [m][TW]; untiled input-major (single GEMV): row stride ldw
        const int64_t rsb = g.row_stride_b ? g.row_stride_b : ROWB;
        const int64_t tsb = g.row_stride_b ? g.tile_stride_b : (int64_t)g.m * ROWB;
        const unsigned char* tbase = reinterpret_cast<const unsigned char*>(g.w) + (int64_t)tile * tsb;
        // untiled matrices: lanes whose columns lie past n (last tile) load
        // nothing; tiled blocks are zero-padded to whole tiles
        const int64_t c0 = (int64_t)tile * TW;
        const bool untiled = g.row_stride_b != 0;
        const bool ok_lo = !untiled || ((WT == TEAL_F32) ? (c0 + 4 * lane < g.n) : (c0 + 8 * lane < g.n));
        const bool ok_hi = !untiled || ((WT == TEAL_F32) ? (c0 + TH + 4 * lane < g.n) : ok_lo);
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int ra = r0; ra < r1; ra += MAXR) {
            const int rb = min(r1, ra + MAXR);
            int cnt;
            if constexpr (WT == TEAL_I4) {
                // the chunk's row-group scales: every load in flight together and
                // under the compaction (thread = column; one round trip, hidden)
                const int gA = ra / g.group, ng = (rb - 1) / g.group - gA + 1;
                float sc[GSC_MAX];
#pragma unroll
                for (int k = 0; k < GSC_MAX; ++k)
                    sc[k] = __ldg(g.gscale + (int64_t)(gA + (k < ng ? k : 0)) * g.ntiles * TW + (int64_t)tile * TW + tid);
                cnt = compact_rows(g, tm, tile, ra, rb, rden, rms, s);
#pragma unroll
                for (int k = 0; k < GSC_MAX; ++k)
                    if (k < ng) s.u.g.gsc[k * TW + tid] = sc[k];
                __syncthreads();
            } else {
                cnt = compact_rows(g, tm, tile, ra, rb, rden, rms, s);
            }
            stream_rows<WT, UB>(tbase + (int64_t)ra * rsb, rsb, cnt, s, acc, pol, ra, g.group > 0 ? g.group : 1,
                                ok_lo, ok_hi);
            __syncthreads();  // rows list is rewritten by the next chunk
        }
        SL_STAMP(segi == 0 ? 3 : 5, gtimer());
#pragma unroll
        for (int j = 0; j < 8; ++j) s.red[warp * TW + acc_col<WT>(lane, j)] = acc[j];
        __syncthreads();
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += s.red[w * TW + tid];
        const int cf = owner_of((int64_t)tile * gpt, F, G);
        const int cl = owner_of((int64_t)(tile + 1) * gpt - 1, F, G);
        if (g.acc) {  // ACC output: add this CTA's partial, bump the counters by its share of CONTRIB
            if (g.col_scale) v *= g.col_scale[(int64_t)tile * TW + tid];
            const int w = g.ranges ? (segi == 0 ? rg.z : rg.w) : (c == cf ? CONTRIB - (cl - cf) : 1);
            if (g.tp_sum && P.tp) {
                tp_accumulate(P, g, tile, to_fx(v), tm.sig0, tm.sig1, w);
            } else {
                red_add_s64(g.acc + (int64_t)tile * TW + tid, to_fx(v));
                signal(P.counters, tm.sig0, tm.sig1, w);
            }
            ++lasts;
            if (segi == 0) SL_STAMP(4, gtimer());
            continue;
        }
        const bool resid = g.epilogue == TEAL_SEPI_RESID && (int64_t)tile * TW + tid < g.n;
        float pre = 0.f;
        if (cl > cf) {
            float* slot = g.partials + ((int64_t)tile * g.maxc + (c - cf)) * TW;
            __stcg(slot + tid, v);
            if (!take_ticket(g.tickets + tile, (unsigned)(cl - cf), s.last)) {
                if (segi == 0) SL_STAMP(4, gtimer());
                continue;
            }
            if (resid) pre = __ldcg(g.resid + (int64_t)tile * TW + tid);  // in flight with the partials
            const float* pb = g.partials + (int64_t)tile * g.maxc * TW + tid;
            const int nc = cl - cf + 1;
            v = 0.f;
            for (int s0 = 0; s0 < nc; s0 += 16) {  // 16 independent loads in flight, summed in order
                float pv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) pv[q] = (s0 + q < nc) ? __ldcg(pb + (int64_t)(s0 + q) * TW) : 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (s0 + q < nc) v += pv[q];
            }
        }
        else if (resid) {
            pre = __ldcg(g.resid + (int64_t)tile * TW + tid);
        }
        if (g.col_scale) v *= g.col_scale[(int64_t)tile * TW + tid];
        finalize(P, g, tile, v, pre);
        ++lasts;
        if (segi == 0) SL_STAMP(4, gtimer());
    }
    (void)lasts;
#undef SL_STAMP
}

// One kernel instantiation per weight format: every GEMV group of a plan
// (layers and LM head) uses the plan's w_dtype.

// ---- attention unit: (kv group g, position chunk) ---------------------------
// Runs on a few CTAs once per layer, so its instructions are cold every time
// (the kernel is far larger than the 32 KB L1.5 instruction cache): the code
// is deliberately small — runtime loops, no unrolling over heads, the K/V
// dtype a runtime switch around two short inner loops — since instruction
// fetch from L2, not arithmetic, sets its latency.
//
// Staging in two parts.  attn_stage_kv runs BEFORE the unit's q/k/v tiles are
// done (the cache rows of earlier positions do not depend on this step): the
// chunk's np K / V rows except the new position's (newrow) -> smem (cache
// dtype; K rows padded by 16 B so row-parallel reads are conflict-free).
// attn_stage_q runs after the wait: q of group g (RoPE applied when it comes
// from the accumulator) and the new row's k (RoPE) and v, which it also
// appends to the cache (rounded to the cache dtype first, as later steps will
// read it).

__device__ __noinline__ void attn_stage_kv(const teal_step_attn& a, int p0, int np, int newrow, int64_t kvbase) {
    Smem& s = smem();
    constexpr int PER = ATT_STAGE / 16 / NT;  // n16 <= ATT_STAGE / 16 = PER * NT
    const int tid = threadIdx.x, hd = a.hd;
    const int kvb = a.kv_dtype == TEAL_BF16 ? 2 : 4;
    const int vpr = hd * kvb / 16;  // 16-byte vectors per row
    const int n16 = np * vpr;
    const uint4* gk = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(a.k_cache) + (kvbase + (int64_t)p0 * hd) * kvb);
    const uint4* gv = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(a.v_cache) + (kvbase + (int64_t)p0 * hd) * kvb);
    uint4 kk[PER], vv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {  // straight-line: out-of-range vectors re-read vector 0 (unused)
        const int v = tid + q * NT;
        const int vc = v < n16 ? v : 0;
        kk[q] = __ldcg(gk + vc);
        vv[q] = __ldcg(gv + vc);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int v = tid + q * NT;
        if (v < n16 && v / vpr != newrow) {
            s.u.a.k[(v / vpr) * (vpr + 1) + v % vpr] = kk[q];
            s.u.a.v[v] = vv[q];
        }
    }
}

__device__ __noinline__ void attn_stage_q(const teal_step_attn& a, int g, int pos, int newrow, int64_t kvbase) {
    Smem& s = smem();
    constexpr int QPT = ATT_MAXG * ATT_MAXHD / NT;
    // the fields, read once: the struct lives in global memory, and a store
    // through one of its pointers would make the compiler re-read the next
    // field it needs after that store (a dependent global load per store)
    const long long* const qkv_acc = a.qkv_acc;
    const float* const rope_cos = a.rope_cos;
    const float* const rope_sin = a.rope_sin;
    void* const k_cache = const_cast<void*>(a.k_cache);
    void* const v_cache = const_cast<void*>(a.v_cache);
    const int kv_dtype = a.kv_dtype, nq = a.nq, nkv = a.nkv;
    const int tid = threadIdx.x, G = a.H / a.KVH, hd = a.hd, half = hd >> 1;
    const bool acc = qkv_acc != nullptr;
    // NT is a multiple of hd: every element this thread touches (q heads and
    // the new k) has head dim d = tid % hd, so one RoPE pair serves all
    const int d = tid % hd, dd = d < half ? d : d - half;
    const int part = d < half ? half : -half;
    const bool rope = acc && rope_cos;
    long long qa[QPT], qp[QPT], ka = 0, kp = 0, va = 0;
    float qf[QPT];
    float cs = 1.f, sn = 0.f;
    if (rope) {
        cs = __ldg(rope_cos + (int64_t)pos * half + dd);
        sn = __ldg(rope_sin + (int64_t)pos * half + dd);
    }
    // straight-line loads (clamped indices; unused values are never consumed)
    const bool nk = newrow >= 0 && tid < hd;
    if (acc) {
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
            const int o = tid + j * NT;
            const int64_t qc = (int64_t)g * G * hd + (o < G * hd ? o : d);
            qa[j] = __ldcg(qkv_acc + qc);
            qp[j] = __ldcg(qkv_acc + qc + part);
            qf[j] = 0.f;
        }
        const int64_t kc = (int64_t)nq + (int64_t)g * hd + d;
        ka = __ldcg(qkv_acc + kc);
        kp = __ldcg(qkv_acc + kc + part);
        va = __ldcg(qkv_acc + kc + nkv);
    } else {
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
            const int o = tid + j * NT;
            qf[j] = __ldcg(a.q + (int64_t)g * G * hd + (o < G * hd ? o : 0));
            qa[j] = qp[j] = 0;
        }
    }
    const float sgn = d < half ? -1.f : 1.f;  // x*cos -/+ partner*sin
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int o = tid + j * NT;
        if (o < G * hd) {
            float r = qf[j];
            if (acc) r = rope ? fmaf(sgn * from_fx(qp[j]), sn, from_fx(qa[j]) * cs) : from_fx(qa[j]);
            s.u.a.q[o] = r;
        }
    }
    if (nk) {
        float kr = rope ? fmaf(sgn * from_fx(kp), sn, from_fx(ka) * cs) : from_fx(ka);
        float vr = from_fx(va);
        const int64_t off = kvbase + (int64_t)pos * hd + d;
        if (kv_dtype == TEAL_BF16) {
            const uint16_t kb = f32_to_bf16_rn(kr), vb = f32_to_bf16_rn(vr);
            __stcg(reinterpret_cast<unsigned short*>(k_cache) + off, kb);
            __stcg(reinterpret_cast<unsigned short*>(v_cache) + off, vb);
        } else {
            __stcg(reinterpret_cast<float*>(k_cache) + off, kr);
            __stcg(reinterpret_cast<float*>(v_cache) + off, vr);
        }
        const int vpr = hd * (kv_dtype == TEAL_BF16 ? 2 : 4) / 16;
        if (kv_dtype == TEAL_BF16) {
            reinterpret_cast<uint16_t*>(s.u.a.k + newrow * (vpr + 1))[d] = f32_to_bf16_rn(kr);
            reinterpret_cast<uint16_t*>(s.u.a.v)[newrow * hd + d] = f32_to_bf16_rn(vr);
        } else {
            reinterpret_cast<float*>(s.u.a.k + newrow * (vpr + 1))[d] = kr;
            reinterpret_cast<float*>(s.u.a.v)[newrow * hd + d] = vr;
        }
    }
}

__device__ __noinline__ void attn_unit(const teal_step_plan& P, const teal_step_attn& a, int g, int ch, int L) {
    Smem& s = smem();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = a.H / a.KVH, hd = a.hd;
    const int p0 = ch * a.chunk;
    const int p1 = min(L, p0 + a.chunk);
    const int np = max(0, p1 - p0);
    const int rec = G * hd + 2 * G;
    float* my = a.partials + ((int64_t)g * a.nchunks + ch) * rec;
    const int64_t kvbase = (int64_t)g * a.max_seq * hd;
    unsigned long long* dbg = a.dbg ? a.dbg + ((int64_t)g * a.nchunks + ch) * 6 : nullptr;
    // stamps 0, 1: %globaltimer (ns); 2..5: SM clock cycles since stamp 1
    long long ck1 = 0;
#define ATT_STAMP(k) do { if (dbg && tid == 0) { if ((k) < 2) { dbg[k] = gtimer(); ck1 = clock64(); } else dbg[k] = (unsigned long long)(clock64() - ck1); } } while (0)
    ATT_STAMP(0);
    const int pos = L - 1;
    const int newrow = (a.qkv_acc && pos >= p0 && pos < p1) ? pos - p0 : -1;
    if (np > 0) attn_stage_kv(a, p0, np, newrow, kvbase);
    wait_range(P.counters, a.dep_base + g, a.dep_base + g, a.dep_target[g]);  // q / new row ready
    ATT_STAMP(1);
    if (np > 0) {
        attn_stage_q(a, g, pos, newrow, kvbase);
        __syncthreads();
        ATT_STAMP(2);
        // scores: thread -> (head, position) pairs, 4 independent chains
        const float rs = rsqrtf((float)hd);
        const bool bf = a.kv_dtype == TEAL_BF16;
        const int vpr = hd * (bf ? 2 : 4) / 16;
#pragma unroll 1
        for (int i = tid; i < G * np; i += NT) {
            const int h = i / np, p = i - h * np;
            const float4* qv = reinterpret_cast<const float4*>(s.u.a.q + h * hd);
            const uint4* kv = s.u.a.k + p * (vpr + 1);
            float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bf) {
#pragma unroll 2
                for (int c = 0; c < vpr; ++c) {  // 8 elements per 16 B
                    const uint4 y = kv[c];
                    const float4 x0 = qv[2 * c], x1 = qv[2 * c + 1];
                    acc4.x = fmaf(x0.x, bf16_lo(y.x), acc4.x);
                    acc4.y = fmaf(x0.y, bf16_hi(y.x), acc4.y);
                    acc4.z = fmaf(x0.z, bf16_lo(y.y), acc4.z);
                    acc4.w = fmaf(x0.w, bf16_hi(y.y), acc4.w);
                    acc4.x = fmaf(x1.x, bf16_lo(y.z), acc4.x);
                    acc4.y = fmaf(x1.y, bf16_hi(y.z), acc4.y);
                    acc4.z = fmaf(x1.z, bf16_lo(y.w), acc4.z);
                    acc4.w = fmaf(x1.w, bf16_hi(y.w), acc4.w);
                }
            } else {
#pragma unroll 2
                for (int c = 0; c < vpr; ++c) {
                    const uint4 y = kv[c];
                    const float4 x = qv[c];
                    acc4.x = fmaf(x.x, __uint_as_float(y.x), acc4.x);
                    acc4.y = fmaf(x.y, __uint_as_float(y.y), acc4.y);
                    acc4.z = fmaf(x.z, __uint_as_float(y.z), acc4.z);
                    acc4.w = fmaf(x.w, __uint_as_float(y.w), acc4.w);
                }
            }
            s.u.a.sc[h * ATT_MAXCHUNK + p] = ((acc4.x + acc4.y) + (acc4.z + acc4.w)) * rs;
        }
        __syncthreads();
        ATT_STAMP(3);
        // softmax statistics: warp per head
#pragma unroll 1
        for (int h = warp; h < G; h += NW) {
            float mx = -INFINITY;
            for (int p = lane; p < np; p += 32) mx = fmaxf(mx, s.u.a.sc[h * ATT_MAXCHUNK + p]);
            mx = warp_max(mx);
            float l = 0.f;
            for (int p = lane; p < np; p += 32) {
                const float e = expf(s.u.a.sc[h * ATT_MAXCHUNK + p] - mx);
                s.u.a.sc[h * ATT_MAXCHUNK + p] = e;
                l += e;
            }
            l = warp_sum(l);
            if (lane == 0) { s.am[h] = mx; s.al[h] = l; }
        }
        __syncthreads();
        // context partial: thread -> (head, pair of dims), positions in four
        // independent chains (p mod 4, summed (0+1)+(2+3)) so the chain depth
        // is np/4; 32-bit V loads (bf16 pair) / 64-bit (fp32 pair), the
        // probabilities as float4 broadcasts.  A single chunk holding every
        // position is final: normalise and write the context (no record,
        // ticket, combine).
        const bool single = (p0 == 0 && p1 == L);
        const int hp = hd >> 1;
#pragma unroll 1
        for (int o = tid; o < G * hp; o += NT) {
            const int h = o / hp, dp = o - h * hp;
            const float* pr = s.u.a.sc + h * ATT_MAXCHUNK;
            float cx[4] = {0.f, 0.f, 0.f, 0.f}, cy[4] = {0.f, 0.f, 0.f, 0.f};
            int p = 0;
            if (bf) {
                const uint32_t* vc = reinterpret_cast<const uint32_t*>(s.u.a.v) + dp;
#pragma unroll 2
                for (; p + 3 < np; p += 4) {
                    const float4 pp = *reinterpret_cast<const float4*>(pr + p);
                    const uint32_t u0 = vc[p * hp], u1 = vc[(p + 1) * hp], u2 = vc[(p + 2) * hp], u3 = vc[(p + 3) * hp];
                    cx[0] = fmaf(pp.x, bf16_lo(u0), cx[0]); cy[0] = fmaf(pp.x, bf16_hi(u0), cy[0]);
                    cx[1] = fmaf(pp.y, bf16_lo(u1), cx[1]); cy[1] = fmaf(pp.y, bf16_hi(u1), cy[1]);
                    cx[2] = fmaf(pp.z, bf16_lo(u2), cx[2]); cy[2] = fmaf(pp.z, bf16_hi(u2), cy[2]);
                    cx[3] = fmaf(pp.w, bf16_lo(u3), cx[3]); cy[3] = fmaf(pp.w, bf16_hi(u3), cy[3]);
                }
#pragma unroll
                for (int k = 0; k < 3; ++k)  // tail (< 4 positions): chain k
                    if (p + k < np) {
                        const uint32_t u = vc[(p + k) * hp];
                        cx[k] = fmaf(pr[p + k], bf16_lo(u), cx[k]);
                        cy[k] = fmaf(pr[p + k], bf16_hi(u), cy[k]);
                    }
            } else {
                const float2* vc = reinterpret_cast<const float2*>(s.u.a.v) + dp;
#pragma unroll 2
                for (; p + 3 < np; p += 4) {
                    const float4 pp = *reinterpret_cast<const float4*>(pr + p);
                    const float2 u0 = vc[p * hp], u1 = vc[(p + 1) * hp], u2 = vc[(p + 2) * hp], u3 = vc[(p + 3) * hp];
                    cx[0] = fmaf(pp.x, u0.x, cx[0]); cy[0] = fmaf(pp.x, u0.y, cy[0]);
                    cx[1] = fmaf(pp.y, u1.x, cx[1]); cy[1] = fmaf(pp.y, u1.y, cy[1]);
                    cx[2] = fmaf(pp.z, u2.x, cx[2]); cy[2] = fmaf(pp.z, u2.y, cy[2]);
                    cx[3] = fmaf(pp.w, u3.x, cx[3]); cy[3] = fmaf(pp.w, u3.y, cy[3]);
                }
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (p + k < np) {
                        const float2 u = vc[(p + k) * hp];
                        cx[k] = fmaf(pr[p + k], u.x, cx[k]);
                        cy[k] = fmaf(pr[p + k], u.y, cy[k]);
                    }
            }
            float2 r = make_float2((cx[0] + cx[1]) + (cx[2] + cx[3]), (cy[0] + cy[1]) + (cy[2] + cy[3]));
            const int oo = h * hd + 2 * dp;
            if (single) {
                r.x = r.x / s.al[h];
                r.y = r.y / s.al[h];
                *reinterpret_cast<float2*>(a.ctx + (int64_t)g * G * hd + oo) = r;
            } else {
                __stcg(reinterpret_cast<float2*>(my + oo), r);
            }
        }
        if (single) {
            ATT_STAMP(4);
            signal(P.counters, a.sig_base + g, a.sig_base + g);
            ATT_STAMP(5);
            return;
        }
        if (tid < G) {
            __stcg(my + G * hd + tid, s.am[tid]);
            __stcg(my + G * hd + G + tid, s.al[tid]);
        }
    } else if (tid < G) {
        __stcg(my + G * hd + tid, -INFINITY);
        __stcg(my + G * hd + G + tid, 0.f);
    }
    // only the chunks holding positions take part (the attn phase skips the rest)
    const int nact = min(a.nchunks, (L + a.chunk - 1) / a.chunk);
    const bool last = take_ticket(a.tickets + g, (unsigned)nact - 1u, s.last);
    if (!last) return;
    const float* rb = a.partials + (int64_t)g * a.nchunks * rec;
    for (int q = tid; q < nact * 2 * G; q += NT) {  // (m, l) of every active chunk -> smem
        const int c = q / (2 * G), k = q % (2 * G);
        s.u.a.sc[q] = __ldcg(rb + (int64_t)c * rec + G * hd + k);
    }
    __syncthreads();
#pragma unroll 1
    for (int o = tid; o < G * hd; o += NT) {
        const int h = o / hd;
        float M = -INFINITY;
        for (int c = 0; c < nact; ++c)
            if (s.u.a.sc[c * 2 * G + G + h] > 0.f) M = fmaxf(M, s.u.a.sc[c * 2 * G + h]);
        float num = 0.f, dn = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < nact; c0 += 4) {
            float pv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pv[q] = (c0 + q < nact) ? __ldcg(rb + (int64_t)(c0 + q) * rec + o) : 0.f;
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                const int c = c0 + q;
                if (c < nact) {
                    const float ls = s.u.a.sc[c * 2 * G + G + h];
                    if (ls > 0.f) {
                        const float sc = expf(s.u.a.sc[c * 2 * G + h] - M);
                        num = fmaf(pv[q], sc, num);
                        dn = fmaf(ls, sc, dn);
                    }
                }
            }
        }
        a.ctx[(int64_t)g * G * hd + o] = num / dn;
    }
    ATT_STAMP(4);
    signal(P.counters, a.sig_base + g, a.sig_base + g);
    ATT_STAMP(5);
#undef ATT_STAMP
}


// Long-context attention unit (kernel variant long_ctx): unit (g, su) walks
// chunks [su*S, su*S + S) with an online softmax — per chunk the staged K/V,
// scores, running max / sum update (previous context rescaled by
// exp(m_old - m_new)) — and writes ONE record for the S chunks, so a long
// context has S x fewer units and records for the last arriver to combine.
__device__ __noinline__ void attn_unit_multi(const teal_step_plan& P, const teal_step_attn& a, int g, int su, int L) {
    Smem& s = smem();
    constexpr int QO = ATT_MAXG * ATT_MAXHD / NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = a.H / a.KVH, hd = a.hd, S = a.super_chunks;
    const int nact = min(a.nchunks, (L + a.chunk - 1) / a.chunk);
    const int nsu = (nact + S - 1) / S;
    const int c0 = su * S, c1 = min(nact, c0 + S);
    const int rec = G * hd + 2 * G;
    float* my = a.partials + ((int64_t)g * a.nchunks + su) * rec;
    const int64_t kvbase = (int64_t)g * a.max_seq * hd;
    const int pos = L - 1;
    const float rs = rsqrtf((float)hd);
    const bool bf = a.kv_dtype == TEAL_BF16;
    const int vpr = hd * (bf ? 2 : 4) / 16;
    float accv[QO];
#pragma unroll
    for (int j = 0; j < QO; ++j) accv[j] = 0.f;
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        const int p0 = c * a.chunk, p1 = min(L, p0 + a.chunk), np = p1 - p0;
        const int newrow = (a.qkv_acc && pos >= p0 && pos < p1) ? pos - p0 : -1;
        attn_stage_kv(a, p0, np, newrow, kvbase);
        if (c == c0) wait_range(P.counters, a.dep_base + g, a.dep_base + g, a.dep_target[g]);
        attn_stage_q(a, g, pos, newrow, kvbase);
        __syncthreads();
#pragma unroll 1
        for (int i = tid; i < G * np; i += NT) {
            const int h = i / np, p = i - h * np;
            const float4* qv = reinterpret_cast<const float4*>(s.u.a.q + h * hd);
            const uint4* kv = s.u.a.k + p * (vpr + 1);
            float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bf) {
#pragma unroll 2
                for (int e = 0; e < vpr; ++e) {
                    const uint4 y = kv[e];
                    const float4 x0 = qv[2 * e], x1 = qv[2 * e + 1];
                    acc4.x = fmaf(x0.x, bf16_lo(y.x), acc4.x);
                    acc4.y = fmaf(x0.y, bf16_hi(y.x), acc4.y);
                    acc4.z = fmaf(x0.z, bf16_lo(y.y), acc4.z);
                    acc4.w = fmaf(x0.w, bf16_hi(y.y), acc4.w);
                    acc4.x = fmaf(x1.x, bf16_lo(y.z), acc4.x);
                    acc4.y = fmaf(x1.y, bf16_hi(y.z), acc4.y);
                    acc4.z = fmaf(x1.z, bf16_lo(y.w), acc4.z);
                    acc4.w = fmaf(x1.w, bf16_hi(y.w), acc4.w);
                }
            } else {
#pragma unroll 2
                for (int e = 0; e < vpr; ++e) {
                    const uint4 y = kv[e];
                    const float4 x = qv[e];
                    acc4.x = fmaf(x.x, __uint_as_float(y.x), acc4.x);
                    acc4.y = fmaf(x.y, __uint_as_float(y.y), acc4.y);
                    acc4.z = fmaf(x.z, __uint_as_float(y.z), acc4.z);
                    acc4.w = fmaf(x.w, __uint_as_float(y.w), acc4.w);
                }
            }
            s.u.a.sc[h * ATT_MAXCHUNK + p] = ((acc4.x + acc4.y) + (acc4.z + acc4.w)) * rs;
        }
        __syncthreads();
        // online softmax: warp per head; s.col[h] = rescale of the previous context
#pragma unroll 1
        for (int h = warp; h < G; h += NW) {
            float mx = -INFINITY;
            for (int p = lane; p < np; p += 32) mx = fmaxf(mx, s.u.a.sc[h * ATT_MAXCHUNK + p]);
            mx = warp_max(mx);
            const float mold = c == c0 ? -INFINITY : s.am[h];
            const float mnew = fmaxf(mold, mx);
            float l = 0.f;
            for (int p = lane; p < np; p += 32) {
                const float e = expf(s.u.a.sc[h * ATT_MAXCHUNK + p] - mnew);
                s.u.a.sc[h * ATT_MAXCHUNK + p] = e;
                l += e;
            }
            l = warp_sum(l);
            if (lane == 0) {
                const float sc = c == c0 ? 0.f : expf(mold - mnew);
                s.col[h] = sc;
                s.am[h] = mnew;
                s.al[h] = (c == c0 ? 0.f : s.al[h] * sc) + l;
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < QO; ++j) {
            const int o = tid + j * NT;
            if (o >= G * hd) continue;
            const int h = o / hd, dd = o - h * hd;
            const float* pr = s.u.a.sc + h * ATT_MAXCHUNK;
            float x0 = 0.f, x1 = 0.f;
            if (bf) {
                const uint16_t* vc = reinterpret_cast<const uint16_t*>(s.u.a.v) + dd;
                for (int p = 0; p + 1 < np; p += 2) {
                    x0 = fmaf(pr[p], bf16_to_f32(vc[p * hd]), x0);
                    x1 = fmaf(pr[p + 1], bf16_to_f32(vc[(p + 1) * hd]), x1);
                }
                if (np & 1) x0 = fmaf(pr[np - 1], bf16_to_f32(vc[(np - 1) * hd]), x0);
            } else {
                const float* vc = reinterpret_cast<const float*>(s.u.a.v) + dd;
                for (int p = 0; p + 1 < np; p += 2) {
                    x0 = fmaf(pr[p], vc[p * hd], x0);
                    x1 = fmaf(pr[p + 1], vc[(p + 1) * hd], x1);
                }
                if (np & 1) x0 = fmaf(pr[np - 1], vc[(np - 1) * hd], x0);
            }
            accv[j] = fmaf(accv[j], s.col[h], x0 + x1);
        }
        __syncthreads();  // the next chunk's staging rewrites K/V, q and the scores
    }
    if (nsu == 1) {  // one unit holds every position: the context is final
#pragma unroll
        for (int j = 0; j < QO; ++j) {
            const int o = tid + j * NT;
            if (o < G * hd) a.ctx[(int64_t)g * G * hd + o] = accv[j] / s.al[o / hd];
        }
        signal(P.counters, a.sig_base + g, a.sig_base + g);
        return;
    }
#pragma unroll
    for (int j = 0; j < QO; ++j) {
        const int o = tid + j * NT;
        if (o < G * hd) __stcg(my + o, accv[j]);
    }
    if (tid < G) {
        __stcg(my + G * hd + tid, s.am[tid]);
        __stcg(my + G * hd + G + tid, s.al[tid]);
    }
    if (!take_ticket(a.tickets + g, (unsigned)nsu - 1u, s.last)) return;
    const float* rb = a.partials + (int64_t)g * a.nchunks * rec;
    for (int q = tid; q < nsu * 2 * G; q += NT) {  // (m, l) of every record -> smem
        const int c = q / (2 * G), k = q % (2 * G);
        s.u.a.sc[q] = __ldcg(rb + (int64_t)c * rec + G * hd + k);
    }
    __syncthreads();
#pragma unroll 1
    for (int o = tid; o < G * hd; o += NT) {
        const int h = o / hd;
        float M = -INFINITY;
        for (int c = 0; c < nsu; ++c)
            if (s.u.a.sc[c * 2 * G + G + h] > 0.f) M = fmaxf(M, s.u.a.sc[c * 2 * G + h]);
        float num = 0.f, dn = 0.f;
#pragma unroll 1
        for (int cb = 0; cb < nsu; cb += 16) {  // 16 records in flight (clamped indices)
            float pv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pv[q] = __ldcg(rb + (int64_t)(cb + q < nsu ? cb + q : 0) * rec + o);
#pragma unroll 1
            for (int q = 0; q < 16; ++q) {
                const int c = cb + q;
                if (c < nsu) {
                    const float ls = s.u.a.sc[c * 2 * G + G + h];
                    if (ls > 0.f) {
                        const float sc = expf(s.u.a.sc[c * 2 * G + h] - M);
                        num = fmaf(pv[q], sc, num);
                        dn = fmaf(ls, sc, dn);
                    }
                }
            }
        }
        a.ctx[(int64_t)g * G * hd + o] = num / dn;
    }
    signal(P.counters, a.sig_base + g, a.sig_base + g);
}

template <bool LC>
__device__ void attn_phase(const teal_step_plan& P, const teal_step_phase& ph, Smem& s) {
    const teal_step_attn& a = P.attns[ph.group];
    // the sequence length is written by this step's load phase: a CTA that had
    // no qkv slice reaches this point without having waited for it (the
    // phase's GLOBAL dependency; none when the load ran in an earlier launch)
    if (ph.dep_kind == TEAL_DEP_GLOBAL) {
        if (P.tp) wait_range_sys(P.counters, ph.dep, ph.dep, ph.target);
        else wait_range(P.counters, ph.dep, ph.dep, ph.target);
    }
    const int L = __ldcg(P.state + 1);
    const int nact = min(a.nchunks, (L + a.chunk - 1) / a.chunk);  // chunks holding positions
    const int nu = LC ? a.KVH * ((nact + a.super_chunks - 1) / a.super_chunks) : a.KVH * nact;
    const int G = gridDim.x;
    // the units fit on the CTAs the qkv phase leaves idle: unit u on CTA home + u
    // (they stage their K/V rows while qkv streams and poll from the start)
    if (a.home > 0 && nu <= G - a.home) {
        const int u = (int)blockIdx.x - a.home;
        if (u >= 0 && u < nu) {
            const int g = u % a.KVH, ch = u / a.KVH;
            if constexpr (LC) attn_unit_multi(P, a, g, ch, L);
            else attn_unit(P, a, g, ch, L);
        }
        return;
    }
    // otherwise unit u = (chunk u / KVH, kv group u % KVH) runs on CTA G-1 - (u*G)/nu:
    // spread over the grid from its end (the qkv phase leaves the last CTAs idle)
    const int cr = G - 1 - (int)blockIdx.x;
    for (int u = (int)(((int64_t)cr * nu + G - 1) / G); u < nu && (int64_t)u * G / nu == cr; ++u) {
        const int g = u % a.KVH, ch = u / a.KVH;  // (the unit waits for its q/k/v tiles itself)
        if constexpr (LC) attn_unit_multi(P, a, g, ch, L);
        else attn_unit(P, a, g, ch, L);
        __syncthreads();
    }
}

// Counter 0 (the step's load / accumulator zeroing) — with fused tensor
// parallelism on every rank: no rank adds into a peer's accumulators before
// that peer has zeroed them (targets world x grid).
__device__ __forceinline__ void load_signal(const teal_step_plan& P) {
    if (!P.tp) {
        signal(P.counters, 0, 0);
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < P.tp->world; ++j) red_release_sys(P.tp->counters[j], 1);
}

// ---- residual load: x = emb[token] (or x_in); ss partials; {pos, len} ---------
__device__ __noinline__ void load_phase(const teal_step_plan& P) {
    Smem& s = smem();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (P.tp) {  // every rank has finished (and reset) the previous step before anyone signals this one
        if (tid == 0) {
            const unsigned* ep = P.tp->epoch[P.tp->rank];
            const int mine = ld_acquire_sys(reinterpret_cast<const int*>(ep + P.tp->rank));
            const unsigned long long t0 = gtimer_();
            for (int j = 0; j < P.tp->world; ++j)
                while (ld_acquire_sys(reinterpret_cast<const int*>(ep + j)) < mine) {
                    __nanosleep(128);
                    if (gtimer_() - t0 > 10000000000ull) asm volatile("trap;");
                }
        }
        __syncthreads();
    }
    if (P.acc_zero) {  // every CTA zeroes its share of this step's ACC accumulators (16 B stores)
        int4* z = reinterpret_cast<int4*>(P.acc_zero);
        const int64_t n2 = P.acc_zero_n >> 1;
        for (int64_t i = (int64_t)blockIdx.x * NT + tid; i < n2; i += (int64_t)gridDim.x * NT) z[i] = make_int4(0, 0, 0, 0);
    }
    if (blockIdx.x != 0) {
        load_signal(P);
        return;
    }
    if (tid == 0) {
        const int len = P.state[1];
        // the step writes K/V row `len`: past max_seq it would land in the next
        // head's / layer's cache slice — fail loudly (the engines also check
        // on the host; inside a graph replay only this guard can)
        if (len < 0 || (P.max_seq > 0 && len >= P.max_seq)) asm volatile("trap;");
        P.state[0] = len;
        P.state[1] = len + 1;
    }
    const int tok = P.emb ? __ldcg(P.token) : 0;
    const int nt = P.d / TW;  // <= NT tiles (d <= 65536)
    float* sq = s.u.g.xs;     // squares of 16 tiles (scratch)
    // Each source type in its own straight-line batch of loads (a branch per
    // element would let the compiler wait on every load at the reconvergence
    // point: 13 us instead of one round trip for the embedding row).
#pragma unroll 1
    for (int t0 = 0; t0 < nt; t0 += 16) {
        float xv[16];
        if (P.emb && P.emb_dtype == TEAL_BF16) {
            const uint16_t* row = reinterpret_cast<const uint16_t*>(P.emb) + (int64_t)tok * P.d;
            uint16_t u[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) u[q] = (t0 + q < nt) ? __ldg(row + (t0 + q) * TW + tid) : (uint16_t)0;
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = bf16_to_f32(u[q]);
        } else if (P.emb) {
            const float* row = reinterpret_cast<const float*>(P.emb) + (int64_t)tok * P.d;
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = (t0 + q < nt) ? __ldg(row + (t0 + q) * TW + tid) : 0.f;
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = (t0 + q < nt) ? __ldcg(P.x_in + (t0 + q) * TW + tid) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if (t0 + q < nt) P.x[(int64_t)(t0 + q) * TW + tid] = xv[q];
            sq[q * TW + tid] = xv[q] * xv[q];
        }
        __syncthreads();
        // per tile: warp w sums tiles w, w + 8 (lane-strided, then a fixed shuffle tree)
        for (int q = warp; q < 16 && t0 + q < nt; q += NW) {
            float a = 0.f;
            for (int k = lane; k < TW; k += 32) a += sq[q * TW + k];
            a = warp_sum(a);
            if (lane == 0) P.ss[t0 + q] = a;
        }
        __syncthreads();
    }
    load_signal(P);
}

// ---- residual materialisation (plans without an LM head) --------------------
__device__ void resid_phase(const teal_step_plan& P, const teal_step_phase& ph, const teal_step_group& g) {
    wait_range(P.counters, ph.dep, ph.dep, ph.target);
    for (int i = blockIdx.x * NT + threadIdx.x; i < g.m; i += gridDim.x * NT)
        g.x_out[i] = __ldcg(g.x + i) + from_fx(__ldcg(g.in_acc + i));
}

// MINB resident CTAs per SM (register budget 65536 / (NT * MINB)); UB rows in
// flight per warp per pipeline stage.
template <int WT, int MINB, int UB, bool LC = false>
__global__ void __launch_bounds__(NT, MINB) step_kernel(const __grid_constant__ teal_step_plan P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint64_t pol = l2_evict_first_policy();
    const int pend = P.phase_end > 0 ? P.phase_end : P.nphases;
    for (int p = P.phase_begin; p < pend; ++p) {
        const teal_step_phase ph = P.phases[p];
        unsigned long long* tl = P.timeline ? P.timeline + ((int64_t)blockIdx.x * P.nphases + p) * 8 : nullptr;
        if (tl && tid == 0) tl[0] = gtimer();
        if (ph.kind == TEAL_PHASE_GEMV) gemv_slice_t<WT, UB>(P, ph, P.groups[ph.group], s, pol, tl);
        else if (ph.kind == TEAL_PHASE_ATTN) attn_phase<LC>(P, ph, s);
        else if (ph.kind == TEAL_PHASE_RESID) resid_phase(P, ph, P.groups[ph.group]);
        else load_phase(P);
        __syncthreads();
        if (tl && tid == 0) tl[1] = gtimer();
    }
    if (tid == 0) {
        if (P.tp) __threadfence_system();
        else __threadfence();
        const unsigned prev = atomicAdd(P.ctrl, 1u);
        if (prev == gridDim.x - 1u) {
            for (int i = 0; i < P.ncounters; ++i) P.counters[(int64_t)i * CSTRIDE] = 0;
            P.ctrl[0] = 0u;
            __threadfence();
            if (P.tp) {  // this rank completed one more step: tell every rank
                const teal_step_tp& T = *P.tp;
                const unsigned e = T.epoch[T.rank][T.rank] + 1u;
                __threadfence_system();
                for (int j = 0; j < T.world; ++j)
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(T.epoch[j] + T.rank), "r"(e) : "memory");
            }
        }
    }
}

// Kernel variants: 2 CTAs/SM with 6 rows per pipeline stage (128 registers;
// measured on the 8B step: UB 5 / 6 / 7 / 8 / 10 -> 370 / 413 / 410 / 406 /
// 361 tok/s at 50%; 3 CTAs/SM with 4 rows per stage spilled and was slower),
// and the long-context attention variant of the same configuration.
template <int WT>
static void* kernel_ptr_t(bool lc) {
    if (lc) return (void*)step_kernel<WT, 2, 6, true>;
    return (void*)step_kernel<WT, 2, 6>;
}

static void* kernel_ptr(int w_dtype, bool lc = false) {
    switch (w_dtype) {
        case TEAL_BF16: return kernel_ptr_t<TEAL_BF16>(lc);
        case TEAL_I8: return kernel_ptr_t<TEAL_I8>(lc);
        case TEAL_I4: return kernel_ptr_t<TEAL_I4>(lc);
        default: return kernel_ptr_t<TEAL_F32>(lc);
    }
}

static int occupancy(int w_dtype) {
    static int cached[4] = {-1, -1, -1, -1};
    int& cache = cached[w_dtype & 3];
    if (cache < 0) {
        const void* k = kernel_ptr(w_dtype);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, NT, kSmemBytes) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        cache = b;
    }
    return cache;
}

// ---- single sparse/dense GEMV on the step streaming core -----------------------
// y = s_t(x) W^T over an UNTILED input-major W (row stride ldw): one ordinary
// launch with a single GEMV phase (no dependencies, no signals), split tiles
// combined by tickets.  Used by teal_fused_gemv for plain single-projection
// calls (kernel.sparse_gemv, matmul_dense, the GEMV sweep).
struct OneArgs {
    teal_step_plan P;
    teal_step_group g;
    teal_step_phase ph;
};

template <int WT, int MINB, int UB>
__global__ void __launch_bounds__(NT, MINB) gemv_one_kernel(const __grid_constant__ OneArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const uint64_t pol = l2_evict_first_policy();
    gemv_slice_t<WT, UB>(A.P, A.ph, A.g, s, pol, nullptr);
}

template <int WT>
static void* one_kernel_ptr() { return (void*)gemv_one_kernel<WT, 2, 8>; }

static int max_contrib(int ntiles, int m, int G) {
    const int64_t gpt = (m + 31) / 32, F = (int64_t)ntiles * gpt;
    int mc = 1;
    for (int t = 0; t < ntiles; ++t) {
        const int cf = (int)(((int64_t)t * gpt + 1) * G - 1) / F;
        const int cl = (int)((((int64_t)t + 1) * gpt) * G - 1) / F;
        if (cl - cf + 1 > mc) mc = cl - cf + 1;
    }
    return mc;
}

// participants() on the host (mirror of the device rule)
static int host_participants(int ntiles, int64_t F, int grid) {
    if (F <= grid) return (int)F;
    const int aligned = ntiles * (grid / ntiles);
    if (2 * ntiles <= grid && 10 * aligned >= 9 * grid) return aligned;
    return grid;
}

}  // namespace step

// eligibility + workspace of the single-GEMV path (-1: not eligible)
int step_gemv_eligible(const teal_gemv_args* a, int64_t* ws_floats, int64_t* tickets, int* grid_out) {
    using namespace step;
    if (!a || a->nseg != 1 || a->prologue != TEAL_PRO_PLAIN || a->epilogue != TEAL_EPI_STORE) return -1;
    if (a->x_dtype != TEAL_F32) return -1;
    if (a->w_dtype != TEAL_BF16 && a->w_dtype != TEAL_F32 && a->w_dtype != TEAL_I8) return -1;
    const teal_seg& sg = a->seg[0];
    if (sg.n % 8 || sg.ldw % 8 || (reinterpret_cast<uintptr_t>(sg.w) & 15) || sg.dbg_bits) return -1;
    if (a->m > (1 << 29)) return -1;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    cudaGetLastError();
    int grid = a->ctas > 0 ? a->ctas : 2 * sms;
    const int ntiles = (int)((sg.n + TW - 1) / TW);
    const int64_t F = (int64_t)ntiles * ((a->m + 31) / 32);
    grid = (int)min64(grid, F);
    const int G = host_participants(ntiles, F, grid);
    if (ws_floats) *ws_floats = (int64_t)ntiles * max_contrib(ntiles, (int)a->m, G) * TW;
    if (tickets) *tickets = ntiles;
    if (grid_out) *grid_out = grid;
    return 0;
}

int step_gemv_single(const teal_gemv_args* a, cudaStream_t stream) {
    using namespace step;
    int grid = 0;
    int64_t wsf = 0, ntk = 0;
    if (step_gemv_eligible(a, &wsf, &ntk, &grid) != 0) return -1;
    const teal_seg& sg = a->seg[0];
    OneArgs A;
    memset(&A, 0, sizeof(A));
    teal_step_group& g = A.g;
    const int esz = a->w_dtype == TEAL_F32 ? 4 : (a->w_dtype == TEAL_BF16 ? 2 : 1);
    g.w = sg.w;
    g.col_scale = sg.col_scale;
    g.tiles = nullptr;
    g.t_all = sg.t32;
    g.x = reinterpret_cast<const float*>(a->x);
    g.partials = a->ws;
    g.tickets = a->tickets;
    g.y = sg.y;
    g.kept[0] = sg.kept;
    g.m = (int)a->m;
    g.n = (int)sg.n;
    g.ntiles = (int)((sg.n + TW - 1) / TW);
    const int64_t F = (int64_t)g.ntiles * ((a->m + 31) / 32);
    g.maxc = max_contrib(g.ntiles, g.m, host_participants(g.ntiles, F, grid));
    g.prologue = TEAL_PRO_PLAIN;
    g.epilogue = TEAL_SEPI_STORE;
    g.w_dtype = a->w_dtype;
    g.row_stride_b = sg.ldw * esz;
    g.tile_stride_b = (int64_t)TW * esz;
    A.ph.kind = TEAL_PHASE_GEMV;
    A.ph.dep_kind = TEAL_DEP_NONE;
    A.ph.dep_rows = 1;
    void* k = a->w_dtype == TEAL_BF16 ? one_kernel_ptr<TEAL_BF16>()
              : a->w_dtype == TEAL_F32 ? one_kernel_ptr<TEAL_F32>() : one_kernel_ptr<TEAL_I8>();
    static bool attr_done[4] = {false, false, false, false};
    if (!attr_done[a->w_dtype & 3]) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        attr_done[a->w_dtype & 3] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[1] = {(void*)&A};
    cudaLaunchKernelExC(&cfg, k, args);
    return check_launch("teal_sparse_gemv");
}

}  // namespace teal

using namespace teal;
using namespace teal::step;

extern "C" {

int teal_step_ctas_per_sm(int w_dtype) {
    if (w_dtype == TEAL_BF16 || w_dtype == TEAL_F32 || w_dtype == TEAL_I8 || w_dtype == TEAL_I4) return occupancy(w_dtype);
    return 0;
}

int teal_step_launch(const teal_step_plan* p, cudaStream_t stream) {
    TEAL_REQUIRE(p && p->groups && p->phases && p->counters && p->ctrl && p->x && p->ss && p->state,
                 "teal_step_launch: null plan field");
    TEAL_REQUIRE(p->nphases >= 1 && p->ncounters >= 1, "teal_step_launch: empty plan");
    TEAL_REQUIRE(p->phase_begin >= 0 && p->phase_end >= 0 && p->phase_end <= p->nphases &&
                     (p->phase_end == 0 || p->phase_begin < p->phase_end),
                 "teal_step_launch: bad phase range [%d, %d)", p->phase_begin, p->phase_end);
    TEAL_REQUIRE(!p->acc_zero || (p->acc_zero_n % 2 == 0 && (reinterpret_cast<uintptr_t>(p->acc_zero) & 15) == 0),
                 "teal_step_launch: acc_zero must be 16-byte aligned with an even element count");
    TEAL_REQUIRE(p->d >= TW && p->d % TW == 0, "teal_step_launch: d must be a multiple of %d", TW);
    TEAL_REQUIRE(p->w_dtype == TEAL_BF16 || p->w_dtype == TEAL_F32 || p->w_dtype == TEAL_I8 || p->w_dtype == TEAL_I4,
                 "teal_step_launch: weights must be bf16, fp32, int8 or int4");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per = teal_step_ctas_per_sm(p->w_dtype);
    TEAL_REQUIRE(per >= 1, "teal_step_launch: kernel cannot be resident");
    TEAL_REQUIRE(p->ctas >= 1 && p->ctas <= per * sms,
                 "teal_step_launch: plan built for %d CTAs, %d resident", p->ctas, per * sms);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p->ctas);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p->noncoop ? 0 : 1;
    void* args[1] = {(void*)p};
    const void* k = kernel_ptr(p->w_dtype, p->long_ctx != 0);
    if (p->long_ctx) {  // (the default variant gets its attribute in occupancy())
        static bool lc_attr[4] = {false, false, false, false};
        if (!lc_attr[p->w_dtype & 3]) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
            lc_attr[p->w_dtype & 3] = true;
        }
    }
    cudaLaunchKernelExC(&cfg, k, args);
    return check_launch("teal_step_launch");
}

}  // extern "C"
