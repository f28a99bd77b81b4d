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
//     stream, so CTAs finish a phase together.  A range spans a few tiles;
//     a tile shared by several CTAs is finished by its last-arriving
//     contributor (ticket), which sums the fp32 partials in contributor order
//     (deterministic two-phase reduction) and runs the fused epilogue.
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
//   2. warp w takes kept rows w, w+8, ...; its lane 0 keeps S row chunks in
//      flight with cp.async.bulk (TMA engine, L2 evict-first) into the warp's
//      private shared-memory ring (one mbarrier per slot, only the kept
//      halves are copied); lanes read 16 B each and FMA into fp32 registers;
//   3. fixed-order cross-warp reduction -> TW column sums.
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
constexpr int ATT_MAXG = 8;
constexpr int ATT_MAXHD = 128;
constexpr int ATT_MAXCHUNK = 256;
constexpr int ATT_STAGE = 16384;  // bytes of K (and of V) staged per attention unit
static_assert(NT == TW, "epilogues map one thread per tile column");

struct Smem {
    union {
        struct {
            int idx[MAXR];    // row - r0 | keep_lo << 30 | keep_hi << 31
            float h[MAXR];
        } g;
        struct {
            float q[ATT_MAXG * ATT_MAXHD];
            float sc[ATT_MAXG * ATT_MAXCHUNK];
            uint4 k[ATT_STAGE / 16];   // K rows of the chunk (raw cache dtype)
            uint4 v[ATT_STAGE / 16];   // V rows of the chunk
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

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Each counter lives in its own 128-byte line (index * CSTRIDE) so hundreds
// of pollers of one counter do not contend with the other counters' updates.
constexpr int CSTRIDE = 32;

// thread 0 polls with backoff; the barrier publishes the result to the CTA
__device__ __forceinline__ void wait_range(const int* counters, int c0, int c1, int target) {
    if (threadIdx.x == 0) {
        for (int c = c0; c <= c1; ++c) {
            unsigned ns = 32;
            while (ld_acquire(counters + (int64_t)c * CSTRIDE) < target) {
                __nanosleep(ns);
                ns = ns < 128 ? ns * 2 : 128;
            }
        }
    }
    __syncthreads();
}

// Publish the CTA's prior global writes, then bump the counters: the barrier
// orders every thread's writes before thread 0, whose gpu-scope fence makes
// them (cumulatively) visible before its atomics — the cooperative-groups
// grid-sync pattern, one fence per CTA instead of one per thread.
__device__ __forceinline__ void signal(int* counters, int c0, int c1) {
    __syncthreads();
    if (threadIdx.x == 0 && c0 >= 0) {
        __threadfence();
        for (int c = c0; c <= c1; ++c) atomicAdd(counters + (int64_t)c * CSTRIDE, 1);
    }
}

// Take a split-K ticket after storing this CTA's partial: returns (to every
// thread) whether this CTA arrived last; the last arriver's thread 0 fences
// again (acquire side) before the barrier that precedes the partial reads.
__device__ __forceinline__ bool take_ticket(unsigned* ticket, unsigned expected_prev, int& s_last) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(ticket, 1u);
        const int last = prev == expected_prev;
        if (last) {
            *ticket = 0u;
            __threadfence();
        }
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

// ---- epilogue of one finished column tile (thread c = column c) --------------
__device__ __noinline__ void finalize(const teal_step_plan& P, const teal_step_group& g, int tile, float v, Smem& s) {
    const int c = threadIdx.x;
    const int64_t col = (int64_t)tile * TW + c;
    const teal_step_tile tm = g.tiles[tile];
    switch (g.epilogue) {
        case TEAL_SEPI_STORE: {
            if (col < g.n) g.y[col] = v;
            break;
        }
        case TEAL_SEPI_RESID: {
            float xn = 0.f;
            if (col < g.n) {
                xn = __ldcg(g.resid + col) + v;
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
                __threadfence();
                const unsigned prev = atomicAdd(P.lm_done, 1u);
                s.last = prev == (unsigned)g.ntiles - 1u;
                if (s.last) {
                    *P.lm_done = 0u;
                    __threadfence();
                }
            }
            __syncthreads();
            if (s.last) {  // the last tile: argmax over the per-tile candidates, whole CTA
                float gv = -INFINITY;
                int gi = 0x7fffffff;
                for (int t = c; t < g.ntiles; t += NT) {
                    const float cv = __ldcg(P.cand_v + t);
                    const int ci = __ldcg(P.cand_i + t);
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
                    *P.token_out = s.wcnt[0] == 0x7fffffff ? 0 : s.wcnt[0];
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

// Per-lane accumulator columns: bf16 lane l owns [8l, 8l+8) (lanes 16..31 =
// hi half); fp32 lane l owns [4l, 4l+4) (lo) and [128+4l, 128+4l+4) (hi).
template <int ESZ>
__device__ __forceinline__ int acc_col(int lane, int j) {
    if constexpr (ESZ == 2) return lane * 8 + j;
    else return j < 4 ? lane * 4 + j : TH + lane * 4 + (j - 4);
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

// CTAs taking part in a GEMV phase: never more than the 32-row groups (every
// range non-empty) and, when the phase has at most half as many tiles as the
// grid has CTAs, a multiple of the tile count so that every range lies inside
// one tile (no CTA pays the fixed cost of a second segment; each tile has the
// same number of contributors).  Mirrored by engine.participants().
__device__ __forceinline__ int participants(int ntiles, int64_t F) {
    const int grid = gridDim.x;
    if (F <= grid) return (int)F;
    if (2 * ntiles <= grid) return ntiles * (grid / ntiles);
    return grid;
}

__device__ __forceinline__ int owner_of(int64_t gidx, int64_t F, int G) {
    return (int)(((gidx + 1) * (int64_t)G - 1) / F);
}

// Threshold + compact rows [r0, r1) of one tile into s.u.g (ordered).
__device__ int compact_rows(const teal_step_group& g, const teal_step_tile& tm, int tile, int r0, int r1,
                            float rden, bool rms, Smem& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool two = tm.seg_hi != tm.seg_lo;
    constexpr int RPT = MAXR / NT;  // rows per thread
    float hx[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {  // all x (and gain) loads in flight at once
        const int i = r0 + q * NT + tid;
        hx[q] = 0.f;
        if (i < r1) {
            const float xv = __ldcg(g.x + i);
            hx[q] = rms ? (xv / rden) * __ldg(g.gain + i) : xv;
        }
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
// the next batch of U rows' 16-byte loads issued before the current batch is
// consumed (software pipeline: 2U row chunks in flight per warp).  Only the
// kept half of a row is loaded (bf16: lanes 0-15 = lo, 16-31 = hi; fp32:
// every lane loads 16 B of each kept half).
template <int ESZ, int UB>
__device__ __forceinline__ void stream_rows(const unsigned char* tb, int cnt, const Smem& s, float acc[8],
                                            uint64_t pol) {
    constexpr int ROWB = TW * ESZ;
    constexpr int HB = ROWB / 2;
    constexpr int U = ESZ == 2 ? UB : UB / 2;
    constexpr int NV = ESZ == 2 ? 1 : 2;  // 16-byte vectors per lane per row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4 a[U][NV], b[U][NV];
    float ha[U][NV], hb[U][NV];
    auto fetch = [&](int e0, uint4 (&d)[U][NV], float (&hh)[U][NV]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                d[u][v] = make_uint4(0u, 0u, 0u, 0u);
                hh[u][v] = 0.f;
            }
            if (e < cnt) {
                const unsigned pk = (unsigned)s.u.g.idx[e];
                const float h = s.u.g.h[e];
                const unsigned char* row = tb + (int64_t)(pk & 0x3fffffffu) * ROWB + lane * 16;
                if constexpr (ESZ == 2) {
                    if ((pk >> (lane < 16 ? 30 : 31)) & 1u) {
                        d[u][0] = ldg128_stream_pol(row, pol);
                        hh[u][0] = h;
                    }
                } else {
                    if ((pk >> 30) & 1u) { d[u][0] = ldg128_stream_pol(row, pol); hh[u][0] = h; }
                    if ((pk >> 31) & 1u) { d[u][NV - 1] = ldg128_stream_pol(row + HB, pol); hh[u][NV - 1] = h; }
                }
            }
        }
    };
    auto consume = [&](const uint4 (&d)[U][NV], const float (&hh)[U][NV]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (ESZ == 2) {
                const uint32_t w4[4] = {d[u][0].x, d[u][0].y, d[u][0].z, d[u][0].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] = fmaf(hh[u][0], bf16_lo(w4[q]), acc[2 * q]);
                    acc[2 * q + 1] = fmaf(hh[u][0], bf16_hi(w4[q]), acc[2 * q + 1]);
                }
            } else {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    acc[4 * v + 0] = fmaf(hh[u][v], __uint_as_float(d[u][v].x), acc[4 * v + 0]);
                    acc[4 * v + 1] = fmaf(hh[u][v], __uint_as_float(d[u][v].y), acc[4 * v + 1]);
                    acc[4 * v + 2] = fmaf(hh[u][v], __uint_as_float(d[u][v].z), acc[4 * v + 2]);
                    acc[4 * v + 3] = fmaf(hh[u][v], __uint_as_float(d[u][v].w), acc[4 * v + 3]);
                }
            }
        }
    };
    int e0 = warp * U;
    if (e0 >= cnt) return;
    fetch(e0, a, ha);
    for (;;) {
        const int en = e0 + NW * U;
        if (en < cnt) fetch(en, b, hb);
        consume(a, ha);
        if (en >= cnt) break;
        e0 = en;
        if (e0 + NW * U < cnt) fetch(e0 + NW * U, a, ha);
        consume(b, hb);
        if (e0 + NW * U >= cnt) break;
        e0 += NW * U;
    }
}

template <int ESZ, int UB>
__device__ void gemv_slice(const teal_step_plan& P, const teal_step_phase& ph, Smem& s, uint64_t pol,
                           unsigned long long* tl) {
    const teal_step_group& g = P.groups[ph.group];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gpt = (g.m + 31) / 32;
    const int64_t F = (int64_t)g.ntiles * gpt;
    const int G = participants(g.ntiles, F), c = blockIdx.x;
    if (c >= G) return;
    const int64_t g0 = (int64_t)c * F / G, g1 = (int64_t)(c + 1) * F / G;
    const bool rms = g.prologue == TEAL_PRO_RMSNORM;
    if (ph.dep_kind == TEAL_DEP_GLOBAL) wait_range(P.counters, ph.dep, ph.dep, ph.target);
    float rden = 1.f;
    if (rms) {
        if (warp == 0) s.rden = rms_den(g, lane);
        __syncthreads();
        rden = s.rden;
    }
    constexpr int ROWB = TW * ESZ;
    int segi = 0, lasts = 0;
#define SL_STAMP(k, v) do { if (tl && tid == 0) tl[k] = (v); } while (0)
    for (int64_t gs = g0; gs < g1; ++segi) {
        const int tile = (int)(gs / gpt);
        const int64_t ge = min64(g1, (int64_t)(tile + 1) * gpt);
        const int r0 = (int)(gs - (int64_t)tile * gpt) * 32;
        const int r1 = min(g.m, (int)(ge - (int64_t)tile * gpt) * 32);
        gs = ge;
        if (ph.dep_kind == TEAL_DEP_ROWS)
            wait_range(P.counters, ph.dep + r0 / ph.dep_rows, ph.dep + (r1 - 1) / ph.dep_rows, ph.target);
        if (segi == 0) SL_STAMP(2, gtimer());
        const teal_step_tile tm = g.tiles[tile];
        const unsigned char* tbase = reinterpret_cast<const unsigned char*>(g.w) + (int64_t)tile * g.m * ROWB;
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int ra = r0; ra < r1; ra += MAXR) {
            const int rb = min(r1, ra + MAXR);
            const int cnt = compact_rows(g, tm, tile, ra, rb, rden, rms, s);
            stream_rows<ESZ, UB>(tbase + (int64_t)ra * ROWB, cnt, s, acc, pol);
            __syncthreads();  // rows list is rewritten by the next chunk
        }
        SL_STAMP(segi == 0 ? 3 : 5, gtimer());
#pragma unroll
        for (int j = 0; j < 8; ++j) s.red[warp * TW + acc_col<ESZ>(lane, j)] = acc[j];
        __syncthreads();
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += s.red[w * TW + tid];
        const int cf = owner_of((int64_t)tile * gpt, F, G);
        const int cl = owner_of((int64_t)(tile + 1) * gpt - 1, F, G);
        if (cl > cf) {
            float* slot = g.partials + ((int64_t)tile * g.maxc + (c - cf)) * TW;
            __stcg(slot + tid, v);
            if (!take_ticket(g.tickets + tile, (unsigned)(cl - cf), s.last)) {
                if (segi == 0) SL_STAMP(4, gtimer());
                continue;
            }
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
        if (g.col_scale) v *= g.col_scale[(int64_t)tile * TW + tid];
        finalize(P, g, tile, v, s);
        ++lasts;
        if (segi == 0) SL_STAMP(4, gtimer());
    }
    SL_STAMP(6, (unsigned long long)segi);
    SL_STAMP(7, (unsigned long long)lasts);
#undef SL_STAMP
}

// ---- attention unit: (kv head g, position chunk) -------------------------------
// Deliberately compact code (runtime loops over heads and head_dim chunks):
// this path runs on a few CTAs once per layer, so its instructions are cold
// in the instruction cache every time; unrolled code here costs more in
// instruction fetch than it saves in issue slots.
template <typename KT>
__device__ __noinline__ void attn_unit_t(const teal_step_plan& P, const teal_step_attn& a, int g, int ch, Smem& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = a.H / a.KVH, hd = a.hd, ndc = (hd + 31) / 32;
    const int L = __ldcg(P.state + 1);
    const int p0 = ch * a.chunk;
    const int p1 = min(L, p0 + a.chunk);
    const int np = max(0, p1 - p0);
    const int rec = G * hd + 2 * G;
    float* my = a.partials + ((int64_t)g * a.nchunks + ch) * rec;
    const int64_t kvbase = (int64_t)g * a.max_seq * hd;
    unsigned long long* dbg = a.dbg ? a.dbg + ((int64_t)g * a.nchunks + ch) * 6 : nullptr;
#define ATT_STAMP(k) do { if (dbg && tid == 0) dbg[k] = gtimer(); } while (0)
    ATT_STAMP(0);
    if (np > 0) {
        // stage q, and the chunk's K and V rows (contiguous in the cache), with
        // 16-byte loads all in flight together: one L2/HBM round trip
        constexpr int KB = (int)sizeof(KT);
        const int n16 = np * hd * KB / 16;
        const uint4* gk = reinterpret_cast<const uint4*>(reinterpret_cast<const KT*>(a.k_cache) + kvbase + (int64_t)p0 * hd);
        const uint4* gv = reinterpret_cast<const uint4*>(reinterpret_cast<const KT*>(a.v_cache) + kvbase + (int64_t)p0 * hd);
        for (int o = tid; o < G * hd; o += NT) s.u.a.q[o] = __ldcg(a.q + (int64_t)g * G * hd + o);
#pragma unroll 1
        {  // n16 <= ATT_STAGE / 16 = 4 * NT: every thread's loads in flight together
            constexpr int PER = ATT_STAGE / 16 / NT;
            uint4 kk[PER], vv[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int v = tid + q * NT;
                if (v < n16) { kk[q] = __ldcg(gk + v); vv[q] = __ldcg(gv + v); }
            }
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int v = tid + q * NT;
                if (v < n16) { s.u.a.k[v] = kk[q]; s.u.a.v[v] = vv[q]; }
            }
        }
        __syncthreads();
        const KT* ks = reinterpret_cast<const KT*>(s.u.a.k);
        const KT* vs = reinterpret_cast<const KT*>(s.u.a.v);
        const float den = sqrtf((float)hd);
        // scores: warp per position, lanes over head_dim
#pragma unroll 1
        for (int p = warp; p < np; p += NW) {
            float kr[ATT_MAXHD / 32];
#pragma unroll
            for (int dc = 0; dc < ATT_MAXHD / 32; ++dc)
                kr[dc] = (dc < ndc && lane + 32 * dc < hd) ? to_f32<KT>(ks[p * hd + lane + 32 * dc]) : 0.f;
#pragma unroll 1
            for (int h = 0; h < G; ++h) {
                float dot = 0.f;
#pragma unroll
                for (int dc = 0; dc < ATT_MAXHD / 32; ++dc)
                    if (dc < ndc && lane + 32 * dc < hd) dot = fmaf(s.u.a.q[h * hd + lane + 32 * dc], kr[dc], dot);
                dot = warp_sum(dot);
                if (lane == 0) s.u.a.sc[h * ATT_MAXCHUNK + p] = dot / den;
            }
        }
        __syncthreads();
        ATT_STAMP(1);
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
        // context partial: thread -> (head, d), positions ascending.  A
        // single chunk holding every position is final: normalise and write
        // the context directly (no partial record, ticket or combine).
        const bool single = (p0 == 0 && p1 == L);
#pragma unroll 1
        for (int o = tid; o < G * hd; o += NT) {
            const int h = o / hd, d = o - h * hd;
            const float* pr = s.u.a.sc + h * ATT_MAXCHUNK;
            float acc = 0.f;
#pragma unroll 4
            for (int p = 0; p < np; ++p) acc = fmaf(pr[p], to_f32<KT>(vs[p * hd + d]), acc);
            if (single) a.ctx[(int64_t)g * G * hd + o] = acc / s.al[h];
            else __stcg(my + o, acc);
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
    ATT_STAMP(2);
    // only the chunks holding positions take part (the attn phase skips the rest)
    const int nact_t = min(a.nchunks, (L + a.chunk - 1) / a.chunk);
    const bool last = take_ticket(a.tickets + g, (unsigned)nact_t - 1u, s.last);
    ATT_STAMP(3);
    if (!last) return;
    const float* rb = a.partials + (int64_t)g * a.nchunks * rec;
    const int nact = min(a.nchunks, (L + a.chunk - 1) / a.chunk);  // chunks holding positions
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
        float num = 0.f, dd = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < nact; c0 += 4) {
            float pv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pv[q] = (c0 + q < nact) ? __ldcg(rb + (int64_t)(c0 + q) * rec + o) : 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = c0 + q;
                if (c < nact) {
                    const float ls = s.u.a.sc[c * 2 * G + G + h];
                    if (ls > 0.f) {
                        const float sc = expf(s.u.a.sc[c * 2 * G + h] - M);
                        num = fmaf(pv[q], sc, num);
                        dd = fmaf(ls, sc, dd);
                    }
                }
            }
        }
        a.ctx[(int64_t)g * G * hd + o] = num / dd;
    }
    ATT_STAMP(4);
    signal(P.counters, a.sig_base + g, a.sig_base + g);
    ATT_STAMP(5);
#undef ATT_STAMP
}

__device__ void attn_phase(const teal_step_plan& P, const teal_step_phase& ph, Smem& s) {
    const teal_step_attn& a = P.attns[ph.group];
    // the sequence length is written by this step's load phase: a CTA that had
    // no qkv slice reaches this point without having waited for it
    wait_range(P.counters, 0, 0, 1);
    const int L = __ldcg(P.state + 1);
    const int nact = min(a.nchunks, (L + a.chunk - 1) / a.chunk);  // chunks holding positions
    const int nu = a.KVH * nact;
    const int G = gridDim.x;
    // unit u = (chunk u / KVH, kv group u % KVH) runs on CTA G-1 - (u*G)/nu:
    // spread over the grid from its end (the qkv phase leaves the last CTAs idle)
    const int cr = G - 1 - (int)blockIdx.x;
    for (int u = (int)(((int64_t)cr * nu + G - 1) / G); u < nu && (int64_t)u * G / nu == cr; ++u) {
        const int g = u % a.KVH, ch = u / a.KVH;
        wait_range(P.counters, a.dep_base + g, a.dep_base + g, a.dep_target[g]);
        if (a.kv_dtype == TEAL_BF16) attn_unit_t<uint16_t>(P, a, g, ch, s);
        else attn_unit_t<float>(P, a, g, ch, s);
        __syncthreads();
    }
}

// ---- residual load: x = emb[token] (or x_in); ss partials; {pos, len} ---------
__device__ __noinline__ void load_phase(const teal_step_plan& P, Smem& s) {
    if (blockIdx.x != 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        const int len = P.state[1];
        P.state[0] = len;
        P.state[1] = len + 1;
    }
    const int tok = P.emb ? __ldcg(P.token) : 0;
    const int nt = P.d / TW;  // <= NT tiles (d <= 65536)
    // every column this thread owns is loaded before any is used
#pragma unroll 1
    for (int t0 = 0; t0 < nt; t0 += 16) {
        float xv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            xv[q] = 0.f;
            if (t0 + q < nt) {
                const int64_t c = (int64_t)(t0 + q) * TW + tid;
                if (P.emb) {
                    const int64_t off = (int64_t)tok * P.d + c;
                    xv[q] = P.emb_dtype == TEAL_BF16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(P.emb)[off])
                                                     : reinterpret_cast<const float*>(P.emb)[off];
                } else {
                    xv[q] = __ldcg(P.x_in + c);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if (t0 + q < nt) P.x[(int64_t)(t0 + q) * TW + tid] = xv[q];
            const float w = warp_sum(xv[q] * xv[q]);
            if (lane == 0) s.red[warp * TW + q] = w;
        }
        __syncthreads();
        if (tid < 16 && t0 + tid < nt) {  // per tile: warps summed in ascending order
            float a = 0.f;
            for (int w = 0; w < NW; ++w) a += s.red[w * TW + tid];
            P.ss[t0 + tid] = a;
        }
        __syncthreads();
    }
    signal(P.counters, 0, 0);
}

// MINB resident CTAs per SM (register budget 65536 / (NT * MINB)); UB rows in
// flight per warp per pipeline stage.
template <int ESZ, int MINB, int UB>
__global__ void __launch_bounds__(NT, MINB) step_kernel(const __grid_constant__ teal_step_plan P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint64_t pol = l2_evict_first_policy();
    for (int p = 0; p < P.nphases; ++p) {
        const teal_step_phase ph = P.phases[p];
        unsigned long long* tl = P.timeline ? P.timeline + ((int64_t)blockIdx.x * P.nphases + p) * 8 : nullptr;
        if (tl && tid == 0) tl[0] = gtimer();
        if (ph.kind == TEAL_PHASE_GEMV) gemv_slice<ESZ, UB>(P, ph, s, pol, tl);
        else if (ph.kind == TEAL_PHASE_ATTN) attn_phase(P, ph, s);
        else load_phase(P, s);
        __syncthreads();
        if (tl && tid == 0) tl[1] = gtimer();
    }
    if (tid == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(P.ctrl, 1u);
        if (prev == gridDim.x - 1u) {
            for (int i = 0; i < P.ncounters; ++i) P.counters[(int64_t)i * CSTRIDE] = 0;
            P.ctrl[0] = 0u;
            __threadfence();
        }
    }
}

// Kernel variant: default 2 CTAs/SM with 8 rows per pipeline stage (128
// registers, no spills in the streaming loop); TEAL_STEP_OCC=3 selects 3
// CTAs/SM with 4 rows per stage (80 registers; measured slower: spills).
static int occ_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TEAL_STEP_OCC");
        v = (e && e[0] == '3') ? 3 : 2;
    }
    return v;
}

template <int ESZ>
static void* kernel_ptr() {
    if (occ_mode() == 2) return (void*)step_kernel<ESZ, 2, 8>;
    return (void*)step_kernel<ESZ, 3, 4>;
}

template <int ESZ>
static int occupancy() {
    static int cached = -1;
    if (cached < 0) {
        const void* k = kernel_ptr<ESZ>();
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, NT, kSmemBytes) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        cached = b;
    }
    return cached;
}

}  // namespace step
}  // namespace teal

using namespace teal;
using namespace teal::step;

extern "C" {

int teal_step_ctas_per_sm(int w_dtype) {
    if (w_dtype == TEAL_BF16) return occupancy<2>();
    if (w_dtype == TEAL_F32) return occupancy<4>();
    return 0;
}

int teal_step_launch(const teal_step_plan* p, cudaStream_t stream) {
    TEAL_REQUIRE(p && p->groups && p->phases && p->counters && p->ctrl && p->x && p->ss && p->state,
                 "teal_step_launch: null plan field");
    TEAL_REQUIRE(p->nphases >= 1 && p->ncounters >= 1, "teal_step_launch: empty plan");
    TEAL_REQUIRE(p->d >= TW && p->d % TW == 0, "teal_step_launch: d must be a multiple of %d", TW);
    TEAL_REQUIRE(p->w_dtype == TEAL_BF16 || p->w_dtype == TEAL_F32, "teal_step_launch: weights must be bf16 or fp32");
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
    cfg.numAttrs = 1;
    void* args[1] = {(void*)p};
    cudaLaunchKernelExC(&cfg, p->w_dtype == TEAL_BF16 ? kernel_ptr<2>() : kernel_ptr<4>(), args);
    return check_launch("teal_step_launch");
}

}  // extern "C"
