// Persistent decode-step kernel (sm_100a): one cooperative launch per token.
//
// Replaces the per-projection launch sequence of a decode step — the seven
// `gated(name, a) @ W.T` products of model._forward
// (pkg/src/actsparse/model.py:158-198) with their RMSNorm / SiLU*up /
// residual epilogues, causal attention (model.py:135-150, one query row over
// a KV cache), the dense LM head and greedy argmax.
//
// Execution model
//   * grid = (CTAs per SM at full occupancy) x #SMs, all co-resident
//     (cooperative launch).  Each CTA pulls work units from one device queue
//     (atomic head) in the plan's topological order, prefetching the next
//     index while it works.
//   * A unit may depend on one counter reaching a target; counters are
//     bumped (release) by the units that finish the producing data.  Since a
//     unit only waits on units that were dequeued before it and every
//     dequeued unit runs on a resident CTA, the queue cannot deadlock.
//     There is no grid-wide barrier: attention for kv-head g starts when the
//     q/k/v tiles of g are final, the o-projection split of g when g's
//     context is final, each down split when its gate/up tiles are final;
//     only RMSNorm inputs (full residual + sum of squares) are global joins.
//   * The last CTA to leave resets the queue and all counters, so a CUDA
//     graph of the launch replays token after token.
//
// GEMV unit (group, column tile, K-range [r0, r1)) over TILED input-major
// weights: tile t of a group is the contiguous block w[t][i][0..TW), so a
// kept input channel is one contiguous TW*esz-byte row chunk (512 B bf16).
//   1. prologue: h_i = x_i (or RMSNorm: x_i / sqrt(sum(ss)/m + eps) * g_i
//      from fixed-order sum-of-squares partials), keep_lo/hi =
//      !(|h_i| <= t_lo/hi) (closed prune boundary, NaN kept), ordered
//      CTA-local compaction of kept rows with warp ballot/popc;
//   2. stream: warps take kept rows round-robin, UR rows in flight per warp,
//      one 16-byte non-allocating load per lane per row half that is kept,
//      fp32 FMA into per-lane column accumulators;
//   3. fixed-order cross-warp reduction -> TW column partials;
//   4. K-split tiles: partial -> workspace slot, ticket; the last-arriving
//      unit sums the slots in split order (deterministic two-phase
//      reduction) and runs the epilogue (store / residual + sum of squares /
//      SiLU(gate)*up / RoPE + KV-cache write / logits + argmax), then
//      signals its counters.
// No tensor cores: a batch-1 matvec is ~1 flop/byte.
#include "teal_common.cuh"
#include <string.h>

namespace teal {
namespace step {

constexpr int TW = TEAL_STEP_TW;  // columns per tile
constexpr int TH = TW / 2;        // columns per half
constexpr int NT = 256;           // threads per CTA (== TW: one column per thread in epilogues)
constexpr int NW = NT / 32;
constexpr int MAXR = 1024;        // rows per GEMV unit
constexpr int ATT_MAXG = 8;
constexpr int ATT_MAXHD = 128;
constexpr int ATT_MAXCHUNK = 256;
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
        } a;
    } u;
    float red[NW * TW];
    float col[TW];
    float am[ATT_MAXG], al[ATT_MAXG];
    float scr[NW + 1];
    int wcnt[NW];
    float rden;
    int unit, next, last;
    float bv;
    int bi;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void wait_counter(const int* c, int target) {
    if (threadIdx.x == 0) {
        int spins = 0;
        while (ld_acquire(c) < target) {
            if (++spins > 4) __nanosleep(32);
        }
    }
    __syncthreads();
}

// every writer thread fences, then one thread bumps the counters
__device__ __forceinline__ void signal(int* counters, int c0, int c1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && c0 >= 0)
        for (int c = c0; c <= c1; ++c) atomicAdd(counters + c, 1);
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
__device__ __forceinline__ float ld_kv(const void* base, int64_t off) {
    return to_f32<T>(__ldcg(reinterpret_cast<const T*>(base) + off));
}
template <>
__device__ __forceinline__ float ld_kv<uint16_t>(const void* base, int64_t off) {
    const unsigned short v = __ldcg(reinterpret_cast<const unsigned short*>(base) + off);
    return bf16_to_f32(v);
}

// ---- epilogue of one finished column tile (thread c = column c) --------------
__device__ void finalize(const teal_step_plan& P, const teal_step_group& g, int tile, float v, Smem& s) {
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
                if (prev == (unsigned)g.ntiles - 1u) {
                    *P.lm_done = 0u;
                    __threadfence();
                    float gv = -INFINITY;
                    int gi = 0x7fffffff;
                    for (int t = 0; t < g.ntiles; ++t) {
                        const float cv = __ldcg(P.cand_v + t);
                        const int ci = __ldcg(P.cand_i + t);
                        if (cv > gv || (cv == gv && ci < gi)) { gv = cv; gi = ci; }
                    }
                    *P.token_out = gi == 0x7fffffff ? 0 : gi;
                }
            }
            break;
        }
        default:
            break;
    }
    signal(P.counters, tm.sig0, tm.sig1);
}

// ---- GEMV unit ---------------------------------------------------------------
// ESZ = weight element bytes (2: bf16, 4: fp32).  Per lane 8 column
// accumulators: bf16 lane l owns columns [8l, 8l+8) (lanes 16..31 = hi half);
// fp32 lane l owns [4l, 4l+4) (lo) and [128+4l, 128+4l+4) (hi).
template <int ESZ>
__device__ __forceinline__ int acc_col(int lane, int j) {
    if constexpr (ESZ == 2) return lane * 8 + j;
    else return j < 4 ? lane * 4 + j : TH + lane * 4 + (j - 4);
}

template <int ESZ>
__device__ void gemv_unit(const teal_step_plan& P, const teal_step_group& g, const teal_step_unit& U, Smem& s) {
    constexpr int UR = ESZ == 2 ? 8 : 4;      // rows in flight per warp
    constexpr int ROWB = TW * ESZ;            // bytes per row chunk
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const teal_step_tile tm = g.tiles[U.tile];
    const bool rms = g.prologue == TEAL_PRO_RMSNORM;
    if (rms && tid == 0) {
        float a = 0.f;
        for (int p = 0; p < g.nss; ++p) a += __ldcg(g.ss + p);
        s.rden = sqrtf(a / (float)g.m + g.eps);
    }
    __syncthreads();
    const float rden = rms ? s.rden : 1.f;
    const bool two = tm.seg_hi != tm.seg_lo || tm.t_hi != tm.t_lo;

    // 1. threshold + ordered compaction
    int base = 0;
    for (int i0 = U.r0; i0 < U.r1; i0 += NT) {
        const int i = i0 + tid;
        const bool v = i < U.r1;
        float h = 0.f;
        if (v) {
            const float xv = __ldcg(g.x + i);
            h = rms ? (xv / rden) * __ldg(g.gain + i) : xv;
        }
        const bool klo = v && !(fabsf(h) <= tm.t_lo);
        const bool khi = v && !(fabsf(h) <= tm.t_hi);
        const bool k = klo || khi;
        const unsigned bk = __ballot_sync(0xffffffffu, k);
        const bool wv = (i - lane) < U.r1;  // this warp's 32 rows start inside the range
        if (g.dbg_h && U.tile == 0 && v) g.dbg_h[i] = h;
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
            s.u.g.idx[pos] = (i - U.r0) | (klo ? (1 << 30) : 0) | (khi ? (int)(1u << 31) : 0);
            s.u.g.h[pos] = h;
        }
        base += tot;
        __syncthreads();
    }
    const int cnt = base;

    // 2. stream kept row chunks
    const unsigned char* tb =
        reinterpret_cast<const unsigned char*>(g.w) + ((int64_t)U.tile * g.m + U.r0) * ROWB;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int e0 = warp * UR; e0 < cnt; e0 += NW * UR) {
        if constexpr (ESZ == 2) {
            const int sh = lane < 16 ? 30 : 31;
            uint4 d[UR];
            float hh[UR];
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                const int e = e0 + u;
                d[u] = make_uint4(0u, 0u, 0u, 0u);
                hh[u] = 0.f;
                if (e < cnt) {
                    const unsigned pk = (unsigned)s.u.g.idx[e];
                    if ((pk >> sh) & 1u) {
                        hh[u] = s.u.g.h[e];
                        d[u] = ldg128_stream(tb + (int64_t)(pk & 0x3fffffffu) * ROWB + lane * 16);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                const uint32_t w4[4] = {d[u].x, d[u].y, d[u].z, d[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] = fmaf(hh[u], bf16_lo(w4[q]), acc[2 * q]);
                    acc[2 * q + 1] = fmaf(hh[u], bf16_hi(w4[q]), acc[2 * q + 1]);
                }
            }
        } else {
            uint4 d0[UR], d1[UR];
            float h0[UR], h1[UR];
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                const int e = e0 + u;
                d0[u] = d1[u] = make_uint4(0u, 0u, 0u, 0u);
                h0[u] = h1[u] = 0.f;
                if (e < cnt) {
                    const unsigned pk = (unsigned)s.u.g.idx[e];
                    const float hv = s.u.g.h[e];
                    const unsigned char* row = tb + (int64_t)(pk & 0x3fffffffu) * ROWB + lane * 16;
                    if ((pk >> 30) & 1u) { h0[u] = hv; d0[u] = ldg128_stream(row); }
                    if ((pk >> 31) & 1u) { h1[u] = hv; d1[u] = ldg128_stream(row + TH * 4); }
                }
            }
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                acc[0] = fmaf(h0[u], __uint_as_float(d0[u].x), acc[0]);
                acc[1] = fmaf(h0[u], __uint_as_float(d0[u].y), acc[1]);
                acc[2] = fmaf(h0[u], __uint_as_float(d0[u].z), acc[2]);
                acc[3] = fmaf(h0[u], __uint_as_float(d0[u].w), acc[3]);
                acc[4] = fmaf(h1[u], __uint_as_float(d1[u].x), acc[4]);
                acc[5] = fmaf(h1[u], __uint_as_float(d1[u].y), acc[5]);
                acc[6] = fmaf(h1[u], __uint_as_float(d1[u].z), acc[6]);
                acc[7] = fmaf(h1[u], __uint_as_float(d1[u].w), acc[7]);
            }
        }
    }

    // 3. fixed-order cross-warp reduction
#pragma unroll
    for (int j = 0; j < 8; ++j) s.red[warp * TW + acc_col<ESZ>(lane, j)] = acc[j];
    __syncthreads();
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += s.red[w * TW + tid];

    // 4. split-K combine (deterministic, split order) + epilogue
    if (g.nsplit > 1) {
        float* slot = g.partials + ((int64_t)U.tile * g.nsplit + U.split) * TW;
        __stcg(slot + tid, v);
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(g.tickets + U.tile, 1u);
            const int last = prev == (unsigned)g.nsplit - 1u;
            if (last) g.tickets[U.tile] = 0u;
            s.last = last;
        }
        __syncthreads();
        if (!s.last) return;
        __threadfence();
        const float* pb = g.partials + (int64_t)U.tile * g.nsplit * TW + tid;
        v = 0.f;
        int sp = 0;
        for (; sp + 4 <= g.nsplit; sp += 4) {
            const float a0 = __ldcg(pb + (int64_t)sp * TW), a1 = __ldcg(pb + (int64_t)(sp + 1) * TW);
            const float a2 = __ldcg(pb + (int64_t)(sp + 2) * TW), a3 = __ldcg(pb + (int64_t)(sp + 3) * TW);
            v += a0;
            v += a1;
            v += a2;
            v += a3;
        }
        for (; sp < g.nsplit; ++sp) v += __ldcg(pb + (int64_t)sp * TW);
    }
    if (g.col_scale) v *= g.col_scale[(int64_t)U.tile * TW + tid];
    finalize(P, g, U.tile, v, s);
}

// ---- attention unit: (kv head g, position chunk) -------------------------------
template <typename KT>
__device__ void attn_unit_t(const teal_step_plan& P, const teal_step_attn& a, const teal_step_unit& U, Smem& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = U.tile, ch = U.split;
    const int G = a.H / a.KVH, hd = a.hd;
    const int L = __ldcg(P.state + 1);
    const int p0 = ch * a.chunk;
    const int p1 = min(L, p0 + a.chunk);
    const int np = max(0, p1 - p0);
    const int rec = G * hd + 2 * G;
    float* my = a.partials + ((int64_t)g * a.nchunks + ch) * rec;
    const int64_t kvbase = (int64_t)g * a.max_seq * hd;
    if (np > 0) {
        for (int o = tid; o < G * hd; o += NT) s.u.a.q[o] = __ldcg(a.q + (int64_t)g * G * hd + o);
        __syncthreads();
        const float den = sqrtf((float)hd);
        for (int p = warp; p < np; p += NW) {
            const int64_t krow = kvbase + (int64_t)(p0 + p) * hd;
            float dot[ATT_MAXG];
#pragma unroll
            for (int h = 0; h < ATT_MAXG; ++h) dot[h] = 0.f;
            for (int d = lane; d < hd; d += 32) {
                const float kv = ld_kv<KT>(a.k_cache, krow + d);
#pragma unroll
                for (int h = 0; h < ATT_MAXG; ++h)
                    if (h < G) dot[h] = fmaf(s.u.a.q[h * hd + d], kv, dot[h]);
            }
#pragma unroll
            for (int h = 0; h < ATT_MAXG; ++h) {
                if (h < G) {
                    const float sv = warp_sum(dot[h]);
                    if (lane == 0) s.u.a.sc[h * ATT_MAXCHUNK + p] = sv / den;
                }
            }
        }
        __syncthreads();
        if (warp < G) {
            float mx = -INFINITY;
            for (int p = lane; p < np; p += 32) mx = fmaxf(mx, s.u.a.sc[warp * ATT_MAXCHUNK + p]);
            mx = warp_max(mx);
            float l = 0.f;
            for (int p = lane; p < np; p += 32) {
                const float e = expf(s.u.a.sc[warp * ATT_MAXCHUNK + p] - mx);
                s.u.a.sc[warp * ATT_MAXCHUNK + p] = e;
                l += e;
            }
            l = warp_sum(l);
            if (lane == 0) { s.am[warp] = mx; s.al[warp] = l; }
        }
        __syncthreads();
        // context partial: thread -> (d, head set); positions ascending
        const int hsets = NT / hd > 0 ? NT / hd : 1;
        const int d = tid % hd, hs = tid / hd;
        if (hs < hsets && d < hd) {
            float accv[ATT_MAXG];
#pragma unroll
            for (int h = 0; h < ATT_MAXG; ++h) accv[h] = 0.f;
            for (int p = 0; p < np; ++p) {
                const float vv = ld_kv<KT>(a.v_cache, kvbase + (int64_t)(p0 + p) * hd + d);
#pragma unroll
                for (int h = 0; h < ATT_MAXG; ++h)
                    if (h % hsets == hs && h < G) accv[h] = fmaf(s.u.a.sc[h * ATT_MAXCHUNK + p], vv, accv[h]);
            }
#pragma unroll
            for (int h = 0; h < ATT_MAXG; ++h)
                if (h % hsets == hs && h < G) __stcg(my + h * hd + d, accv[h]);
        }
        if (tid < G) {
            __stcg(my + G * hd + tid, s.am[tid]);
            __stcg(my + G * hd + G + tid, s.al[tid]);
        }
    } else if (tid < G) {
        __stcg(my + G * hd + tid, -INFINITY);
        __stcg(my + G * hd + G + tid, 0.f);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(a.tickets + g, 1u);
        const int last = prev == (unsigned)a.nchunks - 1u;
        if (last) a.tickets[g] = 0u;
        s.last = last;
    }
    __syncthreads();
    if (!s.last) return;
    __threadfence();
    const float* rb = a.partials + (int64_t)g * a.nchunks * rec;
    for (int o = tid; o < G * hd; o += NT) {
        const int h = o / hd;
        float M = -INFINITY;
        for (int c = 0; c < a.nchunks; ++c) {
            const float* r = rb + (int64_t)c * rec;
            if (__ldcg(r + G * hd + G + h) > 0.f) M = fmaxf(M, __ldcg(r + G * hd + h));
        }
        float num = 0.f, dd = 0.f;
        for (int c = 0; c < a.nchunks; ++c) {
            const float* r = rb + (int64_t)c * rec;
            const float ls = __ldcg(r + G * hd + G + h);
            if (ls > 0.f) {
                const float sc = expf(__ldcg(r + G * hd + h) - M);
                num = fmaf(__ldcg(r + o), sc, num);
                dd = fmaf(ls, sc, dd);
            }
        }
        a.ctx[(int64_t)g * G * hd + o] = num / dd;
    }
    signal(P.counters, a.sig_base + g, a.sig_base + g);
}

// ---- residual load: x = emb[token] (or x_in); ss partials; {pos, len} ---------
__device__ void load_unit(const teal_step_plan& P, Smem& s) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        const int len = P.state[1];
        P.state[0] = len;
        P.state[1] = len + 1;
    }
    const int tok = P.emb ? __ldcg(P.token) : 0;
    for (int t = 0; t < P.d / TW; ++t) {
        const int64_t c = (int64_t)t * TW + tid;
        float xv;
        if (P.emb) {
            const int64_t off = (int64_t)tok * P.d + c;
            xv = P.emb_dtype == TEAL_BF16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(P.emb)[off])
                                          : reinterpret_cast<const float*>(P.emb)[off];
        } else {
            xv = __ldcg(P.x_in + c);
        }
        P.x[c] = xv;
        const float ss = block_sum_nt(xv * xv, s);
        if (tid == 0) P.ss[t] = ss;
    }
    signal(P.counters, 0, 0);
}

template <int ESZ>
__global__ void __launch_bounds__(NT, 3) step_kernel(const __grid_constant__ teal_step_plan P) {
    __shared__ Smem s;
    const int tid = threadIdx.x;
    if (tid == 0) s.next = (int)atomicAdd(P.ctrl, 1u);
    for (;;) {
        __syncthreads();
        const int u = s.next;
        if (u >= P.nunits) break;
        __syncthreads();
        if (tid == 0) s.next = (int)atomicAdd(P.ctrl, 1u);  // prefetch the next index
        const teal_step_unit U = P.units[u];
        if (U.dep >= 0) wait_counter(P.counters + U.dep, U.target);
        if (U.kind == TEAL_UNIT_GEMV) {
            gemv_unit<ESZ>(P, P.groups[U.group], U, s);
        } else if (U.kind == TEAL_UNIT_ATTN) {
            const teal_step_attn& a = P.attns[U.group];
            if (a.kv_dtype == TEAL_BF16) attn_unit_t<uint16_t>(P, a, U, s);
            else attn_unit_t<float>(P, a, U, s);
        } else {
            load_unit(P, s);
        }
    }
    if (tid == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(P.ctrl + 1, 1u);
        if (prev == gridDim.x - 1u) {
            for (int i = 0; i < P.ncounters; ++i) P.counters[i] = 0;
            P.ctrl[0] = 0u;
            P.ctrl[1] = 0u;
            __threadfence();
        }
    }
}

template <int ESZ>
static int occupancy() {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, step_kernel<ESZ>, NT, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return b;
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
    TEAL_REQUIRE(p && p->groups && p->units && p->counters && p->ctrl && p->x && p->ss && p->state,
                 "teal_step_launch: null plan field");
    TEAL_REQUIRE(p->nunits >= 1 && p->ncounters >= 1, "teal_step_launch: empty plan");
    TEAL_REQUIRE(p->d >= TW && p->d % TW == 0, "teal_step_launch: d must be a multiple of %d", TW);
    TEAL_REQUIRE(p->w_dtype == TEAL_BF16 || p->w_dtype == TEAL_F32, "teal_step_launch: weights must be bf16 or fp32");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per = teal_step_ctas_per_sm(p->w_dtype);
    TEAL_REQUIRE(per >= 1, "teal_step_launch: kernel cannot be resident");
    int ctas = per * sms;
    if (p->ctas > 0 && p->ctas < ctas) ctas = p->ctas;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p->w_dtype == TEAL_BF16) cudaLaunchKernelEx(&cfg, step_kernel<2>, *p);
    else cudaLaunchKernelEx(&cfg, step_kernel<4>, *p);
    return check_launch("teal_step_launch");
}

}  // extern "C"
