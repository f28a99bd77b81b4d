// Fused threshold + sparse GEMV over input-channel-major weights (sm_100a).
//
// Replaces the reference's column-skipping numba GEMV
// (pkg/src/actsparse/kernel.py:30-44, `_skip_gemv`) and the seven masked
// `gated(name, a) @ W.T` products of model._forward (model.py:166-198).
//
// Work decomposition (one launch = one fused projection group):
//   grid.x = column tiles over all segments (TILE output columns each),
//   grid.y = K chunks (kchunk input channels each, multiple of 32).
// Each CTA
//   1. forms h over its K chunk (plain x, or RMSNorm of the residual stream
//      from fixed-order sum-of-squares partials),
//   2. compares keep_i = !(|h_i| <= t) and compacts the surviving channel
//      indices CTA-locally with warp ballot/popc into shared memory (ascending
//      channel order preserved),
//   3. streams only the surviving rows' TILE-column segments with 256-bit
//      non-coherent loads (one row segment per warp instruction), fp32 FMA,
//   4. reduces its 8 warps in fixed order, writes an fp32 partial, and the
//      last-arriving CTA of the tile (ticket counter) sums the ksplit partials
//      in ascending chunk order — a deterministic two-phase reduction — and
//      runs the fused epilogue (store / residual+sumsq / SiLU(gate)*up /
//      RoPE+KV-cache write).
// No tensor cores: a batch-1 matvec is ~1 flop/byte, far below the ridge.
#include "teal_common.cuh"
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

namespace teal {

constexpr int KCH_MAX = 2048;  // max input channels per CTA (smem index list)

struct KParams {
    teal_gemv_args a;
    int tile;           // TILE columns per CTA
    int tile0[4];       // first global tile of each segment (+ sentinel)
    int64_t wscol0[3];  // column offset of each segment inside a ws row
    int64_t ldws;       // ws row length (sum of n)
};

// ---- raw vector fetch / expand ---------------------------------------------
template <typename WT, int VE> struct Raw;
template <> struct Raw<uint16_t, 16> { U8 r; };
template <> struct Raw<float, 8> { U8 r; };
template <> struct Raw<int8_t, 16> { uint4 r; };
template <typename WT> struct Raw<WT, 1> { WT r; };

template <typename WT, int VE>
__device__ __forceinline__ void fetch(Raw<WT, VE>& d, const WT* p) {
    if constexpr (VE == 1) {
        d.r = __ldg(p);
    } else if constexpr (sizeof(WT) == 1) {
        d.r = ldg128_stream(p);
    } else {
        d.r = ldg256_stream(p);
    }
}
template <typename WT, int VE>
__device__ __forceinline__ void zero(Raw<WT, VE>& d) {
    if constexpr (VE == 1) {
        d.r = WT(0);
    } else if constexpr (sizeof(WT) == 1) {
        d.r = make_uint4(0u, 0u, 0u, 0u);
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) d.r.v[k] = 0u;
    }
}
template <typename WT, int VE>
__device__ __forceinline__ void fma_into(float* acc, const Raw<WT, VE>& d, float x) {
    if constexpr (VE == 1) {
        acc[0] = fmaf(x, to_f32<WT>(d.r), acc[0]);
    } else if constexpr (sizeof(WT) == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc[2 * k] = fmaf(x, bf16_lo(d.r.v[k]), acc[2 * k]);
            acc[2 * k + 1] = fmaf(x, bf16_hi(d.r.v[k]), acc[2 * k + 1]);
        }
    } else if constexpr (sizeof(WT) == 4) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fmaf(x, __uint_as_float(d.r.v[k]), acc[k]);
    } else {  // int8 x 16
        const uint32_t w4[4] = {d.r.x, d.r.y, d.r.z, d.r.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t u = w4[k];
#pragma unroll
            for (int b = 0; b < 4; ++b)
                acc[4 * k + b] = fmaf(x, (float)(int8_t)((u >> (8 * b)) & 0xffu), acc[4 * k + b]);
        }
    }
}

__device__ __forceinline__ float silu(float z) { return z / (1.0f + expf(-z)); }

template <typename XT>
__device__ __forceinline__ float load_x(const void* x, int64_t i) {
    return to_f32<XT>(reinterpret_cast<const XT*>(x)[i]);
}

template <typename WT, typename XT, int VE, int NV>
__global__ void __launch_bounds__(kThreads, 2) fused_gemv_kernel(const __grid_constant__ KParams P) {
    constexpr int TILE = 32 * VE * NV;
    constexpr int U = (VE == 1) ? 8 : 4;  // rows in flight per warp
    constexpr int QN = (TILE + kThreads - 1) / kThreads;

    __shared__ int s_idx[KCH_MAX];
    __shared__ float s_val[KCH_MAX];
    __shared__ __align__(32) float s_red[kWarps * TILE];
    __shared__ int s_wcnt[kWarps];
    __shared__ float s_scr[kWarps + 1];
    __shared__ float s_rden;
    __shared__ int s_last;

    const teal_gemv_args& A = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gt = blockIdx.x;
    const int seg = (A.nseg > 1 && gt >= P.tile0[1]) ? ((A.nseg > 2 && gt >= P.tile0[2]) ? 2 : 1) : 0;
    const teal_seg& S = A.seg[seg];
    const int tis = gt - P.tile0[seg];
    const int64_t c0 = (int64_t)tis * TILE;
    const int ncols = (int)min64(TILE, S.n - c0);
    const int ks = blockIdx.y;
    const int64_t k0 = (int64_t)ks * A.kchunk;
    const int64_t k1 = min64(A.m, k0 + A.kchunk);
    const float t32 = S.t32;

    // ---- 1. prologue: h over the K chunk ----------------------------------
    const bool rms = (A.prologue == TEAL_PRO_RMSNORM);
    if (rms) {
        if (tid == 0) {
            float s = 0.f;
            for (int p = 0; p < A.ss_count; ++p) s += A.ss_part[p];
            s_rden = sqrtf(s / (float)A.m + A.eps);
        }
        __syncthreads();
    }
    const float rden = rms ? s_rden : 1.f;

    // ---- 2. threshold + CTA-local compaction (ballot/popc) -----------------
    int base = 0;
    const bool first_tile = (tis == 0);
    for (int64_t cbeg = k0; cbeg < k1; cbeg += kThreads) {
        const int64_t i = cbeg + tid;
        const bool valid = i < k1;
        float h = 0.f;
        if (valid) {
            h = load_x<XT>(A.x, i);
            if (rms) h = h / rden * A.norm_scale[i];
        }
        const bool keep = valid && !(fabsf(h) <= t32);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        if (first_tile) {
            if (S.dbg_bits && lane == 0 && cbeg + warp * 32 < k1) S.dbg_bits[(cbeg + warp * 32) >> 5] = bal;
            if (seg == 0 && A.dbg_h && valid) A.dbg_h[i] = h;
        }
        __syncthreads();
        int off = base, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = s_wcnt[w];
            off += (w < warp) ? c : 0;
            tot += c;
        }
        if (keep) {
            const int pos = off + __popc(bal & ((1u << lane) - 1u));
            s_idx[pos] = (int)(i - k0);
            s_val[pos] = h;
        }
        base += tot;
        __syncthreads();
    }
    const int count = base;
    if (first_tile && tid == 0 && S.kept && count) atomicAdd(S.kept, (unsigned long long)count);

    // ---- 3. stream the surviving rows -------------------------------------
    float acc[NV][VE];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[v][e] = 0.f;

    const WT* wseg = reinterpret_cast<const WT*>(S.w) + c0 + k0 * S.ldw;
    bool colok[NV];
    int coloff[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        coloff[v] = (v * 32 + lane) * VE;
        colok[v] = coloff[v] < ncols;
    }
    for (int r = warp * U; r < count; r += kWarps * U) {
        Raw<WT, VE> raw[U][NV];
        float xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int rr = r + u;
            if (rr < count) {
                const WT* row = wseg + (int64_t)s_idx[rr] * S.ldw;
                xv[u] = s_val[rr];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if (colok[v]) fetch<WT, VE>(raw[u][v], row + coloff[v]);
                    else zero<WT, VE>(raw[u][v]);
                }
            } else {
                xv[u] = 0.f;
#pragma unroll
                for (int v = 0; v < NV; ++v) zero<WT, VE>(raw[u][v]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) fma_into<WT, VE>(acc[v], raw[u][v], xv[u]);
    }

    // ---- 4. fixed-order reduction over warps ------------------------------
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        float* dst = s_red + warp * TILE + coloff[v];
        if constexpr (VE % 4 == 0) {
#pragma unroll
            for (int e = 0; e < VE; e += 4)
                *reinterpret_cast<float4*>(dst + e) = make_float4(acc[v][e], acc[v][e + 1], acc[v][e + 2], acc[v][e + 3]);
        } else {
#pragma unroll
            for (int e = 0; e < VE; ++e) dst[e] = acc[v][e];
        }
    }
    __syncthreads();
    float tot[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int c = tid + q * kThreads;
        float s = 0.f;
        if (c < TILE) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += s_red[w * TILE + c];
        }
        tot[q] = s;
    }

    const int epi = A.epilogue;
    const bool direct = (A.ksplit == 1) && (epi != TEAL_EPI_SILU);
    float tot_up[QN];  // SILU: the paired up-projection totals
    if (!direct) {
        float* wsrow = A.ws + (int64_t)ks * P.ldws + P.wscol0[seg] + c0;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (c < ncols) __stcg(wsrow + c, tot[q]);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int tk = (epi == TEAL_EPI_SILU) ? tis : gt;
            const unsigned expected = (unsigned)A.ksplit * ((epi == TEAL_EPI_SILU) ? 2u : 1u);
            const unsigned prev = atomicAdd(&A.tickets[tk], 1u);
            const int last = (prev == expected - 1u);
            if (last) A.tickets[tk] = 0u;  // self-reset for the next launch
            s_last = last;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        const int sa = (epi == TEAL_EPI_SILU) ? 0 : seg;
        const float* wcol = A.ws + P.wscol0[sa] + c0;
        const float* wcol_up = A.ws + P.wscol0[1] + c0;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            float s = 0.f, su = 0.f;
            if (c < ncols) {
                for (int k = 0; k < A.ksplit; ++k) s += ldcg_f32(wcol + (int64_t)k * P.ldws + c);
                if (epi == TEAL_EPI_SILU)
                    for (int k = 0; k < A.ksplit; ++k) su += ldcg_f32(wcol_up + (int64_t)k * P.ldws + c);
            }
            tot[q] = s;
            tot_up[q] = su;
        }
    }

    // ---- 5. fused epilogue ------------------------------------------------
    if (epi == TEAL_EPI_STORE) {
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (c < ncols) {
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
            if (c < ncols) {
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
            if (c < ncols) {
                float g = tot[q], u = tot_up[q];
                if (A.seg[0].col_scale) g *= A.seg[0].col_scale[c0 + c];
                if (A.seg[1].col_scale) u *= A.seg[1].col_scale[c0 + c];
                A.inter[c0 + c] = silu(g) * u;
            }
        }
    } else {  // TEAL_EPI_QKV: seg 0 = q, 1 = k, 2 = v
        float* s_tile = s_red;  // reuse (all warps are past the reduction)
        __syncthreads();
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (c < TILE) {
                float v = (c < ncols) ? tot[q] : 0.f;
                if (c < ncols && S.col_scale) v *= S.col_scale[c0 + c];
                s_tile[c] = v;
            }
        }
        __syncthreads();
        const int hd = A.head_dim, half = hd >> 1;
        const int pos = *A.pos;
        const bool rope = (A.rope_cos != nullptr) && (seg < 2);
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int c = tid + q * kThreads;
            if (c < ncols) {
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
    }
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

static int elem_bytes(int dt) { return dt == TEAL_F32 ? 4 : dt == TEAL_BF16 ? 2 : 1; }
static int wide_ve(int dt) { return dt == TEAL_F32 ? 8 : 16; }

static bool seg_wide_ok(const teal_gemv_args* a) {
    const int ve = wide_ve(a->w_dtype);
    for (int s = 0; s < a->nseg; ++s) {
        const teal_seg& g = a->seg[s];
        if (g.n % ve) return false;
        if (g.ldw % ve) return false;
        if (reinterpret_cast<uintptr_t>(g.w) % 32) return false;
    }
    return true;
}

static int tile_width(const teal_gemv_args* a) {
    if (a->w_dtype == TEAL_I8) return 32 * 16;  // int8 is wide-only
    if (seg_wide_ok(a)) return 32 * wide_ve(a->w_dtype);
    return 32 * 8;  // scalar path: VE=1, NV=8
}

static int sm_count_cached() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        cudaGetLastError();
    }
    return sms;
}

template <typename WT, typename XT, int VE, int NV>
static void launch(const KParams& P, dim3 grid, cudaStream_t st) {
    fused_gemv_kernel<WT, XT, VE, NV><<<grid, kThreads, 0, st>>>(P);
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

int teal_gemv_plan(int64_t m, int64_t ncols_total, int w_dtype, int nseg, int* ksplit, int* kchunk) {
    TEAL_REQUIRE(m >= 1 && ncols_total >= 1, "teal_gemv_plan: invalid shape m=%lld n=%lld", (long long)m, (long long)ncols_total);
    TEAL_REQUIRE(ksplit && kchunk, "teal_gemv_plan: null output");
    (void)nseg;
    const int tile = (w_dtype == TEAL_F32) ? 256 : 512;
    const int64_t tiles = (ncols_total + tile - 1) / tile;
    int per_sm = 4;
    if (const char* e = getenv("TEAL_CTAS_PER_SM")) per_sm = atoi(e) > 0 ? atoi(e) : 4;
    const int64_t target = (int64_t)sm_count_cached() * per_sm;
    int64_t ks = (target + tiles - 1) / tiles;
    // keep >= ~64 channels per chunk so the prologue amortises
    const int64_t ks_max_amort = (m + 63) / 64;
    if (ks > ks_max_amort) ks = ks_max_amort;
    if (ks < 1) ks = 1;
    int64_t kc = (m + ks - 1) / ks;
    kc = ((kc + 31) / 32) * 32;
    if (kc > KCH_MAX) kc = KCH_MAX;
    ks = (m + kc - 1) / kc;
    *ksplit = (int)ks;
    *kchunk = (int)kc;
    return TEAL_OK;
}

int teal_gemv_tile_width(const teal_gemv_args* a) { return a ? tile_width(a) : -1; }

int teal_gemv_tiles(const teal_gemv_args* a) {
    if (!a) return -1;
    const int tile = tile_width(a);
    int t = 0;
    for (int s = 0; s < a->nseg; ++s) t += (int)((a->seg[s].n + tile - 1) / tile);
    return t;
}

int teal_fused_gemv(const teal_gemv_args* a, cudaStream_t stream) {
    TEAL_REQUIRE(a, "teal_fused_gemv: null args");
    TEAL_REQUIRE(a->nseg >= 1 && a->nseg <= 3, "teal_fused_gemv: nseg must be 1..3, got %d", a->nseg);
    TEAL_REQUIRE(a->m >= 1, "teal_fused_gemv: m must be >= 1");
    TEAL_REQUIRE(a->x, "teal_fused_gemv: null x");
    TEAL_REQUIRE(a->w_dtype == TEAL_F32 || a->w_dtype == TEAL_BF16 || a->w_dtype == TEAL_I8,
                 "teal_fused_gemv: unsupported weight dtype %d", a->w_dtype);
    TEAL_REQUIRE(a->x_dtype == TEAL_F32 || a->x_dtype == TEAL_BF16, "teal_fused_gemv: unsupported x dtype %d", a->x_dtype);
    TEAL_REQUIRE(a->kchunk >= 32 && a->kchunk % 32 == 0 && a->kchunk <= KCH_MAX,
                 "teal_fused_gemv: kchunk must be a multiple of 32 in [32, %d], got %d", KCH_MAX, a->kchunk);
    TEAL_REQUIRE(a->ksplit >= 1 && (int64_t)a->ksplit * a->kchunk >= a->m && (int64_t)(a->ksplit - 1) * a->kchunk < a->m,
                 "teal_fused_gemv: ksplit*kchunk does not tile m (ksplit=%d kchunk=%d m=%lld)", a->ksplit, a->kchunk, (long long)a->m);
    for (int s = 0; s < a->nseg; ++s) {
        const teal_seg& g = a->seg[s];
        TEAL_REQUIRE(g.w && g.n >= 1 && g.ldw >= g.n, "teal_fused_gemv: bad segment %d (n=%lld ldw=%lld)", s, (long long)g.n, (long long)g.ldw);
        TEAL_REQUIRE(g.t32 == g.t32 && (!(g.t32 < 0.f) || g.t32 == -INFINITY), "teal_fused_gemv: threshold must be >= 0 (or -inf for dense), got %g", (double)g.t32);
        TEAL_REQUIRE(a->w_dtype != TEAL_I8 || g.col_scale, "teal_fused_gemv: int8 weights need col_scale");
        if (a->epilogue == TEAL_EPI_STORE) TEAL_REQUIRE(g.y, "teal_fused_gemv: STORE epilogue needs seg[%d].y", s);
    }
    if (a->prologue == TEAL_PRO_RMSNORM) {
        TEAL_REQUIRE(a->x_dtype == TEAL_F32 && a->norm_scale && a->ss_part && a->ss_count >= 1,
                     "teal_fused_gemv: RMSNORM prologue needs fp32 x, norm_scale and ss_part");
    } else {
        TEAL_REQUIRE(a->prologue == TEAL_PRO_PLAIN, "teal_fused_gemv: unknown prologue %d", a->prologue);
    }
    switch (a->epilogue) {
        case TEAL_EPI_STORE: break;
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
    const int tile = tile_width(a);
    P.tile = tile;
    if (a->epilogue == TEAL_EPI_QKV) {
        TEAL_REQUIRE(tile % a->head_dim == 0 && a->seg[0].n % a->head_dim == 0 && a->seg[1].n % a->head_dim == 0,
                     "teal_fused_gemv: QKV epilogue needs head_dim | tile (%d) and head_dim | n", tile);
    }
    int t = 0;
    int64_t col = 0;
    for (int s = 0; s < a->nseg; ++s) {
        P.tile0[s] = t;
        P.wscol0[s] = col;
        t += (int)((a->seg[s].n + tile - 1) / tile);
        col += a->seg[s].n;
    }
    P.tile0[a->nseg] = t;
    for (int s = a->nseg + 1; s < 4; ++s) P.tile0[s] = t;
    P.ldws = col;
    const bool needs_ws = !(a->ksplit == 1 && a->epilogue != TEAL_EPI_SILU);
    if (needs_ws) TEAL_REQUIRE(a->ws && a->tickets, "teal_fused_gemv: split-K needs ws and tickets");
    int grid_x = t;
    if (a->epilogue == TEAL_EPI_SILU) grid_x = t;  // both segments' tiles, paired tickets
    dim3 grid(grid_x, a->ksplit);
    const bool wide = (a->w_dtype == TEAL_I8) || seg_wide_ok(a);
    TEAL_REQUIRE(a->w_dtype != TEAL_I8 || seg_wide_ok(a), "teal_fused_gemv: int8 rows need n%%16==0, ldw%%16==0 and 32B alignment");
    const bool xb = (a->x_dtype == TEAL_BF16);
    if (a->w_dtype == TEAL_BF16) {
        if (wide) { if (xb) launch<uint16_t, uint16_t, 16, 1>(P, grid, stream); else launch<uint16_t, float, 16, 1>(P, grid, stream); }
        else      { if (xb) launch<uint16_t, uint16_t, 1, 8>(P, grid, stream);  else launch<uint16_t, float, 1, 8>(P, grid, stream); }
    } else if (a->w_dtype == TEAL_F32) {
        if (wide) { if (xb) launch<float, uint16_t, 8, 1>(P, grid, stream); else launch<float, float, 8, 1>(P, grid, stream); }
        else      { if (xb) launch<float, uint16_t, 1, 8>(P, grid, stream);  else launch<float, float, 1, 8>(P, grid, stream); }
    } else {
        if (xb) launch<int8_t, uint16_t, 16, 1>(P, grid, stream); else launch<int8_t, float, 16, 1>(P, grid, stream);
    }
    return check_launch("teal_fused_gemv");
}

int teal_sparse_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw,
                     const void* x, int x_dtype, float t32, float* y, const float* col_scale,
                     float* ws, uint32_t* tickets, int ksplit, int kchunk,
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
    a.ksplit = ksplit;
    a.kchunk = kchunk;
    a.ws = ws;
    a.tickets = tickets;
    return teal_fused_gemv(&a, stream);
}

int teal_dense_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw,
                    const void* x, int x_dtype, float* y, const float* col_scale,
                    float* ws, uint32_t* tickets, int ksplit, int kchunk, cudaStream_t stream) {
    return teal_sparse_gemv(w, w_dtype, m, n, ldw, x, x_dtype, -INFINITY, y, col_scale, ws, tickets,
                            ksplit, kchunk, nullptr, stream);
}

}  // extern "C"
