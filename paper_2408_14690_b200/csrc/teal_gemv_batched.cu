// Batched (B <= 16) shared-mask sparse GEMV over bf16 / int8 / int4 weight
// rows (sm_100a) — BASELINE config 5 (small-batch decode with weight-quantized
// rows).
//
// Semantics = the reference's batched sparsification followed by the dense
// product (pkg/src/actsparse/sparsifier.py:136-155 `sparsify_batched`, then
// tensor.py:130-140 `matmul_dense` per row):
//   column i of X [B][m] is pruned in every row iff mean_b |X[b,i]| <= t
//   (fp32 sum in ascending b, then the fp64 quotient rounded to fp32, exactly
//   as teal_threshold_batched), and Y[b] = sum over kept i of X[b,i] * W[i,:].
// Each kept input channel's weight row is read ONCE for all B batch rows.
//
// Weights (input-major, row i = n outputs, row stride ldw elements):
//   bf16 ; int8 with a per-output-column fp32 scale (W = q * s[j]) ;
//   int4 two's-complement nibbles, two per byte (low nibble = even column),
//   with an fp32 scale per (group of `group` input rows, column):
//   W[i,j] = q * s[i / group][j].
//
// Decomposition as teal_fused_gemv: the flattened (column tile, 32-row group)
// space is cut into equal contiguous CTA ranges; a lane owns CPL consecutive
// columns of a TC = 32*CPL column tile and all B batch rows (fp32
// accumulators acc[B][CPL]); warps take kept rows round-robin with U rows in
// flight; warps are reduced in fixed order, split tiles by the last-arriving
// CTA in ascending-CTA order (deterministic).  The FMA kernel (CUDA cores)
// serves B < 4; bf16 / int8 / int4 (group % 128 == 0) rows at B >= 4 (where
// the FMA loop is issue-bound, 2*B flops per weight element) run the
// mma.sync variant below.  At B = 1 the fused single-row kernels are the fast path.
#include "teal_common.cuh"
#include <string.h>

namespace teal {
namespace batched {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int CHUNK = 256;   // rows compacted per round
constexpr int BMAX = 16;

// bytes of CPL consecutive elements of a row
template <int WT, int CPL> struct RowLoad;
template <int CPL> struct RowLoad<TEAL_BF16, CPL> { static constexpr int BYTES = 2 * CPL; };
template <int CPL> struct RowLoad<TEAL_I8, CPL> { static constexpr int BYTES = CPL; };
template <int CPL> struct RowLoad<TEAL_I4, CPL> { static constexpr int BYTES = CPL / 2; };

template <int BYTES>
__device__ __forceinline__ uint4 ld_row(const void* p) {
    uint4 r = make_uint4(0u, 0u, 0u, 0u);
    if constexpr (BYTES == 16) {
        r = ldg128_stream(p);
    } else if constexpr (BYTES == 8) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        r.x = v.x;
        r.y = v.y;
    } else if constexpr (BYTES == 4) {
        r.x = __ldg(reinterpret_cast<const unsigned int*>(p));
    } else {
        r.x = __ldg(reinterpret_cast<const unsigned short*>(p));
    }
    return r;
}

// dequantise CPL packed elements (without scale)
template <int WT, int CPL>
__device__ __forceinline__ void unpack(const uint4 d, float* w) {
    const uint32_t u[4] = {d.x, d.y, d.z, d.w};
    if constexpr (WT == TEAL_BF16) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) w[k] = (k & 1) ? bf16_hi(u[k >> 1]) : bf16_lo(u[k >> 1]);
    } else if constexpr (WT == TEAL_I8) {
        // magic-number conversion (no quarter-rate I2F): b ^ 0x80 = b + 128 in
        // the mantissa of 2^23 (PRMT), minus 2^23 + 128 (FADD)
#pragma unroll
        for (int k = 0; k < CPL; ++k)
            w[k] = __uint_as_float(__byte_perm(u[k >> 2] ^ 0x80808080u, 0x4B000000u, 0x7540u | (k & 3))) - 8388736.0f;
    } else {
        // nibble n ^ 8 = n + 8 in the mantissa of 2^23, minus 2^23 + 8
#pragma unroll
        for (int k = 0; k < CPL; ++k)
            w[k] = __uint_as_float((((u[k >> 3] ^ 0x88888888u) >> (4 * (k & 7))) & 0xfu) | 0x4B000000u) - 8388616.0f;
    }
}

struct KP {
    teal_gemv_batched_args a;
    int gpt;        // 32-row groups per tile
    int ntiles;
    int64_t F;
    int G;
    int maxc;       // partial slots per tile
};

__host__ __device__ __forceinline__ int owner_of(int64_t g, int64_t F, int G) { return (int)(((g + 1) * G - 1) / F); }


// Last arriver's split-K combine of one tile: out[q] = sum over contributors
// k = 0..nc-1 (ascending, from 0.f) of base[k * SLOT + q], q < nout (a
// multiple of 4).  Each thread owns QPT float4 outputs and, per round, has
// 4 contributors x QPT float4 loads in flight (clamped indices, masked adds):
// ceil(nc / 4) L2 round trips instead of one per (output, 16 contributors).
template <int SLOT>
__device__ __forceinline__ void combine_tile(const float* base, int nc, int nout, float* out) {
    constexpr int QPT = (SLOT / 4 + NT - 1) / NT;
    const int tid = threadIdx.x, nq4 = nout >> 2;
    const float4* b4 = reinterpret_cast<const float4*>(base);
    float4 v[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < nc; k0 += 4) {
        float4 pv[4][QPT];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int j = 0; j < QPT; ++j) {
                const int k = min(k0 + kk, nc - 1), q4 = min(tid + j * NT, nq4 - 1);
                pv[kk][j] = __ldcg(b4 + (int64_t)k * (SLOT / 4) + q4);
            }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            if (k0 + kk < nc)
#pragma unroll
                for (int j = 0; j < QPT; ++j) {
                    v[j].x += pv[kk][j].x;
                    v[j].y += pv[kk][j].y;
                    v[j].z += pv[kk][j].z;
                    v[j].w += pv[kk][j].w;
                }
    }
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int q4 = tid + j * NT;
        if (q4 < nq4) reinterpret_cast<float4*>(out)[q4] = v[j];
    }
}

template <int WT, int BM, int CPL>
__global__ void __launch_bounds__(NT, 2) gemv_batched_kernel(const __grid_constant__ KP P) {
    constexpr int TC = 32 * CPL;
    constexpr int LB = RowLoad<WT, CPL>::BYTES;
    constexpr int U = 4;
    __shared__ int s_idx[CHUNK];
    __shared__ __align__(16) float s_x[CHUNK * BM];
    __shared__ __align__(16) float s_red[BM * TC];
    __shared__ int s_wcnt[NW];
    __shared__ int s_last;
    const teal_gemv_batched_args& A = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t g0 = (int64_t)c * P.F / P.G, g1 = (int64_t)(c + 1) * P.F / P.G;
    const int B = A.B;
    unsigned kcount = 0;
    for (int64_t gs = g0; gs < g1;) {
        const int tile = (int)(gs / P.gpt);
        const int64_t ge = min64(g1, (int64_t)(tile + 1) * P.gpt);
        const int r0 = (int)(gs - (int64_t)tile * P.gpt) * 32;
        const int r1 = (int)min64(A.m, (ge - (int64_t)tile * P.gpt) * 32);
        gs = ge;
        const int64_t col0 = (int64_t)tile * TC + lane * CPL;
        float acc[BM][CPL];
#pragma unroll
        for (int b = 0; b < BM; ++b)
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[b][k] = 0.f;
        int sgrp = -1;
        float sc[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) sc[k] = 1.f;
        for (int ra = r0; ra < r1; ra += CHUNK) {
            const int rb = min(r1, ra + CHUNK);
            // shared mask of this chunk (ordered compaction)
            const int i = ra + tid;
            const bool v = i < rb;
            float xs[BM];
            float s = 0.f;
            // straight-line loads (clamped indices, masked after): a load
            // inside a per-element branch is waited for at the branch's
            // reconvergence point, i.e. B round trips instead of one
#pragma unroll
            for (int b = 0; b < BM; ++b) xs[b] = __ldg(A.x + (int64_t)(b < B ? b : 0) * A.m + (v ? i : ra));
#pragma unroll
            for (int b = 0; b < BM; ++b) {
                xs[b] = (v && b < B) ? xs[b] : 0.f;
                if (b < B) s = __fadd_rn(s, fabsf(xs[b]));
            }
            const float mean = (float)__ddiv_rn((double)s, (double)B);
            const bool keep = v && !(mean <= A.t32);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (tile == 0) {
                if (A.mask && v) A.mask[i] = keep ? 0 : 1;
                kcount += (lane == 0) ? __popc(bal) : 0u;
            }
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            int off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int cw = s_wcnt[w];
                off += (w < warp) ? cw : 0;
                tot += cw;
            }
            if (keep) {
                const int pos = off + __popc(bal & ((1u << lane) - 1u));
                s_idx[pos] = i;
#pragma unroll
                for (int b = 0; b < BM; ++b) s_x[pos * BM + b] = xs[b];
            }
            __syncthreads();
            // stream the kept rows: warp w takes entries w*U.., the next U
            // rows' loads issued before the current U are consumed (double
            // buffer: 2U row chunks in flight per warp)
            auto fetch = [&](int e0, uint4 (&d)[U], int (&rows)[U]) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + u;
                    rows[u] = e < tot ? s_idx[e] : -1;
                    d[u] = make_uint4(0u, 0u, 0u, 0u);
                    if (rows[u] >= 0 && col0 < A.n) {
                        const int64_t el = (int64_t)rows[u] * A.ldw + col0;
                        const unsigned char* p = reinterpret_cast<const unsigned char*>(A.w) +
                                                 (WT == TEAL_BF16 ? el * 2 : (WT == TEAL_I8 ? el : el / 2));
                        d[u] = ld_row<LB>(p);
                    }
                }
            };
            auto consume = [&](int e0, const uint4 (&d)[U], const int (&rows)[U]) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (rows[u] < 0) continue;
                    float w[CPL];
                    unpack<WT, CPL>(d[u], w);
                    if constexpr (WT == TEAL_I4) {
                        const int grp = rows[u] / A.group;
                        if (grp != sgrp) {  // rows ascend: the group scale changes rarely
                            sgrp = grp;
#pragma unroll
                            for (int k = 0; k < CPL; ++k)
                                sc[k] = (col0 + k < A.n) ? __ldg(A.scale + (int64_t)grp * A.n + col0 + k) : 0.f;
                        }
#pragma unroll
                        for (int k = 0; k < CPL; ++k) w[k] *= sc[k];
                    }
                    const float* xr = s_x + (e0 + u) * BM;
                    float xv[BM];
                    if constexpr (BM % 4 == 0) {  // 16-byte shared loads of the batch's x values
#pragma unroll
                        for (int b = 0; b < BM; b += 4) {
                            const float4 q = *reinterpret_cast<const float4*>(xr + b);
                            xv[b] = q.x; xv[b + 1] = q.y; xv[b + 2] = q.z; xv[b + 3] = q.w;
                        }
                    } else {
#pragma unroll
                        for (int b = 0; b < BM; ++b) xv[b] = xr[b];
                    }
#pragma unroll
                    for (int b = 0; b < BM; ++b) {
#pragma unroll
                        for (int k = 0; k < CPL; ++k) acc[b][k] = fmaf(xv[b], w[k], acc[b][k]);
                    }
                }
            };
            {
                uint4 da[U], db[U];
                int ra_[U], rb_[U];
                int e0 = warp * U;
                if (e0 < tot) {
                    fetch(e0, da, ra_);
                    for (;;) {
                        const int en = e0 + NW * U;
                        if (en < tot) fetch(en, db, rb_);
                        consume(e0, da, ra_);
                        if (en >= tot) break;
                        e0 = en;
                        if (e0 + NW * U < tot) fetch(e0 + NW * U, da, ra_);
                        consume(e0, db, rb_);
                        if (e0 + NW * U >= tot) break;
                        e0 += NW * U;
                    }
                }
            }
            __syncthreads();
        }
        // fixed-order warp reduction: warp 0 writes, warps 1..7 add in turn
        for (int w = 0; w < NW; ++w) {
            if (warp == w) {
#pragma unroll
                for (int b = 0; b < BM; ++b)
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        float* r = s_red + b * TC + lane * CPL + k;
                        *r = (w == 0) ? acc[b][k] : *r + acc[b][k];
                    }
            }
            __syncthreads();
        }
        // split-K combine (ascending CTA order) + store
        const int cf = owner_of((int64_t)tile * P.gpt, P.F, P.G);
        const int cl = owner_of((int64_t)(tile + 1) * P.gpt - 1, P.F, P.G);
        bool fin = true;
        if (cl > cf) {
            float* slot = A.ws + ((int64_t)tile * P.maxc + (c - cf)) * (BM * TC);
            for (int q = tid; q < BM * TC; q += NT) __stcg(slot + q, s_red[q]);
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                const unsigned prev = atomicAdd(A.tickets + tile, 1u);
                s_last = prev == (unsigned)(cl - cf);
                if (s_last) {
                    A.tickets[tile] = 0u;
                    __threadfence();
                }
            }
            __syncthreads();
            fin = s_last != 0;
            if (fin) {
                // every contributor's partial of this thread's outputs in flight
                // together (16 at a time, clamped indices), then summed in
                // ascending contributor order
                combine_tile<BM * TC>(A.ws + (int64_t)tile * P.maxc * (BM * TC), cl - cf + 1, B * TC, s_red);
                __syncthreads();
            }
        }
        if (fin) {
            for (int q = tid; q < B * TC; q += NT) {
                const int b = q / TC, cc = q - b * TC;
                const int64_t col = (int64_t)tile * TC + cc;
                if (col < A.n) {
                    float v = s_red[b * TC + cc];
                    if constexpr (WT == TEAL_I8) v *= A.scale[col];
                    A.y[(int64_t)b * A.n + col] = v;
                }
            }
        }
        __syncthreads();
    }
    if (A.kept && lane == 0 && kcount) atomicAdd(A.kept, (unsigned long long)kcount);
}


// ---- bf16 rows, B >= 4: tensor-core (mma.sync m16n8k16) variant ----------
// Same decomposition, mask and deterministic split-K combine as above; the
// per-row FMA loop (FMA-issue bound at B >= 4: 2*B flops per weight element)
// is replaced by warp MMAs over the chunk's gathered rows:
//   D[b][col] += sum_k X[b][k] * W[idx_k][col]   (M = batch padded to 16,
//   N = 32 columns per warp, K = kept rows of the chunk in steps of 16).
// Kept rows' TCM-column slices are gathered into shared memory with
// cp.async (16 B per request, zero-filled past n), row stride padded by 16 B
// so ldmatrix(.trans) phases are bank-conflict free.  X is fp32: it is split
// exactly into three bf16 terms x = h1 + h2 + h3 (h_i = RN(x - h_1 - ...)),
// each product with a bf16 weight is exact in fp32, so the result matches an
// fp32 GEMV to accumulation rounding (the rel 1e-5 bar of the FMA kernel).
constexpr int MC = 128;               // candidate rows per chunk
constexpr int TCM = 256;              // columns per tile: 8 warps x 32
constexpr int WSTR = TCM * 2 + 16;    // staged row stride (bytes)
constexpr int XSTR = MC * 2 + 16;     // staged x row stride (bytes): [b][k]
constexpr int NSPLIT = 3;
constexpr size_t kMmaW = (size_t)MC * WSTR;
constexpr size_t kMmaX = (size_t)NSPLIT * 16 * XSTR;
constexpr size_t kMmaSmem = kMmaW + kMmaX + MC * 4 + NW * 4 + 16;
static_assert((size_t)16 * TCM * 4 <= kMmaW, "combine buffer aliases the row stage");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int WT>
__global__ void __launch_bounds__(NT, 2) gemv_batched_mma_kernel(const __grid_constant__ KP P) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* s_w = sm;                                // [MC][WSTR]
    unsigned char* s_xb = sm + kMmaW;                       // [NSPLIT][16][XSTR]
    int* s_idx = reinterpret_cast<int*>(sm + kMmaW + kMmaX);
    int* s_wcnt = s_idx + MC;
    int* s_last = s_wcnt + NW;
    float* s_red = reinterpret_cast<float*>(sm);            // [16][TCM], after the last chunk
    const teal_gemv_batched_args& A = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t g0 = (int64_t)c * P.F / P.G, g1 = (int64_t)(c + 1) * P.F / P.G;
    const int B = A.B;
    const unsigned char* W = reinterpret_cast<const unsigned char*>(A.w);
    // bytes of one row slice; int8 / int4 slices land at the end of the
    // slot (upper half / last quarter) and are widened to bf16 in place
    constexpr int RB = WT == TEAL_I8 ? TCM : (WT == TEAL_I4 ? TCM / 2 : TCM * 2);
    constexpr int SEGS = RB / 16;                      // 16-byte requests per row slice
    constexpr int EPS = TCM / SEGS;                    // elements per request
    constexpr int SOFF = 2 * TCM - RB;
    unsigned kcount = 0;
    const int mi = lane >> 3, mr = lane & 7;  // ldmatrix: matrix / row this lane addresses
    for (int64_t gs = g0; gs < g1;) {
        const int tile = (int)(gs / P.gpt);
        const int64_t ge = min64(g1, (int64_t)(tile + 1) * P.gpt);
        const int r0 = (int)(gs - (int64_t)tile * P.gpt) * 32;
        const int r1 = (int)min64(A.m, (ge - (int64_t)tile * P.gpt) * 32);
        gs = ge;
        const int64_t tcol0 = (int64_t)tile * TCM;
        float acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][q] = 0.f;
        float gtot[4][4];  // int4: scaled sum over the chunks (one row group each)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) gtot[j][q] = 0.f;
        // chunks end at multiples of MC, so with group % MC == 0 a chunk lies
        // inside one int4 scale group
        for (int ra = r0, rb; ra < r1; ra = rb) {
            rb = min(r1, (ra / MC + 1) * MC);
            // shared mask of the chunk (threads 0..MC-1 own one row each)
            const int i = ra + tid;
            const bool v = tid < MC && i < rb;
            float xs[BMAX];
            float sabs = 0.f;
#pragma unroll
            for (int b = 0; b < BMAX; ++b) xs[b] = __ldg(A.x + (int64_t)(b < B ? b : 0) * A.m + (v ? i : ra));
#pragma unroll
            for (int b = 0; b < BMAX; ++b) {
                xs[b] = (v && b < B) ? xs[b] : 0.f;
                if (b < B) sabs = __fadd_rn(sabs, fabsf(xs[b]));
            }
            const float mean = (float)__ddiv_rn((double)sabs, (double)B);
            const bool keep = v && !(mean <= A.t32);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (tile == 0) {
                if (A.mask && v) A.mask[i] = keep ? 0 : 1;
                kcount += (lane == 0) ? __popc(bal) : 0u;
            }
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            int off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int cw = s_wcnt[w];
                off += (w < warp) ? cw : 0;
                tot += cw;
            }
            const int kpad = (tot + 15) & ~15;
            // slot of this thread's row: kept rows first (ascending), then the
            // pad slots [tot, kpad) take zero x and a valid (finite) row
            int slot = -1;
            if (keep) slot = off + __popc(bal & ((1u << lane) - 1u));
            else if (tid >= MC && tid - MC < kpad - tot) slot = tot + (tid - MC);  // row-less threads
            if (slot >= 0) {
                s_idx[slot] = keep ? i : ra;
#pragma unroll
                for (int b = 0; b < 16; ++b) {
                    const float x0 = keep ? xs[b] : 0.f;
                    const uint16_t h1 = f32_to_bf16_rn(x0);
                    const float e1 = x0 - __uint_as_float((uint32_t)h1 << 16);
                    const uint16_t h2 = f32_to_bf16_rn(e1);
                    const float e2 = e1 - __uint_as_float((uint32_t)h2 << 16);
                    const uint16_t h3 = f32_to_bf16_rn(e2);
                    *reinterpret_cast<uint16_t*>(s_xb + (0 * 16 + b) * XSTR + slot * 2) = h1;
                    *reinterpret_cast<uint16_t*>(s_xb + (1 * 16 + b) * XSTR + slot * 2) = h2;
                    *reinterpret_cast<uint16_t*>(s_xb + (2 * 16 + b) * XSTR + slot * 2) = h3;
                }
            }
            __syncthreads();
            if (kpad == 0) continue;  // uniform: nothing kept in this chunk
            // gather the kept rows' tile slices (16 B per request, zero past n)
            for (int q = tid; q < kpad * SEGS; q += NT) {
                const int k = q / SEGS, sg = q % SEGS;
                const int64_t col = tcol0 + sg * EPS;
                const bool inb = col < A.n;
                const unsigned char* src = W + ((int64_t)s_idx[k] * A.ldw + (inb ? col : 0)) * RB / TCM;
                cp_async16(smem_u32(s_w + k * WSTR + SOFF + sg * 16), src, inb ? 16 : 0);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            if constexpr (WT == TEAL_I8) {
                // widen in place, one half-warp per row: every lane loads its
                // 16 int8 from the slot's upper half before any lane stores its
                // 16 bf16 (exact: |q| <= 128) over the row
                const int c = lane & 15;
#pragma unroll 1
                for (int k = warp * 2 + (lane >> 4); k < kpad; k += NW * 2) {
                    const uint4 q = *reinterpret_cast<const uint4*>(s_w + k * WSTR + TCM + c * 16);
                    __syncwarp();
                    const uint32_t u[4] = {q.x, q.y, q.z, q.w};
                    uint32_t o[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int k0 = 2 * e, k1 = 2 * e + 1;
                        const float f0 = __uint_as_float(__byte_perm(u[k0 >> 2] ^ 0x80808080u, 0x4B000000u, 0x7540u | (k0 & 3))) - 8388736.0f;
                        const float f1 = __uint_as_float(__byte_perm(u[k1 >> 2] ^ 0x80808080u, 0x4B000000u, 0x7540u | (k1 & 3))) - 8388736.0f;
                        o[e] = (__float_as_uint(f0) >> 16) | (__float_as_uint(f1) & 0xffff0000u);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(s_w + k * WSTR + c * 32);
                    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
                    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
                    __syncwarp();
                }
                __syncthreads();
            }
            if constexpr (WT == TEAL_I4) {
                // widen in place, one quarter-warp per row (32 nibbles per
                // lane, low nibble = even column; exact in bf16)
                const int c = lane & 7;
#pragma unroll 1
                for (int kb = warp * 4; kb < kpad; kb += NW * 4) {  // kpad % 4 == 0: uniform per warp
                    const int k = kb + (lane >> 3);
                    const uint4 q = *reinterpret_cast<const uint4*>(s_w + k * WSTR + SOFF + c * 16);
                    __syncwarp();
                    const uint32_t u[4] = {q.x ^ 0x88888888u, q.y ^ 0x88888888u, q.z ^ 0x88888888u, q.w ^ 0x88888888u};
                    uint4* dst = reinterpret_cast<uint4*>(s_w + k * WSTR + c * 64);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        uint32_t o[4];
#pragma unroll
                        for (int e2 = 0; e2 < 4; ++e2) {
                            const int e0 = v4 * 8 + e2 * 2, e1 = e0 + 1;
                            const float f0 = __uint_as_float(((u[e0 >> 3] >> (4 * (e0 & 7))) & 0xfu) | 0x4B000000u) - 8388616.0f;
                            const float f1 = __uint_as_float(((u[e1 >> 3] >> (4 * (e1 & 7))) & 0xfu) | 0x4B000000u) - 8388616.0f;
                            o[e2] = (__float_as_uint(f0) >> 16) | (__float_as_uint(f1) & 0xffff0000u);
                        }
                        dst[v4] = make_uint4(o[0], o[1], o[2], o[3]);
                    }
                    __syncwarp();
                }
                __syncthreads();
            }
            float2 gsc[4];  // int4: this chunk's group scales of the thread's 8 columns
            if constexpr (WT == TEAL_I4) {
                const int64_t grow = (int64_t)(ra / A.group) * A.n;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t col = tcol0 + warp * 32 + j * 8 + 2 * (lane & 3);
                    gsc[j] = __ldg(reinterpret_cast<const float2*>(A.scale + grow + (col < A.n ? col : 0)));
                    if (col >= A.n) gsc[j] = make_float2(0.f, 0.f);
                }
            }
            const uint32_t xb = smem_u32(s_xb), wb = smem_u32(s_w);
            const int n0 = warp * 32;
#pragma unroll 1
            for (int k0 = 0; k0 < kpad; k0 += 16) {
                uint32_t bf[2][4];
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
                    ldsm_x4_t(wb + (k0 + mr + 8 * (mi & 1)) * WSTR + (n0 + jj * 16 + 8 * (mi >> 1)) * 2,
                              bf[jj][0], bf[jj][1], bf[jj][2], bf[jj][3]);
#pragma unroll
                for (int sp = 0; sp < NSPLIT; ++sp) {
                    uint32_t af[4];
                    ldsm_x4(xb + (sp * 16 + mr + 8 * (mi & 1)) * XSTR + (k0 + 8 * (mi >> 1)) * 2, af[0], af[1], af[2], af[3]);
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        mma_bf16(acc[2 * jj], af, bf[jj][0], bf[jj][1]);
                        mma_bf16(acc[2 * jj + 1], af, bf[jj][2], bf[jj][3]);
                    }
                }
            }
            if constexpr (WT == TEAL_I4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    gtot[j][0] = fmaf(acc[j][0], gsc[j].x, gtot[j][0]);
                    gtot[j][1] = fmaf(acc[j][1], gsc[j].y, gtot[j][1]);
                    gtot[j][2] = fmaf(acc[j][2], gsc[j].x, gtot[j][2]);
                    gtot[j][3] = fmaf(acc[j][3], gsc[j].y, gtot[j][3]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[j][q] = 0.f;
                }
            }
            __syncthreads();  // the stage is rewritten by the next chunk
        }
        if constexpr (WT == TEAL_I4) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[j][q] = gtot[j][q];
        }
        // warp-owned columns: D fragment -> s_red[b][col] (no cross-warp sum)
        {
            const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int col = warp * 32 + j * 8 + 2 * tq;
                s_red[gq * TCM + col] = acc[j][0];
                s_red[gq * TCM + col + 1] = acc[j][1];
                s_red[(gq + 8) * TCM + col] = acc[j][2];
                s_red[(gq + 8) * TCM + col + 1] = acc[j][3];
            }
        }
        __syncthreads();
        // split-K combine (ascending CTA order) + store, as the FMA kernel
        const int cf = owner_of((int64_t)tile * P.gpt, P.F, P.G);
        const int cl = owner_of((int64_t)(tile + 1) * P.gpt - 1, P.F, P.G);
        bool fin = true;
        if (cl > cf) {
            float* slot = A.ws + ((int64_t)tile * P.maxc + (c - cf)) * (16 * TCM);
            for (int q = tid; q < B * TCM; q += NT) __stcg(slot + q, s_red[q]);
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                const unsigned prev = atomicAdd(A.tickets + tile, 1u);
                *s_last = prev == (unsigned)(cl - cf);
                if (*s_last) {
                    A.tickets[tile] = 0u;
                    __threadfence();
                }
            }
            __syncthreads();
            fin = *s_last != 0;
            if (fin) {
                combine_tile<16 * TCM>(A.ws + (int64_t)tile * P.maxc * (16 * TCM), cl - cf + 1, B * TCM, s_red);
                __syncthreads();
            }
        }
        if (fin) {
            for (int q = tid; q < B * TCM; q += NT) {
                const int b = q / TCM, cc = q - b * TCM;
                const int64_t col = tcol0 + cc;
                if (col < A.n) {
                    float v = s_red[b * TCM + cc];
                    if constexpr (WT == TEAL_I8) v *= A.scale[col];
                    A.y[(int64_t)b * A.n + col] = v;
                }
            }
        }
        __syncthreads();
    }
    if (A.kept && lane == 0 && kcount) atomicAdd(A.kept, (unsigned long long)kcount);
}

// Narrow outputs at B > 8 (few 256-column tiles: many split-K contributors
// per tile and a long combine) stay on the FMA kernel's 128-column tiles.
#ifndef TEAL_MMA_MIN_B
#define TEAL_MMA_MIN_B 4
#endif
static bool use_mma(const teal_gemv_batched_args* a) {
    const bool fmt = (a->w_dtype == TEAL_BF16 && a->n % 8 == 0 && a->ldw % 8 == 0) ||
                     (a->w_dtype == TEAL_I8 && a->n % 16 == 0 && a->ldw % 16 == 0) ||
                     (a->w_dtype == TEAL_I4 && a->n % 32 == 0 && a->ldw % 32 == 0 && a->group % MC == 0);
    return fmt && a->B >= TEAL_MMA_MIN_B;
}

static int cpl_of(int B) { return B > 8 ? 4 : 8; }
static int tc_of(int B) { return 32 * cpl_of(B); }
static int bm_of(int B) { return B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : 16; }

static int plan(const teal_gemv_batched_args* a, KP* P) {
    const int tc = use_mma(a) ? TCM : tc_of(a->B);
    P->ntiles = (int)((a->n + tc - 1) / tc);
    P->gpt = (int)((a->m + 31) / 32);
    P->F = (int64_t)P->ntiles * P->gpt;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    cudaGetLastError();
    // MMA variant over few column tiles (k/v: n = 1024, 4 tiles): one CTA per
    // SM halves the split-K contributors per tile (k/v B = 16 19 -> 16 us);
    // wider outputs keep two resident CTAs to overlap their chunk chains
    const bool narrow = use_mma(a) && P->ntiles <= 4;
    int64_t G = a->ctas > 0 ? a->ctas : (narrow ? 1LL : 2LL) * sms;
    if (G > P->F) G = P->F;
    P->G = (int)G;
    int maxc = 1;
    for (int t = 0; t < P->ntiles; ++t) {
        const int cf = owner_of((int64_t)t * P->gpt, P->F, P->G);
        const int cl = owner_of((int64_t)(t + 1) * P->gpt - 1, P->F, P->G);
        if (cl - cf + 1 > maxc) maxc = cl - cf + 1;
    }
    P->maxc = maxc;
    return TEAL_OK;
}

static int validate(const teal_gemv_batched_args* a) {
    TEAL_REQUIRE(a, "teal_gemv_batched: null args");
    TEAL_REQUIRE(a->B >= 1 && a->B <= BMAX, "teal_gemv_batched: batch must be in [1, %d], got %d", BMAX, a->B);
    TEAL_REQUIRE(a->m >= 1 && a->n >= 1 && a->ldw >= a->n, "teal_gemv_batched: bad shape m=%lld n=%lld ldw=%lld",
                 (long long)a->m, (long long)a->n, (long long)a->ldw);
    TEAL_REQUIRE(a->w_dtype == TEAL_BF16 || a->w_dtype == TEAL_I8 || a->w_dtype == TEAL_I4,
                 "teal_gemv_batched: weights must be bf16, int8 or int4 (got %d)", a->w_dtype);
    TEAL_REQUIRE(a->w_dtype == TEAL_BF16 || a->scale, "teal_gemv_batched: quantised weights need scales");
    TEAL_REQUIRE(a->w_dtype != TEAL_I4 || a->group >= 1, "teal_gemv_batched: int4 needs a row-group size");
    const int cpl = cpl_of(a->B);
    TEAL_REQUIRE(a->n % cpl == 0 && a->ldw % cpl == 0,
                 "teal_gemv_batched: n and ldw must be multiples of %d for batch %d", cpl, a->B);
    TEAL_REQUIRE(a->t32 == a->t32 && (!(a->t32 < 0.f) || a->t32 == -INFINITY),
                 "teal_gemv_batched: threshold must be >= 0 (or -inf for dense), got %g", (double)a->t32);
    TEAL_REQUIRE(a->x && a->y && a->w, "teal_gemv_batched: null pointer");
    return TEAL_OK;
}

template <int WT>
static int launch_mma(const KP& P, cudaStream_t st) {
    // the dynamic shared memory opt-in is per device
    static unsigned long long done = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("teal_gemv_batched (device)");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit)) {
        if (cudaFuncSetAttribute(gemv_batched_mma_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMmaSmem) != cudaSuccess)
            return check_launch("teal_gemv_batched (smem attribute)");
        __atomic_fetch_or(&done, bit, __ATOMIC_RELEASE);
    }
    gemv_batched_mma_kernel<WT><<<P.G, NT, kMmaSmem, st>>>(P);
    return check_launch("teal_gemv_batched");
}

template <int WT>
static int launch_w(const KP& P, cudaStream_t st) {
    const int bm = bm_of(P.a.B);
    dim3 grid(P.G), block(NT);
#define TEAL_BL(BMv, CPLv) gemv_batched_kernel<WT, BMv, CPLv><<<grid, block, 0, st>>>(P)
    switch (bm) {
        case 1: TEAL_BL(1, 8); break;
        case 2: TEAL_BL(2, 8); break;
        case 4: TEAL_BL(4, 8); break;
        case 8: TEAL_BL(8, 8); break;
        default: TEAL_BL(16, 4); break;
    }
#undef TEAL_BL
    return check_launch("teal_gemv_batched");
}

}  // namespace batched
}  // namespace teal

using namespace teal;
using namespace teal::batched;

namespace teal {
bool gemv_tc_eligible(const teal_gemv_batched_args* a);  // teal_gemv_tc.cu: bf16, 4 <= B <= 16
int64_t gemv_tc_workspace_floats(const teal_gemv_batched_args* a, int64_t* tickets);
int gemv_tc_launch(const teal_gemv_batched_args* a, cudaStream_t stream);
}  // namespace teal

extern "C" {

int teal_gemv_batched_workspace(const teal_gemv_batched_args* a, int* ctas, int64_t* ws_floats, int64_t* tickets) {
    int st = validate(a);
    if (st) return st;
    if (gemv_tc_eligible(a)) {  // tcgen05 path: compaction + tensor-core contraction
        if (ctas) *ctas = 0;
        const int64_t f = gemv_tc_workspace_floats(a, tickets);
        if (ws_floats) *ws_floats = f;
        return TEAL_OK;
    }
    KP P;
    memset(&P, 0, sizeof(P));
    plan(a, &P);
    if (ctas) *ctas = P.G;
    if (ws_floats) *ws_floats = use_mma(a) ? (int64_t)P.ntiles * P.maxc * 16 * TCM
                                           : (int64_t)P.ntiles * P.maxc * bm_of(a->B) * tc_of(a->B);
    if (tickets) *tickets = P.ntiles;
    return TEAL_OK;
}

int teal_gemv_batched(const teal_gemv_batched_args* a, cudaStream_t stream) {
    int st = validate(a);
    if (st) return st;
    if (gemv_tc_eligible(a)) return gemv_tc_launch(a, stream);
    KP P;
    memset(&P, 0, sizeof(P));
    P.a = *a;
    plan(a, &P);
    TEAL_REQUIRE(P.G == 1 || P.maxc == 1 || (a->ws && a->tickets), "teal_gemv_batched: ws and tickets are required");
    if (use_mma(a))
        return a->w_dtype == TEAL_I8 ? launch_mma<TEAL_I8>(P, stream)
             : a->w_dtype == TEAL_I4 ? launch_mma<TEAL_I4>(P, stream) : launch_mma<TEAL_BF16>(P, stream);
    if (a->w_dtype == TEAL_BF16) return launch_w<TEAL_BF16>(P, stream);
    if (a->w_dtype == TEAL_I8) return launch_w<TEAL_I8>(P, stream);
    return launch_w<TEAL_I4>(P, stream);
}

}  // extern "C"
