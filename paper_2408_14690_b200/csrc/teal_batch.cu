// Small-batch decode helpers (BASELINE config 5: B = 1..16 sequences decoded
// in lockstep, one shared sparsity mask per projection, sparsifier.py:136-155).
// The projections run in teal_gemv_batched (each kept weight row read once for
// all B rows); these kernels are the elementwise / per-sequence steps around
// them, each one launch for the whole batch:
//   teal_batch_embed       x[b] = emb[token[b]]                       (model input)
//   teal_batch_rmsnorm     x[b] += delta[b] (optional); h[b] = RMSNorm(x[b])
//                          (model.py:126-128, residuals model.py:184/198)
//   teal_batch_rope_cache  RoPE of q[b] / k[b] (in place), k[b] / v[b] appended
//                          to sequence b's KV cache at this step's position
//   teal_batch_silu_mul    inter[b] = SiLU(gate[b]) * up[b]           (model.py:190-193)
//   teal_batch_argmax      token[b] = argmax logits[b] (lowest index on ties,
//                          NaN ignored)
// Batched attention over the B caches is teal_batch_attention (teal_decode.cu).
#include "teal_common.cuh"

namespace teal {
namespace batch {

template <typename ST>
__global__ void __launch_bounds__(kThreads) embed_kernel(const ST* __restrict__ emb, const int* __restrict__ tokens,
                                                         int64_t d, float* __restrict__ x, int* state) {
    const int b = blockIdx.y;
    if (state && blockIdx.x == 0 && b == 0 && threadIdx.x == 0) {  // {pos, len}: this step writes position len
        const int len = state[1];
        state[0] = len;
        state[1] = len + 1;
    }
    const ST* row = emb + (int64_t)tokens[b] * d;
    for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < d; c += (int64_t)gridDim.x * kThreads)
        x[(int64_t)b * d + c] = to_f32<ST>(row[c]);
}

// one CTA per row: x (+= delta), sum of squares in a fixed order (per-thread
// partials over its float4 slots, then block_sum), h = x / sqrt(mean + eps) * g.
// Every load of the row is issued before any is consumed (d <= 8192: at most
// 8 float4 per thread), so the row costs one memory round trip, not d/256.
constexpr int RMS_V4 = 8;
__global__ void __launch_bounds__(kThreads) rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ delta,
                                                           const float* __restrict__ gain, float eps, int64_t d,
                                                           float* __restrict__ h) {
    __shared__ float s_scr[kWarps + 1];
    const int b = blockIdx.x, tid = threadIdx.x;
    float4* xr = reinterpret_cast<float4*>(x + (int64_t)b * d);
    const float4* dr = delta ? reinterpret_cast<const float4*>(delta + (int64_t)b * d) : nullptr;
    const float4* gr = reinterpret_cast<const float4*>(gain);
    float4* hr = reinterpret_cast<float4*>(h + (int64_t)b * d);
    const int n4 = (int)(d >> 2);
    float4 v[RMS_V4], dv[RMS_V4], gv[RMS_V4];
#pragma unroll
    for (int q = 0; q < RMS_V4; ++q) {  // straight-line: slots past n4 read slot 0 (unused)
        const int i = tid + q * kThreads;
        const int ic = i < n4 ? i : 0;
        v[q] = xr[ic];
        dv[q] = dr ? dr[ic] : make_float4(0.f, 0.f, 0.f, 0.f);
        gv[q] = gr[ic];
    }
    float sq = 0.f;
#pragma unroll
    for (int q = 0; q < RMS_V4; ++q) {
        const int i = tid + q * kThreads;
        if (i < n4) {
            if (dr) {
                v[q].x += dv[q].x; v[q].y += dv[q].y; v[q].z += dv[q].z; v[q].w += dv[q].w;
                xr[i] = v[q];
            }
            sq = fmaf(v[q].x, v[q].x, sq);
            sq = fmaf(v[q].y, v[q].y, sq);
            sq = fmaf(v[q].z, v[q].z, sq);
            sq = fmaf(v[q].w, v[q].w, sq);
        }
    }
    const float den = sqrtf(block_sum(sq, s_scr) / (float)d + eps);
#pragma unroll
    for (int q = 0; q < RMS_V4; ++q) {
        const int i = tid + q * kThreads;
        if (i < n4)
            hr[i] = make_float4((v[q].x / den) * gv[q].x, (v[q].y / den) * gv[q].y, (v[q].z / den) * gv[q].z,
                                (v[q].w / den) * gv[q].w);
    }
}

// grid (heads q + kv, B); thread = dimension pair (d, d + hd/2)
template <typename KT>
__global__ void __launch_bounds__(kThreads) rope_cache_kernel(float* __restrict__ q, float* __restrict__ k,
                                                              const float* __restrict__ v, KT* __restrict__ kc,
                                                              KT* __restrict__ vc, const float* __restrict__ cosv,
                                                              const float* __restrict__ sinv, const int* __restrict__ state,
                                                              int H, int KVH, int hd, int64_t max_seq) {
    const int head = blockIdx.x, b = blockIdx.y, half = hd >> 1;
    const int pos = state[0];
    if (pos < 0 || pos >= max_seq) asm volatile("trap;");  // past the cache: fail loudly
    for (int dd = threadIdx.x; dd < half; dd += kThreads) {
        const float cs = cosv ? cosv[(int64_t)pos * half + dd] : 1.f;
        const float sn = sinv ? sinv[(int64_t)pos * half + dd] : 0.f;
        if (head < H) {
            float* r = q + ((int64_t)b * H + head) * hd;
            const float x0 = r[dd], x1 = r[dd + half];
            r[dd] = fmaf(-x1, sn, x0 * cs);
            r[dd + half] = fmaf(x0, sn, x1 * cs);
        } else {
            const int kh = head - H;
            float* r = k + ((int64_t)b * KVH + kh) * hd;
            const float x0 = r[dd], x1 = r[dd + half];
            const float k0 = fmaf(-x1, sn, x0 * cs), k1 = fmaf(x0, sn, x1 * cs);
            const float* vr = v + ((int64_t)b * KVH + kh) * hd;
            const int64_t off = (((int64_t)b * KVH + kh) * max_seq + pos) * hd;
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

__global__ void __launch_bounds__(kThreads) silu_mul_kernel(const float* __restrict__ gate, const float* __restrict__ up,
                                                            int64_t n, float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        const float z = gate[i];
        out[i] = z / (1.0f + expf(-z)) * up[i];
    }
}

// one CTA per row: largest value, lowest index on ties, NaN ignored
__global__ void __launch_bounds__(kThreads) argmax_rows_kernel(const float* __restrict__ logits, int64_t n,
                                                               int* __restrict__ out) {
    __shared__ float s_v[kWarps];
    __shared__ int s_i[kWarps];
    const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* r = logits + (int64_t)b * n;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) {
        const float v = r[i];
        if (v == v && (v > bv || (v == bv && (int)i < bi))) { bv = v; bi = (int)i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { s_v[warp] = bv; s_i[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; ++w)
            if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi)) { bv = s_v[w]; bi = s_i[w]; }
        out[b] = bi == 0x7fffffff ? 0 : bi;
    }
}

}  // namespace batch
}  // namespace teal

using namespace teal;
using namespace teal::batch;

extern "C" {

int teal_batch_embed(const void* emb, int emb_dtype, const int* tokens, int B, int64_t d, float* x, int* state,
                     cudaStream_t stream) {
    TEAL_REQUIRE(emb && tokens && x && B >= 1 && B <= 65535 && d >= 1, "teal_batch_embed: bad arguments");
    const dim3 grid((unsigned)((d + kThreads - 1) / kThreads), B);
    if (emb_dtype == TEAL_BF16)
        embed_kernel<uint16_t><<<grid, kThreads, 0, stream>>>((const uint16_t*)emb, tokens, d, x, state);
    else if (emb_dtype == TEAL_F32)
        embed_kernel<float><<<grid, kThreads, 0, stream>>>((const float*)emb, tokens, d, x, state);
    else
        TEAL_REQUIRE(false, "teal_batch_embed: unsupported dtype %d", emb_dtype);
    return check_launch("teal_batch_embed");
}

int teal_batch_rmsnorm(float* x, const float* delta, const float* gain, float eps, int B, int64_t d, float* h,
                       cudaStream_t stream) {
    TEAL_REQUIRE(x && gain && h && B >= 1 && d >= 4 && d % 4 == 0 && d <= 4LL * RMS_V4 * kThreads,
                 "teal_batch_rmsnorm: need 4 | d <= %d", 4 * RMS_V4 * kThreads);
    TEAL_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(h) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(gain) & 15) == 0 && (reinterpret_cast<uintptr_t>(delta) & 15) == 0,
                 "teal_batch_rmsnorm: 16-byte aligned rows");
    rmsnorm_kernel<<<B, kThreads, 0, stream>>>(x, delta, gain, eps, d, h);
    return check_launch("teal_batch_rmsnorm");
}

int teal_batch_rope_cache(float* q, float* k, const float* v, void* k_cache, void* v_cache, int kv_dtype,
                          const float* rope_cos, const float* rope_sin, const int* state, int B, int H, int KVH,
                          int hd, int64_t max_seq, cudaStream_t stream) {
    TEAL_REQUIRE(q && k && v && k_cache && v_cache && state && B >= 1 && H >= 1 && KVH >= 1 && hd >= 2 && hd % 2 == 0,
                 "teal_batch_rope_cache: bad arguments");
    TEAL_REQUIRE((rope_cos == nullptr) == (rope_sin == nullptr), "teal_batch_rope_cache: cos and sin go together");
    const dim3 grid(H + KVH, B);
    if (kv_dtype == TEAL_BF16)
        rope_cache_kernel<uint16_t><<<grid, kThreads, 0, stream>>>(q, k, v, (uint16_t*)k_cache, (uint16_t*)v_cache,
                                                                   rope_cos, rope_sin, state, H, KVH, hd, max_seq);
    else if (kv_dtype == TEAL_F32)
        rope_cache_kernel<float><<<grid, kThreads, 0, stream>>>(q, k, v, (float*)k_cache, (float*)v_cache, rope_cos,
                                                                rope_sin, state, H, KVH, hd, max_seq);
    else
        TEAL_REQUIRE(false, "teal_batch_rope_cache: unsupported kv dtype %d", kv_dtype);
    return check_launch("teal_batch_rope_cache");
}

int teal_batch_silu_mul(const float* gate, const float* up, int64_t n, float* out, cudaStream_t stream) {
    TEAL_REQUIRE(gate && up && out && n >= 1, "teal_batch_silu_mul: bad arguments");
    int64_t g = (n + kThreads - 1) / kThreads;
    if (g > 148 * 8) g = 148 * 8;
    silu_mul_kernel<<<(int)g, kThreads, 0, stream>>>(gate, up, n, out);
    return check_launch("teal_batch_silu_mul");
}

int teal_batch_argmax(const float* logits, int B, int64_t n, int* tokens, cudaStream_t stream) {
    TEAL_REQUIRE(logits && tokens && B >= 1 && n >= 1 && n < 0x7fffffff, "teal_batch_argmax: bad arguments");
    argmax_rows_kernel<<<B, kThreads, 0, stream>>>(logits, n, tokens);
    return check_launch("teal_batch_argmax");
}

// ---- stream ordering for concurrent projections (same runtime as the launches) ----
int teal_stream_create(cudaStream_t* s) {
    TEAL_REQUIRE(s, "teal_stream_create: null pointer");
    if (cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) != cudaSuccess) return check_launch("teal_stream_create");
    return TEAL_OK;
}
int teal_stream_destroy(cudaStream_t s) {
    cudaStreamDestroy(s);
    return check_launch("teal_stream_destroy");
}
int teal_event_create(cudaEvent_t* e) {
    TEAL_REQUIRE(e, "teal_event_create: null pointer");
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return check_launch("teal_event_create");
    return TEAL_OK;
}
int teal_event_destroy(cudaEvent_t e) {
    cudaEventDestroy(e);
    return check_launch("teal_event_destroy");
}
int teal_stream_order(cudaStream_t waiter, cudaStream_t signaler, cudaEvent_t e) {
    TEAL_REQUIRE(e, "teal_stream_order: null event");
    if (cudaEventRecord(e, signaler) != cudaSuccess || cudaStreamWaitEvent(waiter, e, 0) != cudaSuccess)
        return check_launch("teal_stream_order");
    return TEAL_OK;
}

}  // extern "C"
