// Decode-step helpers around the sparse GEMVs (sm_100a):
//   teal_decode_attention — one query row of model._causal_attention
//                           (pkg/src/actsparse/model.py:135-150) over a KV cache,
//                           GQA-capable, split over positions with a
//                           deterministic ticketed combine;
//   teal_load_residual    — residual-stream load (embedding row or a given
//                           hidden row) + per-tile sum of squares for the
//                           next RMSNorm prologue (model.py:126-128);
//   teal_argmax           — greedy next token from the LM-head logits.
#include "teal_common.cuh"

namespace teal {

constexpr int ATT_MAX_G = 8;       // q heads per kv head
constexpr int ATT_MAX_HD = 256;
constexpr int ATT_MAX_CHUNK = 512;  // positions per CTA

template <typename KT>
__global__ void __launch_bounds__(kThreads) attention_kernel(const float* __restrict__ q, const KT* __restrict__ kc,
                                                             const KT* __restrict__ vc, int H, int KVH, int hd,
                                                             int64_t max_seq, const int* __restrict__ len_ptr,
                                                             int chunk, float* __restrict__ ctx,
                                                             float* __restrict__ ws, uint32_t* __restrict__ tickets,
                                                             int64_t kv_bstride) {
    __shared__ float s_q[ATT_MAX_G * ATT_MAX_HD];
    __shared__ float s_sc[ATT_MAX_G * ATT_MAX_CHUNK];
    __shared__ float s_m[ATT_MAX_G], s_l[ATT_MAX_G];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kvh = blockIdx.x, sp = blockIdx.y, nsplit = gridDim.y;
    const int G = H / KVH;
    // batch (blockIdx.z): sequence b's q / ctx rows, its cache slice and its
    // split-combine records and tickets
    {
        const int b = blockIdx.z;
        q += (int64_t)b * H * hd;
        ctx += (int64_t)b * H * hd;
        kc += (int64_t)b * kv_bstride;
        vc += (int64_t)b * kv_bstride;
        if (ws) ws += (int64_t)b * KVH * nsplit * (G * hd + 2 * G);
        if (tickets) tickets += (int64_t)b * KVH;
    }
    const int L = *len_ptr;
    const int p0 = sp * chunk;
    const int p1 = min(L, p0 + chunk);
    const int np = max(0, p1 - p0);
    const KT* kb = kc + (int64_t)kvh * max_seq * hd;
    const KT* vb = vc + (int64_t)kvh * max_seq * hd;
    const float inv_den = sqrtf((float)hd);

    for (int o = tid; o < G * hd; o += kThreads) s_q[o] = q[(int64_t)kvh * G * hd + o];
    __syncthreads();

    // scores: one warp per position, lanes strided over head_dim
    for (int p = warp; p < np; p += kWarps) {
        const KT* krow = kb + (int64_t)(p0 + p) * hd;
        float dot[ATT_MAX_G];
#pragma unroll
        for (int g = 0; g < ATT_MAX_G; ++g) dot[g] = 0.f;
        for (int d = lane; d < hd; d += 32) {
            const float kv = to_f32<KT>(krow[d]);
#pragma unroll
            for (int g = 0; g < ATT_MAX_G; ++g)
                if (g < G) dot[g] = fmaf(s_q[g * hd + d], kv, dot[g]);
        }
#pragma unroll
        for (int g = 0; g < ATT_MAX_G; ++g) {
            if (g < G) {
                const float s = warp_sum(dot[g]);
                if (lane == 0) s_sc[g * chunk + p] = s / inv_den;
            }
        }
    }
    __syncthreads();
    // local softmax statistics per head (one warp per head)
    if (warp < G) {
        float mx = -INFINITY;
        for (int p = lane; p < np; p += 32) mx = fmaxf(mx, s_sc[warp * chunk + p]);
        mx = warp_max(mx);
        float l = 0.f;
        for (int p = lane; p < np; p += 32) {
            const float e = expf(s_sc[warp * chunk + p] - mx);
            s_sc[warp * chunk + p] = e;
            l += e;
        }
        l = warp_sum(l);
        if (lane == 0) { s_m[warp] = mx; s_l[warp] = l; }
    }
    __syncthreads();
    // partial context: thread per (head, dim), positions in ascending order
    float accs[(ATT_MAX_G * ATT_MAX_HD) / kThreads];
    int nacc = 0;
    for (int o = tid; o < G * hd; o += kThreads, ++nacc) {
        const int g = o / hd, d = o - g * hd;
        float a = 0.f;
        for (int p = 0; p < np; ++p) a = fmaf(s_sc[g * chunk + p], to_f32<KT>(vb[(int64_t)(p0 + p) * hd + d]), a);
        accs[nacc] = a;
    }
    if (nsplit == 1) {
        nacc = 0;
        for (int o = tid; o < G * hd; o += kThreads, ++nacc) {
            const int g = o / hd;
            ctx[(int64_t)kvh * G * hd + o] = accs[nacc] / s_l[g];
        }
        return;
    }
    // split combine: ws[(kvh*nsplit + sp)] = {o[G*hd], m[G], l[G]}
    const int rec = G * hd + 2 * G;
    float* my = ws + ((int64_t)kvh * nsplit + sp) * rec;
    nacc = 0;
    for (int o = tid; o < G * hd; o += kThreads, ++nacc) __stcg(my + o, accs[nacc]);
    if (tid < G) { __stcg(my + G * hd + tid, s_m[tid]); __stcg(my + G * hd + G + tid, s_l[tid]); }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&tickets[kvh], 1u);
        s_last = (prev == (unsigned)nsplit - 1u);
        if (s_last) tickets[kvh] = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* base = ws + (int64_t)kvh * nsplit * rec;
    for (int o = tid; o < G * hd; o += kThreads) {
        const int g = o / hd;
        float M = -INFINITY;
        for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(base + (int64_t)s * rec + G * hd + g));
        float num = 0.f, den = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float* r = base + (int64_t)s * rec;
            const float ls = __ldcg(r + G * hd + G + g);
            if (ls > 0.f) {
                const float sc = expf(__ldcg(r + G * hd + g) - M);
                num = fmaf(__ldcg(r + o), sc, num);
                den = fmaf(ls, sc, den);
            }
        }
        ctx[(int64_t)kvh * G * hd + o] = num / den;
    }
}

template <typename ST>
__global__ void __launch_bounds__(kThreads) load_residual_kernel(const ST* __restrict__ src, const int* __restrict__ token,
                                                                 int64_t d, float* __restrict__ x,
                                                                 float* __restrict__ ss_out, int tile, int* step_state) {
    __shared__ float s_scr[kWarps + 1];
    if (step_state && blockIdx.x == 0 && threadIdx.x == 0) {  // {pos, len}: this step writes position len_prev
        const int len = step_state[1];
        step_state[0] = len;
        step_state[1] = len + 1;
    }
    const ST* row = token ? src + (int64_t)(*token) * d : src;
    const int64_t c0 = (int64_t)blockIdx.x * tile;
    const int64_t c1 = min64(d, c0 + tile);
    float sq = 0.f;
    for (int64_t c = c0 + threadIdx.x; c < c1; c += kThreads) {
        const float v = to_f32<ST>(row[c]);
        x[c] = v;
        sq += v * v;
    }
    const float s = block_sum(sq, s_scr);
    if (threadIdx.x == 0 && ss_out) ss_out[blockIdx.x] = s;
}

// x += delta (fp32); ss_out[t] = sum of x^2 over columns [t*tile, (t+1)*tile).
__global__ void __launch_bounds__(kThreads) residual_add_kernel(float* __restrict__ x, const float* __restrict__ delta,
                                                                int64_t d, float* __restrict__ ss_out, int tile) {
    __shared__ float s_scr[kWarps + 1];
    const int64_t c0 = (int64_t)blockIdx.x * tile;
    const int64_t c1 = min64(d, c0 + tile);
    float sq = 0.f;
    for (int64_t c = c0 + threadIdx.x; c < c1; c += kThreads) {
        const float v = x[c] + delta[c];
        x[c] = v;
        sq += v * v;
    }
    const float s = block_sum(sq, s_scr);
    if (threadIdx.x == 0 && ss_out) ss_out[blockIdx.x] = s;
}

__device__ __forceinline__ void argmax_merge(float& bv, long long& bi, float v, long long i) {
    if (v != v) return;  // NaN ignored
    if (bi < 0 || v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__global__ void __launch_bounds__(kThreads) argmax_kernel(const float* __restrict__ logits, int64_t n, int* __restrict__ out,
                                                          float* __restrict__ ws, uint32_t* __restrict__ tickets) {
    __shared__ float s_v[kThreads];
    __shared__ long long s_i[kThreads];
    __shared__ int s_last;
    float bv = -INFINITY;
    long long bi = -1;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
        argmax_merge(bv, bi, logits[i], i);
    s_v[threadIdx.x] = bv;
    s_i[threadIdx.x] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = -INFINITY;
        long long ix = -1;
        for (int t = 0; t < kThreads; ++t)
            if (s_i[t] >= 0) argmax_merge(v, ix, s_v[t], s_i[t]);
        __stcg(ws + 2 * blockIdx.x, v);
        __stcg(reinterpret_cast<int*>(ws) + 2 * blockIdx.x + 1, (int)ix);
        __threadfence();
        const unsigned prev = atomicAdd(tickets, 1u);
        s_last = (prev == gridDim.x - 1u);
        if (s_last) {
            tickets[0] = 0u;
            __threadfence();
            float gv = -INFINITY;
            long long gi = -1;
            for (unsigned b = 0; b < gridDim.x; ++b) {
                const int ib = __ldcg(reinterpret_cast<const int*>(ws) + 2 * b + 1);
                if (ib >= 0) argmax_merge(gv, gi, __ldcg(ws + 2 * b), ib);
            }
            *out = (int)(gi < 0 ? 0 : gi);
        }
    }
}

}  // namespace teal

using namespace teal;

static int launch_attention(const float* q, const void* k_cache, const void* v_cache, int kv_dtype, int H, int KVH,
                            int hd, int64_t max_seq, const int* len, int chunk, int nsplit, int B, int64_t kv_bstride,
                            float* ctx, float* ws, uint32_t* tickets, cudaStream_t stream, const char* what) {
    dim3 grid(KVH, nsplit, B);
    if (kv_dtype == TEAL_F32)
        attention_kernel<float><<<grid, kThreads, 0, stream>>>(q, (const float*)k_cache, (const float*)v_cache, H, KVH, hd,
                                                               max_seq, len, chunk, ctx, ws, tickets, kv_bstride);
    else if (kv_dtype == TEAL_BF16)
        attention_kernel<uint16_t><<<grid, kThreads, 0, stream>>>(q, (const uint16_t*)k_cache, (const uint16_t*)v_cache, H,
                                                                  KVH, hd, max_seq, len, chunk, ctx, ws, tickets, kv_bstride);
    else
        TEAL_REQUIRE(false, "%s: unsupported kv dtype %d", what, kv_dtype);
    return check_launch(what);
}

extern "C" {

int teal_decode_attention(const float* q, const void* k_cache, const void* v_cache, int kv_dtype, int H, int KVH, int hd,
                          int64_t max_seq, const int* len, int max_len, float* ctx, float* ws, uint32_t* tickets,
                          int nsplit, cudaStream_t stream) {
    TEAL_REQUIRE(q && k_cache && v_cache && len && ctx, "teal_decode_attention: null pointer");
    TEAL_REQUIRE(H >= 1 && KVH >= 1 && H % KVH == 0 && H / KVH <= ATT_MAX_G,
                 "teal_decode_attention: need KVH | H and H/KVH <= %d (H=%d KVH=%d)", ATT_MAX_G, H, KVH);
    TEAL_REQUIRE(hd >= 1 && hd <= ATT_MAX_HD, "teal_decode_attention: head_dim must be in [1, %d]", ATT_MAX_HD);
    TEAL_REQUIRE(max_len >= 1 && max_len <= max_seq, "teal_decode_attention: bad max_len %d", max_len);
    TEAL_REQUIRE(nsplit >= 1, "teal_decode_attention: nsplit must be >= 1");
    const int chunk = (max_len + nsplit - 1) / nsplit;
    TEAL_REQUIRE(chunk <= ATT_MAX_CHUNK, "teal_decode_attention: %d positions per split exceeds %d; raise nsplit",
                 chunk, ATT_MAX_CHUNK);
    TEAL_REQUIRE(nsplit == 1 || (ws && tickets), "teal_decode_attention: nsplit > 1 needs ws and tickets");
    return launch_attention(q, k_cache, v_cache, kv_dtype, H, KVH, hd, max_seq, len, chunk, nsplit, 1, 0, ctx, ws,
                            tickets, stream, "teal_decode_attention");
}

int teal_batch_attention(const float* q, const void* k_cache, const void* v_cache, int kv_dtype, int B, int H, int KVH,
                         int hd, int64_t max_seq, const int* len, int max_len, float* ctx, float* ws,
                         uint32_t* tickets, int nsplit, cudaStream_t stream) {
    TEAL_REQUIRE(q && k_cache && v_cache && len && ctx, "teal_batch_attention: null pointer");
    TEAL_REQUIRE(B >= 1 && B <= 65535, "teal_batch_attention: bad batch %d", B);
    TEAL_REQUIRE(H >= 1 && KVH >= 1 && H % KVH == 0 && H / KVH <= ATT_MAX_G,
                 "teal_batch_attention: need KVH | H and H/KVH <= %d (H=%d KVH=%d)", ATT_MAX_G, H, KVH);
    TEAL_REQUIRE(hd >= 1 && hd <= ATT_MAX_HD, "teal_batch_attention: head_dim must be in [1, %d]", ATT_MAX_HD);
    TEAL_REQUIRE(max_len >= 1 && max_len <= max_seq, "teal_batch_attention: bad max_len %d", max_len);
    TEAL_REQUIRE(nsplit >= 1, "teal_batch_attention: nsplit must be >= 1");
    const int chunk = (max_len + nsplit - 1) / nsplit;
    TEAL_REQUIRE(chunk <= ATT_MAX_CHUNK, "teal_batch_attention: %d positions per split exceeds %d; raise nsplit",
                 chunk, ATT_MAX_CHUNK);
    TEAL_REQUIRE(nsplit == 1 || (ws && tickets), "teal_batch_attention: nsplit > 1 needs ws and tickets");
    return launch_attention(q, k_cache, v_cache, kv_dtype, H, KVH, hd, max_seq, len, chunk, nsplit, B,
                            (int64_t)KVH * max_seq * hd, ctx, ws, tickets, stream, "teal_batch_attention");
}

int teal_load_residual(const void* src, int src_dtype, const int* token, int64_t d, float* x, float* ss_out, int tile,
                       int* step_state, cudaStream_t stream) {
    TEAL_REQUIRE(src && x && d >= 1 && tile >= 1, "teal_load_residual: bad arguments");
    const int grid = (int)((d + tile - 1) / tile);
    if (src_dtype == TEAL_F32)
        load_residual_kernel<float><<<grid, kThreads, 0, stream>>>((const float*)src, token, d, x, ss_out, tile, step_state);
    else if (src_dtype == TEAL_BF16)
        load_residual_kernel<uint16_t><<<grid, kThreads, 0, stream>>>((const uint16_t*)src, token, d, x, ss_out, tile, step_state);
    else
        TEAL_REQUIRE(false, "teal_load_residual: unsupported dtype %d", src_dtype);
    return check_launch("teal_load_residual");
}

int teal_residual_add(float* x, const float* delta, int64_t d, float* ss_out, int tile, cudaStream_t stream) {
    TEAL_REQUIRE(x && delta && d >= 1 && tile >= 1, "teal_residual_add: bad arguments");
    const int grid = (int)((d + tile - 1) / tile);
    residual_add_kernel<<<grid, kThreads, 0, stream>>>(x, delta, d, ss_out, tile);
    return check_launch("teal_residual_add");
}

int teal_argmax(const float* logits, int64_t n, int* out_token, float* ws, uint32_t* tickets, cudaStream_t stream) {
    TEAL_REQUIRE(logits && out_token && ws && tickets && n >= 1, "teal_argmax: bad arguments");
    int64_t g = (n + kThreads * 8 - 1) / (kThreads * 8);
    if (g > 256) g = 256;
    argmax_kernel<<<(int)g, kThreads, 0, stream>>>(logits, n, out_token, ws, tickets);
    return check_launch("teal_argmax");
}

}  // extern "C"
