// Thresholding, batched shared-mask thresholding and GPU histogram
// calibration (sm_100a).
//
//   teal_threshold          <- sparsify / realized_sparsity (sparsifier.py:120-133)
//   teal_threshold_batched  <- sparsify_batched (sparsifier.py:136-155)
//   teal_hist_record        <- ActivationHistogram.record (sparsifier.py:68-83)
//   teal_hist_threshold     <- ActivationHistogram.threshold (sparsifier.py:94-117)
#include "teal_common.cuh"

namespace teal {

// keep_i = !(|x_i| <= t32): closed prune boundary, NaN kept, pruned -> +0.0.
template <typename XT>
__global__ void __launch_bounds__(kThreads) threshold_kernel(const XT* __restrict__ x, int64_t m, float t32,
                                                             uint32_t* __restrict__ bits, XT* __restrict__ xs,
                                                             unsigned long long* __restrict__ pruned) {
    const int lane = threadIdx.x & 31;
    unsigned npr = 0;
    for (int64_t b = (int64_t)blockIdx.x * kThreads; b < m; b += (int64_t)gridDim.x * kThreads) {
        const int64_t i = b + threadIdx.x;
        const bool valid = i < m;
        const XT xv = valid ? x[i] : XT(0);
        const float v = to_f32<XT>(xv);
        const bool keep = valid && !(fabsf(v) <= t32);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bits && lane == 0 && (i - lane) < m) bits[(i - lane) >> 5] = bal;
        if (xs && valid) xs[i] = keep ? xv : XT(0);
        npr += (valid && !keep) ? 1u : 0u;
    }
    if (pruned) {
        const unsigned w = __reduce_add_sync(0xffffffffu, npr);
        if (lane == 0 && w) atomicAdd(pruned, (unsigned long long)w);
    }
}

// Column mean of |X| over B rows: fp32 sequential sum in ascending b, then
// divided by B the way numpy's mean does it (fp64 quotient rounded to fp32).
__global__ void __launch_bounds__(kThreads) threshold_batched_kernel(const float* __restrict__ xs, int64_t B, int64_t m,
                                                                     float t32, uint8_t* __restrict__ mask,
                                                                     float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < m; i += (int64_t)gridDim.x * kThreads) {
        float s = 0.f;
        for (int64_t b = 0; b < B; ++b) s = __fadd_rn(s, fabsf(xs[b * m + i]));
        const float mean = (float)__ddiv_rn((double)s, (double)B);
        const bool pr = (mean <= t32);
        if (mask) mask[i] = pr ? 1 : 0;
        if (out)
            for (int64_t b = 0; b < B; ++b) out[b * m + i] = pr ? 0.f : xs[b * m + i];
    }
}

// Histogram of |x| on [0, hi] in fp64: idx = floor(|x| / hi * bins), clipped to
// the last bin, |x| > hi -> overflow.  Shared-memory privatised 32-bit bins,
// flushed with 64-bit global atomics (integer, so order-independent).
// the value binned: fp64 input as is (the reference bins np.asarray(x,
// float64), sparsifier.py:75-80), fp32 / bf16 widened exactly
__device__ __forceinline__ double hist_value(double v) { return v; }
__device__ __forceinline__ double hist_value(float v) { return (double)v; }
__device__ __forceinline__ double hist_value(uint16_t v) { return (double)bf16_to_f32(v); }

template <typename XT>
__global__ void __launch_bounds__(kThreads) hist_kernel(const XT* __restrict__ x, int64_t cnt, double hi, int bins,
                                                        unsigned long long* __restrict__ counts,
                                                        unsigned long long* __restrict__ overflow,
                                                        unsigned int* __restrict__ nan_flag, int use_smem) {
    extern __shared__ unsigned int s_bins[];
    if (use_smem) {
        for (int b = threadIdx.x; b < bins; b += kThreads) s_bins[b] = 0u;
        __syncthreads();
    }
    const double dbins = (double)bins;
    unsigned ov = 0;
    bool nan = false;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * kThreads) {
        const double v = fabs(hist_value(x[i]));
        if (isnan(v)) {
            nan = true;
        } else if (v > hi) {
            ++ov;
        } else {
            long long idx = (long long)floor(__dmul_rn(__ddiv_rn(v, hi), dbins));
            if (idx < 0) idx = 0;
            if (idx > bins - 1) idx = bins - 1;
            if (use_smem) atomicAdd(&s_bins[idx], 1u);
            else atomicAdd(&counts[idx], 1ull);
        }
    }
    if (nan) atomicExch(nan_flag, 1u);
    const unsigned ovw = __reduce_add_sync(0xffffffffu, ov);
    if ((threadIdx.x & 31) == 0 && ovw) atomicAdd(overflow, (unsigned long long)ovw);
    if (use_smem) {
        __syncthreads();
        for (int b = threadIdx.x; b < bins; b += kThreads)
            if (s_bins[b]) atomicAdd(&counts[b], (unsigned long long)s_bins[b]);
    }
}

// One CTA.  cum = cumsum(counts) / total (exact int64 prefix, fp64 division),
// idx = first bin with cum >= p (numpy searchsorted 'left'), then linear
// interpolation inside the bin — identical fp64 operation sequence to
// sparsifier.py:94-117, with no FMA contraction.
__global__ void __launch_bounds__(1024) hist_threshold_kernel(const unsigned long long* __restrict__ counts, int bins,
                                                              const unsigned long long* __restrict__ overflow, double hi,
                                                              const double* __restrict__ p, int np_, double* __restrict__ out) {
    extern __shared__ unsigned long long s_cum[];  // [bins]
    __shared__ unsigned long long s_part[1024];
    __shared__ int s_idx;
    const int T = blockDim.x, tid = threadIdx.x;
    // block prefix sum: each thread owns a contiguous run of bins
    const int per = (bins + T - 1) / T;
    const int b0 = tid * per, b1 = min(bins, b0 + per);
    unsigned long long run = 0;
    for (int b = b0; b < b1; ++b) { run += counts[b]; s_cum[b] = run; }
    s_part[tid] = run;
    __syncthreads();
    if (tid == 0) {
        unsigned long long acc = 0;
        for (int t = 0; t < T; ++t) { const unsigned long long v = s_part[t]; s_part[t] = acc; acc += v; }
    }
    __syncthreads();
    for (int b = b0; b < b1; ++b) s_cum[b] += s_part[tid];
    __syncthreads();
    const unsigned long long total = s_cum[bins - 1] + *overflow;
    const double dtot = (double)total;
    for (int j = 0; j < np_; ++j) {
        const double pj = p[j];
        if (tid == 0) s_idx = bins;
        __syncthreads();
        int my = bins;
        for (int b = b0; b < b1; ++b)
            if (__ddiv_rn((double)s_cum[b], dtot) >= pj) { my = b; break; }
        if (my < bins) atomicMin(&s_idx, my);
        __syncthreads();
        if (tid == 0) {
            double r;
            if (total < 1) r = __longlong_as_double(0x7ff8000000000000ll);  // NaN: empty histogram
            else if (pj == 0.0) r = 0.0;
            else if (pj == 1.0) r = hi;
            else {
                const int idx = s_idx;
                if (idx >= bins) r = hi;
                else {
                    const double prev = idx > 0 ? __ddiv_rn((double)s_cum[idx - 1], dtot) : 0.0;
                    const double cur = __ddiv_rn((double)s_cum[idx], dtot);
                    const double mass = __dsub_rn(cur, prev);
                    const double width = __ddiv_rn(hi, (double)bins);
                    const double left = __dmul_rn((double)idx, width);
                    if (mass <= 0.0) r = left;
                    else r = __dadd_rn(left, __dmul_rn(__ddiv_rn(__dsub_rn(pj, prev), mass), width));
                }
            }
            out[j] = r;
        }
        __syncthreads();
    }
}

static int grid_for(int64_t n, int per_block_elems, int max_blocks) {
    int64_t g = (n + per_block_elems - 1) / per_block_elems;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

}  // namespace teal

using namespace teal;

extern "C" {

int teal_threshold(const void* x, int x_dtype, int64_t m, float t32, uint32_t* keep_bits, void* x_sparse,
                   unsigned long long* pruned, cudaStream_t stream) {
    TEAL_REQUIRE(m >= 0, "teal_threshold: m must be >= 0");
    TEAL_REQUIRE(t32 >= 0.f, "threshold must be non-negative, got %g", (double)t32);
    if (m == 0) return TEAL_OK;
    TEAL_REQUIRE(x, "teal_threshold: null x");
    const int g = grid_for(m, kThreads, 148 * 8);
    if (x_dtype == TEAL_F32)
        threshold_kernel<float><<<g, kThreads, 0, stream>>>((const float*)x, m, t32, keep_bits, (float*)x_sparse, pruned);
    else if (x_dtype == TEAL_BF16)
        threshold_kernel<uint16_t><<<g, kThreads, 0, stream>>>((const uint16_t*)x, m, t32, keep_bits, (uint16_t*)x_sparse, pruned);
    else
        TEAL_REQUIRE(false, "teal_threshold: unsupported dtype %d", x_dtype);
    return check_launch("teal_threshold");
}

int teal_threshold_batched(const float* xs, int64_t B, int64_t m, float t32, uint8_t* mask, float* xs_sparse,
                           cudaStream_t stream) {
    TEAL_REQUIRE(B >= 1 && m >= 1, "expected a [B, m] batch with B >= 1, got [%lld, %lld]", (long long)B, (long long)m);
    TEAL_REQUIRE(t32 >= 0.f, "threshold must be non-negative, got %g", (double)t32);
    TEAL_REQUIRE(xs, "teal_threshold_batched: null xs");
    const int g = grid_for(m, kThreads, 148 * 8);
    threshold_batched_kernel<<<g, kThreads, 0, stream>>>(xs, B, m, t32, mask, xs_sparse);
    return check_launch("teal_threshold_batched");
}

int teal_hist_record(const void* x, int x_dtype, int64_t count, double hi, int bins, unsigned long long* counts,
                     unsigned long long* overflow, unsigned int* nan_flag, cudaStream_t stream) {
    TEAL_REQUIRE(bins >= 1, "bin_count must be >= 1, got %d", bins);
    TEAL_REQUIRE(hi > 0, "histogram upper bound must be positive, got %g", hi);
    TEAL_REQUIRE(count >= 0, "teal_hist_record: negative count");
    if (count == 0) return TEAL_OK;
    TEAL_REQUIRE(x && counts && overflow && nan_flag, "teal_hist_record: null pointer");
    const int use_smem = bins <= 16384;
    const size_t smem = use_smem ? (size_t)bins * 4 : 0;
    if (use_smem && smem > 48 * 1024) {
        cudaFuncSetAttribute(hist_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(hist_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(hist_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const int g = grid_for(count, kThreads * 16, 148 * 4);
    if (x_dtype == TEAL_F32)
        hist_kernel<float><<<g, kThreads, smem, stream>>>((const float*)x, count, hi, bins, counts, overflow, nan_flag, use_smem);
    else if (x_dtype == TEAL_BF16)
        hist_kernel<uint16_t><<<g, kThreads, smem, stream>>>((const uint16_t*)x, count, hi, bins, counts, overflow, nan_flag, use_smem);
    else if (x_dtype == TEAL_F64)
        hist_kernel<double><<<g, kThreads, smem, stream>>>((const double*)x, count, hi, bins, counts, overflow, nan_flag, use_smem);
    else
        TEAL_REQUIRE(false, "teal_hist_record: unsupported dtype %d", x_dtype);
    return check_launch("teal_hist_record");
}

int teal_hist_threshold(const unsigned long long* counts, int bins, const unsigned long long* overflow, double hi,
                        const double* p, int np_, double* t_out, cudaStream_t stream) {
    TEAL_REQUIRE(bins >= 1 && bins <= 16384, "teal_hist_threshold: bins must be in [1, 16384], got %d", bins);
    TEAL_REQUIRE(counts && overflow && p && t_out && np_ >= 0, "teal_hist_threshold: null pointer");
    if (np_ == 0) return TEAL_OK;
    const size_t smem = (size_t)bins * 8;
    cudaFuncSetAttribute(hist_threshold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hist_threshold_kernel<<<1, 1024, smem, stream>>>(counts, bins, overflow, hi, p, np_, t_out);
    return check_launch("teal_hist_threshold");
}

}  // extern "C"
