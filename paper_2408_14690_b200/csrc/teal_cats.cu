// CATS-style output-sparse GEMV (sm_100a) — the paper's output-sparsity
// baseline for the MLP (the reference's
// mlp_forward_output_sparse, pkg/src/actsparse/model.py:331-341):
//
//   inter[j] = keep_j ? gate[j] * (x . W_up[j, :]) : 0,   keep_j = !(|gate_j| <= t)
//
// with the SiLU(gate) vector already computed (dense).  The mask selects
// OUTPUT rows, so W_up is stored row-major (output-major: row j = the m
// input weights of output j, contiguous) and each kept output streams one
// contiguous row.  Per CTA: the gate values of its output range are
// thresholded and compacted (warp ballot, ordered), x is staged in shared
// memory once, then each warp takes kept rows round-robin with the whole row
// in flight (m * 2 B of 16-byte loads across 32 lanes), a fixed-order warp
// reduction, and the product with the gate.  Memory-bound: bytes =
// kept * m * w_bytes + m * 4 + n * 4.
#include "teal_common.cuh"

namespace teal {
namespace cats {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int ROWS = 32;     // output rows per CTA (one warp's ballot; ~3 CTAs per SM at n = 14336)
constexpr int XMAX = 16384;  // staged x (fp32)
constexpr int V16 = 16;      // 16-byte loads per lane per pass (bf16: 16 * 8 * 32 = 4096 elements)

template <typename WT>
__global__ void __launch_bounds__(NT) cats_kernel(const WT* __restrict__ w, int64_t n, int64_t m, int64_t ldw,
                                                  const float* __restrict__ x, const float* __restrict__ gate,
                                                  float t32, float* __restrict__ out, uint32_t* __restrict__ bits,
                                                  unsigned long long* __restrict__ kept) {
    extern __shared__ __align__(16) float s_x[];
    __shared__ int s_rows[ROWS];
    __shared__ int s_tot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    if (warp == 0) {  // threshold + ordered compaction of this CTA's 32 output rows
        const int64_t j = r0 + lane;
        const bool valid = j < n;
        const float g = valid ? gate[j] : 0.f;
        const bool keep = valid && !(fabsf(g) <= t32);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bits && lane == 0) bits[r0 >> 5] = bal;
        if (keep) s_rows[__popc(bal & ((1u << lane) - 1u))] = lane;
        if (!keep && valid) out[j] = 0.f;
        if (lane == 0) {
            s_tot = __popc(bal);
            if (kept && bal) atomicAdd(kept, (unsigned long long)__popc(bal));
        }
    }
    for (int64_t i = tid; i < m; i += NT) s_x[i] = x[i];
    __syncthreads();
    const int tot = s_tot;
    constexpr int EPL = 16 / sizeof(WT);  // elements per 16-byte load
    for (int e = warp; e < tot; e += NW) {
        const int64_t row = r0 + s_rows[e];
        const WT* wr = w + row * ldw;
        float acc = 0.f;
        for (int64_t c0 = 0; c0 < m; c0 += (int64_t)V16 * 32 * EPL) {
            uint4 v[V16];
#pragma unroll
            for (int q = 0; q < V16; ++q) {  // every load of the pass in flight (clamped: unused past m)
                const int64_t c = c0 + ((int64_t)q * 32 + lane) * EPL;
                v[q] = ldg128_stream(wr + (c < m ? c : 0));
            }
#pragma unroll
            for (int q = 0; q < V16; ++q) {
                const int64_t c = c0 + ((int64_t)q * 32 + lane) * EPL;
                if (c < m) {
                    if constexpr (sizeof(WT) == 2) {
                        const uint32_t u[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            acc = fmaf(bf16_lo(u[k]), s_x[c + 2 * k], acc);
                            acc = fmaf(bf16_hi(u[k]), s_x[c + 2 * k + 1], acc);
                        }
                    } else {
                        acc = fmaf(__uint_as_float(v[q].x), s_x[c], acc);
                        acc = fmaf(__uint_as_float(v[q].y), s_x[c + 1], acc);
                        acc = fmaf(__uint_as_float(v[q].z), s_x[c + 2], acc);
                        acc = fmaf(__uint_as_float(v[q].w), s_x[c + 3], acc);
                    }
                }
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) out[row] = gate[row] * acc;
    }
}

}  // namespace cats
}  // namespace teal

using namespace teal;
using namespace teal::cats;

extern "C" {

int teal_output_sparse_gemv(const void* w, int w_dtype, int64_t n, int64_t m, int64_t ldw, const float* x,
                            const float* gate, float t32, float* out, uint32_t* keep_bits,
                            unsigned long long* kept, cudaStream_t stream) {
    TEAL_REQUIRE(w && x && gate && out, "teal_output_sparse_gemv: null pointer");
    TEAL_REQUIRE(n >= 1 && m >= 1 && ldw >= m, "teal_output_sparse_gemv: bad shape n=%lld m=%lld ldw=%lld",
                 (long long)n, (long long)m, (long long)ldw);
    TEAL_REQUIRE(m <= XMAX, "teal_output_sparse_gemv: m must be <= %d", XMAX);
    TEAL_REQUIRE(t32 == t32 && (t32 >= 0.f || t32 == -INFINITY), "threshold must be non-negative, got %g", (double)t32);
    const int esz = w_dtype == TEAL_BF16 ? 2 : (w_dtype == TEAL_F32 ? 4 : 0);
    TEAL_REQUIRE(esz, "teal_output_sparse_gemv: weights must be bf16 or fp32 (got %d)", w_dtype);
    TEAL_REQUIRE((m * esz) % 16 == 0 && (ldw * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0,
                 "teal_output_sparse_gemv: rows must be 16-byte aligned multiples of 16 bytes");
    const int grid = (int)((n + ROWS - 1) / ROWS);
    const size_t smem = (size_t)m * 4;
    static unsigned long long attr = 0ull;  // dynamic shared-memory opt-in, per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("teal_output_sparse_gemv (device)");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&attr, __ATOMIC_ACQUIRE) & bit)) {
        cudaFuncSetAttribute(cats_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, XMAX * 4);
        cudaFuncSetAttribute(cats_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, XMAX * 4);
        __atomic_fetch_or(&attr, bit, __ATOMIC_RELEASE);
    }
    if (w_dtype == TEAL_BF16)
        cats_kernel<uint16_t><<<grid, NT, smem, stream>>>((const uint16_t*)w, n, m, ldw, x, gate, t32, out, keep_bits, kept);
    else
        cats_kernel<float><<<grid, NT, smem, stream>>>((const float*)w, n, m, ldw, x, gate, t32, out, keep_bits, kept);
    return check_launch("teal_output_sparse_gemv");
}

}  // extern "C"
