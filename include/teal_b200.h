/*
 * teal_b200.h — C ABI of the B200-native TEAL decode hot path.
 *
 * Every entry point takes caller-owned DEVICE pointers, plain sizes and a
 * cudaStream_t, returns an int status (TEAL_OK = 0) and never allocates,
 * frees or synchronises.  The last error message of the calling thread is
 * available from teal_last_error().  No C++ exception crosses this boundary.
 * All launches are stream-ordered and CUDA-graph capturable.  The library
 * reads no environment variables; its only process-wide state is a per-
 * process cache of immutable device facts (SM count, kernel occupancy) and
 * of one-time kernel attributes (dynamic shared-memory opt-in), all
 * idempotent.
 *
 * teal_sparse_gemv / teal_dense_gemv / teal_fused_gemv calls with one
 * segment, the PLAIN prologue, the STORE epilogue, fp32 x and bf16 / fp32 /
 * int8 rows run on the persistent step kernel's streaming core
 * (gemv_one_kernel in teal_step.cu, split tiles combined in contributor
 * order); every other fused variant runs the gemv_tma / register kernels of
 * teal_gemv.cu.  Both paths have the same masks and MAC counts.
 *
 * Reference interfaces replaced (paths relative to the reference tree):
 *   teal_threshold         <- sparsifier.sparsify / realized_sparsity
 *                             (pkg/src/actsparse/sparsifier.py:120-133)
 *   teal_threshold_batched <- sparsifier.sparsify_batched (sparsifier.py:136-155)
 *   teal_sparse_gemv       <- kernel.sparse_gemv -> _skip_gemv numba FFI
 *                             (pkg/src/actsparse/kernel.py:30-65, call site :62)
 *   teal_dense_gemv        <- tensor.matmul_dense -> _gemv_{row,col}major
 *                             (pkg/src/actsparse/tensor.py:107-140)
 *   teal_fused_gemv        <- the seven `gated(name, a) @ W.T` sites of
 *                             model._forward (pkg/src/actsparse/model.py:166-198)
 *                             with RMSNorm prologue (model.py:126-128),
 *                             SiLU(gate)*up epilogue (model.py:131-132,191-193)
 *                             and residual adds (model.py:184,198)
 *   teal_hist_record       <- ActivationHistogram.record (sparsifier.py:68-83)
 *   teal_hist_threshold    <- ActivationHistogram.threshold (sparsifier.py:94-117)
 *   teal_decode_attention  <- model._causal_attention, row t (model.py:135-150)
 *   teal_gemv_batched      <- sparsifier.sparsify_batched + matmul_dense per row
 *                             (sparsifier.py:136-155, tensor.py:130-140)
 *   teal_output_sparse_gemv <- model.mlp_forward_output_sparse's up projection
 *                             (model.py:331-341, the paper's CATS baseline)
 *   teal_prefill_gate / teal_prefill_gemm <- sparsify + matmul_dense over the
 *                             prompt rows >= sparse_from (
 *                             the reference has no prefill)
 */
#ifndef TEAL_B200_H
#define TEAL_B200_H

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TEAL_ABI_VERSION 1

/* status codes */
#define TEAL_OK 0
#define TEAL_EINVAL 1   /* invalid argument (message via teal_last_error) */
#define TEAL_ECUDA 2    /* CUDA launch / runtime error */

/* element types */
#define TEAL_F32 0
#define TEAL_BF16 1
#define TEAL_F64 4      /* teal_hist_record input only (the reference bins float64) */
#define TEAL_I8 2       /* int8 rows, per-output-column fp32 scale */
#define TEAL_I4 3       /* int4 rows (two per byte, low nibble = even column),
                           fp32 scale per (group of input rows, column) */

/* fused-GEMV prologues: how the input h is formed from x */
#define TEAL_PRO_PLAIN 0     /* h_i = x_i */
#define TEAL_PRO_RMSNORM 1   /* h_i = x_i / sqrt(sum(ss_part)/m + eps) * norm_scale_i */

/* fused-GEMV epilogues */
#define TEAL_EPI_STORE 0     /* seg.y[j] = acc_j                          */
#define TEAL_EPI_RESID 1     /* resid[j] += acc_j ; ss_out[tile] = sum x^2 */
#define TEAL_EPI_SILU 2      /* inter[j] = silu(acc_gate_j) * acc_up_j    */
#define TEAL_EPI_QKV 3       /* q -> rope -> q_out ; k -> rope -> k cache ; v -> v cache */

const char* teal_last_error(void);
int teal_abi_version(void);
int teal_device_sm_count(int device);

/* ---- thresholding ------------------------------------------------------ */

/* keep_i = !(|x_i| <= t32)  (closed prune boundary, NaN kept).
 * keep_bits (nullable): bit i%32 of word i/32 set iff kept; [ceil(m/32)] words.
 * x_sparse  (nullable): x with pruned entries replaced by +0.0, same dtype as x.
 * pruned    (nullable): atomically incremented by the number of pruned entries. */
int teal_threshold(const void* x, int x_dtype, int64_t m, float t32,
                   uint32_t* keep_bits, void* x_sparse,
                   unsigned long long* pruned, cudaStream_t stream);

/* Shared column mask over a [B, m] fp32 batch: column i pruned iff
 * (sum_b |X[b,i]| in ascending b, fp32) / B <= t32.  mask[i] = 1 if pruned.
 * xs_sparse (nullable) receives the batch with pruned columns zeroed. */
int teal_threshold_batched(const float* xs, int64_t B, int64_t m, float t32,
                           uint8_t* mask, float* xs_sparse, cudaStream_t stream);

/* ---- GEMV over input-major (transposed) weights ------------------------ */

/* One projection inside a fused launch.  Element (input i, output j) of the
 * segment lives at w[i*ldw + j] (the reference's COL_MAJOR layout of the
 * logical [n_out, m_in] matrix, tensor.py:47-48). */
typedef struct teal_seg {
    const void* w;               /* weights, w_dtype elements                   */
    int64_t ldw;                 /* row stride in elements (>= n)              */
    int64_t n;                   /* output columns                              */
    float t32;                   /* keep iff !(|h_i| <= t32); -INFINITY = dense */
    float* y;                    /* EPI_STORE output [n] fp32                   */
    const float* col_scale;      /* TEAL_I8 only: per-output-column scale [n]   */
    uint32_t* dbg_bits;          /* nullable: keep bitmask of h [ceil(m/32)]    */
    unsigned long long* kept;    /* nullable: += kept input channels            */
} teal_seg;

typedef struct teal_gemv_args {
    int w_dtype;                 /* TEAL_F32 / TEAL_BF16 / TEAL_I8              */
    int x_dtype;                 /* TEAL_F32 / TEAL_BF16 (PRO_PLAIN only)       */
    const void* x;               /* input vector [m]                            */
    int64_t m;                   /* input channels                              */
    int nseg;                    /* 1..3                                        */
    teal_seg seg[3];
    /* prologue */
    int prologue;
    const float* norm_scale;     /* RMSNorm gain [m]                            */
    const float* ss_part;        /* fp32 partial sums of x^2, summed in order   */
    int ss_count;
    float eps;
    float* dbg_h;                /* nullable: h [m] fp32 (written once)         */
    /* epilogue */
    int epilogue;
    float* resid;                /* EPI_RESID: residual stream [n], updated     */
    float* ss_out;               /* EPI_RESID: [tiles] partial sum of squares   */
    float* inter;                /* EPI_SILU: [n]                               */
    float* q_out;                /* EPI_QKV: rotated q [n_q]                    */
    void* k_cache;               /* EPI_QKV: [kv_heads][max_seq][head_dim]      */
    void* v_cache;
    int kv_dtype;                /* TEAL_F32 / TEAL_BF16                        */
    int64_t max_seq;
    const int* pos;              /* device scalar: position being written       */
    int head_dim;
    const float* rope_cos;       /* nullable (no RoPE): [max_seq][head_dim/2]   */
    const float* rope_sin;
    /* persistent split-K grid and workspace (caller-owned) */
    int ctas;                    /* CTAs (0 = auto: CTAS_PER_SM x #SMs)         */
    float* ws;                   /* split-K partials, teal_gemv_workspace() floats */
    uint32_t* tickets;           /* one per column tile, zero before first use;
                                    self-resetting (graph-replay safe)          */
} teal_gemv_args;

/* Work decomposition: the (column tile, 32-channel group) space of all
 * segments is flattened tile-major and split into `ctas` equal contiguous
 * ranges, one per CTA of a single persistent wave; a column tile shared by
 * several CTAs is reduced by its last-arriving CTA in ascending-CTA order.
 * teal_gemv_workspace() resolves ctas=0 and reports the ws/ticket sizes. */
int teal_gemv_workspace(const teal_gemv_args* a, int* ctas, int64_t* ws_floats,
                        int64_t* tickets);
int teal_gemv_tile_width(const teal_gemv_args* a);
/* Debug: copy n per-CTA phase timestamps of the last launch run with
 * TEAL_TIMELINE=1 in the environment (synchronous; not for the hot path). */
int teal_debug_timeline(unsigned long long* host_dst, int n);
int teal_fused_gemv(const teal_gemv_args* a, cudaStream_t stream);

/* Convenience single-projection forms (kernel.py:30-65 / tensor.py:137-140). */
int teal_sparse_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw,
                     const void* x, int x_dtype, float t32, float* y,
                     const float* col_scale,
                     float* ws, uint32_t* tickets, int ctas,
                     unsigned long long* kept, cudaStream_t stream);
int teal_dense_gemv(const void* w, int w_dtype, int64_t m, int64_t n, int64_t ldw,
                    const void* x, int x_dtype, float* y, const float* col_scale,
                    float* ws, uint32_t* tickets, int ctas, cudaStream_t stream);


/* ---- batched shared-mask sparse GEMV over bf16 / int8 / int4 rows ---------
 * Replaces sparsify_batched followed by the dense product
 * (sparsifier.py:136-155, tensor.py:130-140) for B <= 16 decode rows:
 * column i is pruned in every row iff mean_b |x[b,i]| <= t32 (fp32 sum in
 * ascending b, fp64 quotient rounded to fp32), and
 * y[b] = sum over kept i of x[b,i] * W[i,:] — each kept row read once.
 * Routes: bf16 rows, 4 <= B <= 16, n a multiple of 128 with n >= 8192 (and a
 * 16-byte aligned w): a compaction launch + a tcgen05 / TMEM contraction
 * (teal_gemv_tc.cu; ctas is ignored and reported 0 by the workspace query;
 * ws must be 256-byte aligned); other shapes at B >= 4: the mma.sync kernel;
 * B < 4: the CUDA-core kernel.  All routes give the same mask and kept count
 * and the fp32-GEMV accuracy. */
typedef struct teal_gemv_batched_args {
    const void* w;               /* input-major rows, row stride ldw elements   */
    const float* scale;          /* I8: [n]; I4: [ceil(m/group)][n]             */
    const float* x;              /* [B][m] fp32                                 */
    float* y;                    /* [B][n] fp32                                 */
    uint8_t* mask;               /* nullable: [m], 1 = pruned                   */
    unsigned long long* kept;    /* nullable: += kept input channels            */
    float* ws;                   /* split-K partials (teal_gemv_batched_workspace) */
    uint32_t* tickets;           /* zeroed, self-resetting                      */
    int64_t m, n, ldw;
    int w_dtype;                 /* TEAL_BF16 / TEAL_I8 / TEAL_I4               */
    int group;                   /* I4 row-group size                           */
    int B;                       /* 1..16                                       */
    float t32;                   /* -INFINITY = dense                           */
    int ctas;                    /* 0 = auto                                    */
    int pad_;
} teal_gemv_batched_args;

int teal_gemv_batched_workspace(const teal_gemv_batched_args* a, int* ctas, int64_t* ws_floats, int64_t* tickets);
int teal_gemv_batched(const teal_gemv_batched_args* a, cudaStream_t stream);

/* ---- calibration ------------------------------------------------------- */

/* counts[b] += #{i : floor(|x_i|/hi*bins) clipped to bins-1 == b, |x_i| <= hi}
 * overflow  += #{i : |x_i| > hi};  nan_flag set to 1 if any NaN.
 * Binning in fp64 exactly as numpy (sparsifier.py:75-80); x_dtype TEAL_F32,
 * TEAL_BF16 or TEAL_F64 (float64 input is binned unrounded, as the reference
 * does with np.asarray(x, float64)). */
int teal_hist_record(const void* x, int x_dtype, int64_t count, double hi, int bins,
                     unsigned long long* counts, unsigned long long* overflow,
                     unsigned int* nan_flag, cudaStream_t stream);

/* Thresholds for np levels p[] from one histogram (sparsifier.py:94-117);
 * total = sum(counts) + overflow.  One CTA, fp64, results bit-identical to
 * the reference's numpy arithmetic. */
int teal_hist_threshold(const unsigned long long* counts, int bins,
                        const unsigned long long* overflow, double hi,
                        const double* p, int np_, double* t_out, cudaStream_t stream);

/* ---- decode-step helpers ----------------------------------------------- */

/* ctx[h*hd + d] = softmax_u(q_h . k_u / sqrt(hd)) v_u over positions u < *len,
 * GQA: q head h reads kv head h / (H / KVH). */
int teal_decode_attention(const float* q, const void* k_cache, const void* v_cache,
                          int kv_dtype, int H, int KVH, int hd, int64_t max_seq,
                          const int* len, int max_len, float* ctx,
                          float* ws, uint32_t* tickets, int nsplit,
                          cudaStream_t stream);

/* x = float(src) (src row = emb + (*token)*d when token != NULL, else src);
 * ss_out[t] = sum of x^2 over columns [t*tile, (t+1)*tile).
 * step_state (nullable) = {pos, len}: starts a decode step — pos = len,
 * len = len + 1 (pos is the KV position this step writes, len the attended
 * length), so a captured graph of one step replays token after token. */
int teal_load_residual(const void* src, int src_dtype, const int* token, int64_t d,
                       float* x, float* ss_out, int tile, int* step_state,
                       cudaStream_t stream);

/* Tensor-parallel row-parallel epilogue after the all-reduce of the partial
 * projections: x += delta; ss_out[t] = sum of x^2 over tile t (model.py:184,198). */
int teal_residual_add(float* x, const float* delta, int64_t d, float* ss_out, int tile, cudaStream_t stream);

/* out_token = argmax(logits) (lowest index on ties, NaN ignored). */
int teal_argmax(const float* logits, int64_t n, int* out_token,
                float* ws, uint32_t* tickets, cudaStream_t stream);


/* ---- CATS output-sparse GEMV (the paper's output-sparsity baseline) -----
 * out[j] = keep_j ? gate[j] * (x . W[j, :]) : 0, keep_j = !(|gate_j| <= t32),
 * W row-major [n][ldw] (output-major: row j = output j's m input weights,
 * bf16 / fp32), x [m] fp32, gate [n] fp32 (SiLU already applied).  Replaces
 * the up-projection of mlp_forward_output_sparse (model.py:331-341) at
 * decode time: only the rows of kept outputs are read.  keep_bits (nullable)
 * [ceil(n/32)], kept (nullable) += kept outputs.  m <= 16384. */
int teal_output_sparse_gemv(const void* w, int w_dtype, int64_t n, int64_t m, int64_t ldw, const float* x,
                            const float* gate, float t32, float* out, uint32_t* keep_bits,
                            unsigned long long* kept, cudaStream_t stream);

/* ---- sparse prefill (the prompt pass before decode) ----------------------
 * TEAL's prefill recipe (not in the reference,
 * SPEC.md:8): prompt positions t < sparse_from stay dense (attention sinks),
 * later ones are thresholded with decode's test, then multiplied — per row,
 * the reference's sparsify + matmul_dense (sparsifier.py:120-134,
 * tensor.py:130-140).  Two launches:
 *
 * teal_prefill_gate: G = mask(X) of X fp32 [T][ldx] (keep = t < sparse_from
 * || !(|x| <= t32)), written as bf16 x_hi = rn(G) and (x_lo non-NULL)
 * x_lo = rn(G - x_hi), both [T][ldo]; m, ldx, ldo multiples of 4.  kept
 * (nullable) += kept values among the thresholded rows.
 *
 * teal_prefill_gemm: y[t][:] (+)= (x_hi + x_lo)[t][:] @ W on the tcgen05
 * tensor cores (TMA-staged, fp32 TMEM accumulator), W bf16 input-major
 * [m][ldw] (the decode engines' layout); x_lo NULL: one bf16 term.
 * m multiple of 64, n multiple of 128, 16-byte aligned operands.  A
 * persistent launch (one CTA per SM, double-buffered TMEM accumulators);
 * grids smaller than the SM count split K, the last-arriving split summing
 * the partials in ascending split order (deterministic). */
typedef struct teal_prefill_args {
    const void* w;      /* bf16 [m][ldw] */
    int64_t m, n, ldw;
    const void* x_hi;   /* bf16 [T][ldx] */
    const void* x_lo;   /* bf16 [T][ldx] or NULL */
    int64_t T, ldx;
    float* y;           /* fp32 [T][ldy] */
    int64_t ldy;
    int accumulate;     /* 0: y = G @ W; 1: y += G @ W (residual add) */
    int splits;         /* K splits: 0 = auto (fill the SMs), 1 = none */
    float* ws;          /* split-K partials [splits][T][n] (teal_prefill_workspace) or NULL: no split */
    uint32_t* tickets;  /* [output tiles], zeroed, self-resetting */
} teal_prefill_args;

int teal_prefill_gate(const float* x, int64_t T, int64_t m, int64_t ldx, float t32, int64_t sparse_from,
                      void* x_hi, void* x_lo, int64_t ldo, unsigned long long* kept, cudaStream_t stream);
int teal_prefill_workspace(const teal_prefill_args* a, int* splits, int64_t* ws_floats, int64_t* tickets);
int teal_prefill_gemm(const teal_prefill_args* a, cudaStream_t stream);
/* RoPE of the prompt rows (rotate-half, as teal_batch_rope_cache; row t is
 * position pos0 + t): q [T][ldq] rotated in place, rotated k [T][ldk] and v
 * [T][ldv] written to the caches [KVH][max_seq][hd] rows pos0 .. pos0+T-1. */
int teal_prefill_rope_cache(float* q, int64_t ldq, const float* k, int64_t ldk, const float* v, int64_t ldv, int T,
                            int H, int KVH, int hd, int64_t pos0, const float* rope_cos, const float* rope_sin,
                            void* k_cache, void* v_cache, int kv_dtype, int64_t max_seq, cudaStream_t stream);

/* ---- small-batch decode (config 5: B sequences in lockstep) -------------
 * The projections run in teal_gemv_batched (one shared mask per projection,
 * sparsifier.sparsify_batched, sparsifier.py:136-155); these are the steps
 * around them, one launch for all B rows each. */

/* teal_decode_attention for B sequences: q / ctx [B][H*hd], caches
 * [B][KVH][max_seq][hd] (sequence b's slice at b*KVH*max_seq*hd), *len
 * positions each (model.py:135-150); ws / tickets: B times the B = 1 sizes. */
int teal_batch_attention(const float* q, const void* k_cache, const void* v_cache, int kv_dtype, int B, int H,
                         int KVH, int hd, int64_t max_seq, const int* len, int max_len, float* ctx, float* ws,
                         uint32_t* tickets, int nsplit, cudaStream_t stream);
/* x[b] = float(emb[tokens[b]]), x [B][d]; state (nullable) {pos, len}: this
 * step writes position len (pos = len, len += 1) */
int teal_batch_embed(const void* emb, int emb_dtype, const int* tokens, int B, int64_t d, float* x, int* state,
                     cudaStream_t stream);
/* x[b] += delta[b] (delta nullable); h[b] = x[b] / sqrt(mean(x[b]^2) + eps) * gain
 * (model.py:126-128 with the residual adds of model.py:184,198) */
int teal_batch_rmsnorm(float* x, const float* delta, const float* gain, float eps, int B, int64_t d, float* h,
                       cudaStream_t stream);
/* RoPE (rotate-half, cos/sin tables [max_seq][hd/2]; NULL: none) of q [B][H][hd]
 * and k [B][KVH][hd] in place at position state[0]; k and v [B][KVH][hd]
 * appended to the caches [B][KVH][max_seq][hd] (kv dtype TEAL_BF16 / F32).
 * Traps when state[0] is outside [0, max_seq). */
int teal_batch_rope_cache(float* q, float* k, const float* v, void* k_cache, void* v_cache, int kv_dtype,
                          const float* rope_cos, const float* rope_sin, const int* state, int B, int H, int KVH,
                          int hd, int64_t max_seq, cudaStream_t stream);
/* out = SiLU(gate) * up elementwise over n = B * d_ff values (model.py:190-193) */
int teal_batch_silu_mul(const float* gate, const float* up, int64_t n, float* out, cudaStream_t stream);
/* tokens[b] = argmax of logits[b] ([B][n]; lowest index on ties, NaN ignored) */
int teal_batch_argmax(const float* logits, int B, int64_t n, int* tokens, cudaStream_t stream);
/* Stream plumbing for running independent projections concurrently (the
 * batch decoder's q / k / v and gate / up), in the same CUDA runtime as the
 * library's launches: non-blocking streams, timing-free events, and
 * teal_stream_order = record e on `signaler`, make `waiter` wait for it
 * (graph-capture safe: the fork / join pattern). */
int teal_stream_create(cudaStream_t* s);
int teal_stream_destroy(cudaStream_t s);
int teal_event_create(cudaEvent_t* e);
int teal_event_destroy(cudaEvent_t e);
int teal_stream_order(cudaStream_t waiter, cudaStream_t signaler, cudaEvent_t e);

/* ---- persistent decode step (one launch per token) ----------------------
 *
 * Replaces the per-projection launches of a decode step (the seven
 * `gated(name, a) @ W.T` products of model._forward, model.py:158-198, plus
 * attention, residual load, LM head and argmax) with ONE persistent
 * cooperative launch.  Every CTA walks the same list of PHASES (per layer:
 * qkv, attention, o, gate/up, down; then the LM head) and owns a static,
 * equal slice of every GEMV phase: the flattened (column tile, 32-channel
 * group) space of the phase is cut into G equal contiguous ranges, one per
 * CTA, so all CTAs finish a phase together.  Ordering between phases uses
 * dependency counters instead of grid barriers: a slice waits only for the
 * input rows it reads (attention groups for o, gate/up tiles for down); the
 * RMSNorm inputs (whole residual + sum of squares) are the only global joins.
 *
 * Weights are stored TILED input-major: a group's output columns are cut
 * into tiles of TEAL_STEP_TW columns and tile t is the contiguous block
 * w[t][i][0..TW) over input channels i (element (out t*TW + c, in i) =
 * w[(t*m + i)*TW + c]); a kept channel streams one contiguous row chunk per
 * tile, register-streamed by the warps (16-byte non-allocating loads, L2
 * evict-first, the next rows' loads in flight while the current ones are
 * consumed).  Each tile carries two column halves with their own thresholds
 * (gate | up interleaved for the MLP).  Layer outputs are int64 fixed-point
 * accumulators (ACC, 2^-32 units) that every contributor of a tile adds its
 * column partials into with red.add — integer addition is associative, so
 * the result does not depend on arrival order; the LM head's split tiles are
 * finished by their last-arriving contributor, summing fp32 partials in
 * contributor order (deterministic two-phase reduction). */
#define TEAL_STEP_TW 256
#define TEAL_PHASE_LOAD 0
#define TEAL_PHASE_GEMV 1
#define TEAL_PHASE_ATTN 2
#define TEAL_PHASE_RESID 3   /* x_out = x + fx(in_acc), CTA-partitioned (plans without an LM head) */
/* Step-engine prologues reading a fixed-point accumulator (see ACC below) */
#define TEAL_PRO_RMS_ACC 2   /* x' = x + fx(in_acc); h = RMSNorm(x'); each CTA writes its share of x' to x_out */
#define TEAL_PRO_SILU_ACC 3  /* h_i = silu(fx(in_acc[gate_i])) * fx(in_acc[up_i]) (gate/up tile layout) */
/* ACC output (group.acc != NULL): every split-K contributor adds its column
 * partials to an int64 fixed-point accumulator (2^-TEAL_STEP_FX_BITS units,
 * integer addition: order-independent, so deterministic) and bumps the
 * tile's counters so that each finished tile adds TEAL_STEP_CONTRIB in total.
 * Range |value| < 2^31. */
#define TEAL_STEP_FX_BITS 32
#define TEAL_STEP_CONTRIB 1024
#define TEAL_DEP_NONE 0
#define TEAL_DEP_GLOBAL 1    /* counters[dep] >= target                          */
#define TEAL_DEP_ROWS 2      /* counters[dep + r / dep_rows] >= target for every input row r read */

#define TEAL_SEPI_STORE 0    /* y[col] = v                                   */
#define TEAL_SEPI_RESID 1    /* resid[col] += v ; ss_out[tile] = sum resid^2 */
#define TEAL_SEPI_SILU 2     /* inter[t*TW/2 + c] = silu(lo_c) * hi_c         */
#define TEAL_SEPI_QKV 3      /* q -> rope -> q_out ; k -> rope -> k cache ; v -> v cache */
#define TEAL_SEPI_LOGITS 4   /* y[col] = v ; per-tile argmax candidate; last tile -> token */

typedef struct teal_step_tile {
    float t_lo, t_hi;        /* keep iff !(|h| <= t); -INFINITY = dense      */
    int seg_lo, seg_hi;      /* debug segment of each half (0..2)            */
    int first_lo, first_hi;  /* 1 if this tile is the first of its segment  */
    int sig0, sig1;          /* counters [sig0, sig1] += 1 on finalize (sig0 < 0: none) */
} teal_step_tile;

typedef struct teal_step_group {
    const void* w;           /* tiled weights [ntiles][m][TW]               */
    const float* col_scale;  /* int8 rows: per-column scale [ntiles*TW]      */
    const teal_step_tile* tiles;  /* [ntiles]                               */
    const float* x;          /* input vector [m] (written earlier in the step) */
    const float* gain;       /* PRO_RMSNORM gain [m]                         */
    const float* ss;         /* PRO_RMSNORM: sum-of-squares partials [nss]   */
    float* partials;         /* [ntiles][maxc][TW]                            */
    unsigned* tickets;       /* [ntiles], zero, self-resetting               */
    float* y;                /* STORE / LOGITS output [n]                    */
    float* resid;            /* RESID residual stream [n]                    */
    float* ss_out;           /* RESID: [ntiles] partial sums of squares       */
    float* inter;            /* SILU output [ntiles*TW/2]                    */
    float* q_out;            /* QKV                                          */
    void* k_cache;
    void* v_cache;
    const float* rope_cos;   /* nullable [max_seq][hd/2]                      */
    const float* rope_sin;
    float* dbg_h;            /* nullable: prologue h [m]                     */
    uint32_t* dbg_bits[3];   /* nullable: keep bits per segment [ceil(m/32)] */
    unsigned long long* kept[3];  /* nullable: kept channels per segment    */
    int64_t max_seq;
    int m, n, ntiles, maxc;  /* maxc: partial slots per tile                 */
    int prologue, nss;
    float eps;
    int epilogue;
    int nq, nkv, head_dim, kv_dtype;
    int w_dtype;             /* TEAL_F32 / TEAL_BF16 / TEAL_I8 (col_scale) / TEAL_I4 (gscale) */
    const float* gscale;     /* TEAL_I4: [ceil(m/group)][ntiles*TW] fp32      */
    int group;               /* TEAL_I4 row-group size (>= 128)              */
    float t_all;             /* tiles == NULL: one threshold for every tile  */
    int64_t tile_stride_b;   /* row_stride_b == 0: tiled (m*TW*esz, TW*esz)   */
    int64_t row_stride_b;    /* else untiled input-major: TW*esz, ldw*esz    */
    long long* acc;          /* nullable ACC output [ntiles*TW] (zero at step start) */
    const long long* in_acc; /* PRO_RMS_ACC: delta [m]; PRO_SILU_ACC: gate/up accumulator */
    float* x_out;            /* PRO_RMS_ACC / PHASE_RESID: materialised x' [m]  */
    const int4* ranges;      /* nullable ACC work split: CTA c < nranges takes 32-row
                                groups [x, y) (at most two tiles) and bumps its first /
                                second tile's counters by z / w; NULL: equal split */
    int nranges;
    int xsig;                /* PRO_RMS_ACC: counter bumped by each CTA once its x_out share is
                                written (-1: none)                                      */
    int xwait, xwait_target; /* PRO_RMS_ACC: x (the previous version) is complete when
                                counters[xwait] >= xwait_target; it is then staged before
                                the phase's own dependency wait (-1: stage after it)   */
    int tp_sum;              /* tensor parallel (plan.tp != NULL): a row-parallel ACC output —
                                every contributor adds its partials to EVERY rank's
                                accumulator and bumps every rank's tile counters (the
                                consumers' targets are world x CONTRIB per tile)        */
} teal_step_group;

typedef struct teal_step_attn {
    const float* q;          /* [H*hd]                                       */
    const void* k_cache;     /* [KVH][max_seq][hd]                            */
    const void* v_cache;
    float* ctx;              /* [H*hd]                                       */
    float* partials;         /* [KVH][nchunks][G*hd + 2G]                    */
    unsigned* tickets;       /* [KVH]                                        */
    int64_t max_seq;
    int H, KVH, hd, kv_dtype;
    int chunk, nchunks;
    int sig_base;            /* counter sig_base + g += 1 when group g's ctx is final */
    int dep_base;            /* unit (g, *) waits for counters[dep_base + g] >= dep_target[g] */
    const int* dep_target;   /* [KVH]                                         */
    unsigned long long* dbg; /* nullable debug: [KVH*nchunks][6] %globaltimer stamps */
    const long long* qkv_acc;  /* nullable: q|k|v ACC accumulator of the qkv group; the
                                  units then apply RoPE themselves and the unit holding
                                  the new position writes its k, v to the cache */
    const float* rope_cos;   /* nullable [max_seq][hd/2]                      */
    const float* rope_sin;
    int nq, nkv;             /* q / k columns (qkv_acc offsets)               */
    int super_chunks;        /* long-context kernel (plan.long_ctx): one unit walks this
                                many chunks with an online softmax (>= 1)           */
    int home;                /* > 0: CTAs [home, grid) take no part in the qkv phase; when
                                the units fit there, unit u runs on CTA home + u (it stages
                                its K/V rows while qkv streams and waits ready) */
} teal_step_attn;

typedef struct teal_step_phase {
    int kind, group;         /* TEAL_PHASE_*; index into groups / attns      */
    int dep_kind, dep;       /* TEAL_DEP_*; counter (base) index             */
    int target, dep_rows;
} teal_step_phase;

/* Tensor-parallel group of a fused step launch (one launch per rank per
 * token; peers reached through peer-mapped pointers — CUDA IPC / NVLink — or,
 * for single-GPU validation, other ranks' buffers on the same device). */
#define TEAL_TP_MAX 8
typedef struct teal_step_tp {
    long long* acc[TEAL_TP_MAX];      /* each rank's accumulator block (same layout)        */
    int* counters[TEAL_TP_MAX];       /* each rank's dependency counters                   */
    unsigned* epoch[TEAL_TP_MAX];     /* each rank's [world] completed-step counts; rank j
                                         writes entry j of every rank's array at exit       */
    int* token[TEAL_TP_MAX];          /* each rank's token word                            */
    float* cand_v;                    /* rank 0: LM argmax candidates [world * ntiles]      */
    int* cand_i;
    unsigned* lm_ticket;              /* rank 0: LM tiles finished over all ranks          */
    int world, rank;
    int vocab_off;                    /* this rank's first vocabulary index                */
    int pad_;
} teal_step_tp;

typedef struct teal_step_plan {
    const teal_step_group* groups;   /* device arrays */
    const teal_step_attn* attns;
    const teal_step_phase* phases;
    int* counters;                   /* [ncounters * 32] zero (counter i at i*32, one 128-B line each);
                                        reset at the end of every launch */
    unsigned* ctrl;                  /* [4] zero: exit count                   */
    const void* emb;                 /* LOAD: embedding [vocab][d] (NULL: x_in) */
    const float* x_in;               /* LOAD: hidden row [d] when emb == NULL  */
    const int* token;                /* LOAD: token id (device)                */
    float* x;                        /* residual stream [d]                    */
    float* ss;                       /* [d / TW] partial sums of squares       */
    int* state;                      /* {pos, len}: LOAD sets pos = len, len += 1 */
    float* cand_v;                   /* LOGITS: per-tile argmax candidates     */
    int* cand_i;
    int* token_out;                  /* LOGITS: argmax token                   */
    unsigned* lm_done;               /* LOGITS: tiles finished (self-resetting) */
    unsigned long long* timeline;    /* nullable debug: [ctas][nphases][8] %globaltimer */
    int nphases, ncounters;
    int prefetch_bytes;              /* per CTA per GEMV phase: L2 prefetch of its weight range head (0: off) */
    int max_seq;                     /* KV-cache positions: LOAD traps when len >= max_seq (0: unchecked) */
    int d, emb_dtype;
    int w_dtype, ctas;               /* ctas: grid size (<= resident capacity)  */
    long long* acc_zero;             /* LOAD: ACC accumulators zeroed each step */
    int64_t acc_zero_n;              /* (elements)                              */
    const teal_step_tp* tp;          /* nullable device pointer: fused tensor parallel     */
    int noncoop, long_ctx;           /* noncoop 1: ordinary launch (single-GPU TP validation runs the
                                        ranks' launches concurrently on one device);
                                        long_ctx 1: the kernel variant whose attention units
                                        walk attn.super_chunks chunks each (long contexts) */
    int phase_begin, phase_end;      /* this launch runs phases [begin, end) (end 0: all).
                                        Dependencies on earlier launches are met by stream
                                        order: the host drops them from the phase list
                                        (tensor parallel: an all-reduce of the row-parallel
                                        accumulators between launches).                  */
} teal_step_plan;

/* Resident CTAs per SM of the step kernel for a weight dtype; the plan's
 * static slicing must be built for ctas = this x #SMs (or fewer). */
int teal_step_ctas_per_sm(int w_dtype);
int teal_step_launch(const teal_step_plan* plan, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TEAL_B200_H */
