/*
 * TEST INFRASTRUCTURE — plain-C restatement of the reference CPU kernels on
 * the TEAL decode hot path.  Used only by tests/ (as a checker) and by
 * bench.py's CPU-baseline leg / `--impl reference` arm (as the timed CPU
 * reference).  Never linked into the product library.
 *
 *   oracle_skip_gemv   <- kernel.py:30-44 `_skip_gemv` (numba, 1 thread):
 *                         for i ascending: skip iff |x_i| <= t (fp64 compare),
 *                         else y[j] += x_i * W[i*n + j] in fp32 (no FMA).
 *   oracle_skip_gemv_mt   the same loop with output columns split across
 *                         pthreads (disjoint outputs);
 *                         per-column arithmetic is unchanged, so results are
 *                         bit-identical to the single-thread version.
 *   oracle_skip_gemv_bf16 the same loop over bf16 rows widened to fp32.
 *   oracle_gemv_dense  <- tensor.py:107-116 `_gemv_rowmajor` order on
 *                         input-major storage (fp32, ascending i).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -pthread).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

long long oracle_skip_gemv(const float* x, const float* w, long long m, long long n, double t, float* y) {
    long long used = 0;
    for (long long j = 0; j < n; ++j) y[j] = 0.0f;
    for (long long i = 0; i < m; ++i) {
        const float xi = x[i];
        if (fabs((double)xi) <= t) continue;
        ++used;
        const float* row = w + i * n;
        for (long long j = 0; j < n; ++j) y[j] += xi * row[j];
    }
    return used;
}

static inline float bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Column-block worker shared by the multi-threaded variants. */
typedef struct {
    const float* x;
    const void* w;
    int w_bf16;
    long long m, n, j0, j1;
    double t;
    float* y;
} oracle_job;

static void* oracle_worker(void* arg) {
    const oracle_job* jb = (const oracle_job*)arg;
    for (long long j = jb->j0; j < jb->j1; ++j) jb->y[j] = 0.0f;
    for (long long i = 0; i < jb->m; ++i) {
        const float xi = jb->x[i];
        if (fabs((double)xi) <= jb->t) continue;
        if (jb->w_bf16) {
            const uint16_t* row = (const uint16_t*)jb->w + i * jb->n;
            for (long long j = jb->j0; j < jb->j1; ++j) jb->y[j] += xi * bf16_to_f32(row[j]);
        } else {
            const float* row = (const float*)jb->w + i * jb->n;
            for (long long j = jb->j0; j < jb->j1; ++j) jb->y[j] += xi * row[j];
        }
    }
    return NULL;
}

static long long run_mt(const float* x, const void* w, int w_bf16, long long m, long long n, double t, float* y,
                        int threads) {
    long long used = 0;
    for (long long i = 0; i < m; ++i) used += !(fabs((double)x[i]) <= t);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    oracle_job jobs[256];
    long long per = ((n + threads - 1) / threads + 15) / 16 * 16;
    int launched = 0;
    for (int k = 0; k < threads; ++k) {
        long long j0 = (long long)k * per, j1 = j0 + per;
        if (j1 > n) j1 = n;
        if (j0 >= j1) break;
        jobs[k] = (oracle_job){x, w, w_bf16, m, n, j0, j1, t, y};
        if (k == 0) continue;
        if (pthread_create(&th[k], NULL, oracle_worker, &jobs[k]) != 0) { oracle_worker(&jobs[k]); th[k] = 0; }
        launched = k;
    }
    oracle_worker(&jobs[0]);
    for (int k = 1; k <= launched; ++k)
        if (th[k]) pthread_join(th[k], NULL);
    return used;
}

long long oracle_skip_gemv_mt(const float* x, const float* w, long long m, long long n, double t, float* y,
                              int threads) {
    return run_mt(x, w, 0, m, n, t, y, threads);
}

long long oracle_skip_gemv_bf16_mt(const float* x, const uint16_t* w, long long m, long long n, double t, float* y,
                                   int threads) {
    return run_mt(x, w, 1, m, n, t, y, threads);
}

void oracle_gemv_dense(const float* x, const float* w, long long m, long long n, float* y) {
    for (long long j = 0; j < n; ++j) y[j] = 0.0f;
    for (long long i = 0; i < m; ++i) {
        const float xi = x[i];
        const float* row = w + i * n;
        for (long long j = 0; j < n; ++j) y[j] += xi * row[j];
    }
}

int oracle_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}
