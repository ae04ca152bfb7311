/*
 * CPU ORACLE — test infrastructure only (see oracle_router.c header).
 *
 * fp32 per-expert gated FFN (SwiGLU) over the coalesced batch:
 *     h = silu(x W1^T) * (x W3^T),   y = h W2^T
 * "gated FFN execution per expert" with three weight matrices (
 * weight_bytes.per_expert = 3*dt*d*ff in workload.py:182-189), run over the whole
 * coalesced batch of each expert (costmodel.py:240-258).
 * The inputs are the bf16-rounded values upcast exactly to fp32; all arithmetic
 * is fp32 (this file may contract a*b+c into fma: it is compared with tolerance).
 *
 * Also the timed "reference CPU path" for bench.py's cpu_baseline leg: OpenMP
 * over all host threads, AVX2/FMA vector extensions (x86-64-v3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef float v8f __attribute__((vector_size(32)));

static inline v8f ld8(const float* p) {
    v8f v;
    memcpy(&v, p, sizeof(v));
    return v;
}
static inline float hsum8(v8f v) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += v[i];
    return s;
}

/* C[i, j] = sum_k A[i, k] * B[j, k]   (A: n x K, B: N x K, both K-contiguous). */
static void gemm_nt(const float* A, long lda, const float* B, long ldb, float* C, long ldc, int n, int N, int K) {
    const int NB = 64;
    int nblk_j = (N + NB - 1) / NB;
    int nblk_i = (n + 3) / 4;
    long total = (long)nblk_j * nblk_i;
#pragma omp parallel for schedule(dynamic, 4)
    for (long task = 0; task < total; ++task) {
        int jb = (int)(task / nblk_i);
        int ib = (int)(task % nblk_i);
        int i0 = ib * 4;
        int j_end = (jb + 1) * NB < N ? (jb + 1) * NB : N;
        for (int j0 = jb * NB; j0 < j_end; j0 += 4) {
            v8f acc[4][4];
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) acc[a][b] = (v8f){0, 0, 0, 0, 0, 0, 0, 0};
            const float* ap[4];
            const float* bp[4];
            for (int a = 0; a < 4; ++a) ap[a] = A + (long)((i0 + a) < n ? (i0 + a) : (n - 1)) * lda;
            for (int b = 0; b < 4; ++b) bp[b] = B + (long)((j0 + b) < j_end ? (j0 + b) : (j_end - 1)) * ldb;
            int kk = 0;
            for (; kk + 8 <= K; kk += 8) {
                v8f av[4], bv[4];
                for (int a = 0; a < 4; ++a) av[a] = ld8(ap[a] + kk);
                for (int b = 0; b < 4; ++b) bv[b] = ld8(bp[b] + kk);
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * bv[b];
            }
            for (int a = 0; a < 4; ++a) {
                if (i0 + a >= n) break;
                for (int b = 0; b < 4; ++b) {
                    if (j0 + b >= j_end) break;
                    float s = hsum8(acc[a][b]);
                    for (int r = kk; r < K; ++r) s += ap[a][r] * bp[b][r];
                    C[(long)(i0 + a) * ldc + j0 + b] = s;
                }
            }
        }
    }
}

static inline float silu(float g) { return g / (1.0f + expf(-g)); }

/* One expert over n coalesced rows: x [n,d] -> y [n,d]; w1,w3 [ff,d], w2 [d,ff].
 * h_out (nullable) receives the fp32 intermediate [n,ff]. */
void oracle_expert_ffn(const float* x, int n, int d, int ff, const float* w1, const float* w3, const float* w2,
                       float* y, float* h_out) {
    if (n <= 0) return;
    float* g = (float*)malloc(sizeof(float) * (size_t)n * ff);
    float* u = (float*)malloc(sizeof(float) * (size_t)n * ff);
    gemm_nt(x, d, w1, d, g, ff, n, ff, d);
    gemm_nt(x, d, w3, d, u, ff, n, ff, d);
#pragma omp parallel for
    for (long i = 0; i < (long)n * ff; ++i) g[i] = silu(g[i]) * u[i];
    if (h_out) memcpy(h_out, g, sizeof(float) * (size_t)n * ff);
    gemm_nt(g, ff, w2, ff, y, d, n, d, ff);
    free(g);
    free(u);
}

/* All experts over a permuted batch: rows [offsets[e], offsets[e]+counts[e]) of
 * x_perm belong to expert e.  Weights are stacked per expert: w1/w3 [E,ff,d],
 * w2 [E,d,ff].  Padding rows of y_perm are left untouched. */
void oracle_grouped_ffn(const float* x_perm, const int32_t* offsets, const int32_t* counts, int E, int d, int ff,
                        const float* w1, const float* w3, const float* w2, float* y_perm) {
    for (int e = 0; e < E; ++e) {
        long r0 = offsets[e];
        oracle_expert_ffn(x_perm + r0 * d, counts[e], d, ff, w1 + (long)e * ff * d, w3 + (long)e * ff * d,
                          w2 + (long)e * d * ff, y_perm + r0 * d, NULL);
    }
}

/* gather rows: x_perm[dst[t*k+j]] = x[t] */
void oracle_gather(const float* x, int T, int d, const int32_t* dst, int k, float* x_perm) {
#pragma omp parallel for
    for (long t = 0; t < T; ++t)
        for (int j = 0; j < k; ++j) memcpy(x_perm + (long)dst[t * k + j] * d, x + t * d, sizeof(float) * d);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
