/*
 * CPU ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product path (paper_2605_17889_b200) never does.
 *
 * Router, top-k, stable permutation and combine for the coalesced MoE expert
 * stage, restated in plain C.  The reference (moeplan) has NO router, permute or
 * combine code; the semantics restated here come from:
 *   - PAPER.md:67          top-k routing of each token over the N-expert pool;
 *   - PAPER.md:191,282     OP3 runs coalesced over the ordinary batch B;
 *   - eas.py:364-374       ties broken toward the lower expert index (the
 *                          reference's own tie convention, reused for top-k);
 *   - public Mixtral config (renormalised softmax over the k selected logits)
 *     and DeepSeek-V2 config (full softmax, norm_topk_prob=false) — these are
 *     ASSUMPTIONS, not reference code.
 * Parity of routing/permutation against the reference is therefore UNPINNED by
 * the reference itself; the restatement is cross-checked against an independent
 * numpy float64 implementation and committed golden vectors (tests/golden/).
 *
 * Canonical summation order (shared bit-for-bit with the CUDA router,
 * paper_2605_17889_b200/csrc/router.cu): logit(t,e) is computed by 32 "lanes";
 * lane l owns the 8-element chunks c = 32*j + l (j = 0,1,...) of the d-vector
 * and accumulates acc = fmaf(x[8c+q], wg[8c+q], acc) for j ascending, q = 0..7
 * ascending, starting from +0.0f.  The 32 partials are then combined by an xor
 * butterfly: for off in 16,8,4,2,1: p[l] = p[l] + p[l^off].  The result is p[0].
 *
 * Compiled with -ffp-contract=off (see Makefile) so no add is fused.  The
 * token loop is OpenMP-parallel (tokens are independent; per-token arithmetic
 * is unchanged), so full 262,144-token batches are checked in seconds.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LANES 32

float oracle_router_logit(const float* x, const float* wg, int d) {
    float p[LANES];
    for (int l = 0; l < LANES; ++l) {
        float acc = 0.0f;
        for (int j = 0;; ++j) {
            long s = 8L * (LANES * (long)j + l);
            if (s >= d) break;
            for (int q = 0; q < 8; ++q) acc = fmaf(x[s + q], wg[s + q], acc);
        }
        p[l] = acc;
    }
    for (int off = 16; off >= 1; off >>= 1) {
        float np_[LANES];
        for (int l = 0; l < LANES; ++l) np_[l] = p[l] + p[l ^ off];
        memcpy(p, np_, sizeof(p));
    }
    return p[0];
}

/* One token: logits -> top-k indices and weights; selected experts are
 * added to cnt.  mode 0: Mixtral (softmax over the k selected logits, i.e.
 * renormalised top-k); mode 1: DeepSeek-V2 (softmax over all E, selected
 * probabilities, no renorm).  Selection is on logits (softmax is monotone);
 * strict '>' keeps the lower index on ties. */
static void route_token(const float* xt, const float* wg, int d, int E, int k, int mode, float* logits_out,
                        int32_t* idx, float* w, int32_t* cnt) {
    float lg[256];
    unsigned char taken[256];
    for (int e = 0; e < E; ++e) {
        lg[e] = oracle_router_logit(xt, wg + (long)e * d, d);
        if (isnan(lg[e])) lg[e] = -INFINITY; /* NaN ranks below every number (GPU: nan_low) */
        if (logits_out) logits_out[e] = lg[e];
        taken[e] = 0;
    }
    for (int j = 0; j < k; ++j) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < E; ++e) {
            if (taken[e]) continue;
            if (best < 0 || lg[e] > bv) { best = e; bv = lg[e]; }
        }
        taken[best] = 1;
        idx[j] = best;
        cnt[best] += 1;
    }
    float m = lg[idx[0]];
    if (mode == 0) {
        float s = 0.0f;
        for (int j = 0; j < k; ++j) s = s + expf(lg[idx[j]] - m);
        for (int j = 0; j < k; ++j) w[j] = expf(lg[idx[j]] - m) / s;
    } else {
        float s = 0.0f;
        for (int e = 0; e < E; ++e) s = s + expf(lg[e] - m);
        for (int j = 0; j < k; ++j) w[j] = expf(lg[idx[j]] - m) / s;
    }
}

/* Tokens are independent: the token loop runs on OpenMP threads (each token's
 * arithmetic is unchanged; counts are integer sums, order-free).  x is fp32
 * (x_bf16 == NULL) or bf16 bit patterns (x == NULL), widened exactly. */
static int router_topk_impl(const float* x, const uint16_t* x_bf16, const float* wg, int T, int d, int E, int k,
                            int mode, float* logits_out, int32_t* idx, float* w, int32_t* counts) {
    if (T < 0 || d <= 0 || (d % 8) != 0 || E <= 0 || E > 256 || k <= 0 || k > E || (mode != 0 && mode != 1))
        return -1;
    for (int e = 0; e < E; ++e) counts[e] = 0;
#pragma omp parallel
    {
        int32_t cnt[256];
        for (int e = 0; e < E; ++e) cnt[e] = 0;
        float* row = x_bf16 ? (float*)malloc(sizeof(float) * (size_t)d) : NULL;
#pragma omp for schedule(static)
        for (long t = 0; t < T; ++t) {
            const float* xt;
            if (x_bf16) {
                const uint16_t* src = x_bf16 + t * (long)d;
                for (int i = 0; i < d; ++i) {
                    uint32_t u = (uint32_t)src[i] << 16;
                    memcpy(row + i, &u, 4);
                }
                xt = row;
            } else {
                xt = x + t * (long)d;
            }
            route_token(xt, wg, d, E, k, mode, logits_out ? logits_out + t * E : NULL, idx + t * k, w + t * k, cnt);
        }
#pragma omp critical
        for (int e = 0; e < E; ++e) counts[e] += cnt[e];
        free(row);
    }
    return 0;
}

/* Returns 0, or -1 on invalid arguments. */
int oracle_router_topk(const float* x, const float* wg, int T, int d, int E, int k, int mode,
                       float* logits_out /* nullable [T,E] */, int32_t* idx, float* w,
                       int32_t* counts /* [E], zeroed here */) {
    return router_topk_impl(x, NULL, wg, T, d, E, k, mode, logits_out, idx, w, counts);
}

/* Same over bf16 tokens (bit patterns), e.g. a full 262,144-token batch
 * without a 4-byte copy of it. */
int oracle_router_topk_bf16(const uint16_t* x, const float* wg, int T, int d, int E, int k, int mode,
                            float* logits_out, int32_t* idx, float* w, int32_t* counts) {
    return router_topk_impl(NULL, x, wg, T, d, E, k, mode, logits_out, idx, w, counts);
}

/* Stable permutation by expert: within expert e the (t, j) pairs appear in
 * ascending token order (a token selects an expert at most once).  Segment e
 * starts at offsets[e]; segments are padded up to a multiple of tile_m rows. */
int oracle_permute(const int32_t* idx, int T, int k, int E, int tile_m, int32_t* offsets /*[E+1]*/,
                   int32_t* dst /*[T*k]*/) {
    if (T < 0 || k <= 0 || E <= 0 || tile_m <= 0) return -1;
    long cnt[256];
    if (E > 256) return -1;
    for (int e = 0; e < E; ++e) cnt[e] = 0;
    for (long i = 0; i < (long)T * k; ++i) {
        if (idx[i] < 0 || idx[i] >= E) return -1;
        cnt[idx[i]]++;
    }
    offsets[0] = 0;
    for (int e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + (int32_t)(((cnt[e] + tile_m - 1) / tile_m) * tile_m);
    long pos[256];
    for (int e = 0; e < E; ++e) pos[e] = offsets[e];
    for (long t = 0; t < T; ++t)
        for (int j = 0; j < k; ++j) {
            int e = idx[t * k + j];
            dst[t * k + j] = (int32_t)pos[e]++;
        }
    return 0;
}

/* out[t] = sum_{j<k} w[t,j] * y_perm[dst[t,j]]  (+ shared[t]), fp32, j ascending. */
void oracle_combine(const float* y_perm, const int32_t* dst, const float* w, int T, int k, int d,
                    const float* shared /* nullable */, float* out) {
    for (long t = 0; t < T; ++t) {
        float* o = out + t * (long)d;
        for (int c = 0; c < d; ++c) {
            float acc = 0.0f;
            for (int j = 0; j < k; ++j) acc = acc + w[t * k + j] * y_perm[(long)dst[t * k + j] * d + c];
            if (shared) acc = acc + shared[t * (long)d + c];
            o[c] = acc;
        }
    }
}
