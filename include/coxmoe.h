/*
 * coxmoe.h — C ABI of libcoxmoe.so, the B200 (sm_100a) coalesced MoE expert stage.
 *
 * The reference (arxiv/paper_2605_17889, package `moeplan`) has no FFI layer: its
 * expert stage exists only as the analytical row
 *     expert_stage_parts(strategy, phase, system, model, batch, activation_map, coalesced)
 *         (pkg/src/moeplan/costmodel.py:225-275)
 * and its OP3 accounting (workload.py:156-165).  Each entry point below is one
 * stage of the execution that row models; the Python host layer
 * (paper_2605_17889_b200/executor.py) binds them with ctypes and mirrors the
 * reference's types and error behaviour (ValueError on invalid input,
 * costmodel.py:92-97, workload.py:157-158).  See INTEGRATION.md.
 *
 * Conventions
 *   - All tensor arguments are DEVICE pointers owned by the caller; the library
 *     never allocates device memory on these paths.  Work is stream-ordered on
 *     the given cudaStream_t (passed as void* so no CUDA header is required).
 *   - Row-major, contiguous.  bf16 = IEEE bfloat16 bit pattern (uint16).
 *   - Return 0 on success, COX_EINVAL (-1) for invalid shapes/alignment,
 *     COX_ECUDA (-2) for a CUDA error, COX_EUNSUPPORTED (-3) for an unsupported
 *     device (anything but sm_100).  cox_last_error() returns a thread-local
 *     message for the last failure.
 */
#ifndef COXMOE_H
#define COXMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COX_OK 0
#define COX_EINVAL (-1)
#define COX_ECUDA (-2)
#define COX_EUNSUPPORTED (-3)

#define COX_DTYPE_F32 0
#define COX_DTYPE_BF16 1

#define COX_ROUTE_MIXTRAL 0  /* softmax over the k selected logits (renormalised) */
#define COX_ROUTE_DEEPSEEK 1 /* softmax over all E, selected probabilities, no renorm */

/* Library / device checks. */
const char* cox_last_error(void);
int cox_version(void);
/* 0 if the current device is sm_100 (B200) and the kernels can launch. */
int cox_device_check(void);

/* K1 — router.  Replaces the top-k routing of PAPER.md:67 that the reference
 * only accounts for analytically (workload.py:156-165 — OP3's D_X term).
 *   x      [T, d]  (x_dtype: COX_DTYPE_BF16 or COX_DTYPE_F32), d % 8 == 0
 *   wg     [E, d]  router weight (wg_dtype: COX_DTYPE_BF16 or COX_DTYPE_F32)
 *   idx    [T, k]  int32 expert ids, descending logit, ties -> lower index
 *                  (eas.py:364-374 convention)
 *   w      [T, k]  fp32 routing weights
 *   counts [E]     int32 tokens per expert (the per-batch analogue of eas.probe,
 *                  eas.py:346-356)
 *   workspace      >= cox_router_workspace_bytes(T, E) bytes of device memory,
 *                  ZEROED ONCE when allocated (the kernels leave it zeroed);
 *                  one workspace per concurrently executing launch.
 * 1 <= k <= min(E, 8), E <= 256.  Logits are fp32 in the canonical order shared
 * with the CPU oracle, so idx is bit-exact.  A bf16 wg (the checkpoint dtype of
 * Mixtral/DeepSeek routers) gives the same logits as the same values in fp32
 * (bf16 x bf16 products are exact).  bf16 x and wg, E >= 32, T >= 18944: the
 * logits are screened on the tensor cores (fp32 accumulation, per-token error
 * bound) and only the candidates that can reach the top-k are recomputed in the
 * canonical order: same idx and counts; COX_ROUTE_MIXTRAL weights identical;
 * COX_ROUTE_DEEPSEEK weights within ~1e-6 relative (their full-softmax
 * denominator uses the screened logits of the non-candidates). */
size_t cox_router_workspace_bytes(int T, int E);
int cox_router_topk(const void* x, int x_dtype, const void* wg, int wg_dtype, int T, int d, int E, int k, int mode,
                    int32_t* idx, float* w, int32_t* counts, void* workspace, size_t workspace_bytes, void* stream);

/* K2 — stable permutation by expert (coalesced dispatch).
 *   idx      [T, k] expert ids in [0, E) (anything else is dropped)
 *   x        [T, d] bf16, d % 8 == 0
 *   offsets  [E+1]  int32 segment starts (segments padded to tile_m rows)
 *   dst      [T, k] int32 row of x_perm that holds (t, j)
 *   x_perm   [rows_cap, d] bf16, rows_cap >= T*k + E*(tile_m-1); NULL: compute
 *            offsets and dst only (the fused EP dispatch moves the rows itself)
 *   row_tokens [rows_cap] (nullable): the source token of every permuted row
 *            (the gathered-B decode path of cox_small_expert_ffn)
 *   workspace of cox_permute_workspace_bytes(T, E) bytes. */
size_t cox_permute_workspace_bytes(int T, int E);
int cox_permute(const int32_t* idx, int T, int k, int E, int tile_m, const void* x, int d, int32_t* offsets,
                int32_t* dst, void* x_perm, long long rows_cap, int32_t* row_tokens, void* workspace, void* stream);

/* K3 — grouped SwiGLU expert GEMM over the coalesced batch:
 *   h[r, :] = silu(x_perm[r] W1_e^T) * (x_perm[r] W3_e^T) for r in segment e.
 * offsets [E+1] are the segments of cox_permute.  Runs the groups
 * group_experts[0..n_groups) (<= 64, each in [0, E)); w13[g] is the DEVICE
 * pointer of that group's interleaved weight [2*ff, d] bf16 (128-row blocks:
 * W1 rows 128i..128i+127, then W3 rows 128i..128i+127; see
 * cox_interleave_w13).  Resident and streamed (cold) experts are just
 * different groups/pointers, so a cold expert's GEMM can be issued separately
 * once its copy has landed.  max_ctas: the persistent kernel uses at most
 * max_ctas SMs (even, >= 2; 0 = all), so two grouped GEMMs can run
 * concurrently on different streams.  d % 64 == 0, ff % 128 == 0. */
int cox_grouped_swiglu(const void* x_perm, long long rows_cap, const int32_t* offsets, int E, int n_groups,
                       const int32_t* group_experts, const void* const* w13, int d, int ff, void* h, int max_ctas,
                       void* stream);

/* K3 with the permuted rows gathered from x (no x_perm copy): identical
 * results to cox_grouped_swiglu on x_perm[r] = x[row_tokens[r]].  row_tokens
 * [T*k]: the source token of every permuted row (cox_permute with x_perm ==
 * NULL writes it, with offsets and dst and no row copy).  Four extra warps per
 * CTA fill the A stages by cp.async in the 128B-swizzled layout the tensor
 * core reads; B (the weights) still streams by TMA.  Replaces the permute's
 * row copy (T*k*d*2 bytes written, T*d*2 read) in the reference's
 * expert:dispatch step (sim.py:149-202, costmodel.py:266-273).
 * d % 64 == 0, ff % 128 == 0. */
int cox_grouped_swiglu_gather(const void* x, long long T, const int32_t* row_tokens, const int32_t* offsets, int E,
                              int n_groups, const int32_t* group_experts, const void* const* w13, int d, int ff,
                              void* h, int max_ctas, void* stream);

/* K4 — grouped down projection: y_perm[r] = h[r] W2_e^T.  w2[g]: [d, ff] bf16.
 * Same grouping arguments as cox_grouped_swiglu.  ff % 64 == 0, d % 256 == 0. */
int cox_grouped_down(const void* h, long long rows_cap, const int32_t* offsets, int E, int n_groups,
                     const int32_t* group_experts, const void* const* w2, int ff, int d, void* y_perm, int max_ctas,
                     void* stream);

/* K3+K4(+K5) for decode-size batches: ONE
 * persistent, weight-streaming launch runs the SwiGLU and the down projection
 * of every group, the shared experts of a DeepSeek-style layer (one more
 * dense group over x) and, optionally, the weighted combine.  Swap-AB tcgen05
 * tiles: 128 weight rows x up to 64 tokens, so the weights stream from HBM
 * once while the tensor pipe idles; a group's down tiles start as soon as its
 * SwiGLU tiles are stored, and the CTA that stores the last down tile of a
 * 128-column block combines that block for every token (device-side
 * counters, no launch boundaries).
 *   x [T, d]             the step's tokens (shared-expert input; gather source)
 *   row_tokens           source token of every permuted row (cox_permute);
 *                        used when x_perm == NULL: the routed rows are gathered
 *                        from x by TMA tile::gather4, no x_perm copy
 *   x_perm [rows_cap, d] materialised permuted rows (or NULL, see above)
 *   offsets [E+1] / group_experts / w13 / w2 / h / y_perm as for
 *                        cox_grouped_swiglu / cox_grouped_down
 *   w13_shared [2*ff_shared, d] (interleaved), w2_shared [d, ff_shared],
 *   h_shared [T, ff_shared], y_shared [T, d]   (w13_shared == NULL: none)
 *   dst [T, k], w [T, k], out [T, d] bf16: fused combine
 *                        out[t] = sum_j w[t,j] y_perm[dst[t,j]] (+ y_shared[t]),
 *                        bit-identical to cox_combine (out == NULL: skipped)
 * Same results as cox_grouped_swiglu + cox_grouped_down (+ cox_combine) up to
 * fp32 summation order, for any segment length; efficient while segments
 * have <= 64 rows.  d % 128 == 0, ff % 128 == 0, ff_shared % 128 == 0,
 * n_groups <= 64. */
int cox_small_expert_ffn(const void* x, int T, const int32_t* row_tokens, const void* x_perm, long long rows_cap,
                         const int32_t* offsets, int E, int n_groups, const int32_t* group_experts,
                         const void* const* w13, const void* const* w2, int d, int ff, void* h, void* y_perm,
                         const void* w13_shared, const void* w2_shared, int ff_shared, void* h_shared,
                         void* y_shared, const int32_t* dst, const float* w, int k, void* out, void* stream);

/* Same decode-size expert stage straight from the router's output (no
 * permute launch): segments from counts[E] (expert-ascending, written to
 * offsets [E+1] if non-NULL), each routed SwiGLU tile collects its expert's
 * tokens from idx [T, k] and gathers their rows from x, the combine rows are
 * written to dst [T, k] (same order as cox_permute).  Experts 0..E-1 are the
 * groups; h [T*k, ff], y_perm [T*k, d]; out [T, d] bf16 (fused combine).
 * T <= 256, E <= 64, d % 128 == 0, ff % 128 == 0. */
int cox_small_expert_ffn_idx(const void* x, int T, const int32_t* idx, const int32_t* counts, int E,
                             const float* w, int k, const void* const* w13, const void* const* w2, int d, int ff,
                             void* h, void* y_perm, const void* w13_shared, const void* w2_shared, int ff_shared,
                             void* h_shared, void* y_shared, int32_t* dst, int32_t* offsets, void* out,
                             void* stream);

/* The whole MoE layer for a decode step (T <= 64 tokens, E <= 64 experts) in
 * ONE launch: router (bf16 wg, canonical order: idx bit-exact with
 * cox_router_topk), SwiGLU + down projection of EVERY expert over all T tokens
 * (the step streams every expert's weights anyway; the idle tensor pipe
 * computes the unrouted pairs, so routing is off the critical path), shared
 * experts and the weighted combine of the routed pairs.
 *   x [T, d] bf16; wg [E, d] bf16; w13[e] [2 ff, d] (interleaved), w2[e] [d, ff]
 *   h [E*T, ff], y [E*T, d] bf16 scratch (expert e's rows at e*T)
 *   optional shared experts: w13_shared [2 ff_shared, d], w2_shared [d, ff_shared],
 *   h_shared [T, ff_shared], y_shared [T, d]
 *   idx [T, k] int32, w [T, k] fp32: the routing; out [T, d] bf16.
 * Replaces the decode-phase `expert_stage_parts` (costmodel.py:368).
 * d % 128 == 0, ff % 128 == 0, ff_shared % 128 == 0. */
int cox_decode_moe(const void* x, int T, const void* wg, int E, int k, int mode, const void* const* w13,
                   const void* const* w2, int d, int ff, const void* w13_shared, const void* w2_shared, int ff_shared,
                   void* h, void* y, void* h_shared, void* y_shared, int32_t* idx, float* w, void* out,
                   void* stream);

/* K6' — cold-expert fetch decided on the device (decode-size steps,
 * SURVEY.md §8 f1).  For each listed cold expert i
 * (expert_ids[i] in [0, E)), if counts[expert_ids[i]] > 0 (the layer's router
 * routed tokens to it) copy `bytes` from pinned host memory host_src[i] to the
 * device slot dst[i]; untouched cold experts cost no PCIe bytes and the
 * decision needs no host round trip (graph-capturable).  Replaces the
 * unconditional `mig_load` of costmodel.py:252.  fetched [n] (nullable): 1 for
 * every entry copied by this launch.  n <= 64, max_ctas: CTAs used (0 = one
 * per SM). */
int cox_fetch_experts(const int32_t* counts, int E, int n, const int32_t* expert_ids, const void* const* host_src,
                      void* const* dst, const long long* bytes, int max_ctas, int32_t* fetched, void* stream);

/* K5 — weighted top-k combine back to token order (+ optional shared-expert
 * output, DeepSeek-V2):  out[t] = sum_j w[t,j] * y_perm[dst[t,j]] (+ shared[t]).
 * out/shared dtype = out_dtype (bf16 or fp32). */
int cox_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared_out,
                void* out, int out_dtype, void* stream);

/* K7' — fused expert-parallel dispatch/combine over NVLink peer memory
 * (replaces the NCCL all-to-all pair of the EP path; see csrc/ep.cu).  Rank r
 * of `world` owns experts [r*E/world, (r+1)*E/world).  Pointer tables are
 * DEVICE arrays of `world` peer addresses (e.g. CUDA symmetric memory).
 *   cox_ep_counts_put: counts[E] -> counts_all[rank][E] on every peer.
 *   cox_ep_offsets:    counts_all[world][E] -> my receive segments
 *                      recv_seg[E/world + 1] (one per local expert: all
 *                      sources' rows, source-rank order; clamped to cap) and
 *                      send_base[E] (row of my first pair of expert e on its
 *                      owner); overflow[0] = the largest receive count of any
 *                      owner if it exceeds cap, else 0 (rewritten per launch;
 *                      identical on every rank).
 *   cox_ep_dispatch:   stores x[t] into the owners' receive buffers at
 *                      send_base[e] + (dst_local - offsets_local[e]);
 *                      route_row[T,k] records the row for the combine (-1:
 *                      beyond cap, dropped).
 *   cox_ep_combine:    out[t] = sum_j w[t,j] * y_owner[route_row[t,j]] (bf16;
 *                      route_row < 0 contributes nothing).
 * dst_local/offsets_local come from cox_permute (x_perm may be NULL then). */
int cox_ep_counts_put(const int32_t* counts, int E, int rank, int world, int32_t* const* peer_counts, void* stream);
int cox_ep_offsets(const int32_t* counts_all, int world, int E, int rank, long long cap, int32_t* recv_seg,
                   int32_t* send_base, int32_t* overflow, void* stream);
int cox_ep_dispatch(const int32_t* idx, const int32_t* dst_local, const int32_t* offsets_local,
                    const int32_t* send_base, int T, int k, int E, int world, long long cap, const void* x, int d,
                    void* const* peer_recv, int32_t* route_row, void* stream);
int cox_ep_combine(const int32_t* idx, const int32_t* route_row, const float* w, int T, int k, int d, int E,
                   int world, const void* const* peer_y, void* out, void* stream);

/* Layout helper: interleave W1 [ff, d] and W3 [ff, d] (bf16, device) into the
 * K3 layout [2*ff, d] (device).  ff % 128 == 0. */
int cox_interleave_w13(const void* w1, const void* w3, int ff, int d, void* w13, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COXMOE_H */
