// C ABI (include/coxmoe.h): argument validation, error reporting, dispatch.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/coxmoe.h"
#include "common.cuh"

namespace cox {
size_t router_workspace_bytes(int T, int E);
int launch_router(const void* x, int x_is_bf16, const void* wg, int wg_is_bf16, int T, int d, int E, int k,
                  int mode, int32_t* idx, float* w, int32_t* counts, void* ws, int tc, int e8, cudaStream_t s);
size_t permute_workspace_bytes(int T, int E);
int launch_permute(const int32_t* idx, int T, int k, int E, int tile_m, const void* x, int d, int32_t* offsets,
                   int32_t* dst, void* x_perm, void* workspace, cudaStream_t s, int32_t* row_tokens = nullptr,
                   long long rows_cap = 0);
int launch_grouped_gemm(int epi, const void* A, long long rows_cap, int K, const int32_t* offsets, int n_groups,
                        const int32_t* group_expert, const void* const* B, int N, void* out, long long ldo,
                        int max_ctas, cudaStream_t s, const void* gx = nullptr, const int32_t* row_tokens = nullptr,
                        long long gx_ld = 0);
struct SmallDense {
  const void* wg;
  int E, mode;
  int32_t* idx;
  float* w;
};
struct SmallIdx {
  const int32_t* idx;
  const int32_t* counts;
  int E;
  int32_t* dst_out;
  int32_t* offsets_out;
};
int launch_small_ffn(const void* x, int T, const int32_t* row_tokens, const void* act, long long rows_cap,
                     const int32_t* offsets, int n_groups, const int32_t* group_expert, const void* const* w13,
                     const void* const* w2, int d, int ff, void* h, void* y, const void* w13s, const void* w2s,
                     int ffs, void* hs, void* ys, const int32_t* cdst, const float* cw, int k, void* out,
                     int phases, cudaStream_t s, const SmallDense* dense = nullptr,
                     const SmallIdx* fromidx = nullptr);
int launch_fetch_experts(const int32_t* counts, int n, const int32_t* expert_ids, const void* const* src,
                         void* const* dst, const long long* bytes, int max_ctas, int32_t* fetched, cudaStream_t s);
int launch_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared,
                   void* out, int out_is_bf16, cudaStream_t s);

int launch_ep_counts_put(const int32_t* counts, int E, int rank, int world, int32_t* const* peer_counts,
                         cudaStream_t s);
int launch_ep_offsets(const int32_t* counts_all, int G, int E, int rank, long long cap, int32_t* recv_seg,
                      int32_t* send_base, int32_t* overflow, cudaStream_t s);
int launch_ep_dispatch(const int32_t* idx, const int32_t* dst_local, const int32_t* offsets_local,
                       const int32_t* send_base, int T, int k, int L, long long cap, const void* x, int d,
                       void* const* peer_recv, int32_t* route_row, cudaStream_t s);
int launch_ep_combine(const int32_t* idx, const int32_t* route_row, const float* w, int T, int k, int d, int L,
                      const void* const* peer_y, void* out, cudaStream_t s);

__global__ void interleave_w13_kernel(const uint4* __restrict__ w1, const uint4* __restrict__ w3, int ff, int d,
                                      uint4* __restrict__ w13) {
  // row r of w13: block b = r / 128; source = (b even ? w1 : w3), row (b/2)*128 + r%128
  const long vec_per_row = d / 8;
  const long total = 2L * ff * vec_per_row;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long r = i / vec_per_row, c = i % vec_per_row;
    const long b = r / 128, rr = (b / 2) * 128 + (r % 128);
    const uint4* src = (b & 1) ? w3 : w1;
    w13[i] = src[rr * vec_per_row + c];
  }
}
}  // namespace cox

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_status(int rc, const char* what) {
  if (rc == 0) return 0;
  if (rc == COX_ECUDA) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cox::g_last_cuda_error;
    cox::g_last_cuda_error = cudaSuccess;
    return fail(COX_ECUDA, "%s: CUDA error: %s", what, cudaGetErrorString(e));
  }
  if (rc == COX_EINVAL) return fail(COX_EINVAL, "%s: invalid argument (tensor map encode rejected the operand)", what);
  return fail(rc, "%s: error %d", what, rc);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" {

const char* cox_last_error(void) { return g_err.c_str(); }

int cox_version(void) { return 3; }

int cox_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(COX_ECUDA, "no CUDA device");
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(COX_EUNSUPPORTED, "libcoxmoe is built for sm_100a only; device is sm_%d%d", major, minor);
  return 0;
}

size_t cox_router_workspace_bytes(int T, int E) { return cox::router_workspace_bytes(T, E); }

// COX_ROUTER (A/B and tests): "generic" = the CUDA-core kernels of router.cu only
// (no tensor-core screen, no E <= 8 TMA kernel); "tc" = the tensor-core screen
// whenever the shape allows it; unset = automatic choice.
static int router_env() {
  static const int m = [] {
    const char* e = getenv("COX_ROUTER");
    if (!e) return 0;
    if (!strcmp(e, "generic")) return 1;
    if (!strcmp(e, "tc")) return 2;
    return 0;
  }();
  return m;
}

int cox_router_topk(const void* x, int x_dtype, const void* wg, int wg_dtype, int T, int d, int E, int k, int mode,
                    int32_t* idx, float* w, int32_t* counts, void* workspace, size_t workspace_bytes,
                    void* stream) {
  const char* fn = "cox_router_topk";
  if (T < 0 || d <= 0 || d % 8 || E <= 0 || E > 256 || k < 1 || k > E || k > 8)
    return fail(COX_EINVAL, "%s: need T>=0, d%%8==0, 1<=k<=min(E,8), E<=256 (T=%d d=%d E=%d k=%d)", fn, T, d, E, k);
  if (mode != COX_ROUTE_MIXTRAL && mode != COX_ROUTE_DEEPSEEK) return fail(COX_EINVAL, "%s: bad mode %d", fn, mode);
  if (x_dtype != COX_DTYPE_BF16 && x_dtype != COX_DTYPE_F32) return fail(COX_EINVAL, "%s: bad x_dtype", fn);
  if (wg_dtype != COX_DTYPE_BF16 && wg_dtype != COX_DTYPE_F32) return fail(COX_EINVAL, "%s: bad wg_dtype", fn);
  if (!counts || (T > 0 && (!x || !wg || !idx || !w))) return fail(COX_EINVAL, "%s: null pointer", fn);
  if (!aligned16(x) || !aligned16(wg)) return fail(COX_EINVAL, "%s: x and wg must be 16-byte aligned", fn);
  const size_t need = cox::router_workspace_bytes(T, E);
  if (!workspace || !aligned16(workspace) || workspace_bytes < need)
    return fail(COX_EINVAL, "%s: workspace of %zu bytes (16-byte aligned) required, got %zu", fn, need,
                workspace_bytes);
  int rc = cox::launch_router(x, x_dtype == COX_DTYPE_BF16, wg, wg_dtype == COX_DTYPE_BF16, T, d, E, k, mode, idx, w,
                              counts, workspace, router_env() == 1 ? 0 : router_env() == 2 ? 1 : -1,
                              router_env() == 1 ? 0 : 1, static_cast<cudaStream_t>(stream));
  return cuda_status(rc, fn);
}

size_t cox_permute_workspace_bytes(int T, int E) { return cox::permute_workspace_bytes(T, E); }

int cox_permute(const int32_t* idx, int T, int k, int E, int tile_m, const void* x, int d, int32_t* offsets,
                int32_t* dst, void* x_perm, long long rows_cap, int32_t* row_tokens, void* workspace, void* stream) {
  if (T < 0 || k < 1 || k > 8 || E < 1 || E > 256 || tile_m < 1 || d <= 0 || d % 8)
    return fail(COX_EINVAL, "cox_permute: need 1<=k<=8, 1<=E<=256, tile_m>=1, d%%8==0");
  if (rows_cap < (long long)T * k + (long long)E * (tile_m - 1))
    return fail(COX_EINVAL, "cox_permute: rows_cap %lld < T*k + E*(tile_m-1) = %lld", rows_cap,
                (long long)T * k + (long long)E * (tile_m - 1));
  if (!aligned16(x) || (x_perm && !aligned16(x_perm)))
    return fail(COX_EINVAL, "cox_permute: x/x_perm must be 16-byte aligned");
  if (!workspace || !offsets) return fail(COX_EINVAL, "cox_permute: null workspace/offsets");
  int rc = cox::launch_permute(idx, T, k, E, tile_m, x, d, offsets, dst, x_perm, workspace,
                               static_cast<cudaStream_t>(stream), row_tokens, rows_cap);
  return cuda_status(rc, "cox_permute");
}

// Every group's expert id must name a segment of offsets[E + 1]: the kernels
// read offsets[e] and offsets[e + 1].
static int check_groups(const char* fn, int E, int n_groups, const int32_t* group_experts, const void* const* w) {
  if (n_groups < 0 || n_groups > 64) return fail(COX_EINVAL, "%s: n_groups must be in [0, 64]", fn);
  if (n_groups > 0 && (E < 1 || !group_experts || !w)) return fail(COX_EINVAL, "%s: need E >= 1 and the group tables", fn);
  for (int g = 0; g < n_groups; ++g) {
    if (group_experts[g] < 0 || group_experts[g] >= E)
      return fail(COX_EINVAL, "%s: group %d names expert %d outside [0, %d)", fn, g, group_experts[g], E);
    if (!w[g] || !aligned16(w[g])) return fail(COX_EINVAL, "%s: weight pointer %d null or unaligned", fn, g);
  }
  return 0;
}

int cox_grouped_swiglu(const void* x_perm, long long rows_cap, const int32_t* offsets, int E, int n_groups,
                       const int32_t* group_experts, const void* const* w13, int d, int ff, void* h, int max_ctas,
                       void* stream) {
  const char* fn = "cox_grouped_swiglu";
  if (d <= 0 || d % 64 || ff <= 0 || ff % 128)
    return fail(COX_EINVAL, "%s: need d%%64==0 and ff%%128==0 (d=%d ff=%d)", fn, d, ff);
  if (rows_cap < 1) return fail(COX_EINVAL, "%s: rows_cap < 1", fn);
  if (max_ctas < 0 || max_ctas == 1) return fail(COX_EINVAL, "%s: max_ctas must be 0 or >= 2", fn);
  if (!aligned16(x_perm) || !aligned16(h)) return fail(COX_EINVAL, "%s: unaligned x_perm/h", fn);
  if (int rc = check_groups(fn, E, n_groups, group_experts, w13)) return rc;
  if (n_groups > 0 && (!x_perm || !h || !offsets)) return fail(COX_EINVAL, "%s: null x_perm/h/offsets", fn);
  int rc = cox::launch_grouped_gemm(0, x_perm, rows_cap, d, offsets, n_groups, group_experts, w13, 2 * ff, h, ff,
                                    max_ctas, static_cast<cudaStream_t>(stream));
  return cuda_status(rc, fn);
}

int cox_grouped_swiglu_gather(const void* x, long long T, const int32_t* row_tokens, const int32_t* offsets, int E,
                              int n_groups, const int32_t* group_experts, const void* const* w13, int d, int ff,
                              void* h, int max_ctas, void* stream) {
  const char* fn = "cox_grouped_swiglu_gather";
  if (d <= 0 || d % 64 || ff <= 0 || ff % 128)
    return fail(COX_EINVAL, "%s: need d%%64==0 and ff%%128==0 (d=%d ff=%d)", fn, d, ff);
  if (T < 0) return fail(COX_EINVAL, "%s: T < 0", fn);
  if (max_ctas < 0 || max_ctas == 1) return fail(COX_EINVAL, "%s: max_ctas must be 0 or >= 2", fn);
  if (!aligned16(x) || !aligned16(h)) return fail(COX_EINVAL, "%s: unaligned x/h", fn);
  if (int rc = check_groups(fn, E, n_groups, group_experts, w13)) return rc;
  if (n_groups > 0 && (!x || !h || !offsets || !row_tokens))
    return fail(COX_EINVAL, "%s: null x/h/offsets/row_tokens", fn);
  int rc = cox::launch_grouped_gemm(0, nullptr, 0, d, offsets, n_groups, group_experts, w13, 2 * ff, h, ff, max_ctas,
                                    static_cast<cudaStream_t>(stream), x, row_tokens, d);
  return cuda_status(rc, fn);
}

int cox_grouped_down(const void* h, long long rows_cap, const int32_t* offsets, int E, int n_groups,
                     const int32_t* group_experts, const void* const* w2, int ff, int d, void* y_perm, int max_ctas,
                     void* stream) {
  const char* fn = "cox_grouped_down";
  if (d <= 0 || d % 256 || ff <= 0 || ff % 64)
    return fail(COX_EINVAL, "%s: need d%%256==0 and ff%%64==0 (d=%d ff=%d)", fn, d, ff);
  if (rows_cap < 1) return fail(COX_EINVAL, "%s: rows_cap < 1", fn);
  if (max_ctas < 0 || max_ctas == 1) return fail(COX_EINVAL, "%s: max_ctas must be 0 or >= 2", fn);
  if (!aligned16(h) || !aligned16(y_perm)) return fail(COX_EINVAL, "%s: unaligned h/y_perm", fn);
  if (int rc = check_groups(fn, E, n_groups, group_experts, w2)) return rc;
  if (n_groups > 0 && (!h || !y_perm || !offsets)) return fail(COX_EINVAL, "%s: null h/y_perm/offsets", fn);
  int rc = cox::launch_grouped_gemm(1, h, rows_cap, ff, offsets, n_groups, group_experts, w2, d, y_perm, d, max_ctas,
                                    static_cast<cudaStream_t>(stream));
  return cuda_status(rc, fn);
}

int cox_small_expert_ffn(const void* x, int T, const int32_t* row_tokens, const void* x_perm, long long rows_cap,
                         const int32_t* offsets, int E, int n_groups, const int32_t* group_experts,
                         const void* const* w13, const void* const* w2, int d, int ff, void* h, void* y_perm,
                         const void* w13_shared, const void* w2_shared, int ff_shared, void* h_shared,
                         void* y_shared, const int32_t* dst, const float* w, int k, void* out, void* stream) {
  const char* fn = "cox_small_expert_ffn";
  if (T < 0 || d <= 0 || d % 128) return fail(COX_EINVAL, "%s: need T >= 0 and d %% 128 == 0 (d=%d)", fn, d);
  if (T > 0 && (!x || !aligned16(x))) return fail(COX_EINVAL, "%s: x null or unaligned", fn);
  if (n_groups > 0) {
    if (ff <= 0 || ff % 128) return fail(COX_EINVAL, "%s: need ff %% 128 == 0 (ff=%d)", fn, ff);
    if (rows_cap < 1 || !offsets) return fail(COX_EINVAL, "%s: rows_cap < 1 or null offsets", fn);
    if (!x_perm && !row_tokens) return fail(COX_EINVAL, "%s: need x_perm or row_tokens", fn);
    if (!h || !y_perm || !aligned16(x_perm) || !aligned16(h) || !aligned16(y_perm))
      return fail(COX_EINVAL, "%s: null or unaligned x_perm/h/y_perm", fn);
  }
  if (int rc = check_groups(fn, E, n_groups, group_experts, w13)) return rc;
  if (int rc = check_groups(fn, E, n_groups, group_experts, w2)) return rc;
  if (w13_shared) {
    if (ff_shared <= 0 || ff_shared % 128)
      return fail(COX_EINVAL, "%s: need ff_shared %% 128 == 0 (ff_shared=%d)", fn, ff_shared);
    if (!w2_shared || !h_shared || !y_shared || !aligned16(w13_shared) || !aligned16(w2_shared) ||
        !aligned16(h_shared) || !aligned16(y_shared))
      return fail(COX_EINVAL, "%s: null or unaligned shared-expert operand", fn);
  }
  if (out) {
    if (k < 1 || k > 8 || !dst || !w || !aligned16(out)) return fail(COX_EINVAL, "%s: fused combine needs 1<=k<=8, dst, w", fn);
  }
  int rc = cox::launch_small_ffn(x, T, row_tokens, x_perm, rows_cap, offsets, n_groups, group_experts, w13, w2, d, ff,
                                 h, y_perm, w13_shared, w2_shared, ff_shared, h_shared, y_shared, dst, w, k, out, 3,
                                 static_cast<cudaStream_t>(stream));
  return cuda_status(rc, fn);
}

int cox_small_expert_ffn_idx(const void* x, int T, const int32_t* idx, const int32_t* counts, int E,
                             const float* w, int k, const void* const* w13, const void* const* w2, int d, int ff,
                             void* h, void* y_perm, const void* w13_shared, const void* w2_shared, int ff_shared,
                             void* h_shared, void* y_shared, int32_t* dst, int32_t* offsets, void* out,
                             void* stream) {
  const char* fn = "cox_small_expert_ffn_idx";
  if (T < 1 || T > 256) return fail(COX_EINVAL, "%s: need 1 <= T <= 256 (T=%d)", fn, T);
  if (E < 1 || E > 64 || k < 1 || k > 8 || k > E) return fail(COX_EINVAL, "%s: need 1 <= k <= min(E, 8), E <= 64", fn);
  if (d <= 0 || d % 128 || ff <= 0 || ff % 128) return fail(COX_EINVAL, "%s: need d %% 128 == 0, ff %% 128 == 0", fn);
  if (!x || !idx || !counts || !w || !h || !y_perm || !dst || !out || !aligned16(x) || !aligned16(h) ||
      !aligned16(y_perm) || !aligned16(out))
    return fail(COX_EINVAL, "%s: null or unaligned operand", fn);
  if (w13_shared && (ff_shared <= 0 || ff_shared % 128 || !w2_shared || !h_shared || !y_shared ||
                     !aligned16(h_shared) || !aligned16(y_shared)))
    return fail(COX_EINVAL, "%s: bad shared-expert operands", fn);
  int32_t ids[64];
  for (int e = 0; e < E; ++e) ids[e] = e;
  if (int rc = check_groups(fn, E, E, ids, w13)) return rc;
  if (int rc = check_groups(fn, E, E, ids, w2)) return rc;
  cox::SmallIdx fi{idx, counts, E, dst, offsets};
  int rc = cox::launch_small_ffn(x, T, nullptr, nullptr, (long long)T * k, nullptr, E, ids, w13, w2, d, ff, h,
                                 y_perm, w13_shared, w2_shared, ff_shared, h_shared, y_shared, dst, w, k, out, 3,
                                 static_cast<cudaStream_t>(stream), nullptr, &fi);
  return cuda_status(rc, fn);
}

int cox_decode_moe(const void* x, int T, const void* wg, int E, int k, int mode, const void* const* w13,
                   const void* const* w2, int d, int ff, const void* w13_shared, const void* w2_shared, int ff_shared,
                   void* h, void* y, void* h_shared, void* y_shared, int32_t* idx, float* w, void* out,
                   void* stream) {
  const char* fn = "cox_decode_moe";
  if (T < 1 || T > 64) return fail(COX_EINVAL, "%s: need 1 <= T <= 64 (T=%d)", fn, T);
  if (E < 1 || E > 64 || k < 1 || k > 8 || k > E) return fail(COX_EINVAL, "%s: need 1 <= k <= min(E, 8), E <= 64", fn);
  if (mode != COX_ROUTE_MIXTRAL && mode != COX_ROUTE_DEEPSEEK) return fail(COX_EINVAL, "%s: bad mode %d", fn, mode);
  if (d <= 0 || d % 128 || ff <= 0 || ff % 128) return fail(COX_EINVAL, "%s: need d %% 128 == 0, ff %% 128 == 0", fn);
  if (!x || !wg || !h || !y || !idx || !w || !out || !aligned16(x) || !aligned16(wg) || !aligned16(h) ||
      !aligned16(y) || !aligned16(out))
    return fail(COX_EINVAL, "%s: null or unaligned operand", fn);
  if (w13_shared && (ff_shared <= 0 || ff_shared % 128 || !w2_shared || !h_shared || !y_shared ||
                     !aligned16(h_shared) || !aligned16(y_shared)))
    return fail(COX_EINVAL, "%s: bad shared-expert operands", fn);
  int32_t ids[64];
  for (int e = 0; e < E; ++e) ids[e] = e;
  if (int rc = check_groups(fn, E, E, ids, w13)) return rc;
  if (int rc = check_groups(fn, E, E, ids, w2)) return rc;
  cox::SmallDense dn{wg, E, mode, idx, w};
  int rc = cox::launch_small_ffn(x, T, nullptr, nullptr, (long long)E * T, nullptr, E, ids, w13, w2, d, ff, h, y,
                                 w13_shared, w2_shared, ff_shared, h_shared, y_shared, nullptr, nullptr, k, out, 3,
                                 static_cast<cudaStream_t>(stream), &dn);
  return cuda_status(rc, fn);
}

int cox_fetch_experts(const int32_t* counts, int E, int n, const int32_t* expert_ids, const void* const* host_src,
                      void* const* dst, const long long* bytes, int max_ctas, int32_t* fetched, void* stream) {
  const char* fn = "cox_fetch_experts";
  if (n < 0 || n > 64 || E < 1 || max_ctas < 0)
    return fail(COX_EINVAL, "%s: need 0 <= n <= 64, E >= 1 (n=%d E=%d)", fn, n, E);
  if (n == 0) return 0;
  if (!counts || !expert_ids || !host_src || !dst || !bytes) return fail(COX_EINVAL, "%s: null pointer", fn);
  for (int i = 0; i < n; ++i) {
    if (expert_ids[i] < 0 || expert_ids[i] >= E)
      return fail(COX_EINVAL, "%s: expert %d outside [0, %d)", fn, expert_ids[i], E);
    if (!host_src[i] || !dst[i] || !aligned16(host_src[i]) || !aligned16(dst[i]) || bytes[i] < 0 || bytes[i] % 16)
      return fail(COX_EINVAL, "%s: entry %d null, unaligned or not a multiple of 16 bytes", fn, i);
  }
  int rc = cox::launch_fetch_experts(counts, n, expert_ids, host_src, dst, bytes, max_ctas, fetched,
                                     static_cast<cudaStream_t>(stream));
  if (rc == -1) return fail(COX_EINVAL, "%s: a source is not pinned (mapped) host memory", fn);
  return cuda_status(rc, fn);
}

int cox_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared_out,
                void* out, int out_dtype, void* stream) {
  if (T < 0 || k < 1 || k > 8 || d <= 0 || d % 8) return fail(COX_EINVAL, "cox_combine: need 1<=k<=8, d%%8==0");
  if (out_dtype != COX_DTYPE_BF16 && out_dtype != COX_DTYPE_F32) return fail(COX_EINVAL, "cox_combine: bad out_dtype");
  if (!aligned16(y_perm) || !aligned16(out) || !aligned16(shared_out))
    return fail(COX_EINVAL, "cox_combine: unaligned operand");
  int rc = cox::launch_combine(y_perm, dst, w, T, k, d, shared_out, out, out_dtype == COX_DTYPE_BF16,
                               static_cast<cudaStream_t>(stream));
  return cuda_status(rc, "cox_combine");
}

static int check_ep(const char* fn, int E, int world, int rank) {
  if (world < 1 || E < 1 || E % world || rank < 0 || rank >= world || E > 256)
    return fail(COX_EINVAL, "%s: need 1 <= world, E %% world == 0, 0 <= rank < world, E <= 256", fn);
  return 0;
}

int cox_ep_counts_put(const int32_t* counts, int E, int rank, int world, int32_t* const* peer_counts, void* stream) {
  if (int rc = check_ep("cox_ep_counts_put", E, world, rank)) return rc;
  if (!counts || !peer_counts) return fail(COX_EINVAL, "cox_ep_counts_put: null pointer");
  return cuda_status(cox::launch_ep_counts_put(counts, E, rank, world, peer_counts, static_cast<cudaStream_t>(stream)),
                     "cox_ep_counts_put");
}

int cox_ep_offsets(const int32_t* counts_all, int world, int E, int rank, long long cap, int32_t* recv_seg,
                   int32_t* send_base, int32_t* overflow, void* stream) {
  if (int rc = check_ep("cox_ep_offsets", E, world, rank)) return rc;
  if (cap < 1) return fail(COX_EINVAL, "cox_ep_offsets: cap < 1");
  return cuda_status(cox::launch_ep_offsets(counts_all, world, E, rank, cap, recv_seg, send_base, overflow,
                                            static_cast<cudaStream_t>(stream)),
                     "cox_ep_offsets");
}

int cox_ep_dispatch(const int32_t* idx, const int32_t* dst_local, const int32_t* offsets_local,
                    const int32_t* send_base, int T, int k, int E, int world, long long cap, const void* x, int d,
                    void* const* peer_recv, int32_t* route_row, void* stream) {
  if (int rc = check_ep("cox_ep_dispatch", E, world, 0)) return rc;
  if (T < 0 || k < 1 || k > 8 || d <= 0 || d % 8) return fail(COX_EINVAL, "cox_ep_dispatch: need 1<=k<=8, d%%8==0");
  if (!aligned16(x)) return fail(COX_EINVAL, "cox_ep_dispatch: x must be 16-byte aligned");
  return cuda_status(cox::launch_ep_dispatch(idx, dst_local, offsets_local, send_base, T, k, E / world, cap, x, d,
                                             peer_recv, route_row, static_cast<cudaStream_t>(stream)),
                     "cox_ep_dispatch");
}

int cox_ep_combine(const int32_t* idx, const int32_t* route_row, const float* w, int T, int k, int d, int E,
                   int world, const void* const* peer_y, void* out, void* stream) {
  if (int rc = check_ep("cox_ep_combine", E, world, 0)) return rc;
  if (T < 0 || k < 1 || k > 8 || d <= 0 || d % 8) return fail(COX_EINVAL, "cox_ep_combine: need 1<=k<=8, d%%8==0");
  if (!aligned16(out)) return fail(COX_EINVAL, "cox_ep_combine: out must be 16-byte aligned");
  return cuda_status(cox::launch_ep_combine(idx, route_row, w, T, k, d, E / world, peer_y, out,
                                            static_cast<cudaStream_t>(stream)),
                     "cox_ep_combine");
}

int cox_interleave_w13(const void* w1, const void* w3, int ff, int d, void* w13, void* stream) {
  if (ff <= 0 || ff % 128 || d <= 0 || d % 8) return fail(COX_EINVAL, "cox_interleave_w13: need ff%%128==0, d%%8==0");
  if (!aligned16(w1) || !aligned16(w3) || !aligned16(w13)) return fail(COX_EINVAL, "cox_interleave_w13: unaligned");
  cox::interleave_w13_kernel<<<1184, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(w1), static_cast<const uint4*>(w3), ff, d, static_cast<uint4*>(w13));
  return cuda_status(cox::launch_status(), "cox_interleave_w13");
}

}  // extern "C"
