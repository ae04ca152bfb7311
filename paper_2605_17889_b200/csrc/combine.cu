// K5 — weighted top-k combine / unpermute back to token order.
//
// out[t] = sum_{j<k} w[t,j] * y_perm[dst[t,j]]  (+ shared_out[t])
// fp32 accumulation in ascending j with separately rounded multiply and add —
// the exact operation order of oracle/oracle_router.c:oracle_combine, so that
// for identical y_perm the result is bit-identical.  The reference's analogue
// is the analytical `expert:merge` / `return_store` step (sim.py:149-202,
// costmodel.py:266-273).  HBM-bound gather-reduce: one warp per token, k is a
// template parameter (registers), each lane keeps UNROLL 16-byte chunks of
// every selected row in flight.
#include "common.cuh"

namespace cox {

template <typename OT>
COX_DEV void store8(OT* p, const float (&a)[8]);
template <>
COX_DEV void store8<__nv_bfloat16>(__nv_bfloat16* p, const float (&a)[8]) {
  uint4 v = make_uint4(pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]), pack_bf16x2(a[4], a[5]),
                       pack_bf16x2(a[6], a[7]));
  *reinterpret_cast<uint4*>(p) = v;
}
template <>
COX_DEV void store8<float>(float* p, const float (&a)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(a[0], a[1], a[2], a[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(a[4], a[5], a[6], a[7]);
}

template <typename OT>
COX_DEV void load8(const OT* p, float (&f)[8]);
template <>
COX_DEV void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  bf16x8_to_f32(ld_nc_v4(p), f);
}
template <>
COX_DEV void load8<float>(const float* p, float (&f)[8]) {
  const float4* sp = reinterpret_cast<const float4*>(p);
  float4 a = sp[0], b = sp[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

constexpr int CB_UNROLL = 2;

template <typename OT, int K>
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ dst,
                                                      const float* __restrict__ w, int T, int d,
                                                      const OT* __restrict__ shared, OT* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nwarps) {
    const __nv_bfloat16* rows[K];
    float wj[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int r = dst[t * K + j];
      rows[j] = y + (long)(r < 0 ? 0 : r) * d;   // dst < 0 (invalid expert id): no contribution
      wj[j] = r < 0 ? 0.0f : w[t * K + j];
    }
    for (int c0 = lane * 8; c0 < d; c0 += 256 * CB_UNROLL) {
      uint4 v[CB_UNROLL][K];
#pragma unroll
      for (int u = 0; u < CB_UNROLL; ++u)
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (c0 + u * 256 < d) v[u][j] = ld_nc_v4(rows[j] + c0 + u * 256);
#pragma unroll
      for (int u = 0; u < CB_UNROLL; ++u) {
        const int c = c0 + u * 256;
        if (c >= d) break;
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float f[8];
          bf16x8_to_f32(v[u][j], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(wj[j], f[q]));
        }
        if (shared) {
          float sh[8];
          load8<OT>(shared + t * (long)d + c, sh);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], sh[q]);
        }
        store8<OT>(out + t * (long)d + c, acc);
      }
    }
  }
}

template <typename OT>
static void launch_k(int k, int blocks, cudaStream_t s, const __nv_bfloat16* y, const int32_t* dst, const float* w,
                     int T, int d, const OT* shared, OT* out) {
  switch (k) {
#define CB_CASE(KK) \
  case KK:          \
    combine_kernel<OT, KK><<<blocks, 256, 0, s>>>(y, dst, w, T, d, shared, out); \
    break;
    CB_CASE(1) CB_CASE(2) CB_CASE(3) CB_CASE(4) CB_CASE(5) CB_CASE(6) CB_CASE(7) CB_CASE(8)
#undef CB_CASE
    default:
      break;
  }
}

int launch_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared,
                   void* out, int out_is_bf16, cudaStream_t s) {
  if (T == 0) return 0;
  long blocks = (T + 7) / 8;
  if (blocks > 148L * 16) blocks = 148L * 16;
  const __nv_bfloat16* y = static_cast<const __nv_bfloat16*>(y_perm);
  if (out_is_bf16)
    launch_k<__nv_bfloat16>(k, (int)blocks, s, y, dst, w, T, d, static_cast<const __nv_bfloat16*>(shared),
                            static_cast<__nv_bfloat16*>(out));
  else
    launch_k<float>(k, (int)blocks, s, y, dst, w, T, d, static_cast<const float*>(shared), static_cast<float*>(out));
  return launch_status();
}

}  // namespace cox
