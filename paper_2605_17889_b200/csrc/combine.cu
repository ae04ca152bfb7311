// K5 — weighted top-k combine / unpermute back to token order.
//
// out[t] = sum_{j<k} w[t,j] * y_perm[dst[t,j]]  (+ shared_out[t])
// fp32 accumulation in ascending j with separately rounded multiply and add —
// the exact operation order of oracle/oracle_router.c:oracle_combine, so that
// for identical y_perm the result is bit-identical.  The reference's analogue
// is the analytical `expert:merge` / `return_store` step (sim.py:149-202,
// costmodel.py:266-273).  HBM-bound gather-reduce: one warp per token, 16 B
// vector loads of each selected row.
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
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ dst,
                                                      const float* __restrict__ w, int T, int k, int d,
                                                      const OT* __restrict__ shared, OT* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nwarps) {
    int dj[8];
    float wj[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dj[j] = j < k ? dst[t * k + j] : 0;
      wj[j] = j < k ? w[t * k + j] : 0.f;
    }
    for (int c = lane * 8; c < d; c += 256) {
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) v[j] = ld_nc_v4(y + (long)dj[j] * d + c);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < k) {
          float f[8];
          bf16x8_to_f32(v[j], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(wj[j], f[q]));
        }
      }
      if (shared) {
        float sh[8];
        if constexpr (sizeof(OT) == 2) {
          bf16x8_to_f32(ld_nc_v4(shared + t * (long)d + c), sh);
        } else {
          const float4* sp = reinterpret_cast<const float4*>(shared + t * (long)d + c);
          float4 a = sp[0], b = sp[1];
          sh[0] = a.x; sh[1] = a.y; sh[2] = a.z; sh[3] = a.w; sh[4] = b.x; sh[5] = b.y; sh[6] = b.z; sh[7] = b.w;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], sh[q]);
      }
      store8<OT>(out + t * (long)d + c, acc);
    }
  }
}

int launch_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared,
                   void* out, int out_is_bf16, cudaStream_t s) {
  if (T == 0) return 0;
  long blocks = (T + 7) / 8;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (out_is_bf16)
    combine_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(y_perm), dst, w, T, k, d, static_cast<const __nv_bfloat16*>(shared),
        static_cast<__nv_bfloat16*>(out));
  else
    combine_kernel<float><<<(int)blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(y_perm), dst, w, T, k, d,
                                                      static_cast<const float*>(shared), static_cast<float*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace cox
