// K1 — router logits + top-k + routing weights + expert histogram.
//
// Reference context: the reference has no router;
// the top-k semantics follow PAPER.md:67 and the tie rule of
// eas.select_resident_experts (eas.py:364-374): on equal logits the LOWER
// expert index wins.  Routing conventions (Mixtral renormalised top-k softmax,
// DeepSeek-V2 full softmax without renorm) are public-config assumptions.
//
// Bit-exactness: logits are fp32 sums in the canonical order that the CPU
// oracle (oracle/oracle_router.c) replays exactly: lane l owns the 8-element
// chunks c = 32*j + l, accumulating fmaf(x, w, acc) with j then q ascending,
// followed by an xor butterfly 16,8,4,2,1 of __fadd_rn.  CUDA cores only — no
// tensor cores — so the order is fixed.  HBM-bound: x is read exactly once with
// 16-byte vector loads; router weights stay L1/L2-resident.
#include "common.cuh"

namespace cox {

constexpr int RT_TPW = 4;   // tokens per warp (register-blocked)
constexpr int RT_EG = 8;    // experts per register group
constexpr int RT_WARPS = 8;

template <typename XT>
COX_DEV void load_x8(const XT* p, float (&f)[8]);

template <>
COX_DEV void load_x8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  uint4 v = ld_nc_v4(p);
  bf16x8_to_f32(v, f);
}
template <>
COX_DEV void load_x8<float>(const float* p, float (&f)[8]) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p));
  float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <typename XT>
__global__ void __launch_bounds__(RT_WARPS * 32, 2)
router_topk_kernel(const XT* __restrict__ x, const float* __restrict__ wg, int T, int d, int E, int k, int mode,
                   int32_t* __restrict__ idx, float* __restrict__ wout, int32_t* __restrict__ counts) {
  extern __shared__ float s_logits[];  // [RT_WARPS][RT_TPW][E]
  __shared__ int s_hist[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  float* my_logits = s_logits + warp * RT_TPW * E;

  const long n_groups = (T + RT_TPW - 1) / RT_TPW;
  for (long tg = (long)blockIdx.x * RT_WARPS + warp; tg < n_groups; tg += (long)gridDim.x * RT_WARPS) {
    const long t0 = tg * RT_TPW;
    for (int e0 = 0; e0 < E; e0 += RT_EG) {
      float acc[RT_TPW][RT_EG];
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) acc[t][e] = 0.0f;
      for (int s = 8 * lane; s < d; s += 256) {
        float xv[RT_TPW][8];
#pragma unroll
        for (int t = 0; t < RT_TPW; ++t) {
          if (t0 + t < T) {
            load_x8<XT>(x + (t0 + t) * (long)d + s, xv[t]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) xv[t][q] = 0.0f;
          }
        }
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          if (e0 + e < E) {
            const float4* wp = reinterpret_cast<const float4*>(wg + (long)(e0 + e) * d + s);
            float4 wa = __ldg(wp), wb = __ldg(wp + 1);
            const float w8[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[t][e] = __fmaf_rn(xv[t][q], w8[q], acc[t][e]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          float v = acc[t][e];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == 0 && e0 + e < E) my_logits[t * E + e0 + e] = v;
        }
    }
    __syncwarp();
    if (lane < RT_TPW && t0 + lane < T) {
      const float* lg = my_logits + lane * E;
      const long t = t0 + lane;
      uint32_t taken[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // up to 256 experts
      int sel[8];
      float selv[8];
      for (int j = 0; j < k; ++j) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < E; ++e) {
          if (taken[e >> 5] & (1u << (e & 31))) continue;
          float v = lg[e];
          if (best < 0 || v > bv) { best = e; bv = v; }
        }
        taken[best >> 5] |= 1u << (best & 31);
        sel[j] = best;
        selv[j] = bv;
        idx[t * k + j] = best;
        atomicAdd(&s_hist[best], 1);
      }
      const float m = selv[0];
      float ssum = 0.0f;
      if (mode == 0) {
        for (int j = 0; j < k; ++j) ssum = __fadd_rn(ssum, expf(__fsub_rn(selv[j], m)));
      } else {
        for (int e = 0; e < E; ++e) ssum = __fadd_rn(ssum, expf(__fsub_rn(lg[e], m)));
      }
      for (int j = 0; j < k; ++j) wout[t * k + j] = __fdiv_rn(expf(__fsub_rn(selv[j], m)), ssum);
      (void)sel;
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&counts[i], s_hist[i]);
}

int launch_router(const void* x, int x_is_bf16, const float* wg, int T, int d, int E, int k, int mode, int32_t* idx,
                  float* w, int32_t* counts, cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s);
  if (err != cudaSuccess) return -2;
  if (T == 0) return 0;
  const int threads = RT_WARPS * 32;
  long groups = (T + RT_TPW - 1) / RT_TPW;
  long blocks = (groups + RT_WARPS - 1) / RT_WARPS;
  if (blocks > 148L * 16) blocks = 148L * 16;
  size_t smem = sizeof(float) * RT_WARPS * RT_TPW * E;
  if (x_is_bf16)
    router_topk_kernel<__nv_bfloat16><<<(int)blocks, threads, smem, s>>>(
        static_cast<const __nv_bfloat16*>(x), wg, T, d, E, k, mode, idx, w, counts);
  else
    router_topk_kernel<float><<<(int)blocks, threads, smem, s>>>(static_cast<const float*>(x), wg, T, d, E, k,
                                                                 mode, idx, w, counts);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace cox
