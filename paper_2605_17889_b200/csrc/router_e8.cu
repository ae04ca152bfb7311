// K1 for coarse-grained MoE (E <= 8: Mixtral-style layers) on large batches:
// TMA-fed, shared-memory-resident router weights, canonical fp32 order.
//
// Semantics are those of router.cu (PAPER.md:67 top-k over the expert pool;
// ties -> lower expert index, eas.py:364-374; NaN ranks like -inf) and the
// logits are bit-identical to the CPU oracle (oracle/oracle_router.c): lane l
// owns the 8-element chunks c = 32 j + l of the d-vector, fma ascending in
// (j, q) from +0.0f, then an xor-butterfly (16, 8, 4, 2, 1) of fp32 adds.
//
// Why a second kernel.  The general router (router_topk_kernel) loads its x
// chunks and router rows straight from global memory and re-widens the
// router rows for every 4 tokens: at C2 (T = 262,144, d = 4096) it is
// latency/issue-bound at ~0.85 ms, a quarter of the HBM rate.  Here:
//   * a producer warp streams x through a ring of 32 KB TMA boxes
//     (64 tokens x 256 columns = one chunk per lane per token), several boxes
//     in flight per SM, so HBM is kept busy while the FMAs run;
//   * the router weight (E <= 8 rows) is copied into shared memory once per
//     CTA (bf16: 16 d bytes; fp32: 32 d bytes), padded to 8 rows with zeros;
//   * each of the 8 consumer warps owns 8 tokens x 8 experts of a tile (64
//     accumulators per lane; expert pairs share one FFMA2), so every widened
//     router chunk feeds 8 tokens and every widened x chunk 8 experts;
//   * the cross-lane reduction is a recursive-halving reduce-scatter: at step
//     `off` a lane adds its partner's (lane ^ off) partial sum of the SAME
//     logit — exactly the pairs the xor butterfly adds, so the bits are the
//     butterfly's — but it moves half the values per step (62 shuffles for
//     64 logits instead of 320).
// Top-k, routing weights and the expert histogram follow warp_route_token's
// arithmetic (one lane per token here; E <= 8).
#include <cuda.h>

#include "common.cuh"
#include "route_common.cuh"

namespace cox {

int get_map_box(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols,
                unsigned box_cols, unsigned box_rows, bool swizzle128);

constexpr int R8_WARPS = 8;                 // consumer warps
constexpr int R8_TPW = 8;                   // tokens per consumer warp
constexpr int R8_TILE = R8_WARPS * R8_TPW;  // 64 tokens per tile
constexpr int R8_SLAB = 256;                // d columns per stage: one 8-element chunk per lane
constexpr uint32_t R8_STAGE_BYTES = R8_TILE * R8_SLAB * 2;  // 32 KB
constexpr int R8_MAX_STAGES = 6;
constexpr int R8_THREADS = (R8_WARPS + 1) * 32;  // + producer warp
constexpr size_t R8_SMEM_LIMIT = 227 * 1024 - 256;  // beside the static s_hist

// bf16 pair -> fp32 on the ALU pipe (PRMT / LOP3), keeping the FMA pipe for the FFMA2s
COX_DEV float bf16_lo(uint32_t u) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(u));
  return __uint_as_float(r);
}
COX_DEV float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

COX_DEV void widen8(const uint4& v, float (&f)[8]) {
  f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
  f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
}

template <typename WT>
struct WRow;
template <>
struct WRow<__nv_bfloat16> {  // router chunk of 8 from shared memory
  COX_DEV static void load(const __nv_bfloat16* p, float (&f)[8]) { widen8(*reinterpret_cast<const uint4*>(p), f); }
};
template <>
struct WRow<float> {
  COX_DEV static void load(const float* p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

template <typename WT>
__global__ void __launch_bounds__(R8_THREADS, 1)
router_e8_kernel(const __grid_constant__ CUtensorMap xmap, const WT* __restrict__ wg, int T, int d, int E, int k,
                 int mode, int stages, int32_t* __restrict__ idx, float* __restrict__ wout,
                 int32_t* __restrict__ counts) {
  extern __shared__ __align__(128) uint8_t r8_smem[];
  uint8_t* sx = r8_smem;                                                         // [stages][64][256] bf16
  WT* sw = reinterpret_cast<WT*>(r8_smem + (size_t)stages * R8_STAGE_BYTES);     // [8][d]
  float* s_logit = reinterpret_cast<float*>(sw + 8 * (size_t)d);                 // [8 warps][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_logit + R8_WARPS * 64);
  uint64_t* empty = full + R8_MAX_STAGES;
  __shared__ int s_hist[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();

  // router rows -> shared memory (rows >= E are zero: they never win, see below)
  {
    constexpr int V = 16 / sizeof(WT);  // elements per 16-byte vector
    const int vec_per_row = d / V;
    for (int i = threadIdx.x; i < 8 * vec_per_row; i += blockDim.x) {
      const int e = i / vec_per_row, c = i - e * vec_per_row;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (e < E) v = __ldg(reinterpret_cast<const uint4*>(wg + (size_t)e * d) + c);
      reinterpret_cast<uint4*>(sw + (size_t)e * d)[c] = v;
    }
  }
  if (threadIdx.x < 8) s_hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), R8_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int ntiles = (T + R8_TILE - 1) / R8_TILE;
  const int nslab = d / R8_SLAB;

  if (warp == R8_WARPS) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int j = 0; j < nslab; ++j) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          mbar_arrive_expect_tx(smem_u32(&full[stage]), R8_STAGE_BYTES);
          tma_load_2d(smem_u32(sx + (size_t)stage * R8_STAGE_BYTES), &xmap, smem_u32(&full[stage]), j * R8_SLAB,
                      tile * R8_TILE);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  int stage = 0;
  uint32_t phase = 0;
  float* lgw = s_logit + warp * 64;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    float acc[R8_TPW][8];
#pragma unroll
    for (int t = 0; t < R8_TPW; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[t][e] = 0.0f;
    for (int j = 0; j < nslab; ++j) {
      mbar_wait(smem_u32(&full[stage]), phase);
      const __nv_bfloat16* xs =
          reinterpret_cast<const __nv_bfloat16*>(sx + (size_t)stage * R8_STAGE_BYTES) + (warp * R8_TPW) * R8_SLAB +
          8 * lane;
      float xv[R8_TPW][8];
#pragma unroll
      for (int t = 0; t < R8_TPW; ++t) widen8(*reinterpret_cast<const uint4*>(xs + t * R8_SLAB), xv[t]);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));  // x of this stage is in registers
      if (++stage == stages) { stage = 0; phase ^= 1; }
      const WT* wcol = sw + (size_t)j * R8_SLAB + 8 * lane;
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float wa[8], wb[8];
        WRow<WT>::load(wcol + (size_t)e * d, wa);
        WRow<WT>::load(wcol + (size_t)(e + 1) * d, wb);
#pragma unroll
        for (int t = 0; t < R8_TPW; ++t)
#pragma unroll
          for (int q = 0; q < 8; ++q) ffma2(acc[t][e], acc[t][e + 1], xv[t][q], wa[q], wb[q]);
      }
    }
    // cross-lane sums (the butterfly's pairs, reduce-scatter order): logit i = 8 t + e
    float v64[64];
#pragma unroll
    for (int t = 0; t < R8_TPW; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) v64[8 * t + e] = acc[t][e];
    float v32[32], v16[16], v8[8], v4[4], v2[2];
    rs_step<32>(v64, v32, lane, 16);
    rs_step<16>(v32, v16, lane, 8);
    rs_step<8>(v16, v8, lane, 4);
    rs_step<4>(v8, v4, lane, 2);
    rs_step<2>(v4, v2, lane, 1);
    // lane l now holds logits i = 2 l and 2 l + 1 (kept halves: +32 b4 + 16 b3 + ... + 2 b0 of l)
    const int i0 = 2 * lane;
    lgw[i0] = v2[0];
    lgw[i0 + 1] = v2[1];
    __syncwarp();
    // top-k: one lane per token
    if (lane < R8_TPW) {
      const long tok = (long)tile * R8_TILE + warp * R8_TPW + lane;
      if (tok < T) {
        float lg[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float v = lgw[8 * lane + e];
          lg[e] = v != v ? -INFINITY : v;  // NaN ranks like -inf (nan_low)
        }
        int sel[8];
        float selv[8];
        unsigned taken = 0;
        for (int jj = 0; jj < k; ++jj) {
          int best = -1;
          float bv = 0.0f;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (e >= E || ((taken >> e) & 1u)) continue;
            if (best < 0 || lg[e] > bv) { best = e; bv = lg[e]; }  // strict '>': ties -> lower index
          }
          taken |= 1u << best;
          sel[jj] = best;
          selv[jj] = bv;
        }
        const float m = selv[0];
        float ssum = 0.0f;
        if (mode == 0) {
          for (int jj = 0; jj < k; ++jj) ssum = __fadd_rn(ssum, expf(__fsub_rn(selv[jj], m)));
        } else {
          for (int e = 0; e < E; ++e) ssum = __fadd_rn(ssum, expf(__fsub_rn(lg[e], m)));
        }
        for (int jj = 0; jj < k; ++jj) {
          idx[tok * k + jj] = sel[jj];
          wout[tok * k + jj] = __fdiv_rn(expf(__fsub_rn(selv[jj], m)), ssum);
          atomicAdd(&s_hist[sel[jj]], 1);
        }
      }
    }
    __syncwarp();
  }
  // all consumers' histograms are in s_hist once every consumer warp is here
  asm volatile("bar.sync 1, %0;" ::"n"(R8_WARPS * 32));
  if (threadIdx.x < E && s_hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_hist[threadIdx.x]);
}

size_t router_e8_smem(int d, bool wg_bf16, int stages) {
  return (size_t)stages * R8_STAGE_BYTES + (size_t)8 * d * (wg_bf16 ? 2 : 4) + R8_WARPS * 64 * 4 +
         2 * R8_MAX_STAGES * 8;
}

// Returns -3 when the shape is not covered (caller uses the general kernels).
int launch_router_e8(const void* x, const void* wg, int wg_is_bf16, int T, int d, int E, int k, int mode,
                     int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  if (E > 8 || k > E || d % R8_SLAB != 0 || T < R8_TILE) return -3;
  int stages = R8_MAX_STAGES;
  while (stages >= 2 && router_e8_smem(d, wg_is_bf16, stages) > R8_SMEM_LIMIT) --stages;
  if (stages < 2) return -3;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  CUtensorMap xmap;
  int rc = get_map_box(&xmap, x, (unsigned long long)T, (unsigned long long)d, R8_SLAB, R8_TILE, false);
  if (rc) return rc;
  if (cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s) != cudaSuccess) return -2;
  const int ntiles = (T + R8_TILE - 1) / R8_TILE;
  const int grid = ntiles < num_sms ? ntiles : num_sms;
  const size_t smem = router_e8_smem(d, wg_is_bf16, stages);
  if (wg_is_bf16) {
    if (cudaFuncSetAttribute(router_e8_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return launch_status();
    router_e8_kernel<__nv_bfloat16><<<grid, R8_THREADS, smem, s>>>(
        xmap, static_cast<const __nv_bfloat16*>(wg), T, d, E, k, mode, stages, idx, w, counts);
  } else {
    if (cudaFuncSetAttribute(router_e8_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return launch_status();
    router_e8_kernel<float><<<grid, R8_THREADS, smem, s>>>(xmap, static_cast<const float*>(wg), T, d, E, k, mode,
                                                          stages, idx, w, counts);
  }
  return launch_status();
}

}  // namespace cox
