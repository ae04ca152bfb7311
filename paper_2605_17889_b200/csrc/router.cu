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
// tensor cores — so the order is fixed.  Two experts' accumulators share one
// FFMA2 (fma.rn.f32x2: two independently rounded FMAs), which halves the FMA
// instruction count without changing any logit's operation sequence.
//
// Work decomposition: a block of 8 warps covers RT_TPW*NTG tokens x all E
// experts; warp w owns an RT_TPW-token x 8-expert register tile (token group
// w / EGN, expert group w % EGN, EGN = expert groups per block pass).  The
// warps of a block that share tokens read the same x chunks (L1 hits), so x
// is read from HBM once.  The kernel is bound by the fp32 FMA pipe
// (T*E*d FMAs: 8.6 G for C2, 34 G for C4), so x is widened once per chunk and
// each loaded router weight feeds RT_TPW FMAs.  Top-k is a warp-parallel
// argmax (lane-local scan + shuffle reduction, ties to the lower index).
#include <cstdlib>

#include "common.cuh"
#include "route_common.cuh"

namespace cox {

// NaN logits (e.g. from overflowing inputs) rank below every number, like
// -inf, so the top-k always returns valid, distinct expert ids (ties and
// equal -inf -> lower index); the oracle applies the same rule.
COX_DEV float nan_low(float v) { return v != v ? -INFINITY : v; }

constexpr int RT_TPW = 4;    // tokens per warp tile
constexpr int RT_EG = 8;     // experts per warp tile
constexpr int RT_WARPS = 8;  // warps per block

template <typename XT>
struct XChunk;
template <>
struct XChunk<__nv_bfloat16> {
  uint4 v;
  COX_DEV void load(const __nv_bfloat16* p) { v = ld_nc_v4_ordered(p); }
  COX_DEV void zero() { v = make_uint4(0, 0, 0, 0); }
  COX_DEV float get(int q) const {
    const uint32_t w = q < 2 ? v.x : q < 4 ? v.y : q < 6 ? v.z : v.w;
    return (q & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  }
};
template <>
struct XChunk<float> {
  float4 a, b;
  COX_DEV void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  COX_DEV void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  COX_DEV float get(int q) const {
    switch (q) {
      case 0: return a.x; case 1: return a.y; case 2: return a.z; case 3: return a.w;
      case 4: return b.x; case 5: return b.y; case 6: return b.z; default: return b.w;
    }
  }
};

// Tokens per block = RT_TPW * (RT_WARPS / egn); egn in {1,2,4,8}: expert groups
// handled concurrently by the warps of one block (E > 8*egn loops over passes).
template <typename WT>
COX_DEV void load_w8(const WT* p, float (&w8)[8]);
template <>
COX_DEV void load_w8<float>(const float* p, float (&w8)[8]) {
  const float4 wa = __ldg(reinterpret_cast<const float4*>(p)), wb = __ldg(reinterpret_cast<const float4*>(p) + 1);
  w8[0] = wa.x; w8[1] = wa.y; w8[2] = wa.z; w8[3] = wa.w; w8[4] = wb.x; w8[5] = wb.y; w8[6] = wb.z; w8[7] = wb.w;
}
template <>
COX_DEV void load_w8<__nv_bfloat16>(const __nv_bfloat16* p, float (&w8)[8]) {
  bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(p)), w8);
}

template <typename XT, int TPW, typename WT>
__global__ void __launch_bounds__(RT_WARPS * 32, 2)
router_topk_kernel(const XT* __restrict__ x, const WT* __restrict__ wg, int T, int d, int E, int k, int mode,
                   int egn, int32_t* __restrict__ idx, float* __restrict__ wout, int32_t* __restrict__ counts) {
  extern __shared__ float s_logits[];  // [tokens_per_block][E]
  __shared__ int s_hist[256];
  __shared__ int s_sel[RT_WARPS][8];
  __shared__ float s_selv[RT_WARPS][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();  // the permute (a programmatic dependent) may be scheduled now
  const int ntg = RT_WARPS / egn;
  const int tpb = TPW * ntg;
  const int tg = warp / egn, eg = warp % egn;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();

  const long nblk = (T + tpb - 1) / tpb;
  for (long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long tb0 = blk * tpb;
    const long t0 = tb0 + (long)tg * TPW;
    for (int e0 = eg * RT_EG; e0 < E; e0 += egn * RT_EG) {
      float acc[TPW][RT_EG];
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) acc[t][e] = 0.0f;
      for (int s = 8 * lane; s < d; s += 256) {
        float xv[TPW][8];  // widened once per chunk (the FMA pipe is the bound)
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          XChunk<XT> c;
          if (t0 + t < T)
            c.load(x + (t0 + t) * (long)d + s);
          else
            c.zero();
#pragma unroll
          for (int q = 0; q < 8; ++q) xv[t][q] = c.get(q);
        }
#pragma unroll
        for (int e = 0; e < RT_EG; e += 2) {  // expert pairs -> FFMA2
          float wa[8], wb[8];
          const int ea = min(e0 + e, E - 1), eb = min(e0 + e + 1, E - 1);  // clamped rows are never stored
          load_w8<WT>(wg + (long)ea * d + s, wa);
          load_w8<WT>(wg + (long)eb * d + s, wb);
#pragma unroll
          for (int t = 0; t < TPW; ++t)
#pragma unroll
            for (int q = 0; q < 8; ++q) ffma2(acc[t][e], acc[t][e + 1], xv[t][q], wa[q], wb[q]);
        }
      }
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          float v = acc[t][e];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == 0 && e0 + e < E) s_logits[(tg * TPW + t) * E + e0 + e] = nan_low(v);
        }
    }
    __syncthreads();
    // top-k: one warp per token, warp-parallel argmax (ties -> lower index)
    for (int tl = warp; tl < tpb; tl += RT_WARPS) {
      const long t = tb0 + tl;
      if (t >= T) break;
      float* lg = s_logits + tl * E;
      warp_route_token_e(lg, E, k, mode, lane, s_sel[warp], s_selv[warp], idx + t * k, wout + t * k, s_hist);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&counts[i], s_hist[i]);
}

// Staged variant for E > 8 (fine-grained MoE, e.g. C4: E=64, d=2048): the
// block's 32-token x tile is copied once into shared memory (cp.async) and
// reused by all E/8 expert-group passes; each warp owns 4 tokens x 8 experts.
// Router weights stream through L1/L2 once per 32 tokens (vs once per 4).
// Same canonical per-(t,e) summation order as router_topk_kernel.
constexpr int RS_TB = 32;

COX_DEV void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
COX_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(RT_WARPS * 32, 1)
router_topk_staged_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg, int T, int d, int E,
                          int k, int mode, int32_t* __restrict__ idx, float* __restrict__ wout,
                          int32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint8_t rs_smem[];
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(rs_smem);                    // [RS_TB][d]
  float* s_logits = reinterpret_cast<float*>(rs_smem + (size_t)RS_TB * d * 2);      // [RS_TB][E]
  __shared__ int s_hist[256];
  __shared__ int s_sel[RT_WARPS][8];
  __shared__ float s_selv[RT_WARPS][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_hist[i] = 0;
  const int vec_per_row = d / 8;
  const long nblk = (T + RS_TB - 1) / RS_TB;
  for (long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long tb0 = blk * RS_TB;
    __syncthreads();  // previous block's readers of sx / s_logits are done
    for (int i = threadIdx.x; i < RS_TB * vec_per_row; i += blockDim.x) {
      const int row = i / vec_per_row, c = i - row * vec_per_row;
      const bool ok = tb0 + row < T;
      const __nv_bfloat16* src = x + (ok ? (tb0 + row) * (long)d + 8 * c : 0);
      cp_async16(smem_u32(sx + (size_t)row * d + 8 * c), src, ok ? 16u : 0u);
    }
    cp_async_wait_all();
    __syncthreads();
    const int tl0 = warp * RT_TPW;
    for (int e0 = 0; e0 < E; e0 += RT_EG) {
      float acc[RT_TPW][RT_EG];
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) acc[t][e] = 0.0f;
      // register double-buffering: chunk j+1's operands are in flight while chunk j's FMAs issue
      uint4 xn[RT_TPW];
      float4 wna[RT_EG], wnb[RT_EG];
      auto load_chunk = [&](int s) {
#pragma unroll
        for (int t = 0; t < RT_TPW; ++t) xn[t] = *reinterpret_cast<const uint4*>(sx + (size_t)(tl0 + t) * d + s);
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          const int ee = min(e0 + e, E - 1);
          const float4* wp = reinterpret_cast<const float4*>(wg + (long)ee * d + s);
          wna[e] = __ldg(wp);
          wnb[e] = __ldg(wp + 1);
        }
      };
      if (8 * lane < d) load_chunk(8 * lane);
      for (int s = 8 * lane; s < d; s += 256) {
        uint4 xc[RT_TPW];
        float4 wca[RT_EG], wcb[RT_EG];
#pragma unroll
        for (int t = 0; t < RT_TPW; ++t) xc[t] = xn[t];
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          wca[e] = wna[e];
          wcb[e] = wnb[e];
        }
        if (s + 256 < d) load_chunk(s + 256);
        float xv[RT_TPW][8];
#pragma unroll
        for (int t = 0; t < RT_TPW; ++t) bf16x8_to_f32(xc[t], xv[t]);
#pragma unroll
        for (int e = 0; e < RT_EG; e += 2) {
          const float wa[8] = {wca[e].x, wca[e].y, wca[e].z, wca[e].w, wcb[e].x, wcb[e].y, wcb[e].z, wcb[e].w};
          const float wb[8] = {wca[e + 1].x, wca[e + 1].y, wca[e + 1].z, wca[e + 1].w,
                               wcb[e + 1].x, wcb[e + 1].y, wcb[e + 1].z, wcb[e + 1].w};
#pragma unroll
          for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
            for (int q = 0; q < 8; ++q) ffma2(acc[t][e], acc[t][e + 1], xv[t][q], wa[q], wb[q]);
        }
      }
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < RT_EG; ++e) {
          float v = acc[t][e];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == 0 && e0 + e < E) s_logits[(tl0 + t) * E + e0 + e] = nan_low(v);
        }
    }
    __syncthreads();
    for (int tl = warp; tl < RS_TB; tl += RT_WARPS) {
      const long t = tb0 + tl;
      if (t >= T) break;
      float* lg = s_logits + tl * E;
      warp_route_token_e(lg, E, k, mode, lane, s_sel[warp], s_selv[warp], idx + t * k, wout + t * k, s_hist);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&counts[i], s_hist[i]);
}

// bf16 router weights (the checkpoint dtype of Mixtral / DeepSeek routers):
// the block's 32-token x tile AND the current 8-expert slice of wg are both
// staged in shared memory (wg double-buffered: group g+1 streams in with
// cp.async while group g is consumed), so every warp reads conflict-free
// LDS.128 and the router weights cross L2 once per 32 tokens at half the
// bytes.  Products bf16 x bf16 -> fp32 FMA in the canonical order: results are
// identical to the fp32-weight kernels whenever wg is bf16-exact.
constexpr int RB_TB = 32;

// NW = warps per block: 8 (each warp 4 tokens x 8 experts) or 16 (4 tokens x 4
// experts: twice the warps per scheduler to hide the conversion/FMA latencies).
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
router_topk_staged_bf16w_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T,
                                int d, int E, int k, int mode, int32_t* __restrict__ idx, float* __restrict__ wout,
                                int32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint8_t rb_smem[];
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(rb_smem);                         // [RB_TB][d]
  __nv_bfloat16* sw = sx + (size_t)RB_TB * d;                                             // [2][RT_EG][d]
  float* s_logits = reinterpret_cast<float*>(sw + (size_t)2 * RT_EG * d);                // [RB_TB][E]
  __shared__ int s_hist[256];
  __shared__ int s_sel[NW][8];
  __shared__ float s_selv[NW][8];
  constexpr int EPW = RT_EG * RT_WARPS / NW;  // experts per warp tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_hist[i] = 0;
  const int vec_per_row = d / 8;
  const int ngroups = (E + RT_EG - 1) / RT_EG;
  auto stage_w = [&](int g, int buf) {
    for (int i = threadIdx.x; i < RT_EG * vec_per_row; i += blockDim.x) {
      const int r = i / vec_per_row, c = i - r * vec_per_row;
      const int e = g * RT_EG + r;
      const bool ok = e < E;
      cp_async16(smem_u32(sw + ((size_t)buf * RT_EG + r) * d + 8 * c), wg + (ok ? (long)e * d + 8 * c : 0),
                 ok ? 16u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const long nblk = (T + RB_TB - 1) / RB_TB;
  for (long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long tb0 = blk * RB_TB;
    __syncthreads();
    for (int i = threadIdx.x; i < RB_TB * vec_per_row; i += blockDim.x) {
      const int row = i / vec_per_row, c = i - row * vec_per_row;
      const bool ok = tb0 + row < T;
      cp_async16(smem_u32(sx + (size_t)row * d + 8 * c), x + (ok ? (tb0 + row) * (long)d + 8 * c : 0),
                 ok ? 16u : 0u);
    }
    stage_w(0, 0);  // commits x tile + group 0 together
    const int tl0 = (warp % RT_WARPS) * RT_TPW;
    const int eh = (warp / RT_WARPS) * EPW;  // first expert of this warp within the 8-expert slice
    for (int g = 0; g < ngroups; ++g) {
      if (g + 1 < ngroups) {
        stage_w(g + 1, (g + 1) & 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const __nv_bfloat16* swg = sw + (size_t)(g & 1) * RT_EG * d + (size_t)eh * d;
      const int e0 = g * RT_EG + eh;
      float acc[RT_TPW][EPW];
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < EPW; ++e) acc[t][e] = 0.0f;
      for (int s = 8 * lane; s < d; s += 256) {
        float xv[RT_TPW][8];
#pragma unroll
        for (int t = 0; t < RT_TPW; ++t)
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(sx + (size_t)(tl0 + t) * d + s), xv[t]);
#pragma unroll
        for (int e = 0; e < EPW; e += 2) {
          float wa[8], wb[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(swg + (size_t)e * d + s), wa);
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(swg + (size_t)(e + 1) * d + s), wb);
#pragma unroll
          for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
            for (int q = 0; q < 8; ++q) ffma2(acc[t][e], acc[t][e + 1], xv[t][q], wa[q], wb[q]);
        }
      }
#pragma unroll
      for (int t = 0; t < RT_TPW; ++t)
#pragma unroll
        for (int e = 0; e < EPW; ++e) {
          float v = acc[t][e];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == 0 && e0 + e < E) s_logits[(tl0 + t) * E + e0 + e] = nan_low(v);
        }
      __syncthreads();  // all warps done with buffer (g & 1) before it is refilled
    }
    for (int tl = warp; tl < RB_TB; tl += NW) {
      const long t = tb0 + tl;
      if (t >= T) break;
      float* lg = s_logits + tl * E;
      warp_route_token_e(lg, E, k, mode, lane, s_sel[warp], s_selv[warp], idx + t * k, wout + t * k, s_hist);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&counts[i], s_hist[i]);
}

int launch_router_bf16w(const void* x, const void* wg, int T, int d, int E, int k, int mode, int32_t* idx, float* w,
                        int32_t* counts, cudaStream_t s) {
  const size_t smem = (size_t)RB_TB * d * 2 + (size_t)2 * RT_EG * d * 2 + (size_t)RB_TB * E * 4;
  if (smem > 220 * 1024) return -1;
  if (cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s) != cudaSuccess) return -2;
  if (T == 0) return 0;
  constexpr int nw = 16;  // 16 warps of 4 tokens x 4 experts (measured faster than 8 x (4 x 8) on C4)
  long blocks = (T + RB_TB - 1) / RB_TB;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (nw == 16) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(router_topk_staged_bf16w_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           220 * 1024);
      attr = true;
    }
    router_topk_staged_bf16w_kernel<16><<<(int)blocks, 16 * 32, smem, s>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(wg), T, d, E, k, mode, idx, w,
        counts);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(router_topk_staged_bf16w_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           220 * 1024);
      attr = true;
    }
    router_topk_staged_bf16w_kernel<8><<<(int)blocks, 8 * 32, smem, s>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(wg), T, d, E, k, mode, idx, w,
        counts);
  }
  return launch_status();
}

// ---------------------------------------------------------------- decode router
// T <= 64 tokens: block (t, sp) computes the logits of token t for experts
// [sp E/S, (sp + 1) E/S), one expert pair per warp and pass (the canonical
// per-expert order of router_topk_kernel, so the same bits), into a global
// scratch row; the last of the S blocks of token t (acq_rel ticket) selects
// its top-k; the block that completes the last token writes the per-expert
// counts from idx (no memset node, no count atomics) and resets the tickets.
constexpr int RD_TMAX = 64;

COX_DEV int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <typename XT, typename WT>
__global__ void __launch_bounds__(RT_WARPS * 32)
router_decode_kernel(const XT* __restrict__ x, const WT* __restrict__ wg, int T, int d, int E, int k, int mode,
                     int S, int32_t* __restrict__ idx, float* __restrict__ wout, int32_t* __restrict__ counts,
                     float* g_logits, int* g_cnt) {
  __shared__ float lg[256];
  __shared__ int s_hist[256];
  __shared__ int s_sel[8];
  __shared__ float s_selv[8];
  __shared__ int s_last;
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x / S, sp = blockIdx.x - t * S;
  const int ept = E / S, eb0 = sp * ept;
  const XT* xr = x + (long)t * d;
  for (int pr = warp; 2 * pr < ept; pr += RT_WARPS) {
    const int ea = eb0 + 2 * pr, ebb = min(ea + 1, E - 1);
    float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll 8
    for (int s = 8 * lane; s < d; s += 256) {
      XChunk<XT> c;
      c.load(xr + s);
      float wa[8], wb[8];
      load_w8<WT>(wg + (long)ea * d + s, wa);
      load_w8<WT>(wg + (long)ebb * d + s, wb);
#pragma unroll
      for (int q = 0; q < 8; ++q) ffma2(acc0, acc1, c.get(q), wa[q], wb[q]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      acc0 = __fadd_rn(acc0, __shfl_xor_sync(0xffffffffu, acc0, off));
      acc1 = __fadd_rn(acc1, __shfl_xor_sync(0xffffffffu, acc1, off));
    }
    if (lane == 0) {
      g_logits[(long)t * E + ea] = nan_low(acc0);
      if (ea + 1 < E) g_logits[(long)t * E + ea + 1] = nan_low(acc1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) s_last = atom_add_acq_rel(g_cnt + t, 1) == S - 1;
  __syncthreads();
  if (!s_last || warp != 0) return;
  // last block of token t: its top-k
  for (int e = lane; e < E; e += 32) lg[e] = __ldcg(g_logits + (long)t * E + e);
  __syncwarp();
  warp_route_token_e(lg, E, k, mode, lane, s_sel, s_selv, idx + (long)t * k, wout + (long)t * k, nullptr);
  int last_tok = 0;
  if (lane == 0) last_tok = atom_add_acq_rel(g_cnt + RD_TMAX, 1) == T - 1;
  last_tok = __shfl_sync(0xffffffffu, last_tok, 0);
  if (!last_tok) return;
  // every token is routed: counts from idx, then reset the tickets
  for (int e = lane; e < E; e += 32) s_hist[e] = 0;
  __syncwarp();
  for (int i = lane; i < T * k; i += 32) {
    const int e = __ldcg(idx + i);
    if (e >= 0 && e < E) atomicAdd(&s_hist[e], 1);
  }
  __syncwarp();
  for (int e = lane; e < E; e += 32) counts[e] = s_hist[e];
  for (int i = lane; i <= RD_TMAX; i += 32) g_cnt[i] = 0;
}

// Scratch from the caller's workspace (router_workspace_bytes): the per-token
// tickets live in the zero-initialised header (the kernel resets them before
// it exits), the logits rows behind it.
static int launch_router_decode(const void* x, int x_is_bf16, const void* wg, int wg_is_bf16, int T, int d, int E,
                                int k, int mode, int32_t* idx, float* w, int32_t* counts, void* ws, cudaStream_t s) {
  // splits per token: expert pairs spread over the warps of S blocks
  int S = 1;
  while (S < 4 && E % (4 * S) == 0 && E / (2 * S) >= 2 * RT_WARPS) S *= 2;
  int* cs = static_cast<int*>(ws);
  float* lgs = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ROUTER_WS_HEADER);
  static bool carve = false;
  if (!carve) {  // decode: same smem carveout as the expert kernel that follows (no reconfig)
    cudaFuncSetAttribute(router_decode_kernel<__nv_bfloat16, __nv_bfloat16>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
#define RD_LAUNCH(XT, WT)                                                                                        \
  router_decode_kernel<XT, WT><<<T * S, RT_WARPS * 32, 0, s>>>(static_cast<const XT*>(x), static_cast<const WT*>(wg), \
                                                               T, d, E, k, mode, S, idx, w, counts, lgs, cs)
  if (x_is_bf16) {
    if (wg_is_bf16) RD_LAUNCH(__nv_bfloat16, __nv_bfloat16); else RD_LAUNCH(__nv_bfloat16, float);
  } else {
    if (wg_is_bf16) RD_LAUNCH(float, __nv_bfloat16); else RD_LAUNCH(float, float);
  }
#undef RD_LAUNCH
  return launch_status();
}

int launch_router_tc(const void* x, const void* wg, int T, int d, int E, int k, int mode, int32_t* idx, float* w,
                     int32_t* counts, float* scratch, cudaStream_t s);
int launch_router_e8(const void* x, const void* wg, int wg_is_bf16, int T, int d, int E, int k, int mode,
                     int32_t* idx, float* w, int32_t* counts, cudaStream_t s);

size_t router_workspace_bytes(int T, int E) {
  if (T < 0) T = 0;
  return ROUTER_WS_HEADER + sizeof(float) * ((size_t)T * E + (size_t)T + 64);
}

// tc: -1 auto (tensor-core screen for large fine-grained batches), 0 never, 1
// whenever the shape allows it; e8: 0 never use the E <= 8 TMA kernel (A/B).
int launch_router(const void* x, int x_is_bf16, const void* wg, int wg_is_bf16, int T, int d, int E, int k,
                  int mode, int32_t* idx, float* w, int32_t* counts, void* ws, int tc, int e8, cudaStream_t s) {
  // Large batches with bf16 x and router weights: tensor-core screening +
  // exact re-scoring (router_tc.cu), same indices as the CUDA-core kernels.
  // Fine-grained MoE only: with E = 8 the all-CUDA-core kernel is faster
  // (tools/bench_router.py: C2 0.85 ms vs 0.39 + 1.15 ms; C4 3.11 vs 1.77 ms).
  const bool tc_ok = x_is_bf16 && wg_is_bf16 && T > 0;
  if (tc_ok && (tc == 1 || (tc < 0 && E >= 32 && (long)T >= 148L * 128))) {
    float* scratch = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ROUTER_WS_HEADER);
    const int rc = launch_router_tc(x, wg, T, d, E, k, mode, idx, w, counts, scratch, s);
    if (rc != -3) return rc;  // -3: shape not supported by the screen -> CUDA-core kernels
  }
  // coarse-grained MoE (E <= 8) on large batches: TMA-fed kernel with the router
  // rows in shared memory (router_e8.cu)
  // from 2,048 tokens (C1, T = 4,096: 1.5-2 us faster than the generic kernel;
  // decode sizes keep the split-expert decode router)
  if (x_is_bf16 && E <= 8 && e8 != 0 && T >= 2048) {
    const int rc = launch_router_e8(x, wg, wg_is_bf16, T, d, E, k, mode, idx, w, counts, s);
    if (rc != -3) return rc;  // -3: shape not covered -> general kernels
  }
  if (wg_is_bf16 && x_is_bf16 && E > RT_EG && (long)T >= 148L * RB_TB) {
    const int rc = launch_router_bf16w(x, wg, T, d, E, k, mode, idx, w, counts, s);
    if (rc != -1) return rc;  // -1: tile does not fit in smem -> generic kernels below
  }
  // decode batches: split-expert router, counts without a memset
  if (T >= 1 && T <= RD_TMAX && E <= 256 && E % 2 == 0 && d % 8 == 0)
    return launch_router_decode(x, x_is_bf16, wg, wg_is_bf16, T, d, E, k, mode, idx, w, counts, ws, s);
  cudaError_t err = cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s);
  if (err != cudaSuccess) return -2;
  if (T == 0) return 0;
  const size_t staged_smem = (size_t)RS_TB * d * 2 + (size_t)RS_TB * E * 4;
  if (!wg_is_bf16 && x_is_bf16 && E > RT_EG && staged_smem <= 200 * 1024 && (long)T >= 148L * RS_TB) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(router_topk_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    long blocks = (T + RS_TB - 1) / RS_TB;
    if (blocks > 148L * 8) blocks = 148L * 8;
    router_topk_staged_kernel<<<(int)blocks, RT_WARPS * 32, staged_smem, s>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const float*>(wg), T, d, E, k, mode, idx, w, counts);
    return launch_status();
  }
  int groups = (E + RT_EG - 1) / RT_EG;
  int egn = 1;
  while (egn < groups && egn < RT_WARPS) egn <<= 1;
  // Small batches (decode): one token per warp tile so that T*E/8 warps exist.
  const bool small = (long)T * egn < 148L * 16 * RT_TPW;
  const int tpw = small ? 1 : RT_TPW;
  const int tpb = tpw * (RT_WARPS / egn);
  long blocks = (T + tpb - 1) / tpb;
  if (blocks > 148L * 16) blocks = 148L * 16;
  const size_t smem = sizeof(float) * (size_t)tpb * E;
#define RT_LAUNCH(XT, TP, WT)                                                                                   \
  do {                                                                                                          \
    static bool carve = false;                                                                                  \
    if (!carve && small) { /* decode: same smem carveout as the expert kernel that follows (no reconfig) */    \
      cudaFuncSetAttribute(router_topk_kernel<XT, TP, WT>, cudaFuncAttributePreferredSharedMemoryCarveout,     \
                           (int)cudaSharedmemCarveoutMaxShared);                                                \
      carve = true;                                                                                             \
    }                                                                                                           \
    router_topk_kernel<XT, TP, WT><<<(int)blocks, RT_WARPS * 32, smem, s>>>(                                    \
        static_cast<const XT*>(x), static_cast<const WT*>(wg), T, d, E, k, mode, egn, idx, w, counts);          \
  } while (0)
#define RT_BY_W(XT, TP) \
  if (wg_is_bf16) RT_LAUNCH(XT, TP, __nv_bfloat16); else RT_LAUNCH(XT, TP, float)
  if (x_is_bf16) {
    if (small) { RT_BY_W(__nv_bfloat16, 1); } else { RT_BY_W(__nv_bfloat16, RT_TPW); }
  } else {
    if (small) { RT_BY_W(float, 1); } else { RT_BY_W(float, RT_TPW); }
  }
#undef RT_BY_W
#undef RT_LAUNCH
  return launch_status();
}

}  // namespace cox
