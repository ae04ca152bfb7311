// K2 — deterministic, stable token permutation by expert (the coalesced
// dispatch of PAPER.md:191,282: every expert sees its whole-batch token set
// as one contiguous row block).
//
// Order contract (shared with oracle/oracle_router.c:oracle_permute): the
// (token, slot) pairs of expert e occupy rows [offsets[e], offsets[e]+n_e) in
// ascending token order; segments are padded to a multiple of tile_m rows
// (padding rows are zero-filled).  No atomics decide placement:
//   1. perm_hist    — per-block (256 tokens) expert histogram (smem atomics on
//                     integers: order-independent result), stored expert-major
//                     ([E][nb]) so each expert's block counts are contiguous;
//   2. perm_scan    — per-expert exclusive scan over blocks: one warp per
//                     expert walks its row 32 blocks at a time (coalesced
//                     loads, shuffle scan, carried running sum), then the
//                     padded segment offsets;
//   3. perm_scatter — in-block ranks from warp ballots (lane = token, so
//                     popc(ballot & lanemask_lt) is the ascending-token rank);
//   4. perm_copy    — grid-wide, one warp per token: each row is read ONCE
//                     (16 B vector loads) and written to its k destinations.
#include "common.cuh"

namespace cox {

constexpr int PM_TB = 256;  // tokens per block

__global__ void __launch_bounds__(PM_TB) perm_hist(const int32_t* __restrict__ idx, int T, int k, int E,
                                                    int32_t* __restrict__ block_counts) {
  __shared__ int s_h[1024];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  long t = (long)blockIdx.x * PM_TB + threadIdx.x;
  if (t < T)
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      if ((unsigned)e < (unsigned)E) atomicAdd(&s_h[e], 1);  // invalid ids are dropped (dst = -1)
    }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) block_counts[(long)i * gridDim.x + blockIdx.x] = s_h[i];
}

// One block of 1024 threads; warp w scans experts w, w+32, ... over their
// contiguous [nb] rows of block counts (expert-major), 32 blocks per step with
// every step's loads issued before the carried scans.
__global__ void __launch_bounds__(1024) perm_scan(const int32_t* __restrict__ block_counts, int nb, int E, int tile_m,
                                                  int32_t* __restrict__ block_base, int32_t* __restrict__ offsets,
                                                  int32_t* __restrict__ seg_counts) {
  __shared__ int s_tot[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int U = 8;  // 32-block steps whose loads are in flight together
  for (int e = warp; e < E; e += 32) {
    const int32_t* row = block_counts + (long)e * nb;
    int32_t* base = block_base + (long)e * nb;
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32 * U) {
      int v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + 32 * u + lane;
        v[u] = b < nb ? row[b] : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int incl = v[u];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        const int b = b0 + 32 * u + lane;
        if (b < nb) base[b] = carry + incl - v[u];
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) s_tot[e] = carry;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int o = 0;
    offsets[0] = 0;
    for (int e = 0; e < E; ++e) {
      seg_counts[e] = s_tot[e];
      o += ((s_tot[e] + tile_m - 1) / tile_m) * tile_m;
      offsets[e + 1] = o;
    }
  }
}

__global__ void __launch_bounds__(PM_TB) perm_scatter(const int32_t* __restrict__ idx, int T, int k, int E,
                                                       const int32_t* __restrict__ block_base,
                                                       const int32_t* __restrict__ offsets,
                                                       int32_t* __restrict__ dst, int32_t* __restrict__ row_tokens) {
  __shared__ int s_wcnt[PM_TB / 32][256];
  __shared__ int s_wbase[PM_TB / 32][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long t = (long)blockIdx.x * PM_TB + threadIdx.x;
  const bool valid = t < T;
  int ej[8], rj[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    ej[j] = (valid && j < k) ? idx[t * k + j] : -1;
    if ((unsigned)ej[j] >= (unsigned)E) ej[j] = -1;
    rj[j] = 0;
  }
  const uint32_t lt = (1u << lane) - 1u;
  for (int e = 0; e < E; ++e) {
    bool has = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) has |= (ej[j] == e);
    uint32_t bal = __ballot_sync(0xffffffffu, has);
    if (lane == 0) s_wcnt[warp][e] = __popc(bal);
    int r = __popc(bal & lt);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (ej[j] == e) rj[j] = r;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = offsets[e] + block_base[(long)e * gridDim.x + blockIdx.x];
    for (int w = 0; w < PM_TB / 32; ++w) {
      s_wbase[w][e] = run;
      run += s_wcnt[w][e];
    }
  }
  __syncthreads();
  int dj[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    dj[j] = (ej[j] >= 0) ? s_wbase[warp][ej[j]] + rj[j] : -1;
    if (j < k && valid) {
      dst[t * k + j] = dj[j];
      if (row_tokens && dj[j] >= 0) row_tokens[dj[j]] = (int32_t)t;
    }
  }
}

// Small batches (decode: T*k <= PS_MAX_PAIRS): histogram, scan and stable
// scatter in ONE single-CTA launch instead of three.  Same order contract:
// tokens are processed in chunks of 1024 (thread = token), in-warp ranks from
// ballots, warp prefix per expert in shared memory, running per-expert base
// across chunks.
constexpr int PS_THREADS = 1024;
// up to 2,048 pairs (decode-size steps, T <= 256): above, the three parallel
// kernels win (C1, T*k = 8,192: 7 us faster per step under graph replay)
constexpr long PS_MAX_PAIRS = 2048;

__global__ void __launch_bounds__(PS_THREADS) perm_small(const int32_t* __restrict__ idx, int T, int k, int E,
                                                         int tile_m, int32_t* __restrict__ offsets,
                                                         int32_t* __restrict__ dst, int32_t* __restrict__ row_tokens,
                                                         int32_t* __restrict__ seg_counts) {
  __shared__ int s_cnt[256];
  __shared__ int s_base[256];
  __shared__ int s_wcnt[PS_THREADS / 32][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();  // the expert kernel may start its weight prefetch now
  pdl_wait();               // ... while this kernel waits for the router's idx
  for (int e = threadIdx.x; e < E; e += PS_THREADS) s_cnt[e] = 0;
  __syncthreads();
  for (long i = threadIdx.x; i < (long)T * k; i += PS_THREADS) {
    const int e = idx[i];
    if ((unsigned)e < (unsigned)E) atomicAdd(&s_cnt[e], 1);  // invalid ids are dropped (dst = -1)
  }
  __syncthreads();
  if (warp == 0) {  // padded segment offsets: warp scan over E <= 256 (8 experts per lane)
    int loc[8], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane * 8 + q;
      const int n = e < E ? s_cnt[e] : 0;
      loc[q] = ((n + tile_m - 1) / tile_m) * tile_m;
      sum += loc[q];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane * 8 + q;
      if (e < E) {
        s_base[e] = run;
        offsets[e] = run;
        seg_counts[e] = s_cnt[e];
      }
      run += loc[q];
    }
    if (lane == 31) offsets[E] = incl;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  for (int c0 = 0; c0 < T; c0 += PS_THREADS) {
    const long t = c0 + threadIdx.x;
    const bool valid = t < T;
    int ej[8], rj[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ej[j] = (valid && j < k) ? idx[t * k + j] : -1;
      if ((unsigned)ej[j] >= (unsigned)E) ej[j] = -1;
      rj[j] = 0;
    }
    const int nlive = min(PS_THREADS / 32, (T - c0 + 31) / 32);  // warps holding tokens of this chunk
    if (warp < nlive) {
      for (int e = 0; e < E; ++e) {
        bool has = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) has |= (ej[j] == e);
        const uint32_t bal = __ballot_sync(0xffffffffu, has);
        if (lane == 0) s_wcnt[warp][e] = __popc(bal);
        const int r = __popc(bal & lt);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (ej[j] == e) rj[j] = r;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += PS_THREADS) {  // exclusive prefix over warps, per expert
      int run = s_base[e];
      for (int w = 0; w < nlive; ++w) {
        const int n = s_wcnt[w][e];
        s_wcnt[w][e] = run;
        run += n;
      }
      s_base[e] = run;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < k && valid) {
        const int dj = ej[j] >= 0 ? s_wcnt[warp][ej[j]] + rj[j] : -1;
        dst[t * k + j] = dj;
        if (row_tokens && dj >= 0) row_tokens[dj] = (int32_t)t;
      }
    __syncthreads();
  }
}

// Row copies, grid-wide: one warp per token; each row is read once (16 B
// vectors, 4 chunks in flight per lane) and written to its k destinations.
__global__ void __launch_bounds__(256) perm_copy(const int32_t* __restrict__ dst, int T, int k,
                                                 const __nv_bfloat16* __restrict__ x, int d,
                                                 __nv_bfloat16* __restrict__ x_perm) {
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nwarps) {
    int di[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) di[j] = j < k ? dst[t * k + j] : 0;
    const __nv_bfloat16* src = x + t * (long)d;
    for (int c0 = lane * 8; c0 < d; c0 += 32 * 8 * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 256;
        if (c < d) v[u] = ld_nc_v4(src + c);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= k) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * 256;
          if (c < d && di[j] >= 0) *reinterpret_cast<uint4*>(x_perm + (long)di[j] * d + c) = v[u];
        }
      }
    }
  }
}

// Zero the padding rows [offsets[e] + n_e, offsets[e+1]) of every segment.
__global__ void perm_zero_pad(const int32_t* __restrict__ offsets, const int32_t* __restrict__ seg_counts, int E,
                              int d, __nv_bfloat16* __restrict__ x_perm) {
  const int e = blockIdx.y;
  const long r0 = offsets[e] + seg_counts[e], r1 = offsets[e + 1];
  const long n = (r1 - r0) * (long)d / 8;
  uint4 z = make_uint4(0, 0, 0, 0);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(x_perm + r0 * d)[i] = z;
}

size_t permute_workspace_bytes(int T, int E) {
  long nb = (T + PM_TB - 1) / PM_TB;
  if (nb < 1) nb = 1;
  return sizeof(int32_t) * (size_t)(2 * nb * E + E);
}

int launch_permute(const int32_t* idx, int T, int k, int E, int tile_m, const void* x, int d, int32_t* offsets,
                   int32_t* dst, void* x_perm, void* workspace, cudaStream_t s, int32_t* row_tokens,
                   long long rows_cap) {
  long nb = (T + PM_TB - 1) / PM_TB;
  int32_t* block_counts = static_cast<int32_t*>(workspace);
  int32_t* block_base = block_counts + (nb > 0 ? nb : 1) * E;
  int32_t* seg_counts = block_base + (nb > 0 ? nb : 1) * E;
  if (nb == 0) {
    if (cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), s) != cudaSuccess) return -2;
    return 0;
  }
  if (row_tokens && tile_m > 1)  // padding rows gather token 0 (computed, never combined)
    if (cudaMemsetAsync(row_tokens, 0, sizeof(int32_t) * rows_cap, s) != cudaSuccess) return -2;
  if ((long)T * k <= PS_MAX_PAIRS) {
    static bool carve = false;
    if (!carve) {
      cudaFuncSetAttribute(perm_small, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared);
      carve = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(PS_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, perm_small, idx, T, k, E, tile_m, offsets, dst, row_tokens, seg_counts);
  } else {
    perm_hist<<<(int)nb, PM_TB, 0, s>>>(idx, T, k, E, block_counts);
    perm_scan<<<1, 1024, 0, s>>>(block_counts, (int)nb, E, tile_m, block_base, offsets, seg_counts);
    perm_scatter<<<(int)nb, PM_TB, 0, s>>>(idx, T, k, E, block_base, offsets, dst, row_tokens);
  }
  long cb = (T + 7) / 8;
  if (cb > 148L * 16) cb = 148L * 16;
  if (x_perm) perm_copy<<<(int)cb, 256, 0, s>>>(dst, T, k, static_cast<const __nv_bfloat16*>(x), d,
                                    static_cast<__nv_bfloat16*>(x_perm));
  if (tile_m > 1 && x_perm) perm_zero_pad<<<dim3(8, E), 256, 0, s>>>(offsets, seg_counts, E, d, static_cast<__nv_bfloat16*>(x_perm));
  return launch_status();
}

}  // namespace cox
