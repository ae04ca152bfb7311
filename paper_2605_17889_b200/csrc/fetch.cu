// K6' — cold-expert fetch decided on the device.
//
// The reference charges every migrated expert on every pass (`mig_load =
// exp_m * 3*dt*d*ff / BW_link`, costmodel.py:252; Eq. 7).  For
// decode-size batches most cold experts are not routed to at all, and which
// ones are is only known after the layer's router ran.  Instead of reading the
// router's histogram back to the host (a synchronisation per layer) this
// kernel reads it on the device: every CTA takes slices of the listed cold
// experts, skips the experts whose count is 0, and streams the others from
// pinned host memory (SM loads over PCIe: mapped host pointers under UVA) into
// their device slots.  The hit ratio of the residency plan thus turns directly
// into PCIe bytes saved, with no host round trip and graph-capturable.
#include "common.cuh"

namespace cox {

constexpr int FX_MAX = 64;

struct FetchParams {
  const int32_t* counts;            // [E] routed tokens per expert (this layer's router)
  int n;                            // entries listed (a cold expert may span several, e.g. W13 and W2)
  int expert[FX_MAX];               // expert id of each entry
  const uint4* src[FX_MAX];         // device-accessible pinned host memory
  uint4* dst[FX_MAX];               // device slots
  long long vecs[FX_MAX];           // 16-byte vectors of each entry
  long long first[FX_MAX + 1];      // prefix sum of the entries' 16 KB slices
  int* fetched;                     // optional [n]: 1 if entry i was copied this launch
};

constexpr int FX_U = 4;                      // loads in flight per thread
constexpr long long FX_SLICE = 256LL * FX_U;  // vectors per CTA iteration (16 KB)

// Per entry: one check of its expert's count (untouched entries cost one load
// per CTA), then a grid-stride over its 16 KB slices with 4 loads in flight per
// thread before the stores (PCIe round trips are ~1-2 us; 148 CTAs keep
// ~2.4 MB in flight).
__global__ void __launch_bounds__(256) fetch_experts_kernel(const __grid_constant__ FetchParams p) {
  for (int i = 0; i < p.n; ++i) {
    if (__ldg(p.counts + p.expert[i]) <= 0) continue;  // untouched this step: no bytes cross PCIe
    if (p.fetched && blockIdx.x == 0 && threadIdx.x == 0) p.fetched[i] = 1;
    const uint4* __restrict__ src = p.src[i];
    uint4* __restrict__ dst = p.dst[i];
    const long long nv = p.vecs[i];
    const long long nslice = p.first[i + 1] - p.first[i];
    for (long long sl = blockIdx.x; sl < nslice; sl += gridDim.x) {
      const long long s0 = sl * FX_SLICE;
      uint4 v[FX_U];
#pragma unroll
      for (int u = 0; u < FX_U; ++u) {
        const long long j = s0 + threadIdx.x + 256LL * u;
        if (j < nv) v[u] = ld_nc_v4(src + j);
      }
#pragma unroll
      for (int u = 0; u < FX_U; ++u) {
        const long long j = s0 + threadIdx.x + 256LL * u;
        if (j < nv) dst[j] = v[u];
      }
    }
  }
}

__global__ void zero_i32_kernel(int* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

int launch_fetch_experts(const int32_t* counts, int n, const int32_t* expert_ids, const void* const* src,
                         void* const* dst, const long long* bytes, int max_ctas, int32_t* fetched, cudaStream_t s) {
  if (n <= 0) return 0;
  FetchParams p;
  p.counts = counts;
  p.n = n;
  p.fetched = fetched;
  p.first[0] = 0;
  for (int i = 0; i < n; ++i) {
    p.expert[i] = expert_ids[i];
    void* dev = nullptr;
    if (cudaHostGetDevicePointer(&dev, const_cast<void*>(src[i]), 0) != cudaSuccess) {
      cudaGetLastError();
      return -1;  // not pinned / not mapped host memory
    }
    p.src[i] = static_cast<const uint4*>(dev);
    p.dst[i] = static_cast<uint4*>(dst[i]);
    p.vecs[i] = bytes[i] / 16;
    p.first[i + 1] = p.first[i] + (p.vecs[i] + FX_SLICE - 1) / FX_SLICE;
  }
  if (fetched) zero_i32_kernel<<<1, 64, 0, s>>>(fetched, n);
  int grid = max_ctas > 0 ? max_ctas : 148;
  fetch_experts_kernel<<<grid, 256, 0, s>>>(p);
  return launch_status();
}

}  // namespace cox
