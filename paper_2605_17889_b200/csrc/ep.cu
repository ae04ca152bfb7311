// K7' — fused expert-parallel dispatch / combine over NVLink peer memory.
//
// Instead of K2's local x_perm + an NCCL all-to-all (and the reverse for the
// combine), the token rows are stored straight into the owner GPU's receive
// buffer (st.global through peer pointers mapped by CUDA symmetric memory),
// and the combine gathers y rows straight from the owners' output buffers
// (ld.global through peer pointers).  NVLink/NVSwitch carries exactly the
// bytes the all-to-all would; the local x_perm / y_back round trips through
// HBM disappear, and no host synchronisation is needed (the receive layout is
// computed on the device from an all-gathered count matrix).
//
// Receive layout on owner r: one contiguous segment per local expert l, made
// of every source's rows in source-rank order, each source's rows in its
// ascending token order — so the per-expert row order is the global token
// order (results bit-identical to one GPU) and each local expert is ONE
// grouped-GEMM group (its weights stream once per layer).
#include "common.cuh"

namespace cox {

// counts_all[rank][e] = counts[e] on every peer (peer_counts[p] = &counts_all of p).
__global__ void ep_counts_put_kernel(const int32_t* __restrict__ counts, int E, int rank, int world,
                                     int32_t* const* __restrict__ peer_counts) {
  for (int i = threadIdx.x; i < world * E; i += blockDim.x) {
    const int p = i / E, e = i - p * E;
    peer_counts[p][rank * E + e] = counts[e];
  }
}

// From counts_all [G][E]: my receive segments (L+1 offsets, one per local
// expert: every source's rows of local expert l are contiguous, sources in
// rank order) and, for each of my experts e (owned by r = e / L, l = e % L),
// the row where my first (t, e) pair lands on r.
// Capacity: overflow[0] = the largest number of rows any owner would receive
// if that exceeds `cap`, else 0 (written every launch, so the flag never goes
// stale).  Every rank holds the same counts_all, so every rank reaches the
// same verdict.  Memory safety does not depend on the caller reacting: the
// receive segments are clamped to `cap` (the grouped GEMMs never touch rows
// >= cap), the dispatch drops rows >= cap and the combine skips them.
__global__ void ep_offsets_kernel(const int32_t* __restrict__ counts_all, int G, int E, int rank, long long cap,
                                  int32_t* __restrict__ recv_seg, int32_t* __restrict__ send_base,
                                  int32_t* __restrict__ overflow) {
  if (threadIdx.x != 0) return;
  const int L = E / G;
  long long run = 0;
  recv_seg[0] = 0;
  for (int l = 0; l < L; ++l) {
    for (int s = 0; s < G; ++s) run += counts_all[s * E + rank * L + l];
    recv_seg[l + 1] = (int32_t)(run < cap ? run : cap);
  }
  long long worst = 0;
  for (int r = 0; r < G; ++r) {
    long long base = 0;
    for (int l = 0; l < L; ++l)
      for (int s = 0; s < G; ++s) {
        if (s == rank) send_base[r * L + l] = (int32_t)(base < cap ? base : cap);
        base += counts_all[s * E + r * L + l];
      }
    if (base > worst) worst = base;
  }
  overflow[0] = worst > cap ? (int32_t)(worst < 0x7fffffffLL ? worst : 0x7fffffffLL) : 0;
}

// One warp per token: read x[t] once, store it to its k owners' receive rows.
__global__ void __launch_bounds__(256) ep_dispatch_kernel(
    const int32_t* __restrict__ idx, const int32_t* __restrict__ dst_local, const int32_t* __restrict__ offsets_local,
    const int32_t* __restrict__ send_base, int T, int k, int L, long long cap, const __nv_bfloat16* __restrict__ x,
    int d, __nv_bfloat16* const* __restrict__ peer_recv, int32_t* __restrict__ route_row) {
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nwarps) {
    __nv_bfloat16* dstp[8];
    int nk = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dstp[j] = nullptr;
      if (j < k) {
        const int e = idx[t * k + j];
        long row = (long)send_base[e] + (dst_local[t * k + j] - offsets_local[e]);
        if (row >= cap) row = -1;  // over capacity: dropped here, skipped by the combine
        if (lane == 0) route_row[t * k + j] = (int32_t)row;
        if (row >= 0) dstp[j] = peer_recv[e / L] + row * d;
        nk = j + 1;
      }
    }
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
        if (j >= nk) break;
        if (!dstp[j]) continue;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * 256;
          if (c < d) *reinterpret_cast<uint4*>(dstp[j] + c) = v[u];
        }
      }
    }
  }
}

// out[t] = sum_j w[t,j] * y_owner(j)[route_row[t,j]]  — rows read from the owners'
// memory; same operation order as K5 / the oracle combine.  route_row < 0
// (dropped for capacity) contributes nothing.
template <int K>
__global__ void __launch_bounds__(256) ep_combine_kernel(const int32_t* __restrict__ idx,
                                                         const int32_t* __restrict__ route_row,
                                                         const float* __restrict__ w, int T, int d, int L,
                                                         const __nv_bfloat16* const* __restrict__ peer_y,
                                                         __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nwarps) {
    const __nv_bfloat16* rows[K];
    float wj[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int rr = route_row[t * K + j];
      rows[j] = rr >= 0 ? peer_y[idx[t * K + j] / L] + (long)rr * d : nullptr;
      wj[j] = w[t * K + j];
    }
    for (int c = lane * 8; c < d; c += 256) {
      uint4 v[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        v[j] = rows[j] ? *reinterpret_cast<const uint4*>(rows[j] + c) : make_uint4(0u, 0u, 0u, 0u);
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        float f[8];
        bf16x8_to_f32(v[j], f);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(wj[j], f[q]));
      }
      uint4 o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                           pack_bf16x2(acc[6], acc[7]));
      *reinterpret_cast<uint4*>(out + t * (long)d + c) = o;
    }
  }
}

int launch_ep_counts_put(const int32_t* counts, int E, int rank, int world, int32_t* const* peer_counts,
                         cudaStream_t s) {
  ep_counts_put_kernel<<<1, 256, 0, s>>>(counts, E, rank, world, peer_counts);
  return launch_status();
}

int launch_ep_offsets(const int32_t* counts_all, int G, int E, int rank, long long cap, int32_t* recv_seg,
                      int32_t* send_base, int32_t* overflow, cudaStream_t s) {
  ep_offsets_kernel<<<1, 32, 0, s>>>(counts_all, G, E, rank, cap, recv_seg, send_base, overflow);
  return launch_status();
}

int launch_ep_dispatch(const int32_t* idx, const int32_t* dst_local, const int32_t* offsets_local,
                       const int32_t* send_base, int T, int k, int L, long long cap, const void* x, int d,
                       void* const* peer_recv, int32_t* route_row, cudaStream_t s) {
  if (T == 0) return 0;
  long blocks = (T + 7) / 8;
  if (blocks > 148L * 16) blocks = 148L * 16;
  ep_dispatch_kernel<<<(int)blocks, 256, 0, s>>>(idx, dst_local, offsets_local, send_base, T, k, L, cap,
                                                 static_cast<const __nv_bfloat16*>(x), d,
                                                 reinterpret_cast<__nv_bfloat16* const*>(peer_recv), route_row);
  return launch_status();
}

int launch_ep_combine(const int32_t* idx, const int32_t* route_row, const float* w, int T, int k, int d, int L,
                      const void* const* peer_y, void* out, cudaStream_t s) {
  if (T == 0) return 0;
  long blocks = (T + 7) / 8;
  if (blocks > 148L * 16) blocks = 148L * 16;
  const __nv_bfloat16* const* py = reinterpret_cast<const __nv_bfloat16* const*>(peer_y);
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
  switch (k) {
#define EPC(KK) \
  case KK: ep_combine_kernel<KK><<<(int)blocks, 256, 0, s>>>(idx, route_row, w, T, d, L, py, o); break;
    EPC(1) EPC(2) EPC(3) EPC(4) EPC(5) EPC(6) EPC(7) EPC(8)
#undef EPC
    default:
      return -1;
  }
  return launch_status();
}

}  // namespace cox
