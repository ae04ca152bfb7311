// K3+K4 for decode-size batches — one weight-streaming launch for the whole
// expert FFN (the paper's decode regime).
//
// At decode sizes (C4: 64 tokens, top-6 of 64 experts => ~6 rows per expert)
// the expert stage is bound by HBM, not by the tensor pipe: every touched
// expert's W13 and W2 must be streamed once (C4: 1.1 GB per layer) while the
// activations are a few KB.  The prefill kernel (grouped_gemm.cu) tiles
// M = 256 token rows x N = 256 weight rows; here the roles swap ("swap-AB"):
//
//   D[w, t] = sum_k W[w, k] * X[t, k]      M = 128 weight rows (TMEM lanes),
//                                          N = 16..64 tokens (TMEM columns)
//
// so one tcgen05.mma.cta_group::1 consumes a 128 x 64 weight tile and the
// segment's token rows, and the tensor pipe is idle most of the time while TMA
// keeps ~170 KB of weight tiles in flight per SM.
//
// Work units (one per 128 weight rows of one group):
//   SwiGLU pass: unit (g, i) = ff columns [64i, 64i+64) of group g: W13 rows of
//                the 64 gate columns (interleaved block i/2, half i%2) stacked on
//                the 64 matching up rows -> TMEM lanes 0-63 gate, 64-127 up.
//   down pass:   unit (g, i) = output columns [128i, 128i+128): W2 rows.
// All SwiGLU units come first in one persistent launch, then all down units;
// a down unit of group g waits (acquire on a per-group counter) until every
// SwiGLU unit of g has stored its h columns, so the W2 stream starts while the
// last W13 tiles are still in flight and there is no launch boundary or wave
// tail between the two GEMMs.  Units are claimed in order from a global atomic
// counter, so a waiting unit only ever waits on units already running.
//
// The shared experts of DeepSeek-style layers (dense MLP over all tokens) are
// one more group (expert id -1, rows [0, Ts) of x), in the same launch.
// Segments longer than 64 rows are processed in 64-row chunks (the weight tile
// is then re-read from L2).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace cox {

int get_map(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols, unsigned box_rows);

constexpr int SG_BM = 128;     // weight rows per unit (MMA M, TMEM lanes)
constexpr int SG_BK = 64;      // K per stage: one 128-byte swizzle atom of bf16
constexpr int SG_NMAX = 64;    // tokens per MMA chunk (MMA N <= 64)
constexpr int SG_STAGES = 8;
constexpr int SG_MAXG = 66;    // 64 routed groups + shared
constexpr int SG_THREADS = 256;
constexpr int SG_DEPTH = 4;    // unit-id ring between the scheduler and the roles
constexpr uint32_t SG_A_BYTES = SG_BM * SG_BK * 2;    // 16 KB
constexpr uint32_t SG_B_BYTES = SG_NMAX * SG_BK * 2;  // 8 KB
constexpr int SG_PITCH = 33;                          // fp32 staging row pitch (conflict-free)
constexpr uint32_t SG_TMEM_COLS = 2 * SG_NMAX;

struct alignas(64) SmallParams {
  CUtensorMap act3[2];  // SwiGLU B operand: [0] routed rows (x_perm), [1] shared-expert input (x)
  CUtensorMap act4[2];  // down B operand:   [0] h, [1] shared h
  CUtensorMap w13[SG_MAXG];
  CUtensorMap w2[SG_MAXG];
  const int32_t* offsets;
  int* counters;  // [0] unit counter, [1 + g] SwiGLU units of group g whose h columns are stored
  __nv_bfloat16* h[2];
  __nv_bfloat16* y[2];
  int group_expert[SG_MAXG];  // >= 0: routed expert (segment from offsets); -1: shared (rows [0, Ts))
  int group_ff[SG_MAXG];
  int n_groups;
  int Ts;
  int d;
  int phases;  // bit 0: SwiGLU pass, bit 1: down pass
};

constexpr size_t SG_SMEM_BYTES = 1024 + SG_STAGES * (SG_A_BYTES + SG_B_BYTES) + 512 + 16 * (SG_MAXG + 2) +
                                 4 * SG_BM * SG_PITCH + 64;

COX_DEV void mbar_spin_ge(const int* p, int want) {
  int v;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  } while (v < want);
}
COX_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
COX_DEV void named_bar_epi() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __launch_bounds__(SG_THREADS, 1) small_ffn_kernel(const __grid_constant__ SmallParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + SG_STAGES * SG_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + SG_STAGES * SG_B_BYTES);
  uint64_t* empty = full + SG_STAGES;
  uint64_t* tfull = empty + SG_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + SG_DEPTH;
  int* s_tile = reinterpret_cast<int*>(sempty + SG_DEPTH);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_tile + SG_DEPTH);
  int* s_rows = reinterpret_cast<int*>(tmem_slot + 4);
  int* s_row0 = s_rows + SG_MAXG;
  int* s_p3 = s_row0 + SG_MAXG;      // [G+1] prefix of SwiGLU units
  int* s_p4 = s_p3 + SG_MAXG + 1;    // [G+1] prefix of down units
  float* stg = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_p4 + SG_MAXG + 1) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = p.n_groups;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SG_STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 4);  // 4 epilogue warps
    }
    for (int i = 0; i < SG_DEPTH; ++i) {
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), 6);  // producer + MMA + 4 epilogue warps
    }
    fence_mbar_init();
    int a3 = 0, a4 = 0;
    for (int g = 0; g < G; ++g) {
      const int e = p.group_expert[g];
      const int r0 = e >= 0 ? p.offsets[e] : 0;
      const int rows = e >= 0 ? p.offsets[e + 1] - r0 : p.Ts;
      s_row0[g] = r0;
      s_rows[g] = rows;
      s_p3[g] = a3;
      s_p4[g] = a4;
      if (rows > 0) {
        if (p.phases & 1) a3 += p.group_ff[g] / 64;
        if (p.phases & 2) a4 += p.d / SG_BM;
      }
    }
    s_p3[G] = a3;
    s_p4[G] = a4;
  }
  if (warp == 2) tmem_alloc<1>(smem_u32(tmem_slot), SG_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t tmem_base = *tmem_slot;
  const int total3 = s_p3[G];
  const int total = total3 + s_p4[G];

  auto fetch = [&](int& si, bool arrive) -> int {
    const int slot = si % SG_DEPTH;
    mbar_wait(smem_u32(&sfull[slot]), (si / SG_DEPTH) & 1);
    const int t = reinterpret_cast<volatile int*>(s_tile)[slot];
    __syncwarp(__activemask());
    if (arrive) mbar_arrive(smem_u32(&sempty[slot]));
    ++si;
    return t;
  };
  // unit id -> (pass, group, index within the group)
  auto decode = [&](int t, int& pass, int& g, int& i) {
    const int* pre = s_p3;
    pass = 0;
    if (t >= total3) {
      t -= total3;
      pre = s_p4;
      pass = 1;
    }
    g = 0;
    while (t >= pre[g + 1]) ++g;
    i = t - pre[g];
  };

  if (warp == 3) {
    // ------------------------------------------------------------ unit scheduler
    if (lane == 0) {
      for (int i = 0;; ++i) {
        const int slot = i % SG_DEPTH;
        mbar_wait(smem_u32(&sempty[slot]), ((i / SG_DEPTH) & 1) ^ 1);
        // every unit comes from the counter (no static first wave): a unit is only
        // ever owned by a CTA that is running, which the down-pass waits rely on
        int t = atomicAdd(p.counters, 1);
        if (t > total) t = total;
        s_tile[slot] = t;
        mbar_arrive(smem_u32(&sfull[slot]));
        if (t >= total) break;
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      int si = 0;
      for (int t = fetch(si, true); t < total; t = fetch(si, true)) {
        int pass, g, i;
        decode(t, pass, g, i);
        const int rows = s_rows[g], row0 = s_row0[g];
        const int src = p.group_expert[g] < 0 ? 1 : 0;
        const CUtensorMap* wmap = pass == 0 ? &p.w13[g] : &p.w2[g];
        const CUtensorMap* amap = pass == 0 ? &p.act3[src] : &p.act4[src];
        const int nk = (pass == 0 ? p.d : p.group_ff[g]) / SG_BK;
        // weight rows of the two 64-row halves of the A tile
        const int wr0 = pass == 0 ? 256 * (i >> 1) + 64 * (i & 1) : SG_BM * i;
        const int wr1 = pass == 0 ? wr0 + 128 : wr0 + 64;
        bool dep_ok = !(pass == 1 && (p.phases & 1));
        for (int c0 = 0; c0 < rows; c0 += SG_NMAX) {
          const int nb = (min(SG_NMAX, rows - c0) + 15) >> 4;  // 16-row B boxes
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
            const uint32_t fb = smem_u32(&full[stage]);
            mbar_arrive_expect_tx(fb, SG_A_BYTES + nb * 2048u);
            const uint32_t a_dst = smem_u32(sA + stage * SG_A_BYTES);
            tma_load_2d(a_dst, wmap, fb, kb * SG_BK, wr0);
            tma_load_2d(a_dst + SG_A_BYTES / 2, wmap, fb, kb * SG_BK, wr1);
            if (!dep_ok) {
              // h columns of this group come from SwiGLU units of this launch
              mbar_spin_ge(p.counters + 1 + g, p.group_ff[g] / 64);
              fence_proxy_async_global();
              dep_ok = true;
            }
            const uint32_t b_dst = smem_u32(sB + stage * SG_B_BYTES);
            for (int b = 0; b < nb; ++b) tma_load_2d(b_dst + b * 2048u, amap, fb, kb * SG_BK, row0 + c0 + 16 * b);
            if (++stage == SG_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      int si = 0, job = 0;
      for (int t = fetch(si, true); t < total; t = fetch(si, true)) {
        int pass, g, i;
        decode(t, pass, g, i);
        const int rows = s_rows[g];
        const int nk = (pass == 0 ? p.d : p.group_ff[g]) / SG_BK;
        for (int c0 = 0; c0 < rows; c0 += SG_NMAX, ++job) {
          const int npad = ((min(SG_NMAX, rows - c0) + 15) >> 4) << 4;
          const uint32_t idesc = idesc_bf16_f32(SG_BM, npad);
          const int acc = job & 1;
          mbar_wait(smem_u32(&tempty[acc]), ((job >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * SG_NMAX;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + stage * SG_A_BYTES);
            const uint32_t b_base = smem_u32(sB + stage * SG_B_BYTES);
#pragma unroll
            for (int k = 0; k < SG_BK / 16; ++k)
              mma_bf16_ss<1>(d_tmem, sdesc_kmajor_sw128(a_base + k * 32), sdesc_kmajor_sw128(b_base + k * 32), idesc,
                             (kb | k) != 0 ? 1u : 0u);
            mma_commit<1>(smem_u32(&empty[stage]));
            if (++stage == SG_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit<1>(smem_u32(&tfull[acc]));
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // Warp q reads TMEM lanes 32q..32q+31 (= weight rows of the unit), 32
    // token columns at a time, into a shared fp32 tile [128 rows][32 tokens];
    // then the 128 threads write whole 16-byte row pieces of the outputs.
    const int q = warp - 4;
    const int tid = threadIdx.x - 128;
    const int r = q * 32 + lane;
    int si = 0, job = 0;
    for (int t = fetch(si, lane == 0); t < total; t = fetch(si, lane == 0)) {
      int pass, g, i;
      decode(t, pass, g, i);
      const int rows = s_rows[g], row0 = s_row0[g];
      const int src = p.group_expert[g] < 0 ? 1 : 0;
      for (int c0 = 0; c0 < rows; c0 += SG_NMAX, ++job) {
        const int acc = job & 1;
        mbar_wait(smem_u32(&tfull[acc]), (job >> 1) & 1);
        tc_fence_after();
        const int nrem = min(SG_NMAX, rows - c0);
        for (int c32 = 0; c32 < nrem; c32 += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * SG_NMAX + c32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[r * SG_PITCH + j] = __uint_as_float(v[j]);
          named_bar_epi();
          const int nt = min(32, nrem - c32);
          const long long tok0 = (long long)row0 + c0 + c32;
          if (pass == 0) {
            const int ff = p.group_ff[g];
            __nv_bfloat16* hbase = p.h[src] + (long long)i * 64;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
              const int idx = tid + 128 * pp, tt = idx >> 3, cg = idx & 7;
              if (tt < nt) {
                uint32_t pk[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int c = cg * 8 + 2 * j;
                  const float g0 = stg[c * SG_PITCH + tt], g1 = stg[(c + 1) * SG_PITCH + tt];
                  const float u0 = stg[(64 + c) * SG_PITCH + tt], u1 = stg[(65 + c) * SG_PITCH + tt];
                  pk[j] = pack_bf16x2(g0 * __frcp_rn(1.0f + __expf(-g0)) * u0, g1 * __frcp_rn(1.0f + __expf(-g1)) * u1);
                }
                st_global_v4(hbase + (tok0 + tt) * ff + cg * 8, pk[0], pk[1], pk[2], pk[3]);
              }
            }
          } else {
            __nv_bfloat16* ybase = p.y[src] + (long long)i * SG_BM;
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
              const int idx = tid + 128 * pp, tt = idx >> 4, cg = idx & 15;
              if (tt < nt) {
                uint32_t pk[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int c = cg * 8 + 2 * j;
                  pk[j] = pack_bf16x2(stg[c * SG_PITCH + tt], stg[(c + 1) * SG_PITCH + tt]);
                }
                st_global_v4(ybase + (tok0 + tt) * p.d + cg * 8, pk[0], pk[1], pk[2], pk[3]);
              }
            }
          }
          named_bar_epi();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      }
      if (pass == 0 && (p.phases & 2)) {
        // publish this unit's h columns to the down units of group g (their
        // B operand is read by TMA, i.e. through the async proxy)
        fence_proxy_async_global();
        named_bar_epi();
        if (tid == 0) {
          __threadfence();
          atomicAdd(p.counters + 1 + g, 1);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, SG_TMEM_COLS);
  }
}

static int g_sg_sms = 0;

// act: routed rows [rows_cap, d] (x_perm); h: [rows_cap, ff]; y: [rows_cap, d].
// Optional shared expert group (xs != nullptr): xs [Ts, d], w13s [2 ffs, d],
// w2s [d, ffs], hs [Ts, ffs], ys [Ts, d].
int launch_small_ffn(const void* act, long long rows_cap, const int32_t* offsets, int n_groups,
                     const int32_t* group_expert, const void* const* w13, const void* const* w2, int d, int ff,
                     void* h, void* y, const void* xs, int Ts, const void* w13s, const void* w2s, int ffs, void* hs,
                     void* ys, int phases, cudaStream_t s) {
  const int G = n_groups + (xs ? 1 : 0);
  if (G == 0) return 0;
  static SmallParams p;  // 17 KB of tensor maps: built in static storage, copied at launch
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int rc = 0;
  if (n_groups > 0) {
    if ((rc = get_map(&p.act3[0], act, rows_cap, d, 16))) return rc;
    if ((rc = get_map(&p.act4[0], h, rows_cap, ff, 16))) return rc;
  }
  for (int g = 0; g < n_groups; ++g) {
    if ((rc = get_map(&p.w13[g], w13[g], 2ull * ff, d, 64))) return rc;
    if ((rc = get_map(&p.w2[g], w2[g], d, ff, 64))) return rc;
    p.group_expert[g] = group_expert[g];
    p.group_ff[g] = ff;
  }
  if (xs) {
    if ((rc = get_map(&p.act3[1], xs, Ts, d, 16))) return rc;
    if ((rc = get_map(&p.act4[1], hs, Ts, ffs, 16))) return rc;
    if ((rc = get_map(&p.w13[n_groups], w13s, 2ull * ffs, d, 64))) return rc;
    if ((rc = get_map(&p.w2[n_groups], w2s, d, ffs, 64))) return rc;
    p.group_expert[n_groups] = -1;
    p.group_ff[n_groups] = ffs;
  }
  static int* counters = nullptr;
  static unsigned seq = 0;
  constexpr int SLOT = 128;
  if (!counters) {
    if (cudaMalloc(&counters, 256 * SLOT * sizeof(int)) != cudaSuccess) return -2;
  }
  int* c = counters + (seq++ % 256) * SLOT;
  if (cudaMemsetAsync(c, 0, (1 + G) * sizeof(int), s) != cudaSuccess) return -2;
  p.counters = c;
  p.offsets = offsets;
  p.h[0] = static_cast<__nv_bfloat16*>(h);
  p.h[1] = static_cast<__nv_bfloat16*>(hs);
  p.y[0] = static_cast<__nv_bfloat16*>(y);
  p.y[1] = static_cast<__nv_bfloat16*>(ys);
  p.n_groups = G;
  p.Ts = Ts;
  p.d = d;
  p.phases = phases;
  if (g_sg_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sg_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sg_sms <= 0) g_sg_sms = 148;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(small_ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SG_SMEM_BYTES);
    attr = true;
  }
  small_ffn_kernel<<<g_sg_sms, SG_THREADS, SG_SMEM_BYTES, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace cox
