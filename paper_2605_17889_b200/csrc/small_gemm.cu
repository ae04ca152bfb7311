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
// one more group (expert id -1, rows [0, Ts) of x), placed first.  Segments
// longer than 64 rows are processed in 64-row chunks (the weight tile is then
// re-read from L2).  Routed rows are gathered from x by TMA tile::gather4
// (row_tokens) or read from a materialised x_perm.  The CTA that stores the
// last down tile of a 128-column block combines that block for every token
// (same operation order as combine_kernel).
//
// Dense mode (cox_decode_moe): every group runs over all T <= 64 tokens and
// warp 2 routes token blockIdx.x in the canonical order, so the router is off
// the critical path; only the combine waits for it.  Routed mode is launched
// as a programmatic dependent of the permute (griddepcontrol).
//
// Host side: tensor maps in a content-keyed global table (not 17 KB of kernel
// parameters), counters reset by the last CTA to exit (no memset node).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "route_common.cuh"

namespace cox {

int get_map(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols, unsigned box_rows);
int launch_combine(const void* y_perm, const int32_t* dst, const float* w, int T, int k, int d, const void* shared,
                   void* out, int out_is_bf16, cudaStream_t s);

constexpr int SG_BM = 128;     // weight rows per unit (MMA M, TMEM lanes)
constexpr int SG_ATOM = 64;    // K of one 128-byte swizzle atom of bf16
constexpr uint32_t SG_RING_BYTES = 200 * 1024;  // smem for the TMA ring
constexpr int SG_MAXG = 66;    // 64 routed groups + shared
constexpr int SG_THREADS = 256;
constexpr int SG_DEPTH = 4;    // unit-id ring between the scheduler and the roles
constexpr uint32_t SG_A_ATOM = SG_BM * SG_ATOM * 2;  // 16 KB: one K atom of the weight tile
constexpr int SG_PITCH = 33;                         // fp32 staging row pitch (conflict-free)
constexpr int SG_MAX_PAIRS = 2048;                   // T*k of the from_idx path (T <= 256, k <= 8)

// KA = K atoms per pipeline stage (BK = 64 KA: contiguous bytes per weight row
// per stage), NMAX = tokens per MMA chunk (MMA N <= NMAX).
template <int KA, int NMAX>
struct SgCfg {
  static constexpr int BK = SG_ATOM * KA;
  static constexpr uint32_t A_STAGE = SG_A_ATOM * KA;
  static constexpr uint32_t B_ATOM = NMAX * SG_ATOM * 2;
  static constexpr uint32_t B_STAGE = B_ATOM * KA;
  static constexpr int STAGES = (int)(SG_RING_BYTES / (A_STAGE + B_STAGE)) > 12 ? 12
                                                                               : (int)(SG_RING_BYTES / (A_STAGE + B_STAGE));
  static constexpr uint32_t TMEM_COLS = 2 * NMAX < 64 ? 64 : 2 * NMAX;
  static constexpr size_t SMEM = 1024 + STAGES * (A_STAGE + B_STAGE) + 512 + 1120 + 4 * SG_MAX_PAIRS + 1024 + 32 +
                                 256 + 24 * (SG_MAXG + 2) +
                                 4 * SG_BM * SG_PITCH + 64;
};

// Tensor maps live in a global-memory table (17 KB), not in the kernel
// parameters: a 17 KB parameter block costs every launch; the table for a given
// set of operands is uploaded once and reused (graph replays included).
struct alignas(128) SmallMaps {
  CUtensorMap act3[2];  // SwiGLU B operand: [0] routed rows (x_perm, or x for gather4), [1] shared-expert input (x)
  CUtensorMap act4[2];  // down B operand:   [0] h, [1] shared h
  CUtensorMap w13[SG_MAXG];
  CUtensorMap w2[SG_MAXG];
};

struct SmallParams {
  const SmallMaps* maps;
  const int32_t* offsets;
  int* counters;  // [0] unit counter, [1 + g] SwiGLU units of group g whose h columns are stored,
                  // [SG_CB_BASE + i] down tiles of column block i, [SG_COUNTERS - 1] exit ticket;
                  // zero at launch, reset by the last CTA to exit
  __nv_bfloat16* h[2];
  __nv_bfloat16* y[2];
  const int32_t* row_tokens;  // gather mode: routed row r of the SwiGLU pass is x[row_tokens[r]] (act3[0] = x)
  long long rows_cap;
  // fused combine (out != nullptr): out[t, cols of block i] = sum_j w[t,j] y[dst[t,j]] (+ y_shared[t]),
  // done by the CTA that stores the last down tile of column block i
  const int32_t* cdst;
  const float* cw;
  __nv_bfloat16* out;
  int k;
  int T;
  // dense decode (dense != 0): every group runs over all T tokens (B = x rows
  // [0, T); routed group g writes h/y rows [(g - g0) T, +T)) and warp 2 of CTA
  // b routes token b (canonical order, like router_topk_kernel) into ridx/rw;
  // the combine reads y[(expert_slot[e]) T + t]
  int dense;
  const __nv_bfloat16* wg;  // [E, d] bf16 router weight
  const __nv_bfloat16* xtok;  // [T, d] the step's tokens
  int E;
  int mode;
  int32_t* ridx;  // [T, k]
  float* rw;      // [T, k]
  int16_t expert_slot[256];  // routed expert -> its row block in h/y (dense)
  // Launched as a programmatic dependent of the permute (pdl != 0): CTAs may
  // become resident while the routing kernels still run and wait (griddepcontrol)
  // before reading their outputs.  Measured: -3 us/step eager, neutral under a
  // CUDA graph; also prefetching the first units' weights into L2 during the
  // wait was tried and was slower (1 unit/CTA +2 us, 2: +4 us, 4: +10 us).
  int pdl;
  // before waiting for the router, every CTA prefetches its share of the shared
  // experts' weight boxes into L2 (routing-independent bytes; measured C4D
  // 196.96 -> 196.35 us, 3 same-box A/B pairs)
  int prefetch_shared;
  // from_idx != 0: no permute kernel ran.  Segments come from the router's
  // counts (expert-ascending offsets, written to offsets_out by CTA 0), the
  // producer of a routed SwiGLU unit collects its expert's tokens from ridx
  // (ascending token order, like the permute) and gathers their rows from x,
  // and the producer of unit 0 of each group writes the group's dst entries
  // for the combine.
  int from_idx;
  const int32_t* rcounts;  // [E]
  int32_t* dst_out;        // [T, k]
  int32_t* offsets_out;    // [E + 1]
  int group_expert[SG_MAXG];  // >= 0: routed expert (segment from offsets); -1: shared (rows [0, Ts))
  int group_ff[SG_MAXG];
  int n_groups;
  int Ts;
  int d;
  int phases;  // bit 0: SwiGLU pass, bit 1: down pass
};
constexpr int SG_CB_BASE = 1 + SG_MAXG;  // counters[SG_CB_BASE + i]: down tiles stored in column block i
constexpr int SG_COUNTERS = 256;
constexpr int SG_ROUTED = SG_COUNTERS - 2;  // dense: tokens routed so far
constexpr int SG_CTICKET = SG_COUNTERS - 3; // fused combine: work-item ticket


COX_DEV void mbar_spin_ge(const int* p, int want) {
  int v;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  } while (v < want);
}
COX_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
COX_DEV void named_bar_epi() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
COX_DEV void tma_gather4(uint32_t dst, const void* map, uint32_t bar, int32_t col, int32_t r0, int32_t r1, int32_t r2,
                         int32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
COX_DEV uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int KA, int NMAX>
__global__ void __launch_bounds__(SG_THREADS, 1) small_ffn_kernel(const __grid_constant__ SmallParams p) {
  using C = SgCfg<KA, NMAX>;
  constexpr int SG_STAGES = C::STAGES;
  constexpr int SG_BK = C::BK;
  constexpr int SG_NMAX = NMAX;
  constexpr uint32_t SG_A_BYTES = C::A_STAGE;
  constexpr uint32_t SG_B_BYTES = C::B_STAGE;
  constexpr uint32_t SG_TMEM_COLS = C::TMEM_COLS;
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
  int* s_misc = s_p4 + SG_MAXG + 1;  // [0] groups with rows, [1] combine flag
  int* s_act = s_misc + 4;            // [G] active groups (rows > 0), in group order
  float* s_route = reinterpret_cast<float*>(s_act + SG_MAXG);  // [280] dense: logits of the token being routed
                                                                 //   (+ top-k scratch at 264..279);
  int* s_eoff = reinterpret_cast<int*>(s_route);                 //   from_idx: expert offsets [E + 1]
  // from_idx: the stable permutation, computed once per CTA by warp 2:
  // s_perm[row] = token of permuted row (expert-major, ascending tokens),
  // s_pos[t*k + j] = permuted row of (t, j)
  int16_t* s_perm = reinterpret_cast<int16_t*>(s_route + 280);   // [SG_MAX_PAIRS]
  int16_t* s_pos = s_perm + SG_MAX_PAIRS;                         // [SG_MAX_PAIRS]
  int* s_erun = reinterpret_cast<int*>(s_pos + SG_MAX_PAIRS);     // [256] running row per expert
  uint64_t* perm_ready = reinterpret_cast<uint64_t*>(s_erun + 256);
  float* stg = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(perm_ready + 1) + 15) & ~uintptr_t(15));

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
    mbar_init(smem_u32(perm_ready), 1);
    fence_mbar_init();
  }
  // dense decode: warp 2 routes tokens blockIdx.x, + gridDim.x, ... in the
  // canonical order, beside the weight stream (only the combine waits for it)
  auto route_tokens = [&]() {
    const int d = p.d, E = p.E, kk = p.k;
    for (int t = blockIdx.x; t < p.T; t += gridDim.x) {
      const __nv_bfloat16* xr = p.xtok + (long long)t * d;
      for (int e0 = 0; e0 < E; e0 += 8) {
        float acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.f;
#pragma unroll 2
        for (int sc = 8 * lane; sc < d; sc += 256) {
          float xv[8];
          bf16x8_to_f32(ld_nc_v4(xr + sc), xv);
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            float wa[8], wb[8];
            const int ea = min(e0 + u, E - 1), eb = min(e0 + u + 1, E - 1);
            bf16x8_to_f32(ld_nc_v4(p.wg + (long long)ea * d + sc), wa);
            bf16x8_to_f32(ld_nc_v4(p.wg + (long long)eb * d + sc), wb);
#pragma unroll
            for (int q = 0; q < 8; ++q) ffma2(acc[u], acc[u + 1], xv[q], wa[q], wb[q]);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float v = acc[u];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == 0 && e0 + u < E) s_route[e0 + u] = v != v ? -INFINITY : v;  // NaN ranks like -inf
        }
      }
      __syncwarp();
      warp_route_token_e(s_route, E, kk, p.mode, lane, reinterpret_cast<int*>(s_route + 264), s_route + 272,
                       p.ridx + t * kk, p.rw + t * kk, nullptr);
      if (lane == 0) red_release_add(p.counters + SG_ROUTED, 1);  // after idx / w / histogram
      __syncwarp();
    }
  };
  // barrier init and the TMEM allocation do not depend on the routing: done
  // while the router (the PDL primary) is still running
  if (warp == 2) tmem_alloc<1>(smem_u32(tmem_slot), SG_TMEM_COLS);
  if (p.pdl && p.prefetch_shared && p.Ts > 0 && threadIdx.x == 0) {
    const int cb = p.d / 64, ff = p.group_ff[0];
    const int nb13 = (2 * ff / 64) * cb, nb2 = (p.d / 64) * (ff / 64);
    for (int b = blockIdx.x; b < nb13 + nb2; b += gridDim.x) {
      const CUtensorMap* m = b < nb13 ? &p.maps->w13[0] : &p.maps->w2[0];
      const int bb = b < nb13 ? b : b - nb13, w = b < nb13 ? cb : ff / 64;
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                       reinterpret_cast<uint64_t>(m)), "r"((bb % w) * 64), "r"((bb / w) * 64)
                   : "memory");
    }
  }
  if (p.pdl) {
    pdl_wait();  // routing (offsets, row_tokens, dst, w) of this step is complete from here on
  }
  if (warp == 0) {
    if (p.from_idx) {
      // expert offsets from the router's counts (exclusive scan, 8 experts per lane)
      int loc[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = lane * 8 + q;
        loc[q] = e < p.E ? p.rcounts[e] : 0;
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
        if (e <= p.E) {
          s_eoff[e] = run;
          if (blockIdx.x == 0 && p.offsets_out) p.offsets_out[e] = run;
        }
        run += loc[q];
      }
      __syncwarp();
    }
    // group table: rows / first row per group and the unit prefix sums, one
    // group per lane (a serial loop would pay one L2 round trip per group)
    int c3 = 0, c4 = 0, nact = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      int rows = 0, r0 = 0;
      if (g < G) {
        const int e = p.group_expert[g];
        if (p.dense) {
          rows = p.T;
          r0 = e >= 0 ? p.expert_slot[e] * p.T : 0;
        } else if (p.from_idx) {
          r0 = e >= 0 ? s_eoff[e] : 0;
          rows = e >= 0 ? s_eoff[e + 1] - r0 : p.Ts;
        } else {
          r0 = e >= 0 ? p.offsets[e] : 0;
          rows = e >= 0 ? p.offsets[e + 1] - r0 : p.Ts;
        }
        s_row0[g] = r0;
        s_rows[g] = rows;
      }
      const uint32_t live = __ballot_sync(0xffffffffu, g < G && rows > 0);
      if (g < G && rows > 0) s_act[nact + __popc(live & ((1u << lane) - 1u))] = g;
      nact += __popc(live);
      int u3 = (g < G && rows > 0 && (p.phases & 1)) ? p.group_ff[g < G ? g : 0] / 64 : 0;
      int u4 = (g < G && rows > 0 && (p.phases & 2)) ? p.d / SG_BM : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive warp scans
        const int a = __shfl_up_sync(0xffffffffu, u3, o), b = __shfl_up_sync(0xffffffffu, u4, o);
        if (lane >= o) {
          u3 += a;
          u4 += b;
        }
      }
      if (g < G) {
        s_p3[g + 1] = c3 + u3;
        s_p4[g + 1] = c4 + u4;
      }
      c3 += __shfl_sync(0xffffffffu, u3, 31);
      c4 += __shfl_sync(0xffffffffu, u4, 31);
    }
    if (lane == 0) {
      s_p3[0] = 0;
      s_p4[0] = 0;
      s_misc[0] = nact;
    }
  }
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
    int lo = 0, hi = G;  // largest g with pre[g] <= t (empty groups have pre[g] == pre[g + 1])
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= t) lo = mid; else hi = mid;
    }
    g = lo;
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
    // Lane 0 issues the weight tiles and tiled activation boxes; in gather mode
    // lanes 0..4nb-1 each issue one tile::gather4 (4 token rows of x) per atom.
    uint32_t stage = 0, phase = 0;
    int si = 0;
    bool perm_seen = false;
    // expert weights are read once per step: evict_first keeps x, h, y, the
    // router weight and the counters in L2
    const uint64_t wpol = l2_policy_evict_first();
    for (;;) {
      int t = lane == 0 ? fetch(si, true) : 0;
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= total) break;
      int pass, g, i;
      decode(t, pass, g, i);
      const int rows = s_rows[g], row0 = s_row0[g];
      const int src = p.group_expert[g] < 0 ? 1 : 0;
      const bool gat = pass == 0 && src == 0 && !p.dense && (p.row_tokens != nullptr || p.from_idx);
      if (gat && p.from_idx && !perm_seen) {
        mbar_wait(smem_u32(perm_ready), 0);  // warp 2 has built this CTA's copy of the permutation
        perm_seen = true;
      }
      const CUtensorMap* wmap = pass == 0 ? &p.maps->w13[g] : &p.maps->w2[g];
      const CUtensorMap* amap = pass == 0 ? &p.maps->act3[p.dense ? 1 : src] : &p.maps->act4[src];
      const int brow0 = (pass == 0 && p.dense) ? 0 : row0;  // dense SwiGLU: B = x rows [0, T)
      const int K = pass == 0 ? p.d : p.group_ff[g];
      const int nk = (K + SG_BK - 1) / SG_BK;  // the last stage may hold fewer than KA atoms
      // weight rows of the two 64-row halves of the A tile
      const int wr0 = pass == 0 ? 256 * (i >> 1) + 64 * (i & 1) : SG_BM * i;
      const int wr1 = pass == 0 ? wr0 + 128 : wr0 + 64;
      bool dep_ok = !(pass == 1 && (p.phases & 1));
      for (int c0 = 0; c0 < rows; c0 += SG_NMAX) {
        const int nb = (min(SG_NMAX, rows - c0) + 15) >> 4;  // 16-row B boxes
        int rr[4] = {0, 0, 0, 0};
        if (gat && p.from_idx) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = c0 + 4 * lane + q;
            rr[q] = (lane < 4 * nb && r < rows) ? (int)s_perm[row0 + r] : 0;
          }
        } else if (gat) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long r = (long long)row0 + c0 + 4 * lane + q;
            rr[q] = (lane < 4 * nb && r < p.rows_cap) ? p.row_tokens[r] : 0;
          }
        }
        // Down tile whose h rows may still be in production: stream the first
        // weight stages (A only) while waiting, then add their B boxes.
        int npre = 0;
        if (!dep_ok && lane == 0) {
          const int* cnt = p.counters + 1 + g;
          const int want = p.group_ff[g] / 64;
          int v;
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          if (v < want) {
            npre = min(nk, SG_STAGES);
            uint32_t st0 = stage, ph0 = phase;
            for (int kb = 0; kb < npre; ++kb) {
              mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
              const uint32_t fb = smem_u32(&full[stage]);
              const int na = min(KA, (K - kb * SG_BK) / SG_ATOM);
              mbar_arrive_expect_tx(fb, na * (SG_A_ATOM + nb * 2048u));
              const uint32_t a_dst = smem_u32(sA + stage * SG_A_BYTES);
              for (int a = 0; a < na; ++a) {
                tma_load_2d_hint(a_dst + a * SG_A_ATOM, wmap, fb, kb * SG_BK + a * SG_ATOM, wr0, wpol);
                tma_load_2d_hint(a_dst + a * SG_A_ATOM + SG_A_ATOM / 2, wmap, fb, kb * SG_BK + a * SG_ATOM, wr1, wpol);
              }
              if (++stage == SG_STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
            mbar_spin_ge(cnt, want);
            fence_proxy_async_global();
            for (int kb = 0; kb < npre; ++kb) {
              const uint32_t fb = smem_u32(&full[st0]);
              const int na = min(KA, (K - kb * SG_BK) / SG_ATOM);
              const uint32_t b_dst = smem_u32(sB + st0 * SG_B_BYTES);
              for (int a = 0; a < na; ++a)
                for (int b = 0; b < nb; ++b)
                  tma_load_2d(b_dst + a * C::B_ATOM + b * 2048u, amap, fb, kb * SG_BK + a * SG_ATOM,
                              brow0 + c0 + 16 * b);
              if (++st0 == SG_STAGES) {
                st0 = 0;
                ph0 ^= 1;
              }
            }
          } else {
            fence_proxy_async_global();
          }
        }
        dep_ok = true;
        npre = __shfl_sync(0xffffffffu, npre, 0);
        stage = __shfl_sync(0xffffffffu, stage, 0);
        phase = __shfl_sync(0xffffffffu, phase, 0);
        for (int kb = npre; kb < nk; ++kb) {
          if (lane == 0) mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          __syncwarp();
          const uint32_t fb = smem_u32(&full[stage]);
          const int na = min(KA, (K - kb * SG_BK) / SG_ATOM);
          const uint32_t b_dst = smem_u32(sB + stage * SG_B_BYTES);
          if (lane == 0) {
            mbar_arrive_expect_tx(fb, na * (SG_A_ATOM + nb * 2048u));
            const uint32_t a_dst = smem_u32(sA + stage * SG_A_BYTES);
#pragma unroll
            for (int a = 0; a < KA; ++a) {
              if (a >= na) break;
              tma_load_2d_hint(a_dst + a * SG_A_ATOM, wmap, fb, kb * SG_BK + a * SG_ATOM, wr0, wpol);
              tma_load_2d_hint(a_dst + a * SG_A_ATOM + SG_A_ATOM / 2, wmap, fb, kb * SG_BK + a * SG_ATOM, wr1, wpol);
            }
            if (!gat) {
#pragma unroll
              for (int a = 0; a < KA; ++a)
                for (int b = 0; b < nb && a < na; ++b)
                  tma_load_2d(b_dst + a * C::B_ATOM + b * 2048u, amap, fb, kb * SG_BK + a * SG_ATOM,
                              brow0 + c0 + 16 * b);
            }
          }
          if (gat && lane < 4 * nb) {
            __syncwarp(__activemask());
#pragma unroll
            for (int a = 0; a < KA; ++a)
              if (a < na)
                tma_gather4(b_dst + a * C::B_ATOM + lane * 512u, amap, fb, kb * SG_BK + a * SG_ATOM, rr[0], rr[1],
                            rr[2], rr[3]);
          }
          __syncwarp();
          if (++stage == SG_STAGES) {
            stage = 0;
            phase ^= 1;
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
        const int K = pass == 0 ? p.d : p.group_ff[g];
        const int nk = (K + SG_BK - 1) / SG_BK;
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
            const int nkk = min(KA, (K - kb * SG_BK) / SG_ATOM) * (SG_ATOM / 16);
#pragma unroll
            for (int k = 0; k < SG_BK / 16; ++k)
              if (k < nkk)
                mma_bf16_ss<1>(d_tmem, sdesc_kmajor_sw128(a_base + (k >> 2) * SG_A_ATOM + (k & 3) * 32),
                             sdesc_kmajor_sw128(b_base + (k >> 2) * C::B_ATOM + (k & 3) * 32), idesc,
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
  } else if (warp == 2) {
    if (p.from_idx) {
      // ---------------------------------------------------------- stable permutation (from_idx)
      // Entries in (t, j) order, 32 at a time: rank among earlier entries of
      // the same expert = running count + peers before me in this chunk
      // (match_any), so rows are expert-major with ascending tokens -- the
      // order of permute.cu / the oracle.  Every CTA keeps its own copy; CTA 0
      // also publishes dst for the caller.
      for (int e = lane; e < p.E; e += 32) s_erun[e] = s_eoff[e];
      __syncwarp();
      const int nent = p.T * p.k;
      constexpr int PB = 8;  // chunks whose idx loads are in flight together (one L2 round trip per 256 entries)
      for (int c0 = 0; c0 < nent; c0 += 32 * PB) {
      int ev[PB];
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        const int ent = c0 + 32 * b + lane;
        ev[b] = ent < nent ? __ldg(p.ridx + ent) : -1;
      }
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        const int c = c0 + 32 * b;
        if (c >= nent) break;
        const int ent = c + lane;
        const int e = ev[b];
        const uint32_t peers = __match_any_sync(0xffffffffu, e);
        const int before = __popc(peers & ((1u << lane) - 1u));
        int row = -1;
        if (e >= 0 && e < p.E) row = s_erun[e] + before;
        __syncwarp();
        if (e >= 0 && e < p.E && before == 0) s_erun[e] += __popc(peers);
        if (ent < nent) {
          s_pos[ent] = (int16_t)row;
          if (row >= 0) s_perm[row] = (int16_t)(ent / p.k);
          if (blockIdx.x == 0) p.dst_out[ent] = row;
        }
        __syncwarp();
      }
      }
      if (lane == 0) mbar_arrive(smem_u32(perm_ready));  // release: the arrays are visible to waiters
    }
    // ------------------------------------------------------------ dense decode: in-kernel router
    // Token t = blockIdx.x (+ gridDim.x ...): logits in the canonical order of
    // router_topk_kernel (lane chunks s = 8 lane + 256 j, fma ascending, xor
    // butterfly; expert pairs share one FFMA2), top-k with ties to the lower
    // index, Mixtral / DeepSeek weights.  Only the combine needs the result, so
    // this runs beside the weight stream instead of before it.
    if (p.dense) route_tokens();
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
                  pk[j] = pack_bf16x2(silu_fast(g0) * u0, silu_fast(g1) * u1);
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
      if (pass == 1 && p.out) {
        // publish this down tile of column block i to the fused combine
        // (end of the kernel): release after all epilogue threads' y stores
        named_bar_epi();
        if (tid == 0) {
          __threadfence();
          atomicAdd(p.counters + SG_CB_BASE + i, 1);
        }
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
  // ------------------------------------------------------------ fused combine
  // out[t, block] = sum_j w[t,j] y[row(t,j), block] (+ y_shared[t, block]) in
  // ascending j with separately rounded mul/add -- combine_kernel's order, so
  // the same bits.  Work items (column block, 16 tokens) are claimed from a
  // global ticket by every CTA that has finished its units; an item waits
  // (acquire) until all down tiles of its block are stored, so the combine of
  // the last blocks is spread over all SMs instead of trailing on one CTA.
  if (p.out) {
    const int T = p.T, kk = p.k, d = p.d;
    const int tid = threadIdx.x;
    int* s_dst = reinterpret_cast<int*>(stg);
    float* s_w = reinterpret_cast<float*>(stg) + T * kk;
    int* s_item = s_misc + 3;
    if (p.dense && tid == 0) mbar_spin_ge(p.counters + SG_ROUTED, T);  // routing of every token done
    if (p.from_idx) mbar_wait(smem_u32(perm_ready), 0);              // this CTA's permutation is built
    __syncthreads();
    __threadfence();
    for (int e = tid; e < T * kk; e += SG_THREADS) {
      if (p.dense) {
        s_dst[e] = p.expert_slot[p.ridx[e]] * T + e / kk;
        s_w[e] = p.rw[e];
      } else if (p.from_idx) {
        s_dst[e] = s_pos[e];
        s_w[e] = p.cw[e];
      } else {
        s_dst[e] = __ldcg(p.cdst + e);
        s_w[e] = p.cw[e];
      }
    }
    const int ngrp = (T + 15) / 16;
    const int nitems = (d / SG_BM) * ngrp;
    const __nv_bfloat16* y0 = p.y[0];
    const __nv_bfloat16* ys = p.y[1];
    for (;;) {
      __syncthreads();  // staging done / previous item consumed
      if (tid == 0) {
        const int item = atomicAdd(p.counters + SG_CTICKET, 1);
        if (item < nitems) mbar_spin_ge(p.counters + SG_CB_BASE + item / ngrp, s_misc[0]);
        s_item[0] = item;
      }
      __syncthreads();
      const int item = s_item[0];
      if (item >= nitems) break;
      __threadfence();
      const int blk = item / ngrp;
      const int tt = (item % ngrp) * 16 + (tid >> 4);
      const int col = blk * SG_BM + (tid & 15) * 8;
      if (tt < T) {
        uint4 v[9];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < kk) v[j] = ld_cg_v4(y0 + (long long)s_dst[tt * kk + j] * d + col);
        if (ys) v[8] = ld_cg_v4(ys + (long long)tt * d + col);
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= kk) break;
          const float wj = s_w[tt * kk + j];
          float f[8];
          bf16x8_to_f32(v[j], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(wj, f[q]));
        }
        if (ys) {
          float f[8];
          bf16x8_to_f32(v[8], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], f[q]);
        }
        st_global_v4(p.out + (long long)tt * d + col, pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                     pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
      }
    }
  }
  if (threadIdx.x == 0) {
    // the last CTA to exit zeroes the counters for the next launch (no memset node)
    __threadfence();
    const int ticket = atomicAdd(p.counters + SG_COUNTERS - 1, 1);
    if (ticket == (int)gridDim.x - 1) {
      __threadfence();
      const int n = SG_CB_BASE + p.d / SG_BM;
      for (int c = 0; c < n; ++c) p.counters[c] = 0;
      p.counters[SG_ROUTED] = 0;
      p.counters[SG_CTICKET] = 0;
      p.counters[SG_COUNTERS - 1] = 0;
    }
  }
}

static int g_sg_sms = 0;

// Device copies of map tables, keyed by content: a table is uploaded (stream-
// ordered, from its own pinned host copy) the first time a set of operands is
// seen and kept for the life of the process, so a kernel node captured in a
// CUDA graph always finds its table unchanged (no eviction).
static const SmallMaps* upload_maps(const SmallMaps& m, cudaStream_t s) {
  struct Slot {
    SmallMaps* host;
    SmallMaps* dev;
  };
  static std::unordered_map<unsigned long long, std::vector<Slot>> pool;
  unsigned long long h = 1469598103934665603ull;  // FNV-1a over the table
  const unsigned char* b = reinterpret_cast<const unsigned char*>(&m);
  for (size_t i = 0; i < sizeof(SmallMaps); ++i) h = (h ^ b[i]) * 1099511628211ull;
  auto& v = pool[h];
  for (const Slot& sl : v)
    if (memcmp(sl.host, &m, sizeof(SmallMaps)) == 0) return sl.dev;
  Slot sl{nullptr, nullptr};
  if (cudaMallocHost(&sl.host, sizeof(SmallMaps)) != cudaSuccess) return nullptr;
  if (cudaMalloc(&sl.dev, sizeof(SmallMaps)) != cudaSuccess) return nullptr;
  *sl.host = m;
  if (cudaMemcpyAsync(sl.dev, sl.host, sizeof(SmallMaps), cudaMemcpyHostToDevice, s) != cudaSuccess) return nullptr;
  v.push_back(sl);
  return sl.dev;
}

// Routed B rows: x_perm [rows_cap, d] (act != nullptr), or gathered from
// x [T, d] through row_tokens[rows_cap].  h: [rows_cap, ff]; y: [rows_cap, d].
// Shared expert group (w13s != nullptr) over x: w13s [2 ffs, d], w2s [d, ffs],
// hs [T, ffs], ys [T, d].  Fused combine when out != nullptr (bf16 [T, d]).
struct SmallDense {  // in-kernel routing (dense decode), see SmallParams::dense
  const void* wg;
  int E, mode;
  int32_t* idx;
  float* w;
};

struct SmallIdx {  // segments straight from the router (see SmallParams::from_idx)
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
                     const SmallIdx* fromidx = nullptr) {
  const bool shared = w13s != nullptr && T > 0;
  const int G = n_groups + (shared ? 1 : 0);
  if (G == 0) return 0;
  static SmallParams p;
  static SmallMaps m;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  memset(&m, 0, sizeof(m));
  int rc = 0;
  if (dense && fromidx) return -1;
  if (dense) {
    if ((rc = get_map(&m.act3[1], x, T, d, 16))) return rc;  // every group's SwiGLU B = x rows [0, T)
    if ((rc = get_map(&m.act4[0], h, rows_cap, ff, 16))) return rc;
    for (int e = 0; e < 256; ++e) p.expert_slot[e] = -1;
    for (int g = 0; g < n_groups; ++g) p.expert_slot[group_expert[g]] = (int16_t)g;
  } else if (n_groups > 0) {
    if (act) {
      if ((rc = get_map(&m.act3[0], act, rows_cap, d, 16))) return rc;
    } else {
      if ((rc = get_map(&m.act3[0], x, T, d, 1))) return rc;  // tile::gather4 rows
    }
    if ((rc = get_map(&m.act4[0], h, rows_cap, ff, 16))) return rc;
  }
  // the shared group goes first: its SwiGLU tiles finish first, so the
  // column-block-major down pass never waits on it
  const int g0 = shared ? 1 : 0;
  for (int g = 0; g < n_groups; ++g) {
    if ((rc = get_map(&m.w13[g0 + g], w13[g], 2ull * ff, d, 64))) return rc;
    if ((rc = get_map(&m.w2[g0 + g], w2[g], d, ff, 64))) return rc;
    p.group_expert[g0 + g] = group_expert[g];
    p.group_ff[g0 + g] = ff;
  }
  if (shared) {
    if (!dense && (rc = get_map(&m.act3[1], x, T, d, 16))) return rc;
    if ((rc = get_map(&m.act4[1], hs, T, ffs, 16))) return rc;
    if ((rc = get_map(&m.w13[0], w13s, 2ull * ffs, d, 64))) return rc;
    if ((rc = get_map(&m.w2[0], w2s, d, ffs, 64))) return rc;
    p.group_expert[0] = -1;
    p.group_ff[0] = ffs;
  }
  // fused combine stages dst/w of all tokens in the 16.9 KB staging tile
  const bool fuse = out != nullptr && (long long)T * k * 8 <= 4LL * SG_BM * SG_PITCH;
  static int* counters = nullptr;
  static unsigned seq = 0;
  if (!counters) {
    if (cudaMalloc(&counters, 256 * SG_COUNTERS * sizeof(int)) != cudaSuccess) return -2;
    if (cudaMemset(counters, 0, 256 * SG_COUNTERS * sizeof(int)) != cudaSuccess) return -2;
  }
  int* c = counters + (seq++ % 256) * SG_COUNTERS;
  p.maps = upload_maps(m, s);
  if (!p.maps) return -2;
  p.row_tokens = act ? nullptr : row_tokens;
  p.rows_cap = rows_cap;
  p.cdst = cdst;
  p.cw = cw;
  p.out = fuse ? static_cast<__nv_bfloat16*>(out) : nullptr;
  p.k = k;
  p.T = T;
  p.dense = dense ? 1 : 0;
  p.from_idx = fromidx ? 1 : 0;
  if (fromidx) {
    p.ridx = const_cast<int32_t*>(fromidx->idx);
    p.rcounts = fromidx->counts;
    p.E = fromidx->E;
    p.dst_out = fromidx->dst_out;
    p.offsets_out = fromidx->offsets_out;
    p.cdst = fromidx->dst_out;
    p.row_tokens = nullptr;
  }
  // routed decode: launched as a programmatic dependent of the router / permute
  p.pdl = dense ? 0 : 1;
  p.prefetch_shared = 1;
  if (dense) {
    p.wg = static_cast<const __nv_bfloat16*>(dense->wg);
    p.xtok = static_cast<const __nv_bfloat16*>(x);
    p.E = dense->E;
    p.mode = dense->mode;
    p.ridx = dense->idx;
    p.rw = dense->w;
  }
  p.counters = c;
  p.offsets = offsets;
  p.h[0] = static_cast<__nv_bfloat16*>(h);
  p.h[1] = static_cast<__nv_bfloat16*>(hs);
  p.y[0] = static_cast<__nv_bfloat16*>(y);
  p.y[1] = shared ? static_cast<__nv_bfloat16*>(ys) : nullptr;
  p.n_groups = G;
  p.Ts = shared ? T : 0;
  p.d = d;
  p.phases = phases;
  if (g_sg_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sg_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sg_sms <= 0) g_sg_sms = 148;
  }
  // pipeline shape: 2 K atoms per stage, chunks of up to 64 tokens (measured
  // best on C4 decode against 1/4 atoms and 16/32-token chunks)
#define SG_LAUNCH(KA_, NM_)                                                                                \
  do {                                                                                                     \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      cudaFuncSetAttribute(small_ffn_kernel<KA_, NM_>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                           (int)SgCfg<KA_, NM_>::SMEM);                                                    \
      attr = true;                                                                                         \
    }                                                                                                      \
    if (p.pdl) {                                                                                           \
      cudaLaunchConfig_t cfg = {};                                                                         \
      cfg.gridDim = dim3(g_sg_sms);                                                                        \
      cfg.blockDim = dim3(SG_THREADS);                                                                     \
      cfg.dynamicSmemBytes = SgCfg<KA_, NM_>::SMEM;                                                        \
      cfg.stream = s;                                                                                      \
      cudaLaunchAttribute at[1];                                                                           \
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                       \
      at[0].val.programmaticStreamSerializationAllowed = 1;                                                \
      cfg.attrs = at;                                                                                      \
      cfg.numAttrs = 1;                                                                                    \
      cudaLaunchKernelEx(&cfg, small_ffn_kernel<KA_, NM_>, p);                                             \
    } else {                                                                                               \
      small_ffn_kernel<KA_, NM_><<<g_sg_sms, SG_THREADS, SgCfg<KA_, NM_>::SMEM, s>>>(p);                   \
    }                                                                                                      \
  } while (0)
  SG_LAUNCH(2, 64);
#undef SG_LAUNCH
  if (out && !fuse) {
    if (launch_status()) return -2;
    return launch_combine(y, cdst, cw, T, k, d, shared ? ys : nullptr, out, 1, s);
  }
  return launch_status();
}

}  // namespace cox
