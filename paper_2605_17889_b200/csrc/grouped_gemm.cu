// K3/K4 — coalesced grouped expert GEMM on 5th-gen tensor cores (sm_100a).
//
// The paper's OP3 ("gated FFN execution per expert") run over
// the WHOLE ordinary batch of each expert at once (the
// coalesced_expert_batch contract of costmodel.py:45-73): one persistent launch
// covers every (expert, m-tile, n-tile) of every group.
//
//   K3 (EPI_SWIGLU): h[rows, ff]  = silu(A W1^T) * (A W3^T), W13 interleaved in
//                    128-row blocks (gate block, up block, ...) so that one
//                    256-wide accumulator tile holds matching gate/up columns.
//   K4 (EPI_STORE) : y[rows, d]   = h W2^T.
//
// Machine mapping:
//   * 2-CTA pairs (cluster 2x1): tcgen05.mma.cta_group::2, M=256 (128 A rows per
//     CTA), N=256 (128 B rows per CTA), K=16 per instruction, fp32 accumulators
//     in TMEM (2 x 256 columns: the epilogue of tile i overlaps the MMAs of i+1).
//   * TMA (cp.async.bulk.tensor, 128B swizzle) streams K slices of A and B into
//     a 192 KB smem ring guarded by mbarriers (3 stages of K = 128, or 6 of
//     K = 64 when K % 128 != 0); both CTAs' loads complete on the leader's "full"
//     barrier, the leader's MMA commit frees the slot in both CTAs (multicast
//     commit).
//   * Warp roles: w0 TMA producer, w1 MMA issuer (leader CTA, one thread),
//     w2 TMEM allocator, w4..w7 epilogue (TMEM -> registers -> coalesced
//     stores through a smem staging tile; branch-free SiLU for K3 -- see
//     silu_fast -- and a relaxed "accumulator drained" arrive, so the epilogue
//     stays shorter than one tile's MMAs even at K = 1024).
//   * Persistent kernel, 74 pairs on 148 SMs, dynamic tile scheduler (warp 3 of
//     the leader: global atomic counter -> tile-id ring in both CTAs); tiles
//     are rasterised in bands of `band` n-tiles so that concurrently running
//     pairs share A rows and B bands in L2.
// Expert segments need no padding: rows of a partial m-tile that belong to the
// next segment are computed but never stored.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "common.cuh"

namespace cox {

constexpr int GM_BM = 128;  // A rows per CTA (pair: 256)
constexpr int GM_BN = 256;  // MMA N per pair (B rows per CTA: 128)
constexpr int GM_BK = 64;   // one 128-byte swizzle atom of bf16
constexpr int GM_STAGES = 6;
constexpr int GM_MAXG = 64;
constexpr int GM_THREADS = 256;
constexpr int GM_GATHER_WARPS = 4;  // gather mode: A rows by cp.async (warps 8..11)
constexpr uint32_t GM_A_BYTES = GM_BM * GM_BK * 2;         // 16 KB
constexpr uint32_t GM_B_BYTES = (GM_BN / 2) * GM_BK * 2;   // 16 KB
constexpr uint32_t GM_TMEM_COLS = 512;
constexpr int GM_SCHED_DEPTH = 4;  // tile-id ring between the scheduler and the roles
constexpr int EPI_SWIGLU = 0;
constexpr int EPI_STORE = 1;

struct alignas(64) GemmParams {
  CUtensorMap a_map;
  CUtensorMap b_map[GM_MAXG];
  CUtensorMap b_map64[GM_MAXG];  // SwiGLU half tiles: 64-row boxes (gate rows over up rows)
  const int32_t* offsets;
  int* tile_counter;  // zeroed before launch; dynamic tile scheduler
  void* out;
  long long ldo;
  int group_expert[GM_MAXG];
  int n_groups;
  int K;
  int n_tiles;
  int band;
  int l2_mode;  // L2 cache policy of the operand loads, see l2_policies()
  int half_tiles;  // 1: a group's last m-tile with <= 128 rows runs as an M = 128 pair tile
  // gather mode (K3 without x_perm): A row r of group g is token
  // row_tokens[row0_g + r] of gx [*, K] (row pitch gx_ld elements)
  const __nv_bfloat16* gx;
  const int32_t* row_tokens;
  long long gx_ld;
};

struct TileCoord {
  int g, m, n;
  bool half;  // M = 128 pair tile (64 A rows per CTA)
};

// g: the caller's group cursor.  Every role sees increasing tile ids (first
// wave static, then an atomic counter), so the group search resumes where the
// previous tile's ended instead of scanning from group 0 (C4: 64 groups, a
// serial smem scan of ~32 steps per tile delayed the producer's TMA issue).
// half_ok: the group's last m-tile runs as an M = 128 pair tile when at most
// 128 of its rows are left (see grouped_gemm_kernel)
COX_DEV TileCoord decode_tile(int t, const int* s_prefix, const int* s_rows, int band, bool half_ok, int& g) {
  TileCoord c;
  while (t >= s_prefix[g + 1]) ++g;
  const int local = t - s_prefix[g];
  const int mt = (s_rows[g] + 2 * GM_BM - 1) / (2 * GM_BM);
  const int per_band = mt * band;
  const int b = local / per_band;
  const int r = local - b * per_band;
  c.g = g;
  c.m = r / band;
  c.n = b * band + (r - c.m * band);
  c.half = half_ok && c.m == mt - 1 && s_rows[g] - c.m * 2 * GM_BM <= GM_BM;  // compile-time false without HALF
  return c;
}

COX_DEV float silu_f(float g) { return silu_fast(g); }

// KA = 128-byte swizzle atoms of K per pipeline stage: 1 -> BK 64, 6 stages;
// 2 -> BK 128, 3 stages (same smem; 256 contiguous bytes per weight row per
// stage, i.e. better DRAM page locality for weight-streaming shapes).  The
// epilogue stores are coalesced through a 16 KB smem staging tile.
template <int KA>
struct GmRing {
  static constexpr int STAGES = GM_STAGES / KA;
  static constexpr size_t SMEM =
      1024 + (size_t)GM_STAGES * (GM_A_BYTES + GM_B_BYTES) + 512 + 4 * (3 * GM_MAXG + 4) + 16 + 4 * 32 * 128;
};

// L2 cache policies of the operand loads (createpolicy, applied per TMA load):
//   mode 0: no hint (the L2's default LRU);
//   mode 1: the B band (expert weights, reused by every m-tile of the band)
//           evict_last, A (activations, consumed by the band's n-tiles within
//           a short window) evict_normal;
//   mode 2: B evict_last, A evict_first.
// Measured reasoning (ncu, C2 K4): without hints the streamed A evicts the
// band's weights, which are then re-read from DRAM once per wave of m-tiles.
COX_DEV void l2_policies(int mode, uint64_t& pa, uint64_t& pb) {
  uint64_t last, first, normal;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(normal));
  pb = mode >= 1 ? last : normal;
  pa = mode == 2 ? first : normal;
}

// 16-byte cp.async into shared memory (L2 only); src_bytes 0 zero-fills
COX_DEV void cp_async_cg16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// Half tiles: the last m-tile of a group with at most 128 rows left (short
// segments of medium batches; the few rows a segment spills past a multiple of
// 256) runs as an M = 128 pair tile, 64 A rows per CTA, so one SM of the pair
// does not multiply 128 rows past the segment end.  The accumulator of
// cta_group::2 with M = 128 holds N columns [0, 128) in TMEM lanes 0-63 and
// [128, 256) in lanes 64-127 (same column addresses); for the SwiGLU GEMM each
// CTA's 128 B rows are then 64 gate rows over the 64 matching up rows, so every
// epilogue warp finds gate and up in its own lanes (64-row boxes of a second
// tensor map).  A half tile's A box is the usual 128 rows; the MMA reads the
// first 64.
template <int EPI, int KA, bool GATHER = false, bool HALF = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GM_THREADS + (GATHER ? 32 * GM_GATHER_WARPS : 0), 1)
    grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  static_assert(!(GATHER && HALF), "the gather mode runs 256-row pair tiles only");
  constexpr bool half_ok = HALF;
  constexpr int BK = GM_BK * KA;
  constexpr int STAGES = GmRing<KA>::STAGES;
  constexpr int NB = GM_STAGES;  // barrier / atom array length (>= STAGES)
  constexpr uint32_t A_STAGE = GM_A_BYTES * KA;
  constexpr uint32_t B_STAGE = GM_B_BYTES * KA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NB * GM_A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NB * GM_B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + NB;
  uint64_t* tfull = bars + 2 * NB;
  uint64_t* tempty = bars + 2 * NB + 2;
  uint64_t* sfull = bars + 2 * NB + 4;                           // [DEPTH] tile id published
  uint64_t* sempty = sfull + GM_SCHED_DEPTH;                     // [DEPTH] (leader) slot consumed
  uint64_t* afull = sempty + GM_SCHED_DEPTH;                     // [NB] gather mode: this CTA's A copies landed
  int* s_tile = reinterpret_cast<int*>(afull + NB);              // [DEPTH]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_tile + GM_SCHED_DEPTH);
  uint32_t* tx_scratch = tmem_slot + 4;  // [12] gather mode: the relays' 16-byte completion copies
  int* s_prefix = reinterpret_cast<int*>(tx_scratch + 12);
  int* s_rows = s_prefix + GM_MAXG + 1;
  int* s_row0 = s_rows + GM_MAXG;
  uint32_t* s_stage = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(s_row0 + GM_MAXG) + 15) & ~uintptr_t(15));  // 4 warps x 32 rows x 128 B

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // gather mode: + the leader's relay arrive; the peer's relay signals as 16 tx bytes (see below)
      mbar_init(smem_u32(&full[s]), GATHER ? 2 : 1);
      mbar_init(smem_u32(&empty[s]), 1);
      if (GATHER) mbar_init(smem_u32(&afull[s]), 32 * GM_GATHER_WARPS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int i = 0; i < GM_SCHED_DEPTH; ++i) {
      mbar_init(smem_u32(&sfull[i]), 1);
      // producers x2 + MMA + epilogue warps x8 (+ gather warps x8 + relays x2)
      mbar_init(smem_u32(&sempty[i]), GATHER ? 11 + 2 * GM_GATHER_WARPS + 2 : 11);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    // group table, one group per lane (a serial loop pays one L2 round trip per
    // group: ~20 us at 64 groups)
    int acc = 0;
    for (int base = 0; base < p.n_groups; base += 32) {
      const int g = base + lane;
      int tiles = 0;
      if (g < p.n_groups) {
        const int e = p.group_expert[g];
        const int r0 = p.offsets[e];
        const int rows = p.offsets[e + 1] - r0;
        s_row0[g] = r0;
        s_rows[g] = rows;
        tiles = ((rows + 2 * GM_BM - 1) / (2 * GM_BM)) * p.n_tiles;
      }
      int incl = tiles;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (g < p.n_groups) s_prefix[g] = acc + incl - tiles;
      acc += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_prefix[p.n_groups] = acc;
  }
  if (warp == 0 && lane == 0) {
    if (!GATHER) tma_prefetch_desc(&p.a_map);
    for (int g = 0; g < p.n_groups; ++g) tma_prefetch_desc(&p.b_map[g]);
  }
  if (warp == 2) tmem_alloc<2>(smem_u32(tmem_slot), GM_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();

  const uint32_t tmem_base = *tmem_slot;
  const int total = s_prefix[p.n_groups];
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  const int nk = p.K / BK;

  // Dynamic tile scheduler.  The leader's warp 3 publishes tile ids into a
  // ring replicated in both CTAs (first wave static, then a global atomic
  // counter) so that concurrently running pairs always work on neighbouring
  // tiles of the rasterised order and keep sharing A/B in L2 — a static
  // round-robin lets pairs drift apart by whole waves.  Every role consumes
  // the same sequence; a value >= total terminates.
  // Leader-CTA consumers use CTA-scope wait/arrive (cheap); the peer CTA needs
  // cluster scope (its tile id was written remotely by the leader).
  auto fetch_tile = [&](int& si, bool do_arrive) -> int {
    const int slot = si % GM_SCHED_DEPTH;
    const uint32_t ph = (si / GM_SCHED_DEPTH) & 1;
    int t;
    if (rank == 0) {
      mbar_wait(smem_u32(&sfull[slot]), ph);
      t = reinterpret_cast<volatile int*>(s_tile)[slot];
      __syncwarp(__activemask());
      if (do_arrive) mbar_arrive(smem_u32(&sempty[slot]));
    } else {
      mbar_wait_cluster(smem_u32(&sfull[slot]), ph);
      t = reinterpret_cast<volatile int*>(s_tile)[slot];
      __syncwarp(__activemask());
      if (do_arrive) {
        // relaxed arrive (a release.cluster arrive is a GPU-scope membar that
        // would wait for this warp's outstanding global stores); the slot read
        // is ordered before it by a data dependency of the arrive's address
        uint32_t z;
        asm volatile("and.b32 %0, %1, 0;" : "=r"(z) : "r"(t));
        mbar_arrive_cluster_relaxed(mapa(smem_u32(&sempty[slot]), 0) + z);
      }
    }
    ++si;
    return t;
  };

  if (warp == 3) {
    // ------------------------------------------------------------ tile scheduler (leader)
    if (rank == 0 && lane == 0) {
      for (int i = 0;; ++i) {
        const int slot = i % GM_SCHED_DEPTH;
        mbar_wait(smem_u32(&sempty[slot]), ((i / GM_SCHED_DEPTH) & 1) ^ 1);
        int t = (i == 0) ? cid : ncl + atomicAdd(p.tile_counter, 1);
        if (t > total) t = total;
        s_tile[slot] = t;
        st_shared_cluster_u32(mapa(smem_u32(&s_tile[slot]), 1), (uint32_t)t);
        mbar_arrive(smem_u32(&sfull[slot]));
        mbar_arrive_cluster(mapa(smem_u32(&sfull[slot]), 1));
        if (t >= total) break;
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (lane 0)
    if (lane == 0) {
      uint64_t pol_a, pol_b;
      l2_policies(p.l2_mode, pol_a, pol_b);
      const bool hint = p.l2_mode != 0;
      uint32_t stage = 0, phase = 0;
      int si = 0, gcur = 0;
      int t = fetch_tile(si, true);
      while (t < total) {
        const TileCoord c = decode_tile(t, s_prefix, s_rows, p.band, half_ok, gcur);
        const int a_row = s_row0[c.g] + c.m * 2 * GM_BM + (int)rank * (c.half ? GM_BM / 2 : GM_BM);
        const int b_row = c.n * GM_BN + (int)rank * (GM_BN / 2);
        // half SwiGLU tile: 64 gate rows [256 n + 64 rank, +64) over the 64 matching up rows (+128)
        const bool gate_up = HALF && EPI == EPI_SWIGLU && c.half;
        const int b_gate = c.n * GM_BN + (int)rank * 64;
        const CUtensorMap* bmap = &p.b_map[c.g];
        const CUtensorMap* bmap64 = &p.b_map64[c.g];
        int t_next = total;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb_local = smem_u32(&full[stage]);
          const uint32_t fb = mapa(fb_local, 0);
          if (rank == 0) mbar_arrive_expect_tx(fb_local, GATHER ? 2 * B_STAGE + 16u : 2 * (A_STAGE + B_STAGE));
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            const uint32_t da = smem_u32(sA + stage * A_STAGE + a * GM_A_BYTES);
            const uint32_t db = smem_u32(sB + stage * B_STAGE + a * GM_B_BYTES);
            const int kc = kb * BK + a * GM_BK;
            if (HALF && gate_up) {
              tma_load_2d_pair(da, &p.a_map, fb, kc, a_row);
              tma_load_2d_pair(db, bmap64, fb, kc, b_gate);
              tma_load_2d_pair(db + GM_B_BYTES / 2, bmap64, fb, kc, b_gate + GM_BN / 2);
            } else if (hint) {
              if (!GATHER) tma_load_2d_pair_hint(da, &p.a_map, fb, kc, a_row, pol_a);
              tma_load_2d_pair_hint(db, bmap, fb, kc, b_row, pol_b);
            } else {
              if (!GATHER) tma_load_2d_pair(da, &p.a_map, fb, kc, a_row);
              tma_load_2d_pair(db, bmap, fb, kc, b_row);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (kb == 0) t_next = fetch_tile(si, true);  // look ahead: hide the fetch behind this tile
        }
        t = t_next;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc_full = idesc_bf16_f32(2 * GM_BM, GM_BN);
      const uint32_t idesc_half = idesc_bf16_f32(GM_BM, GM_BN);
      uint32_t stage = 0, phase = 0;
      int si = 0, gcur = 0;
      int t = fetch_tile(si, true);
      // the tile's shape is decoded while the previous tile's MMAs run (the
      // MMA issue gap between tiles is on the critical path)
      uint32_t idesc_next = idesc_full;
      if constexpr (HALF)
        if (t < total && decode_tile(t, s_prefix, s_rows, p.band, half_ok, gcur).half) idesc_next = idesc_half;
      for (int it = 0; t < total; ++it) {
        int t_next = total;
        const uint32_t idesc = idesc_next;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * GM_BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_STAGE);
          const uint32_t b_base = smem_u32(sB + stage * B_STAGE);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t off = (k >> 2) * GM_A_BYTES + (k & 3) * 32;  // atom, then 16-wide K step inside it
            mma_bf16_ss<2>(d_tmem, sdesc_kmajor_sw128(a_base + off), sdesc_kmajor_sw128(b_base + off), idesc,
                           (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit<2>(smem_u32(&empty[stage]));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (kb == 0) {  // look ahead while the tensor pipe is busy
            t_next = fetch_tile(si, true);
            if constexpr (HALF)
              if (t_next < total)
                idesc_next = decode_tile(t_next, s_prefix, s_rows, p.band, half_ok, gcur).half ? idesc_half
                                                                                              : idesc_full;
          }
        }
        mma_commit<2>(smem_u32(&tfull[acc]));
        t = t_next;
      }
    }
    __syncwarp();
  } else if (GATHER && warp == 2) {
    // ------------------------------------------------------------ A relay (gather mode)
    // Waits until this CTA's gather threads' copies of a stage have landed
    // (cp.async.mbarrier.arrive on afull) and orders them before the async
    // proxy (fence.proxy.async).  The leader's relay then arrives on its own
    // full barrier (CTA scope); the peer's relay signals the leader with a
    // 16-byte async-proxy bulk copy into the leader's shared memory that
    // completes as transaction bytes on that barrier — the same completion
    // path as the peer's TMA loads.  (An mbarrier.arrive.release.cluster here
    // compiles to a GPU-scope memory barrier per stage and made the gathered
    // K3 ~8% slower.)
    if (lane == 0) {
      const uint32_t full0 = mapa(smem_u32(&full[0]), 0);
      const uint32_t dst = mapa(smem_u32(tx_scratch), 0);
      const uint32_t src = smem_u32(tx_scratch + 8);
      uint32_t stage = 0, phase = 0;
      int si = 0;
      int t = fetch_tile(si, true);
      while (t < total) {
        int t_next = total;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&afull[stage]), phase);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (rank == 0)
            mbar_arrive(smem_u32(&full[stage]));
          else
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                    dst),
                "r"(src), "r"(full0 + stage * 8)
                : "memory");
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (kb == 0) t_next = fetch_tile(si, true);
        }
        t = t_next;
      }
    }
    __syncwarp();
  } else if (GATHER && warp >= 8) {
    // ------------------------------------------------------------ A gather (cp.async)
    // 4 warps fill this CTA's 128 A rows of every stage straight from x: lane
    // (gw, l) copies 16-byte chunk l%8 of rows 4 gw + l/8 + 16 w (w < 8) of
    // each 64-column swizzle atom (a warp instruction = 4 rows x 128 B), into
    // the 128B-swizzled K-major layout TMA would write (chunk c of row r at
    // (c ^ (r & 7)) * 16).  Completion is tracked without blocking: each
    // thread's cp.async.mbarrier.arrive.noinc fires on afull[stage] once its
    // copies have landed (the relay warp publishes the stage).  Rows past the
    // group end are zero-filled.
    const int gw = warp - 8;
    const int c8 = lane & 7;
    uint32_t stage = 0, phase = 0;
    int si = 0, gcur = 0;
    int t = fetch_tile(si, lane == 0);
    while (t < total) {
      const TileCoord c = decode_tile(t, s_prefix, s_rows, p.band, false, gcur);
      const int lrow0 = c.m * 2 * GM_BM + (int)rank * GM_BM;  // first A row of this CTA in the group
      const __nv_bfloat16* src[8];
      uint32_t sbytes[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int r = 4 * gw + (lane >> 3) + 16 * w;
        const bool ok = lrow0 + r < s_rows[c.g];
        const int tok = ok ? __ldg(p.row_tokens + s_row0[c.g] + lrow0 + r) : 0;
        src[w] = p.gx + (long long)tok * p.gx_ld + 8 * c8;
        sbytes[w] = ok ? 16u : 0u;
      }
      int t_next = total;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
#pragma unroll
        for (int a = 0; a < KA; ++a) {
          const uint32_t atom = smem_u32(sA + stage * A_STAGE + a * GM_A_BYTES);
          const int kc = kb * BK + a * GM_BK;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const int r = 4 * gw + (lane >> 3) + 16 * w;
            cp_async_cg16(atom + r * 128 + ((c8 ^ (r & 7)) << 4), src[w] + kc, sbytes[w]);
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&afull[stage])) : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (kb == 0) t_next = fetch_tile(si, lane == 0);
      }
      t = t_next;
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa(smem_u32(&tempty[1]), 0);
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
    int si = 0, gcur = 0;
    for (int it = 0;; ++it) {
      const int t = fetch_tile(si, lane == 0);
      if (t >= total) break;
      const TileCoord c = decode_tile(t, s_prefix, s_rows, p.band, half_ok, gcur);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * GM_BN;
      // Epilogue stores are coalesced through a per-warp 4 KB staging tile:
      // each lane packs 64 bf16 columns of its row (XOR-swizzled 16 B chunks,
      // conflict-free), then every st.global.v4 instruction of the warp writes
      // 4 rows x 128 contiguous bytes (full lines) instead of 32 scattered
      // 16-byte pieces.
      // first row of this warp in the group (half tile: warps 0,1 and 2,3 hold the same 64 rows, N halves)
      const int wrow0 = c.half ? c.m * 2 * GM_BM + (int)rank * (GM_BM / 2) + (ew & 1) * 32
                               : c.m * 2 * GM_BM + (int)rank * GM_BM + ew * 32;
      const int vrows = s_rows[c.g] - wrow0;                               // rows of the warp that are stored
      const long long grow0 = (long long)s_row0[c.g] + wrow0;
      uint32_t* stg = s_stage + ew * (32 * 32);
      auto stage16 = [&](int j, uint32_t a, uint32_t b, uint32_t c2, uint32_t d2) {  // chunk j (0..7) of my row
        *reinterpret_cast<uint4*>(stg + lane * 32 + ((j ^ (lane & 7)) * 4)) = make_uint4(a, b, c2, d2);
      };
      auto flush64 = [&](__nv_bfloat16* col0) {  // write the staged 32 rows x 64 cols
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + (lane >> 3), j = lane & 7;
          const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 32 + ((j ^ (r & 7)) * 4));
          if (r < vrows) st_global_v4(col0 + (grow0 + r) * p.ldo + j * 8, v.x, v.y, v.z, v.w);
        }
        __syncwarp();
      };
      if (HALF && EPI == EPI_SWIGLU && c.half) {
        // N columns 0-63 gate / 64-127 up of h block 2n (lanes 0-63) or 2n+1 (lanes 64-127)
        __nv_bfloat16* ocol = out + (long long)c.n * (GM_BN / 2) + (ew >> 1) * 64;
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          uint32_t gr[32], ur[32];
          tmem_ld2_32x32b_x32(tbase + cc * 32, gr, tbase + 64 + cc * 32, ur);
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float g0 = __uint_as_float(gr[2 * q]), g1 = __uint_as_float(gr[2 * q + 1]);
            const float u0 = __uint_as_float(ur[2 * q]), u1 = __uint_as_float(ur[2 * q + 1]);
            pk[q] = pack_bf16x2(silu_f(g0) * u0, silu_f(g1) * u1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) stage16(cc * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
        flush64(ocol);
      } else if (HALF && EPI == EPI_STORE && c.half) {
        // N columns [128 h, 128 h + 128) of the warp's rows, h = ew >> 1
        __nv_bfloat16* ocol = out + (long long)c.n * GM_BN + (ew >> 1) * (GM_BN / 2);
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + cc * 32, r);
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) pk[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
#pragma unroll
          for (int q = 0; q < 4; ++q) stage16((cc & 1) * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          if (cc & 1) flush64(ocol + (cc >> 1) * 64);
        }
      } else if (EPI == EPI_SWIGLU) {
        __nv_bfloat16* ocol = out + (long long)c.n * (GM_BN / 2);
#pragma unroll 1
        for (int cc = 0; cc < (GM_BN / 2) / 32; ++cc) {
          uint32_t gr[32], ur[32];
          tmem_ld2_32x32b_x32(tbase + cc * 32, gr, tbase + (GM_BN / 2) + cc * 32, ur);
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float g0 = __uint_as_float(gr[2 * q]), g1 = __uint_as_float(gr[2 * q + 1]);
            const float u0 = __uint_as_float(ur[2 * q]), u1 = __uint_as_float(ur[2 * q + 1]);
            pk[q] = pack_bf16x2(silu_f(g0) * u0, silu_f(g1) * u1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) stage16((cc & 1) * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          if (cc & 1) flush64(ocol + (cc >> 1) * 64);
        }
      } else {
        __nv_bfloat16* ocol = out + (long long)c.n * GM_BN;
#pragma unroll 1
        for (int cc = 0; cc < GM_BN / 32; ++cc) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + cc * 32, r);
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) pk[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
#pragma unroll
          for (int q = 0; q < 4; ++q) stage16((cc & 1) * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          if (cc & 1) flush64(ocol + (cc >> 1) * 64);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<2>(tmem_base, GM_TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  unsigned long long rows, cols;
  unsigned box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.ptr) ^ (k.rows * 1000003ull) ^ (k.cols * 998244353ull) ^ k.box_rows;
  }
};

// bf16 row-major [rows, cols] -> TMA map with a {64 cols, box_rows rows} box, 128B swizzle.
int get_map(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols,
                   unsigned box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, cols, box_rows};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return 0;
    }
  }
  auto enc = get_encode_fn();
  if (!enc) return -2;
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return 0;
}

// bf16 row-major [rows, cols] -> TMA map with a {box_cols, box_rows} box, no swizzle or 128B swizzle
// (not cached: for kernels that build their map per launch).
int get_map_box(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols,
                unsigned box_cols, unsigned box_rows, bool swizzle128) {
  auto enc = get_encode_fn();
  if (!enc) return -2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Raster band (n-tiles per band): tiles run expert -> n-band -> m -> n, so the
// B band (band x 256 rows x K) is shared by every m-tile of the expert and A
// is re-read once per band.  Pick the widest band that divides n_tiles and
// whose B band stays within an L2 budget (32 MB for K3, 64 MB for K4); e.g.
// C2 K3 (K=4096): 16, C2 K4 (K=14336): 8, C4 K3 (11 n-tiles, K=2048): 11.
// COX_GEMM_BAND_K3 / COX_GEMM_BAND_K4 override (A/B experiments).
static int pick_band(int epi, int n_tiles, int K) {
  static const int env_band[2] = {env_int("COX_GEMM_BAND_K3", 0), env_int("COX_GEMM_BAND_K4", 0)};
  static const int env_budget[2] = {env_int("COX_GEMM_BUDGET_MB_K3", 32), env_int("COX_GEMM_BUDGET_MB_K4", 64)};
  const int want = env_band[epi ? 1 : 0];
  if (want > 0 && n_tiles % want == 0) return want;
  const long long per_tile = (long long)GM_BN * K * 2;
  // measured (ncu dram__bytes_read, C2): K3 band 16 -> 33 GB (28 -> 57 GB);
  // K4 band 4/8/16 -> 77/69/143 GB, so the long-K down projection gets a larger budget
  const long long budget = (long long)env_budget[epi ? 1 : 0] << 20;
  long long max_band = budget / per_tile;
  if (max_band < 1) max_band = 1;
  for (int b = (int)(max_band < n_tiles ? max_band : n_tiles); b >= 1; --b)
    if (n_tiles % b == 0) return b;
  return 1;
}

static int g_num_sms = 0;

// epi: EPI_SWIGLU (B = W13 interleaved [2ff, K], out = h [rows_cap, ff])
//      EPI_STORE  (B = W2 [N, K],                out = y [rows_cap, N])
// gx != nullptr (EPI_SWIGLU only): gather mode, A row r of a group is row
// row_tokens[r] of gx [*, K] (pitch gx_ld); A / rows_cap are unused.
int launch_grouped_gemm(int epi, const void* A, long long rows_cap, int K, const int32_t* offsets, int n_groups,
                        const int32_t* group_expert, const void* const* B, int N, void* out, long long ldo,
                        int max_ctas, cudaStream_t s, const void* gx, const int32_t* row_tokens, long long gx_ld) {
  if (n_groups <= 0) return 0;
  static GemmParams p;  // large (17 KB): built in static storage, copied at launch
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  const bool gather = gx != nullptr;
  if (gather && epi != EPI_SWIGLU) return -1;
  // half tiles (see grouped_gemm_kernel) for batches whose segments average
  // <= 2,048 rows: there the last m-tile's padding is a visible share of the
  // MMAs (C2 T = 1,024: ~256 +- 16 rows per expert, so half the experts spill a
  // few rows into a second tile); above, the full-tile kernel (same-box A/B:
  // the half-capable kernel costs 0.4-0.7% at T = 262,144).  COX_GEMM_HALF=0/1
  // forbids / forces them (A/B, tests).
  static const int half_env = env_int("COX_GEMM_HALF", -1);
  p.half_tiles = !gather && (half_env >= 0 ? half_env == 1 : rows_cap <= 2048LL * n_groups);
  int rc = gather ? 0 : get_map(&p.a_map, A, (unsigned long long)rows_cap, (unsigned long long)K, GM_BM);
  if (rc) return rc;
  p.gx = static_cast<const __nv_bfloat16*>(gx);
  p.row_tokens = row_tokens;
  p.gx_ld = gx_ld;
  for (int g = 0; g < n_groups; ++g) {
    rc = get_map(&p.b_map[g], B[g], (unsigned long long)N, (unsigned long long)K, GM_BN / 2);
    if (rc) return rc;
    if (epi == EPI_SWIGLU && p.half_tiles) {
      rc = get_map(&p.b_map64[g], B[g], (unsigned long long)N, (unsigned long long)K, GM_BN / 4);
      if (rc) return rc;
    }
    p.group_expert[g] = group_expert[g];
  }
  // per-launch tile counters: a ring of slots, each zeroed (stream-ordered) before its launch
  static int* counters = nullptr;
  static unsigned seq = 0;
  if (!counters) {
    if (cudaMalloc(&counters, 1024 * sizeof(int)) != cudaSuccess) return -2;
    if (cudaMemset(counters, 0, 1024 * sizeof(int)) != cudaSuccess) return -2;
  }
  int* counter = counters + (seq++ % 1024);
  if (cudaMemsetAsync(counter, 0, sizeof(int), s) != cudaSuccess) return -2;
  p.tile_counter = counter;
  p.offsets = offsets;
  p.out = out;
  p.ldo = ldo;
  p.n_groups = n_groups;
  p.K = K;
  p.n_tiles = N / GM_BN;
  p.band = pick_band(epi, p.n_tiles, K);
  static const int l2_env[2] = {env_int("COX_GEMM_L2_K3", 0), env_int("COX_GEMM_L2_K4", 0)};
  p.l2_mode = l2_env[epi ? 1 : 0];
  // evict_last lines live in the persisting set-aside of the L2 (cudaLimitPersistingL2CacheSize;
  // 0 by default, which turns evict_last into evict_normal): COX_L2_PERSIST_MB sets it once
  static const bool persist_set = [] {
    const int mb = env_int("COX_L2_PERSIST_MB", 0);
    if (mb <= 0) return false;
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
    size_t want = (size_t)mb << 20;
    if (want > (size_t)mx) want = (size_t)mx;
    return cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess;
  }();
  (void)persist_set;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  int grid = (g_num_sms / 2) * 2;
  if (max_ctas >= 2 && max_ctas < grid) grid = (max_ctas / 2) * 2;
  // K per stage: BK = 128 (3 stages) wherever K allows it.  Measured: C2 K3
  // 92.2 -> 89.6 ms against BK = 64 / 6 stages; the down projection, same box,
  // interleaved: C4's routed K4 (K = 1408) 6.96 -> 6.63 ms, C2's (K = 14336)
  // 43.9 either way (same-box library A/B).
  const int ka = K % (2 * GM_BK) == 0 ? 2 : 1;
#define GM_LAUNCH(E_, KA_, G_, H_)                                                                             \
  do {                                                                                                         \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      cudaFuncSetAttribute(grouped_gemm_kernel<E_, KA_, G_, H_>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                           (int)GmRing<KA_>::SMEM);                                                            \
      attr = true;                                                                                             \
    }                                                                                                          \
    grouped_gemm_kernel<E_, KA_, G_, H_><<<grid, GM_THREADS + (G_ ? 32 * GM_GATHER_WARPS : 0),                 \
                                           GmRing<KA_>::SMEM, s>>>(p);                                         \
  } while (0)
  const bool h = p.half_tiles != 0;
  if (epi == EPI_SWIGLU) {
    if (gather) {
      if (ka == 2) GM_LAUNCH(EPI_SWIGLU, 2, true, false);
      else GM_LAUNCH(EPI_SWIGLU, 1, true, false);
    } else if (h) {
      if (ka == 2) GM_LAUNCH(EPI_SWIGLU, 2, false, true);
      else GM_LAUNCH(EPI_SWIGLU, 1, false, true);
    } else {
      if (ka == 2) GM_LAUNCH(EPI_SWIGLU, 2, false, false);
      else GM_LAUNCH(EPI_SWIGLU, 1, false, false);
    }
  } else if (h) {
    if (ka == 2) GM_LAUNCH(EPI_STORE, 2, false, true);
    else GM_LAUNCH(EPI_STORE, 1, false, true);
  } else {
    if (ka == 2) GM_LAUNCH(EPI_STORE, 2, false, false);
    else GM_LAUNCH(EPI_STORE, 1, false, false);
  }
#undef GM_LAUNCH
  return launch_status();
}

}  // namespace cox
