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
//     a 192 KB smem ring guarded by mbarriers (K3: 3 stages of K = 128; K4: 6
//     stages of K = 64); both CTAs' loads complete on the leader's "full"
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
constexpr uint32_t GM_A_BYTES = GM_BM * GM_BK * 2;         // 16 KB
constexpr uint32_t GM_B_BYTES = (GM_BN / 2) * GM_BK * 2;   // 16 KB
constexpr uint32_t GM_TMEM_COLS = 512;
constexpr int GM_SCHED_DEPTH = 4;  // tile-id ring between the scheduler and the roles
constexpr int EPI_SWIGLU = 0;
constexpr int EPI_STORE = 1;
// shared-expert down projection with the top-k combine fused into its epilogue:
// out[t] = sum_j w[t,j] * y_perm[dst[t,j]] + bf16(h_shared W2s^T)[t]
constexpr int EPI_COMBINE = 2;
#ifndef CMB_U
#define CMB_U 2  // EPI_COMBINE: rows per lane whose routed-row loads are in flight together (4: 255 regs, slower)
#endif

struct alignas(64) GemmParams {
  CUtensorMap a_map;
  CUtensorMap b_map[GM_MAXG];
  const int32_t* offsets;
  const int32_t* a_rows;  // gather mode: A row r = x[a_rows[r]] (tile::gather4); nullptr = tiled A
  long long a_rows_cap;   // entries of a_rows
  int* tile_counter;  // zeroed before launch; dynamic tile scheduler
  unsigned long long* tile_word;  // die-aware mode: (claimed from head) | (claimed from tail) << 32
  const int* die_map;             // SM id -> die (0/1), nullptr = die-agnostic
  void* out;
  long long ldo;
  const __nv_bfloat16* cy;  // EPI_COMBINE: routed expert outputs y_perm [rows, N] (leading dim ldo)
  const int32_t* cdst;      //   [T, ck] permuted row of (token, slot); < 0 = no contribution
  const float* cw;          //   [T, ck] combine weights
  int ck;                   //   top-k (<= 8)
  int group_expert[GM_MAXG];
  int n_groups;
  int K;
  int n_tiles;
  int band;
};

constexpr size_t GM_SMEM_BYTES =
    1024 + GM_STAGES * (GM_A_BYTES + GM_B_BYTES) + 512 + 4 * (3 * GM_MAXG + 4) + 16 + 4 * 32 * 128;

struct TileCoord {
  int g, m, n;
};

COX_DEV TileCoord decode_tile(int t, const int* s_prefix, const int* s_rows, int band) {
  TileCoord c;
  int g = 0;
  while (t >= s_prefix[g + 1]) ++g;
  const int local = t - s_prefix[g];
  const int mt = (s_rows[g] + 2 * GM_BM - 1) / (2 * GM_BM);
  const int per_band = mt * band;
  const int b = local / per_band;
  const int r = local - b * per_band;
  c.g = g;
  c.m = r / band;
  c.n = b * band + (r - c.m * band);
  return c;
}

COX_DEV float silu_f(float g) { return silu_fast(g); }

// KA = 128-byte swizzle atoms of K per pipeline stage: 1 -> BK 64, 6 stages;
// 2 -> BK 128, 3 stages (same smem; 256 contiguous bytes per weight row per
// stage, i.e. better DRAM page locality for weight-streaming shapes).
// STG: epilogue stores coalesced through a 16 KB smem staging tile (default);
// without it the ring gets a 7th 32 KB stage (KA = 1): more operand bytes in
// flight for feed-bound shapes.
template <int KA, bool STG>
struct GmRing {
  static constexpr int STAGES = STG ? GM_STAGES / KA : (KA == 1 ? 7 : 3);
  static constexpr int ATOMS = STAGES * KA;  // ring size in 16 KB (A) / 16 KB (B) atoms
  static constexpr size_t SMEM = 1024 + (size_t)ATOMS * (GM_A_BYTES + GM_B_BYTES) + 512 + 4 * (3 * GM_MAXG + 4) + 16 +
                                 (STG ? 4 * 32 * 128 : 0);
};

template <int EPI, int KA, bool STG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  constexpr int BK = GM_BK * KA;
  constexpr int STAGES = GmRing<KA, STG>::STAGES;
  constexpr int NB = GmRing<KA, STG>::ATOMS;  // barrier array length (>= STAGES)
  constexpr uint32_t A_STAGE = GM_A_BYTES * KA;
  constexpr uint32_t B_STAGE = GM_B_BYTES * KA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NB * GM_A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NB * GM_B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + NB;  // barrier arrays sized for the max stage count
  uint64_t* tfull = bars + 2 * NB;
  uint64_t* tempty = bars + 2 * NB + 2;
  uint64_t* sfull = bars + 2 * NB + 4;                           // [DEPTH] tile id published
  uint64_t* sempty = sfull + GM_SCHED_DEPTH;                     // [DEPTH] (leader) slot consumed
  int* s_tile = reinterpret_cast<int*>(sempty + GM_SCHED_DEPTH);  // [DEPTH]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_tile + GM_SCHED_DEPTH);
  int* s_prefix = reinterpret_cast<int*>(tmem_slot + 4);
  int* s_rows = s_prefix + GM_MAXG + 1;
  int* s_row0 = s_rows + GM_MAXG;
  uint32_t* s_stage = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(s_row0 + GM_MAXG) + 15) & ~uintptr_t(15));  // 4 warps x 32 rows x 128 B

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int i = 0; i < GM_SCHED_DEPTH; ++i) {
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), 11);  // producers x2 + MMA + epilogue warps x8
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
    tma_prefetch_desc(&p.a_map);
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
      if (do_arrive) mbar_arrive_cluster(mapa(smem_u32(&sempty[slot]), 0));
    }
    ++si;
    return t;
  };

  if (warp == 3) {
    // ------------------------------------------------------------ tile scheduler (leader)
    if (rank == 0 && lane == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      const int my_die = p.die_map ? p.die_map[smid] : 0;
      for (int i = 0;; ++i) {
        const int slot = i % GM_SCHED_DEPTH;
        mbar_wait(smem_u32(&sempty[slot]), ((i / GM_SCHED_DEPTH) & 1) ^ 1);
        int t;
        if (p.die_map) {
          // Two-ended queue: die 0 walks the tile list from the front, die 1 from the
          // back; both claims go through one 64-bit atomic, so they meet exactly.
          const unsigned long long old = atomicAdd(p.tile_word, my_die ? (1ull << 32) : 1ull);
          const int head = (int)(old & 0xffffffffu), tailc = (int)(old >> 32);
          if (my_die == 0)
            t = (head < total - tailc) ? head : total;
          else
            t = (total - 1 - tailc >= head) ? total - 1 - tailc : total;
        } else {
          t = (i == 0) ? cid : ncl + atomicAdd(p.tile_counter, 1);
        }
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
    // ------------------------------------------------------------ TMA producer
    // Tiled A: lane 0 issues one A box and one B box per stage.  Gather A
    // (p.a_rows): the whole warp issues 32 tile::gather4 loads per stage, lane i
    // fetching token rows a_rows[4i..4i+3] of this CTA's 128 permuted rows
    // straight from x — no materialised x_perm.  Correct but ~3x slower at C2
    // (gather issue rate; A re-fetched per n-tile), so it is opt-in only.
    const bool gather = p.a_rows != nullptr;
    uint32_t stage = 0, phase = 0;
    int si = 0;
    int t = lane == 0 ? fetch_tile(si, true) : 0;
    t = __shfl_sync(0xffffffffu, t, 0);
    while (t < total) {
      const TileCoord c = decode_tile(t, s_prefix, s_rows, p.band);
      const int a_row = s_row0[c.g] + c.m * 2 * GM_BM + (int)rank * GM_BM;
      const int b_row = c.n * GM_BN + (int)rank * (GM_BN / 2);
      const CUtensorMap* bmap = &p.b_map[c.g];
      int rr[4] = {0, 0, 0, 0};
      if (gather) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long r = (long long)a_row + lane * 4 + q;
          rr[q] = r < p.a_rows_cap ? p.a_rows[r] : 0;
        }
      }
      int t_next = total;
      for (int kb = 0; kb < nk; ++kb) {
        if (lane == 0) mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        __syncwarp();
        const uint32_t fb_local = smem_u32(&full[stage]);
        const uint32_t fb = mapa(fb_local, 0);
        if (lane == 0) {
          if (rank == 0) mbar_arrive_expect_tx(fb_local, 2 * (A_STAGE + B_STAGE));
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            if (!gather)
              tma_load_2d_pair(smem_u32(sA + stage * A_STAGE + a * GM_A_BYTES), &p.a_map, fb, kb * BK + a * GM_BK,
                               a_row);
            tma_load_2d_pair(smem_u32(sB + stage * B_STAGE + a * GM_B_BYTES), bmap, fb, kb * BK + a * GM_BK, b_row);
          }
        }
        if (gather) {
#pragma unroll
          for (int a = 0; a < KA; ++a)
            tma_gather4_pair(smem_u32(sA + stage * A_STAGE + a * GM_A_BYTES) + lane * 512, &p.a_map, fb,
                             kb * BK + a * GM_BK, rr[0], rr[1], rr[2], rr[3]);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (kb == 0) {  // look ahead: hide the fetch behind this tile
          int tn = lane == 0 ? fetch_tile(si, true) : 0;
          t_next = __shfl_sync(0xffffffffu, tn, 0);
        }
      }
      t = t_next;
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(2 * GM_BM, GM_BN);
      uint32_t stage = 0, phase = 0;
      int si = 0;
      int t = fetch_tile(si, true);
      for (int it = 0; t < total; ++it) {
        int t_next = total;
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
          if (kb == 0) t_next = fetch_tile(si, true);  // look ahead while the tensor pipe is busy
        }
        mma_commit<2>(smem_u32(&tfull[acc]));
        t = t_next;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int row_in_cta = ew * 32 + lane;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa(smem_u32(&tempty[1]), 0);
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
    int si = 0;
    for (int it = 0;; ++it) {
      const int t = fetch_tile(si, lane == 0);
      if (t >= total) break;
      const TileCoord c = decode_tile(t, s_prefix, s_rows, p.band);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      // EPI_COMBINE: this lane's token (row) — its top-k (row, weight) pairs,
      // and an L2 prefetch of the routed rows' 256 columns while the MMA runs
      int cd[8];
      float cwt[8];
      if constexpr (EPI == EPI_COMBINE) {
        const int lrow = c.m * 2 * GM_BM + (int)rank * GM_BM + row_in_cta;
        const bool v = lrow < s_rows[c.g];
        const long long tok = (long long)s_row0[c.g] + lrow;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          cd[j] = 0;
          cwt[j] = 0.0f;
          if (j < p.ck && v) {
            const int r = __ldg(p.cdst + tok * p.ck + j);
            if (r >= 0) {
              cd[j] = r;
              cwt[j] = __ldg(p.cw + tok * p.ck + j);
              const __nv_bfloat16* src = p.cy + (long long)r * p.ldo + (long long)c.n * GM_BN;
#pragma unroll
              for (int l = 0; l < 4; ++l) prefetch_l2(src + l * 64);
            }
          }
        }
      }
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const int local_row = c.m * 2 * GM_BM + (int)rank * GM_BM + row_in_cta;
      const bool valid = local_row < s_rows[c.g];
      const long long grow = (long long)s_row0[c.g] + local_row;
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * GM_BN;
      // Epilogue stores are coalesced through a per-warp 4 KB staging tile:
      // each lane packs 64 bf16 columns of its row (XOR-swizzled 16 B chunks,
      // conflict-free), then every st.global.v4 instruction of the warp writes
      // 4 rows x 128 contiguous bytes (full lines) instead of 32 scattered
      // 16-byte pieces.
      const int wrow0 = c.m * 2 * GM_BM + (int)rank * GM_BM + ew * 32;  // first row of this warp in the group
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
      // EPI_COMBINE: the staged 32 rows x 64 cols are the shared expert's bf16
      // output; add the routed rows in the order of combine.cu (ascending j,
      // separately rounded fp32 multiply and add, shared last) and store `out`
      auto flush64c = [&](__nv_bfloat16* col0, long long gcol) {
        __syncwarp();
        // CMB_U rows per lane per batch: all their routed-row loads are issued
        // before any is consumed (the loads are volatile asm, so the compiler
        // would not hoist them across the previous row's store by itself)
#pragma unroll 1
        for (int i0 = 0; i0 < 8; i0 += CMB_U) {
          uint4 yv[CMB_U][8];
          float wj[CMB_U][8];
#pragma unroll
          for (int u = 0; u < CMB_U; ++u) {
            const int r = (i0 + u) * 4 + (lane >> 3), j = lane & 7;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int dr = __shfl_sync(0xffffffffu, cd[q], r);
              wj[u][q] = __shfl_sync(0xffffffffu, cwt[q], r);
              if (q < p.ck && r < vrows) yv[u][q] = ld_nc_v4(p.cy + (long long)dr * p.ldo + gcol + j * 8);
            }
          }
#pragma unroll
          for (int u = 0; u < CMB_U; ++u) {
            const int r = (i0 + u) * 4 + (lane >> 3), j = lane & 7;
            if (r < vrows) {
              float a[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) a[e] = 0.0f;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                if (q < p.ck) {
                  float f[8];
                  bf16x8_to_f32(yv[u][q], f);
#pragma unroll
                  for (int e = 0; e < 8; ++e) a[e] = __fadd_rn(a[e], __fmul_rn(wj[u][q], f[e]));
                }
              }
              const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 32 + ((j ^ (r & 7)) * 4));
              float sh[8];
              bf16x8_to_f32(v, sh);
#pragma unroll
              for (int e = 0; e < 8; ++e) a[e] = __fadd_rn(a[e], sh[e]);
              st_global_v4(col0 + (grow0 + r) * p.ldo + j * 8, pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]),
                           pack_bf16x2(a[4], a[5]), pack_bf16x2(a[6], a[7]));
            }
          }
        }
        __syncwarp();
      };
      if constexpr (EPI == EPI_SWIGLU) {
        __nv_bfloat16* ocol = out + (long long)c.n * (GM_BN / 2);
#pragma unroll 1
        for (int cc = 0; cc < (GM_BN / 2) / 32; ++cc) {
          uint32_t gr[32], ur[32];
          tmem_ld_32x32b_x32(tbase + cc * 32, gr);
          tmem_ld_32x32b_x32(tbase + (GM_BN / 2) + cc * 32, ur);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float g0 = __uint_as_float(gr[2 * q]), g1 = __uint_as_float(gr[2 * q + 1]);
            const float u0 = __uint_as_float(ur[2 * q]), u1 = __uint_as_float(ur[2 * q + 1]);
            pk[q] = pack_bf16x2(silu_f(g0) * u0, silu_f(g1) * u1);
          }
          if constexpr (STG) {
#pragma unroll
            for (int q = 0; q < 4; ++q) stage16((cc & 1) * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            if (cc & 1) flush64(ocol + (cc >> 1) * 64);
          } else if (valid) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_global_v4(ocol + grow * p.ldo + cc * 32 + 8 * q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      } else {
        __nv_bfloat16* ocol = out + (long long)c.n * GM_BN;
#pragma unroll 1
        for (int cc = 0; cc < GM_BN / 32; ++cc) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + cc * 32, r);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) pk[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
          if constexpr (STG) {
#pragma unroll
            for (int q = 0; q < 4; ++q) stage16((cc & 1) * 4 + q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            if (cc & 1) {
              if constexpr (EPI == EPI_COMBINE)
                flush64c(ocol + (cc >> 1) * 64, (long long)c.n * GM_BN + (cc >> 1) * 64);
              else
                flush64(ocol + (cc >> 1) * 64);
            }
          } else if (valid) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_global_v4(ocol + grow * p.ldo + cc * 32 + 8 * q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
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

// Raster band (n-tiles per band): tiles run expert -> n-band -> m -> n, so the
// B band (band x 256 rows x K) is shared by every m-tile of the expert and A
// is re-read once per band.  Pick the widest band that divides n_tiles and
// whose B band stays within an L2 budget (32 MB for K3, 64 MB for K4); e.g.
// C2 K3 (K=4096): 16, C2 K4 (K=14336): 8, C4 K3 (11 n-tiles, K=2048): 11.  COX_GEMM_BAND_K3 /
// COX_GEMM_BAND_K4 override for experiments.
static int pick_band(int epi, int n_tiles, int K) {
  static int env_band[2] = {
      [] { const char* e = getenv("COX_GEMM_BAND_K3"); return e ? atoi(e) : 0; }(),
      [] { const char* e = getenv("COX_GEMM_BAND_K4"); return e ? atoi(e) : 0; }()};
  const int want = env_band[epi ? 1 : 0];
  if (want > 0 && n_tiles % want == 0) return want;
  const long long per_tile = (long long)GM_BN * K * 2;
  // measured (ncu dram__bytes_read, C2): K3 band 16 -> 33 GB (28 -> 57 GB);
  // K4 band 4/8/16 -> 77/69/143 GB, so the long-K down projection gets a larger budget
  const long long budget = epi ? (64LL << 20) : (32LL << 20);
  long long max_band = budget / per_tile;
  if (max_band < 1) max_band = 1;
  for (int b = (int)(max_band < n_tiles ? max_band : n_tiles); b >= 1; --b)
    if (n_tiles % b == 0) return b;
  return 1;
}

// ------------------------------------------------------------------ die discovery
// B200 has two dies, each with half of the L2; an operand used by SMs of both
// dies is fetched into both halves (the L2 fabric counters show it).  The SM ->
// die map is per GPU (yield-dependent), so it is measured once per process: each
// SM times L2 hits to 256 lines; lines homed on its own die are faster, so SMs
// of one die share a latency pattern (within-group correlation ~0.9, between
// ~ -0.7 on the measured boards).  OFF by default (COX_DIE_AWARE=1 enables):
// measured on C2 it RAISES K3's DRAM reads 33 -> 138 GB and the L2 fabric
// traffic 4x (1.71 vs 1.86 M tok/s) — operands shared by both dies are served
// better than disjoint per-die working sets; C4 gains ~1.5%.  Kept as an
// experiment switch, see DESIGN.md.
__global__ void die_probe_kernel(const int* __restrict__ buf, int nlines, int stride_ints, unsigned* lat,
                                 int* smid_out) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x) return;
  smid_out[blockIdx.x] = (int)smid;
  int sink = 0;
  for (int i = 0; i < nlines; ++i) {
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(buf + (long)i * stride_ints));
    sink += v;
  }
  for (int i = 0; i < nlines; ++i) {
    const long long t0 = clock64();
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(buf + (long)i * stride_ints + (sink & 1)));
    sink += v;
    const long long t1 = clock64();
    lat[blockIdx.x * nlines + i] = (unsigned)(t1 - t0);
  }
  if (sink == 123456789) lat[0] = 0;
}

static const int* die_map_device(int num_sms) {
  static int* d_map = nullptr;
  static bool tried = false;
  if (tried) return d_map;
  tried = true;
  const char* env = getenv("COX_DIE_AWARE");
  if (!env || atoi(env) == 0) return nullptr;
  const int nlines = 256, stride = 1536, nb = num_sms * 4;
  int* buf = nullptr;
  unsigned* lat = nullptr;
  int* sm = nullptr;
  bool ok = cudaMalloc(&buf, (size_t)nlines * stride * 4 + 64) == cudaSuccess &&
            cudaMalloc(&lat, (size_t)nb * nlines * 4) == cudaSuccess && cudaMalloc(&sm, nb * 4) == cudaSuccess &&
            cudaMemset(buf, 0, (size_t)nlines * stride * 4 + 64) == cudaSuccess;
  std::vector<unsigned> h((size_t)nb * nlines);
  std::vector<int> hs(nb);
  if (ok) {
    die_probe_kernel<<<nb, 32>>>(buf, nlines, stride, lat, sm);
    die_probe_kernel<<<nb, 32>>>(buf, nlines, stride, lat, sm);
    ok = cudaDeviceSynchronize() == cudaSuccess &&
         cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(hs.data(), sm, nb * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(buf);
  cudaFree(lat);
  cudaFree(sm);
  if (!ok) {
    cudaGetLastError();
    return nullptr;
  }
  // per-SM mean latency vector (centred), correlation with SM 0's vector
  std::vector<double> M((size_t)num_sms * nlines, 0.0);
  std::vector<int> n(num_sms, 0);
  for (int b = 0; b < nb; ++b) {
    const int id = hs[b];
    if (id < 0 || id >= num_sms) return nullptr;
    n[id]++;
    for (int i = 0; i < nlines; ++i) M[(size_t)id * nlines + i] += h[(size_t)b * nlines + i];
  }
  for (int id = 0; id < num_sms; ++id) {
    if (!n[id]) return nullptr;
    double mean = 0;
    for (int i = 0; i < nlines; ++i) mean += (M[(size_t)id * nlines + i] /= n[id]);
    mean /= nlines;
    for (int i = 0; i < nlines; ++i) M[(size_t)id * nlines + i] -= mean;
  }
  auto corr = [&](int a, int b) {
    double ab = 0, aa = 0, bb = 0;
    for (int i = 0; i < nlines; ++i) {
      const double x = M[(size_t)a * nlines + i], y = M[(size_t)b * nlines + i];
      ab += x * y;
      aa += x * x;
      bb += y * y;
    }
    return ab / std::sqrt(aa * bb + 1e-30);
  };
  std::vector<int> die(num_sms);
  int n1 = 0;
  double worst = 1.0;
  for (int id = 0; id < num_sms; ++id) {
    const double c = corr(0, id);
    die[id] = c > 0 ? 0 : 1;
    n1 += die[id];
    worst = std::min(worst, std::fabs(c));
  }
  // a clean two-way split is required; otherwise stay die-agnostic
  if (worst < 0.3 || n1 < num_sms / 4 || n1 > 3 * num_sms / 4) return nullptr;
  for (int id = 0; id + 1 < num_sms; id += 2)  // CTA pairs (clusters) never straddle dies
    if (die[id] != die[id + 1]) return nullptr;
  if (cudaMalloc(&d_map, num_sms * sizeof(int)) != cudaSuccess) return d_map = nullptr;
  cudaMemcpy(d_map, die.data(), num_sms * sizeof(int), cudaMemcpyHostToDevice);
  return d_map;
}

static int g_num_sms = 0;

// epi: EPI_SWIGLU (B = W13 interleaved [2ff, K], out = h [rows_cap, ff])
//      EPI_STORE  (B = W2 [N, K],                out = y [rows_cap, N])
//      EPI_COMBINE (B = W2 of the shared expert, out = final [T, N]; cmb = routed y_perm / dst / w / k)
int launch_grouped_gemm(int epi, const void* A, long long rows_cap, int K, const int32_t* offsets, int n_groups,
                        const int32_t* group_expert, const void* const* B, int N, void* out, long long ldo,
                        int max_ctas, cudaStream_t s, const int32_t* a_rows, long long a_rows_cap,
                        const GemmCombine* cmb) {
  if (n_groups <= 0) return 0;
  static GemmParams p;  // large (8.6 KB): built in static storage, copied at launch
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  // gather mode: A is x [rows_cap = T, K] read row by row (box of 1 row x 64 cols)
  int rc = get_map(&p.a_map, A, (unsigned long long)rows_cap, (unsigned long long)K, a_rows ? 1u : (unsigned)GM_BM);
  if (rc) return rc;
  for (int g = 0; g < n_groups; ++g) {
    rc = get_map(&p.b_map[g], B[g], (unsigned long long)N, (unsigned long long)K, GM_BN / 2);
    if (rc) return rc;
    p.group_expert[g] = group_expert[g];
  }
  static int* counters = nullptr;
  static unsigned seq = 0;
  if (!counters) {
    if (cudaMalloc(&counters, 1024 * sizeof(int)) != cudaSuccess) return -2;
    if (cudaMemset(counters, 0, 1024 * sizeof(int)) != cudaSuccess) return -2;
  }
  const unsigned slot = seq++ % 1024;
  int* counter = counters + slot;
  if (cudaMemsetAsync(counter, 0, sizeof(int), s) != cudaSuccess) return -2;
  p.tile_counter = counter;
  static unsigned long long* words = nullptr;
  if (!words) {
    if (cudaMalloc(&words, 1024 * sizeof(unsigned long long)) != cudaSuccess) return -2;
  }
  p.tile_word = words + slot;
  if (cudaMemsetAsync(p.tile_word, 0, sizeof(unsigned long long), s) != cudaSuccess) return -2;
  p.offsets = offsets;
  p.a_rows = a_rows;
  p.a_rows_cap = a_rows_cap;
  p.out = out;
  p.ldo = ldo;
  p.cy = cmb ? static_cast<const __nv_bfloat16*>(cmb->y_perm) : nullptr;
  p.cdst = cmb ? cmb->dst : nullptr;
  p.cw = cmb ? cmb->w : nullptr;
  p.ck = cmb ? cmb->k : 0;
  p.n_groups = n_groups;
  p.K = K;
  p.n_tiles = N / GM_BN;
  p.band = pick_band(epi, p.n_tiles, K);
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  p.die_map = die_map_device(g_num_sms);
  int grid = (g_num_sms / 2) * 2;
  if (max_ctas >= 2 && max_ctas < grid) grid = (max_ctas / 2) * 2;
  // K per stage: measured on C2, the SwiGLU GEMM is faster with BK=128 (3 stages;
  // K3 92.2 -> 89.6 ms) while the long-K down projection prefers BK=64 with 6
  // stages (42.6 vs 43.6 ms).  COX_GEMM_BK=64|128 forces one value for both.
  static int env_bk = [] {
    const char* e = getenv("COX_GEMM_BK");
    return e ? atoi(e) : 0;
  }();
  int ka = env_bk == 128 ? 2 : env_bk == 64 ? 1 : (epi == EPI_SWIGLU ? 2 : 1);
  if (epi == EPI_COMBINE) ka = 1;
  if (K % (ka * GM_BK) != 0) ka = 1;
  cudaError_t err;
#define GM_LAUNCH(E_, KA_, STG_)                                                                            \
  do {                                                                                                      \
    static bool attr = false;                                                                               \
    if (!attr) {                                                                                            \
      cudaFuncSetAttribute(grouped_gemm_kernel<E_, KA_, STG_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)GmRing<KA_, STG_>::SMEM);                                                   \
      attr = true;                                                                                          \
    }                                                                                                       \
    grouped_gemm_kernel<E_, KA_, STG_><<<grid, GM_THREADS, GmRing<KA_, STG_>::SMEM, s>>>(p);                \
  } while (0)
  // COX_GEMM_NOSTG=1: BK = 64 kernels without the epilogue staging tile, 7 ring stages (experiment)
  static const bool nostg = [] {
    const char* e = getenv("COX_GEMM_NOSTG");
    return e && atoi(e) == 1;
  }();
  if (epi == EPI_COMBINE) {
    GM_LAUNCH(EPI_COMBINE, 1, true);
  } else if (epi == EPI_SWIGLU) {
    if (ka == 2) GM_LAUNCH(EPI_SWIGLU, 2, true);
    else if (nostg) GM_LAUNCH(EPI_SWIGLU, 1, false);
    else GM_LAUNCH(EPI_SWIGLU, 1, true);
  } else {
    if (ka == 2) GM_LAUNCH(EPI_STORE, 2, true);
    else if (nostg) GM_LAUNCH(EPI_STORE, 1, false);
    else GM_LAUNCH(EPI_STORE, 1, true);
  }
#undef GM_LAUNCH
  err = cudaGetLastError();
  return err == cudaSuccess ? 0 : -2;
}

}  // namespace cox
