// K1 on tensor cores with exact re-scoring: the router's GEMM-shaped bulk
// (T x E x d multiply-adds) runs on tcgen05, and only the few logits that can
// decide the top-k are recomputed on CUDA cores in the canonical order of the
// CPU oracle (oracle/oracle_router.c; router.cu's order), so the routing
// indices stay bit-exact.
//
//   R1 router_screen_kernel (tcgen05, TMEM):  approx[t, e] = x_t . w_e (bf16 x
//      bf16 products, fp32 tensor-core accumulation) for a 128-token tile x all
//      E experts (MMA N = E padded to 16); two helper warps read the same smem
//      tiles to get ||x_t||_inf and every expert's ||w_e||_1, from which the
//      epilogue writes a per-token error bound
//          margin_t = gamma(d) * ||x_t||_inf * max_e ||w_e||_1
//      >= |approx - exact| + |canonical - exact| for every e (gamma: worst-case
//      rounding of d/16 tensor-core accumulation steps plus d/32 + 5 canonical
//      fp32 steps, x4 safety; SURVEY.md §0.5 explains why the canonical order
//      is needed at all).
//   R2 router_rescore_kernel (one warp per token scores, one lane per token
//      selects): k-th largest approx value a_k; candidates C = {e : approx_e >=
//      a_k - 2 margin_t}.  Every e outside C has exact_e < a_k - margin_t <=
//      exact_s for all k screened winners s, so the exact top-k lies in C.
//      Exact canonical logits for C (mixed-precision FHFMA.BF16 chains in the
//      lane chunk order + the xor butterfly's sums), then per lane over a
//      batch of tokens: top-k with ties to the lower index, weights from the
//      exact logits (Mixtral: softmax over the k: bit-exact; DeepSeek:
//      full-softmax denominator uses exact logits for C and the tensor-core
//      logits for the rest).
// Used when x and the router weight are bf16 (the checkpoint dtypes).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "common.cuh"
#include "route_common.cuh"

namespace cox {

int get_map(CUtensorMap* out, const void* ptr, unsigned long long rows, unsigned long long cols, unsigned box_rows);

constexpr int RC_BM = 128;  // tokens per tile (MMA M, TMEM lanes)
constexpr int RC_BK = 64;   // K per stage: one 128-byte swizzle atom
constexpr int RC_MAX_STAGES = 8;  // ring depth: as many 64-column stages as fit ~200 KB (8 at E <= 64)
constexpr int RC_THREADS = 256;
constexpr uint32_t RC_A_BYTES = RC_BM * RC_BK * 2;  // 16 KB

struct RcParams {
  CUtensorMap xmap;  // x [T, d] bf16, box {64, 128}
  CUtensorMap wmap;  // wg [E, d] bf16, box {64, Epad}; rows >= E read as zero
  float* approx;     // [T, E]
  float* margin;     // [T]
  int T, d, E, Epad;
  float gamma;
};

// two CTAs per SM, each with ~100 KB of ring (latency hiding from 16 warps)
__host__ __device__ constexpr int rc_stages(int Epad) {
  return (int)(100u * 1024u / (RC_A_BYTES + (uint32_t)Epad * 128u)) > RC_MAX_STAGES
             ? RC_MAX_STAGES
             : (int)(100u * 1024u / (RC_A_BYTES + (uint32_t)Epad * 128u));
}

constexpr size_t rc_smem_bytes(int Epad) {
  return 1024 + (size_t)rc_stages(Epad) * (RC_A_BYTES + (size_t)Epad * 128) + 1024 + 2 * RC_BM * 4 + 256 * 4 + 64;
}

COX_DEV float bf16_abs_max8(const uint4& v, float m) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m = fmaxf(m, fabsf(__uint_as_float(w[i] << 16)));
    m = fmaxf(m, fabsf(__uint_as_float(w[i] & 0xFFFF0000u)));
  }
  return m;
}
COX_DEV float bf16_abs_sum8(const uint4& v, float s) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s += fabsf(__uint_as_float(w[i] << 16));
    s += fabsf(__uint_as_float(w[i] & 0xFFFF0000u));
  }
  return s;
}

__global__ void __launch_bounds__(RC_THREADS, 2) router_screen_kernel(const __grid_constant__ RcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t B_BYTES = (uint32_t)p.Epad * 128;
  uint8_t* sA = smem;
  const int RC_STAGES = rc_stages(p.Epad);
  uint8_t* sB = smem + RC_STAGES * RC_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + RC_STAGES * B_BYTES);
  uint64_t* empty = full + RC_STAGES;
  uint64_t* tfull = empty + RC_STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained
  uint64_t* xready = tempty + 2;        // [2] row max-abs of the tile ready
  uint64_t* xfree = xready + 2;         // [2] epilogue done with it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfree + 2);
  float* s_xinf = reinterpret_cast<float*>(tmem_slot + 4);  // [2][128]
  float* s_w1 = s_xinf + 2 * RC_BM;                          // [256] ||w_e||_1, then [0] = max
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int acc_stride = p.Epad < 32 ? 32 : p.Epad;
  const uint32_t tmem_cols = acc_stride * 2 <= 32 ? 32 : acc_stride * 2 <= 64 ? 64 : acc_stride * 2 <= 128 ? 128 : acc_stride * 2 <= 256 ? 256 : 512;

  for (int e = threadIdx.x; e < 256; e += blockDim.x) s_w1[e] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RC_STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 3);  // MMA commit + 2 scanner warps
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 4);
      mbar_init(smem_u32(&xready[a]), 2);
      mbar_init(smem_u32(&xfree[a]), 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_slot), tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int ntiles = (p.T + RC_BM - 1) / RC_BM;
  const int nk = p.d / RC_BK;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_arrive_expect_tx(fb, RC_A_BYTES + B_BYTES);
          tma_load_2d(smem_u32(sA + stage * RC_A_BYTES), &p.xmap, fb, kb * RC_BK, tile * RC_BM);
          tma_load_2d(smem_u32(sB + stage * B_BYTES), &p.wmap, fb, kb * RC_BK, 0);
          if (++stage == RC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(RC_BM, p.Epad);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(smem_u32(&tempty[acc]), ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * acc_stride;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * RC_A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < RC_BK / 16; ++k)
            mma_bf16_ss<1>(d_tmem, sdesc_kmajor_sw128(a_base + k * 32), sdesc_kmajor_sw128(b_base + k * 32), idesc,
                           (kb | k) != 0 ? 1u : 0u);
          mma_commit<1>(smem_u32(&empty[stage]));
          if (++stage == RC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit<1>(smem_u32(&tfull[acc]));
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    // ------------------------------------------------------------ scanners
    // Read the same smem tiles as the MMA (conflict-free: each warp
    // instruction covers 512 contiguous bytes).  Warp w2 owns rows
    // [64 w2, 64 w2 + 64); lane l reads chunk l%8 of rows 64 w2 + 4i + l/8
    // (i < 16) and keeps their running max |x| (the swizzle only permutes the
    // chunks of a row, irrelevant for a max).  On the first tile the B slices
    // also give every expert's ||w_e||_1 (deterministic: one owner per row).
    const int w2 = warp - 2;
    uint32_t stage = 0, phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      float m[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = 0.f;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(&full[stage]), phase);
        const uint8_t* a = sA + stage * RC_A_BYTES + w2 * 64 * 128 + lane * 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = bf16_abs_max8(*reinterpret_cast<const uint4*>(a + i * 512), m[i]);
        if (it == 0) {
          const uint8_t* b = sB + stage * B_BYTES + lane * 16;
          for (int i = 0; 8 * i + 4 * w2 < p.Epad; ++i) {
            float sum = bf16_abs_sum8(*reinterpret_cast<const uint4*>(b + (8 * i + 4 * w2) * 128), 0.f);
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            sum += __shfl_xor_sync(0xffffffffu, sum, 4);
            if ((lane & 7) == 0) s_w1[8 * i + 4 * w2 + (lane >> 3)] += sum;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
        if (++stage == RC_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], 1));
        m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], 2));
        m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], 4));
      }
      mbar_wait(smem_u32(&xfree[buf]), ((it >> 1) & 1) ^ 1);
      if ((lane & 7) == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) s_xinf[buf * RC_BM + w2 * 64 + 4 * i + (lane >> 3)] = m[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&xready[buf]));
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 4;
    const int row = q * 32 + lane;
    int it = 0;
    float w1max = 0.f;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      mbar_wait(smem_u32(&xready[acc]), (it >> 1) & 1);
      if (it == 0) {
        for (int e = 0; e < p.E; ++e) w1max = fmaxf(w1max, s_w1[e]);
        // fp32 summation of d terms may under-estimate by (d * 2^-24): inflate
        w1max *= 1.0f + (float)p.d * 1.2e-7f;
      }
      const float xinf = s_xinf[acc * RC_BM + row];
      mbar_wait(smem_u32(&tfull[acc]), (it >> 1) & 1);
      tc_fence_after();
      const long long t = (long long)tile * RC_BM + row;
      float* dst = p.approx + t * p.E;
      for (int c0 = 0; c0 < p.E; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * acc_stride + c0, v);
        if (t < p.T) {
          const int n = min(32, p.E - c0);
          if ((p.E & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              if (j < n) st_global_v4(dst + c0 + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)  // static indices: v stays in registers
              if (j < n) dst[c0 + j] = __uint_as_float(v[j]);
          }
        }
      }
      if (t < p.T) p.margin[t] = p.gamma * xinf * w1max;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(smem_u32(&tempty[acc]));
        mbar_arrive(smem_u32(&xfree[acc]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, tmem_cols);
  }
}

// ---------------------------------------------------------------------------- R2
// One warp per token.  The candidates' exact logits are computed two chains
// at a time, each step one mixed-precision FMA on the packed bf16 operands
// (fma_bf16x2_seq: no widening instructions, bit-identical to fmaf on the
// widened values); a pair's per-lane partial sums are combined over the xor
// butterfly's exact pairs (reduce-scatter at 16, then 8..1), and the top-k,
// routing weights and histogram are warp_route_token's (route_common.cuh) on
// the token's logits: exact for the candidates, screened for the rest (which
// are provably below k exact candidate logits, so they are never selected).
constexpr int RR_WARPS = 8;
constexpr int RR_CH = 2;  // candidate chains in flight per warp (4: +2% time, more discarded chains)

// L1-allocating read-only load (the router rows are re-read by every token)
COX_DEV uint4 ldg_v4(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// NCH = x chunks per lane held in registers (d <= 256 NCH): the token's whole
// x row is requested at once, so a token costs one DRAM round trip.
template <int NCH, int NE, bool FULL>
__global__ void __launch_bounds__(RR_WARPS * 32, NCH <= 8 ? 2 : 1) router_rescore_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, const float* __restrict__ approx,
    const float* __restrict__ margin, int T, int d, int E, int k, int mode, int32_t* __restrict__ idx,
    float* __restrict__ wout, int32_t* __restrict__ counts) {
  // Tokens are scored one per warp (exact candidate logits need the whole
  // warp's lanes: the canonical lane-chunk order), but the per-token top-k and
  // softmax are serial work, so they run one token per LANE over a batch of
  // TB tokens: per warp, TB logit rows (screened, exact for the candidates;
  // pitch 32 NE + 1 so the lanes' row scans hit distinct banks) and each
  // token's candidate bit mask.
  constexpr int TB = 32 / NE < 4 ? 4 : 32 / NE;
  constexpr int PITCH = 32 * NE + 1;
  __shared__ float s_l[RR_WARPS][TB * PITCH];
  __shared__ uint32_t s_mask[RR_WARPS][TB][NE];
  __shared__ long long s_tok[RR_WARPS][TB];
  __shared__ uint8_t s_cand[RR_WARPS][32 * NE];
  __shared__ int s_hist[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  uint8_t* cand = s_cand[warp];
  // lane b < nb selects and weighs batch token b (same operations, in the same
  // order, as warp_route_token: largest value first, ties -> lower index; the
  // top-k lies among the candidates, which hold exact logits)
  auto finish_batch = [&](int nb) {
    __syncwarp();
    if (lane < nb) {
      const float* lr = s_l[warp] + lane * PITCH;
      const long long t = s_tok[warp][lane];
      uint32_t msk[NE];
      int nc = 0;
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        msk[i] = s_mask[warp][lane][i];
        nc += __popc(msk[i]);
      }
      if (nc < k) {  // only with non-finite margins (no candidates): select among all E screened values
#pragma unroll
        for (int i = 0; i < NE; ++i) msk[i] = (32 * i + 32 <= E) ? 0xffffffffu : ((1u << (E - 32 * i)) - 1u);
      }
      int sel[8];
      float selv[8];
      uint32_t taken[NE];
#pragma unroll
      for (int i = 0; i < NE; ++i) taken[i] = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // k <= 8; unrolled so sel / selv stay in registers
        sel[j] = 0;
        selv[j] = 0.f;
        if (j < k) {
          int be = -1, bw = 0, bb = 0;
          float bv = 0.f;
#pragma unroll
          for (int i = 0; i < NE; ++i) {
            for (uint32_t m = msk[i] & ~taken[i]; m; m &= m - 1u) {  // ascending expert order
              const int bit = __ffs(m) - 1;
              const float v = lr[32 * i + bit];
              if (be < 0 || v > bv) {
                be = 32 * i + bit;
                bv = v;
                bw = i;
                bb = bit;
              }
            }
          }
#pragma unroll
          for (int i = 0; i < NE; ++i)
            if (i == bw) taken[i] |= 1u << bb;
          sel[j] = be;
          selv[j] = bv;
        }
      }
      const float m = selv[0];
      float ssum = 0.0f;
      if (mode == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < k) ssum = __fadd_rn(ssum, expf(__fsub_rn(selv[j], m)));
      } else {
        for (int e = 0; e < E; ++e) ssum = __fadd_rn(ssum, expf(__fsub_rn(lr[e], m)));  // ascending e, as the oracle
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) {
          idx[t * k + j] = sel[j];
          wout[t * k + j] = __fdiv_rn(expf(__fsub_rn(selv[j], m)), ssum);
          atomicAdd(&s_hist[sel[j]], 1);
        }
    }
    __syncwarp();
  };
  int nb = 0;
  // the next token's x row, screened logits and margin are requested while
  // the current token is scored (one DRAM round trip hidden per token)
  const long long tstep = (long long)gridDim.x * RR_WARPS;
  long long t = (long long)blockIdx.x * RR_WARPS + warp;
  uint4 xn[NCH];
  float an[NE], mn = 0.f;
  auto fetch = [&](long long tt) {
    if (tt >= T) return;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int s = 8 * lane + 256 * j;
      xn[j] = (FULL || s < d) ? ld_nc_v4(x + tt * d + s) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = lane + 32 * i;
      an[i] = e < E ? approx[tt * E + e] : -INFINITY;
    }
    mn = margin[tt];
  };
  fetch(t);
  for (; t < T; t += tstep) {
    uint4 xq[NCH];
    float av[NE];
#pragma unroll
    for (int j = 0; j < NCH; ++j) xq[j] = xn[j];
#pragma unroll
    for (int i = 0; i < NE; ++i) av[i] = an[i];
    const float mt = mn;
    fetch(t + tstep);
    float* lg = s_l[warp] + nb * PITCH;
    uint32_t key[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = lane + 32 * i;
      av[i] = av[i] != av[i] ? -INFINITY : av[i];  // NaN ranks like -inf (router.cu nan_low)
      if (e < E) lg[e] = av[i];
      key[i] = e < E ? route_key(av[i]) : 0u;
    }
    // k-th largest screened VALUE: k rounds of a warp max over order keys;
    // equal values leave together (that can only lower the threshold: a superset)
    uint32_t mk = 0;
    for (int j = 0; j < k; ++j) {
      uint32_t bk = 0;
#pragma unroll
      for (int i = 0; i < NE; ++i) bk = key[i] > bk ? key[i] : bk;
      mk = __reduce_max_sync(0xffffffffu, bk);
#pragma unroll
      for (int i = 0; i < NE; ++i)
        if (key[i] == mk) key[i] = 0;
    }
    const float kth = __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk);
    const float thr = kth - 2.0f * mt;
    int nc = 0;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = lane + 32 * i;
      const bool c = e < E && av[i] >= thr;
      const uint32_t bal = __ballot_sync(0xffffffffu, c);
      if (c) cand[nc + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)e;
      nc += __popc(bal);
      if (lane == 0) s_mask[warp][nb][i] = bal;
    }
    if (lane == 0) s_tok[warp][nb] = t;
    __syncwarp();
    // candidates RR_CH at a time (a runtime loop: only real candidates cost
    // FMAs; a short last group runs beside discarded duplicates)
    for (int c = 0; c < nc; c += RR_CH) {
      const __nv_bfloat16* wr[RR_CH];
      float a[RR_CH];
#pragma unroll
      for (int u = 0; u < RR_CH; ++u) {
        wr[u] = wg + (long long)cand[c + u < nc ? c + u : c] * d + 8 * lane;
        a[u] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        if (FULL || 8 * lane + 256 * j < d) {  // FULL: d == 256 NCH, every lane owns NCH chunks
          uint4 p[RR_CH];
#pragma unroll
          for (int u = 0; u < RR_CH; ++u) p[u] = ldg_v4(wr[u] + 256 * j);
#pragma unroll
          for (int u = 0; u < RR_CH; ++u) fma_bf16x2_seq(a[u], xq[j].x, p[u].x);
#pragma unroll
          for (int u = 0; u < RR_CH; ++u) fma_bf16x2_seq(a[u], xq[j].y, p[u].y);
#pragma unroll
          for (int u = 0; u < RR_CH; ++u) fma_bf16x2_seq(a[u], xq[j].z, p[u].z);
#pragma unroll
          for (int u = 0; u < RR_CH; ++u) fma_bf16x2_seq(a[u], xq[j].w, p[u].w);
        }
      }
      // butterfly sums of the group over the xor butterfly's exact pairs:
      // reduce-scatter at 16, then plain levels 8, 4, 2, 1; chain u ends in
      // lanes 16 u .. 16 u + 15
      static_assert(RR_CH == 2, "reduce-scatter below is written for 2 chains");
      float v1[1];
      rs_step<1>(a, v1, lane, 16);
      float r = v1[0];
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, off));
      const int u = lane >> 4;
      if ((lane & 15) == 0 && c + u < nc) lg[cand[c + u]] = r != r ? -INFINITY : r;
    }
    __syncwarp();  // this token's cand / lg accesses before the next token's writes
    if (++nb == TB) {
      finish_batch(nb);
      nb = 0;
    }
  }
  if (nb) finish_batch(nb);
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&counts[i], s_hist[i]);
}

// Screening + re-scoring router.  scratch: T*E + T floats from the caller's
// workspace (approx logits, then per-token margins), so concurrent launches
// on different streams or graphs never share it.  Returns -3 if the shape is
// not supported by the tensor-core screen (caller falls back to the CUDA-core
// router).
int launch_router_tc(const void* x, const void* wg, int T, int d, int E, int k, int mode, int32_t* idx, float* w,
                     int32_t* counts, float* scratch, cudaStream_t s) {
  if (d % RC_BK != 0 || d > 24 * 256 || E > 256 || E < 1 || k > 8) return -3;
  if (cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s) != cudaSuccess) return -2;
  if (T == 0) return 0;
  RcParams p;
  const int Epad = ((E + 15) / 16) * 16;
  int rc = get_map(&p.xmap, x, (unsigned long long)T, (unsigned long long)d, RC_BM);
  if (rc) return rc;
  rc = get_map(&p.wmap, wg, (unsigned long long)E, (unsigned long long)d, (unsigned)Epad);
  if (rc) return rc;
  p.approx = scratch;
  p.margin = scratch + (size_t)T * E;
  p.T = T;
  p.d = d;
  p.E = E;
  p.Epad = Epad;
  // worst-case rounding: d/16 tensor-core accumulation steps of <= 4 ulp plus
  // d/32 + 5 canonical fp32 steps of <= 1 ulp, relative to sum |x_i w_i| <=
  // ||x||_inf ||w||_1; x4 safety
  p.gamma = (float)(4.0 * ((d / 16.0 + 16.0) * 4.0 + d / 32.0 + 5.0) * std::ldexp(1.0, -24));
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ntiles = (T + RC_BM - 1) / RC_BM;
  const int grid = ntiles < 2 * num_sms ? ntiles : 2 * num_sms;
  const size_t smem = rc_smem_bytes(Epad);
  // the ring depth depends on E, so the largest footprint is not at E = 256:
  // raise the kernel's dynamic shared-memory limit whenever a launch needs more
  static size_t attr_bytes = 0;
  if (smem > attr_bytes) {
    if (cudaFuncSetAttribute(router_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return -2;
    attr_bytes = smem;
  }
  router_screen_kernel<<<grid, RC_THREADS, smem, s>>>(p);
  long long blocks = ((long long)T + RR_WARPS - 1) / RR_WARPS;
  if (blocks > (long long)num_sms * 8) blocks = (long long)num_sms * 8;
#define RR_LAUNCH3(NCH_, NE_, F_)                                                                                 \
  do {                                                                                                             \
    static bool carve = false;                                                                                     \
    if (!carve) { /* router rows flow through L1: the smallest carveout that fits 2 CTAs (~37 KB each) */          \
      cudaFuncSetAttribute(router_rescore_kernel<NCH_, NE_, F_>, cudaFuncAttributePreferredSharedMemoryCarveout,   \
                           40);                                                                                    \
      carve = true;                                                                                                \
    }                                                                                                              \
    router_rescore_kernel<NCH_, NE_, F_><<<(int)blocks, RR_WARPS * 32, 0, s>>>(                                    \
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(wg), p.approx, p.margin, T, d, E,   \
        k, mode, idx, w, counts);                                                                                  \
  } while (0)
#define RR_LAUNCH(NCH_, NE_)                       \
  do {                                             \
    if (d == 256 * (NCH_)) RR_LAUNCH3(NCH_, NE_, true); \
    else RR_LAUNCH3(NCH_, NE_, false);             \
  } while (0)
#define RR_BY_NE(NCH_)                          \
  do {                                          \
    if (E <= 32) RR_LAUNCH(NCH_, 1);            \
    else if (E <= 64) RR_LAUNCH(NCH_, 2);       \
    else if (E <= 128) RR_LAUNCH(NCH_, 4);      \
    else RR_LAUNCH(NCH_, 8);                    \
  } while (0)
  const int nch = (d + 255) / 256;
  if (nch <= 4) RR_BY_NE(4);
  else if (nch <= 8) RR_BY_NE(8);
  else if (nch <= 16) RR_BY_NE(16);
  else if (nch <= 24) RR_BY_NE(24);
  else return -3;
#undef RR_BY_NE
#undef RR_LAUNCH
#undef RR_LAUNCH3
  return launch_status();
}

}  // namespace cox
