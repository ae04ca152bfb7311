// Per-token top-k selection and routing weights, shared by every router
// kernel that holds a token's E logits in shared memory (router.cu,
// small_gemm.cu's in-kernel router).  One warp per token.
//
// Semantics (oracle/oracle_router.c:oracle_router_topk): the k largest logits
// in descending order, ties -> lower expert index (eas.py:364-374 convention);
// weights: mode 0 (Mixtral) softmax over the k selected logits, mode 1
// (DeepSeek-V2) softmax over all E, denominator summed in ascending e.
#pragma once
#include "common.cuh"

namespace cox {

// Recursive-halving step: lane keeps the half of `v` selected by (lane & off)
// and adds the partner's copy of the same logits.
template <int N>
COX_DEV void rs_step(float (&v)[2 * N], float (&o)[N], int lane, int off) {
  const bool upper = (lane & off) != 0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const float keep = upper ? v[N + m] : v[m];
    const float send = upper ? v[m] : v[N + m];
    o[m] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, off));
  }
}

// lg: the token's E logits in shared memory (overwritten with the exp terms in
// mode 1); s_sel / s_selv: this warp's [8] shared scratch; idx / w: the
// token's k outputs; hist: optional shared/global histogram (+1 per selected
// expert).  E <= 256, k <= 8.
// Order-preserving map of a float to an unsigned key (larger float -> larger
// key; -inf -> 0x007fffff > 0 = "no candidate"; -0 and +0 share a key, so they
// tie as under float comparison).  Logits are NaN-free here (callers map NaN
// to -inf).
COX_DEV uint32_t route_key(float v) {
  const uint32_t b = v == 0.0f ? 0u : __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// NI = logits per lane held as keys (E <= 32 NI): callers that know E is small
// pass a smaller NI (each selection round scans NI registers per lane).
template <int NI = 8>
COX_DEV void warp_route_token(float* lg, int E, int k, int mode, int lane, int* s_sel, float* s_selv,
                              int32_t* idx, float* w, int* hist) {
  // the lane's logits (experts lane + 32 i) in registers, selected ones knocked
  // out; each round: the lane's best (lowest index among equals), then two
  // warp-wide redux steps: max key, then min index among the lanes holding it
  // (= the old shuffle butterfly's choice: largest value, ties -> lower index)
  uint32_t key[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) key[i] = (lane + 32 * i < E) ? route_key(lg[lane + 32 * i]) : 0u;
  for (int j = 0; j < k; ++j) {
    uint32_t bk = 0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (key[i] > bk) {
        bk = key[i];
        bi = lane + 32 * i;
      }
    const uint32_t mk = __reduce_max_sync(0xffffffffu, bk);
    const int e = (int)__reduce_min_sync(0xffffffffu, (uint32_t)(bk == mk ? bi : 0x7fffffff));
    if ((e & 31) == lane) {
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (i == (e >> 5)) key[i] = 0;
    }
    if (lane == 0) {
      s_sel[j] = e;
      s_selv[j] = lg[e];
    }
  }
  __syncwarp();
  if (mode != 0) {  // full softmax: every expf in parallel (in place; the logits are no longer needed)
    const float m0 = s_selv[0];
    for (int e = lane; e < E; e += 32) lg[e] = expf(__fsub_rn(lg[e], m0));
    __syncwarp();
  }
  const float m = s_selv[0];
  float ssum = 0.0f;
  if (lane == 0) {
    if (mode == 0) {
      for (int j = 0; j < k; ++j) ssum = __fadd_rn(ssum, expf(__fsub_rn(s_selv[j], m)));
    } else {
      // ascending e, as the oracle; eight shared loads in flight per step of the add chain
      int e = 0;
      for (; e + 8 <= E; e += 8) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = lg[e + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) ssum = __fadd_rn(ssum, v[q]);
      }
      for (; e < E; ++e) ssum = __fadd_rn(ssum, lg[e]);
    }
  }
  ssum = __shfl_sync(0xffffffffu, ssum, 0);
  if (lane < k) {  // one selected expert per lane: the same expression per weight as a serial loop
    const int e = s_sel[lane];
    idx[lane] = e;
    w[lane] = __fdiv_rn(expf(__fsub_rn(s_selv[lane], m)), ssum);
    if (hist) atomicAdd(&hist[e], 1);
  }
  __syncwarp();
}

// warp_route_token with the key scan sized to E at run time (E is uniform
// across the launch, so the branch is too): E <= 64 scans 2 registers per lane
// per selection round instead of 8.
COX_DEV void warp_route_token_e(float* lg, int E, int k, int mode, int lane, int* s_sel, float* s_selv, int32_t* idx,
                                float* w, int* hist) {
  if (E <= 32) warp_route_token<1>(lg, E, k, mode, lane, s_sel, s_selv, idx, w, hist);
  else if (E <= 64) warp_route_token<2>(lg, E, k, mode, lane, s_sel, s_selv, idx, w, hist);
  else if (E <= 128) warp_route_token<4>(lg, E, k, mode, lane, s_sel, s_selv, idx, w, hist);
  else warp_route_token<8>(lg, E, k, mode, lane, s_sel, s_selv, idx, w, hist);
}

}  // namespace cox
