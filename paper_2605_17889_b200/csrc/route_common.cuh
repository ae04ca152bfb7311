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

// lg: the token's E logits in shared memory (overwritten with the exp terms in
// mode 1); s_sel / s_selv: this warp's [8] shared scratch; idx / w: the
// token's k outputs; hist: optional shared/global histogram (+1 per selected
// expert).  E <= 256, k <= 8.
COX_DEV void warp_route_token(float* lg, int E, int k, int mode, int lane, int* s_sel, float* s_selv,
                              int32_t* idx, float* w, int* hist) {
  uint32_t taken = 0;  // bit i: expert lane + 32 i already selected
  for (int j = 0; j < k; ++j) {
    float bv = 0.0f;
    int bi = -1;
    for (int i = 0; lane + 32 * i < E; ++i) {
      const int e = lane + 32 * i;
      if (taken & (1u << i)) continue;
      const float v = lg[e];
      if (bi < 0 || v > bv) {
        bv = v;
        bi = e;
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    if (lane == 0) {
      s_sel[j] = bi;
      s_selv[j] = bv;
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

}  // namespace cox
