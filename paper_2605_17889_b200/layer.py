"""The coalesced MoE expert stage on one B200: router -> permute -> grouped
SwiGLU -> grouped down -> combine, all in libcoxmoe.so.

``MoELayer.forward`` is the single-GPU, all-resident path (the reference's
``AllocationStrategy(exp_r=E, exp_m=0, exp_c=0)``).  Residency/streaming and
expert parallelism build on the same stage functions (executor.py, ep.py).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import _lib, ops
from .synthetic import LayerWeights

MODES = {"mixtral": _lib.ROUTE_MIXTRAL, "deepseek": _lib.ROUTE_DEEPSEEK}


@dataclass
class StageBuffers:
    T: int
    idx: torch.Tensor
    w: torch.Tensor
    counts: torch.Tensor
    offsets: torch.Tensor
    dst: torch.Tensor
    x_perm: torch.Tensor
    h: torch.Tensor
    y: torch.Tensor
    out: torch.Tensor
    workspace: torch.Tensor
    row_tokens: torch.Tensor | None = None  # gather mode: source token of every permuted row
    x_ref: torch.Tensor | None = None       # gather mode: the step's input (A source of K3)
    shared_offsets: torch.Tensor | None = None
    shared_h: torch.Tensor | None = None
    shared_y: torch.Tensor | None = None


def alloc_buffers(T: int, d: int, ff: int, E: int, k: int, tile_m: int, device, out_dtype=torch.bfloat16,
                  shared_ff: int = 0, gather_a: bool = False) -> StageBuffers:
    cap = ops.rows_capacity(T, k, E, tile_m)
    bf = torch.bfloat16
    b = StageBuffers(
        T=T,
        idx=torch.empty((T, k), dtype=torch.int32, device=device),
        w=torch.empty((T, k), dtype=torch.float32, device=device),
        counts=torch.empty((E,), dtype=torch.int32, device=device),
        offsets=torch.empty((E + 1,), dtype=torch.int32, device=device),
        dst=torch.empty((T, k), dtype=torch.int32, device=device),
        x_perm=torch.empty((1 if gather_a else cap, d), dtype=bf, device=device),
        h=torch.empty((cap, ff), dtype=bf, device=device),
        y=torch.empty((cap, d), dtype=bf, device=device),
        out=torch.empty((T, d), dtype=out_dtype, device=device),
        workspace=torch.empty((max(16, ops.permute_workspace_bytes(T, E)),), dtype=torch.uint8, device=device),
    )
    if gather_a:
        b.row_tokens = torch.empty((cap,), dtype=torch.int32, device=device)
    if shared_ff:
        b.shared_offsets = torch.tensor([0, T], dtype=torch.int32, device=device)
        b.shared_h = torch.empty((max(T, 1), shared_ff), dtype=bf, device=device)
        b.shared_y = torch.empty((max(T, 1), d), dtype=bf, device=device)
    return b


class MoELayer:
    """One MoE layer's expert stage with every expert resident in HBM."""

    def __init__(self, weights: LayerWeights, top_k: int, mode: str = "mixtral", tile_m: int = 1,
                 out_dtype=torch.bfloat16, gather_a: bool | None = None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")
        self.wts = weights
        self.k = int(top_k)
        self.mode = MODES[mode]
        self.tile_m = int(tile_m)
        self.out_dtype = out_dtype
        # gather-fused A loads (TMA tile::gather4): K3 reads token rows from x directly
        if gather_a is None:
            gather_a = os.environ.get("COX_GATHER_A", "0") == "1"
        self.gather_a = bool(gather_a)
        self.E = weights.num_experts
        self.d = weights.hidden_dim
        self.ff = weights.expert_dim
        if not (1 <= self.k <= self.E):
            raise ValueError("top_k must satisfy 1 <= top_k <= experts_per_layer")
        self.groups = list(range(self.E))
        # router weight in bf16 when that is exact (bf16 checkpoints): half the bytes, smem-staged for E > 8
        wgb = weights.wg.to(torch.bfloat16)
        self.wg_router = wgb if torch.equal(wgb.float(), weights.wg) else weights.wg
        self.w13_list = [weights.w13[e] for e in range(self.E)]
        self.w2_list = [weights.w2[e] for e in range(self.E)]
        self.shared_ff = weights.shared_w2.shape[1] if weights.shared_w2 is not None else 0
        if self.shared_ff and out_dtype != torch.bfloat16:
            raise ValueError("shared experts require a bf16 output")
        self._bufs: StageBuffers | None = None
        self.profile_events = None  # optional {"k3": (ev0, ev1), "k4": (ev0, ev1)} recorded around K3/K4

    def launches_per_step(self, T: int | None = None) -> int:
        # router 1 + permute 4 (hist, scan, scatter, copy; +1 pad) + K3 + K4 + combine (+ shared K3/K4);
        # decode-size batches: K3, K4 and the shared experts are one launch
        # permute: single-CTA index kernel for T*k <= 16384 (else hist, scan, scatter) + row copy (+ pad)
        small_perm = T is not None and T * self.k <= 16384
        perm = (1 if small_perm else 3) + 1 + (1 if self.tile_m > 1 else 0)
        if T is not None and self.uses_dense_decode(T):
            return 1  # router + all experts + shared + combine in one launch
        if T is not None and self.uses_routed_one_launch(T):
            return 1  # router in the prologue of the K3/K4/shared/combine launch
        if T is not None and self.uses_idx_decode(T):
            return 2  # router, then one launch for K3/K4/shared/combine reading the router's idx
        if T is not None and self.uses_small_path(T):
            # router + single-CTA permute (indices only; + row copy above the gather
            # threshold) + one launch for K3/K4/shared/combine
            perm_small_path = 1 if small_perm else 3
            return (1 + perm_small_path + (0 if self._small_gather(T) else 1) + 1
                    + (1 if self.out_dtype != torch.bfloat16 else 0))
        if (self.shared_ff and self.SHARED_FUSED_COMBINE and self.k <= 8
                and not (T is not None and 0 < T * self.k <= self.SHARED_SIDE_MAX_ROWS)):
            return 1 + perm + 2 + 2  # shared K3 + shared down with the combine in its epilogue
        return 1 + perm + 2 + 1 + (2 if self.shared_ff else 0)

    def buffers(self, T: int, device) -> StageBuffers:
        if self._bufs is None or self._bufs.T != T:
            self._bufs = None
            self._bufs = alloc_buffers(T, self.d, self.ff, self.E, self.k, self.tile_m, device, self.out_dtype,
                                       self.shared_ff, self.gather_a)
            if self.uses_small_path(T) and self._bufs.row_tokens is None:
                self._bufs.row_tokens = torch.empty((self._bufs.h.shape[0],), dtype=torch.int32, device=device)
        return self._bufs

    # --- stages (all stream-ordered on the current stream) -------------------
    def route(self, x: torch.Tensor, b: StageBuffers):
        ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts))
        if self.gather_a:
            ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, None), workspace=b.workspace,
                        copy_rows=False, row_tokens=b.row_tokens)
            b.x_ref = x
        else:
            ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, b.x_perm), workspace=b.workspace)

    def _k3(self, b: StageBuffers, groups, w13, max_ctas: int = 0):
        if self.gather_a:
            ops.grouped_swiglu_gather(b.x_ref, b.row_tokens, b.offsets, groups, w13, self.ff, h=b.h,
                                      max_ctas=max_ctas)
        else:
            ops.grouped_swiglu(b.x_perm, b.offsets, groups, w13, self.ff, h=b.h, max_ctas=max_ctas)

    def experts(self, b: StageBuffers, groups=None, w13=None, w2=None):
        groups = self.groups if groups is None else groups
        pe = self.profile_events
        if pe:
            pe["k3"][0].record()
        self._k3(b, groups, self.w13_list if w13 is None else w13)
        if pe:
            pe["k3"][1].record()
            pe["k4"][0].record()
        ops.grouped_down(b.h, b.offsets, groups, self.w2_list if w2 is None else w2, self.d, y=b.y)
        if pe:
            pe["k4"][1].record()

    def shared_expert(self, x: torch.Tensor, b: StageBuffers):
        if not self.shared_ff:
            return None
        ops.grouped_swiglu(x, b.shared_offsets, [0], [self.wts.shared_w13], self.shared_ff, h=b.shared_h)
        ops.grouped_down(b.shared_h, b.shared_offsets, [0], [self.wts.shared_w2], self.d, y=b.shared_y)
        return b.shared_y

    def finish(self, b: StageBuffers, shared=None, out=None):
        return ops.combine(b.y, b.dst, b.w, shared, out=b.out if out is None else out)

    # decode-size batches: the shared expert runs beside the routed experts on a
    # side stream with a slice of the SMs (its GEMMs are tiny and would
    # otherwise serialise behind the HBM-bound routed GEMMs)
    SHARED_SIDE_MAX_ROWS = 8192
    SHARED_SIDE_CTAS = 16

    # decode-size batches: one weight-streaming launch for K3+K4 (+ shared
    # experts), csrc/small_gemm.cu; COX_SMALL_T_MAX overrides the crossover
    SMALL_T_MAX = int(os.environ.get("COX_SMALL_T_MAX", "256"))

    def uses_small_path(self, T: int) -> bool:
        return (0 < T <= self.SMALL_T_MAX and not self.gather_a and self.d % 128 == 0 and self.ff % 128 == 0
                and self.E <= 64 and (not self.shared_ff or self.shared_ff % 128 == 0))

    # prefill layers with shared experts: COX_SHARED_FUSE=1 runs the top-k combine
    # in the shared down projection's epilogue (cox_shared_down_combine, bit-identical).
    # Off by default: measured on C4 the fused epilogue is latency-bound on the k
    # routed-row gathers (shared down + combine 3.51 ms fused vs 1.99 + 1.38 separate)
    SHARED_FUSED_COMBINE = os.environ.get("COX_SHARED_FUSE", "0") == "1"
    # prefill layers with shared experts: shared-expert GEMMs on a side stream
    # beside the permute (COX_SHARED_BESIDE=0: in sequence after the routed experts)
    SHARED_BESIDE_PERMUTE = os.environ.get("COX_SHARED_BESIDE", "1") == "1"

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] != self.d:
            raise ValueError(f"x must be bf16 [T, {self.d}]")
        T = x.shape[0]
        b = self.buffers(T, x.device)
        if self.uses_small_path(T):
            return self._forward_small(x, b, out)
        if self.shared_ff and 0 < T * self.k <= self.SHARED_SIDE_MAX_ROWS:
            main = torch.cuda.current_stream(x.device)
            side = self._side_stream(x.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                ops.grouped_swiglu(x, b.shared_offsets, [0], [self.wts.shared_w13], self.shared_ff, h=b.shared_h,
                                   max_ctas=self.SHARED_SIDE_CTAS)
                ops.grouped_down(b.shared_h, b.shared_offsets, [0], [self.wts.shared_w2], self.d, y=b.shared_y,
                                 max_ctas=self.SHARED_SIDE_CTAS)
            self.route(x, b)
            self._k3(b, self.groups, self.w13_list, max_ctas=-(-(148 - self.SHARED_SIDE_CTAS) // 2) * 2)
            ops.grouped_down(b.h, b.offsets, self.groups, self.w2_list, self.d, y=b.y,
                             max_ctas=-(-(148 - self.SHARED_SIDE_CTAS) // 2) * 2)
            main.wait_stream(side)
            return self.finish(b, b.shared_y, out)
        if self.shared_ff and self.SHARED_BESIDE_PERMUTE and not self.SHARED_FUSED_COMBINE:
            # the shared expert does not depend on the routing: its GEMMs run on a
            # side stream right after the router, so the HBM-bound permute copy
            # (a few registers, no shared memory) co-resides with them on the SMs
            main = torch.cuda.current_stream(x.device)
            side = self._side_stream(x.device)
            ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts))
            side.wait_stream(main)
            with torch.cuda.stream(side):
                sh = self.shared_expert(x, b)
            if self.gather_a:
                ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, None), workspace=b.workspace,
                            copy_rows=False, row_tokens=b.row_tokens)
                b.x_ref = x
            else:
                ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, b.x_perm), workspace=b.workspace)
            self.experts(b)
            main.wait_stream(side)
            return self.finish(b, sh, out)
        self.route(x, b)
        self.experts(b)
        if self.shared_ff and self.SHARED_FUSED_COMBINE and self.k <= 8:
            # shared expert K3, then its down projection with the combine in the epilogue
            ops.grouped_swiglu(x, b.shared_offsets, [0], [self.wts.shared_w13], self.shared_ff, h=b.shared_h)
            return ops.shared_down_combine(b.shared_h, b.shared_offsets, self.wts.shared_w2, b.y, b.dst, b.w,
                                           out=b.out if out is None else out)
        sh = self.shared_expert(x, b)
        return self.finish(b, sh, out)

    # experiment switches for the decode path (A/B): gathered vs materialised
    # routed rows, fused vs separate combine
    SMALL_GATHER = os.environ.get("COX_SMALL_GATHER", "1") == "1"
    SMALL_FUSE = os.environ.get("COX_SMALL_FUSE", "1") == "1"
    # Row gathers (TMA tile::gather4 of x rows) only up to this many tokens:
    # above it the permute materialises x_perm and the kernel loads tiled B
    # boxes.  Measured on C4 (tools/sweep_decode_large.py, us/step, gather vs
    # x_perm): T=64 196.5/196.2, 128 222.0/210.9, 192 270.9/234.8, 256 323.4/262.1.
    SMALL_GATHER_T_MAX = int(os.environ.get("COX_SMALL_GATHER_T_MAX", "64"))

    def _small_gather(self, T: int) -> bool:
        return self.SMALL_GATHER and T <= self.SMALL_GATHER_T_MAX

    def _route_small(self, x: torch.Tensor, b: StageBuffers):
        gather = self._small_gather(x.shape[0])
        ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts))
        ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, None if gather else b.x_perm),
                    workspace=b.workspace, copy_rows=not gather, row_tokens=b.row_tokens)

    def _ffn_small(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor):
        shared = (self.wts.shared_w13, self.wts.shared_w2, b.shared_h, b.shared_y) if self.shared_ff else None
        fuse = out.dtype == torch.bfloat16 and self.SMALL_FUSE
        ops.small_expert_ffn(x, b.offsets, self.groups, self.w13_list, self.w2_list, b.h, b.y,
                             x_perm=None if self._small_gather(x.shape[0]) else b.x_perm, row_tokens=b.row_tokens,
                             shared=shared, combine=(b.dst, b.w, out) if fuse else None)
        if not fuse:
            ops.combine(b.y, b.dst, b.w, b.shared_y if self.shared_ff else None, out=out)
        return out

    # Mid-size decode steps: router + every expert over all tokens + shared
    # experts + combine in ONE launch (cox_decode_moe).  It streams EVERY
    # expert, so it only pays when nearly all are touched anyway, and its token
    # tiles grow with T: measured on C4 (tools/sweep_decode.py, us/step, dense
    # vs routed): T=8 129/129, 16 168/169, 24 188/195, 32 190/199, 48 198/204,
    # 64 205/205.  Used when T <= DENSE_T_MAX and P(expert untouched) =
    # (1 - k/E)^T <= 0.1; COX_DECODE_DENSE=0 disables.
    DENSE_T_MAX = 48 if os.environ.get("COX_DECODE_DENSE", "1") == "1" else 0

    def uses_dense_decode(self, T: int) -> bool:
        return (self.uses_small_path(T) and T <= self.DENSE_T_MAX and (1.0 - self.k / self.E) ** T <= 0.1
                and self.wg_router.dtype == torch.bfloat16 and self.out_dtype == torch.bfloat16)

    def _forward_small(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor | None):
        """Decode-size step: router, index-only permute (no row copy), then ONE
        launch for K3 + K4 + shared experts + combine (csrc/small_gemm.cu).
        At <= 64 tokens the router runs inside that launch too (dense decode)."""
        out = b.out if out is None else out
        T = x.shape[0]
        if self.uses_dense_decode(T):
            dh, dy = self._dense_scratch(T, x.device)
            shared = (self.wts.shared_w13, self.wts.shared_w2, b.shared_h, b.shared_y) if self.shared_ff else None
            return ops.decode_moe(x, self.wg_router, self.k, self.mode, self.w13_list, self.w2_list, dh, dy,
                                  b.idx, b.w, out, shared)
        if self.uses_idx_decode(T, out):
            if self.uses_routed_one_launch(T):
                shared = (self.wts.shared_w13, self.wts.shared_w2, b.shared_h, b.shared_y) if self.shared_ff else None
                return ops.decode_moe_routed(x, self.wg_router, self.k, self.mode, self.w13_list, self.w2_list,
                                             b.h, b.y, b.idx, b.w, b.counts, b.dst, b.offsets, out, shared)
            ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts))
            return self._ffn_idx(x, b, out)
        self._route_small(x, b)
        return self._ffn_small(x, b, out)

    # routed decode without a permute launch: the expert kernel reads the
    # router's idx/counts directly (COX_SMALL_FROM_IDX=0: router + permute + FFN)
    SMALL_FROM_IDX = os.environ.get("COX_SMALL_FROM_IDX", "1") == "1"

    def uses_idx_decode(self, T: int, out: torch.Tensor | None = None) -> bool:
        return (self.SMALL_FROM_IDX and self.uses_small_path(T) and self.tile_m == 1 and self.SMALL_FUSE
                and self._small_gather(T) and (out is None or out.dtype == torch.bfloat16)
                and self.out_dtype == torch.bfloat16)

    # routed decode in ONE launch: the router runs in the expert kernel's
    # prologue (cox_decode_moe_routed), COX_DECODE_ROUTE_IN=1.  Off by default:
    # measured on C4 (tools/sweep_decode.py, profiles/r01/sweep_decode_c4_v2.txt)
    # the in-kernel routing of a token (~10 us on one CTA) is slower than the
    # router kernel + PDL hand-off at small T (T=1: 82 vs 56 us) and within
    # noise at T=64..256; C2D (E=8) gains ~1%
    DECODE_ROUTE_IN = os.environ.get("COX_DECODE_ROUTE_IN", "0") == "1"

    def uses_routed_one_launch(self, T: int) -> bool:
        return (self.DECODE_ROUTE_IN and self.uses_idx_decode(T) and self.wg_router.dtype == torch.bfloat16
                and self.E <= 64 and self.d <= 8192)

    def _ffn_idx(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor):
        shared = (self.wts.shared_w13, self.wts.shared_w2, b.shared_h, b.shared_y) if self.shared_ff else None
        return ops.small_expert_ffn_idx(x, b.idx, b.counts, b.w, self.w13_list, self.w2_list, b.h, b.y, b.dst, out,
                                        offsets=b.offsets, shared=shared)

    def _dense_scratch(self, T: int, dev):
        sc = getattr(self, "_dense", None)
        if sc is None or sc[0].shape[0] != self.E * T:
            sc = (torch.empty((self.E * T, self.ff), dtype=torch.bfloat16, device=dev),
                  torch.empty((self.E * T, self.d), dtype=torch.bfloat16, device=dev))
            self._dense = sc
        return sc

    def _side_stream(self, dev):
        st = getattr(self, "_side", None)
        if st is None:
            st = torch.cuda.Stream(dev)
            self._side = st
        return st

    def capture(self, x_static: torch.Tensor):
        """Capture one forward over `x_static` into a CUDA graph (launch-bound
        small-T steps such as decode).  Returns (replay_fn, out_tensor); refill
        x_static in place and call replay_fn() for each step."""
        self.forward(x_static)  # allocate buffers / tensor maps outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.forward(x_static)
        return g.replay, out

    def forward_microbatched(self, x: torch.Tensor, m_tokens: int) -> torch.Tensor:
        """Ablation (costmodel.expert_stage_time(coalesced=False), planner.py:309-366):
        run the expert stage separately per micro-batch of `m_tokens` tokens, so
        every micro-batch re-reads the expert weights and each expert sees only
        its share of the micro-batch.  Same results; for measuring the cost of
        NOT coalescing."""
        T = x.shape[0]
        out = torch.empty((T, self.d), dtype=self.out_dtype, device=x.device)
        subs = {}
        for s0 in range(0, T, m_tokens):
            xs = x[s0:s0 + m_tokens]
            n = xs.shape[0]
            if n not in subs:
                subs[n] = MoELayer(self.wts, self.k, "mixtral" if self.mode == 0 else "deepseek", self.tile_m,
                                   self.out_dtype, self.gather_a)
            subs[n].forward(xs, out=out[s0:s0 + n])
        return out

    # run_host_batches replays a captured step for batches up to this many tokens (COX_HOST_GRAPH_T_MAX)
    HOST_GRAPH_T_MAX = int(os.environ.get("COX_HOST_GRAPH_T_MAX", "8192"))

    def run_host_batches(self, xs_host, outs_host) -> None:
        """End-to-end serving loop over host batches (pinned memory).

        Batch i's H2D copy (copy engine, own stream) overlaps batch i-1's expert
        stage, and batch i's D2H copy overlaps batch i+1's stage: two device
        input and two device output buffers, event-ordered.  Every batch still
        crosses PCIe both ways; only the waiting is hidden.  Batches of up to
        HOST_GRAPH_T_MAX tokens replay a CUDA graph of the step (one per slot).
        Returns once all work is enqueued; the current stream is ordered after
        the last copy."""
        if len(xs_host) != len(outs_host):
            raise ValueError("one output buffer per input batch")
        if not xs_host:
            return
        dev = self.wts.w13.device
        T = xs_host[0].shape[0]
        comp = torch.cuda.current_stream(dev)
        st = self._host_state(T, dev)
        h2d, d2h, xin, yout = st["h2d"], st["d2h"], st["xin"], st["yout"]
        in_free, out_done = st["in_free"], st["out_done"]
        for i, xh in enumerate(xs_host):
            slot = i % 2
            with torch.cuda.stream(h2d):
                if in_free[slot] is not None:
                    h2d.wait_event(in_free[slot])
                xin[slot].copy_(xh, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(h2d)
            comp.wait_event(ready)
            if out_done[slot] is not None:
                comp.wait_event(out_done[slot])
            if st["graphs"] is not None:
                st["graphs"][slot].replay()
            else:
                self.forward(xin[slot], out=yout[slot])
            ev_c = torch.cuda.Event()
            ev_c.record(comp)
            in_free[slot] = ev_c
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_c)
                outs_host[i].copy_(yout[slot], non_blocking=True)
                ev_o = torch.cuda.Event()
                ev_o.record(d2h)
                out_done[slot] = ev_o
        comp.wait_stream(d2h)

    def _host_state(self, T, dev):
        st = getattr(self, "_hs", None)
        if st is None or st["T"] != T:
            st = {"T": T, "h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                  "xin": [torch.empty((T, self.d), dtype=torch.bfloat16, device=dev) for _ in range(2)],
                  "yout": [torch.empty((T, self.d), dtype=self.out_dtype, device=dev) for _ in range(2)],
                  "in_free": [None, None], "out_done": [None, None], "graphs": None}
            if T <= self.HOST_GRAPH_T_MAX:
                # launch-bound batch sizes: one CUDA graph per (input, output) slot pair
                st["graphs"] = []
                for s in range(2):
                    st["xin"][s].zero_()
                    self.forward(st["xin"][s], out=st["yout"][s])  # buffers / tensor maps outside capture
                    torch.cuda.synchronize(dev)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        self.forward(st["xin"][s], out=st["yout"][s])
                    st["graphs"].append(g)
            self._hs = st
        return st

    __call__ = forward

    def stage_times(self, x: torch.Tensor | None = None) -> dict:
        """One instrumented step (CUDA events between stages), in ms."""
        b = self._bufs
        if x is None:
            raise ValueError("stage_times needs the step's input")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        if self.uses_dense_decode(x.shape[0]) or self.uses_routed_one_launch(x.shape[0]):
            ev[0].record()
            self._forward_small(x, b, b.out)
            ev[1].record()
            torch.cuda.synchronize()
            name = "decode_moe_one_launch" if self.uses_dense_decode(x.shape[0]) else "decode_moe_routed_one_launch"
            return {name: ev[0].elapsed_time(ev[1])}
        ev[0].record()
        ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts))
        ev[1].record()
        if self.uses_idx_decode(x.shape[0]):
            self._ffn_idx(x, b, b.out)
            ev[2].record()
            torch.cuda.synchronize()
            return {"router": ev[0].elapsed_time(ev[1]), "expert_ffn_from_idx_shared_combine": ev[1].elapsed_time(ev[2])}
        if self.uses_small_path(x.shape[0]):
            gather = self._small_gather(x.shape[0])
            ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, None if gather else b.x_perm),
                        workspace=b.workspace, copy_rows=not gather, row_tokens=b.row_tokens)
        elif self.gather_a:
            ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, None), workspace=b.workspace,
                        copy_rows=False, row_tokens=b.row_tokens)
            b.x_ref = x
        else:
            ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, b.x_perm), workspace=b.workspace)
        ev[2].record()
        if self.uses_small_path(x.shape[0]):
            self._ffn_small(x, b, b.out)
            ev[3].record()
            torch.cuda.synchronize()
            names = ["router", "permute", "expert_ffn_k3k4_shared_combine"]
            return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}
        self._k3(b, self.groups, self.w13_list)
        ev[3].record()
        ops.grouped_down(b.h, b.offsets, self.groups, self.w2_list, self.d, y=b.y)
        ev[4].record()
        if self.shared_ff and self.SHARED_FUSED_COMBINE and self.k <= 8:
            ops.grouped_swiglu(x, b.shared_offsets, [0], [self.wts.shared_w13], self.shared_ff, h=b.shared_h)
            ev[5].record()
            ops.shared_down_combine(b.shared_h, b.shared_offsets, self.wts.shared_w2, b.y, b.dst, b.w, out=b.out)
            ev[6].record()
            torch.cuda.synchronize()
            names = ["router", "permute", "swiglu_k3", "down_k4", "shared_k3", "shared_down_with_combine"]
            return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}
        sh = self.shared_expert(x, b)
        ev[5].record()
        ops.combine(b.y, b.dst, b.w, sh, out=b.out)
        ev[6].record()
        torch.cuda.synchronize()
        names = ["router", "permute", "swiglu_k3", "down_k4", "shared", "combine"]
        return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}
