"""The coalesced MoE expert stage on one B200: router -> permute -> grouped
SwiGLU -> grouped down -> combine, all in libcoxmoe.so.

``MoELayer.forward`` is the single-GPU, all-resident path (the reference's
``AllocationStrategy(exp_r=E, exp_m=0, exp_c=0)``).  Residency/streaming and
expert parallelism build on the same stage functions (executor.py, ep.py).

Kernel selection by batch size (all measured on B200):
  * T <= DENSE_T_MAX (48) and nearly every expert touched: ONE launch
    (cox_decode_moe: router + every expert + shared experts + combine);
  * T <= SMALL_GATHER_T_MAX (64): router launch + one weight-streaming launch
    that reads the router's idx directly (cox_small_expert_ffn_idx);
  * T <= SMALL_T_MAX (256) and T*k <= 32 E: router + permute (x_perm
    materialised) + one weight-streaming launch (cox_small_expert_ffn);
  * larger batches: router, permute, K3, K4, combine (persistent tcgen05
    grouped GEMMs), shared experts on a side stream.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib, ops
from .hostio import HostIO, run_host_batches
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
    workspace: torch.Tensor          # permute workspace
    router_ws: torch.Tensor          # router workspace (zero-initialised)
    row_tokens: torch.Tensor | None = None  # small path: source token of every permuted row
    shared_offsets: torch.Tensor | None = None
    shared_h: torch.Tensor | None = None
    shared_y: torch.Tensor | None = None
    dense_h: torch.Tensor | None = None     # dense decode scratch [E*T, ff] / [E*T, d]
    dense_y: torch.Tensor | None = None


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
        x_perm=torch.empty((0 if gather_a else cap, d), dtype=bf, device=device),
        h=torch.empty((cap, ff), dtype=bf, device=device),
        y=torch.empty((cap, d), dtype=bf, device=device),
        out=torch.empty((T, d), dtype=out_dtype, device=device),
        workspace=torch.empty((max(16, ops.permute_workspace_bytes(T, E)),), dtype=torch.uint8, device=device),
        router_ws=ops.router_workspace(T, E, device),
    )
    if gather_a:
        b.row_tokens = torch.empty((cap,), dtype=torch.int32, device=device)
    if shared_ff:
        b.shared_offsets = torch.tensor([0, T], dtype=torch.int32, device=device)
        b.shared_h = torch.empty((max(T, 1), shared_ff), dtype=bf, device=device)
        b.shared_y = torch.empty((max(T, 1), d), dtype=bf, device=device)
    return b


class MoELayer:
    """One MoE layer's expert stage with every expert resident in HBM.

    Buffers are kept per batch size.  A CUDA graph captured over a buffer set
    (``capture``, ``run_host_batches``) PINS that set: it is never freed or
    reallocated while the layer lives, so a later forward at another batch
    size cannot hand the graph's memory to other tensors.  Unpinned sets are
    dropped when a new batch size is allocated (one live working set)."""

    # decode-size batches: one weight-streaming launch for K3+K4 (+ shared
    # experts), csrc/small_gemm.cu
    SMALL_T_MAX = 256
    # ... and while an expert averages at most this many rows (the kernel runs
    # segments in 64-token chunks and re-reads them per 128 weight rows).
    # Measured with tools/sweep_tokens.py paths (graph replay, us,
    # weight-streaming vs prefill kernels with their M = 128 pair tiles):
    # C2 (E=8, k=2) T=128 (32 rows) 495 vs 530, T=192 (48 rows) 660 vs 534;
    # C4 (E=64, k=6) T=192 (18 rows) 235 vs 256, T=256 (24 rows) 265 vs 258.
    SMALL_ROWS_PER_EXPERT_MAX = 32
    # Row gathers (TMA tile::gather4 of x rows) only up to this many tokens:
    # above it the permute materialises x_perm and the kernel loads tiled B
    # boxes.  Measured on C4 (tools/sweep_decode_large.py, us/step, gather vs
    # x_perm): T=64 196.5/196.2, 128 222.0/210.9, 192 270.9/234.8, 256 323.4/262.1.
    SMALL_GATHER_T_MAX = 64
    # Mid-size decode steps: router + every expert over all tokens + shared
    # experts + combine in ONE launch (cox_decode_moe).  It streams EVERY
    # expert, so it only pays when nearly all are touched anyway: measured on
    # C4 (tools/sweep_decode.py, us/step, dense vs routed): T=8 129/129, 16
    # 168/169, 24 188/195, 32 190/199, 48 198/204, 64 205/205.  Used when
    # T <= DENSE_T_MAX and P(expert untouched) = (1 - k/E)^T <= 0.1.
    DENSE_T_MAX = 48
    # decode-size batches with shared experts: the shared expert runs beside
    # the routed experts on a side stream with a slice of the SMs
    SHARED_SIDE_MAX_ROWS = 8192
    SHARED_SIDE_CTAS = 16
    # run_host_batches replays a captured step for batches up to this many tokens
    HOST_GRAPH_T_MAX = 8192
    # prefill K3 reading its A rows from x by cp.async gathers (no x_perm copy,
    # saves the T*k*d*2-byte x_perm buffer): bit-identical, measured within
    # 1-2% of (not faster than) the x_perm path on B200 (C4 30.1-30.7 vs
    # 29.9-30.0 ms, C2 137.6-138.1 vs 134.0-135.4 ms per step), so opt-in;
    # DESIGN.md §4 "Gather-fused A loads"
    GATHER_A_DEFAULT = False

    def __init__(self, weights: LayerWeights, top_k: int, mode: str = "mixtral", tile_m: int = 1,
                 out_dtype=torch.bfloat16, gather_a: bool | None = None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")
        self.wts = weights
        self.k = int(top_k)
        self.mode_name = mode
        self.mode = MODES[mode]
        self.tile_m = int(tile_m)
        self.out_dtype = out_dtype
        # prefill K3 gathers its A rows from x (cp.async) instead of a
        # materialised x_perm: the permute writes indices only
        self.gather_a = self.GATHER_A_DEFAULT if gather_a is None else bool(gather_a)
        if self.gather_a and self.tile_m != 1:
            raise ValueError("gather_a needs tile_m == 1")
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
        self._bufs: dict[int, StageBuffers] = {}
        self._pinned: set[int] = set()
        self._hs: dict[int, dict] = {}
        self._side = None
        self.profile_events = None  # optional {"k3": (ev0, ev1), "k4": (ev0, ev1)} recorded around K3/K4

    def launches_per_step(self, T: int | None = None) -> int:
        if T is not None and self.uses_dense_decode(T):
            return 1  # router + all experts + shared + combine in one launch
        if T is not None and self.uses_idx_decode(T):
            return 2  # router, then one launch for K3/K4/shared/combine reading the router's idx
        # permute: single-CTA index kernel for T*k <= 2048 (else hist, scan, scatter) + row copy (+ pad)
        small_perm = T is not None and T * self.k <= 2048
        perm = (1 if small_perm else 3) + 1 + (1 if self.tile_m > 1 else 0)
        if T is not None and self.uses_small_path(T):
            # router + permute (rows materialised) + one launch for K3/K4/shared/combine
            return 1 + perm + 1 + (1 if self.out_dtype != torch.bfloat16 else 0)
        # prefill: the gather path drops the permute's row copy
        return 1 + perm - (1 if self.gather_a else 0) + 2 + 1 + (2 if self.shared_ff else 0)

    # --- buffers ---------------------------------------------------------------
    def buffers(self, T: int, device) -> StageBuffers:
        b = self._bufs.get(T)
        if b is None:
            for t in [t for t in self._bufs if t not in self._pinned]:
                del self._bufs[t]
            gather = self.gather_a and not self.uses_small_path(T)
            b = alloc_buffers(T, self.d, self.ff, self.E, self.k, self.tile_m, device, self.out_dtype,
                              self.shared_ff, gather_a=gather)
            if self.uses_small_path(T):
                b.row_tokens = torch.empty((b.h.shape[0],), dtype=torch.int32, device=device)
            if self.uses_dense_decode(T):
                b.dense_h = torch.empty((self.E * T, self.ff), dtype=torch.bfloat16, device=device)
                b.dense_y = torch.empty((self.E * T, self.d), dtype=torch.bfloat16, device=device)
            self._bufs[T] = b
        return b

    def pin(self, T: int) -> None:
        """Keep the buffer set of batch size T for the life of the layer (graphs reference it)."""
        self._pinned.add(T)

    # --- stages (all stream-ordered on the current stream) -------------------
    def _router(self, x: torch.Tensor, b: StageBuffers):
        ops.router_topk(x, self.wg_router, self.k, self.mode, out=(b.idx, b.w, b.counts), workspace=b.router_ws)

    def route(self, x: torch.Tensor, b: StageBuffers):
        self._router(x, b)
        self._permute(x, b)

    def _gathers(self, b: StageBuffers) -> bool:
        return b.x_perm.shape[0] == 0  # prefill buffers of a gather_a layer

    def _permute(self, x: torch.Tensor, b: StageBuffers):
        ops.permute(b.idx, x, self.E, self.tile_m, out=(b.offsets, b.dst, b.x_perm), workspace=b.workspace,
                    row_tokens=b.row_tokens, copy_rows=not self._gathers(b))
        self._x = x  # the gather K3 reads the permuted rows straight from the step's input

    def _swiglu(self, b: StageBuffers, groups, w13, max_ctas: int = 0):
        if self._gathers(b):
            ops.grouped_swiglu_gather(self._x, b.row_tokens, b.offsets, groups, w13, self.ff, b.h, max_ctas=max_ctas)
        else:
            ops.grouped_swiglu(b.x_perm, b.offsets, groups, w13, self.ff, h=b.h, max_ctas=max_ctas)

    def experts(self, b: StageBuffers, groups=None, w13=None, w2=None):
        groups = self.groups if groups is None else groups
        pe = self.profile_events
        if pe:
            pe["k3"][0].record()
        self._swiglu(b, groups, self.w13_list if w13 is None else w13)
        if pe:
            pe["k3"][1].record()
            pe["k4"][0].record()
        ops.grouped_down(b.h, b.offsets, groups, self.w2_list if w2 is None else w2, self.d, y=b.y)
        if pe:
            pe["k4"][1].record()

    def shared_expert(self, x: torch.Tensor, b: StageBuffers, max_ctas: int = 0):
        if not self.shared_ff:
            return None
        ops.grouped_swiglu(x, b.shared_offsets, [0], [self.wts.shared_w13], self.shared_ff, h=b.shared_h,
                           max_ctas=max_ctas)
        ops.grouped_down(b.shared_h, b.shared_offsets, [0], [self.wts.shared_w2], self.d, y=b.shared_y,
                         max_ctas=max_ctas)
        return b.shared_y

    def finish(self, b: StageBuffers, shared=None, out=None):
        return ops.combine(b.y, b.dst, b.w, shared, out=b.out if out is None else out)

    def uses_small_path(self, T: int) -> bool:
        return (0 < T <= self.SMALL_T_MAX and T * self.k <= self.SMALL_ROWS_PER_EXPERT_MAX * self.E
                and self.d % 128 == 0 and self.ff % 128 == 0 and self.E <= 64
                and (not self.shared_ff or self.shared_ff % 128 == 0))

    def uses_dense_decode(self, T: int) -> bool:
        return (self.uses_small_path(T) and T <= self.DENSE_T_MAX and (1.0 - self.k / self.E) ** T <= 0.1
                and self.wg_router.dtype == torch.bfloat16 and self.out_dtype == torch.bfloat16)

    def uses_idx_decode(self, T: int, out: torch.Tensor | None = None) -> bool:
        """Routed decode without a permute launch: the expert kernel reads the router's idx/counts."""
        return (self.uses_small_path(T) and self.tile_m == 1 and T <= self.SMALL_GATHER_T_MAX
                and (out is None or out.dtype == torch.bfloat16) and self.out_dtype == torch.bfloat16)

    def _side_stream(self, dev):
        if self._side is None:
            self._side = torch.cuda.Stream(dev)
        return self._side

    # --- forward ---------------------------------------------------------------
    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] != self.d:
            raise ValueError(f"x must be bf16 [T, {self.d}]")
        T = x.shape[0]
        b = self.buffers(T, x.device)
        if self.uses_small_path(T):
            return self._forward_small(x, b, out)
        if self.shared_ff and 0 < T * self.k <= self.SHARED_SIDE_MAX_ROWS:
            # small prefill batches: the shared expert on a side stream with a slice of the SMs
            main = torch.cuda.current_stream(x.device)
            side = self._side_stream(x.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.shared_expert(x, b, max_ctas=self.SHARED_SIDE_CTAS)
            self.route(x, b)
            rest = -(-(148 - self.SHARED_SIDE_CTAS) // 2) * 2
            self._swiglu(b, self.groups, self.w13_list, max_ctas=rest)
            ops.grouped_down(b.h, b.offsets, self.groups, self.w2_list, self.d, y=b.y, max_ctas=rest)
            main.wait_stream(side)
            return self.finish(b, b.shared_y, out)
        if self.shared_ff:
            # the shared expert does not depend on the routing: its GEMMs run on a
            # side stream right after the router, so the HBM-bound permute copy
            # (a few registers, no shared memory) co-resides with them on the SMs
            # (C4: +0.5%)
            main = torch.cuda.current_stream(x.device)
            side = self._side_stream(x.device)
            self._router(x, b)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                sh = self.shared_expert(x, b)
            self._permute(x, b)
            self.experts(b)
            main.wait_stream(side)
            return self.finish(b, sh, out)
        self.route(x, b)
        self.experts(b)
        return self.finish(b, None, out)

    __call__ = forward

    def _shared_args(self, b: StageBuffers):
        return (self.wts.shared_w13, self.wts.shared_w2, b.shared_h, b.shared_y) if self.shared_ff else None

    def _forward_small(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor | None):
        """Decode-size step: see the module docstring for the selection."""
        out = b.out if out is None else out
        T = x.shape[0]
        if self.uses_dense_decode(T):
            return ops.decode_moe(x, self.wg_router, self.k, self.mode, self.w13_list, self.w2_list, b.dense_h,
                                  b.dense_y, b.idx, b.w, out, self._shared_args(b))
        self._router(x, b)
        if self.uses_idx_decode(T, out):
            return self._ffn_idx(x, b, out)
        self._permute(x, b)
        return self._ffn_small(x, b, out)

    def _ffn_small(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor):
        fuse = out.dtype == torch.bfloat16
        ops.small_expert_ffn(x, b.offsets, self.groups, self.w13_list, self.w2_list, b.h, b.y, x_perm=b.x_perm,
                             shared=self._shared_args(b), combine=(b.dst, b.w, out) if fuse else None)
        if not fuse:
            ops.combine(b.y, b.dst, b.w, b.shared_y if self.shared_ff else None, out=out)
        return out

    def _ffn_idx(self, x: torch.Tensor, b: StageBuffers, out: torch.Tensor):
        return ops.small_expert_ffn_idx(x, b.idx, b.counts, b.w, self.w13_list, self.w2_list, b.h, b.y, b.dst, out,
                                        offsets=b.offsets, shared=self._shared_args(b))

    # --- CUDA graphs and host batches -------------------------------------------
    def capture(self, x_static: torch.Tensor):
        """Capture one forward over `x_static` into a CUDA graph (launch-bound
        small-T steps such as decode).  Returns (replay_fn, out_tensor); refill
        x_static in place and call replay_fn() for each step.  The batch size's
        buffers are pinned for the life of the layer."""
        T = x_static.shape[0]
        self.pin(T)
        self.forward(x_static)  # allocate buffers / tensor maps outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.forward(x_static)
        keep = (g, x_static, self._bufs[T])

        def replay():
            keep[0].replay()
        return replay, out

    def forward_microbatched(self, x: torch.Tensor, m_tokens: int) -> torch.Tensor:
        """Ablation (costmodel.expert_stage_time(coalesced=False), planner.py:309-366):
        run the expert stage separately per micro-batch of `m_tokens` tokens, so
        every micro-batch re-reads the expert weights and each expert sees only
        its share of the micro-batch.  Same results; for measuring the cost of
        NOT coalescing."""
        T = x.shape[0]
        out = torch.empty((T, self.d), dtype=self.out_dtype, device=x.device)
        subs = getattr(self, "_mb_layers", None)
        if subs is None:
            subs = self._mb_layers = {}
        for s0 in range(0, T, m_tokens):
            xs = x[s0:s0 + m_tokens]
            n = xs.shape[0]
            if n not in subs:
                subs[n] = MoELayer(self.wts, self.k, self.mode_name, self.tile_m, self.out_dtype, self.gather_a)
            subs[n].forward(xs, out=out[s0:s0 + n])
        return out

    def run_host_batches(self, xs_host, outs_host) -> None:
        """End-to-end serving loop over host batches (pinned memory), see
        hostio.run_host_batches.  Batches of up to HOST_GRAPH_T_MAX tokens replay
        a CUDA graph of the step (one per slot; the batch size's buffers are
        pinned)."""
        if not xs_host:
            return
        dev = self.wts.w13.device
        T = xs_host[0].shape[0]
        st = self._host_state(T, dev)
        run_host_batches(st["io"], xs_host, outs_host,
                         (lambda slot: st["graphs"][slot].replay()) if st["graphs"] is not None
                         else (lambda slot: self.forward(st["io"].xin[slot], out=st["io"].yout[slot])))

    def _host_state(self, T, dev):
        st = self._hs.get(T)
        if st is None:
            io = HostIO(T, self.d, dev, out_dtype=self.out_dtype)
            st = {"io": io, "graphs": None}
            if T <= self.HOST_GRAPH_T_MAX:
                # launch-bound batch sizes: one CUDA graph per (input, output) slot pair; the
                # graphs reference this T's stage buffers, which are pinned from here on
                self.pin(T)
                st["graphs"] = []
                for s in range(2):
                    io.xin[s].zero_()
                    self.forward(io.xin[s], out=io.yout[s])  # buffers / tensor maps outside capture
                    torch.cuda.synchronize(dev)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        self.forward(io.xin[s], out=io.yout[s])
                    st["graphs"].append(g)
                st["bufs"] = self._bufs[T]
            self._hs[T] = st
        return st

    def stage_times(self, x: torch.Tensor | None = None) -> dict:
        """One instrumented step (CUDA events between stages), in ms."""
        if x is None:
            raise ValueError("stage_times needs the step's input")
        T = x.shape[0]
        b = self.buffers(T, x.device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]

        def span(names, n):
            torch.cuda.synchronize()
            return {nm: ev[i].elapsed_time(ev[i + 1]) for i, nm in enumerate(names[:n])}

        if self.uses_dense_decode(T):
            ev[0].record()
            self._forward_small(x, b, b.out)
            ev[1].record()
            return span(["decode_moe_one_launch"], 1)
        ev[0].record()
        self._router(x, b)
        ev[1].record()
        if self.uses_idx_decode(T):
            self._ffn_idx(x, b, b.out)
            ev[2].record()
            return span(["router", "expert_ffn_from_idx_shared_combine"], 2)
        self._permute(x, b)
        ev[2].record()
        if self.uses_small_path(T):
            self._ffn_small(x, b, b.out)
            ev[3].record()
            return span(["router", "permute", "expert_ffn_k3k4_shared_combine"], 3)
        self._swiglu(b, self.groups, self.w13_list)
        ev[3].record()
        ops.grouped_down(b.h, b.offsets, self.groups, self.w2_list, self.d, y=b.y)
        ev[4].record()
        sh = self.shared_expert(x, b)
        ev[5].record()
        ops.combine(b.y, b.dst, b.w, sh, out=b.out)
        ev[6].record()
        return span(["router", "permute", "swiglu_k3", "down_k4", "shared", "combine"], 6)
