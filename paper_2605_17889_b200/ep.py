"""Expert parallelism across the GPUs of one box.

One process per GPU.  Rank r owns experts [r*E/G, (r+1)*E/G) and its own
batch of tokens (weak scaling: every rank routes its own ordinary batch, the
coalesced per-expert batch on the owner is the union over all ranks).

Per layer, on every rank (stream-ordered, CUDA kernels from libcoxmoe.so):
  1. K1 route + K2 permute the local tokens by GLOBAL expert id — with
     tile_m=1 the permuted rows are destination-rank-major, so they are the
     all-to-all send buffer as is;
  2. counts exchange: all_to_all of the E/G per-expert counts (one small
     device->host read per layer to size the payload exchange);
  3. dispatch: all_to_all_single (NCCL over NVLink/NVSwitch) of token rows;
     the receive buffer holds, per source rank, that source's rows for each
     local expert — every (source, expert) segment becomes one group of the
     grouped GEMM (same weights, own row range), so no re-permute pass;
  4. K3/K4 grouped expert GEMMs on the received rows;
  5. combine: the reverse all_to_all_single returns y rows to their source;
  6. K5 weighted combine on the home rank.
Order contract: a source's rows arrive in that source's (expert, token)
order, so the per-expert row order on the owner is (source rank, token) —
the global token order when tokens are sharded contiguously — and results
are bit-identical to a single-rank run (tests/test_ep.py checks this with
the gloo backend and the CPU oracle standing in for the kernels).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops
from .hostio import HostIO, run_host_batches
from .layer import MODES
from .synthetic import LayerWeights


class _HostBatches:
    """run_host_batches for the EP layers: the same pipelined H2D / D2H copies
    as MoELayer (hostio.py), one pipeline per rank; every rank feeds its own
    host batches (weak scaling)."""

    def run_host_batches(self, xs_host, outs_host) -> None:
        if not xs_host:
            return
        T = xs_host[0].shape[0]
        io = getattr(self, "_hostio", None)
        if io is None or io.T != T:
            io = self._hostio = HostIO(T, self.d, self._device())
        run_host_batches(io, xs_host, outs_host, lambda slot: self.forward(io.xin[slot], out=io.yout[slot]))


class CudaStage:
    """The per-rank compute of the EP layer, on libcoxmoe.so kernels."""

    def __init__(self, weights: LayerWeights, k: int, mode: int, local_experts: range):
        self.w = weights
        self.k = k
        self.mode = mode
        self.E = weights.num_experts
        self.d = weights.hidden_dim
        self.ff = weights.expert_dim
        self.local = list(local_experts)
        self.w13 = [weights.w13[e] for e in self.local]
        self.w2 = [weights.w2[e] for e in self.local]
        self._ws = None
        self._rws = None
        self._h = None
        self.profile_events = None

    def route_and_permute(self, x):
        T = x.shape[0]
        if self._rws is None or self._rws.numel() < ops.router_workspace_bytes(T, self.E):
            self._rws = ops.router_workspace(T, self.E, x.device)
        idx, w, counts = ops.router_topk(x, self.w.wg, self.k, self.mode, workspace=self._rws)
        if self._ws is None or self._ws.numel() < ops.permute_workspace_bytes(T, self.E):
            self._ws = torch.empty((max(16, ops.permute_workspace_bytes(T, self.E)),), dtype=torch.uint8,
                                   device=x.device)
        offsets, dst, x_perm = ops.permute(idx, x, self.E, 1, workspace=self._ws)
        return idx, w, counts, dst, x_perm

    def experts(self, rows, seg_offsets, n_src, out=None):
        L = len(self.local)
        groups = list(range(n_src * L))
        w13 = [self.w13[g % L] for g in groups]
        w2 = [self.w2[g % L] for g in groups]
        n = rows.shape[0]
        if self._h is None or self._h.shape[0] < n:
            self._h = torch.empty((max(n, 1), self.ff), dtype=torch.bfloat16, device=rows.device)
        h = self._h[: max(n, 1)]
        pe = self.profile_events
        if pe:
            pe["k3"][0].record()
        ops.grouped_swiglu(rows, seg_offsets, groups, w13, self.ff, h=h)
        if pe:
            pe["k3"][1].record()
            pe["k4"][0].record()
        y = ops.grouped_down(h, seg_offsets, groups, w2, self.d, y=out)
        if pe:
            pe["k4"][1].record()
        return y

    def combine(self, y_back, dst, w, out=None):
        return ops.combine(y_back, dst, w, out=out)

    def empty_rows(self, n, like):
        return torch.empty((max(n, 1), self.d), dtype=like.dtype, device=like.device)


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_rows, in_rows, group):
    """Row all-to-all; rows are moved as int32 words (bf16/fp32 payloads alike).

    NCCL moves device rows directly over NVLink/NVSwitch.  Under gloo (CPU
    tests, or several ranks sharing one GPU in tests) device rows are staged
    through host memory."""
    w = inp.shape[1] * inp.element_size() // 4
    o = out.view(torch.int32).view(-1, w)
    i = inp.view(torch.int32).view(-1, w)
    oc = [int(v) for v in out_rows]
    ic = [int(v) for v in in_rows]
    if o.is_cuda and dist.get_backend(group) != "nccl":
        oh = torch.empty(o.shape, dtype=o.dtype)
        dist.all_to_all_single(oh, i.cpu(), oc, ic, group=group)
        o.copy_(oh)
    else:
        dist.all_to_all_single(o, i, oc, ic, group=group)


class EPMoELayer(_HostBatches):
    """MoE expert stage with experts sharded over the ranks of `group`."""

    def __init__(self, weights: LayerWeights, top_k: int, mode: str = "mixtral", group=None, stage=None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")
        self.group = group if group is not None else dist.group.WORLD
        self.G = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.E = weights.num_experts if hasattr(weights, "num_experts") else weights["E"]
        if self.E % self.G:
            raise ValueError(f"{self.E} experts cannot be sharded evenly over {self.G} ranks")
        self.L = self.E // self.G
        if self.G * self.L > 64:
            raise ValueError("at most 64 (source, expert) groups per grouped GEMM")
        self.k = int(top_k)
        self.d = weights.hidden_dim if hasattr(weights, "hidden_dim") else None
        self._wdev = weights.w13.device if hasattr(weights, "w13") else None
        local = range(self.rank * self.L, (self.rank + 1) * self.L)
        self.stage = stage if stage is not None else CudaStage(weights, self.k, MODES[mode], local)
        self._recv = None
        self._yrecv = None
        self._yback = None
        self.last_split = None
        self.profile_events = None

    @property
    def launches_per_step(self) -> int:
        return 1 + 4 + 2 + 1

    def _buf(self, name, n, like):
        b = getattr(self, name)
        if b is None or b.shape[0] < max(n, 1) or b.dtype != like.dtype:
            b = self.stage.empty_rows(n, like)
            setattr(self, name, b)
        return b[:n]

    def _device(self):
        return self._wdev

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        G, L, k = self.G, self.L, self.k
        T = x.shape[0]
        idx, w, counts, dst, x_perm = self.stage.route_and_permute(x)
        # counts exchange: counts[e] for e owned by rank q go to rank q
        recv_counts = torch.empty_like(counts)
        if counts.is_cuda and dist.get_backend(self.group) != "nccl":
            rc = torch.empty(counts.shape, dtype=counts.dtype)
            dist.all_to_all_single(rc, counts.cpu(), group=self.group)
            recv_counts.copy_(rc)
        else:
            dist.all_to_all_single(recv_counts, counts, group=self.group)
        self.stage.profile_events = self.profile_events
        both = torch.cat([counts, recv_counts]).cpu()  # the one host sync per layer
        send_seg = both[: self.E].view(G, L)
        recv_seg = both[self.E:].view(G, L)  # [source rank, local expert]
        send_rows = send_seg.sum(1).tolist()
        recv_rows = recv_seg.sum(1).tolist()
        n_recv = int(sum(recv_rows))
        seg = torch.zeros(G * L + 1, dtype=torch.int32)
        seg[1:] = torch.cumsum(recv_seg.reshape(-1), 0)
        seg_offsets = seg.to(x.device, non_blocking=True)
        self.last_split = (send_rows, recv_rows)

        recv = self._buf("_recv", n_recv, x_perm)
        _a2a(recv, x_perm[: T * k], recv_rows, send_rows, self.group)
        yrecv = self._buf("_yrecv", n_recv, x_perm)
        y = self.stage.experts(recv, seg_offsets, G, out=yrecv) if n_recv else yrecv
        yback = self._buf("_yback", T * k, x_perm)
        _a2a(yback, y[:n_recv], send_rows, recv_rows, self.group)
        return self.stage.combine(yback, dst, w, out=out) if out is not None else self.stage.combine(yback, dst, w)

    __call__ = forward


class SymmMemTransport:
    """Peer-mapped buffers from CUDA symmetric memory + its stream-ordered barrier."""

    def __init__(self, group):
        self.group = group
        self.hdl = None

    def alloc(self, spec: dict, dev) -> dict:
        """spec: name -> (shape, dtype); returns name -> (local tensor, device int64 [world] peer addresses)."""
        import torch.distributed._symmetric_memory as symm
        out = {}
        for name, (shape, dtype) in spec.items():
            t = symm.empty(shape, dtype=dtype, device=dev)
            h = symm.rendezvous(t, self.group)
            if self.hdl is None:
                self.hdl = h
            out[name] = (t, torch.tensor(list(h.buffer_ptrs), dtype=torch.int64, device=dev))
        return out

    def barrier(self) -> None:
        self.hdl.barrier(channel=0, timeout_ms=120000)


class FusedEPMoELayer(_HostBatches):
    """EP expert stage with dispatch/combine fused into kernels that store/load
    token rows directly in the peers' memory (csrc/ep.cu) — no NCCL
    all-to-all, no x_perm/y_back round trip through local HBM.

    Buffers are CUDA symmetric memory (torch.distributed._symmetric_memory):
    every rank maps every peer's receive buffer, output buffer and count
    matrix; the symmetric-memory barrier (stream-ordered, system-scope
    release/acquire on signal pads) separates the phases:
        K1 route -> K2 ranks -> counts put -> barrier -> offsets [-> capacity
        check] -> dispatch -> barrier -> K3/K4 on received rows (one group per
        local expert) -> barrier -> fused combine.
    The next layer's counts put is ordered after this combine on every rank,
    so buffers are never overwritten while a peer still reads them.

    Receive capacity.  The receive buffers hold `cap` rows (capacity_factor x
    T*k + 256).  The offsets kernel reports the largest receive count of any
    owner when it exceeds `cap`; every rank holds the same count matrix, so
    every rank reaches the same verdict.  With check_capacity=True (default)
    each layer reads that verdict back (one 4-byte D2H read after the offsets
    kernel) and, on overflow, all ranks grow their receive buffers to fit
    (a collective symmetric-memory allocation, identical on every rank) and
    redo the offsets — results stay exact for any routing skew.  With
    check_capacity=False nothing waits on the host: overflowing rows are
    dropped by the kernels (never written or read out of bounds) and
    `check()` raises afterwards.
    """

    def __init__(self, weights: LayerWeights, top_k: int, mode: str = "mixtral", group=None,
                 capacity_factor: float = 1.25, transport=None, check_capacity: bool = True):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")
        self.group = group if group is not None else dist.group.WORLD
        self.transport = transport if transport is not None else SymmMemTransport(self.group)
        self.G = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.E = weights.num_experts
        if self.E % self.G:
            raise ValueError(f"{self.E} experts cannot be sharded evenly over {self.G} ranks")
        self.L = self.E // self.G
        if self.L > 64:
            raise ValueError("at most 64 local experts per grouped GEMM")
        self.k = int(top_k)
        self.mode = MODES[mode]
        self.w = weights
        self.d = weights.hidden_dim
        self.ff = weights.expert_dim
        local = range(self.rank * self.L, (self.rank + 1) * self.L)
        self.w13 = [weights.w13[e] for e in local]
        self.w2 = [weights.w2[e] for e in local]
        self.cap_factor = float(capacity_factor)
        self.check_capacity = bool(check_capacity)
        self.regrows = 0
        self._T = None
        self._flag_host = None
        self.profile_events = None

    @property
    def launches_per_step(self) -> int:
        # ours: router, permute ranks x3, counts put, offsets, dispatch, K3, K4, combine (+3 symm-mem barriers, not ours)
        return 1 + 3 + 1 + 1 + 1 + 2 + 1

    def _alloc_rows(self, cap: int, dev):
        bufs = self.transport.alloc({"recv": ((cap, self.d), torch.bfloat16), "y": ((cap, self.d), torch.bfloat16)},
                                    dev)
        (self.recv, self.peer_recv), (self.ysym, self.peer_y) = bufs["recv"], bufs["y"]
        self.h = torch.empty((cap, self.ff), dtype=torch.bfloat16, device=dev)
        self.cap = cap

    def _setup(self, T: int, dev):
        G, E, k, d = self.G, self.E, self.k, self.d
        (self.counts_all, self.peer_counts), = self.transport.alloc({"counts": ((G, E), torch.int32)}, dev).values()
        self._alloc_rows(int(T * k * self.cap_factor) + 256, dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.idx = torch.empty((T, k), **i32)
        self.wts = torch.empty((T, k), dtype=torch.float32, device=dev)
        self.counts = torch.empty((E,), **i32)
        self.offsets = torch.empty((E + 1,), **i32)
        self.dst = torch.empty((T, k), **i32)
        self.route_row = torch.empty((T, k), **i32)
        self.recv_seg = torch.empty((self.L + 1,), **i32)
        self.send_base = torch.empty((E,), **i32)
        self.overflow = torch.zeros((1,), **i32)
        self._flag_host = torch.zeros((1,), dtype=torch.int32, pin_memory=True)
        self.ws = torch.empty((max(16, ops.permute_workspace_bytes(T, E)),), dtype=torch.uint8, device=dev)
        self.rws = ops.router_workspace(T, E, dev)
        self.out = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
        self._T = T

    def _barrier(self):
        self.transport.barrier()

    def _offsets(self):
        ops.ep_offsets(self.counts_all, self.rank, self.cap, self.recv_seg, self.send_base, self.overflow)
        if not self.check_capacity:
            return
        self._flag_host.copy_(self.overflow, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        need = int(self._flag_host.item())
        if need:
            # identical on every rank (same count matrix): grow collectively, redo the offsets
            self.regrows += 1
            self._alloc_rows(int(need * 1.125) + 256, self.recv.device)
            ops.ep_offsets(self.counts_all, self.rank, self.cap, self.recv_seg, self.send_base, self.overflow)

    def _device(self):
        return self.w.w13.device

    # stage names of stage_times(), in order (one CUDA event after each)
    STAGES = ("router_permute", "counts_exchange_offsets", "dispatch_nvlink", "swiglu_k3", "down_k4",
              "barrier", "combine_nvlink")

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, _events=None) -> torch.Tensor:
        T = x.shape[0]
        if self._T != T:
            self._setup(T, x.device)
        G, L = self.G, self.L

        def mark():
            if _events is not None:
                _events.append(torch.cuda.Event(enable_timing=True))
                _events[-1].record()
        mark()
        ops.router_topk(x, self.w.wg, self.k, self.mode, out=(self.idx, self.wts, self.counts), workspace=self.rws)
        ops.permute(self.idx, x, self.E, 1, out=(self.offsets, self.dst, None), workspace=self.ws)
        mark()
        ops.ep_counts_put(self.counts, self.rank, G, self.peer_counts)
        self._barrier()
        self._offsets()
        mark()
        ops.ep_dispatch(self.idx, self.dst, self.offsets, self.send_base, x, G, self.cap, self.peer_recv,
                        self.route_row)
        self._barrier()
        mark()
        groups = list(range(L))  # one group per local expert (all sources' rows contiguous)
        pe = self.profile_events
        if pe:
            pe["k3"][0].record()
        ops.grouped_swiglu(self.recv, self.recv_seg, groups, self.w13, self.ff, h=self.h)
        if pe:
            pe["k3"][1].record()
            pe["k4"][0].record()
        mark()
        ops.grouped_down(self.h, self.recv_seg, groups, self.w2, self.d, y=self.ysym)
        if pe:
            pe["k4"][1].record()
        mark()
        self._barrier()
        mark()
        res = ops.ep_combine(self.idx, self.route_row, self.wts, self.E, G, self.peer_y,
                             self.out if out is None else out)
        mark()
        return res

    def stage_times(self, x: torch.Tensor) -> dict:
        """One instrumented step (CUDA events between the phases), in ms."""
        ev = []
        self.forward(x, _events=ev)
        torch.cuda.synchronize()
        return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(self.STAGES)}

    def exchange_bytes(self) -> dict:
        """Bytes this rank moved over NVLink in the last step (rows to / from
        other ranks' memory; its own rows stay local)."""
        idx = self.idx
        owner = torch.div(idx, self.L, rounding_mode="floor")
        remote = int(((owner != self.rank) & (self.route_row >= 0)).sum().item())
        row = self.d * 2
        return {"dispatch": remote * row, "combine": remote * row}

    __call__ = forward

    def check(self) -> None:
        """Raise if the last step dropped rows for capacity (only possible with
        check_capacity=False; raise capacity_factor)."""
        if self._T is not None and int(self.overflow.item()) != 0:
            raise RuntimeError(f"EP receive capacity {self.cap} rows exceeded (needed {int(self.overflow.item())}); "
                               "raise capacity_factor or use check_capacity=True")
