"""Stratified multi-layer expert stage: hot experts pinned in HBM under a
budget, cold experts streamed from pinned host memory, overlapped with the
resident experts' GEMMs (BASELINE.json configs[2]; SURVEY.md §8a rows a4,
a9-a12, a18).

Reference mapping:
  * AllocationStrategy.exp_r / exp_m (costmodel.py:45-89): per layer, the
    residency plan's experts are exp_r (weights in HBM), the rest exp_m
    (migrated every pass); exp_c must be 0 (no CPU expert path).
  * vram_usage resident term (costmodel.py:460): resident bytes =
    exp_r * 3*dt*d*ff * N; `capacity_per_layer` turns an HBM budget into exp_r.
  * eas.select_resident_experts + probe (eas.py:346-374): `calibrate()` runs
    prototype batches through the stack and accumulates the router's own
    histograms (K1) into an ActivationMap, then picks the resident sets.
  * sim.build_task_graph expert tasks (sim.py:149-202): measured timeline
    records with the same {name, res, ts, dur} schema (sim.py:356-361), with
    finer tasks: expert:gather (route+permute), expert:gpu:resident,
    expert:migrate:L<l> (copy stream), expert:gpu:cold, expert:merge.
    Unlike the reference's `expert:gpu` (which waits for the whole
    migration), resident GEMMs start immediately; only the cold groups wait
    for their copy events.

Synthetic-model caveat (stated in DESIGN.md): expert weights are drawn from a
pool of P distinct experts (expert (l, e) := pool[(l*E + e) % P]) so that the
cold set fits in this host's pinned RAM; resident experts are real, distinct
HBM copies and every cold expert crosses PCIe on every pass.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .config import ExpertStageParts, ResidencyPlan
from .eas import Calibrator, select_resident_experts
from .layer import MODES
from .streaming import HostExpertPool, SlotRing


@dataclass
class _Bufs:
    T: int
    idx: torch.Tensor
    w: torch.Tensor
    counts: torch.Tensor
    offsets: torch.Tensor
    dst: torch.Tensor
    x_perm: torch.Tensor  # also receives y (K4 output) — x_perm is dead after K3
    h: torch.Tensor
    ping: torch.Tensor
    pong: torch.Tensor
    ws: torch.Tensor
    router_ws: torch.Tensor


class StratifiedMoEStack:
    def __init__(self, num_layers: int, wg: torch.Tensor, pool: HostExpertPool, top_k: int,
                 residency: ResidencyPlan, mode: str = "mixtral", pool_map=None, residual: bool = True):
        """wg: [N, E, d] fp32 router weights on the device; pool: host experts.
        residual: layer l+1 consumes x_l + MoE_l(x_l) (the residual stream, added
        inside K5) instead of MoE_l(x_l) alone."""
        self.N = int(num_layers)
        self.wg = wg
        # router weights in bf16 when that is exact (as MoELayer): half the bytes, shared-memory resident
        wgb = wg.to(torch.bfloat16)
        self.wg_router = wgb if torch.equal(wgb.float(), wg) else wg
        self.E = wg.shape[1]
        self.d = wg.shape[2]
        self.ff = pool.w2.shape[2]
        self.k = int(top_k)
        self.mode = MODES[mode]
        self.pool = pool
        self.pool_map = pool_map or (lambda l, e: (l * self.E + e) % pool.size)
        self.device = wg.device
        self.residual = bool(residual)
        self.res_w13: list[dict[int, torch.Tensor]] = []
        self.res_w2: list[dict[int, torch.Tensor]] = []
        self.ring = None
        self._bufs = None
        self.set_residency(residency)

    # ------------------------------------------------------------ residency
    def set_residency(self, plan: ResidencyPlan) -> None:
        if plan.num_layers != self.N:
            raise ValueError("residency plan must cover every layer")
        self.plan = plan
        self.res_w13, self.res_w2 = [], []
        self.ring = None
        torch.cuda.empty_cache()
        for l in range(self.N):
            d13, d2 = {}, {}
            for e in plan.resident[l]:
                if not (0 <= e < self.E):
                    raise ValueError("resident expert id out of range")
                p = self.pool_map(l, e)
                d13[e] = self.pool.w13[p].to(self.device, non_blocking=True)
                d2[e] = self.pool.w2[p].to(self.device, non_blocking=True)
            self.res_w13.append(d13)
            self.res_w2.append(d2)
        self.cold = [[e for e in range(self.E) if e not in set(plan.resident[l])] for l in range(self.N)]
        C = max((len(c) for c in self.cold), default=0)
        self.C = C
        self.ring = SlotRing(2 * C, self.d, self.ff, self.device) if C else None
        torch.cuda.synchronize()

    @property
    def resident_bytes(self) -> int:
        per = self.pool.nbytes_per_expert()
        return per * sum(len(r) for r in self.plan.resident)

    @property
    def launches_per_step(self) -> int:
        return self.launches_per_step_at(1 << 20, "stream")

    def launches_per_step_at(self, T: int, fetch: str = "stream") -> int:
        """Kernel launches of one forward over T tokens (router, permute index
        kernel(s) + row copy, GEMMs, combine; touched mode: one fetch launch per
        layer with cold experts and one K3/K4 over all experts)."""
        perm = (1 if T * self.k <= 2048 else 3) + 1
        if fetch == "touched":
            return sum(1 + perm + (1 if self.cold[l] else 0) + 2 + 1 for l in range(self.N))
        return sum(1 + perm + 1 + (2 if self.plan.resident[l] else 0) + (2 if self.cold[l] else 0)
                   for l in range(self.N))

    def _buffers(self, T: int) -> _Bufs:
        if self._bufs is None or self._bufs.T != T:
            self._bufs = None
            torch.cuda.empty_cache()
            dev, bf = self.device, torch.bfloat16
            cap = ops.rows_capacity(T, self.k, self.E, 1)
            self._bufs = _Bufs(
                T=T, idx=torch.empty((T, self.k), dtype=torch.int32, device=dev),
                w=torch.empty((T, self.k), dtype=torch.float32, device=dev),
                counts=torch.empty((self.E,), dtype=torch.int32, device=dev),
                offsets=torch.empty((self.E + 1,), dtype=torch.int32, device=dev),
                dst=torch.empty((T, self.k), dtype=torch.int32, device=dev),
                x_perm=torch.empty((cap, self.d), dtype=bf, device=dev),
                h=torch.empty((cap, self.ff), dtype=bf, device=dev),
                ping=torch.empty((T, self.d), dtype=bf, device=dev),
                pong=torch.empty((T, self.d), dtype=bf, device=dev),
                ws=torch.empty((max(16, ops.permute_workspace_bytes(T, self.E)),), dtype=torch.uint8, device=dev),
                router_ws=ops.router_workspace(T, self.E, dev))
        return self._bufs

    # ------------------------------------------------------------ forward
    def _stage_layer(self, l: int, timing: bool):
        base = (l % 2) * self.C
        return [self.ring.stage(self.pool, self.pool_map(l, e), base + j, timing) for j, e in enumerate(self.cold[l])]

    # decode-size batches fetch only the cold experts the router touched (on the device)
    TOUCHED_T_MAX = 4096

    def forward(self, x: torch.Tensor, timeline: bool = False, counts_out: torch.Tensor | None = None,
                fetch: str = "auto"):
        """Run all N layers; returns the last layer's output (a view of an internal buffer).

        counts_out: optional [N, E] int32 device tensor receiving each layer's
        routed-token histogram (calibration / hit-ratio accounting).
        fetch: "stream" — every cold expert of every layer is copied (copy
        engine, two layers ahead, overlapped with the resident GEMMs; prefill);
        "touched" — after each layer's router, cox_fetch_experts copies only the
        cold experts that received tokens (decided on the device; decode-size
        steps); "auto" — touched for T <= TOUCHED_T_MAX, else stream."""
        if x.dtype != torch.bfloat16 or x.shape[1] != self.d:
            raise ValueError(f"x must be bf16 [T, {self.d}]")
        if fetch not in ("auto", "stream", "touched"):
            raise ValueError("fetch must be auto, stream or touched")
        T = x.shape[0]
        if fetch == "auto":
            fetch = "touched" if T <= self.TOUCHED_T_MAX else "stream"
        b = self._buffers(T)
        self._records = []
        if self.ring is not None:
            self.ring.copy_events = []
        if fetch == "touched":
            return self._forward_touched(x, b, timeline, counts_out)
        s = torch.cuda.current_stream()
        copy_done = {}
        if self.C:
            for l in range(min(2, self.N)):
                copy_done[l] = self._stage_layer(l, timeline)
        cur = x
        for l in range(self.N):
            out = b.ping if (l % 2 == 0) else b.pong
            e0 = self._mark(timeline)
            self._route(cur, b, l, counts_out)
            e1 = self._mark(timeline)
            res = list(self.plan.resident[l])
            if res:
                ops.grouped_swiglu(b.x_perm, b.offsets, res, [self.res_w13[l][e] for e in res], self.ff, h=b.h)
            e2 = self._mark(timeline)
            cold = self.cold[l]
            if cold:
                for ev in copy_done.pop(l, []):
                    s.wait_event(ev)
            e2w = self._mark(timeline)  # the cold GEMMs' copies have landed
            if cold:
                base = (l % 2) * self.C
                slots = [base + j for j in range(len(cold))]
                ops.grouped_swiglu(b.x_perm, b.offsets, cold, [self.ring.w13[i] for i in slots], self.ff, h=b.h)
                ops.grouped_down(b.h, b.offsets, cold, [self.ring.w2[i] for i in slots], self.d, y=b.x_perm)
                for i in slots:
                    self.ring.release(i, s)
            # layer l+2 reuses layer l's slot half; staged whether or not layer l
            # had cold experts itself (plans may differ in exp_r per layer)
            if self.C and l + 2 < self.N and self.cold[l + 2]:
                copy_done[l + 2] = self._stage_layer(l + 2, timeline)
            e3 = self._mark(timeline)
            if res:
                ops.grouped_down(b.h, b.offsets, res, [self.res_w2[l][e] for e in res], self.d, y=b.x_perm)
            e4 = self._mark(timeline)
            # residual stream: out = x_l + sum_j w_j y_j, fused into K5 (shared_out = x_l)
            ops.combine(b.x_perm, b.dst, b.w, shared=cur if self.residual else None, out=out)
            e5 = self._mark(timeline)
            if timeline:
                self._records += [(f"expert:gather:L{l}", "gpu", e0, e1), (f"expert:gpu:resident:L{l}", "gpu", e1, e2),
                                  (f"expert:wait:L{l}", "wait", e2, e2w), (f"expert:gpu:cold:L{l}", "gpu", e2w, e3),
                                  (f"expert:gpu:resident:L{l}", "gpu", e3, e4), (f"expert:merge:L{l}", "gpu", e4, e5)]
            cur = out
        if timeline and self.ring is not None:
            for i, (slot, a, b2) in enumerate(self.ring.copy_events):
                self._records.append((f"expert:migrate:slot{slot}:{i}", "h2d", a, b2))
        return cur

    __call__ = forward

    @staticmethod
    def _mark(timeline: bool):
        if not timeline:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def _route(self, cur, b, l, counts_out):
        ops.router_topk(cur, self.wg_router[l], self.k, self.mode, out=(b.idx, b.w, b.counts), workspace=b.router_ws)
        ops.permute(b.idx, cur, self.E, 1, out=(b.offsets, b.dst, b.x_perm), workspace=b.ws)
        if counts_out is not None:
            counts_out[l].copy_(b.counts)

    def _forward_touched(self, x, b, timeline, counts_out):
        """Decode-size steps: per layer router -> device-side fetch of the touched
        cold experts (pinned host -> slots [0, C)) -> one grouped K3/K4 over all
        experts (resident copies and fetched slots) -> combine + residual.
        self.fetched_entries accumulates, per layer, how many cold entries (W13 /
        W2 of an expert) crossed PCIe."""
        cur = x
        if self.C:
            if getattr(self, "_fetched", None) is None or self._fetched.shape != (self.N, 2 * self.C):
                self._fetched = torch.zeros((self.N, 2 * self.C), dtype=torch.int32, device=self.device)
        for l in range(self.N):
            out = b.ping if (l % 2 == 0) else b.pong
            e0 = self._mark(timeline)
            self._route(cur, b, l, counts_out)
            e1 = self._mark(timeline)
            cold = self.cold[l]
            w13 = [None] * self.E
            w2 = [None] * self.E
            for e, t in self.res_w13[l].items():
                w13[e], w2[e] = t, self.res_w2[l][e]
            if cold:
                ids, src, dst = [], [], []
                for j, e in enumerate(cold):
                    p = self.pool_map(l, e)
                    ids += [e, e]
                    src += [self.pool.w13[p], self.pool.w2[p]]
                    dst += [self.ring.w13[j], self.ring.w2[j]]
                    w13[e], w2[e] = self.ring.w13[j], self.ring.w2[j]
                ops.fetch_experts(b.counts, ids, src, dst, fetched=self._fetched[l, : 2 * len(cold)])
            e2 = self._mark(timeline)
            groups = list(range(self.E))
            ops.grouped_swiglu(b.x_perm, b.offsets, groups, w13, self.ff, h=b.h)
            ops.grouped_down(b.h, b.offsets, groups, w2, self.d, y=b.x_perm)
            e3 = self._mark(timeline)
            ops.combine(b.x_perm, b.dst, b.w, shared=cur if self.residual else None, out=out)
            e4 = self._mark(timeline)
            if timeline:
                self._records += [(f"expert:gather:L{l}", "gpu", e0, e1), (f"expert:migrate:touched:L{l}", "h2d", e1, e2),
                                  (f"expert:gpu:L{l}", "gpu", e2, e3), (f"expert:merge:L{l}", "gpu", e3, e4)]
            cur = out
        return cur

    def fetched_cold_experts(self) -> float:
        """Mean number of cold experts fetched per layer by the last touched-mode step."""
        if getattr(self, "_fetched", None) is None:
            return 0.0
        return float(self._fetched.sum().item()) / 2.0 / self.N

    # ------------------------------------------------------------ reporting
    def timeline_records(self) -> list[dict]:
        """Measured timeline in sim.timeline_records' schema (sim.py:356-361):
        [{"name", "res", "ts", "dur"}] in seconds from the first event."""
        torch.cuda.synchronize()
        recs = getattr(self, "_records", None) or []
        if not recs:
            return []
        t0 = recs[0][2]
        out = [{"name": n, "res": r, "ts": t0.elapsed_time(a) / 1e3, "dur": a.elapsed_time(b) / 1e3}
               for n, r, a, b in recs]
        return sorted(out, key=lambda r: r["ts"])

    def measured_parts(self) -> ExpertStageParts:
        """Per-layer mean of the measured timeline, in ExpertStageParts' fields
        (costmodel.py:199-222): act_load 0 (activations stay in HBM),
        mig_load = copy-engine busy time, lat_gpu = stage GPU time (kernels
        only: time the stream spent waiting for a copy is excluded)."""
        rec = self.timeline_records()
        n = max(1, self.N)
        mig = sum(r["dur"] for r in rec if r["res"] == "h2d") / n
        gpu = sum(r["dur"] for r in rec if r["res"] == "gpu") / n
        return ExpertStageParts(act_load=0.0, mig_load=mig, lat_gpu=gpu, lat_cpu=0.0, return_store=0.0)

    # ------------------------------------------------------------ orchestrator bridge
    def apply_strategy(self, strategy, model=None, activation_map=None) -> ResidencyPlan:
        """Adopt the expert partition an orchestrator chose — a moeplan
        `AllocationStrategy` or `Plan` (planner.plan, planner.py:246-272; its
        `prefill_strategy` is used): exp_r experts per layer stay resident
        (the hottest ones of `activation_map`, default: the calibration map),
        exp_m are streamed; exp_c must be 0 (no CPU expert path)."""
        strategy = getattr(strategy, "prefill_strategy", strategy)
        total = strategy.exp_r + strategy.exp_m + strategy.exp_c
        if total != self.E:
            raise ValueError(f"expert partition {strategy.exp_r}+{strategy.exp_m}+{strategy.exp_c} "
                             f"does not cover the {self.E} activated experts")
        if strategy.exp_c != 0:
            raise ValueError("the B200 executor runs every expert on the GPU: exp_c must be 0")
        amap = activation_map if activation_map is not None else getattr(self, "calibration_map", None)
        if amap is None:
            from .config import ActivationMap
            amap = ActivationMap.uniform(self.N, self.E)
        plan = select_resident_experts(amap, strategy.exp_r)
        self._bufs = None
        self.set_residency(plan)
        return plan

    # ------------------------------------------------------------ calibration
    def max_capacity(self, T: int, slack_bytes: int = 4 << 30) -> int:
        """Largest exp_r whose resident copies + the T-token activations + the
        2*(E - exp_r) slot ring fit in the free HBM (x, ping, pong, x_perm, h) (the vram_usage feasibility
        test, costmodel.py:440-489, with measured free memory).  Leaves the
        stack with an empty residency plan (every expert cold)."""
        self.ring = None
        self._bufs = None
        self.res_w13, self.res_w2 = [], []
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info(self.device)
        per = self.pool.nbytes_per_expert()
        act = T * self.d * 2 * 3 + ops.rows_capacity(T, self.k, self.E) * (self.d + self.ff) * 2
        best = 0
        for cap in range(self.E, -1, -1):
            need = cap * per * self.N + 2 * (self.E - cap) * per + act + slack_bytes
            if need <= free:
                best = cap
                break
        # the resident copies were freed to measure: continue with every expert cold
        self.set_residency(ResidencyPlan(tuple(() for _ in range(self.N)), 0))
        return best

    def calibrate(self, batches, capacity_per_layer: int) -> ResidencyPlan:
        """Prefill-only probing: run prototype batches through the
        stack, accumulate K1 histograms per layer, choose the hot set per layer
        (eas.select_resident_experts) and re-place the resident copies."""
        cal = Calibrator(self.N, self.E)
        counts = torch.zeros((self.N, self.E), dtype=torch.int32, device=self.device)
        for xb in batches:
            self.forward(xb, counts_out=counts)
            torch.cuda.synchronize()
            c = counts.cpu().numpy()
            for l in range(self.N):
                cal.observe(l, c[l])
        plan = select_resident_experts(cal.activation_map(), capacity_per_layer)
        self._bufs = None
        self.set_residency(plan)
        self.calibration_map = cal.activation_map()
        return plan


_MEASURE_CACHE: dict = {}


def measured_expert_stage_parts(strategy, phase, system, model, batch, activation_map=None, coalesced: bool = True,
                                *, mode: str = "mixtral", warmup: int = 1, device=None) -> ExpertStageParts:
    """The MEASURED counterpart of costmodel.expert_stage_parts, with its
    signature (costmodel.py:225-233): one MoE layer of `model` runs on this
    B200 over batch.batch_size x phase.seq_len synthetic tokens, with
    strategy.exp_r experts resident (the hottest of `activation_map`, summed
    over its layers) and strategy.exp_m streamed from pinned host memory.
    Returns seconds per layer in ExpertStageParts' fields:
      act_load     0 — activations stay in HBM (no PCIe gather on B200);
      mig_load     copy-engine busy time of the exp_m cold experts;
      lat_gpu      GPU time of the expert stage (router .. combine);
      lat_cpu      0 — no CPU expert path (exp_c must be 0);
      return_store 0.
    coalesced=False runs ceil(B / strategy.m) micro-batches of strategy.m
    sequences (the reference's `repeats`, costmodel.py:254-260) and sums them.
    `system` is accepted for signature parity (the hardware is measured)."""
    from .config import ActivationMap
    from .synthetic import make_tokens
    if strategy.exp_r + strategy.exp_m + strategy.exp_c != model.experts_per_layer:
        raise ValueError(f"expert partition {strategy.exp_r}+{strategy.exp_m}+{strategy.exp_c} "
                         f"does not cover the {model.experts_per_layer} activated experts")
    if strategy.exp_c != 0:
        raise ValueError("the B200 executor runs every expert on the GPU: exp_c must be 0")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    E, d, ff, k = model.experts_per_layer, model.hidden_dim, model.expert_dim, model.top_k
    key = (E, d, ff, k, mode, str(dev))
    stack = _MEASURE_CACHE.get(key)
    if stack is None:
        _MEASURE_CACHE.clear()
        pool = make_pool(E, d, ff, seed=0, device=dev)
        wg = make_router_weights(1, E, d, seed=7, device=dev)
        stack = StratifiedMoEStack(1, wg, pool, k, ResidencyPlan(((),), 0), mode, pool_map=lambda l, e: e,
                                   residual=False)
        _MEASURE_CACHE[key] = stack
    counts = np.ones((1, E)) if activation_map is None else \
        np.asarray(activation_map.counts, dtype=float).sum(axis=0, keepdims=True)
    stack.set_residency(select_resident_experts(ActivationMap(counts), strategy.exp_r))
    L = int(phase.seq_len)
    B = int(batch.batch_size)
    m = B if coalesced else int(strategy.m)
    sizes = [min(m, B - s0) for s0 in range(0, B, m)]
    mig = gpu = 0.0
    for nseq in sorted(set(sizes)):
        x = make_tokens(nseq * L, d, seed=1, device=dev)
        for _ in range(warmup):
            stack(x, fetch="stream")
        stack(x, timeline=True, fetch="stream")
        parts = stack.measured_parts()
        reps = sizes.count(nseq)
        mig += reps * parts.mig_load
        gpu += reps * parts.lat_gpu
        del x
    stack._bufs = None
    return ExpertStageParts(act_load=0.0, mig_load=mig, lat_gpu=gpu, lat_cpu=0.0, return_store=0.0)


def make_pool(P: int, d: int, ff: int, seed: int = 0, device="cuda", residual_scale: float = 1.0) -> HostExpertPool:
    """P distinct random experts generated on the device, copied to pinned host memory.

    residual_scale multiplies the down projections (GPT-2-style 1/sqrt(2 N)
    init of residual branches): the stack has no normalisation between layers,
    and with unit-scaled random experts reused every P/E layers the residual
    stream of a deep stack grows geometrically (overflow after ~50 layers)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    w13 = torch.empty((P, 2 * ff, d), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((P, d, ff), dtype=torch.bfloat16, device=device)
    a2 = residual_scale * ff ** -0.5
    for p in range(P):
        w13[p].uniform_(-d ** -0.5, d ** -0.5, generator=g)
        w2[p].uniform_(-a2, a2, generator=g)
    pool = HostExpertPool.from_device(w13, w2)
    del w13, w2
    torch.cuda.empty_cache()
    return pool


def make_router_weights(N: int, E: int, d: int, seed: int = 7, device="cuda") -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    wg = torch.empty((N, E, d), dtype=torch.float32, device=device)
    wg.uniform_(-d ** -0.5, d ** -0.5, generator=g)
    return wg.to(torch.bfloat16).float()


def hit_ratio_of_counts(counts: np.ndarray, plan: ResidencyPlan) -> float:
    from .eas import hit_ratio_from_counts
    return hit_ratio_from_counts(counts, plan)


__all__ = ["StratifiedMoEStack", "make_pool", "make_router_weights", "HostExpertPool", "hit_ratio_of_counts",
           "measured_expert_stage_parts"]
