#!/usr/bin/env python
"""Benchmark of the coalesced MoE expert stage (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C1|C3L|C4]

One "step" = one full expert stage (router -> permute -> grouped SwiGLU ->
grouped down -> combine) over one batch of synthetic tokens.  Default workload
= BASELINE.json configs[1] (C2): Mixtral-8x7B-shaped layer, E=8, top-2,
d=4096, ff=14336, batch 64x4096 = 262,144 tokens per GPU, bf16.

N > 1 (torchrun, one process per GPU): expert parallelism — each rank holds its
own 64x4096 batch (weak scaling) and E/N experts; tokens travel by NCCL
all-to-all (ep.py).  Time = max over ranks of CUDA-event time.

Prints ONE JSON line on rank 0.  `value` is device-resident throughput; `e2e`
is the same metric through the public API (MoELayer / EP layer) with the
tokens copied from pinned host memory and the output copied back inside the
timed region.  `cpu_baseline` times the fp32 CPU oracle (oracle/, the
"reference CPU path": moeplan ships no executable expert stage) on a bounded
token slice on this host.

--impl reference: times that CPU oracle alone (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (T per GPU, d, ff, E, k, mode, shared_ff, description)
    "C2": (64 * 4096, 4096, 14336, 8, 2, "mixtral", 0,
           "C2 Mixtral-8x7B MoE layer (E=8, top-2, d=4096, ff=14336), prefill batch 64x4096 per GPU"),
    "C1": (16 * 256, 1024, 3584, 8, 2, "mixtral", 0,
           "C1 tiny Mixtral-style MoE layer (E=8, top-2, d=1024, ff=3584), batch 16x256 (bf16 on GPU), "
           "CUDA-graph replay"),
    "C3L": (64 * 4096, 6144, 16384, 8, 2, "mixtral", 0,
            "C3/C5 Mixtral-8x22B MoE layer (E=8, top-2, d=6144, ff=16384), batch 64x4096 per GPU"),
    "C4": (64 * 4096, 2048, 1408, 64, 6, "deepseek", 2816,
           "C4 DeepSeek-V2-Lite MoE layer (64 routed top-6 + 2 shared, d=2048, ff=1408), batch 64x4096"),
    "C4D": (64, 2048, 1408, 64, 6, "deepseek", 2816,
            "C4 DeepSeek-V2-Lite MoE layer decode step: 64 sequences x 1 token (64 routed top-6 + 2 shared), "
            "CUDA-graph replay"),
    "C2D": (64, 4096, 14336, 8, 2, "mixtral", 0,
            "C2 Mixtral-8x7B MoE layer decode step: 64 sequences x 1 token (not a BASELINE config: the decode "
            "kernel at 352 MB experts), CUDA-graph replay"),
    "C3": (64 * 4096, 6144, 16384, 8, 2, "mixtral", 0,
           "C3 Mixtral-8x22B-shaped 56-layer MoE stack, batch 64x4096, HBM budget -> calibrated hot experts "
           "resident, cold experts streamed from pinned host memory"),
    "C3D": (8, 6144, 16384, 8, 2, "mixtral", 0,
            "C3 56-layer stack decode step: 8 sequences x 1 token; cold experts fetched only when routed to "
            "(device-side decision), calibrated vs random residency"),
}
STACK_LAYERS = 56


def metric_name(config: str) -> str:
    if config == "C2":
        return "MoE layer tokens/s, Mixtral-8x7B layer, b64x4096"
    return f"MoE layer tokens/s, {config}"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
                for n, v in zip(names, f[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
                pw.append(float(f[6]))
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_max": max(pw) if pw else None, "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(wts_host, x_host, k, mode_id, shared_host, n_tokens):
    """fp32 CPU oracle over the first n_tokens tokens (routed exactly as in the full batch).
    Returns (tokens/s, threads, seconds, oracle result dict)."""
    from oracle import oracle as O
    O.lib()
    threads = len(os.sched_getaffinity(0))
    O.set_num_threads(threads)
    xs = x_host[:n_tokens]
    t0 = time.perf_counter()
    ref = O.moe_layer(xs, wts_host["wg"], wts_host["w1"], wts_host["w3"], wts_host["w2"], k, mode_id,
                      shared=shared_host)
    dt = time.perf_counter() - t0
    return n_tokens / dt, threads, dt, ref


def gpu_routing(layer, x):
    """(idx, counts, offsets, dst) the timed path produced for x (numpy; offsets
    / dst None where the path materialises no permutation)."""
    import torch
    from paper_2605_17889_b200 import ops
    T = x.shape[0]
    c = lambda t: t.cpu().numpy() if t is not None else None  # noqa: E731
    if hasattr(layer, "buffers"):  # MoELayer: buffers of its last step over x
        b = layer.buffers(T, x.device)
        perm = not layer.uses_dense_decode(T)
        return c(b.idx), c(b.counts), c(b.offsets) if perm else None, c(b.dst) if perm else None
    if hasattr(layer, "route_row"):  # fused EP: routing of the rank's own tokens
        return c(layer.idx), c(layer.counts), c(layer.offsets), c(layer.dst)
    # NCCL EP: the same router + permute kernels its stage runs
    idx, _, counts, _, _ = layer.stage.route_and_permute(x)
    offsets = torch.empty((layer.E + 1,), dtype=torch.int32, device=x.device)
    dst = torch.empty_like(idx)
    ops.permute(idx, x, layer.E, out=(offsets, dst, None))
    return c(idx), c(counts), c(offsets), c(dst)


def cpu_baseline_and_parity(args, layer, wts, x, out_full, k, mode):
    """cpu_baseline: the fp32 oracle over the first n tokens of this rank's batch
    (routed as in the full batch), timed on this host.  parity: (1) routing of
    the FULL batch — idx, counts, offsets, dst — against the oracle router
    (OpenMP over tokens) bit for bit; (2) the layer output of the first n tokens
    against the fp32 oracle layer, rel-L2 <= 1e-2."""
    import numpy as np
    import torch
    from oracle import oracle as O
    T, d = x.shape
    E = wts.num_experts
    mode_id = 0 if mode == "mixtral" else 1
    n = min(T, args.cpu_tokens)
    hw, shared = host_weights(wts)
    cps, threads, dt, ref = cpu_baseline(hw, x[:n].float().cpu().numpy(), k, mode_id, shared, n)
    cpu = {"value": cps, "unit": "tokens/s", "cores": threads, "kind": "port",
           "sample": (f"all {T} tokens of the step" if n == T else f"first {n} of {T} tokens (routed as in the full "
                      "batch)") + f", full-size weights, fp32 oracle (oracle/, OpenMP x{threads}) on "
                      f"{cpu_model_name()}: {dt:.2f} s"}
    gi, gc, go, gd = gpu_routing(layer, x)
    t0 = time.perf_counter()
    oi, _, oc = O.router_topk_bf16(x.view(torch.int16).cpu().numpy().view(np.uint16), hw["wg"], k, mode_id)
    oo, od = O.permute(oi, E, 1)
    t_route = time.perf_counter() - t0
    routing_ok = bool(np.array_equal(gi, oi) and np.array_equal(gc, oc)
                      and (go is None or np.array_equal(go, oo)) and (gd is None or np.array_equal(gd, od)))
    gout = out_full[:n].float().cpu().numpy().astype(np.float64)
    err = float(np.linalg.norm(gout - ref["out"]) / max(np.linalg.norm(ref["out"]), 1e-30))
    parity = {"routing_tokens_checked": T, "routing_bitexact": routing_ok,
              "routing_checked": "idx, counts" + (", offsets, dst" if go is not None else ""),
              "routing_oracle_s": round(t_route, 2),
              "tokens_checked": n, "routing_indices_bitexact": bool(np.array_equal(gi[:n], ref["idx"])),
              "out_rel_l2_vs_fp32_oracle": err, "tolerance": 1e-2, "pass": bool(routing_ok and err <= 1e-2)}
    return cpu, parity


def host_weights(wts):
    import numpy as np  # noqa: F401
    from paper_2605_17889_b200.synthetic import split_w13
    w1, w3 = split_w13(wts.w13)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    hw = {"wg": f(wts.wg), "w1": f(w1), "w3": f(w3), "w2": f(wts.w2)}
    shared = None
    if wts.shared_w13 is not None:
        s1, s3 = split_w13(wts.shared_w13)
        shared = (f(s1), f(s3), f(wts.shared_w2))
    return hw, shared


def cpu_model_name():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg):
    """--impl reference: the fp32 CPU oracle (the reference ships no executable expert stage)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
    T, d, ff, E, k, mode, shared_ff, desc = cfg
    sample = min(T, args.ref_tokens)
    # the same seeded generators (and so the same bits) as the GPU arm's inputs:
    # drawn on the GPU when there is one (data generation only, no kernels of
    # ours), then moved to host memory for the CPU oracle
    gen_dev = "cuda" if torch.cuda.is_available() else "cpu"
    wts = make_layer_weights(E, d, ff, seed=0, device=gen_dev, shared_ff=shared_ff)
    x = make_tokens(T if gen_dev == "cuda" else sample, d, seed=1, device=gen_dev)[:sample].float().cpu().numpy()
    hw, shared = host_weights(wts)
    del wts
    if gen_dev == "cuda":
        torch.cuda.empty_cache()
    threads = len(os.sched_getaffinity(0))
    O.set_num_threads(threads)
    mode_id = 0 if mode == "mixtral" else 1
    for _ in range(args.warmup):
        O.moe_layer(x[: max(8, sample // 8)], hw["wg"], hw["w1"], hw["w3"], hw["w2"], k, mode_id, shared=shared)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.moe_layer(x, hw["wg"], hw["w1"], hw["w3"], hw["w2"], k, mode_id, shared=shared)
    dt = time.perf_counter() - t0
    value = sample * args.steps / dt
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (the GPU arm's seeded inputs, generated on {gen_dev})",
        "config": {"workload": desc, "tokens_per_step": sample, "d": d, "ff": ff, "E": E, "k": k},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"first {sample} of {T} tokens per step, full-size weights, fp32 oracle "
                                   f"(oracle/, OpenMP x{threads}) on {cpu_model_name()}"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def _stack_setup(args, cfg, T_eval):
    """C3 stack on one GPU with topic-structured routing; calibrated residency.

    Expert (l, e) weights are pool[(l*E + e) % P] (P distinct experts in pinned
    host RAM); the router rows carry per-(topic, layer) Zipf preferences
    (synthetic.make_topic_router, the GPU analogue of
    eas.generate_synthetic_trace).  Calibration = prefill-only probing
    (PAPER.md:308): candidate sequences are clustered on their embeddings
    (eas.cluster), prototypes chosen nearest-to-centroid (eas.select_prototypes,
    ratio 0.05), run through the stack, and the K1 histograms give the
    ActivationMap from which eas.select_resident_experts picks the hot set
    under the HBM budget (max_capacity: measured free HBM, the vram_usage
    feasibility test)."""
    import torch
    from paper_2605_17889_b200 import eas
    from paper_2605_17889_b200.config import ResidencyPlan
    from paper_2605_17889_b200.executor import StratifiedMoEStack, make_pool
    from paper_2605_17889_b200.synthetic import (make_topic_router, make_topic_tokens, make_topic_workload,
                                                 sequence_embeddings)
    T, d, ff, E, k, mode, _, desc = cfg
    N = args.layers
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    pool = make_pool(args.pool, d, ff, seed=0, device=dev, residual_scale=(2.0 * N) ** -0.5)
    wl = make_topic_workload(d, num_topics=args.topics, device=dev)
    wg = make_topic_router(N, E, d, wl, device=dev)
    stack = StratifiedMoEStack(N, wg, pool, k, ResidencyPlan(tuple(() for _ in range(N)), 0), mode)
    n_cand, cand_len = 256, 256
    xc, _ = make_topic_tokens(wl, n_cand, cand_len, seed=100, device=dev)
    cl = eas.cluster(sequence_embeddings(xc, n_cand), args.topics, seed=0)
    protos = eas.select_prototypes(cl, 0.05)
    xp = xc.reshape(n_cand, cand_len, d)[torch.tensor(protos, device=dev)].reshape(-1, d).contiguous()
    del xc
    cap = stack.max_capacity(T_eval)
    t0 = time.perf_counter()
    plan = stack.calibrate([xp], cap)
    t_cal = time.perf_counter() - t0
    info = {"prototypes": len(protos), "prototype_tokens": int(xp.shape[0]), "candidates": n_cand,
            "clusters": args.topics, "calibration_s": round(t_cal, 2), "capacity_per_layer": cap}
    return stack, wl, plan, cap, info


def _hit_summary(counts, plan, E, cap):
    """Token-weighted hit ratio of the timed batch's K1 histograms: calibrated
    plan, eas.random_baseline (mean of 50 seeds), and the batch's own top-cap."""
    from paper_2605_17889_b200 import eas
    from paper_2605_17889_b200.config import ActivationMap
    c = counts.cpu().numpy().astype(float)
    best = eas.select_resident_experts(ActivationMap(c + 1e-9), cap)
    return {"calibrated": eas.hit_ratio_from_counts(c, plan),
            "random_baseline_mean50": eas.random_hit_ratio(c, E, cap),
            "exact_map_upper_bound": eas.hit_ratio_from_counts(c, best)}


def stack_parity_and_cpu(args, stack, T, mode):
    """C3 / C3D: parity and CPU baseline on the stack's LAST layer of the last
    step (its input is layer N-2's output, still in the ping/pong buffer).
    parity: that layer's routing of the FULL batch (idx, counts, offsets, dst)
    against the oracle router, bit for bit, and its output (residual included)
    on the first n tokens against the fp32 oracle layer (rel-L2 <= 1e-2).
    cpu_baseline: the oracle's rate through that one layer, divided by the
    stack depth (the stack's tokens/s on the host)."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_2605_17889_b200.synthetic import split_w13
    b = stack._bufs
    N, E, k = stack.N, stack.E, stack.k
    if N < 2 or b is None:
        return None, None
    l = N - 1
    x_in = b.ping if (N - 2) % 2 == 0 else b.pong
    out = b.ping if l % 2 == 0 else b.pong
    mode_id = 0 if mode == "mixtral" else 1
    wg = stack.wg[l].float().cpu().numpy()
    gi, gc, go, gd = (t.cpu().numpy() for t in (b.idx, b.counts, b.offsets, b.dst))
    t0 = time.perf_counter()
    oi, _, oc = O.router_topk_bf16(x_in.view(torch.int16).cpu().numpy().view(np.uint16), wg, k, mode_id)
    oo, od = O.permute(oi, E, 1)
    t_route = time.perf_counter() - t0
    routing_ok = bool(np.array_equal(gi, oi) and np.array_equal(gc, oc) and np.array_equal(go, oo)
                      and np.array_equal(gd, od))
    n = min(T, args.cpu_tokens)
    ps = [stack.pool_map(l, e) for e in range(E)]
    w1, w3 = split_w13(torch.stack([stack.pool.w13[p] for p in ps]))
    w2 = torch.stack([stack.pool.w2[p] for p in ps])
    f = lambda t: t.float().numpy()  # noqa: E731
    threads = len(os.sched_getaffinity(0))
    O.set_num_threads(threads)
    xs = x_in[:n].float().cpu().numpy()
    t0 = time.perf_counter()
    ref = O.moe_layer(xs, wg, f(w1), f(w3), f(w2), k, mode_id, shared=None)
    dt = time.perf_counter() - t0
    ref_out = ref["out"] + (xs.astype(np.float64) if stack.residual else 0.0)
    gout = out[:n].float().cpu().numpy().astype(np.float64)
    err = float(np.linalg.norm(gout - ref_out) / max(np.linalg.norm(ref_out), 1e-30))
    cpu = {"value": n / dt / N, "unit": "tokens/s", "cores": threads, "kind": "port",
           "sample": f"first {n} of {T} tokens through one layer (layer {l}: its router rows and experts, "
                     f"full size), fp32 oracle (oracle/, OpenMP x{threads}) on {cpu_model_name()}: {dt:.2f} s; "
                     f"value = that per-layer rate / {N} layers"}
    parity = {"layer_checked": l, "routing_tokens_checked": T, "routing_bitexact": routing_ok,
              "routing_checked": "idx, counts, offsets, dst", "routing_oracle_s": round(t_route, 2),
              "tokens_checked": n, "routing_indices_bitexact": bool(np.array_equal(gi[:n], ref["idx"])),
              "out_rel_l2_vs_fp32_oracle": err, "tolerance": 1e-2, "pass": bool(routing_ok and err <= 1e-2)}
    return cpu, parity


def stack_e2e(stack, xs_dev, steps, fetch):
    """End to end through StratifiedMoEStack.forward with host buffers: each
    step copies its tokens from pinned host memory, runs every layer and reads
    the last layer's output back to pinned host memory, inside the timed region."""
    import torch
    xs_host = [x.cpu().pin_memory() for x in xs_dev]
    T, d = xs_dev[0].shape
    x_dev = torch.empty_like(xs_dev[0])
    out_host = torch.empty((T, d), dtype=torch.bfloat16).pin_memory()
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(steps):
        x_dev.copy_(xs_host[i % len(xs_host)], non_blocking=True)
        o = stack(x_dev, fetch=fetch)
        out_host.copy_(o, non_blocking=True)
    z.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(z) / steps
    return {"value": T / (ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": T * d * 2,
            "d2h_bytes_per_step": T * d * 2, "steps": steps,
            "api": "StratifiedMoEStack.forward (pinned host tokens in, last layer's output out, inside the timed "
                   "region)"}


def run_stack(args, cfg):
    """C3: the 56-layer stratified stack on one GPU (BASELINE.json configs[2])."""
    import torch
    from paper_2605_17889_b200 import costmodel as CM
    from paper_2605_17889_b200.config import ModelConfig, AllocationStrategy, Device, BatchConfig, Phase
    from paper_2605_17889_b200.synthetic import make_topic_tokens

    T, d, ff, E, k, mode, _, desc = cfg
    N = args.layers
    stack, wl, plan, cap, cal = _stack_setup(args, cfg, T)
    x, _ = make_topic_tokens(wl, 64, T // 64, seed=1, device="cuda")
    counts = torch.zeros((N, E), dtype=torch.int32, device="cuda")
    for _ in range(args.warmup):
        stack(x, fetch="stream")
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        a.record(s)
        for i in range(args.steps):
            stack(x, counts_out=counts if i == args.steps - 1 else None, fetch="stream")
        b.record(s)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    stack(x, timeline=True, fetch="stream")
    parts = stack.measured_parts()
    cpu = parity = e2e = None
    if not args.no_cpu_baseline:
        cpu, parity = stack_parity_and_cpu(args, stack, T, mode)
    if not args.no_e2e:
        e2e = stack_e2e(stack, [x], 1, "stream")
    pk = peaks()
    flops = N * (6.0 * T * k * d * ff + 2.0 * T * d * E)
    n_cold = sum(len(c) for c in stack.cold)
    mig_bytes = n_cold * stack.pool.nbytes_per_expert()
    model = ModelConfig(N, d, ff, E, k, 2)
    strat = AllocationStrategy((Device.GPU,) * 3, cap, E - cap, 0, m=64)
    system = CM.load_system_spec(CM.B200_SYSTEM_YAML)
    ana = CM.expert_stage_parts(strat, Phase.prefill(T // 64), system, model, BatchConfig(64, T // 64, 0),
                                stack.calibration_map, count_top_k=True)
    line = {
        "metric": metric_name("C3"), "value": T / (ms / 1e3), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic; topic-structured routing (make_topic_router); expert (l,e) weights = pool[(l*E+e) % P] "
                "(P distinct experts in pinned host RAM)",
        "config": {"workload": desc, "layers": N, "tokens": T, "d": d, "ff": ff, "E": E, "k": k,
                   "resident_per_layer": cap, "resident_bytes": stack.resident_bytes, "host_pool_experts": args.pool,
                   "cold_experts_per_step": n_cold, "h2d_bytes_per_step": mig_bytes, "calibration": cal},
        "stack_tflops": flops / (ms / 1e3) / 1e12,
        "frac_of_bf16_sustained": flops / (ms / 1e3) / 1e12 / pk["bf16_sus"],
        "hit_ratio": _hit_summary(counts, plan, E, cap),
        "measured_parts_per_layer_s": {"act_load": parts.act_load, "mig_load": parts.mig_load,
                                       "lat_gpu": parts.lat_gpu},
        "analytical_parts_per_layer_s": {"act_load": ana.act_load, "mig_load": ana.mig_load, "lat_gpu": ana.lat_gpu,
                                         "system": "configs/system_b200.yaml (measured peaks), k counted"},
        "h2d_gbs": mig_bytes / max(1e-9, parts.mig_load * N) / 1e9,
        "roofline": {"kernel": f"whole {N}-layer stack step (K3/K4 of every layer + router/permute/combine)",
                     "bound": "tensor", "achieved": flops / (ms / 1e3) / 1e12, "peak": pk["bf16_sus"],
                     "unit": "TFLOP/s", "frac": flops / (ms / 1e3) / 1e12 / pk["bf16_sus"], "traffic": None,
                     "peak_kind": f"bf16_tflops_sustained ({pk['src']}); burst {pk['bf16']}"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": stack.launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_stack_decode(args, cfg):
    """C3D: decode steps of the C3 stack (T tokens = T sequences x 1 token).
    Cold experts are fetched only if the layer's router sent them tokens
    (cox_fetch_experts, decided on the device), so the residency plan's hit
    ratio turns into PCIe bytes: the calibrated plan (eas.select_resident_experts
    on prototype histograms) is timed against eas.random_baseline residency."""
    import torch
    from paper_2605_17889_b200 import eas
    from paper_2605_17889_b200.synthetic import make_topic_tokens

    T, d, ff, E, k, mode, _, desc = cfg
    N = args.layers
    stack, wl, plan, cap, cal = _stack_setup(args, cfg, max(T, 4096))
    per_expert = stack.pool.nbytes_per_expert()

    def measure(tag):
        xs = [make_topic_tokens(wl, T, 1, seed=200 + i, device="cuda")[0] for i in range(args.steps + args.warmup)]
        counts = torch.zeros((N, E), dtype=torch.int32, device="cuda")
        tot = torch.zeros((N, E), dtype=torch.int64, device="cuda")
        fetched = 0.0
        for i in range(args.warmup):
            stack(xs[i], fetch="touched")
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            a.record(s)
            for i in range(args.steps):
                stack(xs[args.warmup + i], fetch="touched", counts_out=counts)
                tot += counts
                fetched += stack._fetched.sum()  # device tensor: no sync inside the timed loop
            b.record(s)
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        f = float(fetched) / 2.0 / args.steps  # cold experts fetched per step (W13 + W2 entries)
        hit = eas.hit_ratio_from_counts(tot.cpu().numpy().astype(float), stack.plan)
        return {"tag": tag, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3), "hit_ratio": hit,
                "cold_experts_fetched_per_step": f, "pcie_bytes_per_step": f * per_expert,
                "pcie_gbs": f * per_expert / (ms / 1e3) / 1e9, "clocks": clk.summary()}

    cal_res = measure("calibrated")
    cpu = parity = e2e = None
    if not args.no_cpu_baseline:
        cpu, parity = stack_parity_and_cpu(args, stack, T, mode)
    if not args.no_e2e:
        xs = [make_topic_tokens(wl, T, 1, seed=200 + i, device="cuda")[0] for i in range(args.steps)]
        e2e = stack_e2e(stack, xs, args.steps, "touched")
        e2e["residency"] = "calibrated"
    rnd_plan = eas.random_baseline(E, cap, N, seed=0)
    stack.set_residency(rnd_plan)
    rnd_res = measure("random_baseline")
    line = {
        "metric": metric_name("C3D"), "value": cal_res["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cal_res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic; topic-structured routing; decode tokens drawn per step from the topic mix",
        "config": {"workload": desc, "layers": N, "tokens_per_step": T, "d": d, "ff": ff, "E": E, "k": k,
                   "resident_per_layer": cap, "host_pool_experts": args.pool, "calibration": cal,
                   "fetch": "touched-only (cox_fetch_experts: cold experts with router count > 0)"},
        "calibrated": cal_res, "random_residency": rnd_res,
        "speedup_calibrated_vs_random": rnd_res["ms_per_step"] / cal_res["ms_per_step"],
        "roofline": {"kernel": "cold-expert fetch (PCIe, SM loads of mapped pinned memory)", "bound": "pcie",
                     "achieved": cal_res["pcie_gbs"], "peak": 55.0, "unit": "GB/s",
                     "frac": cal_res["pcie_gbs"] / 55.0, "traffic": None,
                     "peak_kind": "copy-engine H2D rate of the C3 prefill stack (configs/system_b200.yaml)"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": stack.launches_per_step_at(T, "touched") * args.steps,
        "clocks": cal_res["clocks"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default per config: ~4-6 s of device time; C3 5, C4D 2000)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-tokens", type=int, default=2048, help="token slice for the CPU-oracle baseline")
    ap.add_argument("--ref-tokens", type=int, default=512, help="tokens per step for --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--microbatch", type=int, default=0,
                    help="ablation: run the expert stage per micro-batch of this many tokens (not coalesced)")
    ap.add_argument("--layers", type=int, default=STACK_LAYERS, help="C3 stack depth")
    ap.add_argument("--pool", type=int, default=16, help="C3 distinct host-pool experts")
    ap.add_argument("--topics", type=int, default=8, help="C3 latent routing topics (= calibration clusters)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        # enough steps that the end-to-end pipeline's fill (first H2D) and drain
        # (last D2H) are a small share of the e2e number, within ~5 s per arm
        args.steps = {"C3": 5, "C3D": 5, "C4D": 2000, "C2D": 1000, "C1": 200}.get(args.config, 30)
        if args.impl == "reference":
            args.steps = 10
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.config == "C3":
        return run_stack(args, cfg)
    if args.config == "C3D":
        return run_stack_decode(args, cfg)

    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    T, d, ff, E, k, mode, shared_ff, desc = cfg

    from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
    from paper_2605_17889_b200.layer import MoELayer

    wts = make_layer_weights(E, d, ff, seed=0, device=dev, shared_ff=shared_ff)
    x = make_tokens(T, d, seed=1 + rank, device=dev)
    ep_used = None
    if ws > 1:
        from paper_2605_17889_b200.ep import EPMoELayer, FusedEPMoELayer
        want = os.environ.get("COX_EP", "auto")  # auto | fused | nccl
        layer = None
        if want in ("auto", "fused"):
            # probe: the fused peer-memory path must agree bit-for-bit with the NCCL path;
            # every rank reaches the same all_reduce whether or not its probe raised
            px = x[: min(T, 8192)].contiguous()
            a = EPMoELayer(wts, k, mode, dist.group.WORLD)(px).clone()
            why = "probe mismatch"
            try:
                probe = FusedEPMoELayer(wts, k, mode, dist.group.WORLD)
                b = probe(px).clone()
                probe.check()
                ok = torch.tensor([int(torch.equal(a, b))], device=dev)
                del probe
            except Exception as exc:  # noqa: BLE001
                ok = torch.tensor([0], device=dev)
                why = f"unavailable: {type(exc).__name__}"
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 1:
                layer = FusedEPMoELayer(wts, k, mode, dist.group.WORLD)
                ep_used = "fused NVLink peer-memory dispatch/combine (probe == NCCL path)"
            else:
                ep_used = f"nccl all_to_all (fused {why})"
        if layer is None:
            layer = EPMoELayer(wts, k, mode, dist.group.WORLD)
            ep_used = ep_used or "nccl all_to_all"
    else:
        layer = MoELayer(wts, k, mode)
    stream = torch.cuda.current_stream()
    graph = args.config in ("C4D", "C2D", "C1") and ws == 1  # small steps: CUDA-graph replay (launch-bound otherwise)
    if graph:
        replay, _ = layer.capture(x)
        step = lambda: replay()  # noqa: E731
    elif args.microbatch:
        step = lambda: layer.forward_microbatched(x, args.microbatch)  # noqa: E731
    else:
        step = lambda: layer(x)  # noqa: E731

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # --- device-resident throughput ------------------------------------------
    for _ in range(args.warmup):
        step()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    k3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    k4 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    layer.profile_events = None
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record(stream)
        for i in range(args.steps):
            layer.profile_events = {"k3": k3[i], "k4": k4[i]}
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        stop.record(stream)
        barrier()
    layer.profile_events = None
    ms_total = start.elapsed_time(stop)
    t_local = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_total = float(t_local.item())
    ms_step = ms_total / args.steps
    tokens_all = T * ws * args.steps
    value = tokens_all / (ms_total / 1e3)
    decode = args.config in ("C4D", "C2D")
    if graph and not decode:
        # prefill under graph replay: the per-kernel K3/K4 events come from an extra eager pass of the
        # same steps (outside the timed region; `value` is the graph-replay number above)
        for i in range(args.steps):
            layer.profile_events = {"k3": k3[i], "k4": k4[i]}
            layer(x)
        layer.profile_events = None
        barrier()
    k3_ms = sum(a.elapsed_time(b) for a, b in k3) / args.steps if not (decode or args.microbatch) else None
    k4_ms = sum(a.elapsed_time(b) for a, b in k4) / args.steps if not (decode or args.microbatch) else None

    # --- end-to-end through the public API with host buffers ------------------
    e2e = None
    if not args.no_e2e and not args.microbatch:
        # pinned host batches; each step = H2D of its tokens + expert stage + D2H of its output,
        # pipelined across steps (MoELayer / EP layer .run_host_batches, every rank its own batches)
        x_host = x.cpu().pin_memory()
        outs = [torch.empty((T, d), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        layer.run_host_batches([x_host] * 2, outs)
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        layer.run_host_batches([x_host] * args.steps, [outs[i % 2] for i in range(args.steps)])
        s1.record(stream)
        barrier()
        e_ms = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens_all / (float(e_ms.item()) / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": x.numel() * 2 * ws, "d2h_bytes_per_step": T * d * 2 * ws,
               "api": f"{type(layer).__name__}.run_host_batches (pinned host in/out, copies overlapped across steps"
                      + (", every rank its own batches)" if ws > 1 else ")")}
        del x_host, outs

    # --- per-stage breakdown (one extra step, not part of `value`; collective under EP) ---
    stages = layer.stage_times(x) if hasattr(layer, "stage_times") and not args.microbatch else None
    touched = int((layer.buffers(T, dev).counts > 0).sum().item()) if hasattr(layer, "buffers") else E
    # one more (untimed) step of the timed path: its output and routing are what the parity checks
    out_full = layer(x).clone() if not args.microbatch else None
    ep_info = None
    if ws > 1:
        # EP output for this rank's batch == the single-GPU layer on the same batch (bit for bit)
        exch = layer.exchange_bytes() if hasattr(layer, "exchange_bytes") else None
        barrier()
        ep_equal = None
        if rank == 0:
            ref_layer = MoELayer(wts, k, mode)
            ep_equal = bool(torch.equal(ref_layer(x), out_full))
            del ref_layer
            torch.cuda.empty_cache()
        ep_info = {"rank0_output_equals_single_gpu_layer": ep_equal}
        if exch is not None and stages:
            ep_info["rank0_nvlink_bytes"] = exch
            ep_info["rank0_dispatch_gbs"] = exch["dispatch"] / max(1e-9, stages["dispatch_nvlink"] / 1e3) / 1e9
            ep_info["rank0_combine_gbs"] = exch["combine"] / max(1e-9, stages["combine_nvlink"] / 1e3) / 1e9
        barrier()

    if rank == 0:
        pk = peaks()
        flops_k3 = 4.0 * T * k * d * ff
        flops_k4 = 2.0 * T * k * d * ff
        traffic = None
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists() and args.config == "C2":
            traffic = json.loads(tp.read_text()).get("grouped_gemm_kernel<0>", {}).get("dram_bytes_per_launch")
        if k3_ms:
            achieved = flops_k3 / (k3_ms / 1e3) / 1e12
            roof = {"kernel": "grouped_gemm_kernel<EPI_SWIGLU> (K3)" + (" on rank 0" if ws > 1 else ""),
                    "bound": "tensor", "achieved": achieved,
                    "peak": pk["bf16_sus"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_sus"], "traffic": traffic,
                    "traffic_note": "DRAM bytes per K3 launch from one ncu --set full capture (profiles/ncu_traffic.json)"
                    if traffic is not None else "no ncu --set full capture for this config (traffic measured on C2)",
                    "peak_kind": f"bf16_tflops_sustained ({pk['src']}); burst {pk['bf16']}", "k3_ms": k3_ms,
                    "k4_ms": k4_ms, "k4_tflops": flops_k4 / (k4_ms / 1e3) / 1e12}
        else:
            # decode / micro-batched: whole step vs the HBM bound of the weights it must read
            per_exp = 3 * d * ff * 2
            wbytes = touched * per_exp + (3 * d * shared_ff * 2 if shared_ff else 0)
            abytes = T * d * 2 * (2 + 2 * k)
            achieved = (wbytes + abytes) / (ms_step / 1e3) / 1e9
            roof = {"kernel": "whole expert stage (CUDA graph)" if decode else "whole expert stage (micro-batched)",
                    "bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                    "frac": achieved / pk["hbm"], "traffic": None,
                    "bytes_per_step": wbytes + abytes, "experts_touched": touched}
        cpu = None
        parity = None
        if not args.no_cpu_baseline and not args.microbatch:
            cpu, parity = cpu_baseline_and_parity(args, layer, wts, x, out_full, k, mode)
        if ep_info is not None and parity is not None:
            parity["ep"] = ep_info
            parity["pass"] = bool(parity["pass"] and ep_info["rank0_output_equals_single_gpu_layer"])
        line = assemble_line(args, cfg, ws, value, ms_step, pk, roof, stages, cpu, parity, e2e,
                             launches_per_step(layer, args.microbatch or T) * args.steps
                             * (-(-T // args.microbatch) if args.microbatch else 1),
                             clk.summary(), ep_used, touched, decode)
        print(json.dumps(line), flush=True)
    if ws > 1:
        if hasattr(layer, "check"):
            layer.check()
        dist.destroy_process_group()


def assemble_line(args, cfg, ws, value, ms_step, pk, roof, stages, cpu, parity, e2e, gpu_launches, clocks, ep_used,
                  touched, decode) -> dict:
    """The ONE JSON line of bench.py (rank 0).  `value` and `e2e` are whole-job
    tokens/s over all ws ranks; at ws > 1 `parity` carries the EP checks
    (rank 0's output == the single-GPU layer) and `stages_ms` the NVLink phases."""
    T, d, ff, E, k, mode, shared_ff, desc = cfg
    flops_layer = 6.0 * T * k * d * ff + 2.0 * T * d * E + (6.0 * T * d * shared_ff if shared_ff else 0.0)
    wgb = (touched * 3 * d * ff * 2 + 3 * d * shared_ff * 2) / 1e9
    if decode:
        l2_note = (f"expert weights read per step ({wgb:.2f} GB) > 126 MB L2, so every step streams them "
                   "from HBM; no flush")
    else:
        ws_gb = wgb + T * d * 2 * (3 + 2 * k) / 1e9 + T * k * ff * 2 / 1e9
        l2_note = (f"per-step working set {ws_gb:.2f} GB > 126 MB L2 (x {T * d * 2 / 1e9:.3f} GB, x_perm "
                   f"{T * k * d * 2 / 1e9:.3f} GB, h {T * k * ff * 2 / 1e9:.3f} GB, expert weights {wgb:.3f} GB); "
                   "no flush")
    desc_mb = f" [ABLATION: micro-batched, {args.microbatch} tokens per expert-stage launch]" if args.microbatch else ""
    tflops = flops_layer * ws / (ms_step / 1e3) / 1e12  # every rank runs one layer's worth of tokens
    return {
        "metric": metric_name(args.config),
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded N(0,1) tokens, nn.Linear-style U(+-1/sqrt(fan_in)) weights)",
        "config": {"workload": desc + desc_mb, "tokens_per_gpu": T, "global_batch_tokens": T * ws, "d": d, "ff": ff,
                   "E": E, "k": k, "routing": mode, "parallelism": f"ep{ws}" if ws > 1 else "single",
                   "ep_path": ep_used, "l2": l2_note},
        "layer_tflops": tflops,
        "frac_layer_of_bf16_sustained": tflops / ws / pk["bf16_sus"],
        "frac_layer_of_bf16_burst": tflops / ws / pk["bf16"],
        "roofline": roof,
        "stages_ms": stages,
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clocks,
    }


def launches_per_step(layer, T: int) -> int:
    lp = layer.launches_per_step
    return lp(T) if callable(lp) else lp


if __name__ == "__main__":
    main()
