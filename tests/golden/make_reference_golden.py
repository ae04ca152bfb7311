"""Golden values produced by the REAL reference package (moeplan) in the build
container, committed as reference_golden.json so the GPU box (which has no
/root/reference) and the CPU suite can pin this repo's restatements:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reference_golden.py

Covers the hot-path rows of SURVEY.md §8a: expert_stage_parts (a6, incl. the
sweep golden `expert_s` of tests/data/sweep_coalesced_membound.csv),
sorted_share_profile (a5), select_resident_experts (a10), random_baseline and
hit_ratio over a synthetic trace (a11), vram resident term (a9).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from moeplan import configio, eas  # noqa: E402
from moeplan.costmodel import AllocationStrategy, expert_stage_parts, vram_usage  # noqa: E402
from moeplan.hardware import Device, DeviceSpec, LinkSpec, SystemSpec  # noqa: E402
from moeplan.planner import PlanRequest, sweep_microbatch  # noqa: E402
from moeplan.planner import plan as planner_plan  # noqa: E402
from moeplan.workload import BatchConfig, ModelConfig, Phase, PhaseKind  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_golden.json"


def sysd(s):
    return {"gpu": [s.gpu.mem_bandwidth, s.gpu.peak_compute, s.gpu.mem_capacity],
            "cpu": [s.cpu.mem_bandwidth, s.cpu.peak_compute, s.cpu.mem_capacity],
            "link": [s.link.bandwidth, s.link.duplex, s.link.efficiency]}


def main():
    G, C = Device.GPU, Device.CPU
    rng = np.random.default_rng(0)
    systems = {
        "b200like": SystemSpec(DeviceSpec("gpu", 8e12, 2.25e15, 180e9), DeviceSpec("cpu", 3e11, 2e12, 1e12),
                               LinkSpec(55e9)),
        "toy": SystemSpec(DeviceSpec("gpu", 100.0, 1000.0, 1e12), DeviceSpec("cpu", 50.0, 200.0, 1e12),
                          LinkSpec(10.0)),
    }
    models = {
        "mixtral8x7b": ModelConfig(32, 4096, 14336, 8, 2, 2),
        "mixtral8x22b": ModelConfig(56, 6144, 16384, 8, 2, 2),
        "dsv2lite": ModelConfig(26, 2048, 1408, 64, 6, 2),
        "toy": ModelConfig(1, 2, 4, 2, 1, 2),
    }
    batches = {"b64x4096": BatchConfig(64, 4096, 0), "b2x2": BatchConfig(2, 2, 0), "b8x32": BatchConfig(8, 32, 4)}
    cases = []
    for sname, mname, bname, part, m, coalesced, amap_seed in [
        ("b200like", "mixtral8x7b", "b64x4096", (8, 0, 0), 64, True, None),
        ("b200like", "mixtral8x22b", "b64x4096", (4, 4, 0), 64, True, None),
        ("b200like", "mixtral8x22b", "b64x4096", (4, 4, 0), 16, False, 3),
        ("b200like", "dsv2lite", "b64x4096", (40, 24, 0), 32, True, 5),
        ("toy", "toy", "b2x2", (1, 0, 1), 1, True, None),
        ("toy", "toy", "b2x2", (0, 1, 1), 2, True, 7),
        ("b200like", "mixtral8x7b", "b8x32", (2, 2, 4), 2, False, 9),
    ]:
        model = models[mname]
        strat = AllocationStrategy((G, C, G), *part, m=m)
        amap = None
        counts = None
        if amap_seed is not None:
            counts = np.random.default_rng(amap_seed).integers(1, 100, size=(3, model.experts_per_layer)).astype(float)
            amap = eas.ActivationMap(counts)
        phase = Phase.prefill(batches[bname].input_len)
        parts = expert_stage_parts(strat, phase, systems[sname], model, batches[bname], amap, coalesced)
        vram = vram_usage(strat, systems[sname], model, batches[bname], PhaseKind.PREFILL)
        cases.append({"system": sname, "model": mname, "batch": bname, "partition": part, "m": m,
                      "coalesced": coalesced, "counts": None if counts is None else counts.tolist(),
                      "parts": [parts.act_load, parts.mig_load, parts.lat_gpu, parts.lat_cpu, parts.return_store],
                      "resident_expert_bytes": vram.resident_expert_bytes,
                      "share_profile": None if amap is None else amap.sorted_share_profile().tolist()})

    # the committed sweep golden (tests/data/sweep_coalesced_membound.csv)
    s = configio.load_system_spec(REF / "configs/system_rtx6000ada.yaml")
    mdl = configio.load_model_config(REF / "configs/model_sweep_membound.yaml")
    bt = configio.load_batch_config(REF / "configs/batch_sweep_membound.yaml")
    req = PlanRequest(system=s, model=mdl, batch=bt)
    rows = sweep_microbatch(req, "coalesced")
    rows_mb = sweep_microbatch(req, "microbatched")
    sweep = {"system": sysd(s), "model": [mdl.num_layers, mdl.hidden_dim, mdl.expert_dim, mdl.experts_per_layer,
                                          mdl.top_k, mdl.dtype_bytes],
             "batch": [bt.batch_size, bt.input_len, bt.output_len], "m": [r.m for r in rows],
             "expert_s": [r.expert_s for r in rows], "expert_s_microbatched": [r.expert_s for r in rows_mb]}

    residency = []
    for counts, cap in [([[5.0, 1.0, 9.0, 9.0]], 2), ([[5.0, 1.0, 9.0, 9.0]], 0), ([[5.0, 1.0, 9.0, 9.0]], 4),
                        (rng.integers(0, 5, size=(6, 8)).astype(float).tolist(), 3),
                        (rng.integers(0, 1000, size=(26, 64)).astype(float).tolist(), 17)]:
        plan = eas.select_resident_experts(eas.ActivationMap(np.asarray(counts)), cap)
        residency.append({"counts": counts, "capacity": cap, "resident": [list(x) for x in plan.resident]})

    randoms = []
    for E, cap, L, seed in [(8, 4, 3, 0), (64, 16, 4, 5), (8, 0, 2, 1)]:
        randoms.append({"args": [E, cap, L, seed], "resident": [list(x) for x in eas.random_baseline(E, cap, L, seed).resident]})

    # acceptance-5-style hit ratio: synthetic trace -> stratified map -> plan -> hit ratio
    trace = eas.generate_synthetic_trace(2000, 16, 4, 64, 8, 12, 1.2, seed=3)
    cfg = eas.StratificationConfig(num_clusters=12, sample_ratio=0.05, seed=3)
    amap = eas.stratified_activation_map(trace, cfg)
    plan = eas.select_resident_experts(amap, 16)
    full_counts = np.zeros((trace.num_layers, trace.experts_per_layer))
    np.add.at(full_counts, (trace.layer_idx, trace.expert_idx), trace.token_counts)
    hit = {"trace_counts": full_counts.tolist(), "probe_counts": amap.counts.tolist(),
           "resident": [list(x) for x in plan.resident], "capacity": 16, "hit_ratio": eas.hit_ratio(trace, plan),
           "random_hit_ratio": eas.hit_ratio(trace, eas.random_baseline(64, 16, 4, 0))}

    # prototype selection (cluster + select_prototypes) on a small trace
    ptrace = eas.generate_synthetic_trace(600, 12, 2, 16, 2, 5, 1.2, seed=11)
    pcfg = eas.StratificationConfig(num_clusters=5, sample_ratio=0.04, seed=11)
    pcl = eas.cluster(ptrace, pcfg)
    protos = {"embeddings": ptrace.embeddings.tolist(), "num_clusters": 5, "sample_ratio": 0.04, "seed": 11,
              "assignments": pcl.assignments.tolist(), "centroids": pcl.centroids.tolist(),
              "inertia": list(pcl.iteration_inertia), "prototypes": eas.select_prototypes(pcl, 0.04, 11)}

    # planner.plan on this repo's B200 system triple (configs/system_b200.yaml, the reference's YAML schema)
    repo = Path(__file__).resolve().parents[2]
    bsys = configio.load_system_spec(repo / "paper_2605_17889_b200" / "configs" / "system_b200.yaml")
    c3 = ModelConfig(56, 6144, 16384, 8, 2, 2)
    c3b = BatchConfig(64, 4096, 16)
    pl = planner_plan(PlanRequest(system=bsys, model=c3, batch=c3b))

    def strat(st):
        return {"placement": [p.value for p in st.placement], "exp_r": st.exp_r, "exp_m": st.exp_m,
                "exp_c": st.exp_c, "m": st.m}
    plan_c3 = {"system": sysd(bsys), "model": [56, 6144, 16384, 8, 2, 2], "batch": [64, 4096, 16],
               "prefill": strat(pl.prefill_strategy), "decode": strat(pl.decode_strategy),
               "vram_prefill_resident_bytes": pl.vram_prefill.resident_expert_bytes}

    OUT.write_text(json.dumps({"plan_c3_b200": plan_c3, "prototypes": protos, "systems": {k: sysd(v) for k, v in systems.items()},
                               "models": {k: [v.num_layers, v.hidden_dim, v.expert_dim, v.experts_per_layer, v.top_k,
                                              v.dtype_bytes] for k, v in models.items()},
                               "batches": {k: [v.batch_size, v.input_len, v.output_len] for k, v in batches.items()},
                               "expert_stage_cases": cases, "sweep": sweep, "residency": residency,
                               "random_baseline": randoms, "hit_ratio": hit}, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
