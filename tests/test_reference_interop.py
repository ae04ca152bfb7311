"""Drop-in check against the REAL reference objects (build container only):
the executor-side API accepts moeplan's own instances and reproduces moeplan."""
import numpy as np
import pytest

from paper_2605_17889_b200 import costmodel as CM
from paper_2605_17889_b200 import eas


def test_expert_stage_parts_accepts_reference_objects(moeplan):
    from moeplan.costmodel import AllocationStrategy, expert_stage_parts
    from moeplan.eas import ActivationMap
    from moeplan.hardware import Device, DeviceSpec, LinkSpec, SystemSpec
    from moeplan.workload import BatchConfig, ModelConfig, Phase
    system = SystemSpec(DeviceSpec("gpu", 6.5e12, 1.36e15, 183e9), DeviceSpec("cpu", 3e11, 2e12, 1e12), LinkSpec(55e9))
    model = ModelConfig(56, 6144, 16384, 8, 2, 2)
    batch = BatchConfig(64, 4096, 0)
    amap = ActivationMap(np.arange(1, 1 + 56 * 8, dtype=float).reshape(56, 8))
    for part in [(8, 0, 0), (4, 4, 0), (2, 3, 3)]:
        strat = AllocationStrategy((Device.GPU, Device.CPU, Device.GPU), *part, m=16)
        ph = Phase.prefill(4096)
        ref = expert_stage_parts(strat, ph, system, model, batch, amap)
        ours = CM.expert_stage_parts(strat, ph, system, model, batch, amap)
        assert (ours.act_load, ours.mig_load, ours.lat_gpu, ours.lat_cpu, ours.return_store) == \
               (ref.act_load, ref.mig_load, ref.lat_gpu, ref.lat_cpu, ref.return_store)


def test_residency_on_reference_map_and_trace(moeplan):
    from moeplan import eas as R
    trace = R.generate_synthetic_trace(1500, 8, 3, 16, 2, 5, 1.1, seed=9)
    amap = R.stratified_activation_map(trace, R.StratificationConfig(5, 0.1, seed=9))
    for cap in (0, 3, 8, 16):
        assert eas.select_resident_experts(amap, cap).resident == R.select_resident_experts(amap, cap).resident
        plan = R.select_resident_experts(amap, cap)
        counts = np.zeros((3, 16))
        np.add.at(counts, (trace.layer_idx, trace.expert_idx), trace.token_counts)
        assert eas.hit_ratio_from_counts(counts, plan) == pytest.approx(R.hit_ratio(trace, plan), abs=0, rel=1e-15)


def test_planner_plan_drives_residency(moeplan):
    """moeplan.planner.plan on a B200 system spec -> exp_r/exp_m -> our residency
    selection (the executor's apply_strategy uses exactly this rule)."""
    from moeplan.hardware import DeviceSpec, LinkSpec, SystemSpec
    from moeplan.planner import PlanRequest, plan
    from moeplan.workload import BatchConfig, ModelConfig
    from moeplan.eas import ActivationMap
    b2 = CM.b200_system()
    system = SystemSpec(DeviceSpec("gpu", b2.gpu.mem_bandwidth, b2.gpu.peak_compute, b2.gpu.mem_capacity),
                        DeviceSpec("cpu", 3e11, 2e12, 1e12), LinkSpec(55e9))
    model = ModelConfig(56, 6144, 16384, 8, 2, 2)
    amap = ActivationMap(np.random.default_rng(0).integers(1, 100, size=(56, 8)).astype(float))
    p = plan(PlanRequest(system=system, model=model, batch=BatchConfig(64, 4096, 16), activation_map=amap))
    s = p.prefill_strategy
    assert s.exp_r + s.exp_m + s.exp_c == 8 and s.exp_r >= 1
    ours = eas.select_resident_experts(amap, s.exp_r)
    assert all(len(layer) == s.exp_r for layer in ours.resident)
    # the hottest experts of every layer are the resident ones
    for layer, res in enumerate(ours.resident):
        order = np.argsort(-amap.counts[layer], kind="stable")[: s.exp_r]
        assert set(res) == set(int(e) for e in order)


def test_b200_system_yaml_replans_c3(moeplan):
    """configs/system_b200.yaml (the reference's YAML schema, measured B200
    numbers) is read identically by moeplan.configio and by costmodel.
    load_system_spec, and moeplan.planner.plan on it reproduces the committed
    C3 plan that tests/test_gpu_stack.py runs on the GPU."""
    import json
    from pathlib import Path
    from moeplan import configio
    from moeplan.planner import PlanRequest, plan
    from moeplan.workload import BatchConfig, ModelConfig
    ref = configio.load_system_spec(CM.B200_SYSTEM_YAML)
    ours = CM.load_system_spec(CM.B200_SYSTEM_YAML)
    for a, b in ((ref.gpu, ours.gpu), (ref.cpu, ours.cpu)):
        assert (a.mem_bandwidth, a.peak_compute, a.mem_capacity) == (b.mem_bandwidth, b.peak_compute, b.mem_capacity)
    assert (ref.link.bandwidth, ref.link.duplex, ref.link.efficiency) == \
           (ours.link.bandwidth, ours.link.duplex, ours.link.efficiency)
    g = json.loads((Path(__file__).resolve().parent / "golden" / "reference_golden.json").read_text())["plan_c3_b200"]
    p = plan(PlanRequest(system=ref, model=ModelConfig(*g["model"]), batch=BatchConfig(*g["batch"])))
    for ph, st in (("prefill", p.prefill_strategy), ("decode", p.decode_strategy)):
        assert [x.value for x in st.placement] == g[ph]["placement"]
        assert (st.exp_r, st.exp_m, st.exp_c, st.m) == (g[ph]["exp_r"], g[ph]["exp_m"], g[ph]["exp_c"], g[ph]["m"])
    # the prefill partition runs on the B200 executor (no CPU experts); the
    # decode partition's CPU experts are replaced by device-side touched-only
    # fetches (executor.StratifiedMoEStack, fetch="touched")
    assert g["prefill"]["exp_c"] == 0
