"""Host-side logic vs the reference's own values (tests/golden/reference_golden.json,
produced by the real moeplan; see tests/golden/make_reference_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2605_17889_b200 import config as C
from paper_2605_17889_b200 import costmodel as CM
from paper_2605_17889_b200 import eas

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "reference_golden.json").read_text())


def _system(d):
    return CM.SystemSpec(CM.DeviceSpec("gpu", *d["gpu"]), CM.DeviceSpec("cpu", *d["cpu"]), CM.LinkSpec(*d["link"]))


def _model(v):
    return C.ModelConfig(*v)


def _batch(v):
    return C.BatchConfig(*v)


@pytest.mark.parametrize("i", range(len(GOLD["expert_stage_cases"])))
def test_expert_stage_parts_bitexact_vs_reference(i):
    c = GOLD["expert_stage_cases"][i]
    model = _model(GOLD["models"][c["model"]])
    batch = _batch(GOLD["batches"][c["batch"]])
    system = _system(GOLD["systems"][c["system"]])
    strat = C.AllocationStrategy((C.Device.GPU, C.Device.CPU, C.Device.GPU), *c["partition"], m=c["m"])
    amap = C.ActivationMap(np.asarray(c["counts"])) if c["counts"] is not None else None
    parts = CM.expert_stage_parts(strat, C.Phase.prefill(batch.input_len), system, model, batch, amap, c["coalesced"])
    got = [parts.act_load, parts.mig_load, parts.lat_gpu, parts.lat_cpu, parts.return_store]
    assert got == c["parts"]
    assert CM.resident_expert_bytes(strat, model) == c["resident_expert_bytes"]
    if amap is not None:
        assert amap.sorted_share_profile().tolist() == c["share_profile"]


def test_sweep_golden_expert_s():
    """tests/data/sweep_coalesced_membound.csv: expert_s = 1.4199466666666667e-05 for every m,
    and the micro-batched refetch rows (planner.sweep_microbatch)."""
    sw = GOLD["sweep"]
    system, model, batch = _system(sw["system"]), _model(sw["model"]), _batch(sw["batch"])
    for m, exp_c, exp_mb in zip(sw["m"], sw["expert_s"], sw["expert_s_microbatched"]):
        strat = C.AllocationStrategy((C.Device.GPU,) * 3, model.experts_per_layer, 0, 0, m=m)
        ph = C.Phase.prefill(batch.input_len)
        pc = CM.expert_stage_parts(strat, ph, system, model, batch, None, True)
        pm = CM.expert_stage_parts(strat, ph, system, model, batch, None, False)
        assert model.num_layers * pc.t_comp == exp_c
        assert model.num_layers * pm.t_comp == exp_mb
    assert sw["expert_s"][0] == 1.4199466666666667e-05


def test_top_k_count_fix_doubles_top2_flops():
    model = C.ModelConfig(32, 4096, 14336, 8, 2, 2)
    batch = C.BatchConfig(64, 4096, 0)
    system = CM.SystemSpec(CM.DeviceSpec("g", 8e15, 1e12, 1e12), CM.DeviceSpec("c", 1.0, 1.0, 1.0), CM.LinkSpec(1.0))
    strat = C.AllocationStrategy((C.Device.GPU,) * 3, 8, 0, 0, m=64)
    ph = C.Phase.prefill(4096)
    a = CM.expert_stage_parts(strat, ph, system, model, batch)
    b = CM.expert_stage_parts(strat, ph, system, model, batch, count_top_k=True)
    assert b.lat_gpu == pytest.approx(2 * a.lat_gpu)  # compute-bound system


@pytest.mark.parametrize("i", range(len(GOLD["residency"])))
def test_select_resident_experts_vs_reference(i):
    c = GOLD["residency"][i]
    plan = eas.select_resident_experts(C.ActivationMap(np.asarray(c["counts"], float)), c["capacity"])
    assert [list(x) for x in plan.resident] == c["resident"]


@pytest.mark.parametrize("i", range(len(GOLD["random_baseline"])))
def test_random_baseline_vs_reference(i):
    c = GOLD["random_baseline"][i]
    assert [list(x) for x in eas.random_baseline(*c["args"]).resident] == c["resident"]


def test_hit_ratio_and_calibrator_vs_reference():
    h = GOLD["hit_ratio"]
    cal = eas.Calibrator(len(h["probe_counts"]), len(h["probe_counts"][0]))
    for layer, row in enumerate(h["probe_counts"]):
        cal.observe(layer, np.asarray(row))
    plan = cal.residency(h["capacity"])
    assert [list(x) for x in plan.resident] == h["resident"]
    assert eas.hit_ratio_from_counts(np.asarray(h["trace_counts"]), plan) == h["hit_ratio"]
    rnd = eas.random_baseline(64, 16, 4, 0)
    assert eas.hit_ratio_from_counts(np.asarray(h["trace_counts"]), rnd) == h["random_hit_ratio"]
    assert h["hit_ratio"] > h["random_hit_ratio"] + 0.3


def test_cluster_and_prototypes_vs_reference():
    """Prototype selection for calibration: eas.cluster (Lloyd + farthest-point
    seeds) and eas.select_prototypes restated bit-for-bit (eas.py:263-339)."""
    g = GOLD["prototypes"]
    cl = eas.cluster(np.asarray(g["embeddings"]), g["num_clusters"], seed=g["seed"])
    assert cl.assignments.tolist() == g["assignments"]
    assert cl.centroids.tolist() == g["centroids"]
    assert list(cl.iteration_inertia) == g["inertia"]
    assert eas.select_prototypes(cl, g["sample_ratio"]) == g["prototypes"]


def test_mirror_validation_matches_reference_rules():
    with pytest.raises(ValueError):
        C.ModelConfig(1, 8, 8, 4, 5)
    with pytest.raises(ValueError):
        C.ModelConfig(1, 8, 8, 4, 2, dtype_bytes=3)
    with pytest.raises(ValueError):
        C.AllocationStrategy((C.Device.GPU,) * 3, -1, 0, 0, 1)
    with pytest.raises(ValueError):
        C.AllocationStrategy((C.Device.GPU,) * 3, 1, 0, 0, 1, coalesced_expert_batch=False)
    with pytest.raises(ValueError):
        C.check_partition(C.AllocationStrategy((C.Device.GPU,) * 3, 4, 2, 2, 1), C.ModelConfig(1, 8, 8, 8, 2))
    C.check_partition(C.AllocationStrategy((C.Device.GPU,) * 3, 4, 4, 0, 1), C.ModelConfig(1, 8, 8, 8, 2))
    with pytest.raises(ValueError):
        C.Phase(C.PhaseKind.DECODE, 2, 0)
    with pytest.raises(ValueError):
        C.ResidencyPlan(((1, 1),), 2)


def test_capacity_per_layer():
    model = C.ModelConfig(56, 6144, 16384, 8, 2, 2)
    per = CM.per_expert_weight_bytes(model)
    assert per == 3 * 2 * 6144 * 16384
    assert CM.capacity_per_layer(model, 4 * per * 56 + 1) == 4
    assert CM.capacity_per_layer(model, 4 * per * 56 - 1) == 3
    assert CM.capacity_per_layer(model, 0) == 0
    assert CM.capacity_per_layer(model, 1e15) == 8


def test_b200_system_yaml_loads():
    """configs/system_b200.yaml parses into the reference's SystemSpec shape
    (the same YAML is read by moeplan.configio in tests/test_reference_interop.py)."""
    s = CM.load_system_spec(CM.B200_SYSTEM_YAML)
    assert s.gpu.mem_bandwidth == 6.4528e12 and s.gpu.peak_compute == 1430.7e12
    assert s.link.bandwidth == 55e9 and s.link.duplex and s.link.efficiency == 1.0
    g = GOLD["plan_c3_b200"]["system"]
    assert [s.gpu.mem_bandwidth, s.gpu.peak_compute, s.gpu.mem_capacity] == g["gpu"]
    assert [s.cpu.mem_bandwidth, s.cpu.peak_compute, s.cpu.mem_capacity] == g["cpu"]
