"""Stratified multi-layer stack (resident + streamed cold experts) on the GPU."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2605_17889_b200.config import ResidencyPlan  # noqa: E402
from paper_2605_17889_b200.executor import StratifiedMoEStack, make_pool, make_router_weights  # noqa: E402
from paper_2605_17889_b200.synthetic import make_tokens, split_w13  # noqa: E402

DEV = "cuda"
N, E, d, ff, k, P = 4, 8, 256, 256, 2, 5


def _stack(plan):
    pool = make_pool(P, d, ff, seed=0, device=DEV)
    wg = make_router_weights(N, E, d, seed=7, device=DEV)
    return StratifiedMoEStack(N, wg, pool, k, plan, "mixtral"), pool, wg


def _bf16(a):
    return torch.from_numpy(a).to(torch.bfloat16).float().numpy()


def test_stack_matches_layerwise_oracle_and_is_residency_invariant():
    plan_a = ResidencyPlan(tuple((0, 1, 2) for _ in range(N)), 3)
    stack, pool, wg = _stack(plan_a)
    x = make_tokens(777, d, seed=3, device=DEV)
    out_a = stack(x, timeline=True).clone()
    torch.cuda.synchronize()
    rec = stack.timeline_records()
    assert any(r["res"] == "h2d" for r in rec) and all(r["dur"] >= 0 for r in rec)
    # residency must not change the function (same weights, same kernels, per-row results)
    plan_b = ResidencyPlan(tuple((e, (e + 3) % E) for e in range(N)), 2)
    stack.set_residency(plan_b)
    out_b = stack(x).clone()
    allres = ResidencyPlan(tuple(tuple(range(E)) for _ in range(N)), E)
    stack.set_residency(allres)
    out_c = stack(x).clone()
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b) and torch.equal(out_a, out_c)
    # layer-wise fp32 oracle with the same bf16 rounding between layers
    w1, w3 = split_w13(pool.w13)
    w1, w3, w2 = w1.float().numpy(), w3.float().numpy(), pool.w2.float().numpy()
    cur = x.float().cpu().numpy()
    wgn = wg.cpu().numpy()
    for l in range(N):
        sel = [(l * E + e) % P for e in range(E)]
        r = O.moe_layer(cur, wgn[l], w1[sel], w3[sel], w2[sel], k, 0)
        cur = _bf16(r["out"] + cur)  # residual stream (added inside K5 on the GPU)
    got = out_a.float().cpu().numpy()
    err = np.linalg.norm(got - cur) / np.linalg.norm(cur)
    assert err < 2e-2, err


def test_calibration_picks_the_hot_experts():
    plan0 = ResidencyPlan(tuple(() for _ in range(N)), 2)
    stack, pool, wg = _stack(plan0)
    # skewed tokens: a mean component along layer-0 router rows 5 and 6
    x = make_tokens(4096, d, seed=4, device=DEV).float()
    x += 3.0 * d ** 0.5 * (wg[0, 5] + wg[0, 6])
    x = x.to(torch.bfloat16)
    plan = stack.calibrate([x[:2048], x[2048:]], capacity_per_layer=2)
    assert plan.resident[0] == (5, 6)
    cm = stack.calibration_map.counts
    assert cm.sum() == N * 4096 * k
    out = stack(x)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()


def test_apply_strategy_from_orchestrator():
    from paper_2605_17889_b200.config import AllocationStrategy, Device
    stack, pool, wg = _stack(ResidencyPlan(tuple(() for _ in range(N)), 0))
    x = make_tokens(500, d, seed=5, device=DEV)
    ref = stack(x).clone()
    plan = stack.apply_strategy(AllocationStrategy((Device.GPU,) * 3, exp_r=5, exp_m=3, exp_c=0, m=4))
    assert all(len(r) == 5 for r in plan.resident)
    out = stack(x)
    torch.cuda.synchronize()
    assert torch.equal(ref, out)
    with pytest.raises(ValueError):
        stack.apply_strategy(AllocationStrategy((Device.GPU,) * 3, exp_r=4, exp_m=2, exp_c=2, m=4))


def test_touched_fetch_matches_stream_and_skips_untouched():
    """fetch="touched" (cox_fetch_experts after each router) gives the same bits
    as fetch="stream" and copies no bytes for cold experts the router left
    untouched (3 tokens x top-2: at most 6 of 8 experts touched per layer)."""
    pool = make_pool(P, d, ff, seed=0, device=DEV)
    wg = make_router_weights(N, E, d, seed=7, device=DEV)
    plan = ResidencyPlan(tuple((0, 1, 2) for _ in range(N)), 3)
    stack = StratifiedMoEStack(N, wg, pool, k, plan, "mixtral")
    for T in (3, 300):
        x = make_tokens(T, d, seed=4, device=DEV)
        a = stack(x, fetch="stream").clone()
        counts = torch.zeros((N, E), dtype=torch.int32, device=DEV)
        b = stack(x, fetch="touched", counts_out=counts).clone()
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        fetched = stack._fetched.cpu().numpy()
        c = counts.cpu().numpy()
        untouched = 0
        for l in range(N):
            for j, e in enumerate(stack.cold[l]):
                want = 1 if c[l, e] > 0 else 0
                untouched += 1 - want
                assert fetched[l, 2 * j] == want and fetched[l, 2 * j + 1] == want, (l, e)
        if T == 3:
            assert untouched > 0 and stack.fetched_cold_experts() < len(stack.cold[0])


def test_golden_c3_plan_runs_and_measured_parts():
    """The plan moeplan.planner.plan makes for C3 on configs/system_b200.yaml
    (committed golden, tests/test_reference_interop.py) drives a C3-shaped
    stack (3 layers), and measured_expert_stage_parts (costmodel.py:225-233's
    signature) returns hardware-measured parts next to the analytical row."""
    import json
    from pathlib import Path
    from paper_2605_17889_b200 import costmodel as CM
    from paper_2605_17889_b200.config import AllocationStrategy, BatchConfig, Device, ModelConfig, Phase
    from paper_2605_17889_b200.executor import measured_expert_stage_parts
    g = json.loads((Path(__file__).resolve().parent / "golden" / "reference_golden.json").read_text())["plan_c3_b200"]
    pf = g["prefill"]
    strat = AllocationStrategy(tuple(Device(p) for p in pf["placement"]), pf["exp_r"], pf["exp_m"], pf["exp_c"],
                               m=pf["m"])
    Nl, dd, fff = 3, 6144, 16384
    pool = make_pool(8, dd, fff, seed=0, device=DEV, residual_scale=(2.0 * Nl) ** -0.5)
    st = StratifiedMoEStack(Nl, make_router_weights(Nl, E, dd, seed=7, device=DEV), pool, k,
                            ResidencyPlan(tuple(() for _ in range(Nl)), 0), "mixtral", pool_map=lambda l, e: e)
    plan = st.apply_strategy(strat)
    assert all(len(r) == pf["exp_r"] for r in plan.resident) and all(len(c) == pf["exp_m"] for c in st.cold)
    out = st(make_tokens(8192, dd, seed=5, device=DEV), fetch="stream")
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    del st, pool
    torch.cuda.empty_cache()
    model = ModelConfig(56, dd, fff, 8, 2, 2)
    batch = BatchConfig(2, 4096, 0)
    ph = Phase.prefill(4096)
    meas = measured_expert_stage_parts(strat, ph, CM.load_system_spec(CM.B200_SYSTEM_YAML), model, batch)
    ana = CM.expert_stage_parts(strat, ph, CM.load_system_spec(CM.B200_SYSTEM_YAML), model, batch,
                                count_top_k=True)
    assert meas.act_load == 0.0 and meas.lat_cpu == 0.0 and meas.return_store == 0.0
    # 4 cold experts x 604 MB over PCIe; the analytical row charges the same bytes at 55 GB/s
    assert 0.5 < meas.mig_load / ana.mig_load < 2.0, (meas, ana)
    assert 0.2 < meas.lat_gpu / ana.lat_gpu < 5.0, (meas, ana)
