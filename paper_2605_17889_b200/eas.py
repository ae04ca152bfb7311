"""Expert-aware stratification on the B200 path: which experts stay pinned in HBM.

The reference builds an activation map by probing prototype samples of a
routing trace (eas.probe, eas.py:346-356) and keeps the top-`capacity`
experts per layer (eas.select_resident_experts, eas.py:364-374).  Here the map
is calibrated from the REAL router: K1 (cox_router_topk) emits a per-expert
token histogram for every batch it routes, and `Calibrator` accumulates those
histograms over prototype batches into the same (num_layers, E) ActivationMap.
Residency selection, hit ratio and the random baseline restate the reference
algorithms exactly (pinned against the reference in tests/).
"""
from __future__ import annotations

import numpy as np

from .config import ActivationMap, ResidencyPlan


def select_resident_experts(activation_map, capacity_per_layer: int) -> ResidencyPlan:
    """eas.select_resident_experts (eas.py:364-374): per layer the `capacity`
    highest-count experts, ties toward the lower index, returned sorted."""
    if capacity_per_layer < 0:
        raise ValueError("capacity_per_layer must be >= 0")
    counts = np.asarray(activation_map.counts, dtype=float)
    cap = min(capacity_per_layer, counts.shape[1])
    layers = []
    for layer in range(counts.shape[0]):
        order = np.argsort(-counts[layer], kind="stable")
        layers.append(tuple(sorted(int(e) for e in order[:cap])))
    return ResidencyPlan(resident=tuple(layers), capacity_per_layer=capacity_per_layer)


def random_baseline(experts_per_layer: int, capacity: int, num_layers: int, seed: int) -> ResidencyPlan:
    """eas.random_baseline (eas.py:391-406), same RNG stream."""
    if not (0 <= capacity <= experts_per_layer):
        raise ValueError("capacity must be in 0..experts_per_layer")
    rng = np.random.default_rng(seed)
    layers = tuple(
        tuple(sorted(int(e) for e in rng.permutation(experts_per_layer)[:capacity])) for _ in range(num_layers))
    return ResidencyPlan(resident=layers, capacity_per_layer=capacity)


def hit_ratio_from_counts(counts, plan) -> float:
    """Token-weighted fraction of routed (token, expert) pairs that land on a
    resident expert — eas.hit_ratio's definition (eas.py:377-388) evaluated on
    per-layer routed-token histograms instead of trace events."""
    counts = np.asarray(counts, dtype=float)
    if counts.ndim != 2 or plan.num_layers != counts.shape[0]:
        raise ValueError("plan and counts disagree on the number of layers")
    total = counts.sum()
    if total == 0:
        raise ValueError("no routed tokens")
    mask = np.zeros(counts.shape, dtype=bool)
    for layer, experts in enumerate(plan.resident):
        mask[layer, list(experts)] = True
    return float(counts[mask].sum() / total)


class Calibrator:
    """Accumulates K1 expert histograms (GPU router) into an ActivationMap.

    `observe(layer, counts)` takes the int32 [E] histogram the router produced
    for one batch (the per-batch analogue of eas.probe over prototype samples);
    `activation_map()` returns the (num_layers, E) float64 counts.
    """

    def __init__(self, num_layers: int, experts_per_layer: int):
        if num_layers < 1 or experts_per_layer < 1:
            raise ValueError("num_layers and experts_per_layer must be >= 1")
        self.counts = np.zeros((num_layers, experts_per_layer), dtype=np.float64)

    def observe(self, layer: int, counts) -> None:
        c = counts.detach().cpu().numpy() if hasattr(counts, "detach") else np.asarray(counts)
        if c.shape != (self.counts.shape[1],):
            raise ValueError("histogram length must equal experts_per_layer")
        if np.any(c < 0):
            raise ValueError("counts must be non-negative")
        self.counts[layer] += c

    def activation_map(self) -> ActivationMap:
        return ActivationMap(self.counts.copy())

    def residency(self, capacity_per_layer: int) -> ResidencyPlan:
        return select_resident_experts(self.activation_map(), capacity_per_layer)
