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

from dataclasses import dataclass

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


# ---------------------------------------------------------------------------
# Prototype selection (which batches calibrate the map).  Restated from the
# reference so the GPU box needs no moeplan; pinned bit-for-bit against it in
# tests/test_host.py (tests/golden/reference_golden.json).


@dataclass(frozen=True)
class Clustering:
    """eas.Clustering (eas.py:225-240): assignments, centroids, the clustered
    points and the inertia after every assignment step."""
    assignments: np.ndarray
    centroids: np.ndarray
    embeddings: np.ndarray
    iteration_inertia: tuple

    @property
    def num_clusters(self) -> int:
        return self.centroids.shape[0]


def _nearest(points: np.ndarray, centroids: np.ndarray):
    """eas._nearest (eas.py:256-260): nearest centroid (ties -> lower id) and its squared distance."""
    d2 = ((points[:, None, :] - centroids[None, :, :]) ** 2).sum(axis=2)
    assign = d2.argmin(axis=1)
    return assign, d2[np.arange(len(points)), assign]


def _farthest_point_seeds(x: np.ndarray, k: int, seed: int) -> np.ndarray:
    """eas._farthest_point_seeds (eas.py:263-272), same RNG stream."""
    rng = np.random.default_rng(seed)
    first = int(rng.integers(len(x)))
    chosen = [first]
    min_d2 = ((x - x[first]) ** 2).sum(axis=1)
    for _ in range(k - 1):
        nxt = int(min_d2.argmax())
        chosen.append(nxt)
        min_d2 = np.minimum(min_d2, ((x - x[nxt]) ** 2).sum(axis=1))
    return x[chosen].copy()


def cluster(embeddings, num_clusters: int, seed: int = 0, max_iters: int = 100, tolerance: float = 1e-6) -> Clustering:
    """eas.cluster (eas.py:275-317): Lloyd iterations from farthest-point seeds;
    empty clusters reseeded with the point farthest from its centroid.
    Defaults = StratificationConfig's max_kmeans_iters / tolerance."""
    x = np.asarray(embeddings, dtype=np.float64)
    k = int(num_clusters)
    if k < 1 or k > len(x):
        raise ValueError("num_clusters must be in 1..number of samples")
    centroids = _farthest_point_seeds(x, k, seed)
    inertia_log = []
    assign = np.zeros(len(x), dtype=np.int64)
    for _ in range(max_iters):
        assign, d2 = _nearest(x, centroids)
        for c in range(k):
            if not np.any(assign == c):
                outlier = int(d2.argmax())
                centroids = centroids.copy()
                centroids[c] = x[outlier]
                assign[outlier] = c
                d2 = d2.copy()
                d2[outlier] = 0.0
        inertia_log.append(float(d2.sum()))
        new_centroids = centroids.copy()
        for c in range(k):
            members = assign == c
            if np.any(members):
                new_centroids[c] = x[members].mean(axis=0)
        shift = float(np.sqrt(((new_centroids - centroids) ** 2).sum(axis=1)).max())
        centroids = new_centroids
        if shift < tolerance:
            break
    assign, d2 = _nearest(x, centroids)
    inertia_log.append(float(d2.sum()))
    return Clustering(assignments=assign, centroids=centroids, embeddings=x, iteration_inertia=tuple(inertia_log))


def select_prototypes(clustering: Clustering, sample_ratio: float) -> list:
    """eas.select_prototypes (eas.py:320-339): per cluster the
    round(sample_ratio * n_k) members nearest its centroid (>= 1 per non-empty
    cluster), ties by index; sorted sample ids."""
    if not (0.0 < sample_ratio <= 1.0):
        raise ValueError("sample_ratio must be in (0, 1]")
    chosen = []
    for c in range(clustering.num_clusters):
        members = np.flatnonzero(clustering.assignments == c)
        if len(members) == 0:
            continue
        quota = max(1, int(sample_ratio * len(members) + 0.5))
        d2 = ((clustering.embeddings[members] - clustering.centroids[c]) ** 2).sum(axis=1)
        order = np.lexsort((members, d2))
        chosen.extend(int(i) for i in members[order[:quota]])
    return sorted(chosen)


def random_hit_ratio(counts, experts_per_layer: int, capacity: int, seeds=range(50)) -> float:
    """Mean hit ratio of eas.random_baseline plans over `seeds` (the CLI's
    hitratio baseline averages 50 plans, cli.py:442-448)."""
    counts = np.asarray(counts, dtype=float)
    return float(np.mean([hit_ratio_from_counts(counts, random_baseline(experts_per_layer, capacity,
                                                                        counts.shape[0], s)) for s in seeds]))
