"""Mirrors of the reference's configuration / orchestration types.

The executor accepts either these classes or the reference's own objects
(duck-typed on the same field names), so a moeplan user can hand over the
exact `ModelConfig`, `BatchConfig`, `AllocationStrategy`, `ActivationMap` and
`ResidencyPlan` instances the planner produced.

Field names, validation rules and error types follow:
  ModelConfig          pkg/src/moeplan/workload.py:38-56
  BatchConfig          workload.py:59-73
  Phase                workload.py:76-107
  AllocationStrategy   costmodel.py:45-89 (+ _check_partition :92-97)
  ExpertStageParts     costmodel.py:199-222
  ActivationMap        eas.py:65-111
  ResidencyPlan        eas.py:133-154
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np


@dataclass(frozen=True)
class ModelConfig:
    num_layers: int
    hidden_dim: int
    expert_dim: int
    experts_per_layer: int
    top_k: int
    dtype_bytes: int = 2

    def __post_init__(self) -> None:
        for field in ("num_layers", "hidden_dim", "expert_dim", "experts_per_layer"):
            if getattr(self, field) < 1:
                raise ValueError(f"{field} must be >= 1")
        if not (1 <= self.top_k <= self.experts_per_layer):
            raise ValueError("top_k must satisfy 1 <= top_k <= experts_per_layer")
        if self.dtype_bytes not in (1, 2, 4):
            raise ValueError("dtype_bytes must be one of 1, 2, 4")


@dataclass(frozen=True)
class BatchConfig:
    batch_size: int
    input_len: int
    output_len: int

    def __post_init__(self) -> None:
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.input_len < 1:
            raise ValueError("input_len must be >= 1")
        if self.output_len < 0:
            raise ValueError("output_len must be >= 0")


class PhaseKind(Enum):
    PREFILL = "prefill"
    DECODE = "decode"


@dataclass(frozen=True)
class Phase:
    kind: PhaseKind
    seq_len: int
    kv_len: int

    def __post_init__(self) -> None:
        if self.seq_len < 1:
            raise ValueError("seq_len must be >= 1")
        if self.kv_len < 0:
            raise ValueError("kv_len must be >= 0")
        if self.kind is PhaseKind.DECODE and self.seq_len != 1:
            raise ValueError("a decode step processes exactly one token per sequence")

    @classmethod
    def prefill(cls, input_len: int) -> "Phase":
        return cls(PhaseKind.PREFILL, seq_len=input_len, kv_len=0)

    @classmethod
    def decode_step(cls, input_len: int, step: int) -> "Phase":
        if step < 1:
            raise ValueError("decode steps are numbered from 1")
        return cls(PhaseKind.DECODE, seq_len=1, kv_len=input_len + step - 1)


class Device(Enum):
    CPU = "cpu"
    GPU = "gpu"


@dataclass(frozen=True)
class AllocationStrategy:
    """Expert partition: exp_r resident + exp_m migrated (streamed) + exp_c CPU.

    The B200 executor has no CPU expert path (no CPU fallback by design), so it
    requires exp_c == 0; exp_m experts are streamed host->HBM per pass.
    """

    placement: tuple
    exp_r: int
    exp_m: int
    exp_c: int
    m: int
    coalesced_expert_batch: bool = True

    def __post_init__(self) -> None:
        if len(self.placement) != 3:
            raise ValueError("placement must cover ops 0..2")
        if min(self.exp_r, self.exp_m, self.exp_c) < 0:
            raise ValueError("expert partition counts must be >= 0")
        if self.m < 1:
            raise ValueError("micro-batch size m must be >= 1")
        if not self.coalesced_expert_batch:
            raise ValueError("expert execution is always coalesced; see expert_stage_time")

    @property
    def num_gpu_experts(self) -> int:
        return self.exp_r + self.exp_m

    @property
    def expert_total(self) -> int:
        return self.exp_r + self.exp_m + self.exp_c

    def num_micro_batches(self, batch: BatchConfig) -> int:
        return math.ceil(batch.batch_size / self.m)


def check_partition(strategy, model) -> None:
    """costmodel._check_partition (costmodel.py:92-97) + the executor's exp_c == 0 rule."""
    total = strategy.exp_r + strategy.exp_m + strategy.exp_c
    if total != model.experts_per_layer:
        raise ValueError(
            f"expert partition {strategy.exp_r}+{strategy.exp_m}+{strategy.exp_c} "
            f"does not cover the {model.experts_per_layer} activated experts"
        )
    if strategy.exp_c != 0:
        raise ValueError("the B200 executor runs every expert on the GPU: exp_c must be 0")


@dataclass(frozen=True)
class ExpertStageParts:
    """Same fields as costmodel.ExpertStageParts (costmodel.py:199-222); here
    they hold MEASURED seconds (CUDA events) instead of roofline estimates.
    lat_cpu and return_store are always 0 (no CPU expert share)."""

    act_load: float
    mig_load: float
    lat_gpu: float
    lat_cpu: float
    return_store: float

    @property
    def t_load(self) -> float:
        return self.act_load + self.mig_load

    @property
    def t_comp(self) -> float:
        return max(self.lat_gpu, self.lat_cpu)


@dataclass(frozen=True)
class ActivationMap:
    counts: np.ndarray  # (num_layers, experts_per_layer) float64

    def __post_init__(self) -> None:
        if self.counts.ndim != 2:
            raise ValueError("counts must be a (num_layers, experts_per_layer) array")
        if np.any(self.counts < 0):
            raise ValueError("counts must be non-negative")

    @property
    def num_layers(self) -> int:
        return self.counts.shape[0]

    @property
    def experts_per_layer(self) -> int:
        return self.counts.shape[1]

    def sorted_share_profile(self) -> np.ndarray:
        totals = self.counts.sum(axis=1, keepdims=True)
        if np.any(totals <= 0):
            raise ValueError("every layer must have recorded activations")
        shares = np.sort(self.counts / totals, axis=1)[:, ::-1]
        profile = shares.mean(axis=0)
        return profile / profile.sum()

    @classmethod
    def uniform(cls, num_layers: int, experts_per_layer: int) -> "ActivationMap":
        return cls(np.ones((num_layers, experts_per_layer)))


@dataclass(frozen=True)
class ResidencyPlan:
    resident: tuple
    capacity_per_layer: int

    def __post_init__(self) -> None:
        if self.capacity_per_layer < 0:
            raise ValueError("capacity_per_layer must be >= 0")
        for layer_set in self.resident:
            if len(layer_set) > self.capacity_per_layer:
                raise ValueError("a layer exceeds capacity_per_layer")
            if len(set(layer_set)) != len(layer_set):
                raise ValueError("resident experts must be distinct per layer")

    @property
    def num_layers(self) -> int:
        return len(self.resident)
