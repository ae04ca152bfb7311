"""B200-native coalesced MoE expert stage (CoX-MoE, arxiv/paper_2605_17889).

Host side: mirrors of moeplan's types (config.py), the stage executor
(layer.py / executor.py), residency selection (eas.py), cold-expert streaming
(streaming.py) and expert parallelism (ep.py).  Compute: libcoxmoe.so
(csrc/, C ABI in include/coxmoe.h), sm_100a only, no CPU fallback.
"""
from .config import (ActivationMap, AllocationStrategy, BatchConfig, Device, ExpertStageParts, ModelConfig, Phase,
                     PhaseKind, ResidencyPlan)

__all__ = [
    "ActivationMap", "AllocationStrategy", "BatchConfig", "Device", "ExpertStageParts", "ModelConfig", "Phase",
    "PhaseKind", "ResidencyPlan",
]
