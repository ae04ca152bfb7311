"""Deterministic regeneration of the golden-vector inputs (numpy RNG only, so
the CPU container and the GPU box produce identical bits)."""
from __future__ import annotations

import numpy as np

# name: (seed, T, d, E, k)
ROUTING_CASES = {
    "mixtral_c2shape": (11, 65536, 4096, 8, 2),
    "deepseek_c4shape": (12, 16384, 2048, 64, 6),
}


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16 << 16
    return b.astype(np.uint32).view(np.float32)


def routing_inputs(name: str):
    seed, T, d, E, k = ROUTING_CASES[name]
    rng = np.random.default_rng(seed)
    x = bf16_round(rng.standard_normal((T, d), dtype=np.float32))
    wg = bf16_round((rng.random((E, d), dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(d)))
    return x, wg, k


def layer_micro_inputs():
    """Small ragged cases; case 'b' leaves expert 3 empty by construction."""
    cases = {}
    for case, (seed, T, d, ff, E, k, mode) in {"a": (21, 37, 64, 96, 4, 2, 0), "b": (22, 29, 64, 128, 4, 2, 0),
                                                "c": (23, 41, 128, 64, 8, 3, 1)}.items():
        rng = np.random.default_rng(seed)
        x = bf16_round(rng.standard_normal((T, d), dtype=np.float32))
        wg = bf16_round((rng.random((E, d), dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(d)))
        if case == "b":
            wg[3] = 0.0
            x = np.abs(x)  # make expert 3's logit (0) lose to positive logits
            wg[:3] = np.abs(wg[:3])
        w1 = bf16_round((rng.random((E, ff, d), dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(d)))
        w3 = bf16_round((rng.random((E, ff, d), dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(d)))
        w2 = bf16_round((rng.random((E, d, ff), dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(ff)))
        cases[case] = (x, wg, w1, w3, w2, k, mode)
    return cases
