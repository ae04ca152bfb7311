"""Synthetic, seeded inputs and random-init weights (no checkpoints, no datasets).

Weights follow nn.Linear's default U(-1/sqrt(fan_in), +1/sqrt(fan_in)) and are
rounded to bf16; x ~ N(0, 1) rounded to bf16.  Generation uses a seeded
torch.Generator on the target device; whoever needs the same bits on the CPU
(the oracle) copies the generated tensors, so both sides see identical values.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class LayerWeights:
    wg: torch.Tensor                 # [E, d] fp32 (bf16-representable values)
    w1: torch.Tensor | None          # [E, ff, d] bf16 (kept only if keep_split)
    w3: torch.Tensor | None          # [E, ff, d] bf16
    w13: torch.Tensor                # [E, 2ff, d] bf16, K3 interleaved layout
    w2: torch.Tensor                 # [E, d, ff] bf16
    shared_w1: torch.Tensor | None = None   # [ffs, d]
    shared_w3: torch.Tensor | None = None
    shared_w13: torch.Tensor | None = None  # [2ffs, d]
    shared_w2: torch.Tensor | None = None   # [d, ffs]

    @property
    def num_experts(self) -> int:
        return self.w13.shape[0]

    @property
    def hidden_dim(self) -> int:
        return self.w13.shape[2]

    @property
    def expert_dim(self) -> int:
        return self.w2.shape[2]


def _uniform(shape, fan_in, g, device):
    t = torch.empty(shape, dtype=torch.float32, device=device)
    t.uniform_(-1.0, 1.0, generator=g)
    t.mul_(fan_in ** -0.5)
    return t.to(torch.bfloat16)


def interleave_w13_torch(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[.., ff, d] x2 -> [.., 2ff, d]: 128-row blocks (gate_i, up_i, ...). Layout helper."""
    *lead, ff, d = w1.shape
    a = w1.reshape(*lead, ff // 128, 128, d)
    b = w3.reshape(*lead, ff // 128, 128, d)
    return torch.stack([a, b], dim=-3).reshape(*lead, 2 * ff, d).contiguous()


def make_layer_weights(E: int, d: int, ff: int, seed: int = 0, device="cuda", shared_ff: int = 0,
                       keep_split: bool = False) -> LayerWeights:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    wg = _uniform((E, d), d, g, device).float()
    w13 = torch.empty((E, 2 * ff, d), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((E, d, ff), dtype=torch.bfloat16, device=device)
    w1s, w3s = [], []
    for e in range(E):
        w1 = _uniform((ff, d), d, g, device)
        w3 = _uniform((ff, d), d, g, device)
        w13[e] = interleave_w13_torch(w1, w3)
        w2[e] = _uniform((d, ff), ff, g, device)
        if keep_split:
            w1s.append(w1)
            w3s.append(w3)
    lw = LayerWeights(wg=wg, w1=torch.stack(w1s) if keep_split else None,
                      w3=torch.stack(w3s) if keep_split else None, w13=w13, w2=w2)
    if shared_ff:
        sw1 = _uniform((shared_ff, d), d, g, device)
        sw3 = _uniform((shared_ff, d), d, g, device)
        lw.shared_w13 = interleave_w13_torch(sw1, sw3)
        lw.shared_w2 = _uniform((d, shared_ff), shared_ff, g, device)
        if keep_split:
            lw.shared_w1, lw.shared_w3 = sw1, sw3
    return lw


def make_tokens(T: int, d: int, seed: int = 1, device="cuda", dtype=torch.bfloat16) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.empty((T, d), dtype=torch.float32, device=device)
    x.normal_(0.0, 1.0, generator=g)
    return x.to(dtype)


def split_w13(w13: torch.Tensor):
    """Inverse of interleave: [.., 2ff, d] -> (w1, w3) [.., ff, d]."""
    *lead, two_ff, d = w13.shape
    ff = two_ff // 2
    v = w13.reshape(*lead, ff // 128, 2, 128, d)
    return (v[..., 0, :, :].reshape(*lead, ff, d), v[..., 1, :, :].reshape(*lead, ff, d))
