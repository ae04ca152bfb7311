"""Run a few eager steps of one MoE layer at a given batch size (for an ncu
launch list of the kernels a step launches).

    ncu --kernel-name regex:"router|perm|grouped|combine|small_ffn" ... python tools/step_kernels.py C4 512
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

SHAPES = {"C4": (2048, 1408, 64, 6, "deepseek", 2816), "C2": (4096, 14336, 8, 2, "mixtral", 0)}

if __name__ == "__main__":
    cfg, T = sys.argv[1], int(sys.argv[2])
    d, ff, E, k, mode, sff = SHAPES[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, mode)
    for _ in range(3):
        layer(x)
    torch.cuda.synchronize()
