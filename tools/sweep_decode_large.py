"""Decode/small-prefill crossover (C4 layer, T = 64..512): weight-streaming kernel
with row gathers straight from the router's idx (default), with a materialised
x_perm (router + permute copy, tiled B loads), and the prefill kernels
(router + permute + grouped GEMMs + combine); CUDA-graph replay, median of 100.

    python tools/sweep_decode_large.py        # on the GPU box
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402
from sweep_decode import time_layer  # noqa: E402


def main():
    d, ff, E, k, sff = 2048, 1408, 64, 6, 2816
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    for T in (64, 128, 192, 256, 384, 512):
        row = []
        for variant in ("gather", "x_perm", "prefill"):
            layer = MoELayer(wts, k, "deepseek")
            layer.DENSE_T_MAX = 0
            if variant == "gather":
                layer.SMALL_GATHER_T_MAX = 1 << 30  # row gathers at every T
            if variant == "x_perm":
                layer.SMALL_GATHER_T_MAX = 0
            if variant == "prefill":
                layer.SMALL_T_MAX = 0
            if variant != "prefill" and not layer.uses_small_path(T):
                row.append(float("nan"))
                continue
            row.append(time_layer(layer, T, d))
        print(f"T={T:3d}: gather-from-idx {row[0]:7.1f} us   x_perm {row[1]:7.1f} us   prefill kernels {row[2]:7.1f} us",
              flush=True)


if __name__ == "__main__":
    main()
