"""Decode-step latency vs batch size (C4 DeepSeek-V2-Lite layer): dense single-
launch decode (cox_decode_moe, every expert over all tokens), routed single
launch (cox_decode_moe_routed, router in the prologue) and routed two launches
(router kernel + cox_small_expert_ffn_idx); CUDA-graph replay, CUDA events,
median of 200 steps.

    python tools/sweep_decode.py        # on the GPU box
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402


def time_layer(layer, T, d):
    x = make_tokens(T, d, seed=1, device="cuda")
    replay, _ = layer.capture(x)
    for _ in range(20):
        replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def main():
    d, ff, E, k, sff = 2048, 1408, 64, 6, 2816
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    for T in (1, 4, 8, 16, 24, 32, 48, 64, 128, 256):
        row = []
        for variant in ("dense", "routed1", "routed2"):
            layer = MoELayer(wts, k, "deepseek")
            if variant == "dense" and not layer.uses_small_path(T):
                row.append(float("nan"))
                continue
            layer.DENSE_T_MAX = 256 if variant == "dense" else 0
            layer.DECODE_ROUTE_IN = variant == "routed1"
            row.append(time_layer(layer, T, d) if variant != "dense" or T <= 64 else float("nan"))
        print(f"T={T:3d}: dense {row[0]:7.1f} us   routed, one launch {row[1]:7.1f} us   "
              f"routed, router launch + FFN {row[2]:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
