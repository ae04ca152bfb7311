"""Batch-size sweep of the expert stage (one MoE layer) from decode to prefill:
tokens/s and time per step for T = 1 ... 262,144, with the kernel path
MoELayer picks for each T (dense single launch, router + weight-streaming
launch, router + permute + weight-streaming launch, prefill kernels).
Steps up to HOST_GRAPH_T_MAX tokens replay a CUDA graph (they are launch-bound
when eager); larger ones run eagerly.  CUDA events, median of repeated steps.

    python tools/sweep_tokens.py [C4|C2]
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

SHAPES = {"C4": (2048, 1408, 64, 6, "deepseek", 2816), "C2": (4096, 14336, 8, 2, "mixtral", 0)}


def path_of(layer, T):
    if layer.uses_dense_decode(T):
        return "dense 1 launch"
    if layer.uses_idx_decode(T):
        return "router + FFN(idx)"
    if layer.uses_small_path(T):
        return "router + permute + FFN"
    return "prefill kernels"


def time_step(layer, x, reps):
    T = x.shape[0]
    if T <= layer.HOST_GRAPH_T_MAX:
        replay, _ = layer.capture(x)
        fn = replay
    else:
        fn = lambda: layer(x)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        z.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(z))
    ts.sort()
    return ts[len(ts) // 2]


def compare_paths(cfg):
    """Weight-streaming (small) path vs prefill kernels for T = 64 ... 2048."""
    d, ff, E, k, mode, sff = SHAPES[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    for T in (64, 128, 192, 256, 384, 512, 768, 1024, 1536, 2048):
        x = make_tokens(T, d, seed=1, device="cuda")
        row = []
        for name, tmax in (("small", 1 << 30), ("prefill", 0)):
            layer = MoELayer(wts, k, mode)
            layer.SMALL_T_MAX = tmax
            layer.SMALL_ROWS_PER_EXPERT_MAX = tmax
            layer.SMALL_GATHER_T_MAX = min(layer.SMALL_GATHER_T_MAX, tmax)
            layer.DENSE_T_MAX = 0
            try:
                row.append(f"{name} {time_step(layer, x, 100) * 1e3:8.1f} us")
            except Exception as exc:  # noqa: BLE001
                row.append(f"{name} failed ({type(exc).__name__})")
            del layer
            torch.cuda.empty_cache()
        print(f"{cfg} T={T:5d} rows/expert {T * k / E:6.1f}:  " + "   ".join(row), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[2] == "paths":
        compare_paths(sys.argv[1])
        return
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    d, ff, E, k, mode, sff = SHAPES[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    print(f"{cfg}: d={d} ff={ff} E={E} k={k} shared_ff={sff}", flush=True)
    for T in (1, 8, 32, 64, 128, 256, 512, 1024, 2048, 4096, 16384, 65536, 262144):
        layer = MoELayer(wts, k, mode)
        x = make_tokens(T, d, seed=1, device="cuda")
        reps = 200 if T <= 4096 else (30 if T <= 65536 else 8)
        ms = time_step(layer, x, reps)
        flops = 6.0 * T * k * d * ff + (6.0 * T * d * sff if sff else 0.0) + 2.0 * T * d * E
        print(f"T={T:7d}  {ms * 1e3:10.1f} us  {T / ms * 1e3 / 1e6:9.3f} M tok/s  {flops / ms / 1e9:8.1f} TF/s  "
              f"[{path_of(layer, T)}]", flush=True)
        del layer, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
