"""Where the decode step's time goes: CUDA-graph replays of the whole idx-path
step (router + expert kernel), the router alone and the expert kernel alone
(routing precomputed), median of repeated replays.

    python tools/decode_probe.py [C4|C2] [T]
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

SHAPES = {"C4": (2048, 1408, 64, 6, "deepseek", 2816), "C2": (4096, 14336, 8, 2, "mixtral", 0)}


def graph_time(fn, reps=300):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        z.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(z) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    Ts = [int(sys.argv[2])] if len(sys.argv) > 2 else [1, 8, 64]
    d, ff, E, k, mode, sff = SHAPES[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    for T in Ts:
        layer = MoELayer(wts, k, mode)
        layer.DENSE_T_MAX = 0
        x = make_tokens(T, d, seed=1, device="cuda")
        b = layer.buffers(T, x.device)
        out = b.out
        step = graph_time(lambda: layer(x))
        rt = graph_time(lambda: layer._router(x, b))
        layer._router(x, b)
        ffn = graph_time(lambda: layer._ffn_idx(x, b, out))
        both = graph_time(lambda: (layer._router(x, b), layer._ffn_idx(x, b, out)))
        print(f"{cfg} T={T:3d}: step {step:7.1f} us  router alone {rt:6.1f}  expert kernel alone {ffn:7.1f}  "
              f"router+kernel {both:7.1f}  -> router on the critical path {both - ffn:5.1f} us", flush=True)
        dl = MoELayer(wts, k, mode)
        dl.DENSE_T_MAX = 64
        if dl.uses_dense_decode(T):
            print(f"{cfg} T={T:3d}: dense one-launch step {graph_time(lambda: dl(x)):7.1f} us", flush=True)


if __name__ == "__main__":
    main()
