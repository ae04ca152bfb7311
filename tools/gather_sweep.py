"""Time the prefill layer with K3 on materialised x_perm vs K3 gathering its A
rows from x (MoELayer(gather_a=True)), interleaved, CUDA events, steady state.

    python tools/gather_sweep.py C4|C2|C3L

Measured (round 2): a hybrid that moved part of each CTA's A rows to TMA
tile::gather4 was slower the more rows the TMA took (C4: 34.0 ms with all rows
by cp.async, 37.4 with 3/8 by gather4, 55.3 with all by gather4, vs 30.3 on
x_perm), so the library gathers by cp.async only.
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

SHAPES = {"C4": (64 * 4096, 2048, 1408, 64, 6, "deepseek", 2816), "C2": (64 * 4096, 4096, 14336, 8, 2, "mixtral", 0),
          "C3L": (64 * 4096, 6144, 16384, 8, 2, "mixtral", 0)}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    rounds, steps = 3, (10 if cfg == "C4" else 4)
    T, d, ff, E, k, mode, sff = SHAPES[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layers = {"x_perm": MoELayer(wts, k, mode, gather_a=False), "gather": MoELayer(wts, k, mode, gather_a=True)}
    outs = {n: L(x).clone() for n, L in layers.items()}
    same = torch.equal(outs["x_perm"], outs["gather"])
    del outs
    res = {n: [] for n in layers}
    for _ in range(rounds):
        for n, L in layers.items():
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                L(x)
            z.record()
            torch.cuda.synchronize()
            res[n].append(a.elapsed_time(z) / steps)
    print(f"{cfg} outputs bit-identical: {same}  " +
          "  ".join(f"{n} " + " ".join(f"{t:.2f}" for t in v) + " ms" for n, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
