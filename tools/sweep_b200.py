#!/usr/bin/env python
"""Measured counterpart of `moeplan sweep` (planner.sweep_microbatch,
pkg/src/moeplan/planner.py:321-366; the paper's Fig. 2): expert-stage time
with the expert GEMMs coalesced over the whole batch vs launched per
micro-batch of m sequences, on one B200, next to the analytical expert_s of
the restated cost model (paper_2605_17889_b200/costmodel.py, B200 measured
peaks, top-k counted).

    python tools/sweep_b200.py [--config C2] [--m 1,4,16,64] > profiles/r01/sweep_c2.csv

CSV columns follow the reference's sweep output (m, expert_s, ...), one layer.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2605_17889_b200 import costmodel as CM  # noqa: E402
from paper_2605_17889_b200.config import AllocationStrategy, BatchConfig, Device, ModelConfig, Phase  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="1,4,16,64", help="micro-batch sizes in sequences of 4096 tokens")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    B, L, d, ff, E, k = 64, 4096, 4096, 14336, 8, 2
    T = B * L
    dev = torch.device("cuda", 0)
    wts = make_layer_weights(E, d, ff, seed=0, device=dev)
    x = make_tokens(T, d, seed=1, device=dev)
    layer = MoELayer(wts, k)
    model = ModelConfig(1, d, ff, E, k, 2)
    batch = BatchConfig(B, L, 0)
    system = CM.b200_system()
    print("m,mode,expert_s_measured,expert_s_model,tokens_per_s")
    for m in [int(v) for v in args.m.split(",")]:
        for mode in ("coalesced", "microbatched"):
            if mode == "coalesced" and m != B:
                run = lambda: layer(x)  # noqa: E731
            else:
                run = lambda: layer.forward_microbatched(x, m * L)  # noqa: E731
            run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                run()
            b.record()
            torch.cuda.synchronize()
            s = a.elapsed_time(b) / args.reps / 1e3
            strat = AllocationStrategy((Device.GPU,) * 3, E, 0, 0, m=m)
            parts = CM.expert_stage_parts(strat, Phase.prefill(L), system, model, batch, None,
                                          coalesced=(mode == "coalesced"), count_top_k=True)
            print(f"{m},{mode},{s:.6e},{parts.t_comp:.6e},{T / s:.1f}", flush=True)


if __name__ == "__main__":
    main()
