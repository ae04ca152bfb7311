"""Time K1 (router + top-k) alone at the C2 and C4 shapes (CUDA events, median of
20 launches after warm-up), and check its indices against a reference build.

    python tools/bench_router.py            # on the GPU box
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

SHAPES = {"C2": (262144, 4096, 8, 2, 0), "C3L": (262144, 6144, 8, 2, 0), "C4": (262144, 2048, 64, 6, 1),
          "C4D": (64, 2048, 64, 6, 1)}


def main():
    for name, (T, d, E, k, mode) in SHAPES.items():
        wts = make_layer_weights(E, d, 256, seed=0, device="cuda")
        wg = wts.wg.to(torch.bfloat16)
        x = make_tokens(T, d, seed=1, device="cuda")
        out = (torch.empty((T, k), dtype=torch.int32, device="cuda"), torch.empty((T, k), device="cuda"),
               torch.empty((E,), dtype=torch.int32, device="cuda"))
        ws = ops.router_workspace(T, E, "cuda")
        for _ in range(3):
            ops.router_topk(x, wg, k, mode, out=out, workspace=ws)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.router_topk(x, wg, k, mode, out=out, workspace=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        chk = int(out[0].to(torch.int64).sum().item()) ^ int(out[0][:, 0].to(torch.int64).mul(7).sum().item())
        gbs = T * d * 2 / (ts[len(ts) // 2] / 1e3) / 1e9
        print(f"{name}: {gbs:7.0f} GB/s of x  router {ts[len(ts) // 2] * 1e3:8.1f} us  (min {ts[0] * 1e3:.1f})  idx checksum {chk}  "
              f"w sum {out[1].double().sum().item():.6f}", flush=True)


if __name__ == "__main__":
    main()
