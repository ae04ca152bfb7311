"""Power-cap probe: C2's K3 (grouped SwiGLU GEMM) on 148 / 132 / 116 / 100 SMs
(`max_ctas`), steady state, interleaved rounds, with the SM clock sampled by
nvidia-smi.  If the 1 kW cap binds, fewer SMs run at a higher clock and lose
less than their share of throughput — the measure of how much of the GEMM's
power is per-SM (tensor pipe, operand delivery) rather than global.

    python tools/power_sms.py
"""
from __future__ import annotations

import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402


def sample_clock(stop, out):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                               capture_output=True, text=True, timeout=5).stdout.strip().split(",")
            out.append((float(r[0]), float(r[1])))
        except Exception:  # noqa: BLE001
            pass
        time.sleep(0.2)


def main():
    T, d, ff, E, k = 64 * 4096, 4096, 14336, 8, 2
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda")
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, "mixtral")
    b = layer.buffers(T, x.device)
    layer.route(x, b)
    flops = 4.0 * T * k * d * ff
    res = {}
    for _ in range(2):
        for mc in (148, 132, 116, 100):
            for _ in range(2):
                ops.grouped_swiglu(b.x_perm, b.offsets, layer.groups, layer.w13_list, ff, h=b.h, max_ctas=mc)
            stop, clk = threading.Event(), []
            th = threading.Thread(target=sample_clock, args=(stop, clk))
            th.start()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(8):
                ops.grouped_swiglu(b.x_perm, b.offsets, layer.groups, layer.w13_list, ff, h=b.h, max_ctas=mc)
            z.record()
            torch.cuda.synchronize()
            stop.set()
            th.join()
            ms = a.elapsed_time(z) / 8
            c = sorted(v[0] for v in clk)
            p = sorted(v[1] for v in clk)
            res.setdefault(mc, []).append((ms, c[len(c) // 2] if c else 0, p[len(p) // 2] if p else 0))
    for mc, v in res.items():
        print(f"K3 on {mc:3d} SMs: " + "  ".join(f"{ms:.1f} ms ({flops / ms / 1e9:.0f} TF/s, {c:.0f} MHz, {p:.0f} W)"
                                                for ms, c, p in v), flush=True)


if __name__ == "__main__":
    main()
