"""C4 prefill: how should the shared experts be scheduled against the routed stage?
Times whole steps (CUDA events, steady state under the power cap) for
  beside : MoELayer.forward (shared GEMMs on a side stream after the router)
  serial : router, permute, K3, K4, shared K3, shared K4, combine on one stream
and the per-kernel split of the serial order, interleaved over several rounds.

    python tools/c4_order.py [rounds] [steps]
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402


def serial(layer, x, b, ev=None):
    def mark(i):
        if ev is not None:
            ev[i].record()
    mark(0)
    layer._router(x, b)
    mark(1)
    layer._permute(x, b)
    mark(2)
    layer._swiglu(b, layer.groups, layer.w13_list)
    mark(3)
    ops.grouped_down(b.h, b.offsets, layer.groups, layer.w2_list, layer.d, y=b.y)
    mark(4)
    sh = layer.shared_expert(x, b)
    mark(5)
    ops.combine(b.y, b.dst, b.w, sh, out=b.out)
    mark(6)


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    T, d, ff, E, k, sff = 64 * 4096, 2048, 1408, 64, 6, 2816
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, "deepseek")
    b = layer.buffers(T, x.device)
    variants = {"beside": lambda: layer(x), "serial": lambda: serial(layer, x, b)}
    for f in variants.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    res = {n: [] for n in variants}
    for r in range(rounds):
        for n, f in variants.items():
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                f()
            z.record()
            torch.cuda.synchronize()
            res[n].append(a.elapsed_time(z) / steps)
    for n, v in res.items():
        print(f"{n:8s} ms/step " + " ".join(f"{t:.3f}" for t in v), flush=True)
    names = ["router", "permute", "k3", "k4", "shared", "combine"]
    acc = [0.0] * 6
    for _ in range(steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        serial(layer, x, b, ev)
        torch.cuda.synchronize()
        for i in range(6):
            acc[i] += ev[i].elapsed_time(ev[i + 1]) / steps
    print("serial split " + " ".join(f"{n} {t:.3f}" for n, t in zip(names, acc)) + f"  sum {sum(acc):.3f}")




def ablate(rounds=3, steps=10, config="C4", gather=None):
    """What-if: step time with a stage left out (its outputs stale from an earlier
    step), to measure what each non-GEMM stage costs inside the power-capped step."""
    shapes = {"C4": (64 * 4096, 2048, 1408, 64, 6, "deepseek", 2816), "C2": (64 * 4096, 4096, 14336, 8, 2, "mixtral", 0)}
    T, d, ff, E, k, mode, sff = shapes[config]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, mode, gather_a=gather)
    b = layer.buffers(T, x.device)
    layer._permute(x, b)

    def run(skip):
        if "router" not in skip:
            layer._router(x, b)
        if "permute" not in skip:
            layer._permute(x, b)
        layer.experts(b)
        sh = layer.shared_expert(x, b)
        if "combine" not in skip:
            ops.combine(b.y, b.dst, b.w, sh, out=b.out)
    variants = {"full": (), "-router": ("router",), "-permute": ("permute",), "-combine": ("combine",),
                "gemms": ("router", "permute", "combine")}
    for v in variants.values():
        run(v)
    torch.cuda.synchronize()
    res = {n: [] for n in variants}
    for r in range(rounds):
        for n, v in variants.items():
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                run(v)
            z.record()
            torch.cuda.synchronize()
            res[n].append(a.elapsed_time(z) / steps)
    for n, v in res.items():
        print(f"{config}{' gather' if layer.gather_a else ' x_perm'} {n:9s} ms/step " + " ".join(f"{t:.3f}" for t in v),
              flush=True)


def beside_sweep(rounds=3, steps=10):
    """C4: the shared experts on a side stream beside the router/permute, with the
    shared GEMMs limited to `max_ctas` SMs so that the HBM-bound permute keeps
    some SMs; serial order as the reference."""
    T, d, ff, E, k, sff = 64 * 4096, 2048, 1408, 64, 6, 2816
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, "deepseek")
    b = layer.buffers(T, x.device)
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()

    def beside(mc, early):
        if not early:
            layer._router(x, b)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            sh = layer.shared_expert(x, b, max_ctas=mc)
        if early:
            layer._router(x, b)
        layer._permute(x, b)
        layer.experts(b)
        main.wait_stream(side)
        ops.combine(b.y, b.dst, b.w, sh, out=b.out)
    variants = {"serial": lambda: serial(layer, x, b)}
    for mc in (0, 128, 112, 96):
        variants[f"beside{mc}"] = (lambda mc=mc: beside(mc, False))
        variants[f"early{mc}"] = (lambda mc=mc: beside(mc, True))
    for f in variants.values():
        f()
    torch.cuda.synchronize()
    res = {n: [] for n in variants}
    for r in range(rounds):
        for n, f in variants.items():
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                f()
            z.record()
            torch.cuda.synchronize()
            res[n].append(a.elapsed_time(z) / steps)
    for n, v in res.items():
        print(f"C4 {n:10s} ms/step " + " ".join(f"{t:.3f}" for t in v), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "beside":
        beside_sweep()
    elif len(sys.argv) > 1 and sys.argv[1] == "ablate":
        ablate(config=sys.argv[2] if len(sys.argv) > 2 else "C4",
               gather={"gather": True, "xperm": False}.get(sys.argv[3]) if len(sys.argv) > 3 else None)
    else:
        main()
