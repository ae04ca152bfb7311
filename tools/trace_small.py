"""Per-unit timeline of the decode expert FFN kernel (csrc/small_gemm.cu).

Builds a TRACED copy of the library (the kernel source patched to stamp
%globaltimer when the producer picks up a unit and when the epilogue finishes
it) into paper_2605_17889_b200/build/trace/, runs one C4 decode step through it
and prints where the time goes: start-up, per-pass unit durations, idle gaps
and the tail.  Debug tool only; the product library is untouched.

    python tools/trace_small.py [C4D|C2D]  # on the GPU box (gpurun)
"""
from __future__ import annotations

import ctypes
import os
import re
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TRACE_DIR = ROOT / "paper_2605_17889_b200" / "build" / "trace"
LIB = TRACE_DIR / "libcoxmoe_trace.so"
MAXU = 96  # units recorded per CTA (C2D: ~14 per CTA)


def make_traced_sources() -> Path:
    src = TRACE_DIR / "csrc"
    if src.exists():
        shutil.rmtree(src)
    shutil.copytree(ROOT / "paper_2605_17889_b200" / "csrc", src)
    f = src / "small_gemm.cu"
    s = f.read_text()
    s = s.replace("namespace cox {\n", f"""namespace cox {{
__device__ unsigned long long g_trace[160 * {MAXU + 2} * 3];
__device__ __forceinline__ unsigned long long gtimer() {{
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}}
""", 1)
    # kernel entry stamp (before barrier init / PDL wait / routing / group table)
    ent = "  const int warp = threadIdx.x >> 5;\n  const int lane = threadIdx.x & 31;\n  const int G = p.n_groups;\n"
    assert ent in s
    s = s.replace(ent, ent + f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU}) * 3 + 2] = gtimer();\n", 1)
    # route_in prologue: after this CTA's routing, after the grid-wide wait (row MAXU - 1)
    a1 = "      __syncthreads();\n    }\n  }\n  if (warp == 0) {\n    if (p.from_idx) {\n"
    if a1 in s:
        s = s.replace(a1, "      __syncthreads();\n    }\n  }\n"
                      f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU - 1}) * 3] = gtimer();\n"
                      "  if (warp == 0) {\n    if (p.from_idx) {\n", 1)
    a2 = "        if (lane == 0) mbar_spin_ge(p.counters + SG_ROUTED, p.T);  // every CTA's tokens are routed\n"
    if a2 in s:
        s = s.replace(a2, a2 + f"        if (lane == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU - 1}) * 3 + 1] = gtimer();\n", 1)
    # route_in: after the logits of this CTA's first token, after its top-k (row MAXU - 2)
    a3 = "      __syncthreads();\n      if (warp == 2) {\n        warp_route_token("
    if a3 in s:
        s = s.replace(a3, "      __syncthreads();\n"
                      f"      if (threadIdx.x == 0 && t == (int)blockIdx.x) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU - 2}) * 3] = gtimer();\n"
                      "      if (warp == 2) {\n        warp_route_token(", 1)
    a4 = "        if (lane == 0) red_release_add(p.counters + SG_ROUTED, 1);  // after idx / w / histogram\n      }\n"
    if a4 in s:
        s = s.replace(a4, "        if (lane == 0) red_release_add(p.counters + SG_ROUTED, 1);  // after idx / w / histogram\n"
                      f"        if (lane == 0 && t == (int)blockIdx.x) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU - 2}) * 3 + 1] = gtimer();\n"
                      "      }\n", 1)
    # kernel start / end stamps
    s = s.replace("  const uint32_t tmem_base = *tmem_slot;\n",
                  f"  const uint32_t tmem_base = *tmem_slot;\n"
                  f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU}) * 3] = gtimer();\n", 1)
    s = s.replace("  tc_fence_before();\n  __syncthreads();\n  if (warp == 2) {\n    tc_fence_after();\n    tmem_dealloc<1>",
                  f"  tc_fence_before();\n  __syncthreads();\n"
                  f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU}) * 3 + 1] = gtimer();\n"
                  f"  if (warp == 2) {{\n    tc_fence_after();\n    tmem_dealloc<1>", 1)
    # end of the deferred combine
    pat_c = "  if (threadIdx.x == 0) {\n    // the last CTA to exit zeroes the counters"
    if pat_c in s:
        s = s.replace(pat_c, f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU + 1}) * 3] = gtimer();\n" + pat_c, 1)
    # inside the combine: after the dst/w staging
    pat_s = "    __syncthreads();\n    const __nv_bfloat16* y0 = p.y[0];"
    if pat_s in s:
        s = s.replace(pat_s, f"    __syncthreads();\n    if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU + 1}) * 3 + 1] = gtimer();\n"
                      "    const __nv_bfloat16* y0 = p.y[0];", 1)
    pat_b = "  const int npend = s_misc[2];\n"
    if pat_b in s:
        s = s.replace(pat_b, pat_b + f"  if (threadIdx.x == 0) g_trace[(blockIdx.x * {MAXU + 2} + {MAXU + 1}) * 3 + 2] = gtimer();\n", 1)
    # producer: unit pick-up
    s = s.replace("      int t = lane == 0 ? fetch(si, true) : 0;\n      t = __shfl_sync(0xffffffffu, t, 0);\n      if (t >= total) break;\n",
                  f"      int t = lane == 0 ? fetch(si, true) : 0;\n      t = __shfl_sync(0xffffffffu, t, 0);\n      if (t >= total) break;\n"
                  f"      if (lane == 0 && si - 1 < {MAXU}) {{\n"
                  f"        g_trace[(blockIdx.x * {MAXU + 2} + si - 1) * 3] = gtimer();\n"
                  f"        g_trace[(blockIdx.x * {MAXU + 2} + si - 1) * 3 + 2] = t;\n      }}\n", 1)
    # epilogue: unit finished (after its last accumulator is released)
    pat = "        if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));\n      }\n"
    assert pat in s
    s = s.replace(pat, pat + f"      if (tid == 0 && si - 1 < {MAXU}) g_trace[(blockIdx.x * {MAXU + 2} + si - 1) * 3 + 1] = gtimer();\n", 1)
    s += f"""
extern "C" int cox_trace_dump(unsigned long long* host) {{
  return (int)cudaMemcpyFromSymbol(host, cox::g_trace, sizeof(unsigned long long) * 160 * {MAXU + 2} * 3);
}}
extern "C" int cox_trace_clear() {{
  static unsigned long long z[160 * {MAXU + 2} * 3];
  return (int)cudaMemcpyToSymbol(cox::g_trace, z, sizeof(z));
}}
"""
    f.write_text(s)
    return src


def build_traced():
    from paper_2605_17889_b200 import build
    src = make_traced_sources()
    build.build(force=True, out=LIB, csrc=src)


def run(cfg: str = "C4D"):
    os.environ["COXMOE_LIB"] = str(LIB)
    import torch
    from paper_2605_17889_b200.layer import MoELayer
    from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
    from paper_2605_17889_b200 import _lib
    T, d, ff, E, k, sff, mode = {"C4D": (64, 2048, 1408, 64, 6, 2816, "deepseek"),
                                 "C2D": (64, 4096, 14336, 8, 2, 0, "mixtral")}[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda", shared_ff=sff)
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, mode)
    for _ in range(5):
        layer(x)
    torch.cuda.synchronize()
    L = _lib.load()
    L.cox_trace_clear()
    layer(x)
    torch.cuda.synchronize()
    if os.environ.get("TRACE_GRAPH") == "1":
        # steady state under graph replay: the traced buffers keep the LAST replay's stamps
        replay, _ = layer.capture(x)
        for _ in range(3):
            replay()
        torch.cuda.synchronize()
        L.cox_trace_clear()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        replay()
        ev0.record()
        replay()
        ev1.record()
        torch.cuda.synchronize()
        print(f"[{cfg}] graph replay step {ev0.elapsed_time(ev1) * 1e3:.1f} us")
    n = 160 * (MAXU + 2) * 3
    buf = (ctypes.c_ulonglong * n)()
    assert L.cox_trace_dump(buf) == 0
    import numpy as np
    a = np.frombuffer(buf, dtype=np.uint64).reshape(160, MAXU + 2, 3).astype(np.int64)
    nb = 148
    starts, ends, entry = a[:nb, MAXU, 0], a[:nb, MAXU, 1], a[:nb, MAXU, 2]
    t0 = starts.min()
    l1, l2 = a[:nb, MAXU - 2, 0], a[:nb, MAXU - 2, 1]
    if l2.max() > 0:
        m = l2 > 0
        print(f"[{cfg}] route_in first token: logits done median {np.median((l1 - entry)[m]) / 1e3:.1f} us after "
              f"entry (max {np.max((l1 - entry)[m]) / 1e3:.1f}), top-k + publish done median "
              f"{np.median((l2 - entry)[m]) / 1e3:.1f} (max {np.max((l2 - entry)[m]) / 1e3:.1f})")
        a[:nb, MAXU - 2] = 0
    r1, r2 = a[:nb, MAXU - 1, 0], a[:nb, MAXU - 1, 1]
    if r2.max() > 0:
        print(f"[{cfg}] route_in: own routing done median {np.median(r1 - entry) / 1e3:.1f} us after entry "
              f"(max {(r1.max() - entry.min()) / 1e3:.1f} from first entry); grid-wide wait passed median "
              f"{np.median(r2 - entry) / 1e3:.1f} us after entry")
        a[:nb, MAXU - 1] = 0
    print(f"[{cfg}] kernel entry: first {(entry.min() - t0) / 1e3:.1f} us, last {(entry.max() - t0) / 1e3:.1f} us "
          f"(relative to the first CTA past the prologue); prologue per CTA median "
          f"{np.median(starts - entry) / 1e3:.1f} us")
    print(f"CTA start spread {(starts.max() - t0) / 1e3:.1f} us; kernel body {(ends.max() - t0) / 1e3:.1f} us; "
          f"first CTA end {(ends.min() - t0) / 1e3:.1f} us")
    cend = a[:nb, MAXU + 1, 0]
    if cend.max() > 0:
        print(f"after the deferred combine: last CTA {(cend.max() - t0) / 1e3:.1f} us, "
              f"median {(np.median(cend) - t0) / 1e3:.1f} us")
        b = int(np.argmax(cend))
        cst, cbeg = a[b, MAXU + 1, 1], a[b, MAXU + 1, 2]
        print(f"  last CTA {b}: combine begins {(cbeg - t0) / 1e3:.1f}, staged {(cst - t0) / 1e3:.1f}, "
              f"done {(cend[b] - t0) / 1e3:.1f} us")
    rec = []
    for b in range(nb):
        for u in range(MAXU):
            s, e, t = a[b, u]
            if s == 0:
                break
            rec.append((b, u, (s - t0) / 1e3, (e - t0) / 1e3 if e else float("nan"), int(t)))
    total3 = None
    ids = sorted(r[4] for r in rec)
    print(f"units traced {len(rec)} (max id {ids[-1]})")
    durs = np.array([r[3] - r[2] for r in rec])
    print(f"unit pick-up -> done: median {np.nanmedian(durs):.1f} us, p90 {np.nanpercentile(durs, 90):.1f}")
    first = np.array([min(r[2] for r in rec if r[0] == b) for b in range(nb)])
    last_pick = np.array([max(r[2] for r in rec if r[0] == b) for b in range(nb)])
    last_done = np.array([np.nanmax([r[3] for r in rec if r[0] == b]) for b in range(nb)])
    print(f"first pick-up per CTA: median {np.median(first):.1f} us, max {first.max():.1f}")
    print(f"last unit done per CTA: min {last_done.min():.1f} median {np.median(last_done):.1f} max {last_done.max():.1f} us")
    per = {}
    for b, u, s, e, t in rec:
        per.setdefault(b, []).append((s, e, t))
    # time by pass: the id where the down pass starts is where ids jump in duration; report by id quartiles
    by_id = sorted(rec, key=lambda r: r[4])
    for q in range(0, len(by_id), max(1, len(by_id) // 12)):
        chunk = by_id[q:q + max(1, len(by_id) // 12)]
        print(f"  ids {chunk[0][4]:5d}-{chunk[-1][4]:5d}: picked {chunk[0][2]:7.1f}-{chunk[-1][2]:7.1f} us, "
              f"median dur {np.nanmedian([c[3] - c[2] for c in chunk]):5.1f} us")


if __name__ == "__main__":
    if "--run-only" not in sys.argv:
        build_traced()
    for c in [a for a in sys.argv[1:] if not a.startswith("--")] or ["C4D"]:
        run(c)
