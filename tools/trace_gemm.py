"""Per-tile timeline of the prefill grouped GEMM (csrc/grouped_gemm.cu).

Builds a TRACED copy of the library (%globaltimer stamps in the leader CTA of
every pair: MMA warp after it got the accumulator / after its last commit,
epilogue warp 4 after the accumulator arrived / after it released it) into
paper_2605_17889_b200/build/trace_gemm/, runs one layer step of the given
config and prints per-tile MMA / epilogue durations and the gaps between
consecutive tiles of a pair.  Debug tool only.

    python tools/trace_gemm.py C4          # on the GPU box (gpurun)
"""
from __future__ import annotations

import ctypes
import os
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TRACE_DIR = ROOT / "paper_2605_17889_b200" / "build" / "trace_gemm"
LIB = TRACE_DIR / "libcoxmoe_trace.so"
MAXT = 4096  # tiles recorded per CTA pair


def make_traced_sources() -> Path:
    src = TRACE_DIR / "csrc"
    if src.exists():
        shutil.rmtree(src)
    shutil.copytree(ROOT / "paper_2605_17889_b200" / "csrc", src)
    f = src / "grouped_gemm.cu"
    s = f.read_text()
    s = s.replace("namespace cox {\n", f"""namespace cox {{
__device__ unsigned long long g_gtrace[80 * {MAXT} * 4];
__device__ __forceinline__ unsigned long long gtimer2() {{
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}}
""", 1)
    slot = f"((blockIdx.x >> 1) * {MAXT} + it)"
    a = "        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);\n"
    assert a in s
    s = s.replace(a, a + f"        if (it < {MAXT}) g_gtrace[{slot} * 4 + 0] = gtimer2();\n", 1)
    b = "        mma_commit<2>(smem_u32(&tfull[acc]));\n"
    assert b in s
    s = s.replace(b, b + f"        if (it < {MAXT}) g_gtrace[{slot} * 4 + 1] = gtimer2();\n", 1)
    c = "      mbar_wait(smem_u32(&tfull[acc]), acc_phase);\n"
    assert c in s
    s = s.replace(c, c + f"      if (rank == 0 && ew == 0 && lane == 0 && it < {MAXT}) g_gtrace[{slot} * 4 + 2] = gtimer2();\n", 1)
    d = "      if (lane == 0) mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);\n"
    assert d in s
    s = s.replace(d, d + f"      if (rank == 0 && ew == 0 && lane == 0 && it < {MAXT}) g_gtrace[{slot} * 4 + 3] = gtimer2();\n", 1)
    s += f"""
extern "C" int cox_gtrace_dump(unsigned long long* host) {{
  return (int)cudaMemcpyFromSymbol(host, cox::g_gtrace, sizeof(unsigned long long) * 80 * {MAXT} * 4);
}}
extern "C" int cox_gtrace_clear() {{
  static unsigned long long z[80 * {MAXT} * 4];
  return (int)cudaMemcpyToSymbol(cox::g_gtrace, z, sizeof(z));
}}
"""
    f.write_text(s)
    return src


def build_traced():
    from paper_2605_17889_b200 import build
    build.build(force=True, out=LIB, csrc=make_traced_sources())


def run(cfg: str):
    os.environ["COXMOE_LIB"] = str(LIB)
    import numpy as np
    import torch
    from paper_2605_17889_b200 import _lib, ops
    from paper_2605_17889_b200.layer import MoELayer
    from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
    T, d, ff, E, k, mode = {"C1": (4096, 1024, 3584, 8, 2, "mixtral"), "C2": (65536, 4096, 14336, 8, 2, "mixtral"),
                            "C4": (65536, 2048, 1408, 64, 6, "deepseek")}[cfg]
    wts = make_layer_weights(E, d, ff, seed=0, device="cuda")
    x = make_tokens(T, d, seed=1, device="cuda")
    layer = MoELayer(wts, k, mode)
    layer(x)
    torch.cuda.synchronize()
    b = layer.buffers(T, "cuda")
    L = _lib.load()
    for name in ("K3", "K4"):
        L.cox_gtrace_clear()
        torch.cuda.synchronize()
        if name == "K3":
            layer._k3(b, layer.groups, layer.w13_list)
        else:
            ops.grouped_down(b.h, b.offsets, layer.groups, layer.w2_list, layer.d, y=b.y)
        torch.cuda.synchronize()
        n = 80 * MAXT * 4
        buf = (ctypes.c_ulonglong * n)()
        assert L.cox_gtrace_dump(buf) == 0
        a = np.frombuffer(buf, dtype=np.uint64).reshape(80, MAXT, 4).astype(np.int64)[:74]
        valid = a[:, :, 0] > 0
        t0 = a[:, :, 0][valid].min()
        mma = (a[:, :, 1] - a[:, :, 0])[valid] / 1e3
        epi = (a[:, :, 3] - a[:, :, 2])[valid & (a[:, :, 3] > 0)] / 1e3
        lag = (a[:, :, 2] - a[:, :, 1])[valid & (a[:, :, 2] > 0)] / 1e3
        gaps = []
        for p in range(74):
            v = a[p][valid[p]]
            if len(v) > 1:
                gaps.extend(((v[1:, 0] - v[:-1, 1]) / 1e3).tolist())
        ends = a[:, :, 3][valid].max()
        print(f"{cfg} {name}: tiles {valid.sum()}, span {(ends - t0) / 1e3:.1f} us; per tile: MMA issue->commit "
              f"median {np.median(mma):.2f} us, commit->epilogue start {np.median(lag):.2f}, epilogue "
              f"median {np.median(epi):.2f} p90 {np.percentile(epi, 90):.2f} us; MMA idle between tiles median "
              f"{np.median(gaps):.2f} p90 {np.percentile(gaps, 90):.2f} us", flush=True)


if __name__ == "__main__":
    if "--run-only" not in sys.argv:
        build_traced()
    for c in [a for a in sys.argv[1:] if not a.startswith("--")] or ["C4"]:
        run(c)
