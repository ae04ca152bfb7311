"""Build libcoxmoe.so (all sm_100a kernels + the C ABI) in-tree with nvcc.

    python -m paper_2605_17889_b200.build        # or __graft_entry__.build()

The library is placed next to this file so that the gpurun snapshot carries it
to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libcoxmoe.so"
SOURCES = ["capi.cu", "router.cu", "permute.cu", "combine.cu", "grouped_gemm.cu", "small_gemm.cu", "router_tc.cu", "router_e8.cu", "fetch.cu", "ep.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "coxmoe.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, csrc: Path | None = None) -> Path:
    """Compile the sources in `csrc` (default: csrc/) into `out` (default: libcoxmoe.so)."""
    lib = Path(out) if out else LIB
    src_dir = Path(csrc) if csrc else CSRC
    if not force and out is None and csrc is None and not needs_build():
        return LIB
    objdir = PKG / "build" / lib.stem
    objdir.mkdir(parents=True, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              "-I", str(ROOT / "include")]
    objs = []
    procs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        objs.append(o)
        procs.append((s, subprocess.Popen([*common, "-I", str(CSRC), "-c", str(src_dir / s), "-o", str(o)],
                                          stdout=subprocess.PIPE,
                                          stderr=subprocess.STDOUT, text=True)))
    for s, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            raise RuntimeError(f"nvcc failed on {s}")
    tmp = lib.with_suffix(".so.tmp")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
