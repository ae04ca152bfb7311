"""CPU ORACLE (test infrastructure only) — ctypes front end of ``oracle/liboracle.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
and ``--impl reference`` legs) may import this module.  The product package
``paper_2605_17889_b200`` never imports it and has no CPU fallback.

What it restates (see the C sources for the per-function citations):
  * router / top-k / stable permute / combine  -> oracle_router.c
  * per-expert SwiGLU FFN over the coalesced batch -> oracle_ffn.c
Parity status: routing/permutation/FFN are UNPINNED by the reference (moeplan
ships no such code); they are cross-checked against an
independent numpy float64 restatement and frozen as golden vectors under
tests/golden/.  The analytical/residency half is pinned against the reference's
own golden values (tests/test_reference_interop.py).
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _HERE / "liboracle.so"


def lib():
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle.so"
        if not path.exists():
            build()
        L = ctypes.CDLL(str(path))
        L.oracle_router_topk.restype = ctypes.c_int
        L.oracle_router_topk.argtypes = [_f32p, _f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, _i32p, _f32p, _i32p]
        L.oracle_router_topk_bf16.restype = ctypes.c_int
        L.oracle_router_topk_bf16.argtypes = [_u16p, _f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_void_p, _i32p, _f32p, _i32p]
        L.oracle_router_logit.restype = ctypes.c_float
        L.oracle_router_logit.argtypes = [_f32p, _f32p, ctypes.c_int]
        L.oracle_permute.restype = ctypes.c_int
        L.oracle_permute.argtypes = [_i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i32p, _i32p]
        L.oracle_combine.restype = None
        L.oracle_combine.argtypes = [_f32p, _i32p, _f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, _f32p]
        L.oracle_expert_ffn.restype = None
        L.oracle_expert_ffn.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f32p, _f32p, _f32p,
                                        _f32p, ctypes.c_void_p]
        L.oracle_grouped_ffn.restype = None
        L.oracle_grouped_ffn.argtypes = [_f32p, _i32p, _i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         _f32p, _f32p, _f32p, _f32p]
        L.oracle_gather.restype = None
        L.oracle_gather.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, _i32p, ctypes.c_int, _f32p]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def router_topk(x, wg, k: int, mode: int = 0, want_logits: bool = False):
    """-> (idx [T,k] i32, w [T,k] f32, counts [E] i32[, logits [T,E] f32])."""
    x = _f32(x)
    wg = _f32(wg)
    T, d = x.shape
    E = wg.shape[0]
    idx = np.zeros((T, k), np.int32)
    w = np.zeros((T, k), np.float32)
    counts = np.zeros(E, np.int32)
    logits = np.zeros((T, E), np.float32) if want_logits else None
    rc = lib().oracle_router_topk(x, wg, T, d, E, k, mode,
                                  logits.ctypes.data if want_logits else None, idx, w, counts)
    if rc != 0:
        raise ValueError("oracle_router_topk: invalid arguments (d must be a multiple of 8, 1<=k<=E<=256)")
    return (idx, w, counts, logits) if want_logits else (idx, w, counts)


def router_topk_bf16(x_bits, wg, k: int, mode: int = 0):
    """Router over bf16 tokens given as their uint16 bit patterns [T, d] (exact
    widening; same arithmetic as router_topk on the fp32 copy) — for full
    batches: -> (idx, w, counts)."""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    wg = _f32(wg)
    T, d = x_bits.shape
    E = wg.shape[0]
    idx = np.zeros((T, k), np.int32)
    w = np.zeros((T, k), np.float32)
    counts = np.zeros(E, np.int32)
    if lib().oracle_router_topk_bf16(x_bits, wg, T, d, E, k, mode, None, idx, w, counts) != 0:
        raise ValueError("oracle_router_topk_bf16: invalid arguments")
    return idx, w, counts


def permute(idx, E: int, tile_m: int = 1):
    """-> (offsets [E+1] i32, dst [T,k] i32)."""
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    T, k = idx.shape
    offsets = np.zeros(E + 1, np.int32)
    dst = np.zeros((T, k), np.int32)
    if lib().oracle_permute(idx, T, k, E, tile_m, offsets, dst) != 0:
        raise ValueError("oracle_permute: invalid arguments")
    return offsets, dst


def gather(x, dst, rows: int) -> np.ndarray:
    x = _f32(x)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    T, d = x.shape
    out = np.zeros((rows, d), np.float32)
    lib().oracle_gather(x, T, d, dst, dst.shape[1], out)
    return out


def expert_ffn(x, w1, w3, w2, want_h: bool = False):
    x = _f32(x)
    n, d = x.shape
    ff = w1.shape[0]
    y = np.zeros((n, d), np.float32)
    h = np.zeros((n, ff), np.float32) if want_h else None
    lib().oracle_expert_ffn(x, n, d, ff, _f32(w1), _f32(w3), _f32(w2), y, h.ctypes.data if want_h else None)
    return (y, h) if want_h else y


def grouped_ffn(x_perm, offsets, counts, w1, w3, w2) -> np.ndarray:
    x_perm = _f32(x_perm)
    E, ff, d = w1.shape
    y = np.zeros_like(x_perm)
    lib().oracle_grouped_ffn(x_perm, np.ascontiguousarray(offsets, np.int32), np.ascontiguousarray(counts, np.int32),
                             E, d, ff, _f32(w1), _f32(w3), _f32(w2), y)
    return y


def combine(y_perm, dst, w, shared=None) -> np.ndarray:
    y_perm = _f32(y_perm)
    dst = np.ascontiguousarray(dst, np.int32)
    w = _f32(w)
    T, k = dst.shape
    d = y_perm.shape[1]
    out = np.zeros((T, d), np.float32)
    sh = _f32(shared) if shared is not None else None
    lib().oracle_combine(y_perm, dst, w, T, k, d, sh.ctypes.data if sh is not None else None, out)
    return out


def moe_layer(x, wg, w1, w3, w2, k: int, mode: int = 0, tile_m: int = 1, shared=None):
    """Full coalesced MoE expert stage on the CPU.

    shared: optional (ws1 [ffs,d], ws3 [ffs,d], ws2 [d,ffs]) always-on shared
    expert MLP (DeepSeek-V2), added to the routed output.
    Returns dict(out, idx, w, counts, offsets, dst).
    """
    x = _f32(x)
    idx, w, counts = router_topk(x, wg, k, mode)
    offsets, dst = permute(idx, wg.shape[0], tile_m)
    x_perm = gather(x, dst, int(offsets[-1]))
    y_perm = grouped_ffn(x_perm, offsets, counts, w1, w3, w2)
    sh = expert_ffn(x, *shared) if shared is not None else None
    out = combine(y_perm, dst, w, sh)
    return dict(out=out, idx=idx, w=w, counts=counts, offsets=offsets, dst=dst)
