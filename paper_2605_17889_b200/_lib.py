"""ctypes binding of libcoxmoe.so (include/coxmoe.h).

There is deliberately no fallback: if the library is missing or the device is
not sm_100, every op raises.  Error behaviour mirrors the reference: invalid
shapes raise ValueError (moeplan raises ValueError for invalid input,
costmodel.py:92-97, workload.py:157-158); CUDA failures raise RuntimeError.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
import os as _os

# COXMOE_LIB overrides the in-tree library (A/B experiments between builds).
LIB_PATH = Path(_os.environ["COXMOE_LIB"]) if _os.environ.get("COXMOE_LIB") else _PKG / "libcoxmoe.so"

COX_OK = 0
COX_EINVAL = -1
COX_ECUDA = -2
COX_EUNSUPPORTED = -3
DTYPE_F32 = 0
DTYPE_BF16 = 1
ROUTE_MIXTRAL = 0
ROUTE_DEEPSEEK = 1

# Every symbol include/coxmoe.h declares (tests check the .so exports them all).
EXPORTS = (
    "cox_last_error", "cox_version", "cox_device_check", "cox_router_workspace_bytes", "cox_router_topk",
    "cox_permute_workspace_bytes", "cox_permute", "cox_grouped_swiglu", "cox_grouped_swiglu_gather", "cox_grouped_down",
    "cox_small_expert_ffn", "cox_small_expert_ffn_idx", "cox_decode_moe", "cox_combine", "cox_ep_counts_put",
    "cox_ep_offsets", "cox_ep_dispatch", "cox_ep_combine", "cox_interleave_w13", "cox_fetch_experts",
)
ABI_VERSION = 3

_lock = threading.Lock()
_lib = None
_device_ok = None


class CoxError(RuntimeError):
    pass


def _declare(L):
    c_int, c_void_p, c_ll, c_size_t = ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_size_t
    P = c_void_p
    L.cox_last_error.restype = ctypes.c_char_p
    L.cox_last_error.argtypes = []
    L.cox_version.restype = c_int
    L.cox_device_check.restype = c_int
    L.cox_router_workspace_bytes.restype = c_size_t
    L.cox_router_workspace_bytes.argtypes = [c_int, c_int]
    L.cox_router_topk.restype = c_int
    L.cox_router_topk.argtypes = [P, c_int, P, c_int, c_int, c_int, c_int, c_int, c_int, P, P, P, P, c_size_t, P]
    L.cox_permute_workspace_bytes.restype = c_size_t
    L.cox_permute_workspace_bytes.argtypes = [c_int, c_int]
    L.cox_permute.restype = c_int
    L.cox_permute.argtypes = [P, c_int, c_int, c_int, c_int, P, c_int, P, P, P, c_ll, P, P, P]
    L.cox_grouped_swiglu.restype = c_int
    L.cox_grouped_swiglu.argtypes = [P, c_ll, P, c_int, c_int, P, P, c_int, c_int, P, c_int, P]
    L.cox_grouped_swiglu_gather.restype = c_int
    L.cox_grouped_swiglu_gather.argtypes = [P, c_ll, P, P, c_int, c_int, P, P, c_int, c_int, P, c_int, P]
    L.cox_grouped_down.restype = c_int
    L.cox_grouped_down.argtypes = [P, c_ll, P, c_int, c_int, P, P, c_int, c_int, P, c_int, P]
    L.cox_small_expert_ffn.restype = c_int
    L.cox_small_expert_ffn.argtypes = [P, c_int, P, P, c_ll, P, c_int, c_int, P, P, P, c_int, c_int, P, P, P, P,
                                       c_int, P, P, P, P, c_int, P, P]
    L.cox_small_expert_ffn_idx.restype = c_int
    L.cox_small_expert_ffn_idx.argtypes = [P, c_int, P, P, c_int, P, c_int, P, P, c_int, c_int, P, P, P, P, c_int,
                                           P, P, P, P, P, P]
    L.cox_decode_moe.restype = c_int
    L.cox_decode_moe.argtypes = [P, c_int, P, c_int, c_int, c_int, P, P, c_int, c_int, P, P, c_int, P, P, P, P, P,
                                 P, P, P]
    L.cox_fetch_experts.restype = c_int
    L.cox_fetch_experts.argtypes = [P, c_int, c_int, P, P, P, P, c_int, P, P]
    L.cox_combine.restype = c_int
    L.cox_combine.argtypes = [P, P, P, c_int, c_int, c_int, P, P, c_int, P]
    L.cox_ep_counts_put.restype = c_int
    L.cox_ep_counts_put.argtypes = [P, c_int, c_int, c_int, P, P]
    L.cox_ep_offsets.restype = c_int
    L.cox_ep_offsets.argtypes = [P, c_int, c_int, c_int, c_ll, P, P, P, P]
    L.cox_ep_dispatch.restype = c_int
    L.cox_ep_dispatch.argtypes = [P, P, P, P, c_int, c_int, c_int, c_int, c_ll, P, c_int, P, P, P]
    L.cox_ep_combine.restype = c_int
    L.cox_ep_combine.argtypes = [P, P, P, c_int, c_int, c_int, c_int, c_int, P, P, P]
    L.cox_interleave_w13.restype = c_int
    L.cox_interleave_w13.argtypes = [P, P, c_int, c_int, P, P]


def load(path: Path | None = None):
    """Load (without touching the GPU) and declare the C ABI."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path) if path else LIB_PATH
            if not p.exists():
                raise CoxError(f"{p} is missing: run __graft_entry__.build() (no CPU fallback exists)")
            L = ctypes.CDLL(str(p))
            _declare(L)
            if L.cox_version() != ABI_VERSION:
                raise CoxError(f"{p}: ABI version {L.cox_version()} != {ABI_VERSION}: rebuild the library")
            _lib = L
    return _lib


def lib():
    """The loaded library, after checking once that the device is sm_100."""
    global _device_ok
    L = load()
    if _device_ok is None:
        rc = L.cox_device_check()
        _device_ok = rc == 0
        if not _device_ok:
            raise CoxError(L.cox_last_error().decode())
    elif not _device_ok:
        raise CoxError("libcoxmoe: unsupported device")
    return L


def check(rc: int, fn: str) -> None:
    if rc == COX_OK:
        return
    msg = _lib.cox_last_error().decode() if _lib is not None else fn
    if rc == COX_EINVAL:
        raise ValueError(msg)
    raise CoxError(msg)
