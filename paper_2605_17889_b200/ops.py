"""Torch-tensor front end of the C ABI: one function per kernel stage.

Tensors are plain device memory here (torch is the allocator and the stream
owner); every computation happens in libcoxmoe.so.  Functions validate the
tensor metadata, then call the corresponding ``cox_*`` entry point on the
current torch stream.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib

_BF16 = torch.bfloat16


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need(t: torch.Tensor, name: str, dtype=None, ndim=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D")


def _ptrs(ts: Sequence[torch.Tensor]):
    arr = (ctypes.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


def _ids(ids: Sequence[int]):
    arr = (ctypes.c_int32 * max(1, len(ids)))()
    for i, e in enumerate(ids):
        arr[i] = int(e)
    return arr


def router_workspace_bytes(T: int, E: int) -> int:
    return int(_lib.load().cox_router_workspace_bytes(T, E))


def router_workspace(T: int, E: int, device) -> torch.Tensor:
    """A zero-initialised router workspace (the kernels leave it zeroed; one per
    concurrently executing launch, e.g. per layer buffer set)."""
    return torch.zeros((max(16, router_workspace_bytes(T, E)),), dtype=torch.uint8, device=device)


def router_topk(x: torch.Tensor, wg: torch.Tensor, k: int, mode: int = _lib.ROUTE_MIXTRAL, out=None,
                workspace: torch.Tensor | None = None, stream=None):
    """K1: -> (idx [T,k] int32, w [T,k] fp32, counts [E] int32).  wg: fp32 or bf16 [E, d]."""
    _need(x, "x", ndim=2)
    _need(wg, "wg", None, 2)
    if wg.dtype not in (torch.float32, _BF16):
        raise ValueError("wg must be fp32 or bf16")
    T, d = x.shape
    E = wg.shape[0]
    if wg.shape[1] != d:
        raise ValueError("wg must be [E, d]")
    if x.dtype == _BF16:
        xdt = _lib.DTYPE_BF16
    elif x.dtype == torch.float32:
        xdt = _lib.DTYPE_F32
    else:
        raise ValueError("x must be bf16 or fp32")
    if out is None:
        idx = torch.empty((T, k), dtype=torch.int32, device=x.device)
        w = torch.empty((T, k), dtype=torch.float32, device=x.device)
        counts = torch.empty((E,), dtype=torch.int32, device=x.device)
    else:
        idx, w, counts = out
    if workspace is None:
        workspace = router_workspace(T, E, x.device)
    _need(workspace, "workspace", torch.uint8, 1)
    L = _lib.lib()
    wdt = _lib.DTYPE_BF16 if wg.dtype == _BF16 else _lib.DTYPE_F32
    _lib.check(L.cox_router_topk(x.data_ptr(), xdt, wg.data_ptr(), wdt, T, d, E, k, mode, idx.data_ptr(),
                                 w.data_ptr(), counts.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                 _stream(stream)), "cox_router_topk")
    return idx, w, counts


def permute_workspace_bytes(T: int, E: int) -> int:
    return int(_lib.load().cox_permute_workspace_bytes(T, E))


def rows_capacity(T: int, k: int, E: int, tile_m: int = 1) -> int:
    return max(1, T * k + E * (tile_m - 1))


def permute(idx: torch.Tensor, x: torch.Tensor, E: int, tile_m: int = 1, out=None, workspace=None, stream=None,
            copy_rows: bool = True, row_tokens: torch.Tensor | None = None):
    """K2: -> (offsets [E+1] int32, dst [T,k] int32, x_perm [rows_cap, d] bf16 or None).

    copy_rows=False computes offsets/dst only (the fused EP dispatch moves the rows)."""
    _need(idx, "idx", torch.int32, 2)
    _need(x, "x", _BF16, 2)
    T, k = idx.shape
    d = x.shape[1]
    if x.shape[0] != T:
        raise ValueError("idx and x disagree on T")
    cap = rows_capacity(T, k, E, tile_m)
    if out is None:
        offsets = torch.empty((E + 1,), dtype=torch.int32, device=x.device)
        dst = torch.empty((T, k), dtype=torch.int32, device=x.device)
        x_perm = torch.empty((cap, d), dtype=_BF16, device=x.device) if copy_rows else None
    else:
        offsets, dst, x_perm = out
        if not copy_rows:
            x_perm = None
    if workspace is None:
        workspace = torch.empty((permute_workspace_bytes(T, E),), dtype=torch.uint8, device=x.device)
    L = _lib.lib()
    if row_tokens is not None:
        _need(row_tokens, "row_tokens", torch.int32, 1)
        if row_tokens.numel() < cap:
            raise ValueError(f"row_tokens needs {cap} entries")
    _lib.check(L.cox_permute(idx.data_ptr(), T, k, E, tile_m, x.data_ptr(), d, offsets.data_ptr(), dst.data_ptr(),
                             x_perm.data_ptr() if x_perm is not None else None,
                             x_perm.shape[0] if x_perm is not None else cap,
                             row_tokens.data_ptr() if row_tokens is not None else None, workspace.data_ptr(),
                             _stream(stream)), "cox_permute")
    return offsets, dst, x_perm


def grouped_swiglu(x_perm: torch.Tensor, offsets: torch.Tensor, group_experts: Sequence[int],
                   w13: Sequence[torch.Tensor], ff: int, h: torch.Tensor | None = None, stream=None,
                   max_ctas: int = 0):
    """K3: h[r] = silu(x_perm[r] W1_e^T) * (x_perm[r] W3_e^T) for the listed groups."""
    _need(x_perm, "x_perm", _BF16, 2)
    _need(offsets, "offsets", torch.int32, 1)
    rows, d = x_perm.shape
    for i, w in enumerate(w13):
        _need(w, f"w13[{i}]", _BF16, 2)
        if tuple(w.shape) != (2 * ff, d):
            raise ValueError(f"w13[{i}] must be [2*ff, d] = [{2 * ff}, {d}]")
    if len(w13) != len(group_experts):
        raise ValueError("one weight per group")
    if h is None:
        h = torch.empty((rows, ff), dtype=_BF16, device=x_perm.device)
    L = _lib.lib()
    _lib.check(L.cox_grouped_swiglu(x_perm.data_ptr(), rows, offsets.data_ptr(), offsets.numel() - 1,
                                    len(group_experts), _ids(group_experts), _ptrs(w13), d, ff, h.data_ptr(),
                                    max_ctas, _stream(stream)), "cox_grouped_swiglu")
    return h


def grouped_swiglu_gather(x: torch.Tensor, row_tokens: torch.Tensor, offsets: torch.Tensor,
                          group_experts: Sequence[int], w13: Sequence[torch.Tensor], ff: int, h: torch.Tensor,
                          stream=None, max_ctas: int = 0):
    """K3 with the permuted rows gathered from x: h[r] = SwiGLU_e(x[row_tokens[r]]) —
    the same bits as grouped_swiglu on x_perm, without the permute's row copy."""
    _need(x, "x", _BF16, 2)
    _need(row_tokens, "row_tokens", torch.int32, 1)
    _need(offsets, "offsets", torch.int32, 1)
    _need(h, "h", _BF16, 2)
    T, d = x.shape
    for i, w in enumerate(w13):
        _need(w, f"w13[{i}]", _BF16, 2)
        if tuple(w.shape) != (2 * ff, d):
            raise ValueError(f"w13[{i}] must be [2*ff, d] = [{2 * ff}, {d}]")
    if len(w13) != len(group_experts):
        raise ValueError("one weight per group")
    if h.shape[1] != ff or h.shape[0] > row_tokens.numel():
        raise ValueError("h must be [rows, ff] with a row_tokens entry per row")
    L = _lib.lib()
    _lib.check(L.cox_grouped_swiglu_gather(x.data_ptr(), T, row_tokens.data_ptr(), offsets.data_ptr(),
                                           offsets.numel() - 1, len(group_experts), _ids(group_experts), _ptrs(w13),
                                           d, ff, h.data_ptr(), max_ctas, _stream(stream)), "cox_grouped_swiglu_gather")
    return h


def grouped_down(h: torch.Tensor, offsets: torch.Tensor, group_experts: Sequence[int], w2: Sequence[torch.Tensor],
                 d: int, y: torch.Tensor | None = None, stream=None, max_ctas: int = 0):
    """K4: y[r] = h[r] W2_e^T for the listed groups."""
    _need(h, "h", _BF16, 2)
    _need(offsets, "offsets", torch.int32, 1)
    rows, ff = h.shape
    for i, w in enumerate(w2):
        _need(w, f"w2[{i}]", _BF16, 2)
        if tuple(w.shape) != (d, ff):
            raise ValueError(f"w2[{i}] must be [d, ff] = [{d}, {ff}]")
    if len(w2) != len(group_experts):
        raise ValueError("one weight per group")
    if y is None:
        y = torch.empty((rows, d), dtype=_BF16, device=h.device)
    L = _lib.lib()
    _lib.check(L.cox_grouped_down(h.data_ptr(), rows, offsets.data_ptr(), offsets.numel() - 1,
                                  len(group_experts), _ids(group_experts), _ptrs(w2), ff, d, y.data_ptr(), max_ctas,
                                  _stream(stream)), "cox_grouped_down")
    return y


def small_expert_ffn(x: torch.Tensor, offsets: torch.Tensor, group_experts: Sequence[int],
                     w13: Sequence[torch.Tensor], w2: Sequence[torch.Tensor], h: torch.Tensor, y: torch.Tensor,
                     x_perm: torch.Tensor | None = None, row_tokens: torch.Tensor | None = None,
                     shared=None, combine=None, stream=None):
    """K3+K4 (+shared experts, +K5) in one weight-streaming launch for decode-size batches.

    Routed rows come from ``x_perm`` or, if it is None, are gathered from ``x``
    through ``row_tokens``.  ``shared = (w13_shared, w2_shared, h_shared,
    y_shared)`` adds the dense shared-expert MLP over x; ``combine = (dst, w,
    out)`` fuses the weighted combine (bf16 out, same bits as ops.combine)."""
    _need(x, "x", _BF16, 2)
    _need(offsets, "offsets", torch.int32, 1)
    _need(h, "h", _BF16, 2)
    _need(y, "y", _BF16, 2)
    T, d = x.shape
    rows, ff = h.shape
    if tuple(y.shape) != (rows, d):
        raise ValueError("y must be [rows, d] with the rows of h")
    if x_perm is not None:
        _need(x_perm, "x_perm", _BF16, 2)
        if tuple(x_perm.shape) != (rows, d):
            raise ValueError("x_perm must be [rows, d] with the rows of h")
    elif row_tokens is not None:
        _need(row_tokens, "row_tokens", torch.int32, 1)
        if row_tokens.numel() < rows:
            raise ValueError("row_tokens needs one entry per row of h")
    elif len(group_experts):
        raise ValueError("need x_perm or row_tokens")
    if len(w13) != len(group_experts) or len(w2) != len(group_experts):
        raise ValueError("one weight pair per group")
    for i, (a, b) in enumerate(zip(w13, w2)):
        _need(a, f"w13[{i}]", _BF16, 2)
        _need(b, f"w2[{i}]", _BF16, 2)
        if tuple(a.shape) != (2 * ff, d) or tuple(b.shape) != (d, ff):
            raise ValueError(f"group {i}: need w13 [2*ff, d] and w2 [d, ff] with ff={ff}, d={d}")
    sw13 = sw2 = sh = sy = None
    ffs = 0
    if shared is not None:
        sw13, sw2, sh, sy = shared
        for t, n in ((sw13, "w13_shared"), (sw2, "w2_shared"), (sh, "h_shared"), (sy, "y_shared")):
            _need(t, n, _BF16, 2)
        ffs = sh.shape[1]
        if (tuple(sw13.shape) != (2 * ffs, d) or tuple(sw2.shape) != (d, ffs) or sh.shape[0] < T
                or sy.shape[0] < T or sy.shape[1] != d):
            raise ValueError("shared expert operands have inconsistent shapes")
    dst = wt = out = None
    k = 0
    if combine is not None:
        dst, wt, out = combine
        _need(dst, "dst", torch.int32, 2)
        _need(wt, "w", torch.float32, 2)
        _need(out, "out", _BF16, 2)
        k = dst.shape[1]
        if dst.shape[0] != T or tuple(wt.shape) != tuple(dst.shape) or tuple(out.shape) != (T, d):
            raise ValueError("combine operands must be dst/w [T, k] and out [T, d]")
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    L = _lib.lib()
    _lib.check(L.cox_small_expert_ffn(
        x.data_ptr(), T, ptr(row_tokens), ptr(x_perm), rows, offsets.data_ptr(), offsets.numel() - 1,
        len(group_experts),
        _ids(group_experts), _ptrs(w13), _ptrs(w2), d, ff, h.data_ptr(), y.data_ptr(), ptr(sw13), ptr(sw2), ffs,
        ptr(sh), ptr(sy), ptr(dst), ptr(wt), k, ptr(out), _stream(stream)), "cox_small_expert_ffn")
    return out if out is not None else y


def small_expert_ffn_idx(x: torch.Tensor, idx: torch.Tensor, counts: torch.Tensor, w: torch.Tensor,
                         w13: Sequence[torch.Tensor], w2: Sequence[torch.Tensor], h: torch.Tensor, y: torch.Tensor,
                         dst: torch.Tensor, out: torch.Tensor, offsets: torch.Tensor | None = None, shared=None,
                         stream=None):
    """Decode-size expert stage straight from the router output (no permute
    launch); writes dst (and offsets) like ops.permute, out = combined result.
    shared = (w13_shared, w2_shared, h_shared, y_shared)."""
    _need(x, "x", _BF16, 2)
    _need(idx, "idx", torch.int32, 2)
    _need(counts, "counts", torch.int32, 1)
    _need(w, "w", torch.float32, 2)
    _need(dst, "dst", torch.int32, 2)
    for t, n in ((h, "h"), (y, "y"), (out, "out")):
        _need(t, n, _BF16, 2)
    T, d = x.shape
    k = idx.shape[1]
    E = counts.shape[0]
    ff = h.shape[1]
    if (tuple(idx.shape) != (T, k) or tuple(w.shape) != (T, k) or tuple(dst.shape) != (T, k)
            or h.shape[0] < T * k or y.shape[0] < T * k or y.shape[1] != d or tuple(out.shape) != (T, d)
            or len(w13) != E or len(w2) != E):
        raise ValueError("small_expert_ffn_idx: inconsistent shapes")
    sw13 = sw2 = sh = sy = None
    ffs = 0
    if shared is not None:
        sw13, sw2, sh, sy = shared
        ffs = sh.shape[1]
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    L = _lib.lib()
    _lib.check(L.cox_small_expert_ffn_idx(
        x.data_ptr(), T, idx.data_ptr(), counts.data_ptr(), E, w.data_ptr(), k, _ptrs(w13), _ptrs(w2), d, ff,
        h.data_ptr(), y.data_ptr(), ptr(sw13), ptr(sw2), ffs, ptr(sh), ptr(sy), dst.data_ptr(), ptr(offsets),
        out.data_ptr(), _stream(stream)), "cox_small_expert_ffn_idx")
    return out


def decode_moe(x: torch.Tensor, wg: torch.Tensor, k: int, mode: int, w13: Sequence[torch.Tensor],
               w2: Sequence[torch.Tensor], h: torch.Tensor, y: torch.Tensor, idx: torch.Tensor, w: torch.Tensor,
               out: torch.Tensor, shared=None, stream=None):
    """Whole decode-step MoE layer in one launch (router + every expert over all
    T <= 64 tokens + shared experts + combine).  h [E*T, ff], y [E*T, d] scratch;
    shared = (w13_shared, w2_shared, h_shared, y_shared)."""
    _need(x, "x", _BF16, 2)
    _need(wg, "wg", _BF16, 2)
    T, d = x.shape
    E = wg.shape[0]
    ff = h.shape[1]
    for t, n in ((h, "h"), (y, "y"), (out, "out")):
        _need(t, n, _BF16, 2)
    _need(idx, "idx", torch.int32, 2)
    _need(w, "w", torch.float32, 2)
    if (wg.shape[1] != d or h.shape[0] != E * T or tuple(y.shape) != (E * T, d) or tuple(out.shape) != (T, d)
            or tuple(idx.shape) != (T, k) or tuple(w.shape) != (T, k) or len(w13) != E or len(w2) != E):
        raise ValueError("decode_moe: inconsistent shapes")
    sw13 = sw2 = sh = sy = None
    ffs = 0
    if shared is not None:
        sw13, sw2, sh, sy = shared
        ffs = sh.shape[1]
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    L = _lib.lib()
    _lib.check(L.cox_decode_moe(x.data_ptr(), T, wg.data_ptr(), E, k, mode, _ptrs(w13), _ptrs(w2), d, ff, ptr(sw13),
                                ptr(sw2), ffs, h.data_ptr(), y.data_ptr(), ptr(sh), ptr(sy), idx.data_ptr(),
                                w.data_ptr(), out.data_ptr(), _stream(stream)), "cox_decode_moe")
    return out


def fetch_experts(counts: torch.Tensor, expert_ids: Sequence[int], host_src: Sequence[torch.Tensor],
                  dst: Sequence[torch.Tensor], max_ctas: int = 0, fetched: torch.Tensor | None = None, stream=None):
    """K6': copy host_src[i] (pinned host) -> dst[i] (device) for every listed
    entry whose expert has router count > 0; decided on the device, no host sync."""
    _need(counts, "counts", torch.int32, 1)
    if not (len(expert_ids) == len(host_src) == len(dst)):
        raise ValueError("one source and one slot per entry")
    nbytes = (ctypes.c_longlong * max(1, len(dst)))()
    for i, (a, b) in enumerate(zip(host_src, dst)):
        if a.is_cuda or not a.is_pinned() or not a.is_contiguous():
            raise ValueError(f"host_src[{i}] must be contiguous pinned host memory")
        _need(b, f"dst[{i}]")
        if a.numel() * a.element_size() != b.numel() * b.element_size():
            raise ValueError(f"entry {i}: source and slot sizes differ")
        nbytes[i] = a.numel() * a.element_size()
    if fetched is not None:
        _need(fetched, "fetched", torch.int32, 1)
    L = _lib.lib()
    _lib.check(L.cox_fetch_experts(counts.data_ptr(), counts.numel(), len(expert_ids), _ids(expert_ids),
                                   _ptrs(host_src), _ptrs(dst), nbytes, max_ctas,
                                   fetched.data_ptr() if fetched is not None else None, _stream(stream)),
               "cox_fetch_experts")


def combine(y_perm: torch.Tensor, dst: torch.Tensor, w: torch.Tensor, shared: torch.Tensor | None = None,
            out: torch.Tensor | None = None, out_dtype=_BF16, stream=None):
    """K5: out[t] = sum_j w[t,j] y_perm[dst[t,j]] (+ shared[t])."""
    _need(y_perm, "y_perm", _BF16, 2)
    _need(dst, "dst", torch.int32, 2)
    _need(w, "w", torch.float32, 2)
    T, k = dst.shape
    d = y_perm.shape[1]
    if out is None:
        out = torch.empty((T, d), dtype=out_dtype, device=y_perm.device)
    odt = _lib.DTYPE_BF16 if out.dtype == _BF16 else _lib.DTYPE_F32
    if shared is not None:
        _need(shared, "shared", out.dtype, 2)
    L = _lib.lib()
    _lib.check(L.cox_combine(y_perm.data_ptr(), dst.data_ptr(), w.data_ptr(), T, k, d,
                             shared.data_ptr() if shared is not None else None, out.data_ptr(), odt, _stream(stream)),
               "cox_combine")
    return out


def interleave_w13(w1: torch.Tensor, w3: torch.Tensor, out: torch.Tensor | None = None, stream=None):
    """[ff,d] x 2 -> K3 layout [2ff, d] (128-row gate/up blocks)."""
    _need(w1, "w1", _BF16, 2)
    _need(w3, "w3", _BF16, 2)
    ff, d = w1.shape
    if out is None:
        out = torch.empty((2 * ff, d), dtype=_BF16, device=w1.device)
    L = _lib.lib()
    _lib.check(L.cox_interleave_w13(w1.data_ptr(), w3.data_ptr(), ff, d, out.data_ptr(), _stream(stream)),
               "cox_interleave_w13")
    return out


# --------------------------------------------------------------------------- fused EP (K7')
def ep_counts_put(counts: torch.Tensor, rank: int, world: int, peer_counts: torch.Tensor, stream=None):
    """counts[E] -> counts_all[rank] on every peer (peer_counts: device int64 [world] addresses)."""
    L = _lib.lib()
    _lib.check(L.cox_ep_counts_put(counts.data_ptr(), counts.numel(), rank, world, peer_counts.data_ptr(),
                                   _stream(stream)), "cox_ep_counts_put")


def ep_offsets(counts_all: torch.Tensor, rank: int, cap: int, recv_seg, send_base, overflow, stream=None):
    world, E = counts_all.shape
    L = _lib.lib()
    _lib.check(L.cox_ep_offsets(counts_all.data_ptr(), world, E, rank, cap, recv_seg.data_ptr(), send_base.data_ptr(),
                                overflow.data_ptr(), _stream(stream)), "cox_ep_offsets")


def ep_dispatch(idx, dst_local, offsets_local, send_base, x, world: int, cap: int, peer_recv, route_row,
                stream=None):
    T, k = idx.shape
    E = send_base.numel()
    L = _lib.lib()
    _lib.check(L.cox_ep_dispatch(idx.data_ptr(), dst_local.data_ptr(), offsets_local.data_ptr(), send_base.data_ptr(),
                                 T, k, E, world, cap, x.data_ptr(), x.shape[1], peer_recv.data_ptr(),
                                 route_row.data_ptr(), _stream(stream)), "cox_ep_dispatch")


def ep_combine(idx, route_row, w, E: int, world: int, peer_y, out, stream=None):
    T, k = idx.shape
    L = _lib.lib()
    _lib.check(L.cox_ep_combine(idx.data_ptr(), route_row.data_ptr(), w.data_ptr(), T, k, out.shape[1], E, world,
                                peer_y.data_ptr(), out.data_ptr(), _stream(stream)), "cox_ep_combine")
    return out
