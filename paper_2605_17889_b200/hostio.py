"""End-to-end host I/O for the expert stage: pinned host batches in, pinned
host outputs back, with the PCIe copies overlapped with the GPU work.

Batch i's H2D copy (copy engine, its own stream) overlaps batch i-1's expert
stage, and batch i's D2H copy overlaps batch i+1's stage: two device input and
two device output slots, event-ordered.  Every batch still crosses PCIe both
ways; only the waiting is hidden.  Used by MoELayer and by the expert-parallel
layers (one pipeline per rank).
"""
from __future__ import annotations

import torch


class HostIO:
    """The per-batch-size device slots and copy streams of run_host_batches."""

    def __init__(self, T: int, d: int, device, out_dtype=torch.bfloat16):
        self.T = T
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.xin = [torch.empty((T, d), dtype=torch.bfloat16, device=device) for _ in range(2)]
        self.yout = [torch.empty((T, d), dtype=out_dtype, device=device) for _ in range(2)]
        self.in_free = [None, None]
        self.out_done = [None, None]


def run_host_batches(io: HostIO, xs_host, outs_host, step) -> None:
    """Run `step(slot)` (the expert stage reading io.xin[slot], writing
    io.yout[slot] on the current stream) for every host batch.  Returns once all
    work is enqueued; the current stream is ordered after the last copy."""
    if len(xs_host) != len(outs_host):
        raise ValueError("one output buffer per input batch")
    comp = torch.cuda.current_stream(io.xin[0].device)
    for i, xh in enumerate(xs_host):
        if xh.shape[0] != io.T:
            raise ValueError("all host batches must have the same number of tokens")
        slot = i % 2
        with torch.cuda.stream(io.h2d):
            if io.in_free[slot] is not None:
                io.h2d.wait_event(io.in_free[slot])
            io.xin[slot].copy_(xh, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(io.h2d)
        comp.wait_event(ready)
        if io.out_done[slot] is not None:
            comp.wait_event(io.out_done[slot])
        step(slot)
        ev_c = torch.cuda.Event()
        ev_c.record(comp)
        io.in_free[slot] = ev_c
        with torch.cuda.stream(io.d2h):
            io.d2h.wait_event(ev_c)
            outs_host[i].copy_(io.yout[slot], non_blocking=True)
            ev_o = torch.cuda.Event()
            ev_o.record(io.d2h)
            io.out_done[slot] = ev_o
    comp.wait_stream(io.d2h)
