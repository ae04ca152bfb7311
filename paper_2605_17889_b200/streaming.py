"""Cold-expert streaming: pinned host pool -> HBM slot ring on a copy stream.

The reference charges migrated experts as `mig_load = exp_m * 3*dt*d*ff /
BW_link` (costmodel.py:252, Eq. 7) and its simulator lets the
`expert:migrate` task overlap everything before the expert stage
(sim.py:163-175).  Here the copies are real: `cudaMemcpyAsync` from pinned
host memory (copy engine, PCIe) on a dedicated stream into a ring of device
slots; each staged expert gets a CUDA event that the compute stream waits on
right before the GEMM groups that use it — resident experts never wait.
A slot is reused only after the compute stream has passed the event recorded
when its last consumer was enqueued.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class HostExpertPool:
    """Pinned host copies of expert weights: w13 [P, 2ff, d], w2 [P, d, ff] bf16."""

    w13: torch.Tensor
    w2: torch.Tensor

    @property
    def size(self) -> int:
        return self.w13.shape[0]

    @classmethod
    def from_device(cls, w13: torch.Tensor, w2: torch.Tensor) -> "HostExpertPool":
        h13 = torch.empty(w13.shape, dtype=w13.dtype, pin_memory=True)
        h2 = torch.empty(w2.shape, dtype=w2.dtype, pin_memory=True)
        h13.copy_(w13)
        h2.copy_(w2)
        return cls(h13, h2)

    def nbytes_per_expert(self) -> int:
        return (self.w13[0].numel() + self.w2[0].numel()) * self.w13.element_size()


class SlotRing:
    """Device slots for streamed experts + the copy stream that fills them."""

    def __init__(self, n_slots: int, d: int, ff: int, device, priority: int = 0):
        if n_slots < 1:
            raise ValueError("n_slots must be >= 1")
        self.w13 = torch.empty((n_slots, 2 * ff, d), dtype=torch.bfloat16, device=device)
        self.w2 = torch.empty((n_slots, d, ff), dtype=torch.bfloat16, device=device)
        self.n = n_slots
        self.stream = torch.cuda.Stream(device=device, priority=priority)
        self._free = [None] * n_slots  # event: compute stream has finished with the slot
        self.copy_events = []          # (slot, start_ev, end_ev) for timelines

    def stage(self, pool: HostExpertPool, pool_idx: int, slot: int, timing: bool = False):
        """Enqueue H2D of one expert into `slot`; returns the completion event."""
        s = self.stream
        if self._free[slot] is not None:
            s.wait_event(self._free[slot])
        ev0 = torch.cuda.Event(enable_timing=True) if timing else None
        with torch.cuda.stream(s):
            if ev0 is not None:
                ev0.record(s)
            self.w13[slot].copy_(pool.w13[pool_idx], non_blocking=True)
            self.w2[slot].copy_(pool.w2[pool_idx], non_blocking=True)
            done = torch.cuda.Event(enable_timing=timing)
            done.record(s)
        if timing:
            self.copy_events.append((slot, ev0, done))
        return done

    def release(self, slot: int, stream=None):
        """Mark the slot reusable once `stream` (default: current) passes this point."""
        ev = torch.cuda.Event()
        ev.record(stream if stream is not None else torch.cuda.current_stream())
        self._free[slot] = ev
