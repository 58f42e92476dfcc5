"""Host-resident batches through the device preconditioner with overlapped
transfers.

``HostPipeline(prec).run(inputs, outputs)`` applies a preconditioner (any
callable on device vectors, e.g. :func:`mg_preconditioner`) to a sequence of
host right-hand sides and writes the results into host buffers.  Three
streams overlap the host->device copy of step k+1 and the device->host copy
of step k-1 with the V-cycle of step k, so a batch runs at
max(copy-in, compute, copy-out) per step instead of their sum.  Pinned host
tensors are required for the copies to be asynchronous.

This is the host-facing entry a caller holding numpy/pinned data uses; the
device path underneath is the same C-ABI kernels (no CPU work besides
enqueueing).
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

from . import device as dev


class HostPipeline:
    """``depth`` device input buffers; copy-ins are enqueued ``depth - 1``
    steps ahead so the host->device engine streams back to back while the
    V-cycles run (the preconditioner's Krylov scalars use mapped memory, not
    the copy engines, so they never queue behind these copies)."""

    def __init__(self, prec: Callable, dim: int, depth: int = 3):
        if depth < 2:
            raise ValueError("depth must be >= 2")
        self.prec = prec
        self.dim = dim
        self.depth = depth
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self.comp = torch.cuda.current_stream()
        self.din = [dev.empty(dim) for _ in range(depth)]

    def run(self, inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor],
            start_event: torch.cuda.Event = None) -> None:
        """outputs[k] <- prec(inputs[k]) for every k (host tensors, pinned).  With
        ``start_event`` the first copy waits for it; on return the current
        stream is ordered after the last copy-out."""
        if len(inputs) != len(outputs):
            raise ValueError("inputs and outputs must have the same length")
        n = len(inputs)
        if n == 0:
            return
        D = self.depth
        copied = [torch.cuda.Event() for _ in range(D)]
        consumed = [torch.cuda.Event() for _ in range(D)]

        if start_event is not None:
            self.h2d.wait_event(start_event)

        def copy_in(k):
            s = k % D
            with torch.cuda.stream(self.h2d):
                if k >= D:
                    self.h2d.wait_event(consumed[s])   # the V-cycle of step k-D read din[s]
                self.din[s].copy_(inputs[k], non_blocking=True)
                copied[s].record(self.h2d)

        for k in range(min(D - 1, n)):
            copy_in(k)
        for k in range(n):
            s = k % D
            if k + D - 1 < n:
                copy_in(k + D - 1)
            self.comp.wait_event(copied[s])
            out = self.prec(self.din[s])
            consumed[s].record(self.comp)
            ev = torch.cuda.Event()
            ev.record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev)
                outputs[k].copy_(out, non_blocking=True)
                out.record_stream(self.d2h)
        self.comp.wait_stream(self.d2h)
