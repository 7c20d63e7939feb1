"""Overlapped host -> device -> host sweep jobs (throughput path).

A job is one host problem — u (and f for Form D) in pinned memory — that is
uploaded, swept `sweeps` times with the colour-ordered schedule (one
`sl_sweep` call, the same C-ABI entry as `run_sweeps`) and downloaded into a
caller-owned pinned buffer.  A single job is bound by PCIe (it moves 24 B
per grid point over the bus and sweeps them at HBM speed), so the pipeline
keeps `depth` device buffer sets and three CUDA streams: while job i sweeps,
job i+1 uploads and job i-1 downloads; host<->device copies in both
directions run on the two copy engines concurrently with the sweeps.  Every
job's result is bitwise the result of `run_sweeps` on the same inputs.

The reference is a single-process CPU library and has no counterpart; this
is the serving-side wrapper around the drop-in sweep (bench.py's e2e).
"""

from __future__ import annotations

import ctypes

from . import _native
from .kernels import NumericsError, StencilKind, status_error

__all__ = ["SweepPipeline"]


class SweepPipeline:
    """`depth` jobs in flight on one device.

    shape: (n+2,)*dim for one dense grid, or (B, n+2, n+2) with batch=True
    for a batch of independent 2D patches (BASELINE config 5).
    """

    def __init__(self, kind: StencilKind, shape, sweeps: int, omega: float = None,
                 batch: bool = False, depth: int = 2, device=None, flags: int = 0):
        import torch
        self._lib = _native.require_cuda()
        if depth < 1 or sweeps < 0:
            raise ValueError("depth >= 1 and sweeps >= 0 required")
        shape = tuple(int(s) for s in shape)
        dim = 2 if batch else len(shape)
        if kind.dim != dim:
            raise ValueError(f"{kind.name} is {kind.dim}D, the jobs are {dim}D")
        if batch and (len(shape) != 3 or shape[1] != shape[2]):
            raise ValueError("batch jobs have shape (B, n+2, n+2)")
        self.kind, self.shape, self.sweeps, self.flags = kind, shape, sweeps, flags
        self.omega = omega
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        form = _native.SL_FORM_D if omega is not None else _native.SL_FORM_R
        self._stencil = kind.descriptor(form, omega or 0.0)
        side = shape[-1]
        self._slots = []
        for _ in range(depth):
            u = torch.empty(shape, dtype=torch.float64, device=self.device)
            f = torch.empty(shape, dtype=torch.float64, device=self.device) if omega is not None else None
            g = _native.SlGrid()
            g.dim = dim
            for a in range(dim):
                g.n[a] = side - 2
            g.batch = shape[0] if batch else 1
            g.batch_stride = side * side if batch else u.numel()
            g.u = u.data_ptr()
            g.f = f.data_ptr() if f is not None else None
            nb = 0 if flags & ~_native.SL_FLAG_STREAM else self._lib.sl_workspace_bytes(ctypes.byref(g), ctypes.byref(self._stencil))
            ws = torch.empty((nb + 7) // 8, dtype=torch.float64, device=self.device) if nb else None
            self._slots.append({
                "u": u, "f": f, "grid": g, "ws": ws, "ws_bytes": nb,
                "status": torch.zeros(1, dtype=torch.int32, device=self.device),
                "up": torch.cuda.Event(), "done": torch.cuda.Event(), "free": torch.cuda.Event(),
                "used": False})
        self._s_up = torch.cuda.Stream(self.device)
        self._s_comp = torch.cuda.Stream(self.device)
        self._s_down = torch.cuda.Stream(self.device)
        self._next = 0
        self._in_flight = []

    def submit(self, u, f=None, out=None):
        """Queue one job: pinned host u (and f), result into pinned `out`
        (u's shape).  Returns immediately; `drain()` waits for all jobs."""
        import torch
        if (f is None) != (self.omega is None):
            raise ValueError("f is required exactly when the pipeline was built with omega")
        s = self._slots[self._next % len(self._slots)]
        self._next += 1
        if s["used"]:   # the slot's previous job must have left the device
            self._s_up.wait_event(s["free"])
        with torch.cuda.stream(self._s_up):
            s["u"].copy_(torch.as_tensor(u).reshape(self.shape), non_blocking=True)
            if f is not None:
                s["f"].copy_(torch.as_tensor(f).reshape(self.shape), non_blocking=True)
            s["up"].record(self._s_up)
        self._s_comp.wait_event(s["up"])
        ws = s["ws"]
        rc = self._lib.sl_sweep(ctypes.byref(s["grid"]), ctypes.byref(self._stencil), self.sweeps,
                                self.flags, ws.data_ptr() if ws is not None else None, s["ws_bytes"],
                                s["status"].data_ptr(), self._s_comp.cuda_stream)
        _native.check(rc, "pipelined sweep")
        s["done"].record(self._s_comp)
        self._s_down.wait_event(s["done"])
        with torch.cuda.stream(self._s_down):
            if out is not None:
                out.copy_(s["u"].reshape(out.shape), non_blocking=True)
            s["free"].record(self._s_down)
        s["used"] = True
        self._in_flight.append(s)
        return out

    def drain(self):
        """Wait for every queued job; NumericsError if any update was non-finite."""
        for s in self._in_flight:
            s["free"].synchronize()
        bad = 0
        for s in self._slots:
            bad |= int(s["status"].item())
        for s in self._slots:
            s["status"].zero_()
        self._in_flight = []
        if bad:
            raise status_error(bad, "a pipelined sweep")
