"""Batched small patches (BASELINE config 5): many independent meshes.

The reference has no batch API; its semantics for a batch is
"colouring applied to each patch as its own Mesh" (colour parity relative to
the patch's own cell (1,1), halo held fixed).  A `PatchBatch` stores B such
grids back to back in one device buffer — `(B, n+2, n+2)` fp64, each patch in
the reference's layout — and sweeps all of them with one C-ABI call
(`sl_sweep` with `sl_grid.batch = B`): the K3 kernel keeps each 16x16 patch in
one warp's registers for all sweeps; other sizes run the per-colour path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .kernels import CostModel, NumericsError, StencilKind

__all__ = ["PatchBatch", "init_patches"]


class PatchBatch:
    """B independent (n+2)^2 grids with optional right-hand sides (Form D)."""

    def __init__(self, u, f=None, omega: float = 0.8, device=None):
        import torch
        _native.require_cuda()
        u = torch.as_tensor(u, dtype=torch.float64)
        if u.dim() != 3 or u.shape[1] != u.shape[2] or u.shape[1] < 3:
            raise ValueError("u must have shape (B, n+2, n+2)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.u = u.to(dev).contiguous()
        self.f = None
        self.omega = None
        if f is not None:
            f = torch.as_tensor(f, dtype=torch.float64)
            if f.shape != u.shape:
                raise ValueError("f must have u's shape")
            self.f = f.to(dev).contiguous()
            self.omega = float(omega)
        self.batch = u.shape[0]
        self.n = u.shape[1] - 2
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)

    def upload(self, u, f=None):
        """Copy new patch values (and rhs) from the host into the device buffers
        (pinned CPU tensors copy asynchronously on the current stream)."""
        import torch
        self.u.copy_(torch.as_tensor(u, dtype=torch.float64).reshape(self.u.shape), non_blocking=True)
        if f is not None:
            if self.f is None:
                raise ValueError("this batch was built without a right-hand side")
            self.f.copy_(torch.as_tensor(f, dtype=torch.float64).reshape(self.f.shape), non_blocking=True)

    def values(self, out=None) -> np.ndarray:
        """Host copy of the patches; `out` (a pinned CPU tensor of u's shape)
        receives it without allocating."""
        if out is None:
            return self.u.cpu().numpy()
        out.copy_(self.u)
        return out.numpy()

    def _descriptors(self, kind: StencilKind):
        if kind.dim != 2:
            raise ValueError(f"{kind.name} is {kind.dim}D but patches are 2D")
        g = _native.SlGrid()
        g.dim = 2
        g.n[0] = g.n[1] = self.n
        g.batch = self.batch
        g.batch_stride = (self.n + 2) ** 2
        g.u = self.u.data_ptr()
        form, omega = _native.SL_FORM_R, 0.0
        if self.f is not None:
            g.f = self.f.data_ptr()
            form, omega = _native.SL_FORM_D, self.omega
        return g, kind.descriptor(form, omega)

    def sweep(self, kind: StencilKind, sweeps: int = 1, cost: CostModel = CostModel(),
              flags: int = 0, check: bool = True):
        """`sweeps` colour-ordered sweeps of every patch, in place; returns the
        cost-model sine tally (0.0 when k == 0)."""
        import torch
        g, s = self._descriptors(kind)
        stream = torch.cuda.current_stream(self.u.device).cuda_stream
        work = None
        if cost.is_free:
            rc = _native.load().sl_sweep(ctypes.byref(g), ctypes.byref(s), sweeps, flags, None, 0,
                                         self.status.data_ptr(), stream)
        else:
            w = torch.zeros(1, dtype=torch.float64, device=self.u.device)
            c = cost.descriptor(w.data_ptr())
            rc = _native.load().sl_sweep_cost(ctypes.byref(g), ctypes.byref(s), ctypes.byref(c),
                                              sweeps, flags & _native.SL_FLAG_LEX,
                                              self.status.data_ptr(), stream)
            work = w
        _native.check(rc, "patch sweep")
        if check and int(self.status.item()):
            self.status.zero_()
            raise NumericsError("non-finite update in a patch sweep")
        return 0.0 if work is None else float(work.item())


def init_patches(batch: int, n: int, seed: int):
    """Config 5 inputs: u incl. halo ~ U[0,1) =
    default_rng(seed).random((B, n+2, n+2)); f ~ U[-1,1) =
    default_rng(seed+1).uniform(-1, 1, (B, n, n)), dense with zero halo."""
    s = n + 2
    u = np.random.default_rng(seed).random((batch, s, s))
    f = np.zeros((batch, s, s))
    f[:, 1:n + 1, 1:n + 1] = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, (batch, n, n))
    return u, f
