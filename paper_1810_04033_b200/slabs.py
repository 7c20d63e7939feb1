"""Slab decomposition of one grid across ranks (one process per GPU).

The reference is single-process (SPEC non-goal).  For the large
BASELINE configs the grid is split along its slowest axis (z in 3D, y in 2D)
into contiguous slabs, one per rank.  Each rank keeps its slab plus G ghost
planes on each side (and one more plane as its local Dirichlet halo), runs
up to `ghost_sweeps` colour-ordered sweeps locally — the ghost planes are
recomputed redundantly, so the owned planes come out exact — and then
exchanges boundary planes with its two neighbours.  G is the dependency
depth of that many sweeps (`sl_ghost_depth`, the same DP the fused kernels
use).  Planes are contiguous in the reference layout, so every exchange is a
plain contiguous send/recv (NCCL P2P over NVLink on GPUs, gloo on CPU in the
tests); the only collective is the final gather.

Correctness contract: after every exchange each rank holds the global state
on [a - G - 1, b + G + 1]; the gathered result equals the 1-rank result bit
for bit (tests/test_slabs.py, world size 2 on gloo).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .kernels import CostModel, NumericsError, StencilKind

__all__ = ["SlabLayout", "SlabRunner", "ghost_depth"]


def ghost_depth(kind: StencilKind, sweeps: int) -> int:
    d = _native.load().sl_ghost_depth(ctypes.byref(kind.descriptor(_native.SL_FORM_D, 0.0)),
                                      kind.dim, sweeps)
    if d < 0:
        raise ValueError(f"no ghost depth for {kind.name}")
    return d


@dataclass(frozen=True)
class SlabLayout:
    """Where rank `rank`'s slab sits in the global grid (slow-axis indices).

    Global interior planes 1..n are split into `world` contiguous ranges
    [a, b].  The local array holds global planes lo..hi (lo/hi are the local
    halo planes), i.e. local plane k is global plane lo + k.
    """

    n: int
    world: int
    rank: int
    ghost: int

    @property
    def a(self) -> int:
        return 1 + (self.rank * self.n) // self.world

    @property
    def b(self) -> int:
        return ((self.rank + 1) * self.n) // self.world

    @property
    def lo(self) -> int:
        return max(0, self.a - self.ghost - 1)

    @property
    def hi(self) -> int:
        return min(self.n + 1, self.b + self.ghost + 1)

    @property
    def local_interior(self) -> int:
        return self.hi - self.lo - 1

    def check(self):
        if self.b - self.a + 1 < self.ghost + 1:
            raise ValueError(f"slab of {self.b - self.a + 1} planes is thinner than ghost+1 = "
                             f"{self.ghost + 1}: use fewer ranks or fewer sweeps per exchange")


def _rng_slice(seed: int, start: int, count: int, kind: str):
    """count draws of default_rng(seed) starting at draw `start` (PCG64 jump,
    so each rank generates only its own planes of the reference init)."""
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(start)
    if kind == "random":
        return rng.random(count)
    return rng.uniform(-1.0, 1.0, count)


class SlabRunner:
    """One rank's slab of a dim-D grid of interior extent n (cubic)."""

    def __init__(self, dim: int, n: int, kind: StencilKind, world: int = 1, rank: int = 0,
                 ghost_sweeps: int = 1, device=None, group=None, compute=None, ghost: int = None):
        import torch
        if kind.dim != dim:
            raise ValueError(f"{kind.name} is {kind.dim}D, not {dim}D")
        self.dim, self.n, self.kind = dim, n, kind
        self.world, self.rank, self.group = world, rank, group
        self.ghost_sweeps = ghost_sweeps
        g = ghost if ghost is not None else ghost_depth(kind, ghost_sweeps)
        self.layout = SlabLayout(n, world, rank, g)
        if world > 1:
            self.layout.check()
        s = n + 2
        nl = self.layout.local_interior
        self.shape = (nl + 2, s) if dim == 2 else (nl + 2, s, s)
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.u = torch.zeros(self.shape, dtype=torch.float64, device=self.device)
        self.f = None
        self.omega = None
        self._compute = compute or self._gpu_compute
        self._ws = None
        self._status = None

    # -- inputs -----------------------------------------------------------------

    def plane_elems(self) -> int:
        return (self.n + 2) ** (self.dim - 1)

    def init(self, seed: int, rhs_seed: int = None, omega: float = 0.8, boundary: float = 0.0):
        """This rank's part of the reference init (mesh.py:102-112) and of
        init_rhs: interior draws in lex order, so global plane p's interior
        draws start at (p-1)*n^(dim-1)."""
        import torch
        n, L = self.n, self.layout
        inner = n ** (self.dim - 1)
        u = np.full(self.shape, boundary)
        g0 = max(L.lo, 1)
        g1 = min(L.hi, n)   # interior global planes held locally
        cnt = (g1 - g0 + 1) * inner
        vals = _rng_slice(seed, (g0 - 1) * inner, cnt, "random").reshape((g1 - g0 + 1,) + (n,) * (self.dim - 1))
        sl = (slice(g0 - L.lo, g1 - L.lo + 1),) + (slice(1, n + 1),) * (self.dim - 1)
        u[sl] = vals
        self.u.copy_(torch.from_numpy(u))
        if rhs_seed is not None:
            f = np.zeros(self.shape)
            f[sl] = _rng_slice(rhs_seed, (g0 - 1) * inner, cnt, "uniform").reshape(vals.shape)
            self.f = torch.from_numpy(f).to(self.device)
            self.omega = float(omega)
        return self

    def load_global(self, u_global, f_global=None, omega: float = 0.8):
        """Take this rank's planes from full global arrays (tests)."""
        import torch
        L = self.layout
        self.u.copy_(torch.as_tensor(np.ascontiguousarray(u_global[L.lo:L.hi + 1])))
        if f_global is not None:
            self.f = torch.as_tensor(np.ascontiguousarray(f_global[L.lo:L.hi + 1])).to(self.device)
            self.omega = float(omega)
        return self

    # -- sweeping ---------------------------------------------------------------

    def _gpu_compute(self, sweeps: int):
        import torch
        lib = _native.require_cuda()
        g = _native.SlGrid()
        g.dim = self.dim
        g.n[0] = self.n
        if self.dim == 2:
            g.n[1] = self.layout.local_interior
            g.origin[1] = self.layout.lo
        else:
            g.n[1] = self.n
            g.n[2] = self.layout.local_interior
            g.origin[2] = self.layout.lo
        g.batch = 1
        g.batch_stride = self.u.numel()
        g.u = self.u.data_ptr()
        form, omega = _native.SL_FORM_R, 0.0
        if self.f is not None:
            g.f = self.f.data_ptr()
            form, omega = _native.SL_FORM_D, self.omega
        st = self.kind.descriptor(form, omega)
        if self._status is None:
            self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        nb = lib.sl_workspace_bytes(ctypes.byref(g), ctypes.byref(st))
        if nb and (self._ws is None or self._ws.numel() * 8 < nb):
            self._ws = torch.empty((nb + 7) // 8, dtype=torch.float64, device=self.device)
        ws_ptr = self._ws.data_ptr() if nb else None
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = lib.sl_sweep(ctypes.byref(g), ctypes.byref(st), sweeps, 0, ws_ptr, nb,
                          self._status.data_ptr(), stream)
        _native.check(rc, "slab sweep")

    def check_status(self):
        if self._status is not None and int(self._status.item()):
            self._status.zero_()
            raise NumericsError("non-finite update in a slab sweep")

    def exchange(self):
        """Boundary planes to/from the neighbouring slabs (contiguous views)."""
        if self.world == 1:
            return
        import torch.distributed as dist
        L, G = self.layout, self.layout.ghost
        ops = []
        if self.rank > 0:   # lower neighbour: send my [a, a+G], receive its [a-G-1, a-1]
            ops.append(dist.P2POp(dist.isend, self.u[L.a - L.lo:L.a - L.lo + G + 1], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self.u[0:L.a - L.lo], self.rank - 1, self.group))
        if self.rank < self.world - 1:   # upper: send my [b-G, b], receive [b+1, b+G+1]
            ops.append(dist.P2POp(dist.isend, self.u[L.b - G - L.lo:L.b - L.lo + 1], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self.u[L.b + 1 - L.lo:], self.rank + 1, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def sweep(self, count: int, cost: CostModel = CostModel()):
        """`count` colour-ordered sweeps of the global grid (exchanging every
        ghost_sweeps sweeps)."""
        if not cost.is_free:
            raise NotImplementedError("slab sweeps run the k = 0 bandwidth path only; "
                                      "use a single-GPU mesh for the cost model")
        while count > 0:
            k = min(self.ghost_sweeps, count)
            self._compute(k)
            count -= k
            self.exchange()
        if self._compute == self._gpu_compute:
            self.check_status()

    def owned(self):
        """This rank's owned planes (global [a, b]) as a view."""
        L = self.layout
        return self.u[L.a - L.lo:L.b - L.lo + 1]

    def gather(self):
        """Full global array on rank 0 (None elsewhere); halo planes included."""
        import torch
        if self.world == 1:
            return self.u.cpu().numpy()
        import torch.distributed as dist
        L = self.layout
        if self.rank != 0:
            dist.send(self.owned().contiguous(), 0, self.group)
            if self.rank == self.world - 1:
                dist.send(self.u[L.b + 1 - L.lo:L.b + 2 - L.lo].contiguous(), 0, self.group)
            return None
        s = self.n + 2
        out = np.zeros((s,) * self.dim)
        out[0:L.b + 1] = self.u[0:L.b + 1 - L.lo].cpu().numpy()   # lo = 0 on rank 0
        for r in range(1, self.world):
            Lr = SlabLayout(self.n, self.world, r, L.ghost)
            buf = torch.empty((Lr.b - Lr.a + 1,) + self.shape[1:], dtype=torch.float64, device=self.device)
            dist.recv(buf, r, self.group)
            out[Lr.a:Lr.b + 1] = buf.cpu().numpy()
            if r == self.world - 1:
                top = torch.empty((1,) + self.shape[1:], dtype=torch.float64, device=self.device)
                dist.recv(top, r, self.group)
                out[self.n + 1] = top.cpu().numpy()[0]
        return out
