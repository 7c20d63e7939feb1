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

Each sweep is one fused pass between two slab buffers (`sl_sweep_pass`, no
copy back).  The last sweep of a round writes only the owned planes; the
ghost planes of the new state are the received ones, so they are never
recomputed.  With `overlap=True` that last sweep runs as three launches —
the G+1 planes at each end first, whose exchange then starts (NCCL runs on
its own stream after the boundary passes) while the interior pass runs.  It
is off by default: at the BASELINE sizes a 3-plane pass costs a full chunk
warm-up, so the two extra launches cost more than the NVLink transfer they
hide (measured compute per sweep at 8 slabs: config 3 157 vs 115 us,
config 4 1106 vs 977 us, config 2 +13 %; the transfer is ~20 / ~70 / ~5 us).

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
                 ghost_sweeps: int = 1, device=None, group=None, compute=None, ghost: int = None,
                 overlap: bool = False, exchange: str = "nccl"):
        import torch
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', not {exchange!r}")
        if kind.dim != dim:
            raise ValueError(f"{kind.name} is {kind.dim}D, not {dim}D")
        self.dim, self.n, self.kind = dim, n, kind
        self.world, self.rank, self.group = world, rank, group
        self.ghost_sweeps = ghost_sweeps
        self.overlap = overlap   # boundary passes first, exchange during the interior pass
        # "peer": the last pass of a round stores the boundary planes straight into the
        # neighbours' ghost planes (peer memory); a stream-ordered barrier ends the round
        self.exchange_mode = exchange
        g = ghost if ghost is not None else ghost_depth(kind, ghost_sweeps)
        self.layout = SlabLayout(n, world, rank, g)
        if world > 1:
            self.layout.check()
        s = n + 2
        nl = self.layout.local_interior
        self.shape = (nl + 2, s) if dim == 2 else (nl + 2, s, s)
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self._symm = None
        import torch.distributed as dist
        if (exchange == "peer" and world > 1 and self.device.type == "cuda" and dist.is_available()
                and dist.is_initialized()):
            bufs = self._symmetric_buffers()     # one process per GPU: peer memory over NVLink
        else:
            bufs = (torch.zeros(self.shape, dtype=torch.float64, device=self.device),
                    torch.zeros(self.shape, dtype=torch.float64, device=self.device))
        self._bufs = bufs                     # fixed roles: buffer 0 / 1 of the ping-pong
        self._cur = 0                         # index of the buffer holding the current state
        self.u, self._u2 = bufs               # the other buffer of the pass ping-pong
        self._peers = None                    # per dst buffer: (pdn, pup) element pointers
        self.f = None
        self.omega = None
        self._pass = compute or self._gpu_pass   # (src, dst, z0, z1): one sweep into dst planes [z0, z1)
        self._residual = None                    # tests: (runner) -> local max over the owned planes
        self._desc = None
        self._fused = None
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
        self._u2.copy_(self.u)
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
        self._u2.copy_(self.u)
        if f_global is not None:
            self.f = torch.as_tensor(np.ascontiguousarray(f_global[L.lo:L.hi + 1])).to(self.device)
            self.omega = float(omega)
        return self

    # -- sweeping ---------------------------------------------------------------

    def _descriptors(self):
        """(grid, stencil) descriptors of the local slab (u is set per call)."""
        if self._desc is None:
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
            form, omega = _native.SL_FORM_R, 0.0
            if self.f is not None:
                g.f = self.f.data_ptr()
                form, omega = _native.SL_FORM_D, self.omega
            self._desc = (g, self.kind.descriptor(form, omega))
        return self._desc

    def _gpu_pass(self, src, dst, z0: int, z1: int):
        import torch
        lib = _native.require_cuda()
        g, st = self._descriptors()
        if self._status is None:
            self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = lib.sl_sweep_pass(ctypes.byref(g), ctypes.byref(st), src.data_ptr(), dst.data_ptr(),
                               z0, z1, self._status.data_ptr(), stream)
        _native.check(rc, "slab pass")

    def _gpu_fused(self) -> bool:
        """Whether a streaming pass kernel covers this slab (an empty plane
        window probes it without launching)."""
        if self._fused is None:
            import torch
            lib = _native.require_cuda()
            g, st = self._descriptors()
            if self._status is None:
                self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
            rc = lib.sl_sweep_pass(ctypes.byref(g), ctypes.byref(st), self.u.data_ptr(),
                                   self._u2.data_ptr(), 0, 0, self._status.data_ptr(), None)
            if rc not in (_native.SL_OK, _native.SL_E_UNSUPPORTED):
                _native.check(rc, "slab pass")
            self._fused = rc == _native.SL_OK
        return self._fused

    def _gpu_inplace(self, k: int):
        """k sweeps in place with the per-colour kernels (grids no streaming
        pass kernel covers, e.g. an odd row length)."""
        import torch
        lib = _native.require_cuda()
        g, st = self._descriptors()
        g.u = self.u.data_ptr()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = lib.sl_sweep(ctypes.byref(g), ctypes.byref(st), k, 0, None, 0,
                          self._status.data_ptr(), stream)
        _native.check(rc, "slab sweep")

    def check_status(self):
        if self._status is not None and int(self._status.item()):
            self._status.zero_()
            raise NumericsError("non-finite update in a slab sweep")

    def _exchange_ops(self, buf):
        import torch.distributed as dist
        L, G = self.layout, self.layout.ghost
        ops = []
        if self.rank > 0:   # lower neighbour: send my [a, a+G], receive its [a-G-1, a-1]
            ops.append(dist.P2POp(dist.isend, buf[L.a - L.lo:L.a - L.lo + G + 1], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[0:L.a - L.lo], self.rank - 1, self.group))
        if self.rank < self.world - 1:   # upper: send my [b-G, b], receive [b+1, b+G+1]
            ops.append(dist.P2POp(dist.isend, buf[L.b - G - L.lo:L.b - L.lo + 1], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[L.b + 1 - L.lo:], self.rank + 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def exchange(self):
        """Boundary planes of the current state to/from the neighbouring slabs."""
        if self.world == 1:
            return
        for req in self._exchange_ops(self.u):
            req.wait()

    def _swap(self):
        self.u, self._u2 = self._u2, self.u
        self._cur ^= 1

    # -- fused peer exchange ------------------------------------------------------

    def _symmetric_buffers(self):
        """Both slab buffers in symmetric memory (same size on every rank),
        so each rank can address its neighbours' buffers over NVLink."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        nl_max = max(SlabLayout(self.n, self.world, r, self.layout.ghost).local_interior
                     for r in range(self.world))
        full = (nl_max + 2,) + self.shape[1:]
        group = self.group if self.group is not None else dist.group.WORLD
        bufs, hdls = [], []
        for _ in range(2):
            t = symm_mem.empty(*full, dtype=torch.float64, device=self.device)
            hdls.append(symm_mem.rendezvous(t, group))
            t.zero_()
            bufs.append(t[:self.shape[0]])
        self._symm = hdls
        ranks = dist.get_process_group_ranks(group)
        lo_of = [SlabLayout(self.n, self.world, r, self.layout.ghost).lo for r in range(self.world)]
        pe = self.plane_elems() * 8
        peers = []
        for d in range(2):
            ptrs = hdls[d].buffer_ptrs
            dn = ptrs[self.rank - 1] + (self.layout.lo - lo_of[self.rank - 1]) * pe if self.rank > 0 else None
            up = (ptrs[self.rank + 1] + (self.layout.lo - lo_of[self.rank + 1]) * pe
                  if self.rank < self.world - 1 else None)
            peers.append((dn, up))
        del ranks
        self._peer_init = peers
        hdls[0].barrier(channel=0)
        return tuple(bufs)

    def connect_peers(self, lower=None, upper=None):
        """Peer exchange between runners of one process (tests; one device):
        the neighbours' buffers stand in for peer memory."""
        pe = self.plane_elems() * 8
        peers = []
        for d in range(2):
            dn = (lower._bufs[d].data_ptr() + (self.layout.lo - lower.layout.lo) * pe) if lower else None
            up = (upper._bufs[d].data_ptr() + (self.layout.lo - upper.layout.lo) * pe) if upper else None
            peers.append((dn, up))
        self._peers = peers

    def _gpu_pass_peer(self, src, dst, z0: int, z1: int, peers):
        import torch
        lib = _native.require_cuda()
        g, st = self._descriptors()
        if self._status is None:
            self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        L, G = self.layout, self.layout.ghost
        a, b = L.a - L.lo, L.b - L.lo
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = lib.sl_sweep_pass_peer(ctypes.byref(g), ctypes.byref(st), src.data_ptr(), dst.data_ptr(),
                                    z0, z1, peers[0], a + G, peers[1], b - G,
                                    self._status.data_ptr(), stream)
        _native.check(rc, "slab peer pass")

    def round_begin(self, k: int):
        """The k-1 redundant sweeps of a round over the whole local slab."""
        whole = self.shape[0]
        for _ in range(k - 1):
            self._pass(self.u, self._u2, 0, whole)
            self._swap()

    def round_end_peer(self):
        """Last sweep of a round in peer mode: one pass over the owned planes
        whose boundary-plane stores also land in the neighbours' ghost planes."""
        L = self.layout
        if self._peers is None:
            if self._symm is None:
                raise RuntimeError("peer exchange needs connect_peers() or symmetric buffers")
            self._peers = self._peer_init
        self._gpu_pass_peer(self.u, self._u2, L.a - L.lo, L.b - L.lo + 1, self._peers[self._cur ^ 1])
        self._swap()

    def compute_round(self, k: int, exchange: bool = False):
        """k sweeps of the slab (k <= ghost_sweeps); with `exchange`, the
        boundary planes of the result are traded with the neighbours while
        the interior pass runs.  Without it the ghost planes of the result
        are left for the caller to fill (tests emulate the exchange)."""
        L, G = self.layout, self.layout.ghost
        if self._pass == self._gpu_pass and not self._gpu_fused():
            self._gpu_inplace(k)
            if exchange:
                self.exchange()
            return
        self.round_begin(k)
        if self.exchange_mode == "peer" and self.world > 1:
            if k > 1 and self._symm is not None:
                # neighbours' redundant passes write whole buffers, ghost planes included:
                # they must be done before this rank's stores reach those planes
                self._symm[0].barrier(channel=0)
            self.round_end_peer()
            if exchange and self._symm is not None:
                self._symm[0].barrier(channel=0)   # every rank's stores are in before anyone reads
            return
        a, b = L.a - L.lo, L.b - L.lo          # owned planes, local indices
        if self.world == 1 or not self.overlap or b - a + 1 <= 2 * (G + 1):
            self._pass(self.u, self._u2, a, b + 1)
            reqs = self._exchange_ops(self._u2) if exchange and self.world > 1 else []
        else:
            self._pass(self.u, self._u2, a, a + G + 1)
            self._pass(self.u, self._u2, b - G, b + 1)
            reqs = self._exchange_ops(self._u2) if exchange else []
            self._pass(self.u, self._u2, a + G + 1, b - G)   # overlaps the exchange
        for req in reqs:
            req.wait()
        self._swap()

    def sweep(self, count: int, cost: CostModel = CostModel()):
        """`count` colour-ordered sweeps of the global grid (exchanging every
        ghost_sweeps sweeps)."""
        if not cost.is_free:
            raise NotImplementedError("slab sweeps run the k = 0 bandwidth path only; "
                                      "use a single-GPU mesh for the cost model")
        # planes no pass writes (global halo) must agree in both buffers
        self._u2[0].copy_(self.u[0])
        self._u2[-1].copy_(self.u[-1])
        while count > 0:
            k = min(self.ghost_sweeps, count)
            self.compute_round(k, exchange=True)
            count -= k
        if self._pass == self._gpu_pass:
            self.check_status()

    # -- residual (reference kernels.py:254-265, convergence loop bench.py:445-474) --

    def _gpu_residual(self) -> float:
        """max |f - A u| (|A u| without f) over this rank's owned planes, on the
        device: sl_residual_max over a window whose interior is the owned
        planes and whose halo planes are the ghost planes around them."""
        import torch
        lib = _native.require_cuda()
        g0, st = self._descriptors()
        L = self.layout
        off = (L.a - L.lo - 1) * self.plane_elems() * 8
        g = _native.SlGrid()
        ctypes.memmove(ctypes.byref(g), ctypes.byref(g0), ctypes.sizeof(g))
        g.n[self.dim - 1] = L.b - L.a + 1
        g.origin[self.dim - 1] = 0
        g.u = self.u.data_ptr() + off
        if self.f is not None:
            g.f = self.f.data_ptr() + off
        out = torch.zeros(1, dtype=torch.float64, device=self.device)
        rc = lib.sl_residual_max(ctypes.byref(g), ctypes.byref(st), out.data_ptr(),
                                 torch.cuda.current_stream(self.device).cuda_stream)
        _native.check(rc, "slab residual")
        return float(out.item())

    def residual_max(self) -> float:
        """Residual of the global grid's current state: each rank reduces its
        owned planes (the exchanged ghost planes supply their neighbours),
        then all_reduce(MAX) — equal to the single-domain residual_max bit for
        bit (a max does not depend on the order it is taken in)."""
        import torch
        local = self._residual(self) if self._residual is not None else self._gpu_residual()
        if self.world == 1:
            return local
        import torch.distributed as dist
        on_gpu = dist.get_backend(self.group) == "nccl"
        t = torch.tensor([local], dtype=torch.float64,
                         device=self.device if on_gpu else torch.device("cpu"))
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

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
