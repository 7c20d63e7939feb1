"""Stencil definitions and the in-place cell update, on the GPU.

Mirror of the reference `stencil_lab.kernels` (kernels.py:1-265).  The kinds,
canonical offset order (kernels.py:78-80) and the per-point arithmetic are the
reference's; the arithmetic itself runs in the sm_100a library
(paper_1810_04033_b200/csrc, C ABI in include/stencil_sweep.h):

* Form R — the reference update u_c = (sum_j |w_j| u_j)/w_c
  (kernels.py:224-232), bit-exact;
* Form D — when the mesh carries a right-hand side (`Mesh.set_rhs`), the
  damped update of the BASELINE configs,
  u_c <- u_c + omega*((f_c - (w_c u_c + sum_j w_j u_j))/w_c).

Extension over the reference: `StencilKind` accepts
per-offset weights including zeros (skipped), which is what the trilinear Q1
operator FE27Q1 of BASELINE config 4 needs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from itertools import product

import numpy as np

from . import _native
from .mesh import Mesh

__all__ = ["NumericsError", "StencilKind", "FD5", "FE9", "FD7", "FE27", "FE27Q1", "STENCILS",
           "get_stencil", "CostModel", "ScalarCellKernel", "update_cell", "update_cells_batch",
           "residual_max"]


class NumericsError(ArithmeticError):
    """A cell update produced a non-finite value (reference kernels.py:38-39)."""


class ExchangeTimeout(RuntimeError):
    """A resident (cooperative) sweep kernel gave up waiting for a neighbouring
    tile's exchange flag (status bit 1): the result is not valid."""


def status_error(flag: int, what: str) -> Exception:
    """The exception a non-zero device status word stands for."""
    if flag & 2:
        return ExchangeTimeout(f"tile exchange timed out during {what}")
    return NumericsError(f"non-finite update during {what}")


def _canonical(offsets):
    # outer axis slowest: sort by reversed displacement so x varies fastest
    return tuple(sorted(offsets, key=lambda off: tuple(reversed(off))))


def _face_offsets(dim):
    offs = []
    for a in range(dim):
        for s in (-1, 1):
            off = [0] * dim
            off[a] = s
            offs.append(tuple(off))
    return _canonical(offs)


def _box_offsets(dim):
    return _canonical([off for off in product((-1, 0, 1), repeat=dim) if any(off)])


_SHAPES = {
    _native.SL_FD5: _face_offsets(2),
    _native.SL_FE9: _box_offsets(2),
    _native.SL_FD7: _face_offsets(3),
    _native.SL_FE27: _box_offsets(3),
}


@dataclass(frozen=True)
class StencilKind:
    """One stencil shape: neighbour offsets, their weights, centre weight.

    Same fields as the reference (kernels.py:42-75); weights may be zero
    (skipped by every update) but not positive.
    """

    name: str
    dim: int
    offsets: tuple
    weights: tuple
    centre_weight: float
    colours: int

    def __post_init__(self):
        assert len(self.offsets) == len(self.weights)
        assert all(w <= 0.0 for w in self.weights)
        assert any(w < 0.0 for w in self.weights)
        row_sum = self.centre_weight + sum(self.weights)
        assert abs(row_sum) < 1e-12, f"{self.name}: row sum {row_sum}"

    @property
    def entry_count(self) -> int:
        return len(self.offsets) + 1

    def flat_offsets(self, mesh: Mesh) -> tuple:
        return tuple(sum(o * s for o, s in zip(off, mesh.strides)) for off in self.offsets)

    def is_adjacent(self, a, b) -> bool:
        if a == b:
            return False
        delta = tuple(bi - ai for ai, bi in zip(a, b))
        return delta in self._offset_set()

    def _offset_set(self):
        return frozenset(self.offsets)

    # -- C-ABI descriptor ------------------------------------------------------

    def shape_id(self) -> int:
        for sid, offs in _SHAPES.items():
            if offs == tuple(self.offsets):
                return sid
        raise NotImplementedError(
            f"{self.name}: offsets are not one of the canonical FD5/FE9/FD7/FE27 sets")

    def descriptor(self, form: int, omega: float = 0.0) -> _native.SlStencil:
        s = _native.SlStencil()
        s.shape = self.shape_id()
        s.colours = self.colours
        s.form = form
        for j, w in enumerate(self.weights):
            s.w[j] = w
        s.wc = self.centre_weight
        s.omega = omega
        return s


FD5 = StencilKind("fd5", 2, _face_offsets(2), (-1.0,) * 4, 4.0, 2)
FE9 = StencilKind("fe9", 2, _box_offsets(2), (-1.0 / 3.0,) * 8, 8.0 / 3.0, 4)
FD7 = StencilKind("fd7", 3, _face_offsets(3), (-1.0,) * 6, 6.0, 2)
FE27 = StencilKind("fe27", 3, _box_offsets(3), (-1.0,) * 26, 26.0, 8)


def _q1_weight(off):
    return {1: 0.0, 2: -1.0 / 6.0, 3: -1.0 / 12.0}[sum(1 for c in off if c)]


# BASELINE config 4: trilinear Q1 FE Laplacian — centre 8/3, faces 0,
# edges -1/6, corners -1/12; 2x2x2 parity colouring.
FE27Q1 = StencilKind("fe27q1", 3, _box_offsets(3), tuple(_q1_weight(o) for o in _box_offsets(3)),
                     8.0 / 3.0, 8)

STENCILS = {k.name: k for k in (FD5, FE9, FD7, FE27, FE27Q1)}


def get_stencil(name: str) -> StencilKind:
    try:
        return STENCILS[name.lower()]
    except KeyError:
        raise KeyError(f"unknown stencil {name!r}; choose from {sorted(STENCILS)}") from None


@dataclass(frozen=True)
class CostModel:
    """Per-cell extra-work parameter k (reference kernels.py:113-145).

    k = 0 runs the fused bandwidth kernels; k > 0 (const or ramp) runs the
    cost kernel (csrc/k5_cost.cu): k sine evaluations per stencil entry whose
    sum is folded in as 0.0*d, so the values are bit-identical to k = 0 and
    the consumed tally is returned by the sweep.
    """

    mode: str = "const"
    k: int = 0

    def __post_init__(self):
        if self.mode not in ("const", "ramp"):
            raise ValueError(f"cost mode must be 'const' or 'ramp', got {self.mode!r}")
        if self.k < 0:
            raise ValueError("k must be non-negative")

    def k_for_rank(self, rank: int, total: int) -> int:
        if not 0 <= rank < total:
            raise ValueError(f"rank {rank} outside [0, {total})")
        if self.mode == "const":
            return self.k
        return min((100 * rank) // total, 99)

    def k_table(self, total: int) -> np.ndarray:
        if self.mode == "const":
            return np.full(total, self.k, dtype=np.int64)
        return np.minimum((100 * np.arange(total, dtype=np.int64)) // total, 99)

    def describe(self) -> str:
        return f"const:{self.k}" if self.mode == "const" else "ramp"

    @property
    def is_free(self) -> bool:
        """k = 0 everywhere: the bandwidth kernels apply."""
        return self.mode == "const" and self.k == 0

    def descriptor(self, d_work=None):
        c = _native.SlCost()
        c.mode = _native.SL_COST_CONST if self.mode == "const" else _native.SL_COST_RAMP
        c.k = self.k if self.mode == "const" else 0
        c.d_work = d_work
        return c


# ---------------------------------------------------------------------------
# device plumbing shared with strategies.py

class DeviceCall:
    """C-ABI descriptors + status word for one (mesh, kind) pair."""

    __slots__ = ("mesh", "kind", "grid", "stencil", "status", "stream", "_torch", "_u", "_f")

    def __init__(self, mesh: Mesh, kind: StencilKind):
        if kind.dim != mesh.dim:
            raise ValueError(f"{kind.name} is {kind.dim}D but mesh is {mesh.dim}D")
        _native.require_cuda()
        import torch
        self._torch = torch
        self.mesh = mesh
        self.kind = kind
        u = mesh.device_values()
        g = _native.SlGrid()
        g.dim = mesh.dim
        for a in range(3):
            g.n[a] = mesh.n if a < mesh.dim else 0
        g.batch = 1
        g.batch_stride = mesh.size
        g.u = u.data_ptr()
        self._u = u                 # the descriptor's pointers stay owned while bound
        self._f = None
        form = _native.SL_FORM_R
        omega = 0.0
        if mesh.has_rhs:
            form = _native.SL_FORM_D
            self._f = mesh.rhs_device()
            g.f = self._f.data_ptr()
            omega = mesh.omega
        self.grid = g
        self.stencil = kind.descriptor(form, omega)
        self.status = torch.zeros(1, dtype=torch.int32, device=u.device)
        self.stream = torch.cuda.current_stream(u.device).cuda_stream

    def refresh(self):
        """Re-bind u and f before a call: host edits of `values` are uploaded,
        and a right-hand side replaced since the last call (`set_rhs`,
        `init_rhs`) is re-read — the descriptor never keeps a freed f."""
        self._u = self.mesh.device_values()
        self.grid.u = self._u.data_ptr()
        if self.mesh.has_rhs:
            self._f = self.mesh.rhs_device()
            self.grid.f = self._f.data_ptr()
        self.stream = self._torch.cuda.current_stream(self._u.device).cuda_stream

    def check_status(self, what: str):
        flag = int(self.status.item())
        if flag:
            self.status.zero_()
            raise status_error(flag, what)


def _call(mesh: Mesh, kind: StencilKind) -> DeviceCall:
    return DeviceCall(mesh, kind)


class ScalarCellKernel:
    """Single-cell in-place updates (reference kernels.py:148-200), one
    one-cell launch each; bitwise equal to the batch path."""

    __slots__ = ("mesh", "kind", "work_sum")

    def __init__(self, mesh: Mesh, kind: StencilKind):
        if kind.dim != mesh.dim:
            raise ValueError(f"{kind.name} is {kind.dim}D but mesh is {mesh.dim}D")
        self.mesh = mesh
        self.kind = kind
        self.work_sum = 0.0

    def update(self, nbrs, centre: int, k: int) -> float:
        self.work_sum += update_cells_batch(self.mesh, self.kind,
                                            np.array([centre], dtype=np.int64), k)
        return float(self.mesh.device_values()[centre].item())


def update_cell(mesh: Mesh, kind: StencilKind, coord, k: int = 0) -> float:
    if not mesh.is_interior(coord):
        raise IndexError(f"{coord!r} is not an interior cell")
    centre = mesh.flat_index(coord)
    nbrs = tuple(centre + d for d in kind.flat_offsets(mesh))
    return ScalarCellKernel(mesh, kind).update(nbrs, centre, k)


def update_cells_batch(mesh: Mesh, kind: StencilKind, flats, k: int) -> float:
    """In-place update of mutually non-adjacent interior cells (reference
    kernels.py:212-251) on the GPU; returns the consumed sine tally (0.0 when
    k == 0)."""
    if k < 0:
        raise ValueError("k must be non-negative")
    call = _call(mesh, kind)
    import torch
    if isinstance(flats, torch.Tensor):
        d_flats = flats.to(device=call.status.device, dtype=torch.int64)
    else:
        d_flats = torch.from_numpy(np.ascontiguousarray(flats, dtype=np.int64)).to(call.status.device)
    lib = _native.load()
    if k == 0:
        rc = lib.sl_update_cells(ctypes.byref(call.grid), ctypes.byref(call.stencil),
                                 d_flats.data_ptr(), d_flats.numel(),
                                 call.status.data_ptr(), call.stream)
        _native.check(rc, "update_cells_batch")
        call.check_status("update_cells_batch")
        return 0.0
    work = torch.zeros(1, dtype=torch.float64, device=call.status.device)
    cost = CostModel("const", k).descriptor(work.data_ptr())
    rc = lib.sl_update_cells_cost(ctypes.byref(call.grid), ctypes.byref(call.stencil),
                                  d_flats.data_ptr(), d_flats.numel(), ctypes.byref(cost),
                                  call.status.data_ptr(), call.stream)
    _native.check(rc, "update_cells_batch")
    call.check_status("update_cells_batch")
    return float(work.item())


def residual_max(mesh: Mesh, kind: StencilKind) -> float:
    """max over interior cells of |w_c u + sum_j w_j u_j| (reference
    kernels.py:254-265); with a right-hand side, max |f - A u|."""
    call = _call(mesh, kind)
    import torch
    out = torch.zeros(1, dtype=torch.float64, device=call.status.device)
    rc = _native.load().sl_residual_max(ctypes.byref(call.grid), ctypes.byref(call.stencil),
                                        out.data_ptr(), call.stream)
    _native.check(rc, "residual_max")
    return float(out.item())
