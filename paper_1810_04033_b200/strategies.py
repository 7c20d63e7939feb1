"""Colour-scheduled sweeps on the GPU — mirror of reference strategies.py.

Covered strategies:
  colouring   strategies.py:348-393 -> sl_sweep (fused K2 / per-colour K1)
  hyb-sync    strategies.py:503-527 -> same result as colouring, bit for bit
  hyb-depend  strategies.py:490-500    (reference tests/test_strategies.py:142-152),
                                        so they run the same kernel
  serial      strategies.py:341-345 -> lexicographic Gauss-Seidel as hyperplane
  taskgraph   strategies.py:477-487    wavefronts (SL_FLAG_LEX); taskgraph equals
                                        serial bit for bit (tests/test_strategies.py:125-139)
Out of scope: nd (nested dissection) — its order depends on the CPU worker
count; it raises NotImplementedError.

Colour classes are parity relative to cell (1,..,1) (strategies.py:62-69):
face stencils 2-colour on coordinate-sum parity, full neighbourhoods use the
2^d per-axis parity code; colours run 0..c-1 within a sweep.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .kernels import CostModel, DeviceCall, StencilKind
from .mesh import Mesh
from .pool import DevicePool, Schedule

__all__ = ["STRATEGY_IDS", "GPU_STRATEGIES", "canonical_strategy", "colour_count", "colour_of",
           "SweepPlan", "sweep_colouring", "sweep_colouring_reference", "sweep_hyb_sync",
           "sweep_hyb_depend", "sweep_serial", "sweep_nested_dissection", "sweep_taskgraph",
           "run_sweep", "run_sweeps"]

STRATEGY_IDS = ("serial", "colouring", "nd", "taskgraph", "hyb-depend", "hyb-sync")
GPU_STRATEGIES = ("serial", "colouring", "taskgraph", "hyb-depend", "hyb-sync")

_ALIASES = {
    "nested_dissection": "nd",
    "hyb_depend": "hyb-depend",
    "hyb_sync": "hyb-sync",
}


def canonical_strategy(name: str) -> str:
    name = _ALIASES.get(name, name)
    if name not in STRATEGY_IDS:
        raise ValueError(f"unknown strategy {name!r}; choose from {STRATEGY_IDS}")
    return name


def colour_count(kind: StencilKind) -> int:
    return kind.colours


def colour_of(kind: StencilKind, coord) -> int:
    """Colour class of an interior cell (parity relative to cell (1,..,1))."""
    if kind.colours == 2:
        return (sum(coord) - kind.dim) % 2
    code = 0
    for a, c in enumerate(coord):
        code |= ((c - 1) & 1) << a
    return code


class SweepPlan:
    """Per-(mesh, kind, cost) state, reused across sweeps.

    The reference plan materialises per-cell index arrays (~65 B/point,
    SURVEY.md D4); the GPU needs none of that — it holds the C-ABI
    descriptors and the fusion workspace.  The colour partition is still
    available (computed on demand on the host) for API compatibility.
    """

    def __init__(self, mesh: Mesh, kind: StencilKind, cost: CostModel):
        if kind.dim != mesh.dim:
            raise ValueError(f"{kind.name} is {kind.dim}D but mesh is {mesh.dim}D")
        self.mesh = mesh
        self.kind = kind
        self.cost = cost
        self.const_k = cost.k if cost.mode == "const" else None
        self.flat_offsets = kind.flat_offsets(mesh)
        self._call = None
        self._key = None
        self._colour_cells = None

    # host-side colour partition (reference strategies.py:188-222)
    def _colour_ids(self) -> np.ndarray:
        side = self.mesh.side
        rem = self.mesh.interior_flat().copy()
        axes = []
        for _ in range(self.mesh.dim):
            axes.append(rem % side)
            rem //= side
        if self.kind.colours == 2:
            return sum(a - 1 for a in axes) % 2
        code = np.zeros(len(rem), dtype=np.int64)
        for a, ax in enumerate(axes):
            code |= ((ax - 1) & 1) << a
        return code

    @property
    def colour_cells(self) -> list:
        if self._colour_cells is None:
            cid = self._colour_ids()
            interior = self.mesh.interior_flat()
            self._colour_cells = [interior[cid == c] for c in range(self.kind.colours)]
        return self._colour_cells

    def device_call(self) -> DeviceCall:
        key = (self.mesh.has_rhs, self.mesh.omega)
        if self._call is None or self._key != key:
            self._call = DeviceCall(self.mesh, self.kind)
            self._key = key
        else:
            self._call.refresh()
        return self._call


def _plan_for(mesh, kind, cost, plan):
    if plan is None or plan.mesh is not mesh or plan.kind is not kind:
        plan = SweepPlan(mesh, kind, cost)
    return plan


def run_sweeps(mesh: Mesh, kind: StencilKind, cost: CostModel, sweeps: int,
               plan: SweepPlan = None, flags: int = 0) -> float:
    """`sweeps` colour-ordered (or, with SL_FLAG_LEX, lexicographic) sweeps in
    one library call (fused when possible); returns the consumed cost-model
    sine tally (0.0 when k == 0)."""
    plan = _plan_for(mesh, kind, cost, plan)
    call = plan.device_call()
    lib = _native.load()
    if not cost.is_free:
        import torch
        work = torch.zeros(1, dtype=torch.float64, device=call.status.device)
        desc = cost.descriptor(work.data_ptr())
        rc = lib.sl_sweep_cost(ctypes.byref(call.grid), ctypes.byref(call.stencil),
                               ctypes.byref(desc), sweeps, flags & _native.SL_FLAG_LEX,
                               call.status.data_ptr(), call.stream)
        _native.check(rc, "sweep")
        call.check_status("sweep")
        return float(work.item())
    ws_bytes = 0
    ws_ptr = None
    if not flags & (_native.SL_FLAG_PER_COLOUR | _native.SL_FLAG_MERGE_COLOURS | _native.SL_FLAG_LEX):
        # the fused kernels (SL_FLAG_STREAM included) ping-pong through a workspace
        ws_bytes = lib.sl_workspace_bytes(ctypes.byref(call.grid), ctypes.byref(call.stencil))
        ws = mesh.workspace(ws_bytes)
        ws_ptr = ws.data_ptr() if ws is not None else None
    rc = lib.sl_sweep(ctypes.byref(call.grid), ctypes.byref(call.stencil), sweeps, flags,
                      ws_ptr, ws_bytes, call.status.data_ptr(), call.stream)
    _native.check(rc, "sweep")
    call.check_status("sweep")
    return 0.0


def sweep_colouring(pool: DevicePool, mesh: Mesh, kind: StencilKind, cost: CostModel,
                    schedule: Schedule = None, plan: SweepPlan = None,
                    _fault_merge_colours: bool = False):
    """One colour-ordered sweep on the GPU (reference strategies.py:348-393).

    `_fault_merge_colours` (tests only) runs every cell in ONE racy pass —
    the negative control the parity checks must catch (strategies.py:364-369).
    """
    flags = _native.SL_FLAG_MERGE_COLOURS if _fault_merge_colours else 0
    run_sweeps(mesh, kind, cost, 1, plan=plan, flags=flags)


def sweep_colouring_reference(mesh: Mesh, kind: StencilKind, cost: CostModel, log=None):
    """Colour-major pass, one in-place launch per colour (the independent
    K1 path; reference oracle strategies.py:409-433)."""
    if log is not None:
        raise NotImplementedError("per-cell tracing is not available on the GPU path")
    run_sweeps(mesh, kind, cost, 1, flags=_native.SL_FLAG_PER_COLOUR)


def sweep_hyb_sync(pool, mesh, kind, cost, schedule=None, plan=None):
    """Bitwise equal to colouring (reference tests/test_strategies.py:142-152)."""
    run_sweeps(mesh, kind, cost, 1, plan=plan)


def sweep_hyb_depend(pool, mesh, kind, cost, chunk=1, plan=None):
    """Bitwise equal to colouring (reference tests/test_strategies.py:142-152)."""
    run_sweeps(mesh, kind, cost, 1, plan=plan)


def _out_of_scope(name):
    raise NotImplementedError(
        f"strategy {name!r} has a CPU-worker-count-dependent update order; "
        f"the GPU runs {GPU_STRATEGIES}")


def sweep_serial(mesh, kind, cost, plan=None, log=None):
    """Lexicographic Gauss-Seidel sweep (reference strategies.py:341-345), on
    the GPU as hyperplane wavefronts; bitwise equal to the reference."""
    if log is not None:
        raise NotImplementedError("per-cell tracing is not available on the GPU path")
    run_sweeps(mesh, kind, cost, 1, plan=plan, flags=_native.SL_FLAG_LEX)


def sweep_nested_dissection(pool, mesh, kind, cost, plan=None):
    _out_of_scope("nd")


def sweep_taskgraph(pool, mesh, kind, cost, chunk=1, plan=None):
    """Dependence-DAG sweep; equals the serial sweep bit for bit (reference
    tests/test_strategies.py:125-139), so it runs the lexicographic wavefront."""
    run_sweeps(mesh, kind, cost, 1, plan=plan, flags=_native.SL_FLAG_LEX)


def run_sweep(strategy: str, mesh: Mesh, kind: StencilKind, cost: CostModel,
              pool: DevicePool = None, schedule: Schedule = None,
              chunk: int = 1, plan: SweepPlan = None, log=None):
    """Dispatch one full sweep of the given strategy (strategies.py:530-549)."""
    strategy = canonical_strategy(strategy)
    if strategy == "serial":
        sweep_serial(mesh, kind, cost, plan=plan, log=log)
        return
    if pool is None:
        raise ValueError(f"strategy {strategy!r} needs a worker pool")
    if log is not None:
        raise NotImplementedError("per-cell tracing is not available on the GPU path")
    if strategy == "colouring":
        sweep_colouring(pool, mesh, kind, cost, schedule, plan=plan)
    elif strategy == "nd":
        sweep_nested_dissection(pool, mesh, kind, cost, plan=plan)
    elif strategy == "taskgraph":
        sweep_taskgraph(pool, mesh, kind, cost, chunk=chunk, plan=plan)
    elif strategy == "hyb-depend":
        sweep_hyb_depend(pool, mesh, kind, cost, chunk=chunk, plan=plan)
    else:
        sweep_hyb_sync(pool, mesh, kind, cost, schedule, plan=plan)
