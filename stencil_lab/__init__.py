"""`stencil_lab` — the reference package's import name for the GPU path.

`import stencil_lab` (and `from stencil_lab.strategies import ...`, etc.)
reaches the B200 implementation in `paper_1810_04033_b200`, so code written
against the reference (reference pkg/src/stencil_lab/__init__.py:8-27) runs
unchanged on the hot path.  Submodules map as:

    stencil_lab.mesh        -> paper_1810_04033_b200.mesh        (mesh.py)
    stencil_lab.kernels     -> paper_1810_04033_b200.kernels     (kernels.py)
    stencil_lab.strategies  -> paper_1810_04033_b200.strategies  (strategies.py)
    stencil_lab.bench       -> paper_1810_04033_b200.runner      (bench.py)
    stencil_lab.taskrt      -> paper_1810_04033_b200.pool        (taskrt.py: WorkerPool, Schedule)
    stencil_lab.cli         -> paper_1810_04033_b200.cli         (cli.py)

Names of the reference's out-of-scope subsystems (the CPU task runtime's
dependence tracker, nested dissection, per-cell tracing) are
not provided: importing one raises ImportError that says why.
"""

import sys as _sys

import paper_1810_04033_b200 as _impl
from paper_1810_04033_b200 import cli, kernels, mesh, pool, runner, strategies
from paper_1810_04033_b200 import (FD5, FD7, FE9, FE27, FE27Q1, STENCILS, STRATEGY_IDS,  # noqa: F401
                                   BenchConfig, BenchResult, ConfigError, CostModel, Mesh,
                                   NumericsError, Report, ScalarCellKernel, Schedule,
                                   StencilKind, StrategyRunner, SweepPlan, WorkerPool,
                                   colour_count, colour_of, get_stencil, init, init_rhs,
                                   make_mesh, mesh_digest, parse_cost, residual_max,
                                   run_benchmark, run_sweep, run_sweeps, run_verification,
                                   sweep_colouring, sweep_colouring_reference,
                                   sweep_hyb_depend, sweep_hyb_sync, sweep_nested_dissection,
                                   sweep_serial, sweep_taskgraph, update_cell,
                                   update_cells_batch)

bench = runner
taskrt = pool
for _name, _mod in (("mesh", mesh), ("kernels", kernels), ("strategies", strategies),
                    ("bench", runner), ("taskrt", pool), ("cli", cli)):
    _sys.modules[f"{__name__}.{_name}"] = _mod

__version__ = _impl.__version__

# reference names of subsystems that stay on the CPU (out of scope)
_OUT_OF_SCOPE = {
    "Box": "nested dissection", "DissectionNode": "nested dissection", "dissect": "nested dissection",
    "DependencyTracker": "the CPU task runtime", "StallError": "the CPU task runtime",
    "TaskRecord": "the CPU task runtime", "WaitScope": "the CPU task runtime",
    "make_task": "the CPU task runtime", "oracle_edges": "the CPU task runtime",
    "Trace": "per-cell tracing", "TraceLog": "per-cell tracing", "assignment_map": "per-cell tracing",
    "band_contiguity": "per-cell tracing", "check_adjacency_exclusion": "per-cell tracing",
    "check_edge_order": "per-cell tracing", "dump_text": "per-cell tracing",
    "merge_logs": "per-cell tracing", "parse_text": "per-cell tracing",
    "render_assignment_map": "per-cell tracing",
}


def __getattr__(name):
    if name in _OUT_OF_SCOPE:
        raise ImportError(f"stencil_lab.{name} belongs to {_OUT_OF_SCOPE[name]}, which the GPU "
                          f"implementation does not provide (only the colour-scheduled sweep path)")
    raise AttributeError(f"module 'stencil_lab' has no attribute {name!r}")
