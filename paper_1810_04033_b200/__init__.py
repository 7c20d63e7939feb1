"""paper_1810_04033_b200: B200-native colour-scheduled smoother sweeps.

Drop-in for the hot path of the reference `stencil_lab` (arXiv 1810.04033):
the same entry-point names as its package surface (reference
__init__.py:8-27) for the colour-scheduled strategies, backed by hand-written
sm_100a CUDA kernels behind the C ABI in include/stencil_sweep.h.
"""

from .kernels import (FD5, FD7, FE9, FE27, FE27Q1, STENCILS, CostModel, NumericsError,
                      ScalarCellKernel, StencilKind, get_stencil, residual_max, update_cell,
                      update_cells_batch)
from .mesh import Mesh, init, init_rhs, make_mesh
from .patches import PatchBatch, init_patches
from .pipeline import SweepPipeline
from .pool import DevicePool, Schedule, WorkerPool
from .runner import (CONVERGENCE_TOL, BenchConfig, BenchResult, ConfigError, Report,
                     StrategyRunner, mesh_digest, parse_cost, run_benchmark, run_verification,
                     serial_convergence_budget, verify_convergence, verify_oracle)
from .strategies import (GPU_STRATEGIES, STRATEGY_IDS, SweepPlan, colour_count, colour_of,
                         run_sweep, run_sweeps, sweep_colouring, sweep_colouring_reference,
                         sweep_hyb_depend, sweep_hyb_sync, sweep_nested_dissection, sweep_serial,
                         sweep_taskgraph)

__version__ = "0.1.0"
