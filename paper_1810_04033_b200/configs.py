"""The five BASELINE.json workloads as concrete sweep configurations.

Seeded synthetic inputs (no public dataset is involved):
u0 = default_rng(seed).random(n^dim) in lex order (reference mesh.py:110-111),
f = default_rng(seed+1).uniform(-1, 1, n^dim) with a zero halo, omega = 0.8,
Dirichlet-zero halo; config 5 holds a random U[0,1) halo fixed per patch.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["Workload", "CONFIGS", "BYTES_PER_UPDATE", "FP64_OPS_PER_UPDATE"]

# algorithmic bytes per grid-point update: read u_c + read f_c + write u_c
BYTES_PER_UPDATE = 24

# fp64 instructions per update of the on-chip (fp64-bound) patch kernel, config 5
# (K3, Form D FD5: DMUL w_c*u, 4 DSUB, DSUB f-Au, DMUL 1/w_c, DMUL omega, DADD)
FP64_OPS_PER_UPDATE = {5: 9}


@dataclass(frozen=True)
class Workload:
    index: int          # 1-based position in BASELINE.json "configs"
    name: str
    stencil: str
    dim: int
    n: int              # interior extent per axis
    sweeps: int
    batch: int = 1      # independent patches (config 5)
    seed: int = 42
    omega: float = 0.8

    @property
    def points(self) -> int:
        return self.batch * self.n ** self.dim

    @property
    def updates(self) -> int:
        return self.points * self.sweeps

    @property
    def side(self) -> int:
        return self.n + 2

    @property
    def grid_elems(self) -> int:
        return self.batch * self.side ** self.dim


CONFIGS = {
    1: Workload(1, "fd5-1026sq-100sw", "fd5", 2, 1024, 100),
    2: Workload(2, "fe9-8194sq-50sw", "fe9", 2, 8192, 50),
    3: Workload(3, "fd7-514cube-20sw", "fd7", 3, 512, 20),
    4: Workload(4, "fe27q1-1026cube-10sw", "fe27q1", 3, 1024, 10),
    5: Workload(5, "fd5-65536x18sq-patches-200sw", "fd5", 2, 16, 200, batch=65536),
}
