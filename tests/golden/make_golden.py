"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    cd /tmp && python /root/repo/tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src, runs its own
colouring path (StrategyRunner "colouring" = sweep_colouring ->
update_cells_batch, bench.py:143-203, strategies.py:348-393) and its
colour-order oracle (sweep_colouring_reference, strategies.py:409-433), and
writes:

  reference_digests.json   sha256 of mesh.values (bench.py:138-140) for every
                           kind x n in {8, 33} x 100 sweeps, seed 42
                           (acceptance criterion 5, tests/test_acceptance.py:107-130),
                           plus init digests and residual_max values
  reference_small.npz      full buffers after 5 sweeps, seed 11 (verify_oracle
                           sizes, bench.py:477-501) for element-level diffs;
                           "serial_<kind>" = the same after 5 lexicographic sweeps
  reference_digests.json["serial"]  sha256 after serial sweeps (strategies.py:341-345),
                           checked equal to taskgraph here (tests/test_strategies.py:125-139)
  reference_digests.json["convergence"]  serial_convergence_budget (bench.py:433-442)

The GPU box never reads /root/reference: tests compare against these files.
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from stencil_lab.bench import StrategyRunner, mesh_digest, serial_convergence_budget  # noqa: E402
from stencil_lab.kernels import STENCILS, CostModel, residual_max  # noqa: E402
from stencil_lab.mesh import Mesh, init, make_mesh  # noqa: E402
from stencil_lab.strategies import sweep_colouring_reference, sweep_serial  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    digests = {"sweeps": {}, "init": {}, "residual": {}, "serial": {}, "convergence": {}}
    # serial sweep counts to residual < 1e-8 (bench.py:433-442), criterion-6 cases
    for name, n in (("fd5", 33), ("fd7", 17), ("fe9", 17), ("fe27", 9)):
        digests["convergence"][f"{name}/n={n}/seed=7"] = serial_convergence_budget(
            STENCILS[name], n, seed=7)
    # criterion-5 style: all kinds, n in {8, 33}, 100 sweeps, seed 42
    for name, kind in STENCILS.items():
        for n in (8, 33):
            with StrategyRunner(kind.dim, n, kind, CostModel("const", 0), "colouring",
                                threads=2, seed=42) as r:
                r.reinit()
                r.run_sweeps(100)
                digests["sweeps"][f"{name}/n={n}/s=100/seed=42"] = r.digest()
        # a few other sweep counts / a non-zero boundary value
        n = 12 if kind.dim == 2 else 6
        for sweeps in (1, 2, 7):
            with StrategyRunner(kind.dim, n, kind, CostModel("const", 0), "colouring",
                                threads=2, seed=5, boundary=0.75) as r:
                r.reinit()
                r.run_sweeps(sweeps)
                digests["sweeps"][f"{name}/n={n}/s={sweeps}/seed=5/b=0.75"] = r.digest()
    # lexicographic order: serial (and taskgraph, which must agree bit for bit)
    for name, kind in STENCILS.items():
        for n, sweeps, seed, b in (((8, 3, 42, 0.0), (13, 2, 5, 0.75)) if kind.dim == 2
                                   else ((6, 3, 42, 0.0), (7, 2, 5, 0.75))):
            got = []
            for strat, threads in (("serial", 1), ("taskgraph", 3)):
                with StrategyRunner(kind.dim, n, kind, CostModel("const", 0), strat,
                                    threads=threads, seed=seed, boundary=b) as r:
                    r.reinit()
                    r.run_sweeps(sweeps)
                    got.append(r.digest())
            assert got[0] == got[1], (name, n)
            digests["serial"][f"{name}/n={n}/s={sweeps}/seed={seed}/b={b}"] = got[0]
    for dim, n, seed, b in ((2, 5, 7, 0.0), (2, 64, 42, 0.0), (3, 4, 7, 2.5), (3, 20, 42, 0.0)):
        m = make_mesh(dim, n, seed=seed, boundary_value=b)
        digests["init"][f"{dim}/{n}/{seed}/{b}"] = mesh_digest(m)
    for name, kind in STENCILS.items():
        n = 10 if kind.dim == 2 else 6
        m = make_mesh(kind.dim, n, seed=9)
        digests["residual"][f"{name}/n={n}/seed=9"] = residual_max(m, kind).hex()
    small = {}
    for name, kind in STENCILS.items():
        n = 10 if kind.dim == 2 else 6     # verify_oracle sizes (bench.py:477)
        ref = Mesh(kind.dim, n)
        init(ref, 11, 0.0)
        for _ in range(5):
            sweep_colouring_reference(ref, kind, CostModel("const", 0))
        small[name] = ref.values.copy()
        ser = Mesh(kind.dim, n)
        init(ser, 11, 0.0)
        for _ in range(5):
            sweep_serial(ser, kind, CostModel("const", 0))
        small["serial_" + name] = ser.values.copy()
    np.savez_compressed(os.path.join(OUT, "reference_small.npz"), **small)
    with open(os.path.join(OUT, "reference_digests.json"), "w") as fh:
        json.dump(digests, fh, indent=1, sort_keys=True)
    print("wrote", len(digests["sweeps"]), "sweep digests")


if __name__ == "__main__":
    main()
