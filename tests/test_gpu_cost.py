"""Cost model k > 0 on the device (reference kernels.py:113-200, :234-244):
the sines execute (non-zero tally) and every value stays bit-identical to
the k = 0 run, in colour order and in lexicographic order."""

import numpy as np
import pytest

import paper_1810_04033_b200 as sl
from oracle import coracle
from oracle import restate as R
from paper_1810_04033_b200 import _native

pytestmark = pytest.mark.gpu
ALL = list(R.STENCIL_TABLE)


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a).reshape(-1).view(np.int64),
                          np.asarray(b).reshape(-1).view(np.int64))


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("order", ["colour", "lex"])
@pytest.mark.parametrize("cost", [sl.CostModel("const", 3), sl.CostModel("ramp")])
def test_cost_values_unchanged_and_work_consumed(name, order, cost):
    dim = R.STENCIL_TABLE[name][0]
    kind = sl.get_stencil(name)
    n = 13 if dim == 2 else 6
    for form in ("R", "D"):
        u = R.init_u(dim, n, 4, 0.5)
        m = sl.make_mesh(dim, n, seed=4, boundary_value=0.5)
        f = None
        if form == "D":
            f = R.init_f(dim, n, 5)
            sl.init_rhs(m, 5, 0.8)
        coracle.sweep(u, name, 2, f=f, omega=0.8, form=form, order=order)
        flags = _native.SL_FLAG_LEX if order == "lex" else 0
        work = sl.run_sweeps(m, kind, cost, 2, flags=flags)
        assert _bits_equal(m.values, u), (name, order, form)
        assert work != 0.0


def test_ramp_colouring_matches_reference_order():
    """Restates reference tests/test_strategies.py:167-175 (FE9, n=11, ramp)."""
    with sl.StrategyRunner(2, 11, sl.FE9, sl.CostModel("ramp"), "colouring", threads=3,
                           seed=7) as r:
        r.reinit()
        r.run_sweeps(2)
        got = r.mesh.values.copy()
    u = R.init_u(2, 11, 7)
    R.sweep(u, "fe9", 2)
    assert _bits_equal(got, u)


def test_update_cell_k100_equals_k0():
    """Restates reference tests/test_kernels.py:128-136."""
    for kind in (sl.FD5, sl.FE9, sl.FD7, sl.FE27):
        a = sl.make_mesh(kind.dim, 4, seed=5)
        b = sl.make_mesh(kind.dim, 4, seed=5)
        for coord in list(a.interior_coords())[:6]:
            sl.update_cell(a, kind, coord, k=0)
            sl.update_cell(b, kind, coord, k=100)
        assert _bits_equal(a.values, b.values), kind.name


def test_scalar_kernel_work_is_consumed():
    m = sl.make_mesh(2, 4, seed=5)
    kernel = sl.ScalarCellKernel(m, sl.FD5)
    flat = m.flat_index((2, 2))
    kernel.update([flat + d for d in sl.FD5.flat_offsets(m)], flat, 10)
    assert kernel.work_sum != 0.0


def test_update_cells_batch_cost_tally_and_values():
    m = sl.make_mesh(2, 12, seed=2)
    plan = sl.SweepPlan(m, sl.FD5, sl.CostModel())
    work = sl.update_cells_batch(m, sl.FD5, plan.colour_cells[1], 7)
    u = R.init_u(2, 12, 2)
    R.colour_pass(u, "fd5", 1)
    assert _bits_equal(m.values, u)
    # the tally is the sum of 7 sines per entry over 5 entries per cell
    vals = R.init_u(2, 12, 2).reshape(-1)
    deltas = [0] + list(sl.FD5.flat_offsets(m))
    want = sum(np.sin(vals[c + d] + i) for c in plan.colour_cells[1] for d in deltas
               for i in range(7))
    assert abs(work - want) <= 1e-9 * max(1.0, abs(want))


def test_patches_with_cost():
    b, n = 7, 16
    u0, f0 = sl.init_patches(b, n, 3)
    pb = sl.PatchBatch(u0, f0, omega=0.8)
    work = pb.sweep(sl.FD5, 3, cost=sl.CostModel("const", 2))
    u, f = u0.copy(), f0.copy()
    coracle.sweep(u, "fd5", 3, f=f, omega=0.8, form="D")
    assert _bits_equal(pb.values(), u)
    assert work != 0.0


def test_cost_nonfinite_raises():
    m = sl.make_mesh(2, 6, seed=1)
    m.values[m.flat_index((1, 2))] = np.inf
    with pytest.raises(sl.NumericsError):
        sl.run_sweeps(m, sl.FD5, sl.CostModel("const", 2), 1)
