"""GPU parity: the CUDA path against the reference (golden digests) and the
oracle (C / NumPy restatements), bit for bit.

Everything here calls the sm_100a library through the C ABI (via the
drop-in Python surface) and compares against tests/golden/ or oracle/.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1810_04033_b200 as sl
from oracle import coracle
from oracle import restate as R
from paper_1810_04033_b200 import _native, strategies

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALL = list(R.STENCIL_TABLE)


def _digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a).reshape(-1).view(np.int64), np.asarray(b).reshape(-1).view(np.int64))


def _parse(key):
    parts = dict(p.split("=") for p in key.split("/")[1:])
    return key.split("/")[0], int(parts["n"]), int(parts["s"]), int(parts["seed"]), float(parts.get("b", 0.0))


@pytest.fixture(scope="module")
def ref_digests():
    with open(os.path.join(GOLDEN, "reference_digests.json")) as fh:
        return json.load(fh)


# -- Form R vs the reference itself ------------------------------------------

@pytest.mark.parametrize("path", ["fused", "per_sweep", "reference_k1"])
def test_form_r_matches_reference_digests(ref_digests, path):
    """Acceptance criterion 5 digests (reference tests/test_acceptance.py:107-130)."""
    for key, want in ref_digests["sweeps"].items():
        name, n, sweeps, seed, b = _parse(key)
        kind = sl.get_stencil(name)
        with sl.StrategyRunner(kind.dim, n, kind, sl.CostModel(), "colouring", seed=seed,
                               boundary=b) as r:
            r.reinit()
            if path == "fused":
                r.run_sweeps(sweeps)
            elif path == "per_sweep":
                for _ in range(sweeps):
                    r.sweep()
            else:
                for _ in range(sweeps):
                    sl.sweep_colouring_reference(r.mesh, kind, sl.CostModel())
            assert r.digest() == want, (key, path)


def test_form_r_small_buffers_bitwise():
    small = np.load(os.path.join(GOLDEN, "reference_small.npz"))
    for name in ("fd5", "fe9", "fd7", "fe27"):
        kind = sl.get_stencil(name)
        n = 10 if kind.dim == 2 else 6
        m = sl.make_mesh(kind.dim, n, seed=11)
        for strat in ("colouring", "hyb-sync", "hyb-depend"):
            m2 = sl.make_mesh(kind.dim, n, seed=11)
            for _ in range(5):
                sl.run_sweep(strat, m2, kind, sl.CostModel(), pool=sl.DevicePool())
            assert _bits_equal(m2.values, small[name]), (name, strat)
        sl.run_sweeps(m, kind, sl.CostModel(), 5)
        assert _bits_equal(m.values, small[name]), name


# -- Form D / Q1 vs the oracle (self-pinned) ----------------------------------

def _oracle_d(name, n, sweeps, seed=42, boundary=0.0):
    dim = R.STENCIL_TABLE[name][0]
    u = R.init_u(dim, n, seed, boundary)
    f = R.init_f(dim, n, seed + 1)
    coracle.sweep(u, name, sweeps, f=f, omega=0.8, form="D")
    return u


def _gpu_d(name, n, sweeps, seed=42, boundary=0.0, mode="fused"):
    kind = sl.get_stencil(name)
    m = sl.make_mesh(kind.dim, n, seed=seed, boundary_value=boundary)
    sl.init_rhs(m, seed + 1, 0.8)
    if mode == "fused":
        sl.run_sweeps(m, kind, sl.CostModel(), sweeps)
    elif mode == "k1":
        sl.run_sweeps(m, kind, sl.CostModel(), sweeps, flags=_native.SL_FLAG_PER_COLOUR)
    elif mode == "stream":
        sl.run_sweeps(m, kind, sl.CostModel(), sweeps, flags=_native.SL_FLAG_STREAM)
    else:
        for _ in range(sweeps):
            sl.sweep_colouring(sl.DevicePool(), m, kind, sl.CostModel())
    return m.values


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("mode", ["fused", "stream", "k1", "single"])
def test_form_d_matches_oracle_small_and_ragged(name, mode):
    dim = R.STENCIL_TABLE[name][0]
    sizes = (1, 2, 3, 7, 16, 33, 64, 130) if dim == 2 else (1, 2, 3, 5, 8, 17, 32)
    for n in sizes:
        for sweeps in (1, 2, 5, 9):
            want = _oracle_d(name, n, sweeps, seed=n)
            got = _gpu_d(name, n, sweeps, seed=n, mode=mode)
            assert _bits_equal(got, want), (name, n, sweeps, mode)


@pytest.mark.parametrize("name", ALL)
def test_form_r_all_kinds_vs_oracle_ragged(name):
    dim = R.STENCIL_TABLE[name][0]
    kind = sl.get_stencil(name)
    for n in ((1, 4, 9, 31, 100) if dim == 2 else (1, 4, 9, 21)):
        u = R.init_u(dim, n, 3, 0.25)
        R.sweep(u, name, 3)
        m = sl.make_mesh(dim, n, seed=3, boundary_value=0.25)
        sl.run_sweeps(m, kind, sl.CostModel(), 3)
        assert _bits_equal(m.values, u), (name, n)


# -- BASELINE configs at full size (property: equals the C oracle) ------------

def test_config1_fd5_1026_full():
    want = _oracle_d("fd5", 1024, 100)
    got = _gpu_d("fd5", 1024, 100)
    assert _bits_equal(got, want)


def test_config2_fe9_8194_full():
    want = _oracle_d("fe9", 8192, 50)
    got = _gpu_d("fe9", 8192, 50)
    assert _bits_equal(got, want)


def test_config3_fd7_514_full():
    want = _oracle_d("fd7", 512, 20)
    got = _gpu_d("fd7", 512, 20)
    assert _bits_equal(got, want)


def test_config4_fe27q1_1026_full():
    # the full BASELINE config: 1026^3 grid, all 10 sweeps (C oracle on all host threads)
    want = _oracle_d("fe27q1", 1024, 10)
    got = _gpu_d("fe27q1", 1024, 10)
    assert _bits_equal(got, want)


# -- reference unit behaviours on the device -----------------------------------

def test_update_cells_batch_equals_oracle_colour_pass():
    for name in ALL:
        kind = sl.get_stencil(name)
        n = 6 if kind.dim == 2 else 4
        m = sl.make_mesh(kind.dim, n, seed=5)
        plan = sl.SweepPlan(m, kind, sl.CostModel())
        sl.update_cells_batch(m, kind, plan.colour_cells[0], 0)
        u = R.init_u(kind.dim, n, 5)
        R.colour_pass(u, name, 0)
        assert _bits_equal(m.values, u), name


def test_update_cell_known_answers():
    m = sl.Mesh(2, 3)
    m.values.fill(1.0)
    assert sl.update_cell(m, sl.FD5, (2, 2)) == 1.0
    m = sl.Mesh(2, 3)
    m.values[m.flat_index((2, 1))] = 1.0
    assert sl.update_cell(m, sl.FD5, (2, 2)) == 0.25
    with pytest.raises(IndexError):
        sl.update_cell(m, sl.FD5, (0, 1))


def test_nonfinite_raises_numerics_error():
    m = sl.make_mesh(2, 8, seed=1)
    m.values[m.flat_index((1, 2))] = np.inf
    with pytest.raises(sl.NumericsError):
        sl.run_sweeps(m, sl.FD5, sl.CostModel(), 2)
    m = sl.make_mesh(2, 4, seed=1)
    m.values[m.flat_index((0, 1))] = np.nan
    before = m.values.copy()
    flats = np.array([m.flat_index((1, 1)), m.flat_index((3, 3)), m.flat_index((2, 4))])
    with pytest.raises(sl.NumericsError):
        sl.update_cells_batch(m, sl.FD5, flats, 0)
    # like the reference (kernels.py:243-251) the failing batch writes nothing
    assert _bits_equal(m.values, before)
    with pytest.raises(sl.NumericsError):
        sl.update_cells_batch(m, sl.FD5, flats, 3)
    assert _bits_equal(m.values, before)


def test_replaced_rhs_is_used_by_a_reused_plan():
    """set_rhs with the same omega after a sweep: the cached plan must read
    the new f (it once kept the freed tensor's pointer)."""
    for name, n in (("fe9", 40), ("fe27q1", 12)):
        kind = sl.get_stencil(name)
        m = sl.make_mesh(kind.dim, n, seed=5)
        sl.init_rhs(m, 6, 0.8)
        plan = sl.SweepPlan(m, kind, sl.CostModel())
        sl.run_sweeps(m, kind, sl.CostModel(), 2, plan=plan)
        f2 = R.init_f(kind.dim, n, 99)
        m.set_rhs(f2.reshape(-1).copy(), 0.8)
        sl.run_sweeps(m, kind, sl.CostModel(), 3, plan=plan)
        u = R.init_u(kind.dim, n, 5)
        coracle.sweep(u, name, 2, f=R.init_f(kind.dim, n, 6), omega=0.8, form="D")
        coracle.sweep(u, name, 3, f=f2, omega=0.8, form="D")
        assert _bits_equal(m.values, u), name


def test_constant_mesh_unchanged():
    for kind in (sl.FD5, sl.FE27):
        m = sl.Mesh(kind.dim, 4)
        m.values.fill(1.75)
        sl.run_sweep("colouring", m, kind, sl.CostModel(), pool=sl.DevicePool())
        assert (m.values == 1.75).all()


def test_halo_immutable():
    for name in ALL:
        kind = sl.get_stencil(name)
        n = 9 if kind.dim == 2 else 6
        m = sl.make_mesh(kind.dim, n, seed=2, boundary_value=3.25)
        sl.init_rhs(m, 3)
        halo = m.halo_flat()
        sl.run_sweeps(m, kind, sl.CostModel(), 4)
        assert (m.values[halo] == 3.25).all(), name


def test_residual_matches_reference(ref_digests):
    for key, want in ref_digests["residual"].items():
        name = key.split("/")[0]
        kind = sl.get_stencil(name)
        n = 10 if kind.dim == 2 else 6
        assert sl.residual_max(sl.make_mesh(kind.dim, n, seed=9), kind).hex() == want, key


def test_residual_form_d_and_decrease():
    m = sl.make_mesh(2, 33, seed=7)
    sl.init_rhs(m, 8)
    f = R.init_f(2, 33, 8)
    r0 = sl.residual_max(m, sl.FD5)
    assert r0 == R.residual_max(R.init_u(2, 33, 7), "fd5", f=f)
    sl.run_sweeps(m, sl.FD5, sl.CostModel(), 50)
    assert sl.residual_max(m, sl.FD5) < r0


def test_merged_colour_negative_control_mismatches():
    """Reference bench.py:372-395: the racy single-pass variant must be caught."""
    kind = sl.FD5
    want = R.init_u(2, 64, 1)
    R.sweep(want, "fd5", 1)
    m = sl.make_mesh(2, 64, seed=1)
    sl.sweep_colouring(sl.DevicePool(), m, kind, sl.CostModel(), _fault_merge_colours=True)
    assert not _bits_equal(m.values, want)


def test_deterministic_across_repeats_and_paths():
    digests = set()
    for mode in ("fused", "stream", "k1", "single", "fused"):
        digests.add(_digest(_gpu_d("fe27q1", 20, 3, mode=mode)))
    assert len(digests) == 1


def test_host_edits_between_sweeps_are_seen():
    m = sl.make_mesh(2, 6, seed=4)
    sl.run_sweeps(m, sl.FD5, sl.CostModel(), 1)
    m.values.fill(2.0)
    sl.run_sweeps(m, sl.FD5, sl.CostModel(), 1)
    assert (m.values == 2.0).all()


def test_read_values_between_sweeps_keeps_the_device_authoritative():
    """read_values() downloads without flipping the mesh to host-authoritative
    (no re-upload on the next sweep), is read-only, and the sweeps continue
    from the device state: 2 + 3 sweeps with a read in between == 5 sweeps."""
    n, seed = 70, 12
    m = sl.make_mesh(2, n, seed=seed)
    sl.init_rhs(m, seed + 1, 0.8)
    sl.run_sweeps(m, sl.FE9, sl.CostModel(), 2)
    mid = m.read_values()
    assert m._where == "dev" and not mid.flags.writeable
    want = R.init_u(2, n, seed)
    f = R.init_f(2, n, seed + 1)
    coracle.sweep(want, "fe9", 2, f=f, omega=0.8, form="D")
    assert _bits_equal(mid, want)
    m._host.fill(-7.0)                 # a stale host mirror must not come back
    sl.run_sweeps(m, sl.FE9, sl.CostModel(), 3)
    coracle.sweep(want, "fe9", 3, f=f, omega=0.8, form="D")
    assert _bits_equal(m.read_values(), want)


# -- lexicographic order (serial / taskgraph) ---------------------------------

@pytest.mark.parametrize("strategy", ["serial", "taskgraph"])
def test_lex_matches_reference_serial_digests(ref_digests, strategy):
    """Reference serial == taskgraph (strategies.py:341-345, :477-487)."""
    for key, want in ref_digests["serial"].items():
        name, n, sweeps, seed, b = _parse(key)
        kind = sl.get_stencil(name)
        with sl.StrategyRunner(kind.dim, n, kind, sl.CostModel(), strategy, threads=3,
                               seed=seed, boundary=b) as r:
            r.reinit()
            r.run_sweeps(sweeps)
            assert r.digest() == want, (key, strategy)


def test_lex_small_buffers_bitwise():
    small = np.load(os.path.join(GOLDEN, "reference_small.npz"))
    for name in ("fd5", "fe9", "fd7", "fe27"):
        kind = sl.get_stencil(name)
        m = sl.make_mesh(kind.dim, 10 if kind.dim == 2 else 6, seed=11)
        for _ in range(5):
            sl.sweep_serial(m, kind, sl.CostModel())
        assert _bits_equal(m.values, small["serial_" + name]), name


def test_lex_kat_degenerate_row():
    """Restates reference tests/test_strategies.py:74-89 on the device."""
    a, b, c = 0.8, 0.3, 0.5
    m = sl.Mesh(2, 3)
    for x, v in ((1, a), (2, b), (3, c)):
        m.values[m.flat_index((x, 1))] = v
    sl.sweep_serial(m, sl.FD5, sl.CostModel())
    a2 = b / 4
    b2 = (a2 + c) / 4
    got = [m.values[m.flat_index((x, 1))] for x in (1, 2, 3)]
    assert got == [a2, b2, b2 / 4]


@pytest.mark.parametrize("name", ALL)
def test_lex_form_d_matches_oracle_ragged(name):
    dim = R.STENCIL_TABLE[name][0]
    kind = sl.get_stencil(name)
    for n in ((1, 2, 5, 16, 67) if dim == 2 else (1, 2, 5, 12)):
        u = R.init_u(dim, n, n)
        f = R.init_f(dim, n, n + 1)
        coracle.sweep(u, name, 3, f=f, omega=0.8, form="D", order="lex")
        m = sl.make_mesh(dim, n, seed=n)
        sl.init_rhs(m, n + 1, 0.8)
        sl.run_sweeps(m, kind, sl.CostModel(), 3, flags=_native.SL_FLAG_LEX)
        assert _bits_equal(m.values, u), (name, n)


def test_lex_differs_from_colour_order():
    m1 = sl.make_mesh(2, 16, seed=1)
    m2 = sl.make_mesh(2, 16, seed=1)
    sl.sweep_serial(m1, sl.FD5, sl.CostModel())
    sl.run_sweeps(m2, sl.FD5, sl.CostModel(), 1)
    assert not _bits_equal(m1.values, m2.values)


# -- single pass with an output plane window (slab runner building block) -----

@pytest.mark.parametrize("name,n", [("fe27q1", 40), ("fd7", 37 + 1), ("fe9", 150), ("fd5", 130)])
def test_sweep_pass_windows_compose(name, n):
    """sl_sweep_pass over [0, a) + [a, b) + [b, S) along the slowest axis gives
    the same dst as one pass over [0, S), and both equal one oracle sweep."""
    import ctypes

    import torch
    kind = sl.get_stencil(name)
    dim = kind.dim
    u = R.init_u(dim, n, 5)
    f = R.init_f(dim, n, 6)
    lib = _native.require_cuda()
    src = torch.from_numpy(u).cuda()
    fd = torch.from_numpy(f).cuda()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = _native.SlGrid()
    g.dim = dim
    for a in range(dim):
        g.n[a] = n
    g.batch = 1
    g.batch_stride = src.numel()
    g.u = src.data_ptr()
    g.f = fd.data_ptr()
    st = kind.descriptor(_native.SL_FORM_D, 0.8)
    S = n + 2
    whole = torch.zeros_like(src)
    parts = torch.zeros_like(src)
    stream = torch.cuda.current_stream().cuda_stream

    def run(dst, z0, z1):
        rc = lib.sl_sweep_pass(ctypes.byref(g), ctypes.byref(st), src.data_ptr(), dst.data_ptr(),
                               z0, z1, status.data_ptr(), stream)
        assert rc == _native.SL_OK, _native.load().sl_strerror(rc)

    run(whole, 0, S)
    a, b = S // 3, S // 3 + 5
    for z0, z1 in ((b, S), (0, a), (a, b)):
        run(parts, z0, z1)
    torch.cuda.synchronize()
    want = u.copy()
    coracle.sweep(want, name, 1, f=f, omega=0.8, form="D")
    assert _bits_equal(whole.cpu().numpy(), want)
    assert _bits_equal(parts.cpu().numpy(), want)
    assert int(status.item()) == 0


@pytest.mark.parametrize("name,n,flags", [("fe9", 130, _native.SL_FLAG_STREAM), ("fe9", 64, 0),
                                          ("fd5", 130, _native.SL_FLAG_STREAM), ("fd7", 34, 0),
                                          ("fe27q1", 30, 0), ("fe27", 18, 0)])
def test_nonfinite_raises_on_every_fused_kernel(name, n, flags):
    """A non-finite interior value (Form D) or right-hand side surfaces as
    NumericsError from the streaming, tile and Q1 kernels alike."""
    kind = sl.get_stencil(name)
    for where in ("u", "f"):
        m = sl.make_mesh(kind.dim, n, seed=3)
        sl.init_rhs(m, 4, 0.8)
        c = (n // 2,) * kind.dim
        if where == "u":
            m.values[m.flat_index(c)] = np.inf
        else:
            f = m._rhs_host.copy()
            f[m.flat_index(c)] = np.nan
            m.set_rhs(f, 0.8)
        with pytest.raises(sl.NumericsError):
            sl.run_sweeps(m, kind, sl.CostModel(), 2, flags=flags)
