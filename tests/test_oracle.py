"""The oracle itself, pinned against the reference (CPU only).

Both restatements (NumPy strided slices, plain C) must reproduce the
reference's own outputs bit for bit: the sha256 digests and full buffers in
tests/golden/ were produced by running /root/reference/pkg/src
(tests/golden/make_golden.py).  Form D / FE27-Q1 / patches have no reference
counterpart, so there the two restatements must agree with each other.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import coracle
from oracle import restate as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REF_KINDS = ("fd5", "fe9", "fd7", "fe27")


def _digest(u):
    return hashlib.sha256(np.ascontiguousarray(u).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ref_digests():
    with open(os.path.join(GOLDEN, "reference_digests.json")) as fh:
        return json.load(fh)


def _parse(key):
    parts = dict(p.split("=") for p in key.split("/")[1:])
    return key.split("/")[0], int(parts["n"]), int(parts["s"]), int(parts["seed"]), float(parts.get("b", 0.0))


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_form_r_matches_reference_digests(ref_digests, impl):
    for key, want in ref_digests["sweeps"].items():
        name, n, sweeps, seed, b = _parse(key)
        dim = R.STENCIL_TABLE[name][0]
        u = R.init_u(dim, n, seed, b)
        if impl == "numpy":
            R.sweep(u, name, sweeps)
        else:
            coracle.sweep(u, name, sweeps, threads=3)
        assert _digest(u) == want, key


def test_form_r_small_buffers_bitwise():
    small = np.load(os.path.join(GOLDEN, "reference_small.npz"))
    for name in REF_KINDS:
        want = small[name]
        dim = R.STENCIL_TABLE[name][0]
        n = 10 if dim == 2 else 6
        for impl in ("numpy", "c"):
            u = R.init_u(dim, n, 11)
            (R.sweep if impl == "numpy" else coracle.sweep)(u, name, 5)
            assert np.array_equal(u.ravel().view(np.int64), want.view(np.int64)), (name, impl)


def test_init_matches_reference(ref_digests):
    for key, want in ref_digests["init"].items():
        dim, n, seed, b = key.split("/")
        assert _digest(R.init_u(int(dim), int(n), int(seed), float(b))) == want, key


def test_residual_matches_reference(ref_digests):
    for key, want in ref_digests["residual"].items():
        name = key.split("/")[0]
        dim = R.STENCIL_TABLE[name][0]
        n = 10 if dim == 2 else 6
        assert R.residual_max(R.init_u(dim, n, 9), name).hex() == want, key


@pytest.mark.parametrize("name", list(R.STENCIL_TABLE))
@pytest.mark.parametrize("form", ["R", "D"])
def test_numpy_and_c_restatements_agree(name, form):
    dim = R.STENCIL_TABLE[name][0]
    for n in ((1, 2, 5, 16) if dim == 2 else (1, 2, 3, 9)):
        a = R.init_u(dim, n, 3, 0.5)
        f = R.init_f(dim, n, 4)
        b = a.copy()
        R.sweep(a, name, 3, f=f, omega=0.8, form=form)
        coracle.sweep(b, name, 3, f=f, omega=0.8, form=form, threads=4)
        assert np.array_equal(a.view(np.int64), b.view(np.int64)), (name, form, n)


def test_patches_agree():
    u, f = R.init_patches(9, 16, 5)
    v = u.copy()
    R.sweep(u, "fd5", 7, f=f, omega=0.8, form="D")
    coracle.sweep(v, "fd5", 7, f=f, omega=0.8, form="D")
    assert np.array_equal(u, v)


def test_patch_equals_per_patch_mesh_sweep():
    # a batch of patches is exactly B independent meshes with their own halo
    u, f = R.init_patches(4, 6, 1)
    w = u.copy()
    R.sweep(u, "fd5", 5, f=f, omega=0.8, form="D")
    for b in range(4):
        p = w[b].copy()
        R.sweep(p, "fd5", 5, f=f[b].copy(), omega=0.8, form="D")
        assert np.array_equal(p, u[b])


def test_halo_never_written():
    for name in R.STENCIL_TABLE:
        dim = R.STENCIL_TABLE[name][0]
        n = 6 if dim == 2 else 4
        u = R.init_u(dim, n, 2, 3.25)
        f = R.init_f(dim, n, 2)
        coracle.sweep(u, name, 4, f=f, form="D")
        mask = np.ones(u.shape, bool)
        mask[(slice(1, n + 1),) * dim] = False
        assert (u[mask] == 3.25).all()


# -- known-answer updates (reference tests/test_kernels.py:95-126) ------------

def test_kat_fd5_all_neighbours_one():
    u = np.ones((5, 5))
    R.colour_pass(u, "fd5", 0)
    assert u[2, 2] == 1.0


def test_kat_fd5_single_neighbour():
    u = np.zeros((5, 5))
    u[1, 2] = 1.0           # (x=2, y=1): north neighbour of (2,2)
    R.colour_pass(u, "fd5", 0)   # (2,2) has colour 0
    assert u[2, 2] == 0.25


@pytest.mark.parametrize("name", list(R.STENCIL_TABLE))
def test_constant_mesh_fixed_point(name):
    dim = R.STENCIL_TABLE[name][0]
    u = np.full((6,) * dim, 1.75)
    R.sweep(u, name, 2)
    assert np.allclose(u, 1.75, rtol=1e-12, atol=0)


def test_colour_ids():
    # reference tests/test_strategies.py:25-38
    assert R.colour_of("fd5", (1, 1)) == 0 and R.colour_of("fd5", (2, 1)) == 1
    assert R.colour_of("fe9", (2, 2)) == 3
    assert R.colour_of("fd7", (1, 1, 1)) == 0
    assert R.colour_of("fe27", (2, 1, 2)) == 5


def test_q1_weights():
    dim, offs, w, wc, c = R.STENCIL_TABLE["fe27q1"]
    assert wc == 8.0 / 3.0 and c == 8 and len(offs) == 26
    assert sum(1 for x in w if x == 0.0) == 6
    assert sum(1 for x in w if x == -1.0 / 6.0) == 12
    assert sum(1 for x in w if x == -1.0 / 12.0) == 8
    assert abs(wc + sum(w)) < 1e-12


def test_nonfinite_raises():
    u = R.init_u(2, 4, 1)
    u[1, 0] = np.nan
    with pytest.raises(R.OracleNumericsError):
        R.colour_pass(u, "fd5", 0)
    with pytest.raises(R.OracleNumericsError):
        coracle.sweep(u, "fd5", 1)


# -- lexicographic (serial) order ---------------------------------------------

@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_lex_matches_reference_serial_digests(ref_digests, impl):
    """Reference serial == taskgraph digests (strategies.py:341-345, :477-487)."""
    for key, want in ref_digests["serial"].items():
        name, n, sweeps, seed, b = _parse(key)
        u = R.init_u(R.STENCIL_TABLE[name][0], n, seed, b)
        if impl == "numpy":
            R.lex_sweep(u, name, sweeps)
        else:
            coracle.sweep(u, name, sweeps, order="lex")
        assert _digest(u) == want, (key, impl)


def test_lex_small_buffers_bitwise():
    small = np.load(os.path.join(GOLDEN, "reference_small.npz"))
    for name in REF_KINDS:
        dim = R.STENCIL_TABLE[name][0]
        u = R.init_u(dim, 10 if dim == 2 else 6, 11)
        coracle.sweep(u, name, 5, order="lex")
        assert np.array_equal(u.reshape(-1).view(np.int64),
                              small["serial_" + name].view(np.int64)), name


def test_lex_kat_degenerate_row():
    """One live row (a, b, c) under a zero halo: a'=b/4, b'=(a'+c)/4, c'=b'/4
    (restates reference tests/test_strategies.py:74-89)."""
    a, b, c = 0.8, 0.3, 0.5
    u = np.zeros((5, 5))
    u[1, 1:4] = (a, b, c)
    R.lex_sweep(u, "fd5", 1)
    a2 = b / 4
    b2 = (a2 + c) / 4
    assert tuple(u[1, 1:4]) == (a2, b2, b2 / 4)


@pytest.mark.parametrize("name", list(R.STENCIL_TABLE))
def test_lex_numpy_and_c_agree_form_d(name):
    dim = R.STENCIL_TABLE[name][0]
    n = 11 if dim == 2 else 5
    u = R.init_u(dim, n, 2)
    f = R.init_f(dim, n, 3)
    v = u.copy()
    R.lex_sweep(u, name, 2, f=f, omega=0.8, form="D")
    coracle.sweep(v, name, 2, f=f, omega=0.8, form="D", order="lex")
    assert np.array_equal(u.view(np.int64), v.view(np.int64))


def test_lex_convergence_budget_matches_reference(ref_digests):
    """serial_convergence_budget (bench.py:433-442) replayed on the C lex sweep."""
    for key, want in ref_digests["convergence"].items():
        name = key.split("/")[0]
        n = int(key.split("n=")[1].split("/")[0])
        u = R.init_u(R.STENCIL_TABLE[name][0], n, 7)
        got = None
        for s in range(1, 20001):
            coracle.sweep(u, name, 1, order="lex", threads=1)
            if R.residual_max(u, name) < 1e-8:
                got = s
                break
        assert got == want, key
