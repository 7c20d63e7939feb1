"""Batched patches (BASELINE config 5) against the oracle, bit for bit."""

import numpy as np
import pytest

import paper_1810_04033_b200 as sl
from oracle import coracle
from oracle import restate as R

pytestmark = pytest.mark.gpu


def _bits(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def test_init_patches_matches_oracle_definition():
    u, f = sl.init_patches(5, 16, 9)
    ru, rf = R.init_patches(5, 16, 9)
    assert _bits(u, ru) and _bits(f, rf)


@pytest.mark.parametrize("n", [16, 10, 6])
@pytest.mark.parametrize("form", ["R", "D"])
def test_patches_match_oracle(n, form):
    u, f = R.init_patches(257, n, 3)
    want = u.copy()
    coracle.sweep(want, "fd5", 7, f=f if form == "D" else None, omega=0.8, form=form)
    pb = sl.PatchBatch(u, f if form == "D" else None, omega=0.8)
    pb.sweep(sl.FD5, 7)
    assert _bits(pb.values(), want)


def test_patches_split_calls_equal_one_call():
    u, f = R.init_patches(64, 16, 4)
    a = sl.PatchBatch(u, f)
    a.sweep(sl.FD5, 10)
    b = sl.PatchBatch(u, f)
    for _ in range(10):
        b.sweep(sl.FD5, 1)
    assert _bits(a.values(), b.values())


def test_patch_equals_single_mesh_path():
    u, f = R.init_patches(3, 16, 5)
    pb = sl.PatchBatch(u, f)
    pb.sweep(sl.FD5, 9)
    for k in range(3):
        m = sl.Mesh(2, 16)
        m.values[:] = u[k].ravel()
        m.set_rhs(f[k].ravel(), 0.8)
        sl.run_sweeps(m, sl.FD5, sl.CostModel(), 9, flags=1)   # K1 per colour
        assert _bits(m.values, pb.values()[k].ravel())


def test_patches_halo_fixed_and_nonfinite():
    u, f = R.init_patches(8, 16, 6)
    pb = sl.PatchBatch(u, f)
    pb.sweep(sl.FD5, 5)
    v = pb.values()
    assert _bits(v[:, 0, :], u[:, 0, :]) and _bits(v[:, :, 17], u[:, :, 17])
    u[3, 5, 0] = np.inf
    with pytest.raises(sl.NumericsError):
        sl.PatchBatch(u, f).sweep(sl.FD5, 2)


def test_config5_full_size():
    u, f = R.init_patches(65536, 16, 42)
    want = u.copy()
    coracle.sweep(want, "fd5", 200, f=f, omega=0.8, form="D")
    pb = sl.PatchBatch(u, f)
    pb.sweep(sl.FD5, 200)
    assert _bits(pb.values(), want)
