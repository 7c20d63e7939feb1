"""The C-ABI library: loads, exports every declared symbol, validates
arguments before touching the device (CPU only, no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1810_04033_b200 import _native
from paper_1810_04033_b200.kernels import FD5, FE27Q1, FE9

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(_native.HEADER_PATH).read()
    return sorted(set(re.findall(r"SL_API\s+[\w\s\*]+?\b(sl_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    declared = _declared()
    assert declared == sorted(_native.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (sl_\w+)", out))
    assert exported == set(declared)
    for name in declared:
        assert hasattr(lib, name)


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_strerror():
    lib = _native.load()
    assert lib.sl_abi_version() == _native.ABI_VERSION
    assert lib.sl_strerror(0) == b"ok"
    assert b"non-finite" in lib.sl_strerror(1)


def test_struct_layout_matches_header(tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "stencil_sweep.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sl_grid), offsetof(sl_grid,u),'
        ' offsetof(sl_grid,f), sizeof(sl_stencil), offsetof(sl_stencil,w), offsetof(sl_stencil,wc),'
        ' offsetof(sl_stencil,omega));printf("%zu %zu %zu\\n", sizeof(sl_cost), offsetof(sl_cost,k),'
        ' offsetof(sl_cost,d_work));return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(prog)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_native.SlGrid), _native.SlGrid.u.offset, _native.SlGrid.f.offset,
            ctypes.sizeof(_native.SlStencil), _native.SlStencil.w.offset,
            _native.SlStencil.wc.offset, _native.SlStencil.omega.offset,
            ctypes.sizeof(_native.SlCost), _native.SlCost.k.offset, _native.SlCost.d_work.offset]
    assert got == want


def _grid(dim=2, n=8, u=0x1000):
    g = _native.SlGrid()
    g.dim = dim
    for a in range(dim):
        g.n[a] = n
    g.batch = 1
    g.batch_stride = (n + 2) ** dim
    g.u = u
    return g


def _sweep(g, s, sweeps=1, status=0x2000):
    lib = _native.load()
    return lib.sl_sweep(ctypes.byref(g), ctypes.byref(s), sweeps, 0, None, 0, status, None)


def test_invalid_arguments_rejected_before_launch():
    s = FD5.descriptor(_native.SL_FORM_R)
    assert _sweep(_grid(dim=3), s) == _native.SL_E_INVAL          # dim mismatch
    assert _sweep(_grid(u=0), s) == _native.SL_E_INVAL            # null u
    assert _sweep(_grid(), s, sweeps=-1) == _native.SL_E_INVAL
    assert _sweep(_grid(), s, status=0) == _native.SL_E_INVAL     # no status word
    d = FD5.descriptor(_native.SL_FORM_D, 0.8)
    assert _sweep(_grid(), d) == _native.SL_E_INVAL               # form D without f
    bad = FE9.descriptor(_native.SL_FORM_R)
    bad.colours = 2                                               # red-black on a box stencil
    assert _sweep(_grid(), bad) == _native.SL_E_INVAL
    odd = FD5.descriptor(_native.SL_FORM_R)
    odd.w[1] = 0.0                                                # zero pattern without a kernel
    assert _sweep(_grid(), odd) == _native.SL_E_UNSUPPORTED
    g = _grid()
    g.batch = 2
    g.batch_stride = 10                                           # overlapping grids
    assert _sweep(g, s) == _native.SL_E_INVAL
    lib = _native.load()
    st = ctypes.c_int32(0)
    g = _grid()
    src, dst = g.u, g.u + 4096
    for a, b in ((-1, 3), (3, 2), (0, 10 ** 6)):                  # plane window out of range
        assert lib.sl_sweep_pass(ctypes.byref(g), ctypes.byref(s), src, dst, a, b,
                                 ctypes.addressof(st), None) == _native.SL_E_INVAL
    assert lib.sl_sweep_pass(ctypes.byref(g), ctypes.byref(s), src, src, 0, 1,
                             ctypes.addressof(st), None) == _native.SL_E_INVAL   # in place


def test_cost_sweep_arguments_rejected_before_launch():
    lib = _native.load()
    s = FD5.descriptor(_native.SL_FORM_R)

    def call(cost, flags=0, g=None):
        return lib.sl_sweep_cost(ctypes.byref(g or _grid()), ctypes.byref(s),
                                 ctypes.byref(cost), 1, flags, 0x2000, None)

    bad_mode = _native.SlCost(7, 1, None)
    assert call(bad_mode) == _native.SL_E_INVAL
    assert call(_native.SlCost(_native.SL_COST_CONST, -1, None)) == _native.SL_E_INVAL
    assert call(_native.SlCost(_native.SL_COST_CONST, 1, None),
                flags=_native.SL_FLAG_STREAM) == _native.SL_E_INVAL
    g = _grid()
    g.origin[1] = 5                                               # slab: ramp rank is global
    assert call(_native.SlCost(_native.SL_COST_RAMP, 0, None), g=g) == _native.SL_E_UNSUPPORTED
    assert lib.sl_update_cells_cost(ctypes.byref(_grid()), ctypes.byref(s), None, 1,
                                    ctypes.byref(_native.SlCost(_native.SL_COST_CONST, 2, None)),
                                    0x2000, None) == _native.SL_E_INVAL


def test_zero_sweeps_and_empty_grid_are_noops():
    s = FD5.descriptor(_native.SL_FORM_R)
    assert _sweep(_grid(), s, sweeps=0) == _native.SL_OK
    assert _sweep(_grid(n=0), s) == _native.SL_OK


def test_q1_pattern_accepted():
    q = FE27Q1.descriptor(_native.SL_FORM_D, 0.8)
    g = _grid(dim=3)
    g.f = 0x3000
    lib = _native.load()
    # workspace query is pure host arithmetic
    lib.sl_workspace_bytes(ctypes.byref(g), ctypes.byref(q))
    assert _sweep(g, q, sweeps=0) == _native.SL_OK


def test_check_maps_status_to_reference_exceptions():
    with pytest.raises(ValueError):
        _native.check(_native.SL_E_INVAL, "x")
    with pytest.raises(NotImplementedError):
        _native.check(_native.SL_E_UNSUPPORTED, "x")
    _native.check(_native.SL_OK, "x")
