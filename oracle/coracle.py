"""ctypes front end of the C restatement (oracle/sweep_oracle.c).

TEST INFRASTRUCTURE (see oracle/__init__.py): used by tests/ as the
large-size checker and by bench.py as the CPU baseline ("port").
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .restate import STENCIL_TABLE, OracleNumericsError

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_sweep.restype = ctypes.c_int
        lib.oracle_sweep.argtypes = [
            ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
            ctypes.c_double, ctypes.c_int, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return _load().oracle_max_threads()


def sweep(u, name, sweeps=1, f=None, omega=0.8, form="R", threads=0, order="colour"):
    """In-place colour sweeps of u (shape (..., S, S[, S]), C-contiguous fp64).
    order="lex": lexicographic (reference serial) sweeps instead."""
    dim, offsets, weights, wc, colours = STENCIL_TABLE[name]
    if not (u.flags.c_contiguous and u.dtype == np.float64):
        raise ValueError("u must be C-contiguous float64")
    n = u.shape[-1] - 2
    grid = (n + 2) ** dim
    batch = u.size // grid
    keep = [(o, w) for o, w in zip(offsets, weights) if w != 0.0]
    off = np.zeros((len(keep), 3), dtype=np.int32)
    for j, (o, _) in enumerate(keep):
        off[j, :dim] = o
    w = np.array([wj for _, wj in keep], dtype=np.float64)
    fp = None
    if form == "D":
        if f is None or f.shape != u.shape or not f.flags.c_contiguous:
            raise ValueError("form D needs f with u's shape")
        fp = f.ctypes.data
    rc = _load().oracle_sweep(dim, n, batch, grid, u.ctypes.data, fp, len(keep),
                              off.ctypes.data, w.ctypes.data, wc,
                              colours if order == "colour" else 0,
                              0 if form == "R" else 1, omega, sweeps, threads)
    if rc == 1:
        raise OracleNumericsError("non-finite update")
    if rc != 0:
        raise ValueError(f"oracle_sweep rc={rc}")
    return u
