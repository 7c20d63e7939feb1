"""ctypes binding of the sm_100a library (include/stencil_sweep.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every device entry point raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libstencil_sweep.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "stencil_sweep.h")

SL_OK, SL_E_NONFINITE, SL_E_INVAL, SL_E_CUDA, SL_E_UNSUPPORTED = 0, 1, 2, 3, 4
SL_FD5, SL_FE9, SL_FD7, SL_FE27 = 0, 1, 2, 3
SL_FORM_R, SL_FORM_D = 0, 1
SL_FLAG_PER_COLOUR = 0x1
SL_FLAG_MERGE_COLOURS = 0x2
SL_FLAG_STREAM = 0x4
SL_FLAG_LEX = 0x8
SL_COST_CONST, SL_COST_RAMP = 0, 1
ABI_VERSION = 1

# every symbol include/stencil_sweep.h declares (checked by tests/test_abi.py)
EXPORTS = ("sl_abi_version", "sl_strerror", "sl_last_cuda_error", "sl_launch_count",
           "sl_workspace_bytes",
           "sl_sweep", "sl_colour_pass", "sl_update_cells", "sl_residual_max", "sl_ghost_depth",
           "sl_sweep_cost", "sl_update_cells_cost", "sl_sweep_pass", "sl_sweep_pass_peer")


class NativeLibraryError(RuntimeError):
    """The CUDA library or device is unavailable (there is no CPU fallback)."""


class SlGrid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("n", ctypes.c_int64 * 3), ("batch", ctypes.c_int64),
                ("batch_stride", ctypes.c_int64), ("origin", ctypes.c_int64 * 3),
                ("u", ctypes.c_void_p), ("f", ctypes.c_void_p)]


class SlStencil(ctypes.Structure):
    _fields_ = [("shape", ctypes.c_int32), ("colours", ctypes.c_int32),
                ("form", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("w", ctypes.c_double * 26), ("wc", ctypes.c_double),
                ("omega", ctypes.c_double)]


class SlCost(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("k", ctypes.c_int32), ("d_work", ctypes.c_void_p)]


_lib = None

_P = ctypes.POINTER
_SIGS = {
    "sl_abi_version": (ctypes.c_int, []),
    "sl_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "sl_last_cuda_error": (ctypes.c_int, []),
    "sl_launch_count": (ctypes.c_uint64, []),
    "sl_workspace_bytes": (ctypes.c_size_t, [_P(SlGrid), _P(SlStencil)]),
    "sl_sweep": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_int32, ctypes.c_uint32,
                                ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]),
    "sl_sweep_pass": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "sl_sweep_pass_peer": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "sl_colour_pass": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_int32,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "sl_update_cells": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "sl_residual_max": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "sl_ghost_depth": (ctypes.c_int, [_P(SlStencil), ctypes.c_int32, ctypes.c_int32]),
    "sl_sweep_cost": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), _P(SlCost), ctypes.c_int32,
                                     ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]),
    "sl_update_cells_cost": (ctypes.c_int, [_P(SlGrid), _P(SlStencil), ctypes.c_void_p,
                                            ctypes.c_int64, _P(SlCost), ctypes.c_void_p,
                                            ctypes.c_void_p]),
}


def load():
    """Load the library (no device needed); raises NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sl_abi_version() != ABI_VERSION:
        raise NativeLibraryError(f"ABI mismatch: library {lib.sl_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the sweep runs only on the GPU (no CPU fallback)")
    return load()


def check(rc: int, what: str):
    """Map a C-ABI status to the reference's exception types."""
    if rc == SL_OK:
        return
    lib = load()
    msg = lib.sl_strerror(rc).decode()
    if rc == SL_E_INVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == SL_E_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    if rc == SL_E_CUDA:
        raise RuntimeError(f"{what}: {msg} (cudaError {lib.sl_last_cuda_error()})")
    raise RuntimeError(f"{what}: status {rc} ({msg})")
