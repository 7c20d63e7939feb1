"""Cartesian cell-value grids with a one-cell fixed-value halo, device-resident.

Mirror of the reference `stencil_lab.mesh` (mesh.py:1-117): same layout — one
dense fp64 buffer of (n+2)^dim cells, x fastest, index(x,y) = y*(n+2)+x,
index(x,y,z) = (z*(n+2)+y)*(n+2)+x (mesh.py:42-51) — and the same seeded
init (mesh.py:102-112).  The authoritative copy lives in HBM as a torch
float64 tensor; `values` is a host mirror that keeps the reference's
observable semantics (tests read and write `mesh.values` between sweeps,
reference tests/test_strategies.py:97-99, :178-186):

* reading `values` downloads the device copy (into the same host buffer) and
  hands the host buffer out as authoritative — the caller may mutate it;
* the next device operation uploads it again.

Form D (BASELINE configs) attaches a right-hand side f and a damping factor
to the mesh (`set_rhs`), so the reference entry points keep their
signatures; without one the reference update (Form R) runs.
"""

from __future__ import annotations

import numpy as np

__all__ = ["Mesh", "init", "init_rhs", "make_mesh"]


def _torch():
    import torch
    return torch


def _alloc_host(count: int) -> np.ndarray:
    """Zeroed fp64 host buffer; page-locked when a CUDA device is present so
    host<->device mirroring runs at full PCIe/C2C speed."""
    try:
        torch = _torch()
        if torch.cuda.is_available():
            return torch.zeros(count, dtype=torch.float64, pin_memory=True).numpy()
    except Exception:
        pass
    return np.zeros(count, dtype=np.float64)


class Mesh:
    """Flat float64 cell storage for a dim-dimensional grid, halo included."""

    __slots__ = ("dim", "n", "side", "strides", "device", "omega",
                 "_host", "_dev", "_where", "_interior_flat", "_rhs_host", "_rhs_dev",
                 "_ws", "__weakref__")

    def __init__(self, dim: int, n: int, device=None):
        if dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {dim}")
        if n < 1:
            raise ValueError(f"interior extent must be >= 1, got {n}")
        self.dim = dim
        self.n = n
        self.side = n + 2
        self.strides = tuple(self.side ** a for a in range(dim))
        self.device = device
        self.omega = None
        self._host = _alloc_host(self.side ** dim)
        self._dev = None
        self._where = "host"
        self._interior_flat = None
        self._rhs_host = None
        self._rhs_dev = None
        self._ws = None

    # -- host/device mirror ---------------------------------------------------

    @property
    def size(self) -> int:
        return self.side ** self.dim

    @property
    def values(self) -> np.ndarray:
        """Writable host view of the buffer (synchronises with the device
        first).  The caller may mutate it, so the host copy becomes the
        authoritative one and the next device call uploads it again; readers
        that only look use `read_values()`, which skips that upload."""
        if self._where == "dev":
            self._dev_to_host()
        self._where = "host"   # the caller may mutate it
        return self._host

    def read_values(self) -> np.ndarray:
        """Read-only host view of the buffer.  Unlike `values` it leaves the
        device copy authoritative, so the next sweep does not upload the
        whole grid again (8.6 GB for BASELINE config 4): use it for digests,
        comparisons and output.  The view is valid until the next device
        call; writes go through `values`."""
        if self._where == "dev":
            self._dev_to_host()
        view = self._host.view()
        view.flags.writeable = False
        return view

    @values.setter
    def values(self, arr):
        arr = np.asarray(arr, dtype=np.float64).reshape(-1)
        if arr.shape != self._host.shape:
            raise ValueError(f"expected {self._host.shape[0]} values, got {arr.shape[0]}")
        self._host[:] = arr
        self._where = "host"

    def _torch_device(self):
        torch = _torch()
        if self.device is None:
            if not torch.cuda.is_available():
                from ._native import NativeLibraryError
                raise NativeLibraryError("no CUDA device: the sweep runs only on the GPU (no CPU fallback)")
            self.device = torch.device("cuda", torch.cuda.current_device())
        return torch.device(self.device)

    def device_values(self):
        """The authoritative device tensor (uploads pending host edits).

        Callers that write it must not read `values` concurrently; device
        kernels launched through this package keep it authoritative.
        """
        torch = _torch()
        dev = self._torch_device()
        if self._dev is None:
            # no device copy yet: the host buffer is authoritative
            self._dev = torch.empty(self.size, dtype=torch.float64, device=dev)
            self._dev.copy_(torch.from_numpy(self._host))
        elif self._where == "host":
            self._dev.copy_(torch.from_numpy(self._host))
        self._where = "dev"
        return self._dev

    def _dev_to_host(self):
        torch = _torch()
        torch.from_numpy(self._host).copy_(self._dev)

    def adopt_device(self, tensor):
        """Make `tensor` (float64, (n+2)^dim, on a CUDA device) the authoritative buffer."""
        torch = _torch()
        if tensor.dtype != torch.float64 or tensor.numel() != self.size or not tensor.is_cuda:
            raise ValueError("need a CUDA float64 tensor of (n+2)^dim elements")
        self._dev = tensor.reshape(-1)
        self.device = tensor.device
        self._where = "dev"

    # -- right-hand side (Form D) ----------------------------------------------

    def set_rhs(self, f, omega: float = 0.8):
        """Attach f (dense (n+2)^dim, zero halo) and damping omega: sweeps
        then run Form D, u <- u + omega*(f - A u)/w_c."""
        if f is None:
            self._rhs_host = self._rhs_dev = None
            self.omega = None
            return
        torch = _torch()
        if isinstance(f, torch.Tensor) and f.is_cuda:
            if f.numel() != self.size or f.dtype != torch.float64:
                raise ValueError("rhs must be float64 with (n+2)^dim elements")
            self._rhs_host = None
            self._rhs_dev = f.reshape(-1)
        elif isinstance(f, torch.Tensor):
            # host tensor (pinned ones upload asynchronously)
            if f.numel() != self.size or f.dtype != torch.float64:
                raise ValueError("rhs must be float64 with (n+2)^dim elements")
            self._rhs_host = f.reshape(-1)
            self._rhs_dev = None
        else:
            f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
            if f.size != self.size:
                raise ValueError("rhs must have (n+2)^dim elements")
            self._rhs_host = f
            self._rhs_dev = None
        self.omega = float(omega)

    @property
    def has_rhs(self) -> bool:
        return self._rhs_host is not None or self._rhs_dev is not None

    def rhs_device(self):
        if self._rhs_dev is None and self._rhs_host is not None:
            torch = _torch()
            host = self._rhs_host
            if not isinstance(host, torch.Tensor):
                host = torch.from_numpy(host)
            self._rhs_dev = host.to(self._torch_device(), non_blocking=True)
        return self._rhs_dev

    def workspace(self, nbytes: int):
        """Device scratch reused across sweeps (fusion ping-pong buffer)."""
        if nbytes <= 0:
            return None
        torch = _torch()
        if self._ws is None or self._ws.numel() * 8 < nbytes:
            self._ws = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=self._torch_device())
        return self._ws

    # -- index arithmetic (reference mesh.py:38-99) ------------------------------

    @property
    def interior_count(self) -> int:
        return self.n ** self.dim

    def flat_index(self, coord) -> int:
        """Row-major flat index of `coord`; raises IndexError out of bounds."""
        if len(coord) != self.dim:
            raise IndexError(f"expected {self.dim} coordinates, got {coord!r}")
        flat = 0
        for c in reversed(coord):
            if not 0 <= c <= self.n + 1:
                raise IndexError(f"coordinate {coord!r} outside [0, {self.n + 1}]")
            flat = flat * self.side + c
        return flat

    def coord_of(self, flat: int):
        if not 0 <= flat < self.size:
            raise IndexError(f"flat index {flat} outside buffer")
        coord = []
        for _ in range(self.dim):
            flat, c = divmod(flat, self.side)
            coord.append(c)
        return tuple(coord)

    def is_interior(self, coord) -> bool:
        return all(1 <= c <= self.n for c in coord)

    def interior_coords(self):
        rng = range(1, self.n + 1)
        if self.dim == 2:
            for y in rng:
                for x in rng:
                    yield (x, y)
        else:
            for z in rng:
                for y in rng:
                    for x in rng:
                        yield (x, y, z)

    def interior_flat(self) -> np.ndarray:
        if self._interior_flat is None:
            axis = np.arange(1, self.n + 1)
            if self.dim == 2:
                flats = axis[:, None] * self.side + axis[None, :]
            else:
                flats = (axis[:, None, None] * self.side + axis[None, :, None]) * self.side + axis[None, None, :]
            self._interior_flat = flats.ravel().astype(np.int64)
        return self._interior_flat

    def halo_flat(self) -> np.ndarray:
        mask = np.ones(self.size, dtype=bool)
        mask[self.interior_flat()] = False
        return np.flatnonzero(mask)

    def copy(self) -> "Mesh":
        other = Mesh(self.dim, self.n, device=self.device)
        other.values[:] = self.values
        if self.has_rhs:
            other.set_rhs(self._rhs_host if self._rhs_host is not None else self._rhs_dev.clone(), self.omega)
        return other


def init(mesh: Mesh, interior_seed: int, boundary_value: float = 0.0) -> Mesh:
    """Halo = boundary_value, interior = default_rng(seed).random(n^dim) in
    lexicographic order — bit-identical to reference mesh.py:102-112."""
    host = mesh.values
    host.fill(boundary_value)
    rng = np.random.default_rng(interior_seed)
    host[mesh.interior_flat()] = rng.random(mesh.interior_count)
    return mesh


def init_rhs(mesh: Mesh, seed: int, omega: float = 0.8) -> Mesh:
    """f ~ U[-1,1) = default_rng(seed).uniform(-1, 1, n^dim) in lex order,
    zero halo (SURVEY.md §8d convention: seed = u seed + 1)."""
    f = np.zeros(mesh.size, dtype=np.float64)
    f[mesh.interior_flat()] = np.random.default_rng(seed).uniform(-1.0, 1.0, mesh.interior_count)
    mesh.set_rhs(f, omega)
    return mesh


def make_mesh(dim: int, n: int, seed: int = 0, boundary_value: float = 0.0) -> Mesh:
    return init(Mesh(dim, n), seed, boundary_value)
