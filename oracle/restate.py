"""NumPy strided-slice restatement of the reference colour sweep.

TEST INFRASTRUCTURE (see oracle/__init__.py): never imported by the product.

Reference algorithm followed (paths under /root/reference/pkg/src/stencil_lab):

* layout — one dense float64 buffer of (n+2)^dim cells, x fastest
  (mesh.py:20-35, flat index mesh.py:42-51); here held as an ndarray of shape
  (S,)*dim indexed [z, y, x] (identical bytes), optionally with leading batch
  axes (independent patches).
* init — halo = boundary value, interior = default_rng(seed).random(n^dim) in
  lexicographic order (mesh.py:102-112).
* stencils — offsets in canonical order = sorted by reversed displacement =
  ascending flat delta (kernels.py:78-80, :98-101).
* colour id — parity relative to cell (1,..,1): 2 colours ->
  (sum(c) - dim) % 2, 2^d colours -> sum(((c_a - 1) & 1) << a)
  (strategies.py:62-69, :201-214); colours run 0..c-1 within a sweep
  (strategies.py:371-393, oracle strategies.py:420-433).
* Form R arithmetic (bit-exact target) — acc = +0.0; for each neighbour in
  canonical order acc = acc + |w_j| * u_j (|w|==1 makes the multiply exact,
  so this equals the reference's plain add); u_c = acc / w_c
  (kernels.py:224-232 batch path, :168-200 scalar path).
* non-finite results raise (kernels.py:247-249).

Form D (BASELINE.json configs; no reference counterpart) is defined
HERE and mirrored by the CUDA kernels:

    Au = w_c * u_c
    for j in canonical order with w_j != 0:  Au = Au + (w_j * u_j)
    u_c = u_c + omega * ((f_c - Au) / w_c)

every operation a separately rounded IEEE binary64 op (no FMA), zero-weight
offsets skipped (FE27-Q1 faces).  Each colour class is a union of per-axis
parity sub-lattices; each is a strided slice, so a colour pass is a handful of
whole-array ufunc calls with exactly the per-point operation sequence above.
"""

from __future__ import annotations

import itertools

import numpy as np


class OracleNumericsError(ArithmeticError):
    pass


# -- stencil tables (independent restatement of kernels.py:98-101 + Q1) -------

def _canonical(offsets):
    # kernels.py:78-80: sort by reversed displacement (outer axis slowest)
    return tuple(sorted(offsets, key=lambda off: tuple(reversed(off))))


def _face(dim):
    offs = []
    for a in range(dim):
        for s in (-1, 1):
            o = [0] * dim
            o[a] = s
            offs.append(tuple(o))
    return _canonical(offs)


def _box(dim):
    return _canonical([o for o in itertools.product((-1, 0, 1), repeat=dim) if any(o)])


def _q1_weight(off):
    nz = sum(1 for c in off if c)
    return {1: 0.0, 2: -1.0 / 6.0, 3: -1.0 / 12.0}[nz]


# name -> (dim, offsets, weights, centre weight, colours)
STENCIL_TABLE = {
    "fd5": (2, _face(2), (-1.0,) * 4, 4.0, 2),
    "fe9": (2, _box(2), (-1.0 / 3.0,) * 8, 8.0 / 3.0, 4),
    "fd7": (3, _face(3), (-1.0,) * 6, 6.0, 2),
    "fe27": (3, _box(3), (-1.0,) * 26, 26.0, 8),
    # BASELINE config 4: trilinear Q1 (centre 8/3, faces 0, edges -1/6, corners -1/12)
    "fe27q1": (3, _box(3), tuple(_q1_weight(o) for o in _box(3)), 8.0 / 3.0, 8),
}


def colour_of(name, coord):
    dim, _, _, _, colours = STENCIL_TABLE[name]
    if colours == 2:
        return (sum(coord) - dim) % 2
    code = 0
    for a, c in enumerate(coord):
        code |= ((c - 1) & 1) << a
    return code


def _parity_vectors(dim, colours, colour, origin=(0, 0, 0)):
    """Local per-axis parity vectors q (local c_a = 1 + q_a + 2k, a=0 is x)
    of the cells of `colour`; colours use GLOBAL coordinates c_a + origin_a
    (a slab of a larger grid keeps the global colouring)."""
    out = []
    for q in itertools.product((0, 1), repeat=dim):   # q[0] = x parity
        g = [(q[a] + origin[a]) & 1 for a in range(dim)]
        if colours == 2:
            c = sum(g) % 2
        else:
            c = sum(bit << a for a, bit in enumerate(g))
        if c == colour:
            out.append(q)
    return out


def _sl(n, q_axis, shift):
    return slice(1 + q_axis + shift, n + 1 + shift, 2)


# -- sweeps -------------------------------------------------------------------

def colour_pass(u, name, colour, f=None, omega=None, form="R", origin=(0, 0, 0)):
    """One colour phase in place on u (shape (..., S[, S], S)); the slowest
    axis may differ in length (slabs)."""
    dim, offsets, weights, wc, colours = STENCIL_TABLE[name]
    ns = [u.shape[-1 - a] - 2 for a in range(dim)]   # interior extent per axis (x, y, z)
    lead = (slice(None),) * (u.ndim - dim)
    for q in _parity_vectors(dim, colours, colour, origin):
        # array axes are reversed coordinate axes: [.., z, y, x]
        centre = lead + tuple(_sl(ns[a], q[a], 0) for a in reversed(range(dim)))
        if u[centre].size == 0:
            continue
        if form == "R":
            acc = np.zeros(u[centre].shape)
            for off, w in zip(offsets, weights):
                if w == 0.0:
                    continue
                nb = lead + tuple(_sl(ns[a], q[a], off[a]) for a in reversed(range(dim)))
                acc += abs(w) * u[nb]
            out = acc / wc
        elif form == "D":
            uc = u[centre]
            au = wc * uc
            for off, w in zip(offsets, weights):
                if w == 0.0:
                    continue
                nb = lead + tuple(_sl(ns[a], q[a], off[a]) for a in reversed(range(dim)))
                au = au + w * u[nb]
            out = uc + omega * ((f[centre] - au) / wc)
        else:
            raise ValueError(form)
        if not np.isfinite(out).all():
            raise OracleNumericsError(f"non-finite update in colour {colour}")
        u[centre] = out


def sweep(u, name, sweeps=1, f=None, omega=None, form="R", origin=(0, 0, 0)):
    """`sweeps` full colour-ordered sweeps in place (strategies.py:371-393)."""
    colours = STENCIL_TABLE[name][4]
    for _ in range(sweeps):
        for c in range(colours):
            colour_pass(u, name, c, f=f, omega=omega, form=form, origin=origin)
    return u


def lex_sweep(u, name, sweeps=1, f=None, omega=None, form="R"):
    """Lexicographic Gauss-Seidel sweeps in place (reference serial sweep,
    strategies.py:341-345: cells in increasing flat index, strategies.py:226-234,
    each one kernels.py:224-232).  Pure-Python loops: small grids only."""
    dim, offsets, weights, wc, _ = STENCIL_TABLE[name]
    n = u.shape[-1] - 2
    keep = [(off, w) for off, w in zip(offsets, weights) if w != 0.0]
    flat = u.reshape(-1)
    strides = [1, n + 2, (n + 2) ** 2][:dim]
    deltas = [sum(o * s_ for o, s_ in zip(off, strides)) for off, _ in keep]
    ws = [w for _, w in keep]
    aws = [abs(w) for w in ws]
    ff = f.reshape(-1) if f is not None else None
    cells = sorted(sum((c + 1) * s_ for c, s_ in zip(coord, strides))
                   for coord in np.ndindex(*((n,) * dim)))
    for _ in range(sweeps):
        for c in cells:
            if form == "R":
                acc = 0.0
                for d, aw in zip(deltas, aws):
                    acc = acc + aw * float(flat[c + d])
                out = acc / wc
            else:
                uc = float(flat[c])
                au = wc * uc
                for d, w in zip(deltas, ws):
                    au = au + w * float(flat[c + d])
                out = uc + omega * ((float(ff[c]) - au) / wc)
            if not np.isfinite(out):
                raise OracleNumericsError("non-finite update")
            flat[c] = out
    return u


def residual_max(u, name, f=None):
    """max |w_c u + sum_j w_j u_j| (kernels.py:254-265); with f: max |f - Au|."""
    dim, offsets, weights, wc, _ = STENCIL_TABLE[name]
    n = u.shape[-1] - 2
    lead = (slice(None),) * (u.ndim - dim)
    inner = lead + (slice(1, n + 1),) * dim
    acc = wc * u[inner]
    for off, w in zip(offsets, weights):
        if w == 0.0:
            continue
        nb = lead + tuple(slice(1 + off[a], n + 1 + off[a]) for a in reversed(range(dim)))
        acc += w * u[nb]
    if f is not None:
        acc = f[inner] - acc
    return float(np.abs(acc).max()) if acc.size else 0.0


# -- seeded inputs (mesh.py:102-112 for u; f / patches defined here) -

def init_u(dim, n, seed, boundary=0.0):
    s = n + 2
    u = np.full((s,) * dim, boundary, dtype=np.float64)
    u[(slice(1, n + 1),) * dim] = np.random.default_rng(seed).random(n ** dim).reshape((n,) * dim)
    return u


def init_f(dim, n, seed):
    """f ~ U[-1,1) from default_rng(seed) in lex order, dense with zero halo."""
    s = n + 2
    f = np.zeros((s,) * dim, dtype=np.float64)
    f[(slice(1, n + 1),) * dim] = np.random.default_rng(seed).uniform(-1.0, 1.0, n ** dim).reshape((n,) * dim)
    return f


def init_patches(batch, n, seed):
    """Config 5: u incl. halo ~ U[0,1) (default_rng(seed).random((B,S,S))),
    f ~ U[-1,1) (default_rng(seed+1).uniform(-1,1,(B,n,n))) dense, zero halo."""
    s = n + 2
    u = np.random.default_rng(seed).random((batch, s, s))
    f = np.zeros((batch, s, s))
    f[:, 1:n + 1, 1:n + 1] = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, (batch, n, n))
    return u, f
