"""Slab kernels on the GPU: several slabs of one grid emulated on one device.

The exchange is done with device-to-device copies mirroring
SlabRunner.exchange (one process, so no NCCL rendezvous is needed); this
checks the fused kernels with odd slab origins and ghost depths.  The NCCL
P2P path itself is covered on CPU with gloo (tests/test_slabs.py).
"""

import numpy as np
import pytest

import paper_1810_04033_b200 as sl
from oracle import coracle
from oracle import restate as R
from paper_1810_04033_b200.slabs import SlabRunner

pytestmark = pytest.mark.gpu


def _emulated(name, n, sweeps, world, per, overlap=False, runners=None):
    kind = sl.get_stencil(name)
    rs = [SlabRunner(kind.dim, n, kind, world=world, rank=r, ghost_sweeps=per, device="cuda",
                     overlap=overlap) for r in range(world)]
    for r in rs:
        r.init(7, 8, 0.8)
    left = sweeps
    while left > 0:
        k = min(per, left)
        for r in rs:
            r.compute_round(k)
        left -= k
        for r0, r1 in zip(rs, rs[1:]):   # what exchange() sends, as device copies
            L0, L1, G = r0.layout, r1.layout, r0.layout.ghost
            r1.u[0:L1.a - L1.lo].copy_(r0.u[L1.lo - L0.lo:L1.a - L0.lo])
            r0.u[L0.b + 1 - L0.lo:].copy_(r1.u[L0.b + 1 - L1.lo:L0.hi + 1 - L1.lo])
    for r in rs:
        r.check_status()
    if runners is not None:
        runners.extend(rs)
    out = np.zeros((n + 2,) * kind.dim)
    for i, r in enumerate(rs):
        L = r.layout
        lo = 0 if i == 0 else L.a
        hi = n + 1 if i == world - 1 else L.b
        out[lo:hi + 1] = r.u[lo - L.lo:hi + 1 - L.lo].cpu().numpy()
    return out


@pytest.mark.parametrize("name,n,sweeps,world,per", [
    ("fd7", 40, 5, 2, 1), ("fd7", 37, 4, 3, 2), ("fe27q1", 30, 3, 2, 1),
    ("fe9", 130, 4, 2, 1), ("fe9", 97, 5, 3, 2), ("fd5", 66, 6, 2, 2), ("fe27q1", 64, 3, 3, 1),
    ("fd7", 70, 4, 4, 1), ("fe9", 200, 3, 4, 1)])
@pytest.mark.parametrize("overlap", [False, True])
def test_emulated_slabs_equal_single_domain(name, n, sweeps, world, per, overlap):
    dim = R.STENCIL_TABLE[name][0]
    want = R.init_u(dim, n, 7)
    f = R.init_f(dim, n, 8)
    coracle.sweep(want, name, sweeps, f=f, omega=0.8, form="D")
    got = _emulated(name, n, sweeps, world, per, overlap)
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_single_rank_slab_runner():
    kind = sl.FD7
    r = SlabRunner(3, 24, kind, device="cuda")
    r.init(7, 8, 0.8)
    r.sweep(3)
    want = R.init_u(3, 24, 7)
    coracle.sweep(want, "fd7", 3, f=R.init_f(3, 24, 8), omega=0.8, form="D")
    assert np.array_equal(r.gather().view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("name,n,sweeps,world,per", [
    ("fd7", 40, 5, 2, 1), ("fd7", 38, 4, 3, 2), ("fe27q1", 30, 3, 2, 1), ("fe27q1", 36, 2, 3, 1),
    ("fe9", 130, 4, 3, 1), ("fe9", 98, 5, 2, 2), ("fd5", 66, 6, 4, 2), ("fe27", 24, 2, 2, 1)])
def test_emulated_peer_exchange_equals_single_domain(name, n, sweeps, world, per):
    """The fused exchange: each rank's last pass of a round stores its
    boundary planes straight into the neighbours' ghost planes (here the
    neighbours' buffers on the same device stand in for peer memory)."""
    kind = sl.get_stencil(name)
    dim = kind.dim
    rs = [SlabRunner(dim, n, kind, world=world, rank=r, ghost_sweeps=per, device="cuda", exchange="peer")
          for r in range(world)]
    for i, r in enumerate(rs):
        r.init(7, 8, 0.8)
        r.connect_peers(rs[i - 1] if i > 0 else None, rs[i + 1] if i + 1 < world else None)
    left = sweeps
    while left > 0:
        k = min(per, left)
        for r in rs:            # all ranks' redundant sweeps, then all ranks' fused last passes
            r.round_begin(k)
        for r in rs:
            r.round_end_peer()
        left -= k
    for r in rs:
        r.check_status()
    want = R.init_u(dim, n, 7)
    coracle.sweep(want, name, sweeps, f=R.init_f(dim, n, 8), omega=0.8, form="D")
    out = np.zeros((n + 2,) * dim)
    for i, r in enumerate(rs):
        L = r.layout
        lo = 0 if i == 0 else L.a
        hi = n + 1 if i == world - 1 else L.b
        out[lo:hi + 1] = r.u[lo - L.lo:hi + 1 - L.lo].cpu().numpy()
        # the ghost planes a neighbour stored are exactly its owned planes
        if i > 0:
            Lp = rs[i - 1].layout
            assert np.array_equal(r.u[0:L.a - L.lo].cpu().numpy(),
                                  rs[i - 1].u[L.lo - Lp.lo:L.a - Lp.lo].cpu().numpy())
    assert np.array_equal(out.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("name,n,world", [("fd7", 40, 3), ("fe27q1", 30, 2), ("fe9", 130, 4)])
def test_emulated_slab_residual_equals_single_domain(name, n, world):
    """Each slab's device residual over its owned planes; the max over the
    slabs (what all_reduce(MAX) returns) equals the whole-grid residual."""
    dim = R.STENCIL_TABLE[name][0]
    rs = []
    _emulated(name, n, 3, world, 1, runners=rs)
    want = R.init_u(dim, n, 7)
    f = R.init_f(dim, n, 8)
    coracle.sweep(want, name, 3, f=f, omega=0.8, form="D")
    assert max(r._gpu_residual() for r in rs) == R.residual_max(want, name, f)
    one = SlabRunner(dim, n, sl.get_stencil(name), device="cuda")
    one.init(7, 8, 0.8)
    one.sweep(3)
    assert one.residual_max() == R.residual_max(want, name, f)
