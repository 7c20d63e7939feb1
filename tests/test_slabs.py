"""Slab decomposition (multi-GPU host logic) — world size 2 on gloo (CPU).

Each rank sweeps its slab with the oracle restatement as the compute (the
CUDA kernels need a GPU; `tests/test_gpu_slabs.py` runs them) and exchanges
ghost planes through torch.distributed P2P.  The gathered result must equal
the single-domain oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1810_04033_b200 as sl
from oracle import restate as R
from paper_1810_04033_b200.slabs import SlabLayout, SlabRunner, ghost_depth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_pass(runner, name):
    """The slab pass contract on CPU: one sweep of src, planes [z0, z1) -> dst."""
    def run(src, dst, z0, z1):
        u = src.numpy().copy()
        f = runner.f.numpy() if runner.f is not None else None
        origin = [0, 0, 0]
        origin[runner.dim - 1] = runner.layout.lo
        R.sweep(u, name, 1, f=f, omega=runner.omega or 0.8, form="D" if f is not None else "R",
                origin=tuple(origin))
        dst[z0:z1] = torch.from_numpy(u[z0:z1])
    return run


def oracle_residual(name):
    """max |f - A u| over a runner's owned planes (CPU stand-in for sl_residual_max)."""
    def run(runner):
        dim, offsets, weights, wc, _ = R.STENCIL_TABLE[name]
        L = runner.layout
        u, f = runner.u.numpy(), runner.f.numpy()
        a, b, n = L.a - L.lo, L.b - L.lo, runner.n
        inner = (slice(a, b + 1),) + (slice(1, n + 1),) * (dim - 1)
        acc = wc * u[inner]
        for off, w in zip(offsets, weights):
            if w == 0.0:
                continue
            o = tuple(reversed(off))     # (slow axis, ..., x)
            nb = (slice(a + o[0], b + 1 + o[0]),) + tuple(slice(1 + d, n + 1 + d) for d in o[1:])
            acc += w * u[nb]
        return float(np.abs(f[inner] - acc).max())
    return run


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, world, case, q)
    except Exception as exc:  # surface the failure instead of hanging the parent
        q.put(exc)
        raise
    finally:
        dist.destroy_process_group()


def _run(rank, world, case, q):
    if True:
        name, n, sweeps, per = case
        kind = sl.get_stencil(name)
        r = SlabRunner(kind.dim, n, kind, world=world, rank=rank, ghost_sweeps=per,
                       ghost=2 * per, overlap=n >= 20)   # n >= 20: boundary / interior split
        r._pass = oracle_pass(r, name)
        r._residual = oracle_residual(name)
        r.init(7, 8, 0.8)
        r.sweep(sweeps)
        res = r.residual_max()          # all_reduce(MAX) over the ranks' owned planes
        out = r.gather()
        if rank == 0:
            q.put((out, res))


CASES = [("fd7", 11, 5, 2), ("fe9", 14, 4, 1), ("fe27q1", 10, 3, 1), ("fd5", 16, 6, 3), ("fd7", 20, 4, 4),
         ("fd5", 9, 3, 1), ("fd7", 24, 3, 1), ("fe27q1", 22, 2, 1)]   # the last two split boundary/interior


@pytest.mark.parametrize("case", CASES)
def test_two_rank_slabs_equal_single_domain(case):
    name, n, sweeps, per = case
    dim = R.STENCIL_TABLE[name][0]
    want = R.init_u(dim, n, 7)
    f = R.init_f(dim, n, 8)
    R.sweep(want, name, sweeps, f=f, omega=0.8, form="D")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    if isinstance(got, Exception):
        raise got
    got, res = got
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    assert res == R.residual_max(want, name, f)


def test_layout_covers_grid():
    for n, world in ((17, 2), (512, 8), (30, 4)):
        spans = [SlabLayout(n, world, r, 2) for r in range(world)]
        assert spans[0].a == 1 and spans[-1].b == n
        for x, y in zip(spans, spans[1:]):
            assert y.a == x.b + 1
        assert spans[0].lo == 0 and spans[-1].hi == n + 1


def test_layout_rejects_thin_slabs():
    with pytest.raises(ValueError):
        SlabLayout(8, 4, 1, 2).check()


def test_ghost_depth_grows_with_sweeps():
    for kind in (sl.FD5, sl.FE9, sl.FD7, sl.FE27Q1):
        assert [ghost_depth(kind, s) for s in (1, 2, 3)] == [2, 4, 6]


def test_slab_init_matches_global_init():
    for dim, n in ((2, 11), (3, 7)):
        kind = sl.FD5 if dim == 2 else sl.FD7
        u = R.init_u(dim, n, 3)
        f = R.init_f(dim, n, 4)
        for world in (1, 2, 3):
            for rank in range(world):
                r = SlabRunner(dim, n, kind, world=world, rank=rank, ghost=1)
                r.init(3, 4)
                L = r.layout
                assert np.array_equal(r.u.numpy(), u[L.lo:L.hi + 1])
                assert np.array_equal(r.f.numpy(), f[L.lo:L.hi + 1])
