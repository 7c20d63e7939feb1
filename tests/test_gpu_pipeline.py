"""SweepPipeline: overlapped upload / sweep / download jobs give the oracle's
result for every job, bit for bit (grids and patch batches)."""

import numpy as np
import pytest
import torch

import paper_1810_04033_b200 as sl
from oracle import coracle
from oracle import restate as R

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a).reshape(-1).view(np.int64), np.asarray(b).reshape(-1).view(np.int64))


@pytest.mark.parametrize("name,n,sweeps", [("fe9", 130, 3), ("fe27q1", 30, 2), ("fd7", 34, 3), ("fd5", 64, 5)])
def test_pipeline_jobs_match_oracle(name, n, sweeps):
    kind = sl.get_stencil(name)
    dim = kind.dim
    jobs = []
    for seed in (3, 5, 7, 9, 11):
        u = R.init_u(dim, n, seed)
        f = R.init_f(dim, n, seed + 1)
        jobs.append((torch.from_numpy(u).pin_memory(), torch.from_numpy(f).pin_memory()))
    pipe = sl.SweepPipeline(kind, jobs[0][0].shape, sweeps, omega=0.8, depth=2)
    outs = [torch.empty_like(jobs[0][0]).pin_memory() for _ in jobs]
    for (u, f), o in zip(jobs, outs):
        pipe.submit(u, f, o)
    pipe.drain()
    for (u, f), o in zip(jobs, outs):
        want = u.numpy().copy()
        coracle.sweep(want, name, sweeps, f=f.numpy(), omega=0.8, form="D")
        assert _bits_equal(o.numpy(), want)


def test_pipeline_patch_batches():
    u0, f0 = sl.init_patches(64, 16, 4)
    u = torch.from_numpy(np.ascontiguousarray(u0)).pin_memory()
    f = torch.from_numpy(np.ascontiguousarray(f0)).pin_memory()
    pipe = sl.SweepPipeline(sl.FD5, u.shape, 20, omega=0.8, batch=True, depth=2)
    outs = [torch.empty_like(u).pin_memory() for _ in range(3)]
    for o in outs:
        pipe.submit(u, f, o)
    pipe.drain()
    pb = sl.PatchBatch(u.clone(), f.clone(), 0.8, device="cuda")
    pb.sweep(sl.FD5, 20)
    want = pb.values()
    for o in outs:
        assert _bits_equal(o.numpy(), want)


def test_pipeline_rejects_mismatched_rhs():
    with pytest.raises(ValueError):
        pipe = sl.SweepPipeline(sl.FD5, (10, 10), 1, omega=0.8)
        pipe.submit(torch.zeros(10, 10).double().pin_memory(), None, None)
