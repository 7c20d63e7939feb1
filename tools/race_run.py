"""Small-grid runs of every sweep kernel, for compute-sanitizer (racecheck /
synccheck / memcheck).  Each case also checks the result against the oracle,
so a race that changed a value would show as a mismatch too.

    compute-sanitizer --tool racecheck python tools/race_run.py [case ...]

Cases: strip2d (FE9, k2_strip2d), fd5strip (FD5 2 sweeps/pass), block2d (K4, FE9),
resident (K6, FD5 on chip across sweeps),
col3d (FD7, k2_col3d_fd7), q1col (FE27-Q1, k2_q1col), stream3d (FE27 reference
weights), patch (K3), k1 (per-colour), lex (hyperplanes), peer (slab pass with
fused peer stores, emulated on one device).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1810_04033_b200 as sl  # noqa: E402
from oracle import coracle  # noqa: E402
from oracle import restate as R  # noqa: E402
from paper_1810_04033_b200 import _native  # noqa: E402


def grid_case(name, n, sweeps, flags=0):
    kind = sl.get_stencil(name)
    m = sl.make_mesh(kind.dim, n, seed=3)
    sl.init_rhs(m, 4, 0.8)
    sl.run_sweeps(m, kind, sl.CostModel(), sweeps, flags=flags)
    u = R.init_u(kind.dim, n, 3)
    order = "lex" if flags & _native.SL_FLAG_LEX else "colour"
    coracle.sweep(u, name, sweeps, f=R.init_f(kind.dim, n, 4), omega=0.8, form="D", order=order)
    return np.array_equal(m.values.view(np.int64), u.reshape(-1).view(np.int64))


def patch_case():
    u, f = R.init_patches(300, 16, 5)
    want = u.copy()
    coracle.sweep(want, "fd5", 7, f=f, omega=0.8, form="D")
    pb = sl.PatchBatch(u, f)
    pb.sweep(sl.FD5, 7)
    return np.array_equal(pb.values().view(np.int64), want.view(np.int64))


def peer_case():
    from paper_1810_04033_b200.slabs import SlabRunner
    name, n, world = "fd7", 40, 2
    kind = sl.get_stencil(name)
    rs = [SlabRunner(3, n, kind, world=world, rank=r, device="cuda", exchange="peer") for r in range(world)]
    for r in rs:
        r.init(7, 8, 0.8)
    rs[0].connect_peers(upper=rs[1])
    rs[1].connect_peers(lower=rs[0])
    for _ in range(3):
        for r in rs:
            r.round_end_peer()
    out = np.zeros((n + 2,) * 3)
    for i, r in enumerate(rs):
        L = r.layout
        lo = 0 if i == 0 else L.a
        hi = n + 1 if i == world - 1 else L.b
        out[lo:hi + 1] = r.u[lo - L.lo:hi + 1 - L.lo].cpu().numpy()
    want = R.init_u(3, n, 7)
    coracle.sweep(want, name, 3, f=R.init_f(3, n, 8), omega=0.8, form="D")
    return np.array_equal(out.view(np.int64), want.view(np.int64))


CASES = {
    "strip2d": lambda: grid_case("fe9", 300, 2, _native.SL_FLAG_STREAM),   # streaming kernel forced
    "fd5strip": lambda: grid_case("fd5", 300, 2, _native.SL_FLAG_STREAM),
    "block2d": lambda: grid_case("fe9", 150, 3) and grid_case("fe9", 201, 2),
    "resident": lambda: grid_case("fd5", 200, 5) and grid_case("fd5", 1024, 3),   # K6, on-chip across sweeps
    "col3d": lambda: grid_case("fd7", 70, 2),
    "q1col": lambda: grid_case("fe27q1", 70, 2),
    "stream3d": lambda: grid_case("fe27", 40, 2),
    "patch": patch_case,
    "k1": lambda: grid_case("fe27q1", 20, 1, _native.SL_FLAG_PER_COLOUR),
    "lex": lambda: grid_case("fd7", 12, 1, _native.SL_FLAG_LEX),
    "peer": peer_case,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    bad = []
    for nm in names:
        ok = CASES[nm]()
        print(f"{nm}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            bad.append(nm)
    sys.exit(1 if bad else 0)
