import sys, numpy as np
sys.path.insert(0, '.')
import paper_1810_04033_b200 as sl
from oracle import coracle, restate as R
from paper_1810_04033_b200 import _native
for mode in ("fused", "stream"):
    for n in (2, 3, 7, 16, 33, 64, 130, 600):
        for sweeps in (1, 2, 5, 9, 11):
            u = R.init_u(2, n, n); f = R.init_f(2, n, n + 1)
            coracle.sweep(u, "fd5", sweeps, f=f, omega=0.8, form="D")
            m = sl.make_mesh(2, n, seed=n); sl.init_rhs(m, n + 1, 0.8)
            try:
                sl.run_sweeps(m, sl.FD5, sl.CostModel(), sweeps, flags=_native.SL_FLAG_STREAM if mode == "stream" else 0)
                got = m.values.reshape(u.shape)
                bad = np.argwhere(got.view(np.int64) != u.view(np.int64))
                print(mode, n, sweeps, "ok" if len(bad) == 0 else f"MISMATCH {len(bad)} first {bad[:3].tolist()}")
            except Exception as e:
                print(mode, n, sweeps, "EXC", type(e).__name__, e)
