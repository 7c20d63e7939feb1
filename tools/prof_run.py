"""Run a few fused passes of one BASELINE config (for ncu captures).

    python tools/prof_run.py --config 2 --sweeps 3 [--per-colour]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1810_04033_b200 as sl  # noqa: E402
from paper_1810_04033_b200 import _native  # noqa: E402
from paper_1810_04033_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--sweeps", type=int, default=3)
ap.add_argument("--per-colour", action="store_true")
a = ap.parse_args()
wl = CONFIGS[a.config]
kind = sl.get_stencil(wl.stencil)
flags = _native.SL_FLAG_PER_COLOUR if a.per_colour else 0
if wl.batch > 1:
    u0, f0 = sl.init_patches(wl.batch, wl.n, wl.seed)
    pb = sl.PatchBatch(torch.from_numpy(u0), torch.from_numpy(f0), wl.omega)
    pb.sweep(kind, a.sweeps, flags=flags)
else:
    m = sl.Mesh(wl.dim, wl.n)
    sl.init(m, wl.seed)
    sl.init_rhs(m, wl.seed + 1, wl.omega)
    sl.run_sweeps(m, kind, sl.CostModel(), a.sweeps, flags=flags)
torch.cuda.synchronize()
print("ok", wl.name, a.sweeps)
