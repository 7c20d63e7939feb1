"""Per-GPU compute rate of the slab passes at the slab geometry of N ranks,
measured on ONE GPU (no transfer): the middle rank's slab of BASELINE configs
2-4 for N = 1, 2, 4, 8, timed with CUDA events over whole rounds
(`SlabRunner.compute_round(k, exchange=False)`), in two modes:

  plain  the pass a rank runs under the NCCL exchange (exchange itself not timed)
  peer   the same round with the boundary-plane stores fused into the pass
         (`exchange="peer"`); the neighbours' ghost planes are stood in for by
         two more slabs on the same device (HBM stores instead of NVLink stores)

    python tools/slab_geometry.py [--configs 2 3 4] [--ranks 1 2 4 8] > profiles/r02_slab_geometry.json

GLUP/s counts the rank's OWNED updates only (the redundant ghost sweeps of a
deep-ghost round are overhead), so rate(N) / rate(1) is the compute side of
strong-scaling efficiency.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1810_04033_b200 as sl  # noqa: E402
from paper_1810_04033_b200.configs import CONFIGS  # noqa: E402
from paper_1810_04033_b200.slabs import SlabRunner  # noqa: E402


def measure(wl, world, mode, rounds, warm):
    kind = sl.get_stencil(wl.stencil)
    gs = 5 if wl.dim == 2 and wl.sweeps % 5 == 0 else 1      # as bench.py --gpus N
    rank = world // 2
    dev = torch.device("cuda", 0)
    mk = lambda r: SlabRunner(wl.dim, wl.n, kind, world=world, rank=r, ghost_sweeps=gs, device=dev,  # noqa: E731
                              exchange="peer" if mode == "peer" else "nccl")
    sr = mk(rank).init(wl.seed, wl.seed + 1, wl.omega)
    if mode == "peer" and world > 1:
        lower = mk(rank - 1) if rank > 0 else None
        upper = mk(rank + 1) if rank < world - 1 else None
        sr.connect_peers(lower=lower, upper=upper)
    sr._u2[0].copy_(sr.u[0])
    sr._u2[-1].copy_(sr.u[-1])

    def one_round():
        if mode == "peer" and world > 1:
            sr.round_begin(gs)
            sr.round_end_peer()
        else:
            sr.compute_round(gs, exchange=False)

    for _ in range(warm):
        one_round()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(rounds):
        one_round()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / rounds
    owned = sr.layout.b - sr.layout.a + 1
    updates = owned * wl.n ** (wl.dim - 1) * gs
    return {"ms_per_round": ms, "sweeps_per_round": gs, "owned_planes": owned, "ghost": sr.layout.ghost,
            "glups_per_gpu": updates / (ms / 1e3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3, 4])
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    out = {"what": "per-GPU compute at the slab geometry of N ranks, one B200, no transfer",
           "gpu": torch.cuda.get_device_name(0), "results": []}
    for c in a.configs:
        wl = CONFIGS[c]
        base = {}
        for n in a.ranks:
            for mode in ("plain", "peer"):
                if mode == "peer" and n == 1:
                    continue
                r = measure(wl, n, mode, a.rounds, a.warmup)
                r.update({"config": c, "workload": wl.name, "ranks": n, "mode": mode})
                if n == 1:
                    base[c] = r["glups_per_gpu"]
                if c in base:
                    r["vs_1_rank"] = r["glups_per_gpu"] / base[c]
                out["results"].append(r)
                print(f"c{c} N={n} {mode}: {r['glups_per_gpu']:.1f} GLUP/s per GPU "
                      f"({r.get('vs_1_rank', 1.0):.2f} of N=1), {r['ms_per_round']:.3f} ms/round",
                      file=sys.stderr, flush=True)
                torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
