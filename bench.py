#!/usr/bin/env python
"""Benchmark: fp64 grid-point updates/s (GLUP/s) of the colour-scheduled sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the hot path over one batch: the `sweeps` colour-ordered
sweeps of BASELINE.json config C (default 4, the largest single-GPU config:
FE27-Q1 1026^3, 8 colours, 10 sweeps), run through the public API
`run_sweeps` (one C-ABI sl_sweep call).
Protocol mirrors the reference bench (bench.py:206-230): seeded init, W
untimed warm-up steps, K timed steps, CUDA events on the launching stream;
with N>1 (torchrun) the per-rank time is max-reduced.  Rank 0 prints ONE
JSON line.  `--impl reference` times the reference algorithm on the host
cores (the C restatement in oracle/, all threads; the reference itself is
Python and does not exist on the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1810_04033_b200.configs import BYTES_PER_UPDATE, CONFIGS, FP64_OPS_PER_UPDATE  # noqa: E402

METRIC = "fp64 grid-point updates/s (GLUP/s)"
UNIT = "GLUP/s"
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--exchange", choices=("nccl", "peer"), default="nccl",
                    help="slab halo exchange (N > 1): NCCL send/recv after the pass, or stores of the "
                         "boundary planes into the neighbours' ghost planes fused into the pass")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-colour", action="store_true", help="force the unfused K1 path")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Measured fp64 instruction peak of the box (tools/fp64_peak.cu, DADD rate)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as fh:
            return float(json.load(fh)["dadd_ops_per_s"]) / 1e12, "measured (profiles/r02_fp64_peak.json, DADD)"
    except Exception:
        return 148 * 64 * 1.965e9 / 1e12, "nominal 64 fp64 lanes/SM/clk x 148 SMs x 1.965 GHz"


def ncu_traffic(workload_name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(workload_name)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
            return
        # nvidia-smi can take seconds to start on a fresh box: wait for its
        # first sample so the timed region is covered, then keep only what
        # follows
        t0 = time.time()
        while not self.lines and time.time() - t0 < 15 and self.proc.poll() is None:
            time.sleep(0.01)
        self.mark = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        # a short timed region still gets at least two samples (the second
        # may land just after it, at the clocks the load left)
        t0 = time.time()
        while len(self.lines) - getattr(self, "mark", 0) < 2 and time.time() - t0 < 2:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[getattr(self, "mark", 0):]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_config(wl, world, extra=None):
    grid = "x".join([str(wl.side)] * wl.dim)
    if wl.batch > 1:
        grid = f"{wl.batch}x{grid}"
    grid_bytes = wl.grid_elems * 8
    cfg = {"workload": wl.name, "baseline_config_index": wl.index, "stencil": wl.stencil,
           "grid": grid, "sweeps_per_step": wl.sweeps, "update": "form D: u += 0.8*(f - A u)/w_c",
           "seed": wl.seed,
           "l2": ("flushed between steps (256 MiB write)" if 2 * grid_bytes < 2 * L2_BYTES
                  else f"inputs larger than L2 ({2 * grid_bytes / 1e9:.2f} GB u+f)"),
           "parallelism": "single-gpu" if world == 1 else f"replicas x{world}"}
    if extra:
        cfg.update(extra)
    return cfg


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_ram_free():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return 0


def cpu_grid(wl):
    """Interior extent the CPU legs run: the full grid when the host can hold
    u and f (1026^3: 17.3 GB) with margin, else an n=512 sub-grid (said so)."""
    if wl.dim == 3 and wl.n > 512:
        need = 2 * wl.grid_elems * 8
        if host_ram_free() < 1.5 * need + (4 << 30):
            return 512, f"n=512 sub-grid of the {wl.side}^3 config (host RAM < 1.5 x {need / 1e9:.1f} GB)"
    return wl.n, "full grid"


def cpu_inputs(wl, n):
    from oracle import restate as R
    if wl.batch > 1:
        u, f = R.init_patches(min(wl.batch, 4096), wl.n, wl.seed)
        return u, f, u.shape[0] * wl.n ** 2, f"{u.shape[0]} of {wl.batch} patches"
    u = R.init_u(wl.dim, n, wl.seed)
    f = R.init_f(wl.dim, n, wl.seed + 1)
    return u, f, n ** wl.dim, None


def cpu_baseline(wl, budget_s=12.0):
    """Time the C restatement (oracle/, all host threads) on a bounded sample."""
    from oracle import coracle

    threads = coracle.max_threads()
    n, note = cpu_grid(wl)
    u, f, pts, pnote = cpu_inputs(wl, n)
    note = pnote or note
    t0 = time.perf_counter()
    coracle.sweep(u, wl.stencil, 1, f=f, omega=wl.omega, form="D", threads=threads)
    t1 = time.perf_counter()
    sweeps = 1
    per = t1 - t0
    more = max(0, min(wl.sweeps - 1, int(budget_s / max(per, 1e-6)) - 1))
    if more:
        coracle.sweep(u, wl.stencil, more, f=f, omega=wl.omega, form="D", threads=threads)
        sweeps += more
    t2 = time.perf_counter()
    return {"value": pts * sweeps / (t2 - t0) / 1e9, "unit": UNIT, "cores": threads,
            "kind": "port", "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "sample": f"{sweeps} of {wl.sweeps} sweep(s) of {wl.stencil} form D on the {note}, "
                      f"C restatement (oracle/sweep_oracle.c), {threads} pthreads"}


def run_reference(args, wl, rank, world):
    """The reference algorithm on the host cores (C port, all threads)."""
    if rank != 0:
        return
    from oracle import coracle

    threads = coracle.max_threads()
    n, note = cpu_grid(wl)
    u, f, pts, pnote = cpu_inputs(wl, n)
    note = pnote or f"{wl.stencil} {note}"
    # one step = a bounded sample: as many sweeps as fit ~4 s (>= 1)
    t0 = time.perf_counter()
    coracle.sweep(u, wl.stencil, 1, f=f, omega=wl.omega, form="D", threads=threads)
    per = time.perf_counter() - t0
    sweeps = max(1, min(wl.sweeps, int(4.0 / max(per, 1e-6))))
    for _ in range(args.warmup):
        coracle.sweep(u, wl.stencil, sweeps, f=f, omega=wl.omega, form="D", threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        coracle.sweep(u, wl.stencil, sweeps, f=f, omega=wl.omega, form="D", threads=threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = pts * sweeps / (ms / 1e3) / 1e9
    sample = (f"{sweeps} of {wl.sweeps} sweep(s) per step of the {note}, form D, C restatement, "
              f"{threads} pthreads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": workload_config(wl, world, {"parallelism": "host cores"}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def flush_l2(torch, buf):
    buf.add_(1.0)


def run_ours(args, wl, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1810_04033_b200 as sl
    from paper_1810_04033_b200 import _native

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.require_cuda()
    kind = sl.get_stencil(wl.stencil)
    flags = _native.SL_FLAG_PER_COLOUR if args.per_colour else 0

    cost = sl.CostModel()
    total_updates = wl.updates * world          # replicas (config 1): every rank does the grid
    scaling, parallelism = "weak", ("single-gpu" if world == 1 else f"replicas x{world}")
    h2d_bytes = 2 * wl.grid_elems * 8
    d2h_bytes = wl.grid_elems * 8
    if wl.batch > 1:
        # config 5: the patches are split evenly across ranks (no exchange)
        lo, hi = rank * wl.batch // world, (rank + 1) * wl.batch // world
        u0, f0 = sl.init_patches(wl.batch, wl.n, wl.seed)
        pinned_u = torch.from_numpy(np.ascontiguousarray(u0[lo:hi])).pin_memory()
        pinned_f = torch.from_numpy(np.ascontiguousarray(f0[lo:hi])).pin_memory()
        del u0, f0
        pb = sl.PatchBatch(pinned_u, pinned_f, wl.omega, device=dev)
        pinned_out = torch.empty_like(pinned_u).pin_memory()
        if world > 1:
            total_updates, scaling, parallelism = wl.updates, "strong", f"patches split x{world}"
            h2d_bytes = 2 * pinned_u.numel() * 8
            d2h_bytes = pinned_u.numel() * 8

        def step():
            pb.sweep(kind, wl.sweeps, flags=flags)

        def e2e_prep():
            pass

        def e2e_step():
            # the public calls a user makes: host patches in, swept patches out
            pb.upload(pinned_u, pinned_f)
            pb.sweep(kind, wl.sweeps, flags=flags)
            return pb.values(out=pinned_out)

        def e2e_pipeline():
            return (sl.SweepPipeline(kind, pinned_u.shape, wl.sweeps, omega=wl.omega, batch=True,
                                     device=dev, flags=flags), pinned_u, pinned_f, pinned_out)
    elif world > 1 and wl.index in (2, 3, 4):
        # configs 2-4: slabs along the slowest axis, ghost planes exchanged by NCCL P2P
        from paper_1810_04033_b200.slabs import SlabRunner
        # 2D slabs are thin in work per sweep (config 2 at 8 GPUs: ~40 us): exchange every 5
        # sweeps (5-sweep ghost rows, <2% redundant rows) so the host issues ~1.4 launches per
        # sweep; 3D slabs exchange every sweep (a deeper z ghost would cost 6-12% extra planes)
        sr = SlabRunner(wl.dim, wl.n, kind, world=world, rank=rank,
                        ghost_sweeps=5 if wl.dim == 2 and wl.sweeps % 5 == 0 else 1, device=dev,
                        exchange=args.exchange)
        sr.init(wl.seed, wl.seed + 1, wl.omega)
        total_updates, scaling = wl.updates, "strong"
        how = "NCCL P2P" if args.exchange == "nccl" else "peer stores fused into the pass"
        parallelism = f"slabs x{world} (axis {'z' if wl.dim == 3 else 'y'}, ghost {sr.layout.ghost}, {how})"
        u_host = sr.u.cpu().pin_memory()
        f_host = sr.f.cpu().pin_memory()
        out_host = torch.empty_like(sr.owned()).cpu().pin_memory()
        h2d_bytes = 2 * u_host.numel() * 8
        d2h_bytes = out_host.numel() * 8

        def step():
            sr.sweep(wl.sweeps)

        e2e_pipeline = None

        def e2e_prep():
            pass

        def e2e_step():
            sr.u.copy_(u_host, non_blocking=True)
            sr.f.copy_(f_host, non_blocking=True)
            sr.sweep(wl.sweeps)
            out_host.copy_(sr.owned())
            return out_host
    else:
        mesh = sl.Mesh(wl.dim, wl.n, device=dev)
        sl.init(mesh, wl.seed)
        sl.init_rhs(mesh, wl.seed + 1, wl.omega)
        plan = sl.SweepPlan(mesh, kind, cost)
        u0_host = mesh.values.copy()
        f_host = torch.from_numpy(mesh._rhs_host).pin_memory()

        def step():
            sl.run_sweeps(mesh, kind, cost, wl.sweeps, plan=plan, flags=flags)

        def e2e_prep():
            mesh.values[:] = u0_host                # host-side prep (untimed)

        def e2e_step():
            mesh.set_rhs(f_host, wl.omega)          # f re-uploaded inside the step
            step()                                  # uploads u (H2D), sweeps
            return mesh.values                      # D2H of the result

        def e2e_pipeline():
            side = (wl.n + 2,) * wl.dim
            u_pin = torch.from_numpy(u0_host.reshape(side)).pin_memory()
            out = torch.empty(side, dtype=torch.float64).pin_memory()
            return (sl.SweepPipeline(kind, side, wl.sweeps, omega=wl.omega, device=dev, flags=flags),
                    u_pin, f_host.reshape(side), out)

    grid_bytes = wl.grid_elems * 8
    needs_flush = 2 * grid_bytes < 2 * L2_BYTES
    flush_buf = torch.zeros(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev) if needs_flush else None

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()   # before the barrier: its start-up must not delay rank 0's timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.sl_launch_count()
    for i in range(args.steps):
        if flush_buf is not None:
            flush_l2(torch, flush_buf)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    launches = lib.sl_launch_count() - launches0
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop() if clocks else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = total_updates / (ms_per_step / 1e3) / 1e9

    # end to end through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        e2e_times = []
        for i in range(args.steps):
            e2e_prep()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            out = e2e_step()
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t0)
            del out
        te = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        seq_value = total_updates / float(te.item()) / 1e9
        e2e = {"value": seq_value, "unit": UNIT,
               "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
               "mode": "sequential: upload, sweeps, download per step"}
        if world == 1 and e2e_pipeline is not None:
            # the same jobs through SweepPipeline: every step still uploads its
            # u and f from pinned host memory and downloads its result; two
            # steps in flight overlap one step's transfers with another's sweeps
            pipe, pu, pf, out = e2e_pipeline()
            pipe.submit(pu, pf, out)                # warm-up job (untimed)
            pipe.drain()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(args.steps):
                pipe.submit(pu, pf, out)            # each step's result lands in `out`
            pipe.drain()
            tp = (time.perf_counter() - t0) / args.steps
            e2e.update({"value": total_updates / tp / 1e9, "sequential_value": seq_value,
                        "mode": "pipelined (SweepPipeline, 2 steps in flight): per step H2D of u and f, "
                                "sweeps, D2H of u"})
            del pipe, out

    if rank != 0:
        return
    peak, peak_src = peaks()
    achieved = BYTES_PER_UPDATE * total_updates / world / (ms_per_step / 1e3) / 1e9   # per GPU
    per_step_launches = launches / args.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[0,1) u0, U[-1,1) f)",
            "config": workload_config(wl, world, {"path": "k1-per-colour" if args.per_colour else "auto",
                                                  "parallelism": parallelism}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(wl.name),
                         "peak_source": peak_src,
                         "algorithmic_bytes": f"{BYTES_PER_UPDATE} B per grid-point update "
                                              "(u read + f read + u write, once per sweep)",
                         "launches_per_step": per_step_launches},
            "gpu_launches": int(launches),
            "clocks": clock_info,
            "e2e": e2e}
    if wl.batch == 1 and wl.dim == 2 and per_step_launches <= 2 and wl.sweeps > 2 and not args.per_colour:
        # config 1: one cooperative launch runs every sweep with the grid resident on chip (K6);
        # HBM sees u and f once per call, so the 24 B/update figure is an accounting kept for
        # comparison with the streaming kernels, not a claim about DRAM traffic (see `traffic`)
        line["roofline"]["note"] = ("grid resident on chip across all sweeps (K6, one launch per step): "
                                    "DRAM traffic per launch is `traffic`, far below the algorithmic bytes; "
                                    "the kernel is bound by the per-round tile exchange through L2 and by "
                                    "shuffle/smem latency, not by HBM")
    if wl.batch > 1 and not args.per_colour:
        # config 5 keeps every patch on chip for all sweeps: the fp64 pipe bounds it, not HBM
        # (K3 Form D FD5: DMUL w_c u, 4 DSUB, DSUB f - Au, DMUL 1/w_c, DMUL omega, DADD = 9
        # fp64 instructions = 9 flops per update, no FMA)
        fpk, fsrc = fp64_peak()
        fach = FP64_OPS_PER_UPDATE[wl.index] * total_updates / world / (ms_per_step / 1e3) / 1e12
        hbm = line["roofline"]
        line["roofline"] = {"bound": "fp64", "achieved": fach, "peak": fpk, "unit": "TFLOP/s",
                            "frac": fach / fpk, "traffic": hbm["traffic"], "peak_source": fsrc,
                            "algorithmic_ops": f"{FP64_OPS_PER_UPDATE[wl.index]} fp64 instructions per update",
                            "hbm_24B_accounting": {"achieved": hbm["achieved"], "peak": hbm["peak"],
                                                   "unit": "GB/s", "frac": hbm["frac"]},
                            "launches_per_step": hbm["launches_per_step"]}
    return line


def main():
    args = parse_args()
    rank, world, local = dist_env()
    wl = CONFIGS[args.config]
    if world > 1:
        # NCCL init lines (rank/device/transport) for the multi-GPU record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    try:
        if args.impl == "reference":
            run_reference(args, wl, rank, world)
        else:
            line = run_ours(args, wl, rank, world, local)
            if line is not None:
                if world == 1 and not args.no_cpu_baseline:
                    # after run_ours returned: its host/device buffers are freed first
                    import gc
                    import torch
                    gc.collect()
                    torch.cuda.empty_cache()
                    line["cpu_baseline"] = cpu_baseline(wl)
                print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
