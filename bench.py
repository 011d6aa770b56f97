#!/usr/bin/env python
"""Benchmark of the HJ reachability hot path (BASELINE.json metric).

Workload (config.workload): BASELINE config 2 — the 4D near-hover lateral
subsystem on a 51^4 fp64 grid (6.77e6 cells), first-order Godunov / forward
Euler (the reference scheme), wind 0.5 on the position row, tol 1e-4.
A "step" is one chunk of ``--iters`` VI sweeps (default 1000) of that solve,
started from V = c, run by the device-resident loop; metric = grid
cell-updates per second = steps * iters * cells / time.

  value    device-resident inputs (already in HBM), CUDA-event time on the
           library stream, max over ranks
  e2e      the same through the reference-facing C ABI (hjb_solve) with HOST
           buffers: H2D of init + c and D2H of V* inside the timed region
  roofline the sweep kernel: 24 algorithmic bytes per cell-update (read V,
           read c, write V) / average sweep time, against the
           measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the reference's own solve (oracle/_ref, compiled from the
           unmodified reference sources) on the host cores, bounded sample

``--impl reference`` times the reference CPU implementation alone (same
metric/config), rank 0 only.  Multi-GPU (N>1, torchrun): every rank solves its
own replica of the workload (weak scaling; the slab-partitioned single solve
is not in this bench yet), barrier + max over ranks.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "HJ grid cell-updates/sec (first-order Godunov VI sweep, fp64)"
UNIT = "cell-updates/s"
BYTES_PER_CELL = 24  # read V + read c + write V, fp64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hjb", choices=["hjb", "reference"])
    ap.add_argument("--n", type=int, default=51, help="grid points per axis (config 2: 51)")
    ap.add_argument("--iters", type=int, default=1000, help="VI sweeps per step")
    ap.add_argument("--no-converge", dest="converge", action="store_false",
                    help="skip the full solve to tol 1e-4 (time_to_converged, ~50 s on a B200)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config3", dest="config3", action="store_false",
                    help="skip the extra config-3 (ENO3 + TVD-RK3, 101^4) step timing")
    ap.add_argument("--sharded", action="store_true",
                    help="slab-partitioned solve of the --n grid over the ranks (axis 0, NCCL "
                         "halo exchange + residual all-reduce; strong scaling), e.g. "
                         "--n 101 --order 3 --rk 3 for config 3")
    ap.add_argument("--order", type=int, default=1, help="--sharded: ENO order")
    ap.add_argument("--rk", type=int, default=1, help="--sharded: TVD-RK order")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload(n):
    from paper_2101_05916_b200 import configs
    w = configs.config2(n)
    return w


def _per_iter_cost(impl, c, w, cfg):
    """Per-sweep cost of a CPU solve: (t(3 sweeps) - t(1 sweep)) / 2, setup excluded."""
    from paper_2101_05916_b200 import hjsafe as hj
    t = []
    for k in (1, 3):
        cf = hj.SolveConfig(**cfg.__dict__)
        cf.max_iters = k
        t0 = time.perf_counter()
        impl.solve(c, c, w.model, w.dbounds(), cf)
        t.append(time.perf_counter() - t0)
    per = max((t[1] - t[0]) / 2, 1e-6)
    return per, max(t[0] - per, 0.0)


def cpu_reference_rate(n, seconds, threads=0):
    """Reference solve (oracle/_ref) on the host: returns (rate, iters, sample, kind)."""
    from oracle import oracle as o
    from paper_2101_05916_b200 import hjsafe as hj
    sys.path.insert(0, str(ROOT / "tests"))
    from cases import band_np, fmax_np
    w = workload(n)
    c = hj.ScalarField(w.grid, w.constraint(band_np, fmax_np))
    if o.reference_available():
        impl, kind = o.Reference(), "reference"
    else:
        impl, kind = o.Restatement(), "port"
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.threads = threads
    per_iter, _ = _per_iter_cost(impl, c, w, cfg)
    iters = int(max(1, min(500, seconds / max(per_iter, 1e-6))))
    cfg.max_iters = iters
    t0 = time.perf_counter()
    r = impl.solve(c, c, w.model, w.dbounds(), cfg)
    el = time.perf_counter() - t0
    rate = w.grid.size() * r.iterations / el
    sample = (f"{r.iterations} VI sweeps of the {n}^4 config-2 solve from V=c "
              f"({w.grid.size()} cells), wall {el:.2f} s")
    return rate, r.iterations, sample, kind


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as o
    from paper_2101_05916_b200 import hjsafe as hj
    sys.path.insert(0, str(ROOT / "tests"))
    from cases import band_np, fmax_np
    w = workload(args.n)
    c = hj.ScalarField(w.grid, w.constraint(band_np, fmax_np))
    if o.reference_available():
        impl, kind = o.Reference(), "reference"
    else:
        impl, kind = o.Restatement(), "port"
    cores = os.cpu_count() or 1
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.threads = 0
    per_iter, _ = _per_iter_cost(impl, c, w, cfg)
    per_step = int(max(1, min(args.iters, 2.0 / max(per_iter, 1e-6))))
    cfg.max_iters = per_step
    for _ in range(args.warmup):
        impl.solve(c, c, w.model, w.dbounds(), cfg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        impl.solve(c, c, w.model, w.dbounds(), cfg)
    el = time.perf_counter() - t0
    cells = w.grid.size()
    rate = args.steps * per_step * cells / el
    sample = f"{per_step} sweeps of {args.n}^4 per step, {cores} host threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic constraint, constant wind bounds)",
        "config": {"workload": f"BASELINE config 2: 4D planar near-hover, {args.n}^4 grid, "
                               "first-order Godunov + Euler, CFL 0.8, tol 1e-4",
                   "cells": cells, "iters_per_step": per_step},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config3_step(ctx, dev, steps=6):
    """BASELINE config 3's scheme on its grid: ENO3 + TVD-RK3 Godunov steps of
    the 101^4 config-2 model (k_eno3g), device time per step from V=c."""
    import torch
    from paper_2101_05916_b200 import hjsafe as hj
    w = configs_mod().config3(101)
    cells = w.grid.size()
    c = torch.empty(cells, dtype=torch.float64, device=dev)
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(w.grid, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.spatial_order, cfg.time_order, cfg.max_iters = 3, 3, 2
    hj.solve_dev(w.grid, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(), cfg,
                 ctx=ctx)
    cfg.max_iters = steps
    r = hj.solve_dev(w.grid, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(), cfg,
                     ctx=ctx)
    per = r.wall_seconds / r.iterations
    peak, _ = measured_peak()
    gbs = 88 * cells / per / 1e9
    del c, out
    torch.cuda.empty_cache()
    return {"workload": "BASELINE config 3 scheme: ENO3 + TVD-RK3 Godunov, 101^4 config-2 model, "
                        "one GPU, from V=c", "steps": r.iterations, "ms_per_step": per * 1e3,
            "cell_steps_per_s": cells / per, "bytes_per_cell_step": 88,
            "achieved_gbs": gbs, "frac_of_hbm": gbs / peak, "bound": "fp64 issue (see DESIGN §5)",
            "kernel": "k_eno3g x 3 stages"}


def configs_mod():
    from paper_2101_05916_b200 import configs
    return configs


def run_hjb(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2101_05916_b200 import hjsafe as hj

    w = workload(args.n)
    grid, model, db = w.grid, w.model, w.dbounds()
    cells = grid.size()
    ctx = hj.Context(local)
    # constraint built on the device (signed_distance_band kernel)
    dev = torch.device("cuda", local)
    c_t = torch.empty(cells, dtype=torch.float64, device=dev)
    out_t = torch.empty(cells, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    for (dim, lo, hi, sign) in w.bands:
        assert sign > 0 and len(w.bands) == 1
        hj.signed_distance_band_dev(grid, dim, lo, hi, c_t.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters = args.iters
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def step():
        return hj.solve_dev(grid, model, db, c_t.data_ptr(), c_t.data_ptr(), out_t.data_ptr(), cfg,
                            ctx=ctx)

    for _ in range(args.warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sweep_s = []
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
            assert r.iterations == args.iters, r.iterations
            sweep_s.append(r.wall_seconds / r.iterations)
        e1.record(stream)
        torch.cuda.synchronize()
    gpu_launches = ctx.launches - launches0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * args.steps * args.iters * cells / (ms * 1e-3)

    # e2e: reference-facing ABI with host buffers (H2D init + c, D2H V*),
    # page-locked host arrays as a serving caller would keep them
    c_pin = torch.empty(cells, dtype=torch.float64, pin_memory=True)
    c_pin.copy_(c_t)
    i_pin = torch.empty(cells, dtype=torch.float64, pin_memory=True)
    i_pin.copy_(c_t)
    o_pin = torch.empty(cells, dtype=torch.float64, pin_memory=True)
    c_host = hj.ScalarField(grid, c_pin.numpy(), check=False)
    init_host = hj.ScalarField(grid, i_pin.numpy(), check=False)
    out_host = o_pin.numpy()
    for _ in range(max(1, args.warmup // 2)):
        hj.solve(init_host, c_host, model, db, cfg, ctx=ctx, history_capacity=0, out=out_host)
    e2e_steps = max(2, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = hj.solve(init_host, c_host, model, db, cfg, ctx=ctx, history_capacity=0,
                       out=out_host)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_rate = world * args.iters * cells / e2e_s

    peak, peak_src = measured_peak()
    traffic = None
    tp = ROOT / "profiles" / "round1_traffic.json"
    if tp.exists():
        t = json.loads(tp.read_text()).get(str(args.n))
        if t:
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
    sweep = statistics.mean(sweep_s)
    achieved = BYTES_PER_CELL * cells / sweep / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic signed-distance constraint, constant wind bounds; no dataset)",
        "config": {"workload": f"BASELINE config 2: 4D planar near-hover (wind on x row, g=9.81, "
                               f"u in [-pi/9,pi/9]), {args.n}^4 grid, first-order Godunov + Euler, "
                               "CFL 0.8, tol 1e-4, solve chunk of iters sweeps from V=c",
                   "cells": cells, "iters_per_step": args.iters,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": f"working set {3 * cells * 8 / 1e6:.0f} MB (V front/back + c) vs 126 MB L2; "
                         "no explicit flush"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": "profiles/round1_traffic.json (ncu --set full, one launch)",
                     "kernel": "k_fast4d sweep (TMA plane ring; avg device time per sweep incl. launch gaps)",
                     "bytes_per_cell": BYTES_PER_CELL, "peak_source": peak_src,
                     "sweep_us": sweep * 1e6},
        "e2e": {"value": e2e_rate, "unit": UNIT, "h2d_bytes_per_step": 2 * cells * 8,
                "d2h_bytes_per_step": cells * 8, "ms_per_step": e2e_s * 1e3,
                "path": "hjsafe.solve -> hjb_solve (C ABI), page-locked host init/c/out"},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "final_residual": res.final_residual,
    }
    if args.converge:
        cfgc = hj.SolveConfig(**w.cfg.__dict__)
        cfgc.max_iters = 5_000_000
        rc = hj.solve_dev(grid, model, db, c_t.data_ptr(), c_t.data_ptr(), out_t.data_ptr(), cfgc,
                          ctx=ctx)
        safe = int((out_t <= 0).sum().item())
        line["time_to_converged"] = {"seconds": rc.wall_seconds, "iterations": rc.iterations,
                                     "converged": rc.converged, "tolerance": cfgc.tolerance,
                                     "safe_cells": safe, "final_residual": rc.final_residual,
                                     "note": "device time of the whole solve from V=c"}
    if args.config3:
        line["config3"] = config3_step(ctx, dev)
    if rank == 0 and not args.no_cpu_baseline:
        try:
            rate, iters, sample, kind = cpu_reference_rate(args.n, args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": kind, "sample": sample}
            if "time_to_converged" in line:
                # bitwise parity => the reference takes the same number of sweeps
                line["time_to_converged"]["cpu_seconds_extrapolated"] = (
                    line["time_to_converged"]["iterations"] * cells / rate)
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args):
    """Slab-partitioned solve: every rank owns a balanced range
    of axis-0 planes; halos and the residual travel over NCCL inside the
    device loop.  Device time per rank from the library, max over ranks."""
    import torch
    rank, world, local = dist_env()
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2101_05916_b200 import hjsafe as hj
    from paper_2101_05916_b200 import sharded
    w = workload(args.n)
    g, cells = w.grid, w.grid.size()
    dev = torch.device("cuda", local)
    ctx = hj.Context(local)
    c = torch.empty(cells, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    b, e = sharded.slab_partition(args.n, world, rank)
    s0 = cells // args.n
    out = torch.empty((e - b) * s0, dtype=torch.float64, device=dev)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters, cfg.spatial_order, cfg.time_order = args.iters, args.order, args.rk
    comm = sharded.Comm(ctx, rank, world, dev)
    ptr = c.data_ptr() + b * s0 * 8
    try:
        for _ in range(args.warmup):
            sharded.solve_sharded_dev(comm, g, w.model, w.dbounds(), ptr, ptr, out.data_ptr(), cfg,
                                      ctx)
        secs = 0.0
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                r = sharded.solve_sharded_dev(comm, g, w.model, w.dbounds(), ptr, ptr,
                                              out.data_ptr(), cfg, ctx)
                secs += r.wall_seconds
    finally:
        comm.close()
    t = torch.tensor([secs], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    secs = float(t.item())
    per_step = secs / args.steps
    value = cells * r.iterations / per_step
    bpc = 24 + 32 * (args.rk - 1)
    peak, peak_src = measured_peak()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config-2 model on {args.n}^4, ENO{args.order} + TVD-RK{args.rk}, "
                                   f"{r.iterations} steps per bench step",
                       "parallelism": f"slab x{world} (axis 0, NCCL halos + residual all-reduce)",
                       "slab_planes": [e - b]},
            "roofline": {"bound": "hbm", "achieved": bpc * cells * r.iterations / per_step / 1e9 / world,
                         "peak": peak, "unit": "GB/s per GPU", "peak_source": peak_src,
                         "bytes_per_cell_step": bpc},
            "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.sharded:
        run_sharded(args)
    else:
        run_hjb(args)


if __name__ == "__main__":
    main()
