#!/usr/bin/env python
"""bench.py -- composite-cell Sinkhorn solves/s and time-to-solution of the
B200 entropic domain decomposition path (arXiv 2001.10986) on BASELINE.json's
headline workload (config 5: 2048^2, s = 8, ladder to eps = 0.5 h^2).

A step = one full coarse-to-fine / eps-scaling solve (all SURVEY 8(a) rows:
refinements, 72 sweeps of K1 -> K2 -> K3) of one image pair resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

N > 1 (torchrun): ONE problem striped over the ranks: each
rank solves the composite cells of its stripe of basic-cell rows; before and
after every B-sweep one boundary row moves between neighbouring ranks by NCCL
send/recv (torch.distributed over NVLink), plus all-reduces of the statistics
(paper_2001_10986_b200/striped.py).  "scaling": "strong" (fixed total work);
value = whole-problem cell solves / max-over-ranks device time.  Rank 0
prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "composite-cell Sinkhorn solves/sec"
UNIT = "cell_solves/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged transport, lets N ranks share one GPU (protocol test)")
    return ap.parse_args()


def _workload(cfg: int):
    from ddinputs import CONFIGS
    p = CONFIGS[cfg]
    n, s = p["n"], p["s"]
    return dict(
        workload=f"cfg{cfg}: {n}x{n} W2, Gaussian mixtures" + (" + 10% noise" if p["noise"] else "")
        + f", s={s}, ladder {p.get('coarsest', 8)}^2->{n}^2, final eps={p['kappa_final']}h^2, Err=1e-6, tau=1e-15",
        n=n, s=s, kappa_final=p["kappa_final"], coarsest=p.get("coarsest", 8),
        eps_start=p.get("eps_start", 0.0), err_tol=1e-6, trunc_tau=1e-15,
        schedule_sweeps=None)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        loaded = [v for v in sm if mx and v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- oracle leg --
def cpu_baseline(cfg: int, n_sample: int = 32):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    workload: the cfg-5 generator recipe (s = 8 -> 16 x 16-px composite cells,
    10% noise, same Err/tau/final kappa) at n_sample^2 with the full ladder."""
    from ddinputs import gaussian_mixture_image, CONFIGS
    from oracle import Oracle
    from oracle.oracle import SCHED_LADDER
    p = CONFIGS[cfg]
    s = min(p["s"], n_sample // 4)
    mu = gaussian_mixture_image(n_sample, 1, cfg)
    nu = gaussian_mixture_image(n_sample, 2, cfg)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    o = Oracle(mu, nu, p["kappa_final"] / n_sample**2, s, err_tol=1e-6, trunc_tau=1e-15,
               schedule=SCHED_LADDER, coarsest_side=8, n_threads=cores)
    cells = 0
    from oracle.oracle import build_schedule
    sched = build_schedule(n_sample, 8, p["kappa_final"])
    # run stage by stage to count cell solves
    for side, kappa, sweeps in sched:
        while o.state_info()["side"] < side:
            o.refine()
        o.set_eps(kappa / side**2)
        for _ in range(sweeps):
            o.iterate(1)
            cells += o.stats()["cells"]
    dt = time.perf_counter() - t0
    return {"value": cells / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"cfg{cfg} recipe at {n_sample}x{n_sample} (s={s}), full ladder 8^2->{n_sample}^2, "
                      f"{cells} cell solves in {dt:.1f} s, dense fp64 oracle, OpenMP {cores} threads",
            "seconds": dt, "cells": cells}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = _workload(args.config)
    samples = []
    for _ in range(args.warmup if args.warmup < 1 else 0):
        pass
    for _ in range(max(1, args.steps)):
        samples.append(cpu_baseline(args.config))
    v = float(np.median([s["value"] for s in samples]))
    secs = float(np.median([s["seconds"] for s in samples]))
    cb = dict(samples[0])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {**{k: w[k] for k in ("workload", "n", "s")},
                                            "note": "oracle timed on a bounded sample of the workload"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our leg --
def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())   # gloo protocol test: ranks may share a GPU
    if world > 1:
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    staging = "cpu" if args.dist_backend == "gloo" else None

    from ddinputs import config_images
    from paper_2001_10986_b200 import DD, SCHED_LADDER, measure_mufu_peak
    w = _workload(args.config)
    n, s = w["n"], w["s"]
    eps = w["kappa_final"] / n**2
    mu_h, nu_h = config_images(args.config, pair=0)      # one problem, striped over the ranks
    mu_d = torch.from_numpy(mu_h).to(dev)
    nu_d = torch.from_numpy(nu_h).to(dev)
    stream = torch.cuda.Stream(dev)          # a real stream handle (the default stream is 0)
    torch.cuda.set_stream(stream)
    kw = dict(err_tol=w["err_tol"], trunc_tau=w["trunc_tau"], schedule=SCHED_LADDER,
              eps_start=w["eps_start"], coarsest_side=w["coarsest"], device=local)
    g = DD(mu_d, nu_d, eps, s, device_input=True, stream=stream.cuda_stream, **kw)
    run = None
    if world > 1:
        from paper_2001_10986_b200.striped import StripedRun, TorchTransport
        run = StripedRun([(rank, g)], world, TorchTransport(dist, rank, world, dev, staging=staging), device=dev)

    def solve(ctx, striped):
        """One full coarse-to-fine solve (the bench step)."""
        if striped is None:
            ctx.run_schedule()
        else:
            striped.run_schedule(n, w["coarsest"], w["kappa_final"], w["eps_start"])

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        g.reset()
        solve(g, run)
        g.synchronize()
    # ---- timed region: K steps, per-step CUDA events on the library's stream
    g.reset_totals()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    step_ms = []
    cells_step = []
    for _ in range(args.steps):
        flush.fill_(1.0)                       # L2 flush between timed steps (256 MB > 126 MB L2)
        g.reset()                              # state back to the product coupling (untimed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        c0 = run.cells_solved if run else 0
        e0.record(stream)
        solve(g, run)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        cells_step.append(run.cells_solved - c0 if run else None)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    tot = g.totals()
    my_ms = float(np.sum(step_ms))
    if run is not None:
        all_cells = float(np.sum(cells_step))          # whole-problem solves (replicated layers once)
        wall_ms = float(run.tr.allreduce_max(torch.tensor([my_ms], dtype=torch.float64, device=dev))[0])
    else:
        wall_ms, all_cells = my_ms, float(tot["cells"])
    cells_per_step = all_cells / args.steps
    value = all_cells / (wall_ms * 1e-3)
    # ---- quality of the final state (outside the timed region)
    if run is not None:
        cost, ent = run.primal_cost()
        l1x, l1y = run.marginal_error()
    else:
        cost, ent = g.primal_cost()
        l1x, l1y = g.marginal_error()
    last = g.stats()

    # ---- roofline of the dominant kernel (K1): algorithmic MUFU ops / K1 time
    peak = measure_mufu_peak(local)
    nominal = 148 * 16 * (clk["sm_max_mhz"] or 1965.0) * 1e6
    k1_ms = tot["solve_ms"]
    achieved = tot["mufu_ops"] / (k1_ms * 1e-3)
    prof_traffic, traffic_unit = None, None
    try:   # committed ncu capture (dram__bytes_read + write of K1 in one finest-layer sweep)
        pj = json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))
        prof_traffic, traffic_unit = pj.get("bytes_per_launch"), pj.get("unit")
    except Exception:
        pass
    roofline = {"bound": "alu", "pipe": "MUFU/XU ex2+log (SFU)", "achieved": achieved / 1e12,
                "peak": peak / 1e12, "unit": "Top/s", "frac": achieved / peak,
                "peak_source": "measured ex2.approx microbenchmark on this B200 (dd_measure_mufu_peak)",
                "peak_nominal": nominal / 1e12, "traffic": prof_traffic, "traffic_unit": traffic_unit,
                "kernel": "k1_cell_solve", "kernel_share_of_step": k1_ms / my_ms,
                "mufu_ops_per_step": tot["mufu_ops"] / args.steps}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        mu_p = torch.from_numpy(mu_h).pin_memory()
        nu_p = torch.from_numpy(nu_h).pin_memory()
        e2e_ms = []
        for k in range(2):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            # same stream as torch's current stream: NCCL completion (TorchTransport)
            # is ordered against it, so the library never reads an unfinished receive
            ge = DD(mu_p.numpy(), nu_p.numpy(), eps, s, stream=stream.cuda_stream, **kw)
            if run is not None:
                re = StripedRun([(rank, ge)], world, TorchTransport(dist, rank, world, dev, staging=staging), device=dev)
                solve(ge, re)
                c_e, _ = re.primal_cost()
                lx_e, ly_e = re.marginal_error()
            else:
                solve(ge, None)
                c_e, _ = ge.primal_cost()
                lx_e, ly_e = ge.marginal_error()
            dt = time.perf_counter() - t0
            if world > 1:
                dt = float(run.tr.allreduce_max(torch.tensor([dt], dtype=torch.float64, device=dev))[0])
            ge.close()
            if k > 0:
                e2e_ms.append(dt * 1e3)
        e2e_ms_med = float(np.median(e2e_ms))
        e2e = {"value": cells_per_step / (e2e_ms_med * 1e-3),
               "unit": UNIT, "h2d_bytes_per_step": int(mu_h.nbytes + nu_h.nbytes),
               "d2h_bytes_per_step": 4 * 8, "ms_per_step": e2e_ms_med,
               "path": "dd_init(host) + dd_run_schedule + dd_primal_cost + dd_marginal_error + dd_free"}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": wall_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "dtype_detail": "f32 ex2/log arithmetic with exact hi/lo argument assembly; f64 staging, "
                            "balance and marginal sums",
            "data": "synthetic",
            "config": {**{k: w[k] for k in ("workload", "n", "s", "kappa_final", "err_tol", "trunc_tau")},
                       "global_batch": 1,
                       "parallelism": f"stripes{world} (NCCL send/recv of boundary rows)" if world > 1 else "single",
                       "l2": "flushed between steps (256 MB write); nu_i pool > L2"},
            "time_to_solution_ms": wall_ms / args.steps,
            "cells_per_step": cells_per_step,
            "iters_per_cell": tot["iters_sum"] / max(1, tot["cells"]),
            "final": {"transport_cost": cost, "entropic": ent, "l1_x": l1x, "l1_y": l1y,
                      "entries_per_px": last["entries"] / n**2, "max_box": tot["max_box"],
                      "big_cells": tot["big_cells"], "failed": tot["failed"]},
            "roofline": roofline, "clocks": clk, "gpu_launches": int(tot["launches"]),
            "e2e": e2e, "cpu_baseline": cb}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
