"""Run the config-5 ladder (or --cfg k) and print per-sweep statistics; the
sweeps selected by --profile (stage index, sweep index; default: the last
sweep of the schedule) run between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly one finest-layer sweep.

  python tools/profile_sweep.py [--cfg 5] [--profile-last] [--quiet]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule, SCHED_LADDER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--profile-last", action="store_true")
ap.add_argument("--quiet", action="store_true")
ap.add_argument("--bcap", type=int, default=0)
ap.add_argument("--bcap-big", type=int, default=0)
ap.add_argument("--onchip", type=int, default=0, help="testing: boxes above this side go to tier G")
ap.add_argument("--json", default="")
ap.add_argument("--cells-npz", default="", help="dump per-cell (iters, box, mufu, kcycles) of every sweep at side >= n/2")
ap.add_argument("--cells-all", action="store_true", help="--cells-npz for every layer")
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
       eps_start=p.get("eps_start", 0.0), bcap_main=a.bcap, bcap_big=a.bcap_big,
       bcap_onchip=a.onchip)
sched = build_schedule(n, p.get("coarsest", 8), p["kappa_final"], p.get("eps_start", 0.0))
rows = []
cell_dump = {}
t0 = time.time()
for k, (side, kappa, sweeps) in enumerate(sched):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    for j in range(sweeps):
        last = (k == len(sched) - 1 and j == sweeps - 1)
        if last and a.profile_last:
            g.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        g.iterate(1)
        st = g.stats()
        if last and a.profile_last:
            torch.cuda.cudart().cudaProfilerStop()
        row = dict(stage=k, side=side, kappa=kappa, sweep=j,
                   **{q: st[q] for q in ("cells", "iters_sum", "iters_max", "failed", "entries", "ms",
                                         "solve_ms", "big_cells", "max_box", "fallbacks", "mufu_ops")})
        rows.append(row)
        if a.cells_npz and (side >= n // 2 or a.cells_all):
            it, bx, mf, kc = g.cell_stats()
            cell_dump[f"s{side}_k{kappa}_j{j}"] = np.stack([it, bx, mf.astype(np.float64), kc])
        if not a.quiet:
            print(json.dumps(row), flush=True)
tot = g.totals()
print("total wall s", time.time() - t0, json.dumps(tot), g.primal_cost(), g.marginal_error(), flush=True)
if a.cells_npz:
    np.savez(a.cells_npz, **cell_dump)
if a.json:
    json.dump(dict(rows=rows, totals=tot), open(a.json, "w"))
