"""Run a config's ladder and report every cell the solve flagged (bit 0
max_inner_iter, bit 1 non-finite / numerically empty row, bit 2 eps raised):
sweep, cell, flags, iterations, box side.

  python tools/failed_cells.py [--cfg 4] [--pair 0] [--max-iter 100000]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule, SCHED_LADDER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--pair", type=int, default=0)
ap.add_argument("--max-iter", type=int, default=100000)
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg, pair=a.pair)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
       eps_start=p.get("eps_start", 0.0), max_inner_iter=a.max_iter)
tot = 0
for side, kappa, sweeps in build_schedule(n, p.get("coarsest", 8), p["kappa_final"], p.get("eps_start", 0.0)):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    for j in range(sweeps):
        g.iterate(1, check=False)
        it, bx, mf, kc, fl = g.cell_stats(flags=True)
        bad = np.nonzero(fl & 7)[0]
        tot += bad.size
        for c in bad[:8]:
            print(f"side {side} kappa {kappa} sweep {j} part {g.state_info()['last_partition']} cell {c} "
                  f"flags {fl[c]} iters {it[c]} box {bx[c]}", flush=True)
g.synchronize(check=False)
print(f"flagged cells: {tot}; final marginal error {g.marginal_error()}")
