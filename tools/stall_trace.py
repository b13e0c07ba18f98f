"""X-error of one GPU cell solve vs the iteration cap: the GPU state before a
sweep is re-imported and the sweep re-run with max_inner_iter = k for several
k; prints the cell's K1 L1 X-error against its stop tolerance ||mu_J|| Err.

  python tools/stall_trace.py --cfg 4 --side 1024 --kappa 0.5 --sweep 1 --cell 3771
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
ap.add_argument("--side", type=int, default=1024)
ap.add_argument("--kappa", type=float, default=0.5)
ap.add_argument("--sweep", type=int, default=1)
ap.add_argument("--cell", type=int, default=3771)
ap.add_argument("--caps", default="100,200,300,400,420,426,430,450,500,700,1000,2000,5000,20000")
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg, pair=a.pair)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
       max_inner_iter=100000)
done = False
for side, kappa, sweeps in build_schedule(n, p.get("coarsest", 8), p["kappa_final"]):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    for j in range(sweeps):
        if side == a.side and kappa == a.kappa and j == a.sweep:
            done = True
            break
        g.iterate(1, check=False)
    if done:
        break
g.synchronize(check=False)
before = g.get_state()
f = n // a.side
mu_l = mu.reshape(a.side, f, a.side, f).sum((1, 3))
s_l = min(s, a.side // 2)
nb = a.side // s_l
part = 1 if before["info"]["half_index"] % 2 == 0 else 2
nca = nb // 2 if part == 1 else nb // 2 + 1
cp, cq = divmod(a.cell, nca)
span = (lambda q: (2 * q, 2 * q + 1)) if part == 1 else (lambda q: (max(0, 2 * q - 1), min(nb - 1, 2 * q)))
r0, r1 = span(cp)
c0, c1 = span(cq)
muJ = mu_l[r0 * s_l:(r1 + 1) * s_l, c0 * s_l:(c1 + 1) * s_l].sum()
print(f"cell {a.cell}: part {part} basic rows {r0}-{r1} cols {c0}-{c1}, ||mu_J|| = {muJ:.3e}, "
      f"tol = {muJ * 1e-6:.3e}", flush=True)
for k in [int(x) for x in a.caps.split(",")]:
    g.set_max_inner_iter(k)
    g.set_state(before)
    g.iterate(1, check=False)
    it, bx, mf, kc, fl, ex = g.cell_stats(flags=True, err=True)
    print(f"cap {k:6d}: iters {it[a.cell]:6d} flags {fl[a.cell]} err/tol {ex[a.cell] / (muJ * 1e-6):.4f} "
          f"box {bx[a.cell]}", flush=True)
