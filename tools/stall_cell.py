"""A cell the GPU flags (max_inner_iter reached): import the GPU state
before that sweep into the fp64 oracle and solve the same cells there, to
tell an inherently slow cell from a numerical stall of the fp32 path.

  python tools/stall_cell.py --cfg 4 --side 1024 --kappa 0.5 --sweep 1 --cells 3771,4033 [--max-iter 100000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule, SCHED_LADDER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--pair", type=int, default=0)
ap.add_argument("--side", type=int, default=1024)
ap.add_argument("--kappa", type=float, default=0.5)
ap.add_argument("--sweep", type=int, default=1)
ap.add_argument("--cells", default="")
ap.add_argument("--top", type=int, default=0, help="the top-K iteration cells of that sweep instead")
ap.add_argument("--max-iter", type=int, default=100000)
ap.add_argument("--gpu-max-iter", type=int, default=100000)
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg, pair=a.pair)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
       max_inner_iter=a.gpu_max_iter)
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
g.iterate(1, check=False)
it, bx, mf, kc, fl = g.cell_stats(flags=True)
if a.top:
    cells = np.argsort(-it)[:a.top].astype(np.int32)
else:
    cells = np.array([int(c) for c in a.cells.split(",")], np.int32)
part = g.state_info()["last_partition"]
print("gpu:", [(int(c), int(it[c]), int(bx[c]), int(fl[c])) for c in cells], flush=True)
# the layer's images for the oracle: sum-pool the finest images to this side (A20)
f = n // a.side
mu_l = mu.reshape(a.side, f, a.side, f).sum((1, 3))
nu_l = nu.reshape(a.side, f, a.side, f).sum((1, 3))
s_l = min(s, a.side // 2)
o = Oracle(mu_l, nu_l, a.kappa / a.side**2, s_l, empty_init=True, max_inner_iter=a.max_iter)
o.set_state(before)
t0 = time.time()
io = o.solve_cells(part, cells)
print("oracle iters:", [int(x) for x in io], f"{time.time() - t0:.1f} s", flush=True)
