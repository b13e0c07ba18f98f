"""Which cells of the cfg-4 sweep used by tests/test_rescue_gpu.py are rescued in fp64 (flag 16) or
flagged (flag 1): the stall is trajectory-dependent, so the test picks its cell from this set."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ddinputs import CONFIGS, config_images
from paper_2001_10986_b200 import DD, build_schedule

p = CONFIGS[4]
n, s = p["n"], p["s"]
mu, nu = config_images(4)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=1, coarsest_side=8, max_inner_iter=100000)
for side, kappa, sweeps in build_schedule(n, 8, p["kappa_final"]):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    nsw = 1 if (side == n and kappa == 0.5) else sweeps
    for j in range(nsw):
        g.iterate(1, check=False)
        it, bx, _, _, fl, ex = g.cell_stats(flags=True, err=True)
        for c in np.nonzero(fl & 17)[0]:
            print(f"side {side} kappa {kappa} sweep {j} cell {c} flags {fl[c]} iters {it[c]} box {bx[c]}")
    if side == n and kappa == 0.5:
        break
g.synchronize(check=False)
g.iterate(1, check=False)
it, bx, _, _, fl, ex = g.cell_stats(flags=True, err=True)
print("test sweep: part", g.state_info()["last_partition"])
for c in np.nonzero(fl & 17)[0]:
    print(f"TEST cell {c} flags {fl[c]} iters {it[c]} box {bx[c]} err {ex[c]:.3e}")
print("cell 3771:", fl[3771], it[3771], bx[3771], ex[3771])
