"""Two fresh contexts stepped in lockstep on the same input: report the first
sweep whose state differs (bitwise) and where.

  python tools/determinism.py [--n 256] [--s 4] [--seed 100] [--batch]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import gaussian_mixture_image  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--s", type=int, default=4)
ap.add_argument("--seed", type=int, default=100)
ap.add_argument("--serial", action="store_true")
a = ap.parse_args()
mu, nu = gaussian_mixture_image(a.n, a.seed, 3), gaussian_mixture_image(a.n, a.seed + 1, 3)
eps = 0.5 / a.n**2
gs = [DD(mu, nu, eps, a.s, schedule=1, coarsest_side=8, max_inner_iter=100000) for _ in range(2)]
k = 0
for side, kappa, sweeps in build_schedule(a.n, 8, 0.5):
    for g in gs:
        while g.state_info()["side"] < side:
            g.refine()
        g.set_eps(kappa / side**2)
    for j in range(sweeps):
        for g in gs:
            g.iterate(1, check=False)
        sts = [g.get_state() for g in gs]
        cs = [g.cell_stats(flags=True, err=True) for g in gs]
        k += 1
        diff = [key for key in ("boxes", "offsets", "values", "alpha_A", "alpha_B")
                if sts[0][key].shape != sts[1][key].shape or not np.array_equal(sts[0][key], sts[1][key])]
        if diff:
            it0, bx0, _, _, fl0, e0 = cs[0]
            it1, bx1, _, _, fl1, e1 = cs[1]
            dc = np.nonzero((it0 != it1) | (e0 != e1))[0]
            print(f"sweep {k} (side {side} kappa {kappa} j {j}) differs in {diff}; cells with different "
                  f"iters/err: {dc[:10].tolist()} iters {it0[dc[:5]].tolist()} vs {it1[dc[:5]].tolist()} "
                  f"box {bx0[dc[:5]].tolist()} flags {fl0[dc[:5]].tolist()}", flush=True)
            if sts[0]["alpha_A"].shape == sts[1]["alpha_A"].shape:
                for key in ("alpha_A", "alpha_B"):
                    dd = np.abs(sts[0][key] - sts[1][key])
                    if dd.max() > 0:
                        ij = np.unravel_index(np.argmax(dd), dd.shape)
                        print(f"  {key} max diff {dd.max():.3e} at {ij}", flush=True)
            sys.exit(1)
print(f"{k} sweeps bit-identical")
