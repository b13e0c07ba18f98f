"""Batch (dd_run_schedule_batch) vs sequential (dd_run_schedule) final
states, per problem: bitwise equality and the size of any difference.

  python tools/batch_check.py [--n 256] [--s 4] [--k 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import gaussian_mixture_image  # noqa: E402
from paper_2001_10986_b200 import DD  # noqa: E402
from paper_2001_10986_b200.dd import run_schedule_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--s", type=int, default=4)
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
eps = 0.5 / a.n**2
kw = dict(schedule=1, coarsest_side=8, max_inner_iter=100000)
imgs = [(gaussian_mixture_image(a.n, 100 + 2 * k, 3), gaussian_mixture_image(a.n, 101 + 2 * k, 3)) for k in range(a.k)]
seq = []
for mu, nu in imgs:
    g = DD(mu, nu, eps, a.s, **kw)
    g.run_schedule()
    seq.append(g.get_state())
    g.close()


def cmp(st, ref):
    out = {}
    for key in ("boxes", "offsets", "values", "alpha_A", "alpha_B"):
        if st[key].shape != ref[key].shape:
            out[key] = f"shape {st[key].shape} vs {ref[key].shape}"
        elif not np.array_equal(st[key], ref[key]):
            d = np.abs(st[key].astype(np.float64) - ref[key].astype(np.float64))
            out[key] = f"{int((d > 0).sum())} entries differ, max {d.max():.3e}"
    return out or "bit-identical"


for rep in range(a.reps):
    bat = [DD(mu, nu, eps, a.s, **kw) for mu, nu in imgs]
    run_schedule_batch(bat)
    for k, g in enumerate(bat):
        print(f"rep {rep} batch problem {k}: {cmp(g.get_state(), seq[k])}", flush=True)
    for g in bat:
        g.close()
for k, (mu, nu) in enumerate(imgs):
    g = DD(mu, nu, eps, a.s, **kw)
    g.run_schedule()
    print(f"sequential rerun problem {k}: {cmp(g.get_state(), seq[k])}", flush=True)
    g.close()
