"""Debug helper: the s = 8 big-tier parity case (tests/test_gpu_parity.py::
test_big_tier_parity_s8) with the library in $DD_LIB; prints cost, marginal
errors and the plan difference vs the oracle, twice (determinism)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddinputs import gaussian_mixture_image  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2001_10986_b200 import DD  # noqa: E402

n, s = 32, 8
mu, nu = gaussian_mixture_image(n, 11, 3), gaussian_mixture_image(n, 12, 3)
eps = 0.5 / n**2
o = Oracle(mu, nu, eps, s, err_tol=1e-6)
o.iterate(6)
co, _ = o.primal_cost()
Do = o.basic_marginals_dense()
for bb in (0, 40):
    for rep in range(2):
        g = DD(mu, nu, eps, s, err_tol=1e-6, bcap_main=18, bcap_big=bb)
        for k in range(6):
            g.iterate(1)
            st = g.stats()
            print(" sweep", k, {q: st[q] for q in ("cells", "iters_sum", "iters_max", "failed", "big_cells", "fallbacks")})
        cg, _ = g.primal_cost()
        lx, ly = g.marginal_error()
        Dg = g.basic_marginals_dense()
        print(os.environ.get("DD_LIB", "default"), "bcap_big", bb, "rep", rep, "cost rel", (cg - co) / co, "lx", lx, "ly", ly,
              "plan L1", np.abs(Dg - Do).sum(), flush=True)
