"""Stage-by-stage ladder run with a sync after every stage (debug aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ddinputs import gaussian_mixture_image
from paper_2001_10986_b200 import DD, build_schedule
n = int(sys.argv[1]); s = int(sys.argv[2]); cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mu = gaussian_mixture_image(n, 1, cfg); nu = gaussian_mixture_image(n, 2, cfg)
g = DD(mu, nu, 0.5 / n**2, s, schedule=1, coarsest_side=8)
t0 = time.time()
for side, kappa, sweeps in build_schedule(n, 8, 0.5):
    while g.state_info()["side"] < side:
        g.refine(); g.synchronize()
        print("refined", g.state_info(), flush=True)
    g.set_eps(kappa / side**2)
    for k in range(sweeps):
        g.iterate(1)
        st = g.stats()
        print(side, kappa, k, {q: st[q] for q in ("cells", "iters_sum", "iters_max", "failed", "entries", "ms", "solve_ms", "big_cells", "max_box", "fallbacks")}, flush=True)
print("total", time.time() - t0, g.totals(), g.primal_cost(), g.marginal_error())
