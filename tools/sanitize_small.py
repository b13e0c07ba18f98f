"""Small runs over every K1 tier, the ladder (refinement + gluing), the
queries and the stripe primitives, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ddinputs import config_images, gaussian_mixture_image
from paper_2001_10986_b200 import DD
from paper_2001_10986_b200.striped import LocalTransport, StripedRun
mu, nu = config_images(1)
for kw in (dict(), dict(bcap_main=10), dict(bcap_main=10, bcap_big=12)):
    g = DD(mu, nu, 2 / 32**2, 4, **kw)
    g.iterate(4)
    print(kw, g.primal_cost(), g.marginal_error(), g.fetch_plan_coo()[2].sum(), flush=True)
mu2, nu2 = config_images(2)
g = DD(mu2, nu2, 0.5 / 64**2, 4, schedule=1, eps_start=1.0, coarsest_side=16, bcap_main=12)
g.run_schedule()
print("ladder", g.primal_cost(), g.marginal_error(), flush=True)
n = 64
mu3, nu3 = gaussian_mixture_image(n, 3, 3), gaussian_mixture_image(n, 4, 3)
ctxs = [(r, DD(mu3, nu3, 1.0 / n**2, 8, bcap_main=18)) for r in range(2)]
run = StripedRun(ctxs, 2, LocalTransport(2))
run.start()
run.iterate(4)
print("stripes", run.primal_cost(), run.marginal_error(), flush=True)
