import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ddinputs import config_images
from paper_2001_10986_b200 import DD, build_schedule
from paper_2001_10986_b200.striped import LocalTransport, StripedRun
N = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mu, nu = config_images(2); n, s = 64, 4
kw = dict(err_tol=1e-6, eps_start=1.0, coarsest_side=16, schedule=1)
ctxs = [(r, DD(mu, nu, 0.5 / n**2, s, **kw)) for r in range(N)]
run = StripedRun(ctxs, N, LocalTransport(N))
run.start()
side = 16
for sd, kappa, sweeps in build_schedule(n, 16, 0.5, 1.0):
    while side < sd:
        run.refine(); side *= 2
        print("refined", side, run.bounds, flush=True)
    run.set_eps(kappa / sd**2)
    for j in range(sweeps):
        run.sweep()
        for r, dd in ctxs:
            try:
                dd.synchronize()
            except Exception as e:
                st = dd.get_state()
                bx = st["boxes"]; nb = st["info"]["nb"]
                empty_rows = [i for i in range(nb) if (bx[i*nb:(i+1)*nb, 2] * bx[i*nb:(i+1)*nb, 3] == 0).all()]
                print("FAIL rank", r, "side", sd, "sweep", run.half_index - 1, e, "empty rows", empty_rows, "bounds", run.bounds, flush=True)
                sys.exit(1)
print("ok")
