"""Per image pair of a config: the full ladder with a given max_inner_iter,
per-sweep statistics (iters_max, ms, failed) and, optionally, the per-cell
dump of every sweep (tools/cell_times.py input).

  python tools/pair_sweeps.py [--cfg 5] [--pairs 0,1,2,3,4] [--max-iter 100000] [--cells-npz out.npz]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule, SCHED_LADDER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--pairs", default="0,1,2,3,4")
ap.add_argument("--max-iter", type=int, default=100000)
ap.add_argument("--cells-npz", default="")
ap.add_argument("--json", default="")
ap.add_argument("--cluster", type=int, default=0, help="dd_options.reserved[3]")
ap.add_argument("--theta", type=int, default=0, help="dd_options.reserved[4]")
ap.add_argument("--ncl", type=int, default=0, help="dd_options.reserved[5]")
ap.add_argument("--tag", default="")
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
out = {}
dump = {}
for k in [int(x) for x in a.pairs.split(",")]:
    mu, nu = config_images(a.cfg, pair=k)
    g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
           eps_start=p.get("eps_start", 0.0), max_inner_iter=a.max_iter, cluster=a.cluster,
           cluster_theta=a.theta, n_clusters=a.ncl)
    sched = build_schedule(n, p.get("coarsest", 8), p["kappa_final"], p.get("eps_start", 0.0))
    rows = []
    for st_i, (side, kappa, sweeps) in enumerate(sched):
        while g.state_info()["side"] < side:
            g.refine()
        g.set_eps(kappa / side**2)
        for j in range(sweeps):
            g.iterate(1, check=False)
            st = g.stats()
            rows.append(dict(side=side, kappa=kappa, sweep=j, ms=st["ms"], solve_ms=st["solve_ms"],
                             iters_max=st["iters_max"], iters_sum=st["iters_sum"], cells=st["cells"],
                             failed=st["failed"], mufu_ops=st["mufu_ops"], max_box=st["max_box"]))
            if a.cells_npz and k == 0:
                it, bx, mf, kc = g.cell_stats()
                dump[f"s{side}_k{kappa}_j{j}"] = np.stack([it, bx, mf.astype(np.float64), kc])
    g.synchronize(check=False)
    tot_ms = sum(r["ms"] for r in rows)
    print(json.dumps(dict(tag=a.tag, pair=k, ms=tot_ms, cluster_cells=g.totals()["cluster_cells"], iters_max=max(r["iters_max"] for r in rows),
                          failed=sum(r["failed"] for r in rows),
                          layer_ms={str(sd): sum(r["ms"] for r in rows if r["side"] == sd)
                                    for sd in sorted({r["side"] for r in rows})})), flush=True)
    out[k] = rows
    del g
if a.json:
    with open(a.json, "w") as f:
        json.dump(out, f)
if a.cells_npz:
    np.savez(a.cells_npz, **dump)
