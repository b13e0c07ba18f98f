"""Throughput of dd_run_schedule_batch (B image pairs in flight on one GPU)
vs the same pairs solved one after another (dd_run_schedule), host wall time
around each (both wait for completion), cfg 5 by default.

  python tools/batch_time.py [--cfg 5] [--batch 1,2,3,5] [--reps 2] [--cluster -1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, SCHED_LADDER  # noqa: E402
from paper_2001_10986_b200.dd import run_schedule_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--batch", default="1,2,3,5")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cluster", type=int, default=-1)
ap.add_argument("--check", action="store_true", help="batch state == sequential state (bitwise)")
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
bs = [int(x) for x in a.batch.split(",")]
ctxs = []
for k in range(max(bs)):
    mu, nu = config_images(a.cfg, pair=k)
    ctxs.append(DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
                   eps_start=p.get("eps_start", 0.0), max_inner_iter=100000, cluster=a.cluster))
# warm-up
for c in ctxs:
    c.reset()
run_schedule_batch(ctxs)
seq = {}
for k, c in enumerate(ctxs):
    ts = []
    for r in range(a.reps):
        c.reset(); c.synchronize()
        c.reset_totals()
        t0 = time.perf_counter()
        c.run_schedule()
        ts.append(time.perf_counter() - t0)
    seq[k] = (min(ts), c.totals()["cells"] // a.reps)
    print(json.dumps(dict(mode="seq", pair=k, s=min(ts), cells=seq[k][1])), flush=True)
ref_state = ctxs[0].get_state() if a.check else None
for b in bs:
    ts = []
    for r in range(a.reps):
        for c in ctxs[:b]:
            c.reset(); c.synchronize()
        t0 = time.perf_counter()
        run_schedule_batch(ctxs[:b])
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    cells = sum(seq[k][1] for k in range(b))
    tseq = sum(seq[k][0] for k in range(b))
    print(json.dumps(dict(mode="batch", batch=b, s=t, seq_s=tseq, speedup=tseq / t, cells_per_s=cells / t,
                          seq_cells_per_s=cells / tseq)), flush=True)
    if a.check:
        st = ctxs[0].get_state()
        same = all(np.array_equal(st[k], ref_state[k]) for k in ("boxes", "offsets", "values", "alpha_A", "alpha_B"))
        print(json.dumps(dict(batch=b, pair0_bit_identical=bool(same))), flush=True)
