"""Predicted per-stripe work imbalance of the multi-GPU stripes (SURVEY.md
8(e), VERDICT r1 "cost-aware stripe bounds") from a per-cell dump of the
cfg-5 schedule (tools/pair_sweeps.py --cells-npz): per layer >= 128^2 and
N ranks, max/mean of the stripes' algorithmic MUFU work for the equal-row
bounds (striped.stripe_bounds) and for cost-balanced even bounds chosen from
the previous sweep's per-cell work (a greedy prefix split of the A-cell
rows), plus the Amdahl bound of the replicated coarse layers.

  python tools/stripe_balance.py gpurun_out/cells_p0.npz [--out profiles/r02/stripe_balance.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2001_10986_b200.striped import stripe_bounds, owned_cell_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("npz")
ap.add_argument("--out", default="profiles/r02/stripe_balance.json")
ap.add_argument("--s", type=int, default=8)
a = ap.parse_args()
z = np.load(a.npz)


def row_work(key):
    it, bx, mf, kc = z[key]
    side = int(key.split("_")[0][1:])
    nb = side // min(a.s, side // 2)
    j = int(key.split("_")[2][1:])
    return side, nb, j, mf


def stripe_loads(nb, part, mf, bounds):
    nca = nb // 2 if part == 1 else nb // 2 + 1
    w = mf.reshape(nca, nca).sum(1)
    return np.array([w[slice(*owned_cell_rows(nb, part, bounds[r], bounds[r + 1]))].sum()
                     for r in range(len(bounds) - 1)])


def balanced_bounds(nb, wA, nranks):
    """Even bounds (A-cell row boundaries) splitting the A-row work evenly."""
    c = np.concatenate([[0.0], np.cumsum(wA)])
    tot = c[-1]
    b = [0]
    for r in range(1, nranks):
        q = int(np.searchsorted(c, tot * r / nranks))
        q = min(max(q, b[-1] // 2 + 1), nb // 2 - (nranks - r))
        b.append(2 * q)
    b.append(nb)
    return b


keys = sorted(z.files, key=lambda k: (int(k.split("_")[0][1:]), k))
out = {"source": a.npz, "layers": {}}
total_work = sum(z[k][2].sum() for k in keys)
for N in (2, 4, 8):
    res = {}
    repl = 0.0
    prev = {}
    for key in keys:
        side, nb, j, mf = row_work(key)
        b = stripe_bounds(nb, N)
        if b is None:
            repl += mf.sum()
            continue
        part = 1 if mf.size == (nb // 2) ** 2 else 2
        eq = stripe_loads(nb, part, mf, b)
        # cost-aware: bounds from the previous sweep's A-row work of this layer
        pw = prev.get(side)
        bb = balanced_bounds(nb, pw, N) if pw is not None else b
        ba = stripe_loads(nb, part, mf, bb)
        if part == 1:
            prev[side] = mf.reshape(nb // 2, nb // 2).sum(1)
        r = res.setdefault(side, {"equal_rows": [], "cost_aware": [], "work": 0.0})
        r["equal_rows"].append(float(eq.max() / eq.mean()))
        r["cost_aware"].append(float(ba.max() / ba.mean()))
        r["work"] += float(mf.sum())
    layers = {str(k): {"equal_rows_max_over_mean": float(np.mean(v["equal_rows"])),
                       "cost_aware_max_over_mean": float(np.mean(v["cost_aware"])),
                       "share_of_work": v["work"] / total_work} for k, v in res.items()}
    striped = 1.0 - repl / total_work
    eq_t = repl / total_work + sum(l["share_of_work"] * l["equal_rows_max_over_mean"] / N for l in layers.values())
    ca_t = repl / total_work + sum(l["share_of_work"] * l["cost_aware_max_over_mean"] / N for l in layers.values())
    out["layers"][str(N)] = {"per_layer": layers, "replicated_share": repl / total_work,
                            "predicted_speedup_equal_rows": 1.0 / eq_t, "predicted_speedup_cost_aware": 1.0 / ca_t,
                            "note": "work model only (MUFU ops per cell): ignores the latency-bound coarse sweeps "
                                    "and the exchange; an upper bound on strong scaling"}
    print(f"N={N}: replicated {repl / total_work:.3%} of the work; predicted speedup equal rows "
          f"{1 / eq_t:.2f}, cost-aware {1 / ca_t:.2f}")
    for k, l in layers.items():
        print(f"   side {k}: max/mean equal {l['equal_rows_max_over_mean']:.2f} cost-aware "
              f"{l['cost_aware_max_over_mean']:.2f} (work share {l['share_of_work']:.1%})")
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(out, open(a.out, "w"), indent=1)
