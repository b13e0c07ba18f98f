"""f4 worst-case lab (Sec. 3.3) on the
CPU oracle: contraction factors of the three-cell eps- and q-studies and the
chain N-study vs Theorem ThreeConvergence.  Writes JSON.

  python tools/worstcase_lab.py [--out profiles/r02/worstcase.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import worstcase as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/r02/worstcase.json")
a = ap.parse_args()
t0 = time.time()
out = {"source": "oracle/worstcase.py (dense fp64 Algorithm 1, exact cell sub-solves)", "eps_study": [], "q_study": [],
       "chain_study": []}
q = 0.3
for eps in (1.5, 2.0, 2.5, 3.0, 4.0, 5.0):
    inst = W.three_cell(q, eps)
    tr = W.trace(inst, 4000 if eps < 2 else 1200)
    fit = W.fit_lambda(tr["delta"])
    d = tr["delta"]
    ok = d[1:-1] > 1e-11
    out["eps_study"].append(dict(eps=eps, lam=fit["lam"], r2=fit["r2"], fit_window=fit.get("window"),
                                 y=-np.log(1 / fit["lam"] - 1), y_bound=20 / eps - np.log(q / (1 - q)),
                                 theorem1_factor=W.theorem1_factor(inst),
                                 max_sweep_ratio=float((d[2:][ok] / d[1:-1][ok]).max())))
xs = [1 / r["eps"] for r in out["eps_study"]]
ys = [r["y"] for r in out["eps_study"]]
sl, ic = np.polyfit(xs, ys, 1)
out["eps_fit"] = {"slope_vs_1_over_eps": sl, "intercept": ic, "bound_slope": 20.0,
                  "note": "y = -log(lambda^-1 - 1); bound y <= 2||c||/eps - log(q/(1-q)) (eq. LambdaBound)"}
for qq in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3):
    inst = W.three_cell(qq, 10.0)
    fit = W.fit_lambda(W.trace(inst, 400)["delta"])
    g = 1 / fit["lam"] - 1
    out["q_study"].append(dict(q=qq, lam=fit["lam"], r2=fit["r2"], lam_inv_minus_1=g,
                               bound=float(np.exp(-2) * qq / (1 - qq)), ratio_to_bound=g / (np.exp(-2) * qq / (1 - qq)),
                               per_q=g / qq))
for N in (3, 4, 6, 8, 12, 16):
    fit = W.fit_lambda(W.trace(W.chain(N), 3000)["delta"])
    out["chain_study"].append(dict(N=N, eps=1.4, lam=fit["lam"], one_minus_lam=1 - fit["lam"], r2=fit["r2"]))
out["seconds"] = time.time() - t0
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps({k: out[k] for k in ("eps_fit", "seconds")}))
for r in out["eps_study"]:
    print(f"eps {r['eps']}: lambda {r['lam']:.6f} y {r['y']:.3f} <= bound {r['y_bound']:.3f}")
for r in out["q_study"]:
    print(f"q {r['q']}: lambda^-1-1 {r['lam_inv_minus_1']:.4f} >= {r['bound']:.4f} (x{r['ratio_to_bound']:.1f}), /q {r['per_q']:.3f}")
for r in out["chain_study"]:
    print(f"chain N {r['N']}: 1 - lambda {r['one_minus_lam']:.3e}")
