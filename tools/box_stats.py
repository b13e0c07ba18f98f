"""Composite-cell Y-box statistics at the end of each layer of a ladder run:
union bounding box vs. the product of its non-empty rows x non-empty columns
("compressed" box), and the per-iteration separable exp work of each
(a_r a_c b_c + a_r b_r b_c + b_r b_c a_c + b_r a_r a_c).

  python tools/box_stats.py [--cfg 5] [--min-side 256]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--min-side", type=int, default=256)
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=1, coarsest_side=p.get("coarsest", 8),
       eps_start=p.get("eps_start", 0.0))


def analyse(tag):
    st = g.get_state()
    info = st["info"]
    nb, side, sl = info["nb"], info["side"], info["s"]
    boxes, offs, vals = st["boxes"], st["offsets"], st["values"]
    # per basic cell: non-empty row / col masks in global coordinates
    rowm = np.zeros((nb * nb, side), bool)
    colm = np.zeros((nb * nb, side), bool)
    for i in range(nb * nb):
        y0, x0, hr, hc = boxes[i]
        if hr * hc == 0:
            continue
        v = vals[offs[i]:offs[i] + hr * hc].reshape(hr, hc) > 0
        rowm[i, y0:y0 + hr] = v.any(1)
        colm[i, x0:x0 + hc] = v.any(0)
    out = {}
    for part in (1, 2):
        nca = nb // 2 if part == 1 else nb // 2 + 1
        W_u = W_c = 0.0
        U, Cc, works_u, works_c = [], [], [], []
        for pp in range(nca):
            for q in range(nca):
                if part == 1:
                    rows, cols = [2 * pp, 2 * pp + 1], [2 * q, 2 * q + 1]
                else:
                    rows = [r for r in (2 * pp - 1, 2 * pp) if 0 <= r < nb]
                    cols = [c for c in (2 * q - 1, 2 * q) if 0 <= c < nb]
                mem = [r * nb + c for r in rows for c in cols]
                ar, ac = len(rows) * sl, len(cols) * sl
                rm = rowm[mem].any(0)
                cm = colm[mem].any(0)
                ridx, cidx = np.nonzero(rm)[0], np.nonzero(cm)[0]
                br, bc = ridx[-1] - ridx[0] + 1, cidx[-1] - cidx[0] + 1
                brc, bcc = len(ridx), len(cidx)
                wu = ar * ac * bc + ar * br * bc + br * bc * ac + br * ar * ac
                wc = ar * ac * bcc + ar * brc * bcc + brc * bcc * ac + brc * ar * ac
                U.append(max(br, bc))
                Cc.append(max(brc, bcc))
                works_u.append(wu)
                works_c.append(wc)
        U, Cc, wu, wc = map(np.array, (U, Cc, works_u, works_c))
        big = U > 40
        out[part] = dict(cells=len(U), union_p50=float(np.median(U)), union_p90=float(np.percentile(U, 90)),
                         union_p99=float(np.percentile(U, 99)), union_max=int(U.max()),
                         comp_p50=float(np.median(Cc)), comp_p90=float(np.percentile(Cc, 90)),
                         comp_p99=float(np.percentile(Cc, 99)), comp_max=int(Cc.max()),
                         frac_union_gt40=float(big.mean()), frac_comp_gt40=float((Cc > 40).mean()),
                         work_union=float(wu.sum()), work_comp=float(wc.sum()),
                         work_share_big_union=float(wu[big].sum() / wu.sum()))
    print(tag, side, json.dumps(out), flush=True)


for side, kappa, sweeps in build_schedule(n, p.get("coarsest", 8), p["kappa_final"], p.get("eps_start", 0.0)):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    g.iterate(sweeps)
    if side >= a.min_side:
        analyse(f"kappa={kappa}")
