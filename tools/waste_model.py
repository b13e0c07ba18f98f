"""Where does K1's fused big-cell path compute exps that the algorithm does
not need?  Runs the cfg-5 ladder, takes the final state and, for every
composite cell of the next sweep's partition that goes to the fused tiers
(union box side > 24), counts per iteration (in units of a_r exps):

  nz      non-zero points of nu_cell (the algorithmic phase-A / phase-B work)
  rows    points inside each row's [first, last] non-zero column
  groups  4 x (union width of each 4-row group)        (phase B, interleaved)
  chunks  4 x 32 x ceil(union width / 32) per group     (phase A)
  half    the same with a half chunk for a last chunk of <= 16 columns
  quarter the same with 8-column quarter chunks (<= 8: quarter, <= 16: half,
          <= 24: half + quarter), the phase A of DD_PA_Q = 1

  python tools/waste_model.py [--cfg 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, SCHED_LADDER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
a = ap.parse_args()
p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=SCHED_LADDER, coarsest_side=p.get("coarsest", 8),
       eps_start=p.get("eps_start", 0.0))
g.run_schedule()
st = g.get_state()
info = st["info"]
nb = info["nb"]
boxes, offs, vals = st["boxes"], st["offsets"], st["values"]
part = 2 if info["last_partition"] == 1 else 1        # the next sweep's partition


def span(c):
    if part == 1:
        return 2 * c, 2 * c + 1
    return max(2 * c - 1, 0), min(2 * c, nb - 1)


nca = nb // 2 if part == 1 else nb // 2 + 1
tot = dict(nz=0, rows=0, groups=0, chunks=0, half=0, quarter=0, cells=0, full=0)
hist = np.zeros(8, np.int64)          # group union widths by 8-column bins (up to 64+)
for cp in range(nca):
    r0, r1 = span(cp)
    for cq in range(nca):
        c0, c1 = span(cq)
        mem = [r * nb + c for r in range(r0, r1 + 1) for c in range(c0, c1 + 1)]
        bx = [boxes[m] for m in mem if boxes[m][2] > 0 and boxes[m][3] > 0]
        if not bx:
            continue
        y0 = min(b[0] for b in bx); x0 = min(b[1] for b in bx)
        y1 = max(b[0] + b[2] for b in bx); x1 = max(b[1] + b[3] for b in bx)
        br, bc = y1 - y0, x1 - x0
        if max(br, bc) <= 24:
            continue
        m = np.zeros((br, bc), bool)
        for mm in mem:
            b = boxes[mm]
            if b[2] <= 0 or b[3] <= 0:
                continue
            v = vals[offs[mm]:offs[mm] + b[2] * b[3]].reshape(b[2], b[3])
            m[b[0] - y0:b[0] - y0 + b[2], b[1] - x0:b[1] - x0 + b[3]] |= v > 0
        if bc > br:
            m = m.T
        nzr = m.any(1)
        lo = np.where(nzr, m.argmax(1), 0)
        hi = np.where(nzr, m.shape[1] - 1 - m[:, ::-1].argmax(1), -1)
        tot["nz"] += int(m.sum())
        tot["rows"] += int((hi - lo + 1).clip(0).sum())
        tot["full"] += m.size
        for g0 in range(0, m.shape[0], 4):
            l, h = lo[g0:g0 + 4], hi[g0:g0 + 4]
            ok = h >= l
            if not ok.any():
                continue
            w = int(h[ok].max() - l[ok].min() + 1)
            tot["groups"] += 4 * w
            tot["chunks"] += 4 * 32 * ((w + 31) // 32)
            tot["half"] += 4 * 32 * (w // 32) + (4 * 32 if w % 32 > 16 else (4 * 16 if w % 32 else 0))
            r = w % 32       # last chunk: quarter (<= 8), half (<= 16), half + quarter (<= 24), full
            tot["quarter"] += 4 * 32 * (w // 32) + 4 * (0 if r == 0 else 8 if r <= 8 else 16 if r <= 16
                                                          else 24 if r <= 24 else 32)
            hist[min(w // 8, 7)] += 1
        tot["cells"] += 1
print("partition", part, "fused-tier cells", tot["cells"])
print("group widths (8-col bins):", hist.tolist())
for k in ("full", "rows", "groups", "chunks", "half", "quarter"):
    print(f"{k:7s} / nz = {tot[k] / tot['nz']:.3f}")
