"""Fill ratio of composite-cell union boxes: |union of the member boxes| and
the non-zero support vs b_r * b_c, for the final state of a config ladder
(work the separable passes spend on zero-nu points of the union box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ddinputs import config_images, CONFIGS
from paper_2001_10986_b200 import DD
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = CONFIGS[cfg]; n, s = p["n"], p["s"]
mu, nu = config_images(cfg)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=1, coarsest_side=8)
g.run_schedule()
st = g.get_state(); nb = st["info"]["nb"]; side = st["info"]["side"]
B, O, V = st["boxes"], st["offsets"], st["values"]
for part in (1, 2):
    nca = nb // 2 if part == 1 else nb // 2 + 1
    tot_box = tot_union = tot_nz = 0
    w_box = w_nz = 0.0
    for pp in range(nca):
        for q in range(nca):
            rows = [2 * pp, 2 * pp + 1] if part == 1 else [r for r in (2 * pp - 1, 2 * pp) if 0 <= r < nb]
            cols = [2 * q, 2 * q + 1] if part == 1 else [c for c in (2 * q - 1, 2 * q) if 0 <= c < nb]
            mem = [r * nb + c for r in rows for c in cols]
            y0 = min(B[i, 0] for i in mem); x0 = min(B[i, 1] for i in mem)
            y1 = max(B[i, 0] + B[i, 2] for i in mem); x1 = max(B[i, 1] + B[i, 3] for i in mem)
            m_union = np.zeros((y1 - y0, x1 - x0), bool); m_nz = np.zeros_like(m_union)
            for i in mem:
                b = B[i]
                m_union[b[0] - y0:b[0] - y0 + b[2], b[1] - x0:b[1] - x0 + b[3]] = True
                v = V[O[i]:O[i] + b[2] * b[3]].reshape(b[2], b[3]) > 0
                m_nz[b[0] - y0:b[0] - y0 + b[2], b[1] - x0:b[1] - x0 + b[3]] |= v
            a = (y1 - y0) * (x1 - x0)
            tot_box += a; tot_union += m_union.sum(); tot_nz += m_nz.sum()
            wgt = a  # work ~ a * b, weight big cells more
            w_box += a * max(y1 - y0, x1 - x0); w_nz += m_nz.sum() * max(y1 - y0, x1 - x0)
    print(f"part {part}: union-of-boxes / box area {tot_union / tot_box:.3f}, nonzero / box area {tot_nz / tot_box:.3f}, work-weighted nonzero fill {w_nz / w_box:.3f}", flush=True)
