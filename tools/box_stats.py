"""Distribution of composite-cell Y boxes (union bbox vs nonempty rows/cols) after a ladder."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ddinputs import gaussian_mixture_image
from paper_2001_10986_b200 import DD, build_schedule
n = int(sys.argv[1]); s = 8; cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mu = gaussian_mixture_image(n, 1, cfg); nu = gaussian_mixture_image(n, 2, cfg)
g = DD(mu, nu, 0.5 / n**2, s, schedule=1, coarsest_side=8, max_inner_iter=3000)
def analyse(tag):
    st = g.get_state(); info = st["info"]; nb = info["nb"]; side = info["side"]
    boxes = st["boxes"]; offs = st["offsets"]; vals = st["values"]
    bb = boxes[:, 2:4]
    print(tag, "side", side, "basic box side mean/p50/p90/max", bb.max(1).mean(), np.percentile(bb.max(1), 50), np.percentile(bb.max(1), 90), bb.max(), flush=True)
    for part in (1, 2):
        nca = nb // 2 if part == 1 else nb // 2 + 1
        U, Cc = [], []
        for p in range(nca):
            for q in range(nca):
                if part == 1: rows, cols = [2*p, 2*p+1], [2*q, 2*q+1]
                else:
                    rows = [r for r in (2*p-1, 2*p) if 0 <= r < nb]; cols = [c for c in (2*q-1, 2*q) if 0 <= c < nb]
                mem = [r*nb+c for r in rows for c in cols]
                y0 = min(boxes[i,0] for i in mem); x0 = min(boxes[i,1] for i in mem)
                y1 = max(boxes[i,0]+boxes[i,2] for i in mem); x1 = max(boxes[i,1]+boxes[i,3] for i in mem)
                rf = np.zeros(y1-y0, bool); cf = np.zeros(x1-x0, bool)
                for i in mem:
                    b = boxes[i]; v = vals[offs[i]:offs[i]+b[2]*b[3]].reshape(b[2], b[3]) > 0
                    rf[b[0]-y0:b[0]-y0+b[2]] |= v.any(1); cf[b[1]-x0:b[1]-x0+b[3]] |= v.any(0)
                U.append(max(y1-y0, x1-x0)); Cc.append(max(rf.sum(), cf.sum()))
        U = np.array(U); Cc = np.array(Cc)
        print(f"  part {part}: union p50 {np.percentile(U,50):.0f} p90 {np.percentile(U,90):.0f} p99 {np.percentile(U,99):.0f} max {U.max()} | compressed p50 {np.percentile(Cc,50):.0f} p90 {np.percentile(Cc,90):.0f} p99 {np.percentile(Cc,99):.0f} max {Cc.max()} | >32: {np.mean(U>32):.2f} / {np.mean(Cc>32):.2f}  >48: {np.mean(U>48):.2f} / {np.mean(Cc>48):.2f}", flush=True)
for side, kappa, sweeps in build_schedule(n, 8, 0.5):
    while g.state_info()["side"] < side:
        g.refine()
        if side >= 64: analyse("after-refine")
    g.set_eps(kappa / side**2)
    g.iterate(sweeps)
    st = g.stats()
    if side >= 64:
        print(side, kappa, {q: st[q] for q in ("iters_sum", "iters_max", "failed", "ms", "big_cells", "max_box")}, flush=True)
        analyse(f"k={kappa}")
