"""Long-pole analysis of a per-cell dump (tools/profile_sweep.py --cells-npz
--cells-all): per sweep, the device time of the sweep vs the longest single
cell solve (CellOut solve time in kcycles at the SM clock) and the sum of all
cell solve times over the SM slots.  A sweep is latency-bound when its
longest cell is close to the sweep time.

  python tools/cell_times.py dump.npz sweeps.json [--mhz 1965]
"""
import json
import sys

import numpy as np

npz = np.load(sys.argv[1])
rows = json.load(open(sys.argv[2]))["rows"]
mhz = float(sys.argv[sys.argv.index("--mhz") + 1]) if "--mhz" in sys.argv else 1965.0
byname = {}
for r in rows:
    byname.setdefault((r["side"], r["kappa"]), []).append(r)
print(f"{'sweep':>22} {'ms':>8} {'maxcell_ms':>10} {'ratio':>6} {'box@max':>7} {'it@max':>6} "
      f"{'sum_ms/148':>10} {'top5 boxes'}")
tot_sweep = tot_pole = 0.0
for key in npz.files:
    it, bx, mf, kc = npz[key]
    side = int(key.split("_")[0][1:])
    kap = float(key.split("_")[1][1:])
    j = int(key.split("_")[2][1:])
    r = byname[(side, kap)][j]
    t = kc.astype(np.float64) * 1024 / (mhz * 1e3)       # ms per cell solve
    k = int(np.argmax(t))
    top = np.argsort(-t)[:5]
    tot_sweep += r["ms"]
    tot_pole += t[k]
    print(f"{key:>22} {r['ms']:8.2f} {t[k]:10.2f} {t[k] / r['ms']:6.2f} {int(bx[k]):7d} {int(it[k]):6d} "
          f"{t.sum() / 148:10.2f} {[int(b) for b in bx[top]]} it {[int(x) for x in it[top]]}")
print(f"total sweep ms {tot_sweep:.1f}, sum of the longest cell per sweep {tot_pole:.1f}")
