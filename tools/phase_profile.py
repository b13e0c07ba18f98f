"""K1 phase profile: build libdd_gpu_prof.so (-DDD_PHASE_PROF) if needed, run
the config ladder with it and print, per layer side >= --min-side, how the
warps' time splits between the Sinkhorn passes and the barriers.

  python tools/phase_profile.py [--cfg 5] [--min-side 1024] [--build-only]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_SO = os.environ.get("DD_PROF_LIB", os.path.join(ROOT, "paper_2001_10986_b200", "libdd_gpu_prof.so"))

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--min-side", type=int, default=1024)
ap.add_argument("--build-only", action="store_true")
ap.add_argument("--cluster", type=int, default=0, help="dd_options.reserved[3] (1: every big-path cell on the cluster tier)")
a = ap.parse_args()

if a.build_only:
    from paper_2001_10986_b200 import build as b
    cmd = [b.NVCC, *b.FLAGS, "-DDD_PHASE_PROF", "-o", PROF_SO, *b.sources()]
    subprocess.check_call(cmd)
    sys.exit(0)

os.environ["DD_LIB"] = PROF_SO
import numpy as np  # noqa: E402
from ddinputs import config_images, CONFIGS  # noqa: E402
from paper_2001_10986_b200 import DD, build_schedule  # noqa: E402

p = CONFIGS[a.cfg]
n, s = p["n"], p["s"]
mu, nu = config_images(a.cfg)
g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=1, coarsest_side=p.get("coarsest", 8),
       eps_start=p.get("eps_start", 0.0), max_inner_iter=100000, cluster=a.cluster)
names = ["Y1", "bar1", "Y2X1", "bar2", "X2", "errsum", "loop", "prologue", "epilogue(cta)", "iters(cta)"]
for side, kappa, sweeps in build_schedule(n, p.get("coarsest", 8), p["kappa_final"], p.get("eps_start", 0.0)):
    while g.state_info()["side"] < side:
        g.refine()
    g.set_eps(kappa / side**2)
    g.phase_profile()
    g.iterate(sweeps, check=False)
    pp = g.phase_profile().astype(np.float64)
    if side < a.min_side:
        continue
    for mode in (0, 1):
        v = pp[mode]
        loop = v[6]
        if loop <= 0:
            continue
        parts = " ".join(f"{names[k]} {v[k] / loop * 100:5.1f}%" for k in range(6))
        print(f"side {side} kappa {kappa} {'big ' if mode else 'smem'}: loop share of warp time "
              f"{loop / (v[6] + v[7]) * 100:5.1f}% | {parts} | iters {v[9]:.3g} cycles/iter/warp {loop / max(v[9], 1):.0f}",
              flush=True)
