"""Parity at BASELINE.json's full size (config 5: 2048^2, s = 8, 10% noise,
the full ladder), in the launch configuration bench.py times, on sampled
outputs the oracle can compute one by one: the GPU runs the whole schedule
but its last sweep; the oracle imports that exact state (boxes, values,
potentials) and solves a sample of the last sweep's composite cells with its
dense fp64 Sinkhorn (Algorithm 2 lines 8-13); their basic-cell marginals are
compared with the GPU's after that sweep.  Whole-state properties that hold
at any size are checked on the full output."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import CONFIGS, config_images  # noqa: E402
from oracle import Oracle  # noqa: E402


def _members(nb, part, cell):
    nca = nb // 2 if part == 1 else nb // 2 + 1
    p, q = divmod(cell, nca)
    span = (lambda t: [2 * t, 2 * t + 1]) if part == 1 else \
        (lambda t: [r for r in (2 * t - 1, 2 * t) if 0 <= r < nb])
    return [r * nb + c for r in span(p) for c in span(q)]


def _dense_box(st, i):
    y0, x0, hr, hc = st["boxes"][i]
    o = st["offsets"][i]
    return (y0, x0, st["values"][o:o + hr * hc].reshape(hr, hc))


def _l1(a, b):
    """L1 distance of two boxed marginals."""
    (ya, xa, va), (yb, xb, vb) = a, b
    y0, x0 = min(ya, yb), min(xa, xb)
    y1 = max(ya + va.shape[0], yb + vb.shape[0])
    x1 = max(xa + va.shape[1], xb + vb.shape[1])
    A = np.zeros((y1 - y0, x1 - x0)); B = np.zeros_like(A)
    A[ya - y0:ya - y0 + va.shape[0], xa - x0:xa - x0 + va.shape[1]] = va
    B[yb - y0:yb - y0 + vb.shape[0], xb - x0:xb - x0 + vb.shape[1]] = vb
    return np.abs(A - B).sum()


def test_cfg5_sampled_cells_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD, build_schedule
    p = CONFIGS[5]
    n, s = p["n"], p["s"]
    mu, nu = config_images(5)
    eps = p["kappa_final"] / n**2
    g = DD(mu, nu, eps, s, schedule=1, coarsest_side=8)
    sched = build_schedule(n, 8, p["kappa_final"])
    side, total = 8, sum(w for _, _, w in sched)
    done = 0
    for sd, kappa, sweeps in sched:
        while side < sd:
            g.refine()
            side *= 2
        g.set_eps(kappa / sd**2)
        k = sweeps if done + sweeps < total else sweeps - 1
        g.iterate(k)
        done += k
    before = g.get_state()
    g.iterate(1)                                  # the last sweep (partition B)
    after = g.get_state()
    part = after["info"]["last_partition"]
    assert part == 2 and after["info"]["side"] == n
    it_g, box_g, _, _ = g.cell_stats()
    nb = after["info"]["nb"]
    # whole-output properties (any size): Y-feasibility and balanced masses
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
    # a sample of cells the dense oracle finishes quickly, over box sizes
    rng = np.random.default_rng(5)
    picks = []
    for lo, hi in [(0, 20), (20, 28), (28, 40), (40, 56)]:
        cand = np.nonzero((box_g > lo) & (box_g <= hi))[0]
        if cand.size:
            picks += list(rng.choice(cand, size=min(2, cand.size), replace=False))
    assert len(picks) >= 6
    o = Oracle(mu, nu, eps, s, empty_init=True)     # single layer n^2, state imported below
    o.set_state(before)
    o.solve_cells(part, np.array(picks))
    ost = o.get_state()
    mass = mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()
    for cell in picks:
        mem = _members(nb, part, int(cell))
        d = sum(_l1(_dense_box(after, i), _dense_box(ost, i)) for i in mem)
        # both solves stop within Err of the same cell optimum
        assert d <= 4e-6 * mass[mem].sum() + 1e-14, (cell, box_g[cell], d, mass[mem].sum())
