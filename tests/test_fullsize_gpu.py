"""Parity at BASELINE.json's full sizes (config 5: 2048^2, s = 8, 10% noise;
config 4: 1024^2, s = 8), in the launch configuration bench.py times, on
sampled outputs the oracle can compute one by one: the GPU runs the whole
schedule but its last sweep; the oracle imports that exact state (boxes,
values, potentials) and solves a sample of the last sweep's composite cells
with its dense fp64 Sinkhorn (Algorithm 2 lines 8-13); their basic-cell
marginals are compared with the GPU's after that sweep.

The sample is stratified by the cell's union Y-box side, so every K1 tier
and the least-margin numerics are covered: tier 0 (box <= 24), tier 1
(24 < box <= 120; the per-cell hi grid coarsens with the box) and tier 2
(box > 120, up to one cell above 300 px).  Bounds: a
cell where both solves stopped at the same Sinkhorn iteration must agree to
1e-7 ||mu_J|| in L1 (the fp32 arithmetic floor); a one-iteration mismatch
(the GPU stops at (1 - 2^-7) ||mu_J|| Err, A28) to Err ||mu_J||
per solve, i.e. 2 Err ||mu_J||.  The distribution of the stop-iteration
mismatches and the per-cell L1 differences are written to
gpurun_out/fullsize_cfg{4,5}.json (committed copies under profiles/).
Whole-state properties that hold at any size are
checked on the full output."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import CONFIGS, config_images  # noqa: E402
from oracle import Oracle  # noqa: E402

ERR = 1e-6
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


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


def _run_all_but_last(cfg):
    """The bench's schedule (same ladder and options) minus its last sweep."""
    from paper_2001_10986_b200 import DD, build_schedule
    p = CONFIGS[cfg]
    n, s = p["n"], p["s"]
    mu, nu = config_images(cfg)
    eps = p["kappa_final"] / n**2
    g = DD(mu, nu, eps, s, schedule=1, coarsest_side=8, err_tol=ERR)
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
    return g, mu, nu, eps, s, n


BINS = [(0, 20, 2), (20, 28, 2), (28, 40, 2), (40, 56, 2), (56, 90, 2), (90, 120, 2),
        (120, 180, 2), (180, 250, 2), (300, 10**6, 1)]


def _sample(box, iters, rng):
    """Stratified by box side; in the largest bins the cells with the fewest
    iterations (the dense oracle's cost is ~ 2 |X| b^2 per iteration)."""
    picks = []
    for lo, hi, k in BINS:
        cand = np.nonzero((box > lo) & (box <= hi))[0]
        if not cand.size:
            continue
        if lo >= 120:
            cand = cand[np.argsort(iters[cand] * box[cand].astype(np.float64) ** 2)][:max(k, 4)]
        picks += [int(c) for c in rng.choice(cand, size=min(k, cand.size), replace=False)]
    return picks


def _fullsize_parity(cfg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    g, mu, nu, eps, s, n = _run_all_but_last(cfg)
    before = g.get_state()
    g.iterate(1)                                  # the last sweep (partition B)
    after = g.get_state()
    part = after["info"]["last_partition"]
    assert part == 2 and after["info"]["side"] == n
    it_g, box_g, _, _ = g.cell_stats()
    nb = after["info"]["nb"]
    # whole-output properties (any size): X-error bound and Y-feasibility
    lx, ly = g.marginal_error()
    assert lx <= ERR and ly <= ERR, (lx, ly)
    picks = _sample(box_g, it_g, np.random.default_rng(cfg))
    assert len(picks) >= 12
    assert (box_g[picks] > 120).any() and ((box_g[picks] > 24) & (box_g[picks] <= 120)).any()
    o = Oracle(mu, nu, eps, s, empty_init=True)   # single layer n^2, state imported below
    o.set_state(before)
    it_o = o.solve_cells(part, np.array(picks))
    ost = o.get_state()
    mass = mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()
    rows, fails = [], []
    for k, cell in enumerate(picks):
        mem = _members(nb, part, cell)
        d = sum(_l1(_dense_box(after, i), _dense_box(ost, i)) for i in mem)
        mJ = mass[mem].sum()
        dit = int(it_g[cell]) - int(it_o[k])
        rel = d / mJ
        rows.append(dict(cell=cell, box=int(box_g[cell]), it_gpu=int(it_g[cell]), it_oracle=int(it_o[k]),
                         l1_rel=rel))
        if dit == 0:
            ok = rel <= 1e-7                    # same stop iteration: the fp32 floor (P9)
        elif abs(dit) == 1:
            ok = rel <= 2 * ERR                 # each solve within Err of the cell optimum
        else:
            ok = rel <= 4 * ERR
        if not ok:
            fails.append(rows[-1])
    dits = np.array([r["it_gpu"] - r["it_oracle"] for r in rows])
    summary = dict(cfg=cfg, n_cells=len(rows), iteration_mismatch={str(v): int((dits == v).sum())
                                                                    for v in np.unique(dits)},
                   max_rel_same_iter=max([r["l1_rel"] for r in rows if r["it_gpu"] == r["it_oracle"]] or [0.0]),
                   max_rel=max(r["l1_rel"] for r in rows), l1_x=lx, l1_y=ly, cells=rows)
    print(json.dumps({k: v for k, v in summary.items() if k != "cells"}))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"fullsize_cfg{cfg}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    assert not fails, fails
    # the stop iterations agree to within 1 % (+2): the GPU tests the stop on
    # its fp32 potentials with the (1 - 2^-7) margin of DESIGN.md A28, so
    # cells near the threshold stop a few iterations apart (r02: -3 .. +6 of
    # 150 .. 3000); the marginals still agree to ~1e-7 ||mu_J|| (the plan
    # changes by far less than Err per iteration there)
    for r in rows:
        assert abs(r["it_gpu"] - r["it_oracle"]) <= 2 + 0.01 * r["it_oracle"], r


def test_cfg5_sampled_cells_vs_oracle():
    _fullsize_parity(5)


def test_cfg4_sampled_cells_vs_oracle():
    _fullsize_parity(4)
