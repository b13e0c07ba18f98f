"""fp64 rescue of K1: a cell the fp32 passes cannot
finish at the error floor is continued from its potentials by the same four
separable passes in fp64 (rescue_fp64) and must agree with the oracle like any
other cell (within ~2 Err ||mu_J|| when the stop iterations
differ).  Which cells stall depends on the fp32 trajectory (on an earlier
build the border cell 3771 of cfg 4, pair 0, ||mu_J|| = 1.8e-6, stalled at
1.04 ||mu_J|| Err for 1e5 iterations, profiles/r02/stall_cell3771_fp32.log;
with the quarter-chunk phase A it converges in 461 fp32 iterations), so the
test takes the fp64 continuation on that cell through the testing hook
DD_FORCE_RESCUE="cell:it" (dd_common.cuh: the cell leaves the fp32 loop after
`it` iterations exactly as the stall detector would make it)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import CONFIGS, config_images  # noqa: E402
from oracle import Oracle  # noqa: E402

ERR = 1e-6
CELL = 3771


def _members(nb, part, cell):
    nca = nb // 2 if part == 1 else nb // 2 + 1
    p, q = divmod(cell, nca)
    span = (lambda t: [2 * t, 2 * t + 1]) if part == 1 else \
        (lambda t: [r for r in (2 * t - 1, 2 * t) if 0 <= r < nb])
    return [r * nb + c for r in span(p) for c in span(q)]


def _dense(st, i, side):
    y0, x0, hr, hc = st["boxes"][i]
    o = st["offsets"][i]
    D = np.zeros((side, side))
    D[y0:y0 + hr, x0:x0 + hc] = st["values"][o:o + hr * hc].reshape(hr, hc)
    return D


@pytest.fixture(scope="module")
def before_state():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD, build_schedule
    p = CONFIGS[4]
    n, s = p["n"], p["s"]
    mu, nu = config_images(4)
    g = DD(mu, nu, p["kappa_final"] / n**2, s, schedule=1, coarsest_side=8, max_inner_iter=100000)
    for side, kappa, sweeps in build_schedule(n, 8, p["kappa_final"]):
        while g.state_info()["side"] < side:
            g.refine()
        g.set_eps(kappa / side**2)
        if side == n and kappa == 0.5:
            g.iterate(1, check=False)
            break
        g.iterate(sweeps, check=False)
    g.synchronize(check=False)
    return g, g.get_state(), mu, nu


def test_rescue_matches_oracle(before_state):
    g, before, mu, nu = before_state
    n, s = 1024, 8
    g.set_state(before)
    os.environ["DD_FORCE_RESCUE"] = f"{CELL}:64"
    try:
        g.iterate(1, check=False)
        g.synchronize(check=False)
    finally:
        del os.environ["DD_FORCE_RESCUE"]
    after = g.get_state()
    it, bx, _, _, fl, ex = g.cell_stats(flags=True, err=True)
    part = after["info"]["last_partition"]
    assert part == 2
    nb = n // s
    mem = _members(nb, part, CELL)
    mJ = mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()[mem].sum()
    assert fl[CELL] & 16, "the fp64 continuation did not run on the forced cell"
    assert it[CELL] > 64
    assert not fl[CELL] & 1 and ex[CELL] <= ERR * mJ, (fl[CELL], ex[CELL] / (ERR * mJ))
    # only the forced cell (and cells that stall by themselves) take the fp64 path
    assert ((fl & 16) != 0).sum() <= 8
    o = Oracle(mu, nu, 0.5 / n**2, s, empty_init=True, max_inner_iter=100000)
    o.set_state(before)
    io = o.solve_cells(part, np.array([CELL]))
    ost = o.get_state()
    d = sum(np.abs(_dense(after, i, n) - _dense(ost, i, n)).sum() for i in mem)
    assert d <= 2 * ERR * mJ, (d / mJ, int(it[CELL]), int(io[0]))


def test_stall_detector_flags(before_state):
    """The sweep's cells that the stall detector hands to the fp64 path carry
    flag 16; those fp64 cannot finish within its iteration cap either (the
    oracle needs > 4e4 iterations on them) also carry flag 1 (reading A6) and
    keep a Y-feasible plan."""
    g, before, mu, nu = before_state
    g.set_state(before)
    g.iterate(1, check=False)
    g.synchronize(check=False)
    it, bx, _, _, fl, ex = g.cell_stats(flags=True, err=True)
    stalled = np.nonzero(fl & 16)[0]
    assert stalled.size <= 8
    for c in stalled:
        assert it[c] >= 512 + 1
    failed = (fl & 1) != 0
    assert ((fl[failed] & 16) != 0).all(), "a cell hit max_inner_iter in fp32 without the stall detector"
    lx, ly = g.marginal_error()
    assert ly < 1e-8


def test_set_max_inner_iter_full_size(before_state):
    """A6 at full size through dd_set_max_inner_iter: a cap far below the
    needed iterations -> the capped cells are flagged, dd_synchronize returns
    DD_ENOCONV, the state stays Y-feasible (sum_i nu_i = nu); the oracle side
    of A6 is tests/test_abi_harness.py."""
    from paper_2001_10986_b200 import NotConverged
    g, before, mu, nu = before_state
    g.set_state(before)
    g.set_max_inner_iter(5)
    try:
        g.iterate(1, check=False)
        with pytest.raises(NotConverged):
            g.synchronize()
        it, _, _, _, fl = g.cell_stats(flags=True)
        assert (fl & 1).sum() > 100 and it.max() <= 5
    finally:
        g.set_max_inner_iter(100000)
        g.synchronize(check=False)
    lx, ly = g.marginal_error()
    assert ly < 1e-8        # truncation at tau = 1e-15 (A9) only
