"""Pins of the oracle against the worked values stored under tests/golden/
(each file cites its source passage).  CPU only."""
import json
import os

import numpy as np

from oracle import Oracle, build_schedule, sinkhorn_dense
from oracle.oracle import SCHED_LADDER

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return json.load(open(os.path.join(GOLD, name)))


def test_golden_p1_2x2():
    g = _load("p1_2x2.json")
    C = np.array(g["cost"])
    f, gg, it, err, rc = sinkhorn_dense(g["mu"], g["nu"], C, g["eps"], 1e-15)
    P = np.exp((f[:, None] + gg[None, :] - C) / g["eps"])    # absorbed potentials (oracle convention)
    assert rc == 0
    assert abs(P[0, 0] - g["pi11"]) < 1e-15 and abs(P[1, 1] - g["pi11"]) < 1e-15
    assert abs(P[0, 1] - g["pi12"]) < 1e-15 and abs(P[1, 0] - g["pi12"]) < 1e-15
    assert abs(g["pi11"] - np.e / (2 * (1 + np.e))) < 1e-16


def test_golden_schedule_counts():
    g = _load("schedule_counts.json")
    for n, total in g["totals"].items():
        sch = build_schedule(int(n), g["coarsest_side"], g["final_kappa"])
        assert sum(w for _, _, w in sch) == total, n


def test_golden_refinement_s368():
    """S:368 on a grid: fine 16x16 (s=4) under a coarse 8x8 (s=4, nb=2).  The
    coarse cell j = 0 holds share nuhat_j/nuhat = 0.5 at the coarse pixel
    yhat = (0,0); the fine cell i1 = (0,0) holds mu(X_i1)/muhat(X_j) = 0.4 of
    its parent's mass; the children of yhat carry nu in the ratio 0.6 : 0.4
    (rows).  Summing the refined nu_i1^0 over each child row gives the
    S:368 values (0.12, 0.08) times nuhat(yhat)."""
    g = _load("refinement_s368.json")
    n = 16
    mu = np.full((n, n), 1.0)
    # parent j = coarse basic cell (0,0) = fine basic cells (0,0),(0,1),(1,0),(1,1) (4x4 px each)
    ratio = g["mu_Xi"] / g["muhat_Xj"]                  # 0.4
    w = {(0, 0): ratio, (0, 1): (1 - ratio) / 3, (1, 0): (1 - ratio) / 3, (1, 1): (1 - ratio) / 3}
    for (a, b), share in w.items():
        mu[4 * a:4 * a + 4, 4 * b:4 * b + 4] = share * 4.0 / 16.0
    mu /= mu.sum()
    nu = np.full((n, n), 1.0)
    c0, c1 = g["nu_children"]
    nu[0, 0:2] = c0 / 2          # children of yhat = (0,0): fine rows 0 and 1, cols 0..1
    nu[1, 0:2] = c1 / 2
    nu /= nu.sum()
    o = Oracle(mu, nu, 1.0, 4, schedule=SCHED_LADDER, coarsest_side=8)
    st = o.get_state()
    side = 8
    mu8, nu8 = o.layer_marginals()
    share_j = g["nuhat_j"] / g["nuhat"]                  # 0.5 at every coarse pixel
    shares = np.array([share_j, (1 - share_j) / 3, (1 - share_j) / 3, (1 - share_j) / 3])
    st["values"] = np.concatenate([shares[j] * nu8.ravel() for j in range(4)])
    st["offsets"] = np.arange(4, dtype=np.int64) * side * side
    st["boxes"] = np.tile(np.array([0, 0, side, side], np.int32), (4, 1))
    o.set_state(st)
    o.refine()
    D = o.basic_marginals_dense().reshape(16, n, n)
    nuhat_y = nu8[0, 0]
    got = np.array([D[0, 0, 0:2].sum(), D[0, 1, 0:2].sum()]) / nuhat_y
    np.testing.assert_allclose(got, g["expected_nu_i0"], rtol=1e-13)
