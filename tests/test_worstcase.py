"""f4 worst-case lab on the oracle (Sec. 3.3,
P:1197-1268) pinned against the paper's theorems and closed forms:

  * Theorem ThreeConvergence: every sweep contracts the
    sub-optimality at least by (1 + exp(-2||c||/eps) q/(1-q))^-1;
  * Lemma SubOptKL: KL(pi|K) - KL(pi*|K) = KL(pi|pi*), and the
    sub-optimality never increases (exact block coordinate descent);
  * the 1/eps law of Example WorstCaseThree (eq. LambdaBound, Fig.
    WorstCaseThreeEps: -log(lambda^-1 - 1) affine in 1/eps, below the bound);
  * the q-proportionality of Example WorstCaseThreeQ (eq. LambdaBoundQ);
  * Example WorstCaseChain: convergence slows as N grows (Fig. WorstCaseN);
  * the initial coupling is partially optimal on each composite cell
    for the UNregularised cost (a linear program, scipy's HiGHS), i.e. a fixed
    point of the unregularised iteration."""
import numpy as np
import pytest

from oracle import worstcase as W


def test_setups_match_figure():
    inst = W.three_cell(0.3, 2.0)
    np.testing.assert_allclose(inst["mu"], [0.35, 0.3, 0.35])
    for pi in (inst["pi0"],):
        np.testing.assert_allclose(pi.sum(1), inst["mu"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(pi.sum(0), inst["nu"], rtol=0, atol=1e-15)
    c = inst["c"]
    # "embedding ... into R^2 such that c becomes the distance function": a metric
    for i in range(3):
        for j in range(3):
            for k in range(3):
                assert c[i, k] <= c[i, j] + c[j, k]
    ch = W.chain(5)
    expect = np.full((5, 5), 10.0)
    np.fill_diagonal(expect, 0.0)
    expect[0, 4] = expect[4, 0] = 1.0
    np.testing.assert_array_equal(ch["c"], expect)
    np.testing.assert_allclose(ch["pi0"].sum(0), 0.2)
    np.testing.assert_allclose(ch["pi0"].sum(1), 0.2)
    assert ch["A"] == [[0, 1], [2, 3], [4]] and ch["B"] == [[0], [1, 2], [3, 4]]


def test_unregularised_fixed_point():
    """pi0 restricted to X_J x Y is optimal for the unregularised
    cell problem with its own marginals, on every composite cell of A and B."""
    from scipy.optimize import linprog
    inst = W.three_cell(0.3, 1.0)
    pi0, c = inst["pi0"], inst["c"]
    for J in inst["A"] + inst["B"]:
        a = pi0[J, :].sum(1)
        b = pi0[J, :].sum(0)
        nJ, ny = len(J), c.shape[1]
        Aeq, beq = [], []
        for r in range(nJ):
            row = np.zeros(nJ * ny); row[r * ny:(r + 1) * ny] = 1; Aeq.append(row); beq.append(a[r])
        for y in range(ny):
            col = np.zeros(nJ * ny); col[y::ny] = 1; Aeq.append(col); beq.append(b[y])
        res = linprog(c[J, :].ravel(), A_eq=np.array(Aeq), b_eq=np.array(beq), bounds=(0, None), method="highs")
        assert res.status == 0
        assert (c[J, :] * pi0[J, :]).sum() <= res.fun + 1e-12


@pytest.mark.parametrize("eps", [2.0, 3.0, 5.0])
def test_theorem1_every_sweep(eps):
    inst = W.three_cell(0.3, eps)
    tr = W.trace(inst, 400)
    d = tr["delta"]
    fac = W.theorem1_factor(inst)
    ok = d[1:-1] > 1e-11
    ratios = d[2:][ok] / d[1:-1][ok]
    assert ratios.size > 20
    assert ratios.max() <= fac + 1e-9, (ratios.max(), fac)
    # Lemma SubOptKL: the sub-optimality is KL to the optimum, never increasing
    K = W.kl_to_kernel
    pistar = tr["pistar"]
    for pi in (inst["pi0"], tr["pi"]):
        # (exact for feasible pi; the plans meet their marginals to ~1e-13)
        assert abs((K(pi, inst) - K(pistar, inst)) - W.kl(pi, pistar)) <= 1e-10
    assert np.all(np.diff(d[1:]) <= 1e-13)


def test_eps_law_three_cells():
    q = 0.3
    xs, ys = [], []
    for eps in (2.0, 2.5, 3.0, 4.0, 5.0):
        inst = W.three_cell(q, eps)
        fit = W.fit_lambda(W.trace(inst, 700)["delta"])
        assert fit["r2"] > 0.999
        y = -np.log(1.0 / fit["lam"] - 1.0)
        assert y <= 20.0 / eps - np.log(q / (1 - q)) + 1e-9          # eq. LambdaBound
        xs.append(1.0 / eps)
        ys.append(y)
    slope, icpt = np.polyfit(xs, ys, 1)
    r2 = 1 - np.sum((np.polyval([slope, icpt], xs) - ys) ** 2) / np.sum((ys - np.mean(ys)) ** 2)
    assert r2 > 0.99                       # "the 1/eps-behaviour is accurate"
    assert 5.0 <= slope <= 20.0            # below the bound's 2||c|| = 20 (paper: off by ~2)


def test_q_law_three_cells():
    eps = 10.0
    vals = []
    for q in (0.05, 0.1, 0.2, 0.3):
        inst = W.three_cell(q, eps)
        fit = W.fit_lambda(W.trace(inst, 300)["delta"])
        g = 1.0 / fit["lam"] - 1.0
        assert g >= np.exp(-2.0) * q / (1 - q)                         # eq. LambdaBoundQ
        vals.append(g / q)
    vals = np.array(vals)
    assert vals.max() / vals.min() < 1.15  # lambda^-1 - 1 proportional to q


def test_chain_slows_with_n():
    lam = {}
    for N in (4, 8):
        lam[N] = W.fit_lambda(W.trace(W.chain(N), 1200)["delta"])["lam"]
    assert 0.0 < lam[4] < lam[8] < 1.0
