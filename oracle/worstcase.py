"""Worst-case lab of the domain decomposition on the CPU
oracle, fp64.  TEST INFRASTRUCTURE ONLY (oracle side): imported by tests/ and
tools/worstcase_lab.py; the product package never imports it.

Dense discrete problems X = Y = {1..N} with singleton basic cells, run with
Algorithm 1 (P:290-300 / Alg. DomDec) and exact cell sub-solves:

  * three cells, dependency on eps  -- Example WorstCaseThree,
  * three cells, dependency on q    -- Example WorstCaseThreeQ,
  * chain graph, dependency on N    -- Example WorstCaseChain,

each against Theorem ThreeConvergence (eq. ThreeConvergenceKLDecrement):
Delta(pi^l) <= (1 + exp(-2||c||/eps) ||mu_2|| / ||mu_{1,3}||)^-1 Delta(pi^(l-1)),
with Delta(pi) = KL(pi|K) - KL(pi*|K) = KL(pi|pi*) for feasible pi
(Lemma SubOptKL) and pi* a high-precision single Sinkhorn solve
(P:1214-1215).  Costs and initial couplings as in Figure WorstCaseSetup
(P:1184-1186): three cells c = 0 on the diagonal, 1 on (1,3) and (3,1), 10
elsewhere; chain c(i,j) = 0 (i = j), 1 ((i,j) in {(1,N),(N,1)}), 10 else.
Reference measure K = exp(-c/eps) mu (x) nu (reading A2).

Every sub-solve is the oracle's dense log-domain Sinkhorn (dd_oracle.c,
sinkhorn_dense) run to an L1 X-error of 1e-13 ||mu_J|| -- "exact" for these tiny
problems -- ending with a Y-iteration so the Y-marginal is exact.
"""
from __future__ import annotations

import numpy as np

from .oracle import sinkhorn_dense

SUB_TOL = 1e-13


def three_cell(q: float, eps: float) -> dict:
    """Example WorstCaseThree: mu = nu = (p, q, p), p = (1 - q)/2; pi0 moves the
    mass of cell 1 to 3 and back; J_A = {{1,2},{3}},
    J_B = {{1},{2,3}} (Example ThreeCells)."""
    if not 0.0 < q < 1.0:
        raise ValueError("q must lie in (0, 1)")
    p = (1.0 - q) / 2.0
    c = np.array([[0.0, 10.0, 1.0], [10.0, 0.0, 10.0], [1.0, 10.0, 0.0]])
    mu = np.array([p, q, p])
    pi0 = np.array([[0.0, 0.0, p], [0.0, q, 0.0], [p, 0.0, 0.0]])
    return dict(c=c, mu=mu, nu=mu.copy(), pi0=pi0, eps=float(eps),
                A=[[0, 1], [2]], B=[[0], [1, 2]], name=f"three q={q} eps={eps}")


def chain(N: int, eps: float = 1.4) -> dict:
    """Example WorstCaseChain: uniform masses, first and last cell exchange
    their mass through N - 2 intermediate cells."""
    if N < 3:
        raise ValueError("N >= 3")
    c = np.full((N, N), 10.0)
    np.fill_diagonal(c, 0.0)
    c[0, N - 1] = c[N - 1, 0] = 1.0
    mu = np.full(N, 1.0 / N)
    pi0 = np.diag(mu).copy()
    pi0[0, 0] = pi0[N - 1, N - 1] = 0.0
    pi0[0, N - 1] = pi0[N - 1, 0] = 1.0 / N
    A = [[i, i + 1] for i in range(0, N - 1, 2)] + ([[N - 1]] if N % 2 else [])
    B = [[0]] + [[i, i + 1] for i in range(1, N - 1, 2)] + ([] if N % 2 else [[N - 1]])
    return dict(c=c, mu=mu, nu=mu.copy(), pi0=pi0, eps=float(eps), A=A, B=B, name=f"chain N={N} eps={eps}")


def _plan(f, g, c, eps):
    return np.exp((f[:, None] + g[None, :] - c) / eps)


def global_optimum(inst: dict) -> np.ndarray:
    """pi* by a single dense Sinkhorn on the whole problem."""
    f, g, it, err, rc = sinkhorn_dense(inst["mu"], inst["nu"], inst["c"], inst["eps"], 1e-15, max_iter=2000000)
    if rc != 0:
        raise RuntimeError(f"global Sinkhorn rc={rc} err={err}")
    return _plan(f, g, inst["c"], inst["eps"])


def cell_solve(mu_J, nu_J, c_J, eps):
    """Entropic OT of one composite cell with marginals (mu_J,
    nu_J): Y points with nu_J = 0 carry no mass (reading A22)."""
    f, g, it, err, rc = sinkhorn_dense(mu_J, nu_J, c_J, eps, SUB_TOL * max(mu_J.sum(), 1e-300), max_iter=5000000)
    if rc != 0:
        raise RuntimeError(f"cell Sinkhorn rc={rc} err={err}")
    pi = _plan(f, g, c_J, eps)
    pi[:, nu_J <= 0.0] = 0.0
    return pi


def sweep(inst: dict, pi: np.ndarray, parts) -> np.ndarray:
    """One half-iteration of Algorithm 1 over the composite partition
    `parts`: each cell J is re-solved with its X-marginal mu_J and the
    Y-marginal of the current plan on X_J."""
    out = pi.copy()
    for J in parts:
        J = np.asarray(J)
        nu_J = pi[J, :].sum(0)
        # Algorithm 1 assumes exact sub-solves, so ||nu_J|| = ||mu_J||; the
        # previous solves leave a mismatch at their tolerance (~1e-13), which
        # no coupling can absorb: rescale (the role of BalanceMeasures)
        nu_J = nu_J * (inst["mu"][J].sum() / nu_J.sum())
        out[J, :] = cell_solve(inst["mu"][J], nu_J, inst["c"][J, :], inst["eps"])
    return out


def kl(p: np.ndarray, q: np.ndarray) -> float:
    """KL(p|q) = sum p log(p/q) - p + q (0 log 0 = 0)."""
    m = p > 0
    return float(np.sum(p[m] * np.log(p[m] / q[m])) - p.sum() + q.sum())


def kl_to_kernel(pi: np.ndarray, inst: dict) -> float:
    """KL(pi|K), K = exp(-c/eps) mu (x) nu (reading A2)."""
    K = np.exp(-inst["c"] / inst["eps"]) * np.outer(inst["mu"], inst["nu"])
    return kl(pi, K)


def trace(inst: dict, sweeps: int, pistar: np.ndarray | None = None) -> dict:
    """Delta(pi^l) = KL(pi^l | pi*) for l = 0..sweeps (A first)."""
    if pistar is None:
        pistar = global_optimum(inst)
    pi = inst["pi0"].copy()
    deltas = [kl(pi, pistar)]
    for l in range(1, sweeps + 1):
        pi = sweep(inst, pi, inst["A"] if l % 2 == 1 else inst["B"])
        deltas.append(kl(pi, pistar))
    return dict(delta=np.array(deltas), pi=pi, pistar=pistar)


def fit_lambda(delta: np.ndarray, floor: float = 1e-13) -> dict:
    """Empirical contraction factor: exp of the least-squares slope of log
    Delta over the last half of the trace above the numerical floor (the
    paper fits the asymptotic slope of Figs. WorstCaseThreeEps/Q/N)."""
    d = np.asarray(delta, dtype=np.float64)
    idx = np.nonzero(d > floor * max(d[0], 1e-300))[0]
    last = idx[-1] if idx.size else 1
    seg = np.arange(max(1, last // 2), last + 1)
    if seg.size < 4:
        return dict(lam=float("nan"), r2=float("nan"), n=int(seg.size))
    y = np.log(d[seg])
    A = np.vstack([seg, np.ones_like(seg)]).T.astype(np.float64)
    coef, res, _, _ = np.linalg.lstsq(A, y, rcond=None)
    yhat = A @ coef
    ss = np.sum((y - y.mean()) ** 2)
    r2 = 1.0 - np.sum((y - yhat) ** 2) / ss if ss > 0 else 1.0
    return dict(lam=float(np.exp(coef[0])), r2=float(r2), n=int(seg.size), window=(int(seg[0]), int(seg[-1])))


def theorem1_factor(inst: dict) -> float:
    """(1 + exp(-2||c||/eps) ||mu_2|| / ||mu_{1,3}||)^-1 (eq. ThreeConvergenceKLDecrement)."""
    mu = inst["mu"]
    cn = float(np.max(np.abs(inst["c"])))
    return 1.0 / (1.0 + np.exp(-2.0 * cn / inst["eps"]) * mu[1] / (mu[0] + mu[2]))
