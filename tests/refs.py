"""Independent numpy references used to PIN the oracle (test-side only).

These are textbook formulas written directly from the paper's definitions,
deliberately in a different form than oracle/dd_oracle.c (scaling domain /
scipy logsumexp on the full global problem), so that a mistake in the oracle
(dropped term, wrong sign, transposed operand) shows up as a mismatch.
"""
from __future__ import annotations

import numpy as np
from scipy.special import logsumexp


def grid_cost(n: int) -> np.ndarray:
    """c(x,y) = |x-y|^2 on the n x n grid of [0,1]^2 pixel centres."""
    t = (np.arange(n) + 0.5) / n
    p1, p2 = np.meshgrid(t, t, indexing="ij")
    P = np.stack([p1.ravel(), p2.ravel()], axis=1)
    d = P[:, None, :] - P[None, :, :]
    return (d ** 2).sum(-1)


def global_sinkhorn(mu: np.ndarray, nu: np.ndarray, cost: np.ndarray, eps: float,
                    tol: float = 1e-14, max_iter: int = 200000) -> np.ndarray:
    """Plain global log-domain Sinkhorn (Remark Sinkhorn): the
    unique optimum pi* of eps KL(pi | K), K = exp(-c/eps) mu (x) nu."""
    a = mu.ravel()
    b = nu.ravel()
    la, lb = np.log(a), np.log(b)
    f = np.zeros_like(a)
    g = np.zeros_like(b)
    for _ in range(max_iter):
        g = eps * lb - eps * logsumexp((f[:, None] - cost) / eps, axis=0)
        f = eps * la - eps * logsumexp((g[None, :] - cost) / eps, axis=1)
        P = np.exp((f[:, None] + g[None, :] - cost) / eps)
        if np.abs(P.sum(0) - b).sum() < tol:
            break
    return P


def sinkhorn_1d(a, b, cost, eps, tol=1e-15, max_iter=1000000):
    """1D scaling-domain Sinkhorn (u, v form of Remark Sinkhorn) for pin P2."""
    K = np.exp(-cost / eps)
    u = np.ones_like(a)
    v = np.ones_like(b)
    for _ in range(max_iter):
        v = b / (K.T @ u)
        u = a / (K @ v)
        P = u[:, None] * K * v[None, :]
        if np.abs(P.sum(0) - b).sum() + np.abs(P.sum(1) - a).sum() < tol:
            break
    return u[:, None] * K * v[None, :]


def kl(p: np.ndarray, q: np.ndarray) -> float:
    """KL(p|q) = sum phi(p/q) q (Def. KL) for q > 0."""
    m = p > 0
    return float((p[m] * np.log(p[m] / q[m])).sum() - p.sum() + q.sum())


def quadratic_2x2(a1, a2, b1, b2, c, eps):
    """Closed form of the 2x2 entropic optimum (pin P1b).

    pi = [[t, a1-t], [b1-t, a2-b1+t]] and the scaling form (Prop.
    EntropicOTBasic (ii)) forces pi11 pi22 / (pi12 pi21) = rho with
    rho = exp(-(c11 + c22 - c12 - c21)/eps)."""
    rho = np.exp(-(c[0, 0] + c[1, 1] - c[0, 1] - c[1, 0]) / eps)
    A = 1.0 - rho
    B = a2 - b1 + rho * (a1 + b1)
    Cq = -rho * a1 * b1
    lo, hi = max(0.0, b1 - a2), min(a1, b1)
    if abs(A) < 1e-300:
        t = -Cq / B
    else:
        disc = np.sqrt(B * B - 4 * A * Cq)
        roots = [(-B + disc) / (2 * A), (-B - disc) / (2 * A)]
        t = [r for r in roots if lo - 1e-15 <= r <= hi + 1e-15][0]
    return np.array([[t, a1 - t], [b1 - t, a2 - b1 + t]])
