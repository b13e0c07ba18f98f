"""General separable costs c(x,y) = h1(|x1-y1|) + h2(|x2-y2|) (PAPER.md P:1528,
Sec. 7.1 "Test data": the scheme applies to costs h(x-y) with h strictly
convex).  Oracle pins (no GPU) against independent
references in tests/refs.py, and GPU parity (marked gpu) through the C-ABI.

The tables are anisotropic (h1 != h2) and non-quadratic, so an axis mix-up or
a quadratic leftover anywhere fails a pin."""
import numpy as np
import pytest

from ddinputs import gaussian_mixture_image, product_image
from oracle import Oracle
from refs import global_sinkhorn, sinkhorn_1d


def cost_tables(n):
    """h1(t) = |t|^1.5 (strictly convex on t >= 0 ... even extension), h2(t) = 2 t^2 + 4 |t|^3,
    t = d / n for finest-grid pixel differences d = 0..n-1 ([0,1]^2 units)."""
    t = np.arange(n) / n
    return t ** 1.5, 2.0 * t ** 2 + 4.0 * t ** 3


def dense_cost(n, h1, h2, side=None):
    """c[x, y] on the side x side grid (row-major pixels) from the finest-grid tables."""
    side = side or n
    st = n // side
    r = np.arange(side)
    D = np.abs(r[:, None] - r[None, :]) * st
    C1, C2 = h1[D], h2[D]            # [r_x, r_y], [c_x, c_y]
    return (C1[:, None, :, None] + C2[None, :, None, :]).reshape(side * side, side * side)


def _problem(n, seed=1):
    return gaussian_mixture_image(n, seed, 1), gaussian_mixture_image(n, seed + 1, 1)


def test_tables_equal_to_quadratic_reproduce_default():
    """h1 = h2 = t^2 must give the built-in |x-y|^2 path's result exactly."""
    n = 16
    mu, nu = _problem(n, 5)
    eps = 2 / n**2
    t = (np.arange(n) / n)
    a = Oracle(mu, nu, eps, 4)
    b = Oracle(mu, nu, eps, 4)
    b.set_cost(t**2, t**2)
    a.iterate(6)
    b.iterate(6)
    ca, cb = a.primal_cost(), b.primal_cost()
    assert abs(ca[0] - cb[0]) <= 1e-15 * ca[0] and abs(ca[1] - cb[1]) <= 1e-15 * abs(ca[1])


def test_single_cell_equals_global_sinkhorn_general_cost():
    """P6 with a general cost: one A-cell covering the 8x8 grid, one sweep = the
    independent dense global Sinkhorn with the same cost matrix."""
    n = 8
    mu, nu = _problem(n)
    h1, h2 = cost_tables(n)
    eps = 2 / n**2
    o = Oracle(mu, nu, eps, 4, err_tol=1e-14, no_truncate=True)
    o.set_cost(h1, h2)
    o.iterate(1)
    P = o.plan_dense()
    Pstar = global_sinkhorn(mu, nu, dense_cost(n, h1, h2), eps)
    assert np.abs(P - Pstar).sum() < 1e-12
    c_o, _ = o.primal_cost()
    assert abs(c_o - (dense_cost(n, h1, h2) * Pstar).sum()) < 1e-13


def test_dd_converges_to_global_optimum_general_cost():
    """P3 with a general cost: exact sub-solves, no truncation -> the global
    entropic optimum of the general-cost problem (Thm. 2), at a
    linear rate."""
    n = 16
    mu, nu = _problem(n, 3)
    h1, h2 = cost_tables(n)
    eps = 8 / n**2
    Pstar = global_sinkhorn(mu, nu, dense_cost(n, h1, h2), eps)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-13, no_truncate=True)
    o.set_cost(h1, h2)
    o.iterate(20)
    d20 = np.abs(o.plan_dense() - Pstar).sum()
    o.iterate(80)
    d100 = np.abs(o.plan_dense() - Pstar).sum()
    assert d100 < 1e-7 and d100 < 1e-3 * d20


def test_product_marginals_closed_form_general_cost():
    """P2 with an anisotropic separable cost: the optimum is pi1 (x) pi2 of the
    1D problems with costs h1 (rows) and h2 (columns); h1 != h2 pins the axes."""
    n, s = 16, 4
    mu, a1, a2 = product_image(n, 11)
    nu, b1, b2 = product_image(n, 12)
    h1, h2 = cost_tables(n)
    eps = 4 / n**2          # (t^1.5 is sharp at 0: 2 h^2 needs > 100 s of exact sub-solves)
    d = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    P1 = sinkhorn_1d(a1, b1, h1[d], eps)
    P2 = sinkhorn_1d(a2, b2, h2[d], eps)
    o = Oracle(mu, nu, eps, s, err_tol=1e-13, no_truncate=True)
    o.set_cost(h1, h2)
    o.iterate(60)
    D = o.basic_marginals_dense()
    nb = n // s
    for i in range(nb * nb):
        r, c = divmod(i, nb)
        ref = np.outer(P1[r * s:(r + 1) * s].sum(0), P2[c * s:(c + 1) * s].sum(0))
        assert np.abs(D[i] - ref.ravel()).sum() < 1e-10
    cost_o, _ = o.primal_cost()
    assert abs(cost_o - ((h1[d] * P1).sum() + (h2[d] * P2).sum())) < 1e-11


def test_transposition_swaps_the_axis_tables():
    """Transposing both images and swapping h1 <-> h2 is a relabelling of the
    same problem: same cost, same PD gap."""
    n = 16
    mu, nu = _problem(n, 7)
    h1, h2 = cost_tables(n)
    eps = 2 / n**2
    a = Oracle(mu, nu, eps, 4)
    a.set_cost(h1, h2)
    b = Oracle(np.ascontiguousarray(mu.T), np.ascontiguousarray(nu.T), eps, 4)
    b.set_cost(h2, h1)
    a.iterate(8)
    b.iterate(8)
    ca, cb = a.primal_cost(), b.primal_cost()
    assert abs(ca[0] - cb[0]) < 1e-7 * ca[0]
    assert abs(a.dual_gap()[2] - b.dual_gap()[2]) < 1e-6


def test_pd_gap_general_cost_weak_duality():
    """Prop. Duality (ii) with the general cost: gap >= 0, -> 0."""
    n = 16
    mu, nu = _problem(n, 9)
    h1, h2 = cost_tables(n)
    eps = 2 / n**2
    o = Oracle(mu, nu, eps, 4, err_tol=1e-10, no_truncate=True)
    o.set_cost(h1, h2)
    gaps = []
    for k in range(4):
        o.iterate(10)
        gaps.append(o.dual_gap()[2])
    assert all(g >= -1e-9 for g in gaps)        # primal plan feasible up to Err = 1e-10
    assert gaps[-1] < 1e-3 * gaps[0] or gaps[-1] < 1e-9


def test_set_cost_validation():
    n = 16
    mu, nu = _problem(n)
    o = Oracle(mu, nu, 2 / n**2, 4)
    with pytest.raises(RuntimeError):
        o.set_cost(np.zeros(n - 1), np.zeros(n - 1))
    h1, h2 = cost_tables(n)
    h1 = h1.copy()
    h1[3] = np.nan
    with pytest.raises(RuntimeError):
        o.set_cost(h1, h2)


# ------------------------------------------------------------------- GPU --
@pytest.fixture(scope="module")
def DD():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD as _DD
    return _DD


def _mass_i(mu, s):
    nb = mu.shape[0] // s
    return mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()


@pytest.mark.gpu
def test_gpu_general_cost_sweeps_vs_oracle(DD):
    """32^2, s = 4, eps = 2 h^2 with the anisotropic non-quadratic tables:
    per-sweep basic-cell marginals (P9) and the final gates."""
    from ddinputs import config_images
    n, s = 32, 4
    mu, nu = config_images(1)
    h1, h2 = cost_tables(n)
    eps = 2.0 / n**2
    g = DD(mu, nu, eps, s, err_tol=1e-6)
    o = Oracle(mu, nu, eps, s, err_tol=1e-6)
    g.set_cost(h1, h2)
    o.set_cost(h1, h2)
    mass = _mass_i(mu, s)
    for sweep in range(8):
        g.iterate(1)
        o.iterate(1)
        Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
        diff = np.abs(Dg - Do).sum(1)
        assert (diff <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, diff.max())
        assert np.abs(Dg.sum(0) - nu.ravel()).sum() < 1e-11
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
    assert g.stats()["failed"] == 0


@pytest.mark.gpu
def test_gpu_general_cost_ladder_vs_oracle(DD):
    """The cfg-2 ladder (16^2 -> 64^2, eps from 1.0 to 0.5 h^2) with the
    general cost, both warm-started the same way: final cost, marginals and
    the PD gap (glued dual with the general cost on both sides)."""
    from ddinputs import config_images
    from oracle.oracle import SCHED_LADDER as O_LADDER
    n = 64
    mu, nu = config_images(2)
    # smooth strictly convex anisotropic tables (curvature bounded below: the
    # ladder's Sinkhorn converges as for |x-y|^2; t^1.5 needs > 10^4 its at 0.5 h^2)
    t = np.arange(n) / n
    h1, h2 = 1.5 * t**2 + 2.0 * t**4, 0.75 * t**2 + 2.0 * t**3
    eps = 0.5 / n**2
    g = DD(mu, nu, eps, 4, schedule=1, err_tol=1e-6, eps_start=1.0, coarsest_side=16)
    o = Oracle(mu, nu, eps, 4, schedule=O_LADDER, err_tol=1e-6, eps_start=1.0, coarsest_side=16,
               warm_refine=True)
    g.set_cost(h1, h2)
    o.set_cost(h1, h2)
    g.run_schedule()
    o.run_schedule()
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
    rg = g.dual_gap()[2]
    ro = o.dual_gap()[2]
    assert -1e-7 < rg < 1e-3 and abs(rg - ro) <= 1e-4 + 0.5 * abs(ro), (rg, ro)


@pytest.mark.gpu
def test_gpu_general_cost_pd_gap_same_state(DD):
    """The oracle's state imported into the GPU library: primal score and
    glued dual objective with the general cost agree to 1e-10 (evaluation
    kernels K7 and k_dual with the tables)."""
    from ddinputs import config_images
    n = 32
    mu, nu = config_images(1)
    h1, h2 = cost_tables(n)
    eps = 2.0 / n**2
    o = Oracle(mu, nu, eps, 4, err_tol=1e-8)
    o.set_cost(h1, h2)
    o.iterate(6)
    Po, Do, ro = o.dual_gap()
    g = DD(mu, nu, eps, 4, err_tol=1e-8)
    g.set_cost(h1, h2)
    g.set_state(o.get_state())
    Pg, Dg, rg = g.dual_gap()
    assert abs(Pg - Po) <= 1e-10 * abs(Po)
    assert abs(Dg - Do) <= 1e-10 * abs(Do)
    assert g.primal_cost()[0] == pytest.approx(o.primal_cost()[0], rel=1e-12)


@pytest.mark.gpu
def test_gpu_quadratic_tables_match_builtin_path(DD):
    """h1 = h2 = t^2 through the table path (no shifted gauge) agrees with the
    built-in quadratic path to the fp32 floor."""
    from ddinputs import config_images
    n = 32
    mu, nu = config_images(1)
    t = np.arange(n) / n
    eps = 2.0 / n**2
    a = DD(mu, nu, eps, 4, err_tol=1e-6)
    b = DD(mu, nu, eps, 4, err_tol=1e-6)
    b.set_cost(t**2, t**2)
    a.iterate(8)
    b.iterate(8)
    ca, cb = a.primal_cost()[0], b.primal_cost()[0]
    assert abs(ca - cb) <= 2e-7 * ca
    assert np.abs(a.basic_marginals_dense() - b.basic_marginals_dense()).sum() <= 4e-6


@pytest.mark.gpu
@pytest.mark.parametrize("kappa", [2.0])
def test_gpu_cell_size_16_vs_oracle(DD, kappa):
    """s = 16 (the paper's cell-size study): composite X cells of
    32 x 32 px (A: the whole grid; B: 16 x 32 edges, 16 x 16 corners) on the
    SMEM tier; GPU vs oracle sweeps at 32^2 (64^2 costs the dense oracle
    ~13 min)."""
    n, s = 32, 16
    mu, nu = gaussian_mixture_image(n, 41, 3), gaussian_mixture_image(n, 42, 3)
    eps = kappa / n**2
    g = DD(mu, nu, eps, s, err_tol=1e-6)
    o = Oracle(mu, nu, eps, s, err_tol=1e-6)
    mass = _mass_i(mu, s)
    for sweep in range(4):
        g.iterate(1)
        o.iterate(1)
        diff = np.abs(g.basic_marginals_dense() - o.basic_marginals_dense()).sum(1)
        assert (diff <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, diff.max())
    cg, co = g.primal_cost()[0], o.primal_cost()[0]
    assert abs(cg - co) <= 1e-5 * co
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
