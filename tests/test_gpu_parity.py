"""GPU (B200) parity: the CUDA path through the C-ABI vs the fp64 CPU oracle on
the same seeded inputs.  Gates (BASELINE.json north_star):
relative primal transport cost <= 1e-5, GPU marginal L1 errors <= 1e-6.

Tolerances derived in DESIGN.md "Parity tolerances": per composite cell the
GPU's fp32 Sinkhorn floors at ~1e-7 relative in the plan, the oracle's fp64 at
~1e-14; both stop at Err = 1e-6 in the L1 X-error, so two correct solves of
the same cell problem differ by at most ~2 Err ||mu_J|| in L1."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import config_images, gaussian_mixture_image, product_image  # noqa: E402
from oracle import Oracle  # noqa: E402
from oracle.oracle import SCHED_LADDER as O_LADDER  # noqa: E402


@pytest.fixture(scope="module")
def DD():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD as _DD
    return _DD


def _mass_i(mu, s):
    n = mu.shape[0]
    nb = n // s
    return mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()


def test_device_and_library(DD):
    import torch
    from paper_2001_10986_b200 import lib
    assert torch.cuda.get_device_capability(0)[0] == 10
    assert lib().dd_version().decode().startswith("ddot-b200")


def test_single_sweep_parity_from_product_state(DD):
    """Same input state (product coupling) -> one A-sweep and one B-sweep on both;
    compare every basic-cell marginal nu_i (the paper's state)."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    g = DD(mu, nu, eps, 4, err_tol=1e-6)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-6)
    mass = _mass_i(mu, 4)
    for sweep in range(2):
        g.iterate(1)
        o.iterate(1)
        Dg = g.basic_marginals_dense()
        Do = o.basic_marginals_dense()
        diff = np.abs(Dg - Do).sum(1)
        # per basic cell: |nu_i^gpu - nu_i^ora|_1 <= 2 Err ||mu_J|| (both within Err of the cell optimum)
        assert (diff <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, diff.max())
        assert np.abs(Dg - Do).sum() <= 4e-6
        # the paper's invariants on the GPU state
        assert np.abs(Dg.sum(0) - nu.ravel()).sum() < 1e-11
        np.testing.assert_allclose(Dg.sum(1), mass, rtol=1e-10, atol=1e-12)
    sg, so = g.stats(), o.stats()
    assert sg["cells"] == so["cells"] == 25
    assert sg["err_x_sum"] <= 1e-6 * 1.0001


def test_trajectory_parity_cfg1(DD):
    """Config 1 (32^2, s = 4, kappa = 2 fixed): 16 sweeps on both."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    g = DD(mu, nu, eps, 4, err_tol=1e-6)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-6)
    g.iterate(16)
    o.iterate(16)
    cg, eg = g.primal_cost()
    co, eo = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co
    assert abs(eg - eo) <= 1e-5 * abs(eo)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
    lxo, _ = o.marginal_error()
    st = g.totals()
    sto = o.stats()
    assert st["cells"] == 8 * 16 + 8 * 25
    # iteration counts agree within a few percent (stop tests in fp32 vs fp64)
    assert abs(g.stats()["iters_sum"] - sto["iters_sum"]) <= 0.1 * sto["iters_sum"] + 20


def test_plan_parity_small(DD):
    """COO plans of the last sweep agree entrywise (L1) on a 16^2 problem."""
    mu, nu = gaussian_mixture_image(16, 3, 1), gaussian_mixture_image(16, 4, 1)
    eps = 2.0 / 16**2
    g = DD(mu, nu, eps, 4, err_tol=1e-7)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-7)
    g.iterate(8)
    o.iterate(8)
    Pg, Po = g.plan_dense(), o.plan_dense()
    assert np.abs(Pg - Po).sum() <= 1e-6
    assert np.abs(Pg.sum(0) - nu.ravel()).sum() <= 1e-6
    assert np.abs(Pg.sum(1) - mu.ravel()).sum() <= 1e-6


def test_ladder_parity_cfg2(DD):
    """Config 2: 64^2, coarse-to-fine from 16^2 with eps from 1.0 to 0.5 h^2."""
    mu, nu = config_images(2)
    eps = 0.5 / 64**2
    kw = dict(err_tol=1e-6, eps_start=1.0, coarsest_side=16)
    g = DD(mu, nu, eps, 4, schedule=1, **kw)
    o = Oracle(mu, nu, eps, 4, schedule=O_LADDER, **kw)
    g.run_schedule()
    o.run_schedule()
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6, (lx, ly)
    assert g.state_info()["half_index"] == o.state_info()["half_index"] == 38


@pytest.mark.parametrize("n,s,kappa", [(8, 4, 2.0), (16, 4, 0.5), (16, 8, 1.0), (64, 8, 2.0)])
def test_edge_geometries(DD, n, s, kappa):
    """Degenerate partitions: one A-cell (n = 2s), B corner singletons,
    2x1 edge cells, s = 8 composite cells; both sweeps, several sweeps."""
    mu, nu = gaussian_mixture_image(n, 5, 1), gaussian_mixture_image(n, 6, 1)
    eps = kappa / n**2
    g = DD(mu, nu, eps, s)
    o = Oracle(mu, nu, eps, s)
    g.iterate(4)
    o.iterate(4)
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6


def test_no_truncation_exact_mode(DD):
    """tau = 0 and tight Err: GPU reaches its fp32 floor, still <= 1e-6 from the oracle."""
    mu, nu = gaussian_mixture_image(16, 7, 1), gaussian_mixture_image(16, 8, 1)
    eps = 2.0 / 16**2
    g = DD(mu, nu, eps, 4, err_tol=1e-7, no_truncate=True)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-7, no_truncate=True)
    g.iterate(10)
    o.iterate(10)
    Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
    assert np.abs(Dg - Do).sum() <= 1e-6


def test_set_state_roundtrip(DD):
    """The oracle's exported state imported into the GPU library gives the same
    next sweep (state import path of DESIGN.md single-sweep parity)."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    o = Oracle(mu, nu, eps, 4)
    o.iterate(3)
    st = o.get_state()
    g = DD(mu, nu, eps, 4)
    g.set_state(st)
    back = g.get_state()
    assert np.array_equal(back["boxes"], st["boxes"])
    assert np.array_equal(back["values"], st["values"])
    g.iterate(1)
    o.iterate(1)
    assert np.abs(g.basic_marginals_dense() - o.basic_marginals_dense()).sum() <= 4e-6


def test_validation_errors_gpu(DD):
    mu = np.full((16, 16), 1 / 256)
    with pytest.raises(ValueError):
        DD(mu, mu * 1.01, 1.0, 4)
    with pytest.raises(ValueError):
        DD(mu, mu, 1.0, 16)


@pytest.mark.parametrize("bcap_main,bcap_big", [(10, 0), (10, 12)])
def test_big_tier_parity_cfg1(DD, bcap_main, bcap_big):
    """The fused Y2+X1 path (K1 tiers 1 and 2) vs the oracle: routing every
    cell with a union Y box > 10 px away from the SMEM tier (and, with
    bcap_big = 12, everything beyond 12 px to the 512-thread tier)."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    g = DD(mu, nu, eps, 4, err_tol=1e-6, bcap_main=bcap_main, bcap_big=bcap_big)
    o = Oracle(mu, nu, eps, 4, err_tol=1e-6)
    mass = _mass_i(mu, 4)
    for sweep in range(2):
        g.iterate(1)
        o.iterate(1)
        Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
        diff = np.abs(Dg - Do).sum(1)
        assert (diff <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, diff.max())
        assert np.abs(Dg.sum(0) - nu.ravel()).sum() < 1e-11
        np.testing.assert_allclose(Dg.sum(1), mass, rtol=1e-10, atol=1e-12)
    g.iterate(10)
    o.iterate(10)
    assert g.totals()["big_cells"] > 0
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6, (lx, ly)


@pytest.mark.parametrize("bcap_big", [0, 40])
def test_big_tier_parity_s8(DD, bcap_big):
    """s = 8 composite cells (16 x 16 X boxes, 16 x 8 edges, 8 x 8 corners) on
    the fused path: 32^2, kappa = 0.5, all cells off the SMEM tier."""
    n, s = 32, 8
    mu, nu = gaussian_mixture_image(n, 11, 3), gaussian_mixture_image(n, 12, 3)
    eps = 0.5 / n**2
    g = DD(mu, nu, eps, s, err_tol=1e-6, bcap_main=18, bcap_big=bcap_big)
    o = Oracle(mu, nu, eps, s, err_tol=1e-6)
    g.iterate(6)
    o.iterate(6)
    assert g.totals()["big_cells"] > 0
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6, (lx, ly)
    Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
    assert np.abs(Dg - Do).sum() <= 1e-5


@pytest.mark.parametrize("sweeps", [3, 12])
def test_pd_gap_parity(DD, sweeps):
    """Relative PD gap of eq. RelPDGap (f1): the oracle's state
    imported into the GPU library gives the same primal score, glued dual
    objective and gap (same state: only the evaluation arithmetic differs)."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    o = Oracle(mu, nu, eps, 4, err_tol=1e-8)
    o.iterate(sweeps)
    Po, Do, ro = o.dual_gap()
    g = DD(mu, nu, eps, 4, err_tol=1e-8)
    g.set_state(o.get_state())
    Pg, Dg, rg = g.dual_gap()
    assert abs(Pg - Po) <= 1e-10 * abs(Po)
    assert abs(Dg - Do) <= 1e-10 * abs(Do)
    assert abs(rg - ro) <= 1e-9 + 1e-4 * abs(ro)
    assert rg > -1e-8


def test_pd_gap_after_ladder_cfg2(DD):
    """After the cfg-2 ladder the glued dual candidate certifies the GPU
    iterate: small non-negative relative PD gap (P:1713-1717 reports ~1e-4 at
    Err = 1e-4; here Err = 1e-6)."""
    mu, nu = config_images(2)
    g = DD(mu, nu, 0.5 / 64**2, 4, schedule=1, err_tol=1e-6, eps_start=1.0, coarsest_side=16)
    g.run_schedule()
    P, D, rel = g.dual_gap()
    assert -1e-7 < rel < 1e-3, rel


def test_paper_schedule_kappa_quarter(DD):
    """The paper's own tail: +2 sweeps at eps = 0.25 dx^2 on the
    finest layer ((n-2)*8+2 sweeps), on the GPU vs the oracle."""
    n = 64
    mu, nu = gaussian_mixture_image(n, 31, 3), gaussian_mixture_image(n, 32, 3)
    eps = 0.25 / n**2
    g = DD(mu, nu, eps, 4, schedule=1, coarsest_side=8)
    o = Oracle(mu, nu, eps, 4, schedule=O_LADDER, coarsest_side=8)
    g.run_schedule()
    o.run_schedule()
    assert g.state_info()["half_index"] == o.state_info()["half_index"] == (6 - 2) * 8 + 2
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6


def test_ladder_s8_big_tiers_128(DD):
    """cfg-4 recipe (s = 8, anisotropic mixtures) at 128^2 through the whole
    ladder with every cell above 18 px on the fused big-cell tiers."""
    n = 128
    mu, nu = gaussian_mixture_image(n, 41, 4), gaussian_mixture_image(n, 42, 4)
    eps = 0.5 / n**2
    g = DD(mu, nu, eps, 8, schedule=1, coarsest_side=8, bcap_main=18)
    o = Oracle(mu, nu, eps, 8, schedule=O_LADDER, coarsest_side=8)
    g.run_schedule()
    o.run_schedule()
    assert g.totals()["big_cells"] > 0
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6


@pytest.mark.parametrize("dm,ds", [(5e-6, 0.0), (0.0, 1e-3), (2e-6, 1e-4)])
def test_l1y_known_deviation_gpu_vs_oracle(DD, dm, ds):
    """A state of known Y-deviation (tests/test_oracle_pins.py): GPU l1_y =
    oracle l1_y = the closed form, after the same import."""
    from test_oracle_pins import _perturbed_product_state
    mu, nu, st, dev = _perturbed_product_state(dm, ds)
    want = np.abs(dev).sum()
    g = DD(mu, nu, 2.0 / 32**2, 4)
    g.set_state(st)
    o = Oracle(mu, nu, 2.0 / 32**2, 4, empty_init=True)
    o.set_state(st)
    _, lyg = g.marginal_error()
    _, lyo = o.marginal_error()
    assert abs(lyg - want) <= 1e-13 + 1e-9 * want, (lyg, want)
    assert abs(lyg - lyo) <= 1e-13 + 1e-9 * want


def test_l1y_after_ladder_gpu_vs_oracle(DD):
    """l1_y of the GPU's own state vs the oracle's evaluation of the same state."""
    mu, nu = config_images(2)
    g = DD(mu, nu, 0.5 / 64**2, 4, schedule=1, coarsest_side=16, eps_start=1.0)
    g.run_schedule()
    st = g.get_state()
    o = Oracle(mu, nu, 0.5 / 64**2, 4, empty_init=True)
    o.set_state(st)
    lxg, lyg = g.marginal_error()
    lxo, lyo = o.marginal_error()
    assert abs(lyg - lyo) <= 1e-15 + 1e-9 * lyo, (lyg, lyo)
    assert abs(lxg - lxo) <= 1e-9 + 1e-6 * lxo, (lxg, lxo)
    assert lyg <= 1e-6 and lxg <= 1e-6


def test_pool_overflow_reports_enomem(DD):
    """A pool too small for the refined state: the refinement flags it
    (no out-of-bounds reads), dd_synchronize returns DD_ENOMEM."""
    mu, nu = config_images(2)
    g = DD(mu, nu, 0.5 / 64**2, 4, schedule=1, coarsest_side=16, pool_capacity=16 * 16 * 16 * 16 + 64)
    with pytest.raises(RuntimeError, match="rc=6"):
        g.run_schedule()


def test_warm_refine_k5_vs_oracle(DD):
    """K5 (glue + log-space interpolation) vs the oracle's
    warm_refine on the same imported coarse state: the fine potentials of
    both partitions agree (fp64 on both sides; CG tolerances)."""
    from oracle.oracle import SCHED_LADDER as OL
    mu, nu = config_images(2)
    n = 64
    o = Oracle(mu, nu, 0.5 / n**2, 4, schedule=OL, coarsest_side=32, warm_refine=True)
    o.set_eps(1.0 / 32**2)
    o.iterate(6)
    st = o.get_state()
    g = DD(mu, nu, 0.5 / n**2, 4, schedule=1, coarsest_side=32)
    g.set_eps(1.0 / 32**2)
    g.set_state(st)
    g.refine()
    o.refine()
    a, b = g.get_state(), o.get_state()
    scale = np.abs(b["alpha_A"]).max()
    for key in ("alpha_A", "alpha_B"):
        d = a[key] - b[key]
        d -= d.mean()                     # the glued potential's global constant is a gauge
        assert np.abs(d).max() <= 1e-9 * max(scale, 1e-12), (key, np.abs(d).max(), scale)


def test_ladder_parity_both_warm_cfg2(DD):
    """cfg-2 ladder with the paper's warm start on BOTH sides (GPU K5 default,
    oracle warm_refine): the BASELINE gates."""
    from oracle.oracle import SCHED_LADDER as OL
    mu, nu = config_images(2)
    n = 64
    g = DD(mu, nu, 0.5 / n**2, 4, schedule=1, coarsest_side=16, eps_start=1.0)
    o = Oracle(mu, nu, 0.5 / n**2, 4, schedule=OL, coarsest_side=16, eps_start=1.0, warm_refine=True)
    g.run_schedule()
    o.run_schedule()
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6
    Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
    assert np.abs(Dg - Do).sum() <= 4e-6     # sum_J 2 Err ||mu_J|| (P9, different stop iterations)
