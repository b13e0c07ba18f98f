"""Tier G (SURVEY.md 8(f) f2 "tiled fallback"): cells whose
union Y box exceeds every on-chip K1 tier run the SMEM-tier kernel on a
per-CTA global-memory layout instead of failing with DD_ENOMEM.  Same code as
tier 0, so the same cell gives the same bits on either; parity with the
oracle as for every tier."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import config_images, gaussian_mixture_image  # noqa: E402
from oracle import Oracle  # noqa: E402


@pytest.fixture(scope="module")
def DD():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD as _DD
    return _DD


def _same_state(a, b):
    for k in ("boxes", "offsets", "values", "alpha_A", "alpha_B"):
        assert np.array_equal(a[k], b[k]), k


def test_tier_g_bit_identical_to_tier_0(DD):
    """cfg 1 (32^2, s = 4, kappa = 2): every cell on tier 0 (bcap_main = 40)
    vs every cell beyond 10 px on tier G (bcap_main = 10, on-chip cap 10):
    identical states after 6 sweeps."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    a = DD(mu, nu, eps, 4, err_tol=1e-6, bcap_main=40)
    b = DD(mu, nu, eps, 4, err_tol=1e-6, bcap_main=10, bcap_onchip=10)
    a.iterate(6)
    b.iterate(6)
    assert a.totals()["big_cells"] == 0
    _same_state(a.get_state(), b.get_state())
    assert a.primal_cost() == b.primal_cost()


def test_tier_g_ladder_vs_oracle(DD):
    """The cfg-2 ladder with every cell above 12 px on tier G, against the
    oracle (both glued warm starts): cost, marginals."""
    from oracle.oracle import SCHED_LADDER as O_LADDER
    mu, nu = config_images(2)
    n = 64
    eps = 0.5 / n**2
    g = DD(mu, nu, eps, 4, schedule=1, err_tol=1e-6, eps_start=1.0, coarsest_side=16, bcap_main=12,
           bcap_onchip=12)
    o = Oracle(mu, nu, eps, 4, schedule=O_LADDER, err_tol=1e-6, eps_start=1.0, coarsest_side=16, warm_refine=True)
    g.run_schedule()
    o.run_schedule()
    cg, co = g.primal_cost()[0], o.primal_cost()[0]
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6


def test_tier_g_general_cost_whole_image_boxes(DD):
    """A nearly flat general cost keeps the product coupling's whole-image
    boxes (128 px > the SMEM tier's general-cost capacity for s = 4): the
    cells run on tier G and match the oracle."""
    n, s = 128, 4
    mu, nu = gaussian_mixture_image(n, 5, 3), gaussian_mixture_image(n, 6, 3)
    t = np.arange(n) / n
    h = 1e-4 * t**2
    eps = 2.0 / n**2
    g = DD(mu, nu, eps, s, err_tol=1e-6)
    o = Oracle(mu, nu, eps, s, err_tol=1e-6)
    g.set_cost(h, h)
    o.set_cost(h, h)
    g.iterate(1)
    o.iterate(1)
    assert g.totals()["max_box"] == n
    d = np.abs(g.basic_marginals_dense() - o.basic_marginals_dense()).sum()
    assert d <= 2e-6, d
    cg, co = g.primal_cost()[0], o.primal_cost()[0]
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    assert g.synchronize() == 0
