"""K1 cluster tier: one composite cell solved by a
thread-block cluster of CTAs that share its state through DSMEM.

The fused big-cell path's arithmetic does not depend on the CTA shape or the
cluster size (fixed X2 split, fixed-order error and norm sums), so tier 1
(256 threads), tier 2 (768 threads) and the cluster tier (kClusterSize CTAs of
768 threads) must agree BIT FOR BIT on every cell; the routing between them
(box side, the long-pole threshold) then only changes timing.  Parity of the
cluster tier with the oracle is checked directly as well."""
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


from paper_2001_10986_b200.dd import NotConverged  # noqa: E402


def _same_state(a, b):
    for k in ("boxes", "offsets", "values", "alpha_A", "alpha_B"):
        assert a[k].shape == b[k].shape, k
        assert np.array_equal(a[k], b[k]), (k, np.abs(a[k] - b[k]).max() if a[k].dtype.kind == "f" else None)


def test_tiers_bit_identical_ladder_128(DD):
    """cfg-4 recipe (s = 8) at 128^2, full ladder: big-path cells by box side
    (tiers 1 / 2), all on tier 2, all on the cluster tier, auto routing."""
    n = 128
    mu, nu = gaussian_mixture_image(n, 41, 4), gaussian_mixture_image(n, 42, 4)
    eps = 0.5 / n**2
    runs = {}
    for name, kw in (("by_side", dict(cluster=-1)), ("tier2", dict(cluster=-1, bcap_big=19)),
                     ("cluster", dict(cluster=1)), ("auto", dict(cluster=2, cluster_theta=50))):
        g = DD(mu, nu, eps, 8, schedule=1, coarsest_side=8, bcap_main=18, **kw)
        g.run_schedule()
        runs[name] = (g.get_state(), g.totals())
    ref, tref = runs["by_side"]
    assert tref["big_cells"] > 0 and tref["cluster_cells"] == 0
    assert runs["tier2"][1]["cluster_cells"] == 0
    assert runs["cluster"][1]["cluster_cells"] == tref["big_cells"]
    for name in ("tier2", "cluster", "auto"):
        _same_state(ref, runs[name][0])
        assert runs[name][1]["iters_sum"] == tref["iters_sum"], name


@pytest.mark.parametrize("s,bcap_main", [(4, 10), (8, 18)])
def test_cluster_tier_parity_vs_oracle(DD, s, bcap_main):
    """Every cell above bcap_main px on the cluster tier vs the fp64 oracle
    (cfg-1 images at 32^2, kappa = 2; s = 8 has the 16 x 8 edge and 8 x 8
    corner cells), 8 sweeps."""
    mu, nu = config_images(1)
    n = 32
    eps = 2.0 / n**2
    g = DD(mu, nu, eps, s, err_tol=1e-6, bcap_main=bcap_main, cluster=1)
    o = Oracle(mu, nu, eps, s, err_tol=1e-6)
    nb = n // s
    mass = mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()
    for sweep in range(2):
        g.iterate(1)
        o.iterate(1)
        Dg, Do = g.basic_marginals_dense(), o.basic_marginals_dense()
        diff = np.abs(Dg - Do).sum(1)
        assert (diff <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, diff.max())
        assert np.abs(Dg.sum(0) - nu.ravel()).sum() < 1e-11
    g.iterate(6)
    o.iterate(6)
    t = g.totals()
    assert t["cluster_cells"] > 0 and t["cluster_cells"] == t["big_cells"]
    cg, _ = g.primal_cost()
    co, _ = o.primal_cost()
    assert abs(cg - co) <= 1e-5 * co, (cg, co)
    lx, ly = g.marginal_error()
    assert lx <= 1e-6 and ly <= 1e-6, (lx, ly)


def test_cluster_auto_routing_cfg4_bit_identical(DD):
    """cfg 4 (1024^2, s = 8, full ladder): the automatic long-pole routing
    sends cells to the cluster tier and the final state equals the run with
    the cluster tier off bit for bit."""
    mu, nu = config_images(4)
    n = 1024
    eps = 0.5 / n**2
    out = {}
    for name, cl in (("off", 0), ("auto", 2)):
        g = DD(mu, nu, eps, 8, schedule=1, coarsest_side=8, cluster=cl, max_inner_iter=100000)
        try:
            g.run_schedule()
        except NotConverged:
            pass        # a few border cells of cfg 4 are flagged (reading A6); compared bitwise all the same
        out[name] = (g.get_state(), g.totals())
        del g
    assert out["auto"][1]["cluster_cells"] > 0
    assert out["off"][1]["cluster_cells"] == 0
    _same_state(out["off"][0], out["auto"][0])
