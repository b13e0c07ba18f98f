"""The eps-raising safeguard (Sec. 7.3: "localized to small
problems on composite cells which are easy to fix (e.g. by temporarily
increasing eps). We have implemented a corresponding safe-guard"
retry at 2x eps and re-solve at the target eps, S:323 at most 3 attempts;
DESIGN.md reading A29).  Oracle pins on CPU, GPU parity marked gpu.

Forcing it: config 1 (32^2, s = 4) at kappa = 2 from the product coupling
needs ~250-480 Sinkhorn iterations per cell; a cap of 200 makes every cell of
the first sweep fail without the safeguard, and none with it."""
import numpy as np
import pytest

from ddinputs import config_images
from oracle import Oracle

N, S, KAPPA, CAP = 32, 4, 2.0, 200


def _mass_i(mu, s):
    nb = mu.shape[0] // s
    return mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()


def test_safeguard_recovers_capped_cells():
    mu, nu = config_images(1)
    eps = KAPPA / N**2
    plain = Oracle(mu, nu, eps, S, max_inner_iter=CAP)
    safe = Oracle(mu, nu, eps, S, max_inner_iter=CAP, safeguard=True)
    plain.iterate(1)
    safe.iterate(1)
    sp, ss = plain.stats(), safe.stats()
    assert sp["failed"] == 16 and sp["safeguarded"] == 0
    assert ss["failed"] == 0 and ss["safeguarded"] == 16
    # the X-error bound of P:1409 holds again
    assert ss["err_x_sum"] <= 1e-6 < sp["err_x_sum"]


def test_safeguard_gives_the_cell_optimum():
    """The safeguard changes only the path: each retried cell ends at the
    unique optimum of its cell problem, i.e. within 2 Err ||mu_J|| of a
    direct solve with a cap large enough not to fire."""
    mu, nu = config_images(1)
    eps = KAPPA / N**2
    ref = Oracle(mu, nu, eps, S, max_inner_iter=2000)
    safe = Oracle(mu, nu, eps, S, max_inner_iter=CAP, safeguard=True)
    ref.iterate(1)
    safe.iterate(1)
    assert ref.stats()["failed"] == 0
    d = np.abs(ref.basic_marginals_dense() - safe.basic_marginals_dense()).sum(1)
    # both within Err ||mu_J|| of the cell optimum in L1: summed over
    # the 16 A-cells (total mass 1) the two states differ by <= 2 Err
    assert d.sum() <= 2e-6, d.sum()


def test_safeguard_idle_is_identity():
    """When no cell fails the safeguard never runs: bit-identical results."""
    mu, nu = config_images(1)
    eps = KAPPA / N**2
    a = Oracle(mu, nu, eps, S)
    b = Oracle(mu, nu, eps, S, safeguard=True)
    a.iterate(3)
    b.iterate(3)
    assert b.stats()["safeguarded"] == 0
    assert a.primal_cost() == b.primal_cost()
    assert np.array_equal(a.basic_marginals_dense(), b.basic_marginals_dense())


def test_safeguard_exhausted_still_flags():
    """Three attempts that cannot converge (cap 5): the cell stays
    flagged (reading A6), the state Y-feasible."""
    mu, nu = config_images(1)
    eps = KAPPA / N**2
    o = Oracle(mu, nu, eps, S, max_inner_iter=5, safeguard=True)
    o.iterate(1)
    st = o.stats()
    assert st["failed"] == 16 and st["safeguarded"] == 16
    D = o.basic_marginals_dense()
    assert np.abs(D.sum(0) - nu.ravel()).sum() < 1e-11


# ------------------------------------------------------------------- GPU --
@pytest.fixture(scope="module")
def DD():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD as _DD
    return _DD


@pytest.mark.gpu
def test_gpu_safeguard_vs_oracle(DD):
    """K1's safeguard (fp64 stages at 2^k eps, DD_FLAG_SAFEGUARD) against the
    oracle's on the forced configuration: every cell retried (CellOut flag 32),
    none failed, marginals within the P9 bound, then two more sweeps."""
    mu, nu = config_images(1)
    eps = KAPPA / N**2
    g = DD(mu, nu, eps, S, max_inner_iter=CAP, safeguard=True)
    o = Oracle(mu, nu, eps, S, max_inner_iter=CAP, safeguard=True)
    mass = _mass_i(mu, S)
    for sweep in range(3):
        g.iterate(1, check=False)
        o.iterate(1)
        sg, so = g.stats(), o.stats()
        assert sg["failed"] == so["failed"] == 0, (sweep, sg, so)
        flags = g.cell_stats(flags=True)[4]
        assert int(((flags & 32) != 0).sum()) == so["safeguarded"], sweep
        d = np.abs(g.basic_marginals_dense() - o.basic_marginals_dense()).sum(1)
        assert (d <= 4e-6 * np.maximum(mass, 1e-3)).all(), (sweep, d.max())
    cg, co = g.primal_cost()[0], o.primal_cost()[0]
    assert abs(cg - co) <= 1e-5 * co
    assert g.synchronize() == 0


@pytest.mark.gpu
def test_gpu_safeguard_exhausted_reports_enoconv(DD):
    mu, nu = config_images(1)
    g = DD(mu, nu, KAPPA / N**2, S, max_inner_iter=5, safeguard=True)
    g.iterate(1, check=False)
    st = g.stats()
    assert st["failed"] == 16
    flags = g.cell_stats(flags=True)[4]
    assert ((flags & 32) != 0).sum() == 16
    D = g.basic_marginals_dense()
    assert np.abs(D.sum(0) - nu.ravel()).sum() < 1e-11
