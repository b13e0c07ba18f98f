"""Full-trajectory parity at config 3 (256^2, s = 4, anisotropic Gaussian
mixtures, the paper's ladder 8^2 -> 256^2 = 48 sweeps, final eps = 0.5 h^2,
Err = 1e-6, tau = 1e-15): the GPU's whole schedule against the oracle's
whole schedule on the same seeded images (trajectory
parity uses the same gates as a single sweep).  The dense fp64 oracle needs
~1.5 min on 16 host cores here."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import CONFIGS, config_images  # noqa: E402
from oracle import Oracle  # noqa: E402
from oracle.oracle import SCHED_LADDER as O_LADDER  # noqa: E402


@pytest.fixture(scope="module")
def cfg3_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    p = CONFIGS[3]
    mu, nu = config_images(3)
    eps = p["kappa_final"] / p["n"] ** 2
    o = Oracle(mu, nu, eps, p["s"], schedule=O_LADDER, coarsest_side=8, err_tol=1e-6)
    o.run_schedule()
    return dict(mu=mu, nu=nu, eps=eps, s=p["s"], cost=o.primal_cost()[0], err=o.marginal_error(),
                info=o.state_info(), marg=o.basic_marginals_dense())


@pytest.mark.parametrize("cold", [True, False])
def test_cfg3_full_trajectory_vs_oracle(cfg3_oracle, cold):
    """cold = True: the GPU follows the oracle's potential refinement (cold
    start, reading A14) -- the same algorithm sweep for sweep; cold = False:
    the bench's configuration (glued + interpolated warm start),
    which only changes iteration counts."""
    from paper_2001_10986_b200 import DD
    r = cfg3_oracle
    g = DD(r["mu"], r["nu"], r["eps"], r["s"], schedule=1, coarsest_side=8, err_tol=1e-6, cold_refine=cold)
    g.run_schedule()
    cg, _ = g.primal_cost()
    lx, ly = g.marginal_error()
    info = g.state_info()
    assert info["half_index"] == r["info"]["half_index"] == 48
    assert abs(cg - r["cost"]) <= 1e-5 * r["cost"], (cg, r["cost"])
    assert lx <= 1e-6 and ly <= 1e-6, (lx, ly)
    assert r["err"][0] <= 1e-6 and r["err"][1] <= 1e-6
    d = np.abs(g.basic_marginals_dense() - r["marg"]).sum()
    print(f"cfg3 cold={cold}: cost gpu {cg:.12f} oracle {r['cost']:.12f} rel {abs(cg - r['cost']) / r['cost']:.2e}"
          f" l1x {lx:.3e} l1y {ly:.3e} |nu_gpu - nu_ora|_1 {d:.3e}")
    # each cell solve stops within Err ||mu_J|| of its optimum (both sides):
    # sum over the cells of the last sweep <= 2 Err ||mu|| plus what the
    # earlier sweeps' differences leave (they contract, Thm 2)
    assert d <= 1e-5
