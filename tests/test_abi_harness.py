"""The SURVEY 8(b) ABI driven through ONE harness (tests/abi_harness.py) on
both libraries: the oracle's dd_* shim (CPU tests) and libdd_gpu.so vs the
oracle (GPU tests).  Also the failure path of reading A6 (a cell hitting
max_inner_iter -> flag, DD_ENOCONV, Y-feasible state) on both sides, which
at a fixed iteration count is a same-stop-iteration parity case (P9)."""
import numpy as np
import pytest

import abi_harness as H
from ddinputs import config_images


def _oracle_lib():
    from oracle.oracle import build_oracle
    return H.load(build_oracle())


def _gpu_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import SO_PATH, lib
    lib()
    return H.load(SO_PATH)


def test_oracle_shim_exports_common_abi():
    L = _oracle_lib()
    for name in H.COMMON:
        assert hasattr(L, name), name
    assert b"oracle" in L.dd_version()


def test_shim_equals_direct_oracle():
    """The shim only marshals: same numbers as the ddo_* calls."""
    from oracle import Oracle
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    s = H.Solver(_oracle_lib(), mu, nu, eps, 4)
    assert s.iterate(4) == H.OK and s.synchronize() == H.OK
    o = Oracle(mu, nu, eps, 4)
    o.iterate(4)
    assert s.primal_cost() == o.primal_cost()
    assert s.marginal_error() == o.marginal_error()
    np.testing.assert_array_equal(s.basic_marginals().reshape(64, -1), o.basic_marginals_dense())
    s.close()


def test_shim_enoconv_deferred_to_synchronize():
    """A6 on the oracle side: max_inner_iter = 3 from the product coupling
    cannot meet Err = 1e-6; dd_iterate stays OK (as the asynchronous GPU
    call does), dd_synchronize reports DD_ENOCONV once."""
    mu, nu = config_images(1)
    s = H.Solver(_oracle_lib(), mu, nu, 2.0 / 32**2, 4, max_inner_iter=3)
    assert s.iterate(1) == H.OK
    rc, st = s.stats()
    assert rc == H.ENOCONV and st["failed"] == st["cells"] == 16 and st["iters_max"] == 3
    assert s.synchronize() == H.ENOCONV
    assert s.synchronize() == H.OK
    # the returned plans end with a Y-iteration: the state stays Y-feasible
    lx, ly = s.marginal_error()
    assert ly <= 1e-11 and lx > 1e-6             # tau = 1e-15 truncation only (P4)
    s.close()


def _member_masses(mu, nb, s):
    return mu.reshape(nb, s, nb, s).sum((1, 3)).ravel()


@pytest.mark.gpu
def test_same_harness_gpu_vs_oracle_cfg1():
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    out = []
    for L in (_gpu_lib(), _oracle_lib()):
        s = H.Solver(L, mu, nu, eps, 4)
        assert s.iterate(6) == H.OK and s.synchronize() == H.OK
        out.append((s.primal_cost(), s.marginal_error(), s.basic_marginals()))
        s.close()
    (cg, _), (lxg, lyg), bg = out[0]
    (co, _), (lxo, lyo), bo = out[1]
    assert abs(cg - co) <= 1e-5 * co
    assert lxg <= 1e-6 and lyg <= 1e-6 and lxo <= 1e-6 and lyo <= 1e-6
    assert np.abs(bg - bo).sum() <= 64 * 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("max_iter", [1, 3, 7])
def test_max_inner_iter_path_gpu_vs_oracle(max_iter):
    """Reading A6 on both sides, and a fixed-iteration parity case: every
    cell runs exactly max_iter Sinkhorn iterations, so the GPU's basic-cell
    marginals must match the oracle's to the same-stop-iteration bound of
    P9 (1e-7 ||mu_J|| per cell); both report DD_ENOCONV at synchronize and
    keep the state Y-feasible."""
    mu, nu = config_images(1)
    eps = 2.0 / 32**2
    res = []
    for L in (_gpu_lib(), _oracle_lib()):
        s = H.Solver(L, mu, nu, eps, 4, max_inner_iter=max_iter)
        for k in range(3):                       # A, B, A
            assert s.iterate(1) == H.OK
            rc, st = s.stats()
            assert rc == H.ENOCONV and st["failed"] == st["cells"] and st["iters_max"] == max_iter
        assert s.synchronize() == H.ENOCONV
        assert s.synchronize() == H.OK
        lx, ly = s.marginal_error()
        assert ly <= 1e-11                       # Y-feasible up to truncation
        res.append((s.basic_marginals().reshape(64, -1), lx, s.primal_cost()[0]))
        s.close()
    bg, lxg, cg = res[0]
    bo, lxo, co = res[1]
    mass = _member_masses(mu, 8, 4)
    # per basic cell (members of one A cell after the last, A, sweep)
    d = np.abs(bg - bo).sum(1)
    assert np.all(d <= 1e-7 * mass + 1e-15), (d / mass).max()
    assert abs(lxg - lxo) <= 1e-7 * max(lxo, 1e-12) + 1e-9
    assert abs(cg - co) <= 1e-7 * co
