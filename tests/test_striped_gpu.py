"""Multi-GPU stripe path on ONE GPU ("virtual stripes"): N
library contexts of the same problem, each solving its stripe, exchange the
boundary rows through LocalTransport exactly as ranks do over NCCL.  The
per-cell arithmetic does not depend on the stripe, so the basic-cell
marginals must be BIT-identical to one context; sums over ranks agree to
rounding.  Also checks the gathered state against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import config_images, gaussian_mixture_image  # noqa: E402
from oracle import Oracle  # noqa: E402
from oracle.oracle import SCHED_LADDER as O_LADDER  # noqa: E402


@pytest.fixture(scope="module")
def mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD
    from paper_2001_10986_b200.striped import LocalTransport, StripedRun
    return DD, LocalTransport, StripedRun


@pytest.mark.parametrize("nranks", [2, 3])
def test_virtual_stripes_ladder_cfg2(mods, nranks):
    DD, LocalTransport, StripedRun = mods
    mu, nu = config_images(2)                     # 64^2, s = 4, ladder 16 -> 64 from eps = 1
    n, s = 64, 4
    kw = dict(err_tol=1e-6, eps_start=1.0, coarsest_side=16, schedule=1)
    eps = 0.5 / n**2
    ref = DD(mu, nu, eps, s, **kw)
    ref.run_schedule()
    ctxs = [(r, DD(mu, nu, eps, s, **kw)) for r in range(nranks)]
    run = StripedRun(ctxs, nranks, LocalTransport(nranks))
    run.run_schedule(n, 16, 0.5, 1.0)
    assert run.bounds is not None and run.exchanged_bytes > 0
    Dr = ref.basic_marginals_dense()
    Ds = run.basic_marginals_dense()
    assert np.array_equal(Dr, Ds), np.abs(Dr - Ds).max()
    cr, er = ref.primal_cost()
    cs, es = run.primal_cost()
    assert abs(cr - cs) <= 1e-13 * cr and abs(er - es) <= 1e-12 * abs(er)
    lxr, lyr = ref.marginal_error()
    lxs, lys = run.marginal_error()
    assert abs(lxr - lxs) <= 1e-15 + 1e-9 * lxr and abs(lyr - lys) <= 1e-15 + 1e-9 * lyr
    # (rank sums count the replicated coarse layers once per rank; the driver
    # counts whole-problem cell solves itself)
    assert ref.totals()["cells"] == run.cells_solved
    # and the whole striped run matches the fp64 oracle (north_star gates)
    o = Oracle(mu, nu, eps, s, schedule=O_LADDER, err_tol=1e-6, eps_start=1.0, coarsest_side=16)
    o.run_schedule()
    co, _ = o.primal_cost()
    assert abs(cs - co) <= 1e-5 * co
    assert lxs <= 1e-6 and lys <= 1e-6


def test_virtual_stripes_fixed_s8_big_tiers(mods):
    """s = 8 cells on the fused big-cell tiers, 4 stripes of a 128^2 layer."""
    DD, LocalTransport, StripedRun = mods
    n, s, nranks = 128, 8, 4
    mu, nu = gaussian_mixture_image(n, 21, 3), gaussian_mixture_image(n, 22, 3)
    eps = 1.0 / n**2
    ref = DD(mu, nu, eps, s, bcap_main=18)
    ctxs = [(r, DD(mu, nu, eps, s, bcap_main=18)) for r in range(nranks)]
    run = StripedRun(ctxs, nranks, LocalTransport(nranks))
    run.start()
    ref.iterate(6)
    run.iterate(6)
    assert run.bounds == [0, 4, 8, 12, 16]
    assert np.array_equal(ref.basic_marginals_dense(), run.basic_marginals_dense())
    cr, _ = ref.primal_cost()
    cs, _ = run.primal_cost()
    assert abs(cr - cs) <= 1e-13 * cr
    tr, ts = ref.totals(), run.totals()
    assert tr["iters_sum"] == ts["iters_sum"] and tr["cells"] == ts["cells"] == run.cells_solved


def test_bench_two_ranks_one_gpu_gloo(mods, tmp_path):
    """bench.py's N = 2 striped path end to end (torchrun, 2 processes sharing
    the GPU, host-staged gloo transport instead of NCCL): the whole-problem
    cost equals a single context's on the same inputs."""
    import json
    import os
    import subprocess
    import sys
    DD = mods[0]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 300),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "3",
           "--dist-backend", "gloo", "--no-e2e", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    from ddinputs import config_images, CONFIGS
    p = CONFIGS[3]
    mu, nu = config_images(3)
    g = DD(mu, nu, p["kappa_final"] / p["n"]**2, p["s"], schedule=1, coarsest_side=8)
    g.run_schedule()
    c1, _ = g.primal_cost()
    assert abs(line["final"]["transport_cost"] - c1) <= 1e-12 * c1
    assert line["final"]["l1_x"] <= 1e-6 and line["final"]["l1_y"] <= 1e-6
    assert line["cells_per_step"] == g.totals()["cells"]


def test_virtual_stripes_cost_aware_rebalance(mods):
    """Cost-aware stripe bounds (StripedRun.rebalance: rows move between
    ranks at eps-stage boundaries, balancing the last A-sweep's work) on the
    cfg-4 recipe at 128^2 with 4 stripes: bounds do move, and the result is
    still bit-identical to one context (and to equal-row stripes)."""
    DD, LocalTransport, StripedRun = mods
    n, s, nranks = 128, 8, 4
    mu, nu = gaussian_mixture_image(n, 41, 4), gaussian_mixture_image(n, 42, 4)
    eps = 0.5 / n**2
    kw = dict(schedule=1, coarsest_side=8, bcap_main=18)
    ref = DD(mu, nu, eps, s, **kw)
    ref.run_schedule()
    out = {}
    for ca in (True, False):
        ctxs = [(r, DD(mu, nu, eps, s, **kw)) for r in range(nranks)]
        run = StripedRun(ctxs, nranks, LocalTransport(nranks), cost_aware=ca)
        run.run_schedule(n, 8, 0.5)
        out[ca] = (run, run.basic_marginals_dense())
    assert out[True][0].rebalances > 0 and out[False][0].rebalances == 0
    assert out[True][0].bounds != [0, 4, 8, 12, 16]
    Dr = ref.basic_marginals_dense()
    assert np.array_equal(Dr, out[True][1]) and np.array_equal(Dr, out[False][1])
    cr, _ = ref.primal_cost()
    cs, _ = out[True][0].primal_cost()
    assert abs(cr - cs) <= 1e-13 * cr
