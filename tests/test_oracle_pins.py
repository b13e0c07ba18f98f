"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md Sec. 8(c) pins P1-P8).  No GPU; these run with -m "not gpu".

Each reference value below comes from a closed form, an invariant the paper
proves, or an independent textbook implementation in tests/refs.py -- never
from the oracle itself and never from the CUDA path."""
import numpy as np
import pytest

from ddinputs import gaussian_mixture_image, product_image, config_images
from oracle import Oracle, build_schedule, sinkhorn_dense
from oracle.oracle import SCHED_LADDER
from refs import global_sinkhorn, grid_cost, kl, quadratic_2x2, sinkhorn_1d


# ---------------------------------------------------------------- P1 / P1b --
def test_p1_closed_form_2x2():
    """mu = nu = (1/2,1/2), c = [[0,1],[1,0]], eps = 1 ->
    pi11 = e/(2(1+e)), pi12 = 1/(2(1+e)) (symmetric scaling ansatz)."""
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    f, g, it, err, rc = sinkhorn_dense([0.5, 0.5], [0.5, 0.5], C, 1.0, 1e-15)
    P = np.exp(f[:, None] + g[None, :] - C)
    e = np.e
    assert rc == 0
    assert abs(P[0, 0] - e / (2 * (1 + e))) < 1e-15
    assert abs(P[0, 1] - 1 / (2 * (1 + e))) < 1e-15
    assert abs(P[0, 0] - 0.3655292893150025) < 1e-15


@pytest.mark.parametrize("seed", range(4))
def test_p1b_general_2x2(seed):
    """Pin P1b: the optimum of the 2x2 problem is the root of the quadratic
    forced by the scaling form pi = u (x) v K (Prop. EntropicOTBasic (ii))."""
    rng = np.random.default_rng(100 + seed)
    a = rng.uniform(0.1, 1.0, 2); a /= a.sum()
    b = rng.uniform(0.1, 1.0, 2); b /= b.sum()
    C = rng.uniform(0.0, 2.0, (2, 2))
    eps = rng.uniform(0.2, 2.0)
    f, g, it, err, rc = sinkhorn_dense(a, b, C, eps, 1e-15, max_iter=100000)
    P = np.exp((f[:, None] + g[None, :] - C) / eps)
    Q = quadratic_2x2(a[0], a[1], b[0], b[1], C, eps)
    assert rc == 0
    assert np.abs(P - Q).max() < 1e-14


def test_sinkhorn_ends_with_y_iteration_and_meets_tolerance():
    """Sec. 6.2: Y-marginal exact, X-marginal L1 <= tol."""
    rng = np.random.default_rng(7)
    nx, ny = 12, 17
    a = rng.uniform(0.1, 1, nx); a /= a.sum()
    b = rng.uniform(0.1, 1, ny); b /= b.sum()
    C = rng.uniform(0, 1, (nx, ny))
    eps = 0.05
    f, g, it, err, rc = sinkhorn_dense(a, b, C, eps, 1e-9)
    P = np.exp((f[:, None] + g[None, :] - C) / eps)
    assert rc == 0 and it > 1
    assert np.abs(P.sum(0) - b).max() < 1e-15
    assert np.abs(P.sum(1) - a).sum() <= 1e-9
    assert abs(np.abs(P.sum(1) - a).sum() - err) < 1e-14
    # warm start from the returned potential: 1 iteration (fixed point)
    f2, g2, it2, err2, rc2 = sinkhorn_dense(a, b, C, eps, 1e-9, f0=f)
    assert it2 == 1 and rc2 == 0


# --------------------------------------------------------------- partitions --
def test_partition_counts_spec_example():
    """S:132-133 / P:1566-1569: 16x16 px, s = 4 -> |J_A| = 4, |J_B| = 9."""
    mu, nu = gaussian_mixture_image(16, 1, 1), gaussian_mixture_image(16, 2, 1)
    o = Oracle(mu, nu, 2 / 16**2, 4)
    o.iterate(1)
    assert o.stats()["cells"] == 4
    o.iterate(1)
    assert o.stats()["cells"] == 9
    o8 = Oracle(gaussian_mixture_image(8, 1, 1), gaussian_mixture_image(8, 2, 1), 2 / 64, 4)
    o8.iterate(2)   # side 8, s 4: A = one cell, B = 4 singletons
    assert o8.stats()["cells"] == 4


@pytest.mark.parametrize("nb", [2, 4, 8, 16])
def test_partition_graph_conditions(nb):
    """Def. PartitionGraph: no pair of basic cells shares both an
    A-cell and a B-cell, and the partition graph is connected.  Checked on
    the A/B construction of P:1566-1569 (reading A11) for every layer size."""
    def cells(part):
        out = []
        nca = nb // 2 if part == "A" else nb // 2 + 1
        for p in range(nca):
            for q in range(nca):
                if part == "A":
                    rows, cols = [2 * p, 2 * p + 1], [2 * q, 2 * q + 1]
                else:
                    rows = [r for r in (2 * p - 1, 2 * p) if 0 <= r < nb]
                    cols = [c for c in (2 * q - 1, 2 * q) if 0 <= c < nb]
                out.append({r * nb + c for r in rows for c in cols})
        return out
    A, B = cells("A"), cells("B")
    assert sorted(i for J in A for i in J) == list(range(nb * nb))
    assert sorted(i for J in B for i in J) == list(range(nb * nb))
    pairA = {(i, j) for J in A for i in J for j in J if i < j}
    pairB = {(i, j) for J in B for i in J for j in J if i < j}
    assert not (pairA & pairB)
    adj = {i: set() for i in range(nb * nb)}
    for i, j in pairA | pairB:
        adj[i].add(j); adj[j].add(i)
    seen, stack = {0}, [0]
    while stack:
        for j in adj[stack.pop()]:
            if j not in seen:
                seen.add(j); stack.append(j)
    assert len(seen) == nb * nb


# ----------------------------------------------------------------- schedule --
@pytest.mark.parametrize("n,total", [(256, 50), (64, 34), (8, 10)])
def test_schedule_counts_paper(n, total):
    """(n-2)*8 + 2 sweeps with the paper's final eps = 0.25."""
    sch = build_schedule(n, 8, 0.25)
    assert sum(s for _, _, s in sch) == total
    assert [k for s, k, _ in sch if s == n][-1] == 0.25


def test_schedule_baseline_configs():
    """BASELINE configs: final kappa 0.5 -> (n-2)*8 sweeps (reading A12)."""
    assert sum(w for _, _, w in build_schedule(2048, 8, 0.5)) == 72
    assert sum(w for _, _, w in build_schedule(1024, 8, 0.5)) == 64
    assert sum(w for _, _, w in build_schedule(256, 8, 0.5)) == 48
    sch = build_schedule(64, 16, 0.5, eps_start=1.0)
    assert sch[0] == (16, 256.0, 2)
    assert (16, 2.0, 4) in sch
    assert sum(w for _, _, w in sch) == 14 + 8 + 8 + 8
    assert all(w % 2 == 0 for _, _, w in sch)   # every stage starts with A


# ------------------------------------------------------------ init / P4 / P7 --
def test_product_init():
    """S:274 / P:1461: nu_i^0 = ||mu_i|| nu; Alg. 2 input contract holds exactly."""
    mu, nu = config_images(1)
    o = Oracle(mu, nu, 2 / 32**2, 4)
    D = o.basic_marginals_dense()
    mass_i = mu.reshape(8, 4, 8, 4).sum((1, 3)).ravel()
    np.testing.assert_allclose(D, mass_i[:, None] * nu.ravel()[None, :], rtol=0, atol=1e-18)
    assert np.abs(D.sum(0) - nu.ravel()).max() < 1e-17


def test_conservation_every_sweep_P4():
    """Prop. feasibility + Sec. 6.2: after every sweep
    sum_i nu_i = nu pointwise (up to truncation), ||nu_i|| = ||mu_i||, and the
    summed X-error is bounded by Err."""
    mu, nu = config_images(1)
    err = 1e-6
    o = Oracle(mu, nu, 2 / 32**2, 4, err_tol=err)
    mass_i = mu.reshape(8, 4, 8, 4).sum((1, 3)).ravel()
    for _ in range(6):
        o.iterate(1)
        D = o.basic_marginals_dense()
        assert np.abs(D.sum(0) - nu.ravel()).sum() < 1e-11
        # balance is exact up to the mass truncation dropped (tau * #dropped per cell)
        np.testing.assert_allclose(D.sum(1), mass_i, rtol=1e-12, atol=1e-12)
        assert (D >= 0).all()
        st = o.stats()
        assert st["err_x_sum"] <= err * (1 + 1e-12)
        l1x, l1y = o.marginal_error()
        assert l1x <= err * 1.0001
        assert abs(l1x - st["err_x_sum"]) < 1e-12


def test_truncation_and_tight_boxes():
    """P:1386 / P:1524 (readings A9/A10): every stored entry is 0 or >= tau and
    each box is the tight bounding box of its kept entries."""
    mu, nu = config_images(1)
    o = Oracle(mu, nu, 2 / 32**2, 4)
    o.iterate(3)
    st = o.get_state()
    tau = 1e-15
    for i, (y0, x0, hr, hc) in enumerate(st["boxes"]):
        v = st["values"][st["offsets"][i]:st["offsets"][i] + hr * hc].reshape(hr, hc)
        assert ((v == 0) | (v >= tau)).all()
        assert (v[0] > 0).any() and (v[-1] > 0).any()
        assert (v[:, 0] > 0).any() and (v[:, -1] > 0).any()


def test_refinement_identities_P7():
    """Prop. FineBasicMarginals: sum_i nu_i^0 = nu and
    ||nu_i^0|| = ||mu_i|| for the refined initialisation."""
    mu, nu = config_images(2)       # 64 x 64
    o = Oracle(mu, nu, 0.5 / 64**2, 4, schedule=SCHED_LADDER, coarsest_side=16)
    o.set_eps(2 / 16**2)
    o.iterate(4)
    o.refine()
    info = o.state_info()
    assert info["side"] == 32
    mu32, nu32 = o.layer_marginals()
    D = o.basic_marginals_dense()
    nb = info["nb"]
    s = info["s"]
    mass_i = mu32.reshape(nb, s, nb, s).sum((1, 3)).ravel()
    # truncation of the coarse state (tau = 1e-15) is the only slack
    assert np.abs(D.sum(0) - nu32.ravel()).sum() < 1e-12
    np.testing.assert_allclose(D.sum(1), mass_i, rtol=1e-11, atol=1e-13)


def test_refinement_collapses_to_product():
    """refining the product state nuhat_j = ||muhat_j|| nuhat gives
    nu_i^0 = ||mu_i|| nu exactly (the formula collapses)."""
    mu, nu = config_images(2)
    o = Oracle(mu, nu, 0.5 / 64**2, 4, schedule=SCHED_LADDER, coarsest_side=16)
    o.refine()
    mu32, nu32 = o.layer_marginals()
    D = o.basic_marginals_dense()
    mass_i = mu32.reshape(8, 4, 8, 4).sum((1, 3)).ravel()
    np.testing.assert_allclose(D, mass_i[:, None] * nu32.ravel()[None, :], rtol=1e-13, atol=1e-20)


def test_refinement_worked_value():
    """S:368 worked value re-expressed on the grid: for a coarse basic cell j
    whose partial marginal is half of nuhat at a coarse pixel (ratio 0.5) and a
    fine cell with mu(X_i)/muhat(X_j) = 0.4, the fine entry at a child y is
    nu(y) * 0.5 * 0.4.  Built via set_state with hand-chosen coarse values."""
    n = 16
    mu = np.full((n, n), 1.0 / n**2)
    nu = np.full((n, n), 1.0 / n**2)
    o = Oracle(mu, nu, 1.0, 4, schedule=SCHED_LADDER, coarsest_side=8)
    # coarse layer 8x8, s = 4, nb = 2; build state: cell j takes share w_j(y)
    st = o.get_state()
    side = 8
    nuhat = np.full(side * side, 4.0 / n**2)
    shares = np.array([0.5, 0.2, 0.2, 0.1])   # sum = 1 at every coarse y
    vals = np.concatenate([shares[j] * nuhat for j in range(4)])
    st["values"] = vals
    st["offsets"] = np.arange(4, dtype=np.int64) * side * side
    st["boxes"] = np.tile(np.array([0, 0, side, side], np.int32), (4, 1))
    o.set_state(st)
    o.refine()
    D = o.basic_marginals_dense()     # fine: 16x16, s = 4 -> nb = 4 (Pa(i) = 2x2 children)
    # fine cell i = (0,0) has parent j = 0; mu(X_i)/muhat(X_j) = (16/256)/(64/256) = 0.25
    y = 0
    assert abs(D[0, y] - nu.ravel()[y] * 0.5 * 0.25) < 1e-18
    np.testing.assert_allclose(D.sum(0), nu.ravel(), rtol=1e-14)


# ------------------------------------------------------------- P3 / P5 / P6 --
def _small_problem(n, seed=1):
    return gaussian_mixture_image(n, seed, 1), gaussian_mixture_image(n, seed + 1, 1)


def test_single_cell_equals_global_sinkhorn_P6():
    """an 8x8 grid with s = 4 has ONE A-cell; one A-sweep is a global
    Sinkhorn solve and must equal the independent global reference."""
    n = 8
    mu, nu = _small_problem(n)
    eps = 2 / n**2
    o = Oracle(mu, nu, eps, 4, err_tol=1e-14, no_truncate=True)
    o.iterate(1)
    P = o.plan_dense()
    Pstar = global_sinkhorn(mu, nu, grid_cost(n), eps)
    assert np.abs(P - Pstar).sum() < 1e-12


def test_dd_converges_to_global_optimum_P3_P5():
    """Pin P3 (Prop. SimpleConvergence, Thm. 2): with
    exact sub-solves and no truncation the DD iterates converge to the unique
    global entropic optimum pi*.  Pin P5 (Lemma SubOptKL): the
    primal score KL(pi^l|K) is non-increasing and Delta = KL(pi^l|pi*)
    decreases (linearly)."""
    n = 16
    mu, nu = _small_problem(n, 3)
    eps = 2 / n**2
    cost = grid_cost(n)
    Pstar = global_sinkhorn(mu, nu, cost, eps)
    K = np.exp(-cost / eps) * np.outer(mu.ravel(), nu.ravel())
    o = Oracle(mu, nu, eps, 4, err_tol=1e-13, no_truncate=True)
    prev_score = None
    deltas = []
    for k in range(40):
        o.iterate(1)
        P = o.plan_dense()
        score = kl(P, K)
        if prev_score is not None:
            assert score <= prev_score + 1e-12
        prev_score = score
        deltas.append(kl(P, Pstar))
    o.iterate(100)
    P = o.plan_dense()
    assert np.abs(P - Pstar).sum() < 1e-9
    # Delta decreases geometrically over the early phase (before rounding floor)
    assert deltas[30] < 1e-3 * deltas[5]
    # entropic score reported by the oracle = eps (KL(pi|K) - ||K||) (Lemma ScalingKL)
    cost_o, ent_o = o.primal_cost()
    assert abs(ent_o - eps * (kl(P, K) - K.sum())) < 1e-12
    assert abs(cost_o - (cost * P).sum()) < 1e-14


def test_product_marginals_closed_form_P2():
    """Pin P2: for product marginals and separable cost the 2D optimum is
    pi1 (x) pi2 of two 1D problems (Prop. Duality (iii)); the converged DD
    state must have nu_i = (row partial of pi1) (x) (col partial of pi2), and
    <c,pi> = <c1,pi1> + <c2,pi2>."""
    n, s = 16, 4
    mu, a1, a2 = product_image(n, 11)
    nu, b1, b2 = product_image(n, 12)
    eps = 2 / n**2
    t = (np.arange(n) + 0.5) / n
    c1 = (t[:, None] - t[None, :]) ** 2
    P1 = sinkhorn_1d(a1, b1, c1, eps)
    P2 = sinkhorn_1d(a2, b2, c1, eps)
    o = Oracle(mu, nu, eps, s, err_tol=1e-13, no_truncate=True)
    o.iterate(90)
    D = o.basic_marginals_dense()
    nb = n // s
    for i in range(nb * nb):
        r, c = divmod(i, nb)
        ref = np.outer(P1[r * s:(r + 1) * s].sum(0), P2[c * s:(c + 1) * s].sum(0))
        assert np.abs(D[i] - ref.ravel()).sum() < 1e-10
    cost_o, _ = o.primal_cost()
    assert abs(cost_o - ((c1 * P1).sum() + (c1 * P2).sum())) < 1e-11


def test_translation_limit_P8():
    """P8 (units sanity): a blob translated by t pixels with a tiny floor has
    W2^2 = |t|^2 h^2 + O(floor); <c, pi_eps> approaches it as kappa decreases."""
    n = 16
    t = (np.arange(n) + 0.5) / n
    x1, x2 = np.meshgrid(t, t, indexing="ij")
    sig = 0.12
    g = np.exp(-0.5 * ((x1 - 0.45) ** 2 + (x2 - 0.45) ** 2) / sig**2)
    sh = (2, 1)
    gy = np.exp(-0.5 * ((x1 - 0.45 - sh[0] / n) ** 2 + (x2 - 0.45 - sh[1] / n) ** 2) / sig**2)
    phi = 1e-9 * g.max()
    mu = g + phi; mu /= mu.sum()
    nu = gy + phi; nu /= nu.sum()
    w2 = (sh[0] ** 2 + sh[1] ** 2) / n**2
    rel = []
    for kappa in (2.0, 0.5, 0.25):
        o = Oracle(mu, nu, kappa / n**2, 4, err_tol=1e-8)
        o.iterate(30)
        rel.append(abs(o.primal_cost()[0] - w2) / w2)
    assert rel[0] > rel[1] > rel[2]
    assert rel[2] < 0.02


# ------------------------------------------------------------- determinism --
def test_deterministic_across_thread_counts():
    """the post-sweep state is bit-identical for any worker count."""
    mu, nu = _small_problem(16, 5)
    states = []
    for nt in (1, 3):
        o = Oracle(mu, nu, 2 / 16**2, 4, n_threads=nt)
        o.iterate(4)
        states.append(o.get_state())
    a, b = states
    assert np.array_equal(a["boxes"], b["boxes"])
    assert np.array_equal(a["values"], b["values"])
    assert np.array_equal(a["alpha_A"], b["alpha_A"])
    assert np.array_equal(a["alpha_B"], b["alpha_B"])


# -------------------------------------------------------------- validation --
@pytest.mark.parametrize("case", ["npow2", "odd_nb", "negative", "unequal", "zero_cell"])
def test_validation_errors(case):
    n, s = 16, 4
    mu = np.full((n, n), 1 / n**2)
    nu = np.full((n, n), 1 / n**2)
    if case == "npow2":
        mu = np.full((12, 12), 1 / 144); nu = mu.copy(); n = 12
    elif case == "odd_nb":
        s = 8   # n/s = 2 is even; use 16/16? use s = 16 -> n/s = 1 odd
        s = 16
    elif case == "negative":
        mu = mu.copy(); mu[0, 0] = -1e-3; mu[0, 1] += 1e-3
    elif case == "unequal":
        nu = nu * 1.01
    elif case == "zero_cell":
        mu = mu.copy(); mu[:4, :4] = 0; mu /= mu.sum()
    with pytest.raises(ValueError):
        Oracle(mu, nu, 1.0, s)


@pytest.mark.parametrize("concurrent", [False, True])
def test_solve_cells_equals_sweep_subset(concurrent):
    """ddo_solve_cells (one cell at a time with the half-iterations threaded,
    or the cells concurrently) on every cell of a partition reproduces
    ddo_iterate bit for bit."""
    mu, nu = config_images(1)
    a = Oracle(mu, nu, 2 / 32**2, 4)
    b = Oracle(mu, nu, 2 / 32**2, 4)
    a.iterate(1)
    b.solve_cells(1, np.arange(16), concurrent=concurrent)
    assert np.array_equal(a.basic_marginals_dense(), b.basic_marginals_dense())


# ------------------------------------------------------------- PD gap (f1) --
def test_pd_gap_single_cell_is_zero():
    """One A-cell covering X (n = 2s): the A-sweep IS the global problem and
    gluing is trivial, so at Err -> 0 the relative PD gap of eq. RelPDGap
     vanishes: J(u, v) = KL(pi|K) at the optimum (Prop. Duality
    (iii))."""
    m8, n8 = gaussian_mixture_image(8, 1, 1), gaussian_mixture_image(8, 2, 1)
    o = Oracle(m8, n8, 2 / 64, 4, err_tol=1e-12, no_truncate=True)
    o.iterate(1)
    P, D, rel = o.dual_gap()
    assert abs(rel) < 1e-10 and P > 0


def test_pd_gap_weak_duality_and_convergence():
    """Weak duality J <= KL (Prop. Duality (ii)) up to the iterate's
    marginal error, and the gap -> 0 as the DD converges to the global
    optimum (Thm 2): the glued dual candidate of Sec. 6.3."""
    mu, nu = config_images(1)
    o = Oracle(mu, nu, 2 / 32**2, 4, err_tol=1e-10, no_truncate=True)
    gaps = []
    for k in (2, 4, 14, 40):
        o.iterate(k)
        gaps.append(o.dual_gap()[2])
    assert all(g > -1e-9 for g in gaps)
    assert all(b < a for a, b in zip(gaps, gaps[1:]))
    assert gaps[-1] < 1e-7


def _perturbed_product_state(delta_move, delta_scale):
    """The product coupling nu_i = ||mu_i|| nu at 32^2 (Y-feasible: sum_i nu_i
    = nu), then (a) mass delta_move moved inside basic cell 5's box
    from its largest entry to one 13 rows / 5 columns away, (b) every nu_i
    scaled by (1 + delta_scale).  nu is not symmetric, so a transposed or
    shifted accumulation fails by far more than the deviation."""
    mu, nu = config_images(1)
    o = Oracle(mu, nu, 2.0 / 32**2, 4)
    st = o.get_state()
    v = st["values"].copy()
    y0, x0, hr, hc = st["boxes"][5]
    assert (y0, x0, hr, hc) == (0, 0, 32, 32)
    o5 = st["offsets"][5]
    src = int(np.argmax(v[o5:o5 + 1024]))
    r, c = divmod(src, 32)
    dst = ((r + 13) % 32) * 32 + (c + 5) % 32
    assert v[o5 + src] > 2 * delta_move
    v[o5 + src] -= delta_move
    v[o5 + dst] += delta_move
    v *= 1.0 + delta_scale
    st["values"] = v
    dev = delta_scale * nu.ravel().copy()          # the known deviation sum_i nu_i - nu
    dev[src] -= delta_move * (1.0 + delta_scale)
    dev[dst] += delta_move * (1.0 + delta_scale)
    return mu, nu, st, dev


@pytest.mark.parametrize("dm,ds", [(5e-6, 0.0), (0.0, 1e-3), (1e-6, 0.0), (2e-6, 1e-4)])
def test_marginal_error_l1y_pin(dm, ds):
    """Reading A18: l1_y = sum_y |sum_i nu_i(y) - nu(y)|.  A state of known
    deviation: moving mass d inside one box gives exactly 2 d; scaling every
    nu_i by (1 + e) gives e ||nu|| = e.  Pins ddo_marginal_error's l1_y."""
    mu, nu, st, dev = _perturbed_product_state(dm, ds)
    o = Oracle(mu, nu, 2.0 / 32**2, 4, empty_init=True)
    o.set_state(st)
    _, ly = o.marginal_error()
    want = np.abs(dev).sum()                       # 2 dm, resp. ds, when only one is set
    if dm == 0.0 or ds == 0.0:
        assert abs(want - (2 * dm + ds)) <= 1e-15
    assert abs(ly - want) <= 1e-13 + 1e-10 * want, (ly, want)


# ----------------------------------------------- f1: warm-start refinement --
def _bilinear_a26(ph, i, j):
    """Reading A26 written out: fine centre (i + 1/2)/2 - 1/2 in coarse index
    units, bilinear, constant beyond the outermost coarse centres."""
    sc = ph.shape[0]
    u = min(max(0.5 * i - 0.25, 0.0), sc - 1.0)
    v = min(max(0.5 * j - 0.25, 0.0), sc - 1.0)
    i0, j0 = int(u), int(v)
    i1, j1 = min(i0 + 1, sc - 1), min(j0 + 1, sc - 1)
    fu, fv = u - i0, v - j0
    return ((1 - fu) * ((1 - fv) * ph[i0, j0] + fv * ph[i0, j1]) + fu * ((1 - fv) * ph[i1, j0] + fv * ph[i1, j1]))


def test_warm_refine_glues_and_interpolates():
    """P:1507-1508 (f1): alpha_A = phi + k_A(J_A(x)), alpha_B = phi + k_B(J_B(x))
    with arbitrary per-cell constants (the gauge freedom of each cell's
    potential): gluing (Sec. 6.3, reading A25) must recover phi up to
    one global constant, and the fine potentials of BOTH partitions are its
    log-space linear interpolation (reading A26)."""
    from oracle.oracle import SCHED_LADDER
    n, s = 32, 4
    mu, nu = config_images(1)
    o = Oracle(mu, nu, 2.0 / 16**2, s, schedule=SCHED_LADDER, coarsest_side=16, warm_refine=True)
    st = o.get_state()
    side, nb = st["info"]["side"], st["info"]["nb"]
    assert side == 16
    rng = np.random.default_rng(7)
    ii, jj = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    phi = 1e-3 * (np.sin(ii / 3.0) + 0.5 * np.cos(jj / 5.0) + 0.01 * ii * jj)
    na, nbB = nb // 2, nb // 2 + 1
    kA = rng.normal(size=(na, na)) * 1e-2
    kB = rng.normal(size=(nbB, nbB)) * 1e-2
    cellA = (ii // s) // 2, (jj // s) // 2
    cellB = (ii // s + 1) // 2, (jj // s + 1) // 2
    st["alpha_A"] = phi + kA[cellA]
    st["alpha_B"] = phi + kB[cellB]
    st["info"]["last_partition"] = 2
    o.set_state(st)
    o.refine()
    fine = o.get_state()
    aA, aB = fine["alpha_A"], fine["alpha_B"]
    assert aA.shape == (32, 32)
    np.testing.assert_array_equal(aA, aB)
    ref = np.array([[_bilinear_a26(phi, i, j) for j in range(32)] for i in range(32)])
    d = aA - ref
    assert np.ptp(d) < 1e-12, np.ptp(d)


def test_warm_refine_ladder_faster_same_answer():
    """The warm start only changes the Sinkhorn iteration counts (the cell
    optimum is unique): same cost to 1e-6 relative, fewer iterations."""
    from oracle.oracle import SCHED_LADDER, build_schedule
    mu, nu = config_images(2)
    res = {}
    for warm in (False, True):
        o = Oracle(mu, nu, 0.5 / 64**2, 4, schedule=SCHED_LADDER, coarsest_side=16, eps_start=1.0,
                   warm_refine=warm)
        its, side = 0, 16
        for sd, kappa, sweeps in build_schedule(64, 16, 0.5, 1.0):
            while side < sd:
                o.refine()
                side *= 2
            o.set_eps(kappa / sd**2)
            for _ in range(sweeps):
                o.iterate(1)
                its += o.stats()["iters_sum"]
        res[warm] = (o.primal_cost()[0], its, o.marginal_error())
    (c0, i0, m0), (c1, i1, m1) = res[False], res[True]
    assert abs(c1 - c0) <= 1e-6 * c0, (c0, c1)
    assert m1[0] <= 1e-6 and m1[1] <= 1e-6
    assert i1 < i0, (i0, i1)
