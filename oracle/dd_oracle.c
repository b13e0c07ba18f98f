/*
 * dd_oracle.c -- plain, slow, obviously-correct CPU fp64 oracle of entropic
 * domain decomposition for optimal transport (arXiv 2001.10986).
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load this.  It shares no code with the
 * CUDA product path.
 *
 * Every function follows the paper step by step, in its order and notation:
 *   Sinkhorn Y-/X-iteration ........ Remark "Sinkhorn algorithm"
 *   sub-solver semantics ............ Sec. 6.2, P:1402-1411 (warm start from u,
 *                                     start with a Y-iteration, L1 X-error
 *                                     stop <= ||mu_J|| Err, end after Y-iter)
 *   Algorithm 2 (one sweep) ......... P:1337-1374 (lines 8-13)
 *   BalanceMeasures ................. P:1412-1414 (rule: DESIGN.md reading A8)
 *   Truncate ........................ P:1386-1389
 *   partitions A/B .................. P:1566-1569 (reading A11)
 *   coarse-to-fine refinement ....... eq. FineBasicMarginals
 *   eps change keeps eps*log u ...... P:1510
 *   schedule ........................ P:1553-1561 (reading A12)
 *   primal score ..................... P:1419, Lemma ScalingKL
 * The cell solver is DENSE: |X_J| x |Y_J| terms per half-iteration, no
 * separable trick, global coordinates, libm exp/log, max-stabilised LSE.
 */
#include "dd_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAX_LAYERS 16

typedef struct {
    int side, s, nb;
    double* mu;        /* side*side */
    double* nu;        /* side*side */
    double* logmu;     /* side*side, -inf where mu == 0 */
    double* mass_i;    /* nb*nb : ||mu_i|| */
} layer_t;

struct ddo_ctx {
    ddo_options opt;
    double tau;
    int n_layers, cur;
    layer_t L[MAX_LAYERS];
    double eps, eps_final;
    /* state of the current layer: basic-cell Y-marginals nu_i as dense boxes */
    int* box;          /* nb*nb*4: y0r, y0c, hr, hc */
    double** val;      /* nb*nb arrays hr*hc */
    double* alphaA;    /* side*side */
    double* alphaB;
    long long half_index;
    int last_part;
    ddo_sweep_stats stats;
    /* general separable cost: c(x,y) = h1(|x1-y1|) + h2(|x2-y2|),
     * tables over finest-grid pixel differences 0..n_final-1 (NULL: |x-y|^2) */
    double *h1, *h2;
    int n_final;
    char err[512];
};

static void set_err(ddo_ctx* c, const char* fmt, ...) {
    if (!c) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
}

/* ---------------------------------------------------------------- sums -- */
/* Neumaier compensated summation (reading A17). */
typedef struct { double s, c; } ksum_t;
static void ks_add(ksum_t* k, double x) {
    double t = k->s + x;
    if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x;
    else k->c += (x - t) + k->s;
    k->s = t;
}
static double ks_get(const ksum_t* k) { return k->s + k->c; }

/* ------------------------------------------------------- dense Sinkhorn -- */
/* Remark Sinkhorn in log domain with absorbed potentials
 * f = eps log(u mu), g = eps log(v nu):
 *   Y-iteration: g(y) = eps log b(y) - eps LSE_x[(f(x) - c(x,y))/eps]
 *   X-iteration: f(x) = eps log a(x) - eps LSE_y[(g(y) - c(x,y))/eps]
 * Stop test after the X-iteration on the X-marginal of the plan (f_old, g):
 *   P_X pi(x) = a(x) exp((f_old - f_new)/eps). */
static double lse_col(int nx, int ny, const double* f, const double* C, int y, double eps) {
    double m = -INFINITY;
    for (int x = 0; x < nx; ++x) {
        double t = f[x] - C[(size_t)x * ny + y];
        if (t > m) m = t;
    }
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int x = 0; x < nx; ++x) s += exp((f[x] - C[(size_t)x * ny + y] - m) / eps);
    return m + eps * log(s);
}
static double lse_row(int ny, const double* g, const double* Crow, double eps) {
    double m = -INFINITY;
    for (int y = 0; y < ny; ++y) {
        double t = g[y] - Crow[y];
        if (t > m) m = t;
    }
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int y = 0; y < ny; ++y) s += exp((g[y] - Crow[y] - m) / eps);
    return m + eps * log(s);
}

/* The loop of P:1404-1411.  check_every = k (reading A5): the stop test is
 * evaluated after every X-iteration and honoured when it % k == 0.  The two
 * half-iterations are independent per output (y, resp. x), so when called
 * outside a parallel region (a few large sampled cells) their outputs are
 * computed by nt OpenMP threads; every output is the same serial sum, so the
 * result does not depend on the thread count. */
static int sinkhorn_dense_k(int nx, int ny, const double* a, const double* b, const double* C,
                            double eps, double tol, int max_iter, int check_every, int nt,
                            double* f, double* g, int* iters, double* err) {
    double* fn = (double*)malloc(sizeof(double) * (size_t)(nx > 0 ? nx : 1));
    if (!fn) return DDO_ENOMEM;
    if (check_every < 1) check_every = 1;
    int par = 0;
#ifdef _OPENMP
    par = !omp_in_parallel() && nt > 1 && (double)nx * (double)ny > 2e5;
#endif
    (void)nt;
    int it = 0, rc = DDO_ENOCONV;
    double e = INFINITY;
    while (1) {
        /* Y-iteration */
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nt) if (par)
#endif
        for (int y = 0; y < ny; ++y)
            g[y] = (b[y] > 0.0) ? eps * log(b[y]) - lse_col(nx, ny, f, C, y, eps) : -INFINITY;
        /* X-iteration */
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nt) if (par)
#endif
        for (int x = 0; x < nx; ++x)
            fn[x] = (a[x] > 0.0) ? eps * log(a[x]) - lse_row(ny, g, C + (size_t)x * ny, eps)
                                 : -INFINITY;
        /* L1 error of the X-marginal of the plan (f, g) */
        e = 0.0;
        for (int x = 0; x < nx; ++x)
            if (a[x] > 0.0) e += a[x] * fabs(expm1((f[x] - fn[x]) / eps));
        ++it;
        if (e <= tol && it % check_every == 0) { rc = DDO_OK; break; }
        if (it >= max_iter) { rc = DDO_ENOCONV; break; }
        memcpy(f, fn, sizeof(double) * (size_t)nx);
    }
    free(fn);
    if (iters) *iters = it;
    if (err) *err = e;
    if (!isfinite(e)) return DDO_ENUMERIC;
    return rc;
}

int ddo_sinkhorn_dense(int nx, int ny, const double* a, const double* b, const double* C,
                       double eps, double tol, int max_iter, double* f, double* g,
                       int* iters, double* err) {
    return sinkhorn_dense_k(nx, ny, a, b, C, eps, tol, max_iter, 1, 1, f, g, iters, err);
}

/* -------------------------------------------------------------- schedule -- */
/* at each layer eps = 2 dx_l^2 for 4 sweeps, then dx_l^2 and
 * 0.5 dx_l^2 for 2 sweeps each, then refine.  Finest layer: keep halving
 * (2 sweeps each) down to kappa_final (paper: 0.25; BASELINE: 0.5).
 * eps_start (config 2): prepend kappa_start, kappa_start/2, ... > 2 at the
 * coarsest layer, 2 sweeps each (reading A12). */
int ddo_build_schedule(int n_final, int coarsest_side, double kappa_final, double eps_start,
                       int* side, double* kappa, int* sweeps, int max) {
    int k = 0;
#define PUSH(S, K, W)                                                      \
    do {                                                                   \
        if (k < max) { side[k] = (S); kappa[k] = (K); sweeps[k] = (W); }   \
        ++k;                                                               \
    } while (0)
    if (coarsest_side <= 0) coarsest_side = 8;
    if (coarsest_side > n_final) coarsest_side = n_final;
    for (int sd = coarsest_side; sd <= n_final; sd *= 2) {
        int finest = (sd == n_final);
        if (sd == coarsest_side && eps_start > 0.0) {
            double ks = eps_start * (double)sd * (double)sd;
            for (double kk = ks; kk > 2.0 * (1.0 + 1e-12); kk *= 0.5) PUSH(sd, kk, 2);
        }
        if (finest && kappa_final > 2.0 * (1.0 + 1e-12)) {
            PUSH(sd, kappa_final, 4);
            continue;
        }
        PUSH(sd, 2.0, 4);
        if (!finest) {
            PUSH(sd, 1.0, 2);
            PUSH(sd, 0.5, 2);
        } else {
            for (double kk = 1.0; kk >= kappa_final * (1.0 - 1e-12); kk *= 0.5) PUSH(sd, kk, 2);
        }
    }
#undef PUSH
    return k;
}

/* ------------------------------------------------------------ partitions -- */
/* A = 2x2 blocks of basic cells; B = same with an offset of one
 * basic cell (2x1 on edges, 1x1 in corners).  Members in row-major order. */
static int n_cells_axis(int nb, int part) { return part == 1 ? nb / 2 : nb / 2 + 1; }

static void cell_rows(int nb, int part, int p, int* lo, int* hi) {
    if (part == 1) { *lo = 2 * p; *hi = 2 * p + 1; }
    else {
        *lo = 2 * p - 1 < 0 ? 0 : 2 * p - 1;
        *hi = 2 * p > nb - 1 ? nb - 1 : 2 * p;
    }
}

/* ----------------------------------------------------------------- layers -- */
static void free_state(ddo_ctx* c) {
    if (c->val) {
        int nb = c->L[c->cur].nb;
        for (int i = 0; i < nb * nb; ++i) free(c->val[i]);
        free(c->val);
        c->val = NULL;
    }
    free(c->box); c->box = NULL;
    free(c->alphaA); c->alphaA = NULL;
    free(c->alphaB); c->alphaB = NULL;
}

static int alloc_state(ddo_ctx* c) {
    layer_t* L = &c->L[c->cur];
    size_t nb2 = (size_t)L->nb * L->nb, n2 = (size_t)L->side * L->side;
    c->box = (int*)calloc(nb2 * 4, sizeof(int));
    c->val = (double**)calloc(nb2, sizeof(double*));
    c->alphaA = (double*)calloc(n2, sizeof(double));
    c->alphaB = (double*)calloc(n2, sizeof(double));
    return (c->box && c->val && c->alphaA && c->alphaB) ? DDO_OK : DDO_ENOMEM;
}

/* Product initialisation nu_i = ||mu_i|| nu (reading A3), alpha = 0. */
static int product_init(ddo_ctx* c) {
    layer_t* L = &c->L[c->cur];
    int nb = L->nb, n = L->side;
    for (int i = 0; i < nb * nb; ++i) {
        c->box[4 * i + 0] = 0; c->box[4 * i + 1] = 0;
        c->box[4 * i + 2] = n; c->box[4 * i + 3] = n;
        c->val[i] = (double*)malloc(sizeof(double) * (size_t)n * n);
        if (!c->val[i]) return DDO_ENOMEM;
        for (int y = 0; y < n * n; ++y) c->val[i][y] = L->mass_i[i] * L->nu[y];
    }
    return DDO_OK;
}

void ddo_free(ddo_ctx* c) {
    if (!c) return;
    free_state(c);
    for (int k = 0; k < c->n_layers; ++k) {
        free(c->L[k].mu); free(c->L[k].nu); free(c->L[k].logmu); free(c->L[k].mass_i);
    }
    free(c->h1); free(c->h2);
    free(c);
}

const char* ddo_last_error(const ddo_ctx* c) { return c ? c->err : "null context"; }

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

int ddo_init(ddo_ctx** out, int n, const double* mu, const double* nu, double eps,
             int cell_size, const ddo_options* opt) {
    if (!out) return DDO_EINVAL;
    *out = NULL;
    ddo_ctx* c = (ddo_ctx*)calloc(1, sizeof(ddo_ctx));
    if (!c) return DDO_ENOMEM;
    if (opt) c->opt = *opt;
    if (c->opt.err_tol <= 0) c->opt.err_tol = 1e-6;
    if (c->opt.max_inner_iter <= 0) c->opt.max_inner_iter = 10000;
    if (c->opt.check_every <= 0) c->opt.check_every = 1;
    c->tau = c->opt.trunc_tau == 0.0 ? 1e-15 : (c->opt.trunc_tau < 0 ? 0.0 : c->opt.trunc_tau);
    if (c->opt.no_truncate) c->tau = 0.0;
    *out = c;
    if (!is_pow2(n) || n < 4) { set_err(c, "n=%d must be a power of two >= 4", n); return DDO_EINVAL; }
    if (!is_pow2(cell_size) || cell_size > n / 2 || (n / cell_size) % 2) {
        set_err(c, "cell_size=%d must be a power of two with n/s even", cell_size);
        return DDO_EINVAL;
    }
    if (!(eps > 0.0) || !isfinite(eps)) { set_err(c, "eps must be > 0"); return DDO_EINVAL; }
    if (!mu || !nu) { set_err(c, "null marginal"); return DDO_EINVAL; }
    ksum_t ksm = {0, 0}, ksn = {0, 0};      /* compensated (A17): input validation only */
    for (size_t k = 0; k < (size_t)n * n; ++k) {
        if (!isfinite(mu[k]) || mu[k] < 0 || !isfinite(nu[k]) || nu[k] < 0) {
            set_err(c, "marginals must be finite and >= 0 (index %zu)", k);
            return DDO_EINVAL;
        }
        ks_add(&ksm, mu[k]); ks_add(&ksn, nu[k]);
    }
    double smu = ks_get(&ksm), snu = ks_get(&ksn);
    if (!(smu > 0) || fabs(smu - snu) > 1e-12 * smu) {
        set_err(c, "||mu|| = %.17g != ||nu|| = %.17g", smu, snu);
        return DDO_EINVAL;
    }
    int coarsest = n;
    if (c->opt.schedule == DDO_SCHED_LADDER) {
        coarsest = c->opt.coarsest_side > 0 ? c->opt.coarsest_side : 8;
        if (!is_pow2(coarsest) || coarsest < 4) { set_err(c, "bad coarsest_side"); return DDO_EINVAL; }
        if (coarsest > n) coarsest = n;
    }
    /* layers coarsest .. n; images by 2x2 sum pooling of the finest (A20) */
    int nl = 0;
    for (int sd = coarsest; sd <= n; sd *= 2) ++nl;
    if (nl > MAX_LAYERS) { set_err(c, "too many layers"); return DDO_EINVAL; }
    c->n_layers = nl;
    c->n_final = n;
    for (int k = nl - 1; k >= 0; --k) {
        layer_t* L = &c->L[k];
        L->side = coarsest << k;
        L->s = cell_size < L->side / 2 ? cell_size : L->side / 2;   /* reading A19 */
        L->nb = L->side / L->s;
        size_t n2 = (size_t)L->side * L->side;
        L->mu = (double*)malloc(sizeof(double) * n2);
        L->nu = (double*)malloc(sizeof(double) * n2);
        L->logmu = (double*)malloc(sizeof(double) * n2);
        L->mass_i = (double*)calloc((size_t)L->nb * L->nb, sizeof(double));
        if (!L->mu || !L->nu || !L->logmu || !L->mass_i) return DDO_ENOMEM;
        if (k == nl - 1) {
            memcpy(L->mu, mu, sizeof(double) * n2);
            memcpy(L->nu, nu, sizeof(double) * n2);
        } else {
            layer_t* F = &c->L[k + 1];
            for (int i = 0; i < L->side; ++i)
                for (int j = 0; j < L->side; ++j) {
                    size_t a = (size_t)(2 * i) * F->side + 2 * j;
                    L->mu[(size_t)i * L->side + j] =
                        F->mu[a] + F->mu[a + 1] + F->mu[a + F->side] + F->mu[a + F->side + 1];
                    L->nu[(size_t)i * L->side + j] =
                        F->nu[a] + F->nu[a + 1] + F->nu[a + F->side] + F->nu[a + F->side + 1];
                }
        }
        for (size_t q = 0; q < n2; ++q) L->logmu[q] = L->mu[q] > 0 ? log(L->mu[q]) : -INFINITY;
        for (int i = 0; i < L->side; ++i)
            for (int j = 0; j < L->side; ++j)
                L->mass_i[(i / L->s) * L->nb + (j / L->s)] += L->mu[(size_t)i * L->side + j];
        for (int q = 0; q < L->nb * L->nb; ++q)
            if (!(L->mass_i[q] > 0)) {
                set_err(c, "basic cell %d of layer side %d has zero mass (P:299)", q, L->side);
                return DDO_EINVAL;
            }
    }
    c->cur = 0;
    c->eps_final = eps;
    c->eps = (c->opt.schedule == DDO_SCHED_LADDER) ? 2.0 / ((double)coarsest * coarsest) : eps;
    int rc = alloc_state(c);
    if (rc) { set_err(c, "out of memory"); return rc; }
    if (!c->opt.empty_init) {
        rc = product_init(c);
        if (rc) { set_err(c, "out of memory"); return rc; }
    }
    c->half_index = 0;
    c->last_part = 0;
    return DDO_OK;
}

int ddo_set_eps(ddo_ctx* c, double eps) {
    if (!c || !(eps > 0.0)) return DDO_EINVAL;
    c->eps = eps;   /* alpha = eps log u is kept constant (reading A13) */
    return DDO_OK;
}

/* --------------------------------------------------------- one cell solve -- */
typedef struct {
    int members[4], nmem;        /* basic-cell indices */
    int mr[4], mc[4];            /* member basic row/col */
    int R0, C0, ar, ac;          /* X pixel region */
    int yr0, yc0, br, bc;        /* union Y box */
} cellgeo_t;

static void cell_geometry(const ddo_ctx* c, int part, int cidx, cellgeo_t* G) {
    const layer_t* L = &c->L[c->cur];
    int nca = n_cells_axis(L->nb, part);
    int p = cidx / nca, q = cidx % nca;
    int rlo, rhi, clo, chi;
    cell_rows(L->nb, part, p, &rlo, &rhi);
    cell_rows(L->nb, part, q, &clo, &chi);
    G->nmem = 0;
    for (int r = rlo; r <= rhi; ++r)
        for (int cc = clo; cc <= chi; ++cc) {
            G->mr[G->nmem] = r; G->mc[G->nmem] = cc;
            G->members[G->nmem++] = r * L->nb + cc;
        }
    G->R0 = rlo * L->s; G->C0 = clo * L->s;
    G->ar = (rhi - rlo + 1) * L->s; G->ac = (chi - clo + 1) * L->s;
    /* union bounding box of the member boxes (empty boxes ignored) */
    int y0 = 1 << 30, x0 = 1 << 30, y1 = -1, x1 = -1;
    for (int m = 0; m < G->nmem; ++m) {
        const int* b = &c->box[4 * G->members[m]];
        if (b[2] <= 0 || b[3] <= 0) continue;
        if (b[0] < y0) y0 = b[0];
        if (b[1] < x0) x0 = b[1];
        if (b[0] + b[2] - 1 > y1) y1 = b[0] + b[2] - 1;
        if (b[1] + b[3] - 1 > x1) x1 = b[1] + b[3] - 1;
    }
    if (y1 < 0) { G->yr0 = G->yc0 = 0; G->br = G->bc = 0; }
    else { G->yr0 = y0; G->yc0 = x0; G->br = y1 - y0 + 1; G->bc = x1 - x0 + 1; }
}

/* Ground cost between pixels (r1, c1) and (r2, c2) of a layer of the given side,
 * [0,1]^2 units, pixel centres: |x-y|^2 (W2), or the separable table
 * cost h1(|x1-y1|) + h2(|x2-y2|) (ddo_set_cost): a layer pixel difference d is
 * d * n_final / side finest pixels (centres of coarse pixels are finest-grid
 * distances apart). */
static double ground_cost(const ddo_ctx* c, int side, int r1, int c1, int r2, int c2) {
    if (c->h1) {
        const int st = c->n_final / side;
        return c->h1[abs(r1 - r2) * st] + c->h2[abs(c1 - c2) * st];
    }
    const double h = 1.0 / side;
    const double d1 = (r1 - r2) * h, d2 = (c1 - c2) * h;
    return d1 * d1 + d2 * d2;
}

int ddo_set_cost(ddo_ctx* c, int n_entries, const double* h1, const double* h2) {
    if (!c) return DDO_EINVAL;
    free(c->h1); free(c->h2);
    c->h1 = c->h2 = NULL;
    if (!h1 && !h2) return DDO_OK;
    if (!h1 || !h2 || n_entries != c->n_final) {
        set_err(c, "ddo_set_cost: two tables of n = %d entries required", c->n_final);
        return DDO_EINVAL;
    }
    for (int d = 0; d < n_entries; ++d)
        if (!isfinite(h1[d]) || !isfinite(h2[d])) { set_err(c, "ddo_set_cost: non-finite entry %d", d); return DDO_EINVAL; }
    c->h1 = (double*)malloc(sizeof(double) * n_entries);
    c->h2 = (double*)malloc(sizeof(double) * n_entries);
    if (!c->h1 || !c->h2) return DDO_ENOMEM;
    memcpy(c->h1, h1, sizeof(double) * n_entries);
    memcpy(c->h2, h2, sizeof(double) * n_entries);
    return DDO_OK;
}

/* Dense problem of one composite cell: a = mu_J, b = nu_cell = sum_{i in J} nu_i
 * (Alg. 2 line 8), cost c(x,y) (ground_cost), f = alpha + eps log mu. */
typedef struct {
    int nx, ny;
    double *a, *b, *C, *f, *g;
} cellprob_t;

static void free_prob(cellprob_t* P) {
    free(P->a); free(P->b); free(P->C); free(P->f); free(P->g);
    memset(P, 0, sizeof(*P));
}

static int build_prob(const ddo_ctx* c, const cellgeo_t* G, const double* alpha, cellprob_t* P) {
    const layer_t* L = &c->L[c->cur];
    double h = 1.0 / L->side;
    P->nx = G->ar * G->ac;
    P->ny = G->br * G->bc;
    P->a = (double*)malloc(sizeof(double) * (size_t)P->nx);
    P->f = (double*)malloc(sizeof(double) * (size_t)P->nx);
    P->b = (double*)calloc((size_t)(P->ny > 0 ? P->ny : 1), sizeof(double));
    P->g = (double*)malloc(sizeof(double) * (size_t)(P->ny > 0 ? P->ny : 1));
    P->C = (double*)malloc(sizeof(double) * (size_t)P->nx * (size_t)(P->ny > 0 ? P->ny : 1));
    if (!P->a || !P->f || !P->b || !P->g || !P->C) return DDO_ENOMEM;
    for (int xr = 0; xr < G->ar; ++xr)
        for (int xc = 0; xc < G->ac; ++xc) {
            size_t gx = (size_t)(G->R0 + xr) * L->side + (G->C0 + xc);
            int x = xr * G->ac + xc;
            P->a[x] = L->mu[gx];
            P->f[x] = (L->mu[gx] > 0) ? alpha[gx] + c->eps * L->logmu[gx] : -INFINITY;
        }
    for (int m = 0; m < G->nmem; ++m) {
        const int* bx = &c->box[4 * G->members[m]];
        const double* v = c->val[G->members[m]];
        for (int r = 0; r < bx[2]; ++r)
            for (int q = 0; q < bx[3]; ++q) {
                int y = (bx[0] + r - G->yr0) * G->bc + (bx[1] + q - G->yc0);
                P->b[y] += v[(size_t)r * bx[3] + q];
            }
    }
    for (int x = 0; x < P->nx; ++x) {
        if (c->h1) {
            for (int y = 0; y < P->ny; ++y)
                P->C[(size_t)x * P->ny + y] = ground_cost(c, L->side, G->R0 + x / G->ac, G->C0 + x % G->ac,
                                                          G->yr0 + y / G->bc, G->yc0 + y % G->bc);
            continue;
        }
        double x1 = (G->R0 + x / G->ac + 0.5) * h, x2 = (G->C0 + x % G->ac + 0.5) * h;
        for (int y = 0; y < P->ny; ++y) {
            double y1 = (G->yr0 + y / G->bc + 0.5) * h, y2 = (G->yc0 + y % G->bc + 0.5) * h;
            P->C[(size_t)x * P->ny + y] = (x1 - y1) * (x1 - y1) + (x2 - y2) * (x2 - y2);
        }
    }
    return DDO_OK;
}

static double plan_entry(const cellprob_t* P, int x, int y, double eps) {
    if (P->f[x] == -INFINITY || P->g[y] == -INFINITY) return 0.0;
    return exp((P->f[x] + P->g[y] - P->C[(size_t)x * P->ny + y]) / eps);
}

/* BalanceMeasures (reading A8): proportional transfer from
 * donors (d_i > 0) to receivers (d_i < 0), amount T = min(sum d_+, sum -d_-),
 * preserving the pointwise sum and non-negativity, no new support. */
static void balance(int nmem, int ny, double** nu_i, const double* target) {
    double norm[4], d[4], Dsum = 0, Psum = 0, dmax = 0;
    for (int m = 0; m < nmem; ++m) {
        double s = 0;
        for (int y = 0; y < ny; ++y) s += nu_i[m][y];
        norm[m] = s;
        d[m] = s - target[m];
        if (fabs(d[m]) > dmax) dmax = fabs(d[m]);
        if (d[m] > 0) Dsum += d[m];
        else Psum += -d[m];
    }
    if (dmax <= 1e-18 || Dsum <= 0 || Psum <= 0) return;
    double T = Dsum < Psum ? Dsum : Psum;
    for (int y = 0; y < ny; ++y) {
        double r = 0;
        for (int m = 0; m < nmem; ++m)
            if (d[m] > 0) {
                double take = nu_i[m][y] * (d[m] / norm[m]) * (T / Dsum);
                nu_i[m][y] -= take;
                r += take;
            }
        for (int m = 0; m < nmem; ++m)
            if (d[m] < 0) nu_i[m][y] += r * (-d[m]) / Psum;
    }
}

typedef struct { int iters, flag, safeguard; double err; } cellres_t;

/* Algorithm 2 lines 8-13 for one composite cell J of partition part. */
static int solve_cell(ddo_ctx* c, int part, int cidx, cellres_t* res) {
    layer_t* L = &c->L[c->cur];
    double* alpha = part == 1 ? c->alphaA : c->alphaB;
    cellgeo_t G;
    cell_geometry(c, part, cidx, &G);
    cellprob_t P;
    memset(&P, 0, sizeof(P));
    int rc = build_prob(c, &G, alpha, &P);
    if (rc) { free_prob(&P); return rc; }
    double muJ = 0;
    for (int x = 0; x < P.nx; ++x) muJ += P.a[x];
    /* line 9: pi_cell, u_{C,J} <- Sinkhorn(mu_J, nu_cell, u_{C,J}) */
    int it = 0;
    double err = 0;
    int nt = 1;
#ifdef _OPENMP
    nt = c->opt.n_threads > 0 ? c->opt.n_threads : omp_get_max_threads();
#endif
    double* f_in = NULL;
    if (c->opt.safeguard) {
        f_in = (double*)malloc(sizeof(double) * (size_t)(P.nx > 0 ? P.nx : 1));
        if (!f_in) { free_prob(&P); return DDO_ENOMEM; }
        memcpy(f_in, P.f, sizeof(double) * (size_t)P.nx);
    }
    int src = sinkhorn_dense_k(P.nx, P.ny, P.a, P.b, P.C, c->eps, muJ * c->opt.err_tol,
                               c->opt.max_inner_iter, c->opt.check_every, nt, P.f, P.g, &it, &err);
    res->safeguard = 0;
    if (src != DDO_OK && c->opt.safeguard) {
        /* eps-raising safeguard ("temporarily increasing eps"; S:281 retry at
         * 2x eps, rescale the potential back, re-solve at the target eps; S:323 at
         * most 3 attempts; A29): attempt k starts from the cell's input
         * alpha = f_in - eps log mu at eps_k = 2^k eps, then keeps alpha (the eps
         * change rule P:1510) and solves at eps; every stage to the same tolerance
         * and iteration cap. */
        res->safeguard = 1;
        for (int k = 1; k <= 3 && src != DDO_OK; ++k) {
            const double ek = ldexp(c->eps, k);
            for (int x = 0; x < P.nx; ++x)
                P.f[x] = (P.a[x] > 0.0) ? f_in[x] - c->eps * log(P.a[x]) + ek * log(P.a[x]) : -INFINITY;
            int i1 = 0, i2 = 0;
            sinkhorn_dense_k(P.nx, P.ny, P.a, P.b, P.C, ek, muJ * c->opt.err_tol,
                             c->opt.max_inner_iter, c->opt.check_every, nt, P.f, P.g, &i1, &err);
            for (int x = 0; x < P.nx; ++x)
                if (P.a[x] > 0.0) P.f[x] = P.f[x] - ek * log(P.a[x]) + c->eps * log(P.a[x]);
            src = sinkhorn_dense_k(P.nx, P.ny, P.a, P.b, P.C, c->eps, muJ * c->opt.err_tol,
                                   c->opt.max_inner_iter, c->opt.check_every, nt, P.f, P.g, &i2, &err);
            it += i1 + i2;
        }
    }
    free(f_in);
    res->iters = it; res->err = err; res->flag = src;
    /* line 10: nu_i <- P_Y(pi_cell restricted to X_i x Y) */
    double* nu_i[4];
    double target[4];
    for (int m = 0; m < G.nmem; ++m) {
        nu_i[m] = (double*)calloc((size_t)(P.ny > 0 ? P.ny : 1), sizeof(double));
        if (!nu_i[m]) { free_prob(&P); return DDO_ENOMEM; }
        target[m] = L->mass_i[G.members[m]];
    }
    for (int x = 0; x < P.nx; ++x) {
        int xr = x / G.ac, xc = x % G.ac;
        int br = (G.R0 + xr) / L->s, bcc = (G.C0 + xc) / L->s;
        int m = 0;
        while (m < G.nmem && !(G.mr[m] == br && G.mc[m] == bcc)) ++m;
        for (int y = 0; y < P.ny; ++y) nu_i[m][y] += plan_entry(&P, x, y, c->eps);
    }
    /* line 11: BalanceMeasures */
    balance(G.nmem, P.ny, nu_i, target);
    /* line 12: Truncate (entries < tau dropped; tight bounding box kept, reading A9/A10) */
    for (int m = 0; m < G.nmem; ++m) {
        int y0 = 1 << 30, x0 = 1 << 30, y1 = -1, x1 = -1;
        for (int y = 0; y < P.ny; ++y) {
            if (nu_i[m][y] < c->tau || nu_i[m][y] <= 0.0) { nu_i[m][y] = 0.0; continue; }
            int r = y / G.bc, q = y % G.bc;
            if (r < y0) y0 = r;
            if (r > y1) y1 = r;
            if (q < x0) x0 = q;
            if (q > x1) x1 = q;
        }
        int i = G.members[m];
        free(c->val[i]);
        c->val[i] = NULL;
        int* bx = &c->box[4 * i];
        if (y1 < 0) { bx[0] = G.yr0; bx[1] = G.yc0; bx[2] = 0; bx[3] = 0; }
        else {
            bx[0] = G.yr0 + y0; bx[1] = G.yc0 + x0; bx[2] = y1 - y0 + 1; bx[3] = x1 - x0 + 1;
            c->val[i] = (double*)malloc(sizeof(double) * (size_t)bx[2] * bx[3]);
            if (!c->val[i]) { free_prob(&P); return DDO_ENOMEM; }
            for (int r = 0; r < bx[2]; ++r)
                for (int q = 0; q < bx[3]; ++q)
                    c->val[i][(size_t)r * bx[3] + q] = nu_i[m][(size_t)(y0 + r) * G.bc + (x0 + q)];
        }
        free(nu_i[m]);
    }
    /* store u_{C,J} as alpha = f - eps log mu (plan's f; reading A4) */
    for (int xr = 0; xr < G.ar; ++xr)
        for (int xc = 0; xc < G.ac; ++xc) {
            size_t gx = (size_t)(G.R0 + xr) * L->side + (G.C0 + xc);
            double fx = P.f[xr * G.ac + xc];
            alpha[gx] = (L->mu[gx] > 0 && isfinite(fx)) ? fx - c->eps * L->logmu[gx] : 0.0;
        }
    free_prob(&P);
    return DDO_OK;
}

static int n_cells(const ddo_ctx* c, int part) {
    int nca = n_cells_axis(c->L[c->cur].nb, part);
    return nca * nca;
}

/* Algorithm 2 lines 6-14: one sweep over the selected partition. */
static int sweep(ddo_ctx* c) {
    int part = (c->half_index % 2 == 0) ? 1 : 2;   /* l odd -> A (l = half_index+1) */
    int nc = n_cells(c, part);
    cellres_t* res = (cellres_t*)calloc((size_t)nc, sizeof(cellres_t));
    int* rcs = (int*)calloc((size_t)nc, sizeof(int));
    if (!res || !rcs) { free(res); free(rcs); return DDO_ENOMEM; }
#ifdef _OPENMP
    int nt = c->opt.n_threads > 0 ? c->opt.n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int j = 0; j < nc; ++j) rcs[j] = solve_cell(c, part, j, &res[j]);
    int rc = DDO_OK;
    ddo_sweep_stats st;
    memset(&st, 0, sizeof(st));
    st.cells = nc;
    for (int j = 0; j < nc; ++j) {     /* fixed-order reduction */
        if (rcs[j] == DDO_ENOMEM) rc = DDO_ENOMEM;
        st.iters_sum += res[j].iters;
        if (res[j].iters > st.iters_max) st.iters_max = res[j].iters;
        st.err_x_sum += res[j].err;
        st.safeguarded += res[j].safeguard;
        if (res[j].flag != DDO_OK) {
            st.failed++;
            if (rc == DDO_OK) rc = res[j].flag;
        }
    }
    layer_t* L = &c->L[c->cur];
    for (int i = 0; i < L->nb * L->nb; ++i) st.entries += (long long)c->box[4 * i + 2] * c->box[4 * i + 3];
    c->stats = st;
    c->half_index++;
    c->last_part = part;
    free(res);
    free(rcs);
    if (rc == DDO_ENOCONV) set_err(c, "%d cells hit max_inner_iter", st.failed);
    if (rc == DDO_ENUMERIC) set_err(c, "non-finite marginal error in %d cells", st.failed);
    return rc;
}

int ddo_solve_cells(ddo_ctx* c, int part, int n, const int* cells, int* iters) {
    if (!c || (part != 1 && part != 2) || n < 0 || (n && !cells)) return DDO_EINVAL;
    int nc = n_cells(c, part);
    int rc = DDO_OK;
    for (int k = 0; k < n; ++k) {
        if (cells[k] < 0 || cells[k] >= nc) { set_err(c, "cell %d out of range", cells[k]); return DDO_EINVAL; }
        cellres_t r;
        memset(&r, 0, sizeof(r));
        int s = solve_cell(c, part, cells[k], &r);
        if (iters) iters[k] = r.iters;
        if (s == DDO_ENOMEM) return s;
        if (!rc && r.flag) rc = r.flag;
    }
    return rc;
}

/* The same for a batch of cells solved concurrently, one OpenMP thread per
 * cell as in a sweep (cells of one partition are disjoint).  Used to
 * time the oracle's sweep throughput on a sample of a sweep's cells. */
int ddo_solve_cells_par(ddo_ctx* c, int part, int n, const int* cells, int* iters) {
    if (!c || (part != 1 && part != 2) || n < 0 || (n && !cells)) return DDO_EINVAL;
    int nc = n_cells(c, part);
    for (int k = 0; k < n; ++k)
        if (cells[k] < 0 || cells[k] >= nc) { set_err(c, "cell %d out of range", cells[k]); return DDO_EINVAL; }
    cellres_t* res = (cellres_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(cellres_t));
    int* rcs = (int*)calloc((size_t)(n > 0 ? n : 1), sizeof(int));
    if (!res || !rcs) { free(res); free(rcs); return DDO_ENOMEM; }
#ifdef _OPENMP
    int nt = c->opt.n_threads > 0 ? c->opt.n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int k = 0; k < n; ++k) rcs[k] = solve_cell(c, part, cells[k], &res[k]);
    int rc = DDO_OK;
    for (int k = 0; k < n; ++k) {
        if (iters) iters[k] = res[k].iters;
        if (rcs[k] == DDO_ENOMEM) rc = DDO_ENOMEM;
        if (!rc && res[k].flag) rc = res[k].flag;
    }
    free(res);
    free(rcs);
    return rc;
}

int ddo_iterate(ddo_ctx* c, int n_half_iters) {
    if (!c) return DDO_EINVAL;
    int rc = DDO_OK;
    for (int k = 0; k < n_half_iters; ++k) {
        int r = sweep(c);
        if (r == DDO_ENOMEM || r == DDO_ENUMERIC) return r;
        if (r) rc = r;
    }
    return rc;
}

/* ------------------------------------------------------------ refinement -- */
static int glue_alpha(ddo_ctx* c, double* ah);

/* P:1508 "linear interpolation onto the fine points (in log space)": alpha
 * = eps log u is the log-space potential; bilinear in coarse pixel-index
 * coordinates at the fine pixel centres, (i + 1/2)/2 - 1/2, constant
 * beyond the outermost coarse centres (reading A26). */
static double interp_bilinear(const double* ph, int sc, int i, int j) {
    double u = 0.5 * i - 0.25, v = 0.5 * j - 0.25;
    if (u < 0.0) u = 0.0;
    if (v < 0.0) v = 0.0;
    if (u > sc - 1) u = sc - 1;
    if (v > sc - 1) v = sc - 1;
    int i0 = (int)u, j0 = (int)v;
    int i1 = i0 + 1 < sc ? i0 + 1 : i0, j1 = j0 + 1 < sc ? j0 + 1 : j0;
    double fu = u - i0, fv = v - j0;
    double top = ph[(size_t)i0 * sc + j0] * (1.0 - fv) + ph[(size_t)i0 * sc + j1] * fv;
    double bot = ph[(size_t)i1 * sc + j0] * (1.0 - fv) + ph[(size_t)i1 * sc + j1] * fv;
    return top * (1.0 - fu) + bot * fu;
}

/* eq. FineBasicMarginals:
 *   nu_i^0(y) = nu(y) * nuhat_{Pa(i)}(pa(y)) / nuhat(pa(y)) * mu(X_i) / muhat(Xhat_{Pa(i)})
 * with 0/0 := 0.  Fine box = 2x the parent box.  alpha cold start (A14). */
int ddo_refine(ddo_ctx* c) {
    if (!c) return DDO_EINVAL;
    if (c->cur + 1 >= c->n_layers) { set_err(c, "already at the finest layer"); return DDO_EINVAL; }
    layer_t* Lc = &c->L[c->cur];
    layer_t* Lf = &c->L[c->cur + 1];
    int nbc = Lc->nb, nbf = Lf->nb;
    double* ah = NULL;                  /* glued coarse potentials (warm_refine) */
    if (c->opt.warm_refine && c->last_part != 0) {
        ah = (double*)malloc((size_t)Lc->side * Lc->side * sizeof(double));
        if (!ah) return DDO_ENOMEM;
        int rc = glue_alpha(c, ah);
        if (rc) { free(ah); return rc; }
    }
    int* nbox = (int*)calloc((size_t)nbf * nbf * 4, sizeof(int));
    double** nval = (double**)calloc((size_t)nbf * nbf, sizeof(double*));
    if (!nbox || !nval) return DDO_ENOMEM;
    for (int ir = 0; ir < nbf; ++ir)
        for (int ic = 0; ic < nbf; ++ic) {
            int i = ir * nbf + ic;
            int jr = ir * nbc / nbf, jc = ic * nbc / nbf;   /* Pa(i) */
            int j = jr * nbc + jc;
            const int* pb = &c->box[4 * j];
            int* fb = &nbox[4 * i];
            fb[0] = 2 * pb[0]; fb[1] = 2 * pb[1]; fb[2] = 2 * pb[2]; fb[3] = 2 * pb[3];
            double ratio_mu = Lf->mass_i[i] / Lc->mass_i[j];
            size_t area = (size_t)fb[2] * fb[3];
            nval[i] = (double*)malloc(sizeof(double) * (area > 0 ? area : 1));
            if (!nval[i]) return DDO_ENOMEM;
            for (int r = 0; r < fb[2]; ++r)
                for (int q = 0; q < fb[3]; ++q) {
                    int y1 = fb[0] + r, y2 = fb[1] + q;          /* fine Y pixel */
                    int p1 = y1 / 2, p2 = y2 / 2;                /* pa(y) */
                    double nuhat_j = c->val[j][(size_t)(p1 - pb[0]) * pb[3] + (p2 - pb[1])];
                    double nuhat = Lc->nu[(size_t)p1 * Lc->side + p2];
                    double nuy = Lf->nu[(size_t)y1 * Lf->side + y2];
                    nval[i][(size_t)r * fb[3] + q] =
                        (nuhat > 0.0) ? nuy * (nuhat_j / nuhat) * ratio_mu : 0.0;
                }
        }
    free_state(c);
    c->cur += 1;
    c->box = nbox;
    c->val = nval;
    size_t n2 = (size_t)Lf->side * Lf->side;
    c->alphaA = (double*)calloc(n2, sizeof(double));
    c->alphaB = (double*)calloc(n2, sizeof(double));
    if (!c->alphaA || !c->alphaB) { free(ah); return DDO_ENOMEM; }
    if (ah) {                           /* both partitions start from the same alpha */
        for (int i = 0; i < Lf->side; ++i)
            for (int j = 0; j < Lf->side; ++j) {
                double a = interp_bilinear(ah, Lc->side, i, j);
                c->alphaA[(size_t)i * Lf->side + j] = a;
                c->alphaB[(size_t)i * Lf->side + j] = a;
            }
        free(ah);
    }
    c->last_part = 0;
    return DDO_OK;
}

int ddo_run_schedule(ddo_ctx* c) {
    if (!c) return DDO_EINVAL;
    int sides[256], sweeps[256];
    double kap[256];
    int ns;
    if (c->opt.schedule == DDO_SCHED_LADDER) {
        int nf = c->L[c->n_layers - 1].side;
        double kf = c->eps_final * (double)nf * nf;
        ns = ddo_build_schedule(nf, c->L[0].side, kf, c->opt.eps_start, sides, kap, sweeps, 256);
    } else {
        ns = 0;
        set_err(c, "run_schedule needs DDO_SCHED_LADDER");
        return DDO_EINVAL;
    }
    int rc = DDO_OK;
    for (int k = 0; k < ns && k < 256; ++k) {
        while (c->L[c->cur].side < sides[k]) {
            int r = ddo_refine(c);
            if (r) return r;
        }
        double h = 1.0 / sides[k];
        ddo_set_eps(c, kap[k] * h * h);
        int r = ddo_iterate(c, sweeps[k]);
        if (r == DDO_ENOMEM || r == DDO_ENUMERIC) return r;
        if (r) rc = r;
    }
    return rc;
}

/* ------------------------------------------------------------ evaluation -- */
/* Primal evaluation (reading A15): for each cell J of the last swept
 * partition (A if none), rebuild nu_cell = sum_{i in J} nu_i and the cell
 * plan pi_J = exp((f + g - c)/eps) with f = alpha_{C,J} + eps log mu and g
 * from one Y-iteration; pi = sum_J pi_J. */
typedef struct { double cost, ent, l1x, mass; } evalres_t;

static int eval_cell(ddo_ctx* c, int part, int cidx, evalres_t* er, long long* count,
                     int* xi, int* yi, double* mass, long long base) {
    layer_t* L = &c->L[c->cur];
    double* alpha = part == 1 ? c->alphaA : c->alphaB;
    cellgeo_t G;
    cell_geometry(c, part, cidx, &G);
    cellprob_t P;
    memset(&P, 0, sizeof(P));
    int rc = build_prob(c, &G, alpha, &P);
    if (rc) { free_prob(&P); return rc; }
    for (int y = 0; y < P.ny; ++y)
        P.g[y] = (P.b[y] > 0.0) ? c->eps * log(P.b[y]) - lse_col(P.nx, P.ny, P.f, P.C, y, c->eps)
                                : -INFINITY;
    ksum_t cost = {0, 0}, ent = {0, 0}, l1x = {0, 0}, ms = {0, 0};
    long long k = 0;
    for (int x = 0; x < P.nx; ++x) {
        size_t gx = (size_t)(G.R0 + x / G.ac) * L->side + (G.C0 + x % G.ac);
        double px = 0;
        for (int y = 0; y < P.ny; ++y) {
            double p = plan_entry(&P, x, y, c->eps);
            if (!(p > 0.0)) continue;
            size_t gy = (size_t)(G.yr0 + y / G.bc) * L->side + (G.yc0 + y % G.bc);
            double cxy = P.C[(size_t)x * P.ny + y];
            /* log(pi/K) = (f+g-c)/eps - log mu(x) - log nu(y) + c/eps, K = exp(-c/eps) mu nu */
            double logK = -cxy / c->eps + L->logmu[gx] + log(L->nu[gy]);
            ks_add(&cost, cxy * p);
            ks_add(&ent, c->eps * p * (log(p) - logK - 1.0));
            ks_add(&ms, p);
            px += p;
            if (xi) {
                xi[base + k] = (int)gx;
                yi[base + k] = (int)gy;
                mass[base + k] = p;
            }
            ++k;
        }
        ks_add(&l1x, fabs(px - L->mu[gx]));
    }
    if (er) { er->cost = ks_get(&cost); er->ent = ks_get(&ent); er->l1x = ks_get(&l1x); er->mass = ks_get(&ms); }
    if (count) *count = k;
    free_prob(&P);
    return DDO_OK;
}

static int evaluate(ddo_ctx* c, double* cost, double* ent, double* l1x) {
    int part = c->last_part ? c->last_part : 1;
    int nc = n_cells(c, part);
    evalres_t* er = (evalres_t*)calloc((size_t)nc, sizeof(evalres_t));
    int* rcs = (int*)calloc((size_t)nc, sizeof(int));
    if (!er || !rcs) { free(er); free(rcs); return DDO_ENOMEM; }
#ifdef _OPENMP
    int nt = c->opt.n_threads > 0 ? c->opt.n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
    for (int j = 0; j < nc; ++j) rcs[j] = eval_cell(c, part, j, &er[j], NULL, NULL, NULL, NULL, 0);
    ksum_t a = {0, 0}, b = {0, 0}, d = {0, 0};
    int rc = DDO_OK;
    for (int j = 0; j < nc; ++j) {
        if (rcs[j]) rc = rcs[j];
        ks_add(&a, er[j].cost); ks_add(&b, er[j].ent); ks_add(&d, er[j].l1x);
    }
    if (cost) *cost = ks_get(&a);
    if (ent) *ent = ks_get(&b);
    if (l1x) *l1x = ks_get(&d);
    free(er);
    free(rcs);
    return rc;
}


/* ----------------------------------------------------- primal-dual gap -- */
/* Relative primal-dual gap, eq. RelPDGap:
 *   (KL(pi|K) - J(u, v)) / (KL(pi|K) - ||K||)
 * pi = the primal iterate of reading A15; the dual candidate follows Sec. 6.3
 * (P:1416-1456): the X-scalings u_{A,J} are glued by the discrete Helmholtz
 * least squares on the graph of A-cells (edges through B-cells, weights
 * log q of P:1431, sign of reading A25), u_hat = exp(V_J) u_{A,J}; v_hat is
 * the Y-iteration against u_hat (Remark Sinkhorn P:272), so that
 * int u_hat (x) v_hat dK = ||nu|| and, with eq. EntropicOTDualObjective P:250,
 *   J - ||K|| = <log u_hat, mu> + <log v_hat, nu> - ||nu||.
 * Dense fp64, plain CG (no shared code with the GPU path). */
static double cg_dot(const double* a, const double* b, int n) {
    ksum_t s = {0, 0};
    for (int i = 0; i < n; ++i) ks_add(&s, a[i] * b[i]);
    return ks_get(&s);
}

/* y = L x on the A-cell graph: for every B-cell and ordered pair of its
 * member basic cells (i1, i2): (Lx)_{A(i1)} += x_{A(i1)} - x_{A(i2)}. */
static void glue_matvec(int nb, const double* x, double* y) {
    int na = nb / 2, nbc = nb / 2 + 1;
    for (int p = 0; p < na * na; ++p) y[p] = 0.0;
    for (int q1 = 0; q1 < nbc; ++q1)
        for (int q2 = 0; q2 < nbc; ++q2) {
            int mr[4], mc[4], m = 0;
            for (int r = 2 * q1 - 1; r <= 2 * q1; ++r)
                for (int cc = 2 * q2 - 1; cc <= 2 * q2; ++cc)
                    if (r >= 0 && r < nb && cc >= 0 && cc < nb) { mr[m] = r; mc[m] = cc; ++m; }
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) {
                    if (a == b) continue;
                    int pa = (mr[a] / 2) * na + mc[a] / 2, pb = (mr[b] / 2) * na + mc[b] / 2;
                    y[pa] += x[pa] - x[pb];
                }
        }
}

/* Sec. 6.3: glue the partitions' cell potentials into one
 * dual candidate on the current layer: per basic cell i the mu-weighted
 * averages a_i = log avg exp((alpha_A - alpha_B)/eps), b_i = log avg
 * exp((alpha_B - alpha_A)/eps) give the edge weights of the A-cell graph;
 * V = the least-squares solution of V(J2) - V(J1) = log q (reading A25),
 * zero mean; ah = alpha_A + eps V(A(x)).  Plain CG (the Laplacian is
 * singular only in the constants; R has zero sum). */
static int glue_alpha(ddo_ctx* c, double* ah) {
    layer_t* L = &c->L[c->cur];
    int side = L->side, s = L->s, nb = L->nb, na = nb / 2;
    double eps = c->eps;
    int nbb = nb * nb;
    double* ab = (double*)calloc((size_t)2 * nbb, sizeof(double));
    int n = na * na;
    double* V = (double*)calloc((size_t)(n > 0 ? n : 1) * 4, sizeof(double));
    size_t n2 = (size_t)side * side;
    if (!ab || !V) { free(ab); free(V); return DDO_ENOMEM; }
    /* a_i = log avg_{X_i} exp((aA - aB)/eps) dmu, b_i = log avg exp((aB - aA)/eps) dmu */
    for (int i = 0; i < nbb; ++i) {
        int r0 = (i / nb) * s, c0 = (i % nb) * s;
        double mp = -INFINITY, mn = -INFINITY, sm = 0;
        for (int k = 0; k < s * s; ++k) {
            size_t g = (size_t)(r0 + k / s) * side + (c0 + k % s);
            if (L->mu[g] > 0) {
                double d = (c->alphaA[g] - c->alphaB[g]) / eps;
                if (d > mp) mp = d;
                if (-d > mn) mn = -d;
            }
        }
        ksum_t sp = {0, 0}, sn = {0, 0};
        for (int k = 0; k < s * s; ++k) {
            size_t g = (size_t)(r0 + k / s) * side + (c0 + k % s);
            if (L->mu[g] > 0) {
                double d = (c->alphaA[g] - c->alphaB[g]) / eps;
                ks_add(&sp, L->mu[g] * exp(d - mp));
                ks_add(&sn, L->mu[g] * exp(-d - mn));
                sm += L->mu[g];
            }
        }
        ab[2 * i] = mp + log(ks_get(&sp) / sm);
        ab[2 * i + 1] = mn + log(ks_get(&sn) / sm);
    }
    /* right-hand side: edge A(i1) -> A(i2) with log q = a_i1 + b_i2 asks
     * V(A(i2)) - V(A(i1)) = log q; normal equations over both orientations */
    double* R = V + n;
    double* Pd = V + 2 * n;
    double* AP = V + 3 * n;
    for (int p = 0; p < n; ++p) R[p] = 0.0;
    int nbc = nb / 2 + 1;
    for (int q1 = 0; q1 < nbc; ++q1)
        for (int q2 = 0; q2 < nbc; ++q2) {
            int mr[4], mc[4], m = 0;
            for (int r = 2 * q1 - 1; r <= 2 * q1; ++r)
                for (int cc = 2 * q2 - 1; cc <= 2 * q2; ++cc)
                    if (r >= 0 && r < nb && cc >= 0 && cc < nb) { mr[m] = r; mc[m] = cc; ++m; }
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) {
                    if (a == b) continue;
                    int i1 = mr[a] * nb + mc[a], i2 = mr[b] * nb + mc[b];
                    int p1 = (mr[a] / 2) * na + mc[a] / 2;
                    /* gradient of (V2 - V1 - w12)^2/2 + (V1 - V2 - w21)^2/2 w.r.t. V1 */
                    R[p1] += 0.5 * ((ab[2 * i2] + ab[2 * i1 + 1]) - (ab[2 * i1] + ab[2 * i2 + 1]));
                }
        }
    /* plain CG from V = 0 (R has zero sum: the system is consistent) */
    for (int p = 0; p < n; ++p) { V[p] = 0.0; Pd[p] = R[p]; }
    double rr = cg_dot(R, R, n), rr0 = rr;
    for (int it = 0; it < 20 * n + 100 && rr > 1e-28 * rr0 && rr > 0; ++it) {
        glue_matvec(nb, Pd, AP);
        double pap = cg_dot(Pd, AP, n);
        if (!(pap > 0)) break;
        double al = rr / pap;
        for (int p = 0; p < n; ++p) { V[p] += al * Pd[p]; R[p] -= al * AP[p]; }
        double rn = cg_dot(R, R, n);
        for (int p = 0; p < n; ++p) Pd[p] = R[p] + (rn / rr) * Pd[p];
        rr = rn;
    }
    /* glued alpha_hat = alpha_A + eps V(A(x)) */
    for (size_t g = 0; g < n2; ++g) {
        int r = (int)(g / side), q = (int)(g % side);
        ah[g] = c->alphaA[g] + eps * V[(r / s / 2) * na + (q / s / 2)];
    }
    free(ab); free(V);
    return DDO_OK;
}

int ddo_dual_gap(ddo_ctx* c, double* primal, double* dual, double* rel) {
    if (!c) return DDO_EINVAL;
    layer_t* L = &c->L[c->cur];
    int side = L->side;
    double eps = c->eps;
    double ent = 0;
    int rc = evaluate(c, NULL, &ent, NULL);
    if (rc) return rc;
    double P = ent / eps;                                  /* KL(pi|K) - ||K|| */
    size_t n2 = (size_t)side * side;
    double* ah = (double*)malloc(n2 * sizeof(double));
    double* T = (double*)malloc(n2 * sizeof(double));
    if (!ah || !T) { free(ah); free(T); return DDO_ENOMEM; }
    rc = glue_alpha(c, ah);
    if (rc) { free(ah); free(T); return rc; }
    /* Y-iteration against u_hat, dense (log v_hat below) */
    ksum_t dsum = {0, 0};
    for (size_t g = 0; g < n2; ++g)
        if (L->mu[g] > 0) ks_add(&dsum, L->mu[g] * ah[g] / eps);
#ifdef _OPENMP
    int nt = c->opt.n_threads > 0 ? c->opt.n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
#endif
    for (long long y = 0; y < (long long)n2; ++y) {
        if (!(L->nu[y] > 0)) { T[y] = 0.0; continue; }
        int y1 = (int)(y / side), y2 = (int)(y % side);
        double mx = -INFINITY;
        for (size_t x = 0; x < n2; ++x) {
            if (!(L->mu[x] > 0)) continue;
            double cxy = ground_cost(c, side, (int)(x / side), (int)(x % side), y1, y2);
            double t = ah[x] / eps + L->logmu[x] - cxy / eps;
            if (t > mx) mx = t;
        }
        double sm = 0;
        for (size_t x = 0; x < n2; ++x) {
            if (!(L->mu[x] > 0)) continue;
            double cxy = ground_cost(c, side, (int)(x / side), (int)(x % side), y1, y2);
            sm += exp(ah[x] / eps + L->logmu[x] - cxy / eps - mx);
        }
        /* v_hat is the density w.r.t. nu (K = exp(-c/eps) mu nu):
         * log v_hat(y) = -LSE_x(log u_hat + log mu - c/eps) */
        T[y] = L->nu[y] * (-(mx + log(sm)) - 1.0);                     /* nu log v_hat - nu */
    }
    for (size_t y = 0; y < n2; ++y) ks_add(&dsum, T[y]);
    double D = ks_get(&dsum);                                   /* J - ||K|| */
    if (primal) *primal = P;
    if (dual) *dual = D;
    if (rel) *rel = (P - D) / P;
    free(ah); free(T);
    return DDO_OK;
}

int ddo_primal_cost(ddo_ctx* c, double* transport_cost, double* entropic) {
    if (!c) return DDO_EINVAL;
    return evaluate(c, transport_cost, entropic, NULL);
}

int ddo_marginal_error(ddo_ctx* c, double* l1_x, double* l1_y) {
    if (!c) return DDO_EINVAL;
    int rc = evaluate(c, NULL, NULL, l1_x);
    if (rc) return rc;
    /* Y side: sum_i nu_i(y) vs nu(y) (reading A18) */
    layer_t* L = &c->L[c->cur];
    size_t n2 = (size_t)L->side * L->side;
    double* acc = (double*)calloc(n2, sizeof(double));
    if (!acc) return DDO_ENOMEM;
    for (int i = 0; i < L->nb * L->nb; ++i) {
        const int* b = &c->box[4 * i];
        for (int r = 0; r < b[2]; ++r)
            for (int q = 0; q < b[3]; ++q)
                acc[(size_t)(b[0] + r) * L->side + (b[1] + q)] += c->val[i][(size_t)r * b[3] + q];
    }
    ksum_t s = {0, 0};
    for (size_t y = 0; y < n2; ++y) ks_add(&s, fabs(acc[y] - L->nu[y]));
    free(acc);
    if (l1_y) *l1_y = ks_get(&s);
    return DDO_OK;
}

int ddo_fetch_plan_coo(ddo_ctx* c, long long* count, int* xi, int* yi, double* mass) {
    if (!c || !count) return DDO_EINVAL;
    int part = c->last_part ? c->last_part : 1;
    int nc = n_cells(c, part);
    long long total = 0;
    for (int j = 0; j < nc; ++j) {
        long long k = 0;
        int rc = eval_cell(c, part, j, NULL, &k, xi ? xi : NULL, yi, mass, total);
        if (rc) return rc;
        total += k;
    }
    *count = total;
    return DDO_OK;
}

int ddo_get_stats(ddo_ctx* c, ddo_sweep_stats* st) {
    if (!c || !st) return DDO_EINVAL;
    *st = c->stats;
    return DDO_OK;
}

int ddo_get_state_info(ddo_ctx* c, ddo_state_info* info) {
    if (!c || !info) return DDO_EINVAL;
    layer_t* L = &c->L[c->cur];
    info->side = L->side; info->s = L->s; info->nb = L->nb;
    info->last_partition = c->last_part;
    info->half_index = c->half_index;
    info->eps = c->eps;
    long long e = 0;
    for (int i = 0; i < L->nb * L->nb; ++i) e += (long long)c->box[4 * i + 2] * c->box[4 * i + 3];
    info->entries = e;
    return DDO_OK;
}

int ddo_get_state(ddo_ctx* c, int* boxes, long long* offsets, double* values,
                  double* alpha_A, double* alpha_B) {
    if (!c) return DDO_EINVAL;
    layer_t* L = &c->L[c->cur];
    long long off = 0;
    for (int i = 0; i < L->nb * L->nb; ++i) {
        const int* b = &c->box[4 * i];
        if (boxes) memcpy(&boxes[4 * i], b, 4 * sizeof(int));
        if (offsets) offsets[i] = off;
        size_t area = (size_t)b[2] * b[3];
        if (values && area) memcpy(values + off, c->val[i], sizeof(double) * area);
        off += (long long)area;
    }
    size_t n2 = (size_t)L->side * L->side;
    if (alpha_A) memcpy(alpha_A, c->alphaA, sizeof(double) * n2);
    if (alpha_B) memcpy(alpha_B, c->alphaB, sizeof(double) * n2);
    return DDO_OK;
}

int ddo_set_state(ddo_ctx* c, int side, long long half_index, int last_partition,
                  const int* boxes, const long long* offsets, const double* values,
                  const double* alpha_A, const double* alpha_B) {
    if (!c || !boxes || !offsets || !values) return DDO_EINVAL;
    int k = 0;
    while (k < c->n_layers && c->L[k].side != side) ++k;
    if (k == c->n_layers) { set_err(c, "no layer of side %d", side); return DDO_EINVAL; }
    free_state(c);
    c->cur = k;
    int rc = alloc_state(c);
    if (rc) return rc;
    layer_t* L = &c->L[k];
    for (int i = 0; i < L->nb * L->nb; ++i) {
        memcpy(&c->box[4 * i], &boxes[4 * i], 4 * sizeof(int));
        const int* b = &boxes[4 * i];
        if (b[2] < 0 || b[3] < 0 || b[0] < 0 || b[1] < 0 || b[0] + b[2] > side || b[1] + b[3] > side) {
            set_err(c, "box %d out of range", i);
            return DDO_EINVAL;
        }
        size_t area = (size_t)b[2] * b[3];
        c->val[i] = (double*)malloc(sizeof(double) * (area ? area : 1));
        if (!c->val[i]) return DDO_ENOMEM;
        if (area) memcpy(c->val[i], values + offsets[i], sizeof(double) * area);
    }
    size_t n2 = (size_t)side * side;
    if (alpha_A) memcpy(c->alphaA, alpha_A, sizeof(double) * n2);
    if (alpha_B) memcpy(c->alphaB, alpha_B, sizeof(double) * n2);
    c->half_index = half_index;
    c->last_part = last_partition;
    return DDO_OK;
}

int ddo_get_layer_marginals(ddo_ctx* c, double* mu, double* nu) {
    if (!c) return DDO_EINVAL;
    layer_t* L = &c->L[c->cur];
    size_t n2 = (size_t)L->side * L->side;
    if (mu) memcpy(mu, L->mu, sizeof(double) * n2);
    if (nu) memcpy(nu, L->nu, sizeof(double) * n2);
    return DDO_OK;
}
