/*
 * dd_shim.c -- the SURVEY.md Sec. 8(b) C-ABI (dd_init, dd_iterate, ...)
 *              exported by the ORACLE library over its own ddo_* calls, so
 *              one harness (tests/abi_harness.py) can drive both libdd_gpu.so
 *              and liboracle_dd.so through the same entry points.
 *
 * TEST INFRASTRUCTURE ONLY (see dd_oracle.h).  Marshalling only: every step
 * of the method runs in dd_oracle.c.  The structure layouts below restate
 * the published contract (include/dd.h of the product); the header itself is
 * deliberately not included, so the oracle shares no file with the CUDA path.
 * Entry points that only make sense on a GPU (stripes, row export/import,
 * phase profile, MUFU peak) are not exported.
 */
#include <stdlib.h>
#include <string.h>

#include "dd_oracle.h"

#define SHIM_OK 0
#define SHIM_EINVAL 1
#define SHIM_ENOCONV 2
#define SHIM_ENOMEM 6
#define SHIM_FLAG_DEVICE_INPUT 1u
#define SHIM_PLAN_BASIC_MARGINALS 0
#define SHIM_PLAN_COO 1

typedef struct {                /* = dd_options */
    double err_tol;
    double trunc_tau;
    int max_inner_iter;
    int check_every;
    int n_gpus;
    int schedule;
    double eps_start;
    int coarsest_side;
    int no_truncate;
    unsigned int flags;
    int device;
    long long pool_capacity;
    void* stream;
    int reserved[8];
} shim_options;

typedef struct {                /* = dd_sweep_stats */
    long long cells, iters_sum;
    int iters_max, failed;
    double err_x_sum;
    long long entries;
    double ms, mufu_ops, solve_ms;
    long long launches, big_cells;
    int max_box, reserved_i;
    long long cluster_cells;    /* GPU cluster tier only: always 0 here */
} shim_stats;

typedef struct {                /* = dd_state_info */
    int side, s, nb, last_partition;
    long long half_index, entries;
    double eps;
} shim_info;

typedef struct {
    ddo_ctx* o;
    int n, cell_size;
    double eps;
    ddo_options opt;
    double *mu, *nu;            /* kept for dd_reset */
    double *h1, *h2;            /* dd_set_cost tables (re-applied by dd_reset) */
    int pending_fail;           /* ENOCONV reported at the next dd_synchronize (as on the GPU) */
    shim_stats tot;
    char err[256];
} shim_ctx;

static int wrap(shim_ctx* c, int rc) {
    if (rc == DDO_ENOCONV) { c->pending_fail = 1; return SHIM_OK; }
    return rc;
}

const char* dd_version(void) { return "ddot-oracle (CPU fp64, dense; test infrastructure)"; }

const char* dd_last_error(const shim_ctx* c) {
    if (!c) return "null context";
    if (c->err[0]) return c->err;
    return c->o ? ddo_last_error(c->o) : "";
}

int dd_build_schedule(int n_final, int coarsest_side, double kappa_final, double eps_start, int* side,
                      double* kappa, int* sweeps, int max) {
    return ddo_build_schedule(n_final, coarsest_side, kappa_final, eps_start, side, kappa, sweeps, max);
}

int dd_init(shim_ctx** out, int n, const double* mu, const double* nu, int cost, double eps, int cell_size,
            const shim_options* opt) {
    if (!out) return SHIM_EINVAL;
    shim_ctx* c = (shim_ctx*)calloc(1, sizeof(shim_ctx));
    *out = c;
    if (!c) return SHIM_ENOMEM;
    if (cost != 0) { strcpy(c->err, "only the squared Euclidean cost"); return SHIM_EINVAL; }
    if (opt && (opt->flags & SHIM_FLAG_DEVICE_INPUT)) { strcpy(c->err, "the oracle takes host inputs"); return SHIM_EINVAL; }
    if (!mu || !nu || n <= 0) { strcpy(c->err, "null marginal"); return SHIM_EINVAL; }
    memset(&c->opt, 0, sizeof(c->opt));
    if (opt) {
        c->opt.err_tol = opt->err_tol;
        c->opt.trunc_tau = opt->trunc_tau;
        c->opt.max_inner_iter = opt->max_inner_iter;
        c->opt.schedule = opt->schedule;
        c->opt.eps_start = opt->eps_start;
        c->opt.coarsest_side = opt->coarsest_side;
        c->opt.no_truncate = opt->no_truncate;
        c->opt.check_every = opt->check_every;
        c->opt.safeguard = (opt->flags & 2u) ? 1 : 0;      /* DD_FLAG_SAFEGUARD */
    }
    c->n = n; c->cell_size = cell_size; c->eps = eps;
    size_t n2 = (size_t)n * n;
    c->mu = (double*)malloc(n2 * sizeof(double));
    c->nu = (double*)malloc(n2 * sizeof(double));
    if (!c->mu || !c->nu) return SHIM_ENOMEM;
    memcpy(c->mu, mu, n2 * sizeof(double));
    memcpy(c->nu, nu, n2 * sizeof(double));
    return ddo_init(&c->o, n, c->mu, c->nu, eps, cell_size, &c->opt);
}

void dd_free(shim_ctx* c) {
    if (!c) return;
    if (c->o) ddo_free(c->o);
    free(c->mu); free(c->nu); free(c->h1); free(c->h2);
    free(c);
}

int dd_reset(shim_ctx* c) {
    if (!c) return SHIM_EINVAL;
    if (c->o) ddo_free(c->o);
    c->o = NULL;
    c->pending_fail = 0;
    int rc = ddo_init(&c->o, c->n, c->mu, c->nu, c->eps, c->cell_size, &c->opt);
    if (rc == DDO_OK && c->h1) rc = ddo_set_cost(c->o, c->n, c->h1, c->h2);
    return rc;
}

int dd_set_cost(shim_ctx* c, int n_entries, const double* h1, const double* h2) {
    if (!c || !c->o) return SHIM_EINVAL;
    int rc = ddo_set_cost(c->o, n_entries, h1, h2);
    if (rc) return rc;
    free(c->h1); free(c->h2);
    c->h1 = c->h2 = NULL;
    if (h1) {
        c->h1 = (double*)malloc(sizeof(double) * n_entries);
        c->h2 = (double*)malloc(sizeof(double) * n_entries);
        if (!c->h1 || !c->h2) return SHIM_ENOMEM;
        memcpy(c->h1, h1, sizeof(double) * n_entries);
        memcpy(c->h2, h2, sizeof(double) * n_entries);
    }
    return SHIM_OK;
}

static void add_totals(shim_ctx* c) {
    ddo_sweep_stats s;
    ddo_get_stats(c->o, &s);
    c->tot.cells += s.cells;
    c->tot.iters_sum += s.iters_sum;
    if (s.iters_max > c->tot.iters_max) c->tot.iters_max = s.iters_max;
    c->tot.failed += s.failed;
    c->tot.err_x_sum = s.err_x_sum;
    c->tot.entries = s.entries;
}

int dd_iterate(shim_ctx* c, int k) {
    if (!c || k < 0) return SHIM_EINVAL;
    for (int i = 0; i < k; ++i) {
        int rc = wrap(c, ddo_iterate(c->o, 1));
        if (rc) return rc;
        add_totals(c);
    }
    return SHIM_OK;
}

int dd_set_eps(shim_ctx* c, double eps) { return c ? ddo_set_eps(c->o, eps) : SHIM_EINVAL; }
int dd_refine(shim_ctx* c) { return c ? ddo_refine(c->o) : SHIM_EINVAL; }

int dd_run_schedule(shim_ctx* c) {
    if (!c) return SHIM_EINVAL;
    int rc = wrap(c, ddo_run_schedule(c->o));
    if (rc) return rc;
    if (c->pending_fail) { c->pending_fail = 0; return SHIM_ENOCONV; }
    return SHIM_OK;
}

int dd_synchronize(shim_ctx* c) {
    if (!c) return SHIM_EINVAL;
    if (c->pending_fail) { c->pending_fail = 0; return SHIM_ENOCONV; }
    return SHIM_OK;
}

int dd_primal_cost(shim_ctx* c, double* cost, double* ent) { return c ? ddo_primal_cost(c->o, cost, ent) : SHIM_EINVAL; }
int dd_marginal_error(shim_ctx* c, double* lx, double* ly) { return c ? ddo_marginal_error(c->o, lx, ly) : SHIM_EINVAL; }
int dd_dual_gap(shim_ctx* c, double* p, double* d, double* r) { return c ? ddo_dual_gap(c->o, p, d, r) : SHIM_EINVAL; }

int dd_get_stats(shim_ctx* c, shim_stats* s) {
    if (!c || !s) return SHIM_EINVAL;
    ddo_sweep_stats d;
    ddo_get_stats(c->o, &d);
    memset(s, 0, sizeof(*s));
    s->cells = d.cells; s->iters_sum = d.iters_sum; s->iters_max = d.iters_max; s->failed = d.failed;
    s->err_x_sum = d.err_x_sum; s->entries = d.entries;
    return d.failed ? SHIM_ENOCONV : SHIM_OK;
}

int dd_get_totals(shim_ctx* c, shim_stats* s) {
    if (!c || !s) return SHIM_EINVAL;
    *s = c->tot;
    return SHIM_OK;
}

int dd_reset_totals(shim_ctx* c) {
    if (!c) return SHIM_EINVAL;
    memset(&c->tot, 0, sizeof(c->tot));
    return SHIM_OK;
}

int dd_get_state_info(shim_ctx* c, shim_info* info) {
    if (!c || !info) return SHIM_EINVAL;
    ddo_state_info d;
    int rc = ddo_get_state_info(c->o, &d);
    info->side = d.side; info->s = d.s; info->nb = d.nb; info->last_partition = d.last_partition;
    info->half_index = d.half_index; info->entries = d.entries; info->eps = d.eps;
    return rc;
}

int dd_get_state(shim_ctx* c, int* boxes, long long* offsets, double* values, double* aA, double* aB) {
    return c ? ddo_get_state(c->o, boxes, offsets, values, aA, aB) : SHIM_EINVAL;
}

int dd_set_state(shim_ctx* c, int side, long long half_index, int last_partition, const int* boxes,
                 const long long* offsets, const double* values, long long n_values, const double* aA,
                 const double* aB) {
    (void)n_values;
    return c ? ddo_set_state(c->o, side, half_index, last_partition, boxes, offsets, values, aA, aB) : SHIM_EINVAL;
}

int dd_fetch_plan(shim_ctx* c, int format, void* buf, size_t* bytes) {
    if (!c || !bytes) return SHIM_EINVAL;
    if (format == SHIM_PLAN_BASIC_MARGINALS) {
        ddo_state_info d;
        ddo_get_state_info(c->o, &d);
        size_t nb2 = (size_t)d.nb * d.nb;
        size_t need = nb2 * 4 * sizeof(int) + nb2 * sizeof(long long) + (size_t)d.entries * sizeof(double);
        if (!buf) { *bytes = need; return SHIM_OK; }
        if (*bytes < need) { strcpy(c->err, "buffer too small"); return SHIM_EINVAL; }
        char* p = (char*)buf;
        *bytes = need;
        return ddo_get_state(c->o, (int*)p, (long long*)(p + nb2 * 4 * sizeof(int)),
                             (double*)(p + nb2 * 4 * sizeof(int) + nb2 * sizeof(long long)), NULL, NULL);
    }
    if (format == SHIM_PLAN_COO) {
        long long cnt = 0;
        int rc = ddo_fetch_plan_coo(c->o, &cnt, NULL, NULL, NULL);
        if (rc) return rc;
        size_t need = (size_t)cnt * (2 * sizeof(int) + sizeof(double));
        if (!buf) { *bytes = need; return SHIM_OK; }
        if (*bytes < need) { strcpy(c->err, "buffer too small"); return SHIM_EINVAL; }
        char* p = (char*)buf;
        *bytes = need;
        return ddo_fetch_plan_coo(c->o, &cnt, (int*)p, (int*)(p + cnt * sizeof(int)),
                                  (double*)(p + 2 * cnt * sizeof(int)));
    }
    strcpy(c->err, "unknown plan format");
    return SHIM_EINVAL;
}
