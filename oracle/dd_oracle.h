/*
 * dd_oracle.h -- CPU fp64 ORACLE for entropic domain decomposition
 *                (arXiv 2001.10986, Algorithm 2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (include/dd.h, paper_2001_10986_b200/csrc/).  Its own prefix is ddo_.
 *
 * Units: the grid is [0,1]^2 with N x N pixels, h = 1/N, pixel centres
 * ((i+1/2)h, (j+1/2)h); cost c(x,y) = |x-y|^2; eps in the same
 * units (reading A1).  Potentials are stored as alpha = eps*log u in cost
 * units (reading A2).  Arrays are row-major, index [i*N + j] with
 * i = row (x1), j = column (x2).
 */
#ifndef DD_ORACLE_H
#define DD_ORACLE_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

#define DDO_OK 0
#define DDO_EINVAL 1
#define DDO_ENOCONV 2
#define DDO_ENUMERIC 3
#define DDO_ENOMEM 6

#define DDO_SCHED_FIXED 0
#define DDO_SCHED_LADDER 1

typedef struct ddo_ctx ddo_ctx;

typedef struct {
    double err_tol;        /* Err; 0 -> 1e-6 */
    double trunc_tau;      /* truncation threshold; <0 -> 0, 0 -> 1e-15 */
    int max_inner_iter;    /* 0 -> 10000 */
    int n_threads;         /* OpenMP threads over cells; 0 -> default */
    int schedule;          /* DDO_SCHED_FIXED | DDO_SCHED_LADDER */
    double eps_start;      /* ladder: eps at the coarsest layer if > 2 h_0^2 (0 = none) */
    int coarsest_side;     /* ladder: coarsest layer side (0 -> 8) */
    int no_truncate;       /* 1 -> tau = 0 exactly (pins P3/P5) */
    int empty_init;        /* 1 -> no product initialisation: empty state, a state is imported next */
    int check_every;       /* stop-test cadence k (reading A5): stop at it % k == 0; 0 -> 1 */
    int warm_refine;       /* 1 -> ddo_refine warm-starts alpha as P:1507-1508 does: the
                              coarse potentials glued (Sec. 6.3) and
                              interpolated linearly in log space onto the fine pixel
                              centres (readings A25, A26); 0 -> cold start alpha = 0 (A14) */
    int safeguard;         /* 1 -> eps-raising safeguard (A29):
                              a cell whose Sinkhorn fails (max_inner_iter or non-finite) is
                              retried from its input alpha at 2^k eps (k = 1, 2, 3), the
                              result re-solved at eps with alpha kept */
} ddo_options;

typedef struct {
    long long cells, iters_sum;
    int iters_max, failed;
    double err_x_sum;
    long long entries;
    int safeguarded;       /* cells the eps-raising safeguard retried (ddo_options.safeguard) */
    int pad_;
} ddo_sweep_stats;

typedef struct {
    int side;              /* N_l of the current layer */
    int s;                 /* basic cell side s_l */
    int nb;                /* basic cells per axis */
    int last_partition;    /* 0 none, 1 A, 2 B */
    long long half_index;  /* sweeps done so far (global) */
    long long entries;     /* stored nu_i entries (sum of box areas) */
    double eps;            /* current eps ([0,1]^2 units) */
} ddo_state_info;

/* Textbook log-domain Sinkhorn on one (composite-cell) problem:
 * target X masses a[nx], Y masses b[ny], cost C[nx*ny] (row-major x,y), eps.
 * f[nx] (in: initial absorbed X potential f = alpha + eps log mu; out: the
 * returned plan's f), g[ny] (out).  Starts and ends with a Y-iteration,
 * stops when sum_x a(x)|exp((f-fn)/eps)-1| <= tol (reading A4).
 * Returns DDO_OK or DDO_ENOCONV (max_iter reached; plan of the last
 * Y-iteration returned). */
int ddo_sinkhorn_dense(int nx, int ny, const double* a, const double* b, const double* C,
                       double eps, double tol, int max_iter, double* f, double* g,
                       int* iters, double* err);

/* Schedule builder (reading A12).  Writes up to max stages;
 * returns the number of stages.  side[k], kappa[k] = eps/h_l^2, sweeps[k]. */
int ddo_build_schedule(int n_final, int coarsest_side, double kappa_final, double eps_start,
                       int* side, double* kappa, int* sweeps, int max);

int ddo_init(ddo_ctx** out, int n, const double* mu, const double* nu, double eps,
             int cell_size, const ddo_options* opt);
int ddo_set_eps(ddo_ctx* c, double eps);
/* General separable cost: c(x,y) = h1(|x1-y1|) + h2(|x2-y2|)
 * in [0,1]^2 cost units; h1[d], h2[d] for finest-grid pixel differences d = 0..n-1
 * (n = the finest side; copied).  Both NULL restores |x-y|^2.  Call before iterating. */
int ddo_set_cost(ddo_ctx* c, int n_entries, const double* h1, const double* h2);
int ddo_iterate(ddo_ctx* c, int n_half_iters);
/* Algorithm 2 lines 8-13 for the listed composite cells of partition `part`
 * only (1 = A, 2 = B; row-major cell index), on the current state; cells of
 * one partition are disjoint, so this is exactly what a sweep does to them.
 * Does not advance the half-iteration.  iters[k] receives each solve's
 * Sinkhorn iteration count (may be NULL).  For sampled full-size parity. */
/* Relative primal-dual gap, eq. RelPDGap, dual candidate glued
 * as in Sec. 6.3: primal = KL(pi|K) - ||K||, dual = J(u_hat, v_hat) - ||K||. */
int ddo_dual_gap(ddo_ctx* c, double* primal, double* dual, double* rel);
int ddo_solve_cells(ddo_ctx* c, int part, int n, const int* cells, int* iters);
/* The same with the listed cells solved concurrently (OpenMP over cells, as
 * in a sweep); for timing the oracle on a sample of a sweep. */
int ddo_solve_cells_par(ddo_ctx* c, int part, int n, const int* cells, int* iters);
int ddo_refine(ddo_ctx* c);
int ddo_run_schedule(ddo_ctx* c);
int ddo_primal_cost(ddo_ctx* c, double* transport_cost, double* entropic);
int ddo_marginal_error(ddo_ctx* c, double* l1_x, double* l1_y);
/* COO plan (x index, y index, mass) of the last sweep's cell plans; two-call. */
int ddo_fetch_plan_coo(ddo_ctx* c, long long* count, int* xi, int* yi, double* mass);
int ddo_get_stats(ddo_ctx* c, ddo_sweep_stats* st);
int ddo_get_state_info(ddo_ctx* c, ddo_state_info* info);
/* boxes[nb*nb*4] = (y0r, y0c, hr, hc); offsets[nb*nb] into values (basic-cell
 * order, compact); alpha_A/alpha_B [side*side] (cost units). */
int ddo_get_state(ddo_ctx* c, int* boxes, long long* offsets, double* values,
                  double* alpha_A, double* alpha_B);
int ddo_set_state(ddo_ctx* c, int side, long long half_index, int last_partition,
                  const int* boxes, const long long* offsets, const double* values,
                  const double* alpha_A, const double* alpha_B);
/* Layer marginals (side*side) of the current layer. */
int ddo_get_layer_marginals(ddo_ctx* c, double* mu, double* nu);
void ddo_free(ddo_ctx* c);
const char* ddo_last_error(const ddo_ctx* c);

#ifdef __cplusplus
}
#endif
#endif
