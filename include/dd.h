/*
 * dd.h -- C-ABI of the B200 (sm_100a) entropic domain decomposition library
 *         libdd_gpu.so  (arXiv 2001.10986).
 *
 * The hot path is Algorithm 2 of the paper: per
 * half-iteration ("sweep") every composite cell J of partition A (then B) is
 * solved as an independent entropic OT problem by log-domain Sinkhorn with
 * the cell's fixed X-mass mu_J and Y-marginal nu_cell = sum_{i in J} nu_i
 * (line 8), split back into basic-cell marginals (line 10), balanced
 * (line 11) and truncated (line 12).  A coarse-to-fine /
 * eps-scaling driver runs on top.
 *
 * Conventions (apply to every entry point):
 *  - Grid: N x N pixels on [0,1]^2, h = 1/N, pixel centres ((i+1/2)h,(j+1/2)h),
 *    arrays row-major [i*N + j], i = row (x1), j = column (x2).  X and Y use
 *    the same grid.  Cost c(x,y) = |x-y|^2.  eps in the same units;
 *    kappa = eps/h^2 is eps in squared pixels.
 *  - Potentials: alpha = eps*log u in cost units; the plan of a cell
 *    is pi(x,y) = exp((alpha(x) + beta(y) - c(x,y))/eps) mu(x) nu(y)
 *    (K = exp(-c/eps) mu (x) nu).
 *  - Return codes: DD_OK (0) or one of DD_E*.  No exceptions cross the ABI;
 *    the message of the last failure is dd_last_error(ctx).
 *  - Memory: inputs are copied at dd_init (the caller keeps ownership).
 *    Outputs go to caller buffers; variable-size outputs use the two-call
 *    pattern (buf == NULL -> required size).  The context owns every device
 *    allocation and frees it in dd_free.
 *  - Streams: all device work of a context is issued on one CUDA stream
 *    (dd_options.stream, or a stream the library creates).  Every entry
 *    point that returns host data synchronises that stream.
 *  - Threading: one context per host thread; calls on a context are not
 *    thread-safe.  One device per context (dd_options.device).
 *  - Determinism: per-cell arithmetic does not depend on scheduling; all
 *    reductions are fixed-order.  Results are bit-reproducible run to run.
 *  - There is NO CPU fallback: without a usable sm_100 device dd_init
 *    returns DD_ECUDA.
 */
#ifndef DD_H
#define DD_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

#define DD_OK 0
#define DD_EINVAL 1    /* invalid argument (n not 2^k, n/s odd, bad mass, ...) */
#define DD_ENOCONV 2   /* some cell hit max_inner_iter; state stays Y-feasible */
#define DD_ENUMERIC 3  /* non-finite value in a cell solve */
#define DD_ECUDA 4     /* CUDA runtime error / no sm_100 device */
#define DD_ENCCL 5     /* reserved: multi-GPU communication error */
#define DD_ENOMEM 6    /* device allocation failed or pool capacity exceeded */

#define DD_COST_SQEUCLID 0

#define DD_SCHED_FIXED 0   /* single layer (the input grid), eps fixed by the caller */
#define DD_SCHED_LADDER 1  /* multiscale + eps-scaling (A12) */

#define DD_FLAG_DEVICE_INPUT 1u  /* dd_init: mu, nu are device pointers (fp64) */
#define DD_FLAG_SAFEGUARD 2u     /* eps-raising safeguard (A29): a
                                    cell whose Sinkhorn hits max_inner_iter or turns non-finite is
                                    retried from its input alpha at 2^k eps (k = 1, 2, 3; fp64),
                                    alpha kept and re-solved at eps; CellOut flag 32.
                                    Cells that still fail are flagged as before (DD_ENOCONV). */

#define DD_PLAN_BASIC_MARGINALS 0
#define DD_PLAN_COO 1

typedef struct dd_ctx dd_ctx;

typedef struct {                /* zero-initialised fields take the defaults */
    double err_tol;             /* Err: cell stop when L1 X-error <= ||mu_J|| Err; 0 -> 1e-6 */
    double trunc_tau;           /* truncation threshold; 0 -> 1e-15, <0 -> 0 */
    int max_inner_iter;         /* Sinkhorn iterations per cell solve; 0 -> 10000 */
    int check_every;            /* stop-test cadence k (A5): a cell stops at the first iteration
                                   it with it % k == 0 and err <= ||mu_J|| Err; 0/1 -> every
                                   iteration (parity mode).  The error itself is fused into the
                                   X-iteration, so k > 1 only delays the stop. */
    int n_gpus;                 /* reserved for striping; 0/1 -> one GPU */
    int schedule;               /* DD_SCHED_FIXED | DD_SCHED_LADDER */
    double eps_start;           /* ladder: eps at the coarsest layer if > 2 h_0^2 (0 = none) */
    int coarsest_side;          /* ladder: coarsest layer side (0 -> 8) */
    int no_truncate;            /* 1 -> tau = 0 */
    unsigned int flags;         /* DD_FLAG_* */
    int device;                 /* CUDA device ordinal */
    long long pool_capacity;    /* nu_i pool entries per buffer; 0 -> 64 * N^2 + 2^22.  Each of
                                   the two pool buffers holds this plus a halo region of
                                   pool_capacity / 3 entries for imported multi-GPU boundary
                                   rows (fp64: 2 * 4/3 * 8 B per entry in total) */
    void* stream;               /* cudaStream_t to use, or NULL */
    int reserved[8];            /* [0] > 0: box-side cap of the SMEM tier (tier 0);
                                   [1] > 0: box-side cap of the 3-CTA/SM fused tier (tier 1);
                                   testing knobs that route cells to the other K1 tiers;
                                   [2] = 1: cold-start potentials at dd_refine (reading A14)
                                   instead of the glued + interpolated warm start;
                                   [3] K1 cluster tier (one cell on a cluster of CTAs, DSMEM):
                                   0 / -1 off (default), 2 auto (the sweep's long poles), 1 every
                                   cell of the fused big-cell path (testing); results are
                                   bit-identical whichever tier solves a cell;
                                   [4] > 0: cluster routing threshold theta in % (default 300:
                                   predicted work >= theta * sweep work / #SMs);
                                   [5] > 0: persistent clusters (default 6, capped by
                                   cudaOccupancyMaxActiveClusters);
                                   [6] > 0: testing: box-side cap of the on-chip tiers; larger
                                   cells run on tier G (the SMEM-tier kernel on global-memory
                                   layouts, which serves boxes of any size) */
} dd_options;

typedef struct {                /* one sweep (or accumulated totals) */
    long long cells;            /* composite-cell solves */
    long long iters_sum;        /* Sinkhorn iterations summed over cells */
    int iters_max;
    int failed;                 /* cells that hit max_inner_iter or went non-finite */
    double err_x_sum;           /* sum_J L1 X-error of the returned plans (<= Err) */
    long long entries;          /* stored nu_i entries after the sweep */
    double ms;                  /* device time of the sweep(s), CUDA events */
    double mufu_ops;            /* MUFU (ex2/lg2/rcp) operations executed by the cell solve */
    double solve_ms;            /* device time of the cell-solve kernel launches only */
    long long launches;         /* kernel launches issued */
    long long big_cells;        /* cells routed to the large-box path */
    int max_box;                /* largest composite Y-box side seen */
    int reserved_i;             /* outputs recomputed with an exact max (speculative misses) */
    long long cluster_cells;    /* cells solved by the K1 cluster tier (a subset of big_cells) */
} dd_sweep_stats;

typedef struct {
    int side;                   /* N_l of the current layer */
    int s;                      /* basic cell side s_l */
    int nb;                     /* basic cells per axis */
    int last_partition;         /* 0 none, 1 A, 2 B */
    long long half_index;       /* sweeps done so far */
    long long entries;          /* stored nu_i entries */
    double eps;                 /* current eps ([0,1]^2 units) */
} dd_state_info;

/* dd_init -- create a context.
 *  n: grid side (power of two >= 4); mu, nu: n*n fp64 row-major, >= 0,
 *  finite, ||mu|| = ||nu|| (1e-12 rel.), every basic cell of every layer with
 *  ||mu_i|| > 0.  Host pointers unless opt->flags has
 *  DD_FLAG_DEVICE_INPUT.  cost: DD_COST_SQEUCLID.  eps: FIXED -> the eps of
 *  the sweeps; LADDER -> the final eps.  cell_size: basic cell side s (power
 *  of two, n/s even).  The state starts at the coarsest layer with the
 *  product coupling nu_i = ||mu_i|| nu and alpha = 0 (A3). */
int dd_init(dd_ctx** out, int n, const double* mu, const double* nu, int cost, double eps,
            int cell_size, const dd_options* opt);

/* dd_iterate -- n_half_iters sweeps A, B, A, ... (Alg. 2 lines 5-14).
 * Asynchronous (enqueued on the context stream; no host wait per sweep).
 * Cells that hit max_inner_iter (reading A6) are reported by the next
 * dd_synchronize / dd_run_schedule as DD_ENOCONV. */
int dd_iterate(dd_ctx* ctx, int n_half_iters);

/* dd_set_eps -- change eps keeping alpha = eps log u constant. */
int dd_set_eps(dd_ctx* ctx, double eps);

/* dd_set_max_inner_iter -- the Sinkhorn iteration cap of the following sweeps
 * (dd_options.max_inner_iter; reading A6).  k >= 1, else DD_EINVAL. */
int dd_set_max_inner_iter(dd_ctx* ctx, int k);

/* dd_set_cost -- general separable ground cost (Sec. 7.1 "Test data":
 * the scheme applies to costs h(x - y)):
 *   c(x, y) = h1(|x1 - y1|) + h2(|x2 - y2|)   ([0,1]^2 cost units, x1 = row)
 * h1, h2: host arrays of n entries (n = the finest side), h_k[d] = the cost of a
 * difference of d finest-grid pixels (d = 0..n-1); copied.  A coarse layer of
 * side m uses h_k[d * n / m] (pixel centres of the coarse grid are finest-grid
 * distances apart).  Both NULL restores |x - y|^2.  Call between sweeps (it
 * synchronises the context).  Numerics: per cell, every table entry / eps is
 * split into a hi part on the cell's 2^-q grid and a lo remainder (DESIGN.md
 * "general costs"), so the hi arithmetic of K1 stays exact for any real table.
 * Scope: general costs (and s = 16) run on the SMEM tier; a cell whose union
 * Y box exceeds its capacity is flagged and dd_synchronize returns DD_ENOMEM.
 * Errors: DD_EINVAL (wrong length, one table NULL, non-finite entry). */
int dd_set_cost(dd_ctx* ctx, int n_entries, const double* h1, const double* h2);

/* dd_refine -- move to the next finer layer: nu_i^0 by eq. FineBasicMarginals
 * (P:1471-1474); alpha warm start = the coarse potentials glued by the
 * discrete Helmholtz least squares and interpolated linearly in
 * log space, or a cold start (alpha = 0, reading A14) when
 * dd_options.reserved[2] = 1 or a multi-GPU stripe is set. */
int dd_refine(dd_ctx* ctx);

/* dd_run_schedule -- LADDER mode: run the whole schedule (refinements, eps
 * stages, sweeps) on the context stream, then wait once at the end: returns
 * DD_ENOCONV if any cell hit max_inner_iter (A6; the state stays
 * Y-feasible), DD_ENOMEM on a pool overflow. */
int dd_run_schedule(dd_ctx* ctx);

/* dd_run_schedule_batch -- dd_run_schedule on n independent problems at once
 * (e.g. the image pairs of a batch; every context LADDER mode with the same
 * grid side, cell size, coarsest side and final eps, on the same device, each
 * with its OWN stream).  The sweeps are enqueued round-robin over the
 * contexts, so the cells of one problem fill the SMs that another problem's
 * latency-bound sweeps (a sweep lasts as long as its slowest cell) leave idle;
 * every problem's arithmetic is unchanged (its state is bit-identical to
 * dd_run_schedule's).  Ordering: work queued on ctxs[0]'s stream before the
 * call precedes every context's first sweep, and ctxs[0]'s stream waits for
 * every context's last sweep.  Waits once at the end; returns the first
 * non-zero code of the contexts' dd_synchronize (DD_ENOCONV, DD_ENOMEM) or
 * DD_EINVAL if the contexts do not match. */
int dd_run_schedule_batch(dd_ctx* const* ctxs, int n);

/* dd_reset -- return to the initial state (coarsest layer, product coupling). */
int dd_reset(dd_ctx* ctx);

/* dd_primal_cost -- evaluate the plan pi = sum_J pi_J of the last swept
 * partition (A if none), each pi_J rebuilt from alpha_{C,J} and
 * nu_cell = sum_{i in J} nu_i by one Y-iteration (A15):
 * transport_cost = <c, pi>; entropic = eps (KL(pi|K) - ||K||). */
int dd_primal_cost(dd_ctx* ctx, double* transport_cost, double* entropic);

/* dd_dual_gap -- relative primal-dual gap of eq. RelPDGap:
 * (KL(pi|K) - J(u_hat, v_hat)) / (KL(pi|K) - ||K||), pi as in
 * dd_primal_cost; u_hat = the potentials of the current layer glued by the
 * discrete Helmholtz least squares (reading A25), v_hat = the
 * Y-iteration against u_hat over the whole grid (dense in x, two separable
 * fp64 passes: O(n^3), a diagnostic).  primal = KL - ||K||, dual = J - ||K||.
 * Needs the whole layer (no multi-GPU stripe). */
int dd_dual_gap(dd_ctx* ctx, double* primal, double* dual, double* rel_gap);

/* dd_marginal_error -- l1_x = sum_x |P_X pi(x) - mu(x)| of that plan;
 * l1_y = sum_y |sum_i nu_i(y) - nu(y)| (A18). */
int dd_marginal_error(dd_ctx* ctx, double* l1_x, double* l1_y);

/* dd_fetch_plan -- two-call export.
 *  DD_PLAN_BASIC_MARGINALS: the paper's state: nb*nb int32 boxes
 *   (y0r, y0c, hr, hc), nb*nb int64 offsets, then fp64 values (row-major per
 *   box), all packed back to back in buf.
 *  DD_PLAN_COO: (int32 x, int32 y, fp64 mass) records of the cell plans of
 *   the last sweep; intended for n <= 256.
 *  *bytes: in = capacity of buf, out = bytes required/written. */
int dd_fetch_plan(dd_ctx* ctx, int format, void* buf, size_t* bytes);

/* Statistics: last sweep / totals since init or dd_reset_totals. */
int dd_get_stats(dd_ctx* ctx, dd_sweep_stats* last);
int dd_get_totals(dd_ctx* ctx, dd_sweep_stats* totals);
int dd_reset_totals(dd_ctx* ctx);

/* dd_get_cell_stats -- per composite cell of the last sweep (cell index =
 * row-major over the partition's cell grid): Sinkhorn iterations, union
 * Y-box side max(b_r, b_c), MUFU ops of the solve, its duration on its SM
 * in units of 1024 cycles and its flags (bit 0: max_inner_iter reached, bit 1:
 * non-finite value / numerically empty kernel row, bit 2: eps raised by the
 * safeguard, bit 3: pool overflow) and the L1 X-error of its returned plan
 * as K1 evaluated it (relative to 1, not to ||mu_J||).  Any output may
 * be NULL.  Returns the number of cells (<= max_cells are written), or < 0 on
 * error (-DD_E*). */
int dd_get_cell_stats(dd_ctx* ctx, int* iters, int* box_side, double* mufu_ops, int* kcycles, int* flags,
                      float* err_x, int max_cells);

/* ---- multi-GPU stripes ----
 * One context per rank holds the whole layer but solves only the composite
 * cells of its stripe of basic-cell rows [row_lo, row_hi) (even bounds):
 * A-cell rows q with 2q in the stripe, B-cell rows q with 2q in the stripe
 * plus the last B row for the bottom stripe.  Before a B-sweep the row above
 * the stripe (row_lo - 1) must be imported from the rank above and the
 * stripe's last row (row_hi - 1) exported to the rank below and cleared;
 * after it row_lo - 1 goes back (export + clear here, import above).  The
 * caller moves the byte buffers (NCCL send/recv over NVLink via
 * torch.distributed in paper_2001_10986_b200/striped.py).  Per-cell
 * arithmetic does not depend on the stripe: results are bit-identical to
 * one context for every rank count. */

/* dd_set_stripe -- restrict sweeps and queries of the CURRENT layer to the
 * stripe; rows outside become empty.  (0, 0) = the whole layer (replicated).
 * dd_refine and dd_reset return to (0, 0). */
int dd_set_stripe(dd_ctx* ctx, int row_lo, int row_hi);

/* dd_clear_rows -- mark basic rows [row, row+nrows) empty (owned elsewhere). */
int dd_clear_rows(dd_ctx* ctx, int row, int nrows);

/* dd_export_rows -- pack basic rows [row, row+nrows) into a DEVICE buffer:
 * int4 boxes[nrows*nb] | int64 total, int64 count | fp64 values (each box
 * row-major, padded to an even length).  buf == NULL: *bytes = size needed
 * (synchronises).  The caller owns buf. */
int dd_export_rows(dd_ctx* ctx, int row, int nrows, void* buf, size_t* bytes);

/* dd_import_rows -- install rows exported by another context of the same
 * problem (same layer) from a DEVICE buffer; the values go to the pool's
 * halo region (one boundary row at a time; DD_ENOMEM if it does not fit). */
int dd_import_rows(dd_ctx* ctx, int row, int nrows, const void* buf, size_t bytes);

/* dd_compact -- K2 over the current pool: every stored box (including rows
 * imported into the halo region) moves into the main pool in basic-cell
 * order, freeing the halo slots (the multi-GPU driver calls it after moving
 * rows between stripes).  Asynchronous. */
int dd_compact(dd_ctx* ctx);

/* dd_export_rows_slab / dd_import_rows_slab -- the same rows through a
 * fixed-capacity DEVICE slab with no host-visible size, fully asynchronous
 * on the context stream (the multi-GPU exchange sends the whole slab with a
 * fixed NCCL count; no host synchronisation per exchange):
 *   int64 header[8] {magic, n boxes, padded entries, bytes needed, overflow}
 *   | int4 boxes[nrows*nb] | fp64 values (row-major, each padded to even).
 * A slab too small for the rows (header: overflow = 1) or one that fails
 * validation on import leaves the imported rows empty and is reported as
 * DD_ENOMEM by the next dd_synchronize.  slab_bytes >= 64 + 16*nrows*nb + 16;
 * size it from dd_export_rows(buf = NULL) once per layer.  Caller owns slab. */
int dd_export_rows_slab(dd_ctx* ctx, int row, int nrows, void* slab, size_t slab_bytes);
int dd_import_rows_slab(dd_ctx* ctx, int row, int nrows, const void* slab, size_t slab_bytes);

/* dd_copy_alpha -- copy pixel rows [row0, row0+nrows) of the X-potential
 * image alpha_A (partition 1) or alpha_B (2) of the current layer (fp64,
 * cost units, row-major, side columns) to (to_ctx = 0) or from (to_ctx = 1)
 * a caller DEVICE buffer.  The multi-GPU driver gathers the potentials of
 * all stripes with it before dd_refine glues them. */
int dd_copy_alpha(dd_ctx* ctx, int partition, int row0, int nrows, void* buf, int to_ctx);

/* dd_y_accumulate -- add this context's sum_i nu_i(y) (2^60 fixed point,
 * deterministic) into a caller-zeroed DEVICE array acc[side*side] of uint64;
 * sum the arrays of all ranks (allreduce), then dd_y_l1 gives
 * l1_y = sum_y |sum_i nu_i(y) - nu(y)| of the whole problem (A18). */
int dd_y_accumulate(dd_ctx* ctx, unsigned long long* acc);
int dd_y_l1(dd_ctx* ctx, const unsigned long long* acc, double* l1_y);

/* dd_phase_profile -- diagnostic: per-phase cycle counters of K1 summed over
 * warps since the last call (32 uint64: [mode][16], mode 0 = SMEM tier,
 * 1 = fused big-cell tiers; slots 0..5 = Y1 pass, barrier, Y2+X1, barrier,
 * X2 pass, error reduction; 6 = Sinkhorn loop, 7 = prologue, 8 = epilogue,
 * 9 = iterations).  All zero unless the library was built with
 * -DDD_PHASE_PROF (tools/phase_profile.py).  Resets the counters. */
int dd_phase_profile(dd_ctx* ctx, unsigned long long* out32);

/* State export/import for single-sweep parity.  Layout as in
 * DD_PLAN_BASIC_MARGINALS plus alpha_A, alpha_B (side*side fp64, cost units).
 * Host buffers; values sized by dd_get_state_info().entries. */
int dd_get_state_info(dd_ctx* ctx, dd_state_info* info);
int dd_get_state(dd_ctx* ctx, int* boxes, long long* offsets, double* values,
                 double* alpha_A, double* alpha_B);
int dd_set_state(dd_ctx* ctx, int side, long long half_index, int last_partition,
                 const int* boxes, const long long* offsets, const double* values,
                 long long n_values, const double* alpha_A, const double* alpha_B);

/* Schedule of the LADDER driver: up to max stages
 * (side, kappa, sweeps); returns the stage count. */
int dd_build_schedule(int n_final, int coarsest_side, double kappa_final, double eps_start,
                      int* side, double* kappa, int* sweeps, int max);

/* Measured MUFU (ex2.approx) throughput of this device in ops/s, and the SM
 * clock (MHz) the measurement ran at (roofline denominator). */
int dd_measure_mufu_peak(int device, double* ops_per_s);

/* dd_synchronize -- wait for the context's work.  DD_ENOMEM on a pool or
 * box-size overflow; DD_ENOCONV if cells hit max_inner_iter since the last
 * report (each failure is reported once; dd_reset_totals forgets them). */
int dd_synchronize(dd_ctx* ctx);
void dd_free(dd_ctx* ctx);
const char* dd_last_error(const dd_ctx* ctx);
const char* dd_version(void);

#ifdef __cplusplus
}
#endif
#endif
