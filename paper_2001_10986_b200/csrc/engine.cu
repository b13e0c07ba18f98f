// engine.cu -- host side of libdd_gpu.so: the C-ABI of include/dd.h, device
// memory management, the sweep pipeline (K1 -> K2 -> K3) and the
// coarse-to-fine / eps-scaling driver.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dd.h"
#include "dd_aux.cuh"

using namespace dd;

namespace {

constexpr int kMaxLayers = 16;

struct Layer {
    int side = 0, s = 0, nb = 0;
    double* mu = nullptr;
    double* nu = nullptr;
    double* logmu = nullptr;
    double* mass = nullptr;
};

struct SweepEvents {
    cudaEvent_t e[3];
};

}  // namespace

struct dd_ctx {
    dd_options opt{};
    int device = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int n_layers = 0, cur = 0;
    Layer L[kMaxLayers];
    double eps = 0, eps_final = 0, tau = 1e-15;
    int cell_size = 0;
    // state (sized for the finest layer)
    double* alphaA = nullptr;
    double* alphaB = nullptr;
    int4* box = nullptr;
    int4* box2 = nullptr;
    long long* off = nullptr;
    long long* off2 = nullptr;
    double* pool = nullptr;
    double* scratch = nullptr;
    long long cap = 0;
    // sweep plumbing
    unsigned long long* bump = nullptr;
    int* lists = nullptr;           // tier lists [3][ncell_max] (K0) + LPT-sorted tiers 1, 2 [2][ncell_max]
                                    // + the cluster tier's list [ncell_max] (K0c)
    int* bside = nullptr;           // LPT sort key per cell (K0)
    int* ipred = nullptr;           // [2][ncell_max] iterations of each cell's last solve, per partition
    int ipred_layer = -1;           // layer the predictions belong to
    int* counters = nullptr;        // [0..2] tier counts, [3..5] work counters, [6] overflow,
                                    // [8] cluster-tier count, [9] its work counter, [10..11] sum of K0 work (u64)
    unsigned char* slices[2] = {nullptr, nullptr};   // BIG tiers: per-CTA global slices (log nu_cell, ACC)
    long long slice_bytes[2] = {0, 0};
    int slice_cap[2] = {0, 0};      // box side the slices were sized for
    int grid_t[2] = {0, 0};         // persistent grid of tiers 1, 2
    cudaStream_t st_t[2] = {nullptr, nullptr};   // tier 1 / tier 2 streams
    // cluster tier: ncl persistent clusters of kClusterSize CTAs,
    // one global slice per cluster, its own high-priority stream
    int ncl = 0;
    int cl_mode = 0;                // 0 auto (long poles), 1 every big-path cell
    float cl_theta = 1.0f;
    int nsm = 148;
    unsigned char* cl_slices = nullptr;
    cudaStream_t st_cl = nullptr;
    cudaEvent_t ev_join_cl = nullptr;
    cudaEvent_t ev_batch = nullptr;  // dd_run_schedule_batch fork / join
    int poison = 0;                 // DD_POISON (testing): poisoned buffers and K1 SMEM
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
    CellOut* cellout = nullptr;
    long long* d_total = nullptr;   // [0] padded pool length, [1] entries
    DevStats* d_last = nullptr;
    DevStats* d_tot = nullptr;
    int ncell_max = 0;
    int bcap_main = 32, bcap_big = 32, bcap_big2 = 32;
    size_t smem_main = 0, smem_big = 0, smem_big2 = 0;
    int grid_big = 148;
    // evaluation scratch
    double* eval_scratch = nullptr;
    size_t eval_scratch_bytes = 0;
    double* eval_res = nullptr;
    size_t eval_res_n = 0;
    double* d_sums = nullptr;       // 4 doubles
    unsigned long long* yacc = nullptr;
    double* partial = nullptr;
    // multi-GPU stripe of the current layer: basic rows [stripe_lo, stripe_hi)
    // (0, 0 = the whole layer); imported boundary rows live in the last
    // halo_cap entries of the pool
    int stripe_lo = 0, stripe_hi = 0;
    long long halo_cap = 0;
    long long* d_xoff = nullptr;    // row export/import offsets scratch
    double* glue = nullptr;         // K5 potential refinement scratch
    // general separable cost (dd_set_cost): finest-grid tables h1 (rows), h2 (columns)
    double* d_h1 = nullptr;
    double* d_h2 = nullptr;
    // tier G: per-CTA global-memory layouts of the SMEM-tier kernel
    // for the cells beyond every on-chip tier (allocated at the first layer
    // whose boxes can exceed the on-chip caps)
    unsigned char* gslab = nullptr;
    long long gslab_bytes = 0;
    size_t gslab_alloc = 0;
    bool serial = false;            // DD_SERIAL_TIERS=1: all K1 tiers on one stream (profiling)
    long long xoff_n = 0;
    // host bookkeeping
    long long half_index = 0;
    int last_part = 0;
    std::vector<SweepEvents> pending;
    std::vector<SweepEvents> free_events;
    double ms_last = 0, solve_ms_last = 0, ms_tot = 0, solve_ms_tot = 0;
    long long failed_seen = 0;      // failed cells already reported by dd_synchronize
    long long launches_last = 0, launches_tot = 0, launches_pending = 0;
    std::string err;
};

namespace {

void set_err(dd_ctx* c, const char* fmt, ...) {
    if (!c) return;
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    c->err = buf;
}

#define CK(call)                                                                     \
    do {                                                                             \
        cudaError_t _e = (call);                                                     \
        if (_e != cudaSuccess) {                                                     \
            set_err(c, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
            return _e == cudaErrorMemoryAllocation ? DD_ENOMEM : DD_ECUDA;           \
        }                                                                            \
    } while (0)

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

int cells_axis(int nb, int part) { return part == 1 ? nb / 2 : nb / 2 + 1; }

// Partition cell rows [cr0, cr1) a context solves: A-cell row q covers basic
// rows 2q, 2q+1; B-cell row q covers 2q-1, 2q.  A stripe owns
// the cells whose LOWER basic row lies in it, plus the last B row at the end.
void cell_rows(const dd_ctx* c, int part, int nb, int* cr0, int* cr1) {
    if (c->stripe_hi <= c->stripe_lo) { *cr0 = 0; *cr1 = cells_axis(nb, part); return; }
    *cr0 = c->stripe_lo / 2;
    *cr1 = c->stripe_hi / 2 + ((part == 2 && c->stripe_hi == nb) ? 1 : 0);
}

// Schedule of P:1553-1561 (A12).  Independent of the oracle's copy.
int build_schedule(int n_final, int coarsest, double kappa_final, double eps_start, int* side, double* kappa,
                   int* sweeps, int max) {
    int k = 0;
    auto push = [&](int sd, double kk, int w) {
        if (k < max) { side[k] = sd; kappa[k] = kk; sweeps[k] = w; }
        ++k;
    };
    if (coarsest <= 0) coarsest = 8;
    if (coarsest > n_final) coarsest = n_final;
    for (int sd = coarsest; sd <= n_final; sd *= 2) {
        const bool finest = (sd == n_final);
        if (sd == coarsest && eps_start > 0.0) {
            const double ks = eps_start * (double)sd * (double)sd;
            for (double kk = ks; kk > 2.0 * (1.0 + 1e-12); kk *= 0.5) push(sd, kk, 2);
        }
        if (finest && kappa_final > 2.0 * (1.0 + 1e-12)) { push(sd, kappa_final, 4); continue; }
        push(sd, 2.0, 4);
        if (!finest) { push(sd, 1.0, 2); push(sd, 0.5, 2); }
        else
            for (double kk = 1.0; kk >= kappa_final * (1.0 - 1e-12); kk *= 0.5) push(sd, kk, 2);
    }
    return k;
}

int alloc_events(dd_ctx* c, SweepEvents& ev) {
    if (!c->free_events.empty()) {
        ev = c->free_events.back();
        c->free_events.pop_back();
        return DD_OK;
    }
    for (int k = 0; k < 3; ++k) CK(cudaEventCreate(&ev.e[k]));
    return DD_OK;
}

// Harvest the timings of finished sweeps (synchronises the stream).
int harvest(dd_ctx* c) {
    CK(cudaStreamSynchronize(c->st));
    for (auto& ev : c->pending) {
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, ev.e[0], ev.e[2]));
        CK(cudaEventElapsedTime(&b, ev.e[0], ev.e[1]));
        c->ms_last = a;
        c->solve_ms_last = b;
        c->ms_tot += a;
        c->solve_ms_tot += b;
        c->free_events.push_back(ev);
    }
    c->pending.clear();
    c->launches_tot += c->launches_pending;
    c->launches_pending = 0;
    return DD_OK;
}

int check_overflow(dd_ctx* c);
// Wait for the context's work and report pool / box-size overflows.
int sync_state(dd_ctx* c) {
    int rc = harvest(c);
    if (rc) return rc;
    return check_overflow(c);
}

int check_overflow(dd_ctx* c) {
    int ov = 0;
    CK(cudaMemcpyAsync(&ov, c->counters + 6, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (ov & 1) {
        set_err(c, "nu_i pool capacity (%lld entries) exceeded; raise dd_options.pool_capacity", c->cap);
        return DD_ENOMEM;
    }
    if (ov & 2) {
        set_err(c, "a composite cell's Y box exceeds the largest supported box side (%d)", c->bcap_big2);
        return DD_ENOMEM;
    }
    if (ov & 4) {
        set_err(c, "a row slab overflowed its capacity or failed validation (dd_export_rows_slab / "
                   "dd_import_rows_slab); the imported rows were left empty");
        return DD_ENOMEM;
    }
    return DD_OK;
}

// Box-side capacities of the three K1 tiers for basic cell side s:
//   tier 0 (SMEM path, 256 threads, 3 CTAs/SM): union Y box <= bcap_main;
//   tier 1 (BIG path, kT1Threads = 256 threads, kT1PerSM = 3 CTAs/SM, <= 80 regs): <= bcap_big (<= kCap1);
//   tier 2 (BIG path, kT2Threads = 768 threads, 1 CTA/SM, <= 80 regs): <= bcap_big2 (<= kCap2).
#ifndef DD_T1_CAP
#define DD_T1_CAP 120
#endif
constexpr int kCap1 = DD_T1_CAP, kCap2 = 704;
#ifndef DD_NCL
#define DD_NCL 6
#endif
constexpr int kDefaultClusters = DD_NCL;   // persistent clusters of the cluster tier
constexpr int kTierG = 4;                  // CTAs of tier G (global-memory layouts)
// SMEM per CTA: 228 KB per SM shared by the resident CTAs, 1 KB reserved per CTA, ~1 KB static
constexpr size_t kSmem1 = 233472 / kT1PerSM - 2048, kSmem2 = kT2PerSM == 1 ? 220 * 1024 : 233472 / kT2PerSM - 2048;
void tier_caps(int s, int opt_main, int opt_big, int* b0, int* b1, int* b2) {
    int want = (s <= 4) ? 32 : 24;   // measured: the fused path wins above ~24 px (s = 8)
    if (opt_main > 0) want = opt_main;
    if (want < 2 * s + 2) want = 2 * s + 2;
    *b0 = want;
    int big = want;
    while (big < kCap1 && k1_smem_bytes_host(s, big + 1, true, kT1Threads / 32) <= kSmem1) ++big;
    int big2 = big;
    if (opt_big > 0 && opt_big >= want && opt_big < big) big = opt_big;   // testing: force tier 2
    *b1 = big;
    while (big2 < kCap2 && k1_smem_bytes_host(s, big2 + 1, true, kT2Threads / 32) <= kSmem2) ++big2;
    *b2 = big2;
}

void choose_caps(dd_ctx* c, int s) {
    int b0, b1, b2;
    if (c->d_h1 || s > 8) {
        // general costs and s = 16 run on the SMEM tier only (DESIGN.md "general
        // costs, s = 16"): its box capacity is raised to what one SM holds
        // (1 CTA/SM at the largest boxes); a cell beyond it is flagged by the
        // big tiers (DD_ENOMEM), never solved with the wrong arithmetic
        const bool gc = c->d_h1 != nullptr;
        int b = std::max(2 * s + 2, 24);
        while (b < 4096 && k1_smem_bytes_host(s, b + 1, false, 0, gc) <= kSmem2) ++b;
        c->bcap_main = b;
        c->smem_main = k1_smem_bytes_host(s, b, false, 0, gc);
        c->bcap_big = c->bcap_big2 = b;
        c->smem_big = k1_smem_bytes_host(s < 8 ? s : 8, std::min(b, c->slice_cap[0]), true, kT1Threads / 32);
        c->smem_big2 = k1_smem_bytes_host(s < 8 ? s : 8, std::min(b, c->slice_cap[1]), true, kT2Threads / 32);
        return;
    }
    tier_caps(s, c->opt.reserved[0], c->opt.reserved[1], &b0, &b1, &b2);
    c->bcap_main = b0;
    c->smem_main = k1_smem_bytes_host(s, b0);
    c->bcap_big = std::min(b1, c->slice_cap[0]);
    c->smem_big = k1_smem_bytes_host(s, c->bcap_big, true, kT1Threads / 32);
    c->bcap_big2 = std::min(b2, c->slice_cap[1]);
    if (c->opt.reserved[6] > 0) {     // testing: cells above this side go to tier G
        c->bcap_big2 = std::max(std::min(c->bcap_big2, c->opt.reserved[6]), c->bcap_main);
        c->bcap_big = std::min(c->bcap_big, c->bcap_big2);
        c->smem_big = k1_smem_bytes_host(s, c->bcap_big, true, kT1Threads / 32);
    }
    c->smem_big2 = k1_smem_bytes_host(s, c->bcap_big2, true, kT2Threads / 32);
}

// BIG tiers: layout of a CTA's global slice for box side cap q.bcap:
// log nu_cell (b^2 float2) | phase-A stabilisers (b^2 float) | extraction sums (b^2 float4)
void slice_offsets(SweepParams& q) {
    auto al = [](long long v) { return (v + 255) & ~255LL; };
    const long long b2 = (long long)q.bcap * q.bcap;
    q.sl_off = al(b2 * (long long)sizeof(float2));
    q.acc_off = q.sl_off + al(b2 * (long long)sizeof(float));
}

// One sweep (Alg. 2 lines 6-14) over the partition selected by the parity of
// the half-iteration index (line 7: odd l -> A).
//   K0 classify cells by union Y-box side -> tier lists (big tiers LPT-sorted)
//   tiers 2 | 1 | 0 run concurrently on three streams (fork/join events)
//   K2 deterministic compaction, K3 fixed-order statistics
int sweep(dd_ctx* c) {
    Layer& Lr = c->L[c->cur];
    const int part = (c->half_index % 2 == 0) ? 1 : 2;
    const int nca = cells_axis(Lr.nb, part);
    const int ncells = nca * nca;
    choose_caps(c, Lr.s);
    CK(cudaMemsetAsync(c->bump, 0, sizeof(unsigned long long), c->st));
    CK(cudaMemsetAsync(c->counters, 0, 6 * sizeof(int), c->st));
    CK(cudaMemsetAsync(c->counters + 8, 0, 6 * sizeof(int), c->st));
    SweepParams p{};
    p.part = part;
    p.side = Lr.side; p.s = Lr.s; p.nb = Lr.nb; p.nca = nca; p.ncells = ncells;
    cell_rows(c, part, Lr.nb, &p.cr0, &p.cr1);
    p.eps = c->eps;
    p.h1 = c->d_h1; p.h2 = c->d_h2; p.hst = c->L[c->n_layers - 1].side / Lr.side;
    p.safeguard = (c->opt.flags & DD_FLAG_SAFEGUARD) ? 1 : 0;
    p.force_cell = -1;
    p.force_it = 0;
    if (const char* e = getenv("DD_FORCE_RESCUE")) {
        int a = -1, b = 0;
        if (sscanf(e, "%d:%d", &a, &b) == 2 && b >= 1) { p.force_cell = a; p.force_it = b; }
    }
    p.kappa = c->eps * (double)Lr.side * (double)Lr.side;
    p.tau = c->tau;
    p.err_tol = c->opt.err_tol;
    p.max_iter = c->opt.max_inner_iter;
    p.check_every = c->opt.check_every;
    p.box = c->box; p.off = c->off;
    p.pool_in = c->pool; p.scratch = c->scratch; p.bump = c->bump; p.cap = c->cap - c->halo_cap;
    p.alpha = part == 1 ? c->alphaA : c->alphaB;
    p.mu = Lr.mu; p.logmu = Lr.logmu; p.mass_i = Lr.mass;
    p.out = c->cellout;
    p.overflow = c->counters + 6;
    p.poison = c->poison;
    // work predictor for the LPT order (order only: results do not depend on it)
    if (c->ipred_layer != c->cur) {
        CK(cudaMemsetAsync(c->ipred, 0, (size_t)2 * c->ncell_max * sizeof(int), c->st));
        c->ipred_layer = c->cur;
    }
    p.ipred = c->ipred + (size_t)(part - 1) * c->ncell_max;
    SweepEvents ev;
    int rc = alloc_events(c, ev);
    if (rc) return rc;
    CK(cudaEventRecord(ev.e[0], c->st));
    int* sorted = c->lists + 3 * (size_t)c->ncell_max;
    CK(launch_k0(p, c->bcap_main, c->bcap_big, c->bcap_big2, c->lists, c->counters, c->ncell_max, c->bside, sorted,
                 c->st));
    int* list3 = c->lists + 5 * (size_t)c->ncell_max;
    if (c->ncl > 0)
        CK(launch_k0_cluster(sorted, c->counters, c->ncell_max, c->bside, c->cl_theta, c->nsm, c->cl_mode, list3,
                             c->st));
    CK(cudaEventRecord(c->ev_fork, c->st));
    CK(cudaStreamWaitEvent(c->st_t[0], c->ev_fork, 0));
    CK(cudaStreamWaitEvent(c->st_t[1], c->ev_fork, 0));
    if (c->ncl > 0) {
        // cluster tier first: its clusters need kClusterSize free SMs of a GPC at once
        CK(cudaStreamWaitEvent(c->st_cl, c->ev_fork, 0));
        SweepParams q = p;
        q.bcap = c->bcap_big2;
        q.list_in = list3; q.n_in = c->counters + 8; q.work_counter = c->counters + 9;
        q.gscratch = c->cl_slices; q.gslice = c->slice_bytes[1];
        slice_offsets(q);
        const cudaError_t e3 = launch_k1(q, 3, c->ncl, c->smem_big2, c->serial ? c->st : c->st_cl);
        if (e3 != cudaSuccess) {
            set_err(c, "K1 cluster tier launch (%d clusters of %d, smem %zu): %s", c->ncl, kClusterSize,
                    c->smem_big2, cudaGetErrorString(e3));
            return DD_ECUDA;
        }
    }
    {   // tier 2: the largest boxes (LPT order), fused path, 768 threads, 1 CTA/SM
        SweepParams q = p;
        q.bcap = c->bcap_big2;
        q.list_in = sorted + c->ncell_max; q.n_in = c->counters + 2; q.work_counter = c->counters + 5;
        q.gscratch = c->slices[1]; q.gslice = c->slice_bytes[1];
        slice_offsets(q);
        CK(launch_k1(q, 2, std::min(c->grid_t[1], ncells), c->smem_big2, c->serial ? c->st : c->st_t[1]));
    }
    {   // tier 1: fused path, 256 threads, 3 CTAs/SM (LPT order)
        SweepParams q = p;
        q.bcap = c->bcap_big;
        q.list_in = sorted; q.n_in = c->counters + 1; q.work_counter = c->counters + 4;
        q.gscratch = c->slices[0]; q.gslice = c->slice_bytes[0];
        slice_offsets(q);
        const cudaError_t e1 = launch_k1(q, 1, std::min(c->grid_t[0], ncells), c->smem_big, c->serial ? c->st : c->st_t[0]);
        if (e1 != cudaSuccess) {
            set_err(c, "K1 tier 1 launch (grid %d, smem %zu, bcap %d): %s", std::min(c->grid_t[0], ncells),
                    c->smem_big, q.bcap, cudaGetErrorString(e1));
            return DD_ECUDA;
        }
    }
    {   // tier 0: the bulk, several CTAs per SM
        SweepParams q = p;
        q.bcap = c->bcap_main;
        q.list_in = c->lists; q.n_in = c->counters; q.work_counter = c->counters + 3;
        CK(launch_k1(q, 0, std::min(ncells, c->grid_big * 8), c->smem_main, c->st));
    }
    bool tier_g = false;
    if (Lr.side > c->bcap_big2) {
        // tier G: cells whose union box exceeds every on-chip tier (K0 list 6)
        // run the SMEM-tier kernel on a global-memory layout, kTierG CTAs
        const bool gc = c->d_h1 != nullptr;
        const long long per = (long long)((k1_smem_bytes_host(Lr.s, Lr.side, false, 0, gc) + 255) & ~size_t(255));
        const size_t need = (size_t)per * kTierG;
        if (need > c->gslab_alloc) {
            CK(cudaStreamSynchronize(c->st));
            if (c->gslab) CK(cudaFree(c->gslab));
            c->gslab = nullptr;
            c->gslab_alloc = 0;
            CK(cudaMalloc(&c->gslab, need));
            c->gslab_alloc = need;
        }
        SweepParams q = p;
        q.bcap = Lr.side;
        q.list_in = c->lists + 6 * (size_t)c->ncell_max; q.n_in = c->counters + 12; q.work_counter = c->counters + 13;
        q.gbase = c->gslab; q.gbase_bytes = per;
        q.poison = 0;
        CK(launch_k1(q, 0, kTierG, 0, c->st));
        tier_g = true;
    }
    CK(cudaEventRecord(c->ev_join[0], c->st_t[0]));
    CK(cudaEventRecord(c->ev_join[1], c->st_t[1]));
    CK(cudaStreamWaitEvent(c->st, c->ev_join[0], 0));
    CK(cudaStreamWaitEvent(c->st, c->ev_join[1], 0));
    if (c->ncl > 0) {
        CK(cudaEventRecord(c->ev_join_cl, c->st_cl));
        CK(cudaStreamWaitEvent(c->st, c->ev_join_cl, 0));
    }
    CK(cudaEventRecord(ev.e[1], c->st));
    // K2: deterministic compaction of the new boxes into the pool
    const int nb2 = Lr.nb * Lr.nb;
    CK(launch_scan_areas(c->box, c->off2, c->d_total, nb2, c->d_total + 1, c->st));
    CK(launch_copy_boxes(c->box, c->off, c->off2, c->scratch, c->pool, nb2, c->cap - c->halo_cap, c->st));
    std::swap(c->off, c->off2);
    // K3: fixed-order sweep statistics
    CK(launch_reduce_stats(c->cellout, ncells, c->d_last, c->d_tot, c->d_total + 1, c->counters + 1,
                           c->counters + 6, c->counters + 2, c->st));
    CK(cudaEventRecord(ev.e[2], c->st));
    c->pending.push_back(ev);
    c->launches_pending += (c->ncl > 0 ? 10 : 8) + (tier_g ? 1 : 0);
    c->half_index++;
    c->last_part = part;
    if (c->pending.size() > 512) return harvest(c);
    return DD_OK;
}

int product_init(dd_ctx* c) {
    Layer& Lr = c->L[c->cur];
    const long long need = (long long)Lr.nb * Lr.nb * Lr.side * Lr.side;
    if (need > c->cap - c->halo_cap) {
        set_err(c, "pool capacity too small for the product initialisation");
        return DD_ENOMEM;
    }
    CK(launch_product_init(c->box, c->off, c->pool, Lr.mass, Lr.nu, Lr.side, Lr.nb, c->st));
    const size_t n2 = (size_t)c->L[c->n_layers - 1].side * c->L[c->n_layers - 1].side;
    CK(cudaMemsetAsync(c->alphaA, 0, n2 * sizeof(double), c->st));
    CK(cudaMemsetAsync(c->alphaB, 0, n2 * sizeof(double), c->st));
    CK(cudaMemsetAsync(c->counters, 0, 8 * sizeof(int), c->st));
    c->half_index = 0;
    c->last_part = 0;
    return DD_OK;
}

void free_all(dd_ctx* c) {
    for (int k = 0; k < c->n_layers; ++k) {
        cudaFree(c->L[k].mu); cudaFree(c->L[k].nu); cudaFree(c->L[k].logmu); cudaFree(c->L[k].mass);
    }
    void* ptrs[] = {c->alphaA, c->alphaB, c->box, c->box2, c->off, c->off2, c->pool, c->scratch,
                    c->bump, c->lists, c->bside, c->ipred, c->slices[0], c->slices[1], c->counters, c->cellout, c->d_total, c->d_last, c->d_tot,
                    c->eval_scratch, c->eval_res, c->d_sums, c->yacc, c->partial, c->d_xoff, c->glue, c->cl_slices,
                    c->d_h1, c->d_h2, c->gslab};
    for (void* q : ptrs) if (q) cudaFree(q);
    for (auto& ev : c->pending) for (int k = 0; k < 3; ++k) cudaEventDestroy(ev.e[k]);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (int k = 0; k < 2; ++k) {
        if (c->ev_join[k]) cudaEventDestroy(c->ev_join[k]);
        if (c->st_t[k]) cudaStreamDestroy(c->st_t[k]);
    }
    if (c->ev_join_cl) cudaEventDestroy(c->ev_join_cl);
    if (c->ev_batch) cudaEventDestroy(c->ev_batch);
    if (c->st_cl) cudaStreamDestroy(c->st_cl);
    for (auto& ev : c->free_events) for (int k = 0; k < 3; ++k) cudaEventDestroy(ev.e[k]);
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
}

// Evaluate the plan of the last swept partition (K7) -> sums[0..2] = cost, ent, l1x.
int evaluate(dd_ctx* c, double* out3, bool coo, long long* coo_count, int* cx, int* cy, double* cm) {
    Layer& Lr = c->L[c->cur];
    const int part = c->last_part ? c->last_part : 1;
    const int nca = cells_axis(Lr.nb, part);
    const int ncells = nca * nca;
    const int nb2 = Lr.nb * Lr.nb;
    std::vector<int4> hbox(nb2);
    CK(cudaMemcpyAsync(hbox.data(), c->box, nb2 * sizeof(int4), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    // per-cell union boxes on the host (sizes only) for the scratch and COO
    // layouts: cell k's scratch (nu_cell, g: ny each; f: nx) starts at the
    // prefix sum of the earlier cells' 2 ny + nx (no per-cell worst case)
    std::vector<long long> coo_off(ncells + 1, 0), scr_off(ncells + 1, 0);
    int cr0, cr1;
    cell_rows(c, part, Lr.nb, &cr0, &cr1);
    for (int cell = 0; cell < ncells; ++cell) {
        const int cp = cell / nca, cq = cell % nca;
        int rlo, rhi, clo, chi;
        auto span = [&](int q, int& lo, int& hi) {
            if (part == 1) { lo = 2 * q; hi = 2 * q + 1; }
            else { lo = std::max(2 * q - 1, 0); hi = std::min(2 * q, Lr.nb - 1); }
        };
        span(cp, rlo, rhi);
        span(cq, clo, chi);
        int y0 = 1 << 30, x0 = 1 << 30, y1 = -1, x1 = -1;
        for (int r = rlo; r <= rhi; ++r)
            for (int q = clo; q <= chi; ++q) {
                const int4 b = hbox[r * Lr.nb + q];
                if (b.z <= 0 || b.w <= 0) continue;
                y0 = std::min(y0, b.x); x0 = std::min(x0, b.y);
                y1 = std::max(y1, b.x + b.z - 1); x1 = std::max(x1, b.y + b.w - 1);
            }
        const long long ny = y1 >= 0 ? (long long)(y1 - y0 + 1) * (x1 - x0 + 1) : 0;
        const long long nx = (long long)(rhi - rlo + 1) * (chi - clo + 1) * Lr.s * Lr.s;
        const bool own = cp >= cr0 && cp < cr1;
        coo_off[cell + 1] = coo_off[cell] + (own ? nx * ny : 0LL);
        scr_off[cell + 1] = scr_off[cell] + (own ? 2 * ny + nx : 0LL);
    }
    const size_t need = (size_t)std::max(1LL, scr_off[ncells]) * sizeof(double) + (size_t)(ncells + 1) * sizeof(long long);
    if (need > c->eval_scratch_bytes) {
        if (c->eval_scratch) cudaFree(c->eval_scratch);
        c->eval_scratch = nullptr;
        c->eval_scratch_bytes = 0;
        CK(cudaMalloc(&c->eval_scratch, need));
        c->eval_scratch_bytes = need;
    }
    long long* d_scr_off = reinterpret_cast<long long*>(c->eval_scratch + std::max(1LL, scr_off[ncells]));
    CK(cudaMemcpyAsync(d_scr_off, scr_off.data(), (ncells + 1) * sizeof(long long), cudaMemcpyHostToDevice, c->st));
    if ((size_t)3 * ncells > c->eval_res_n) {
        if (c->eval_res) cudaFree(c->eval_res);
        c->eval_res = nullptr;
        CK(cudaMalloc(&c->eval_res, 3 * ncells * sizeof(double)));
        c->eval_res_n = 3 * ncells;
    }
    EvalParams p{};
    p.part = part; p.side = Lr.side; p.s = Lr.s; p.nb = Lr.nb; p.nca = nca;
    p.eps = c->eps;
    p.h1 = c->d_h1; p.h2 = c->d_h2; p.hst = c->L[c->n_layers - 1].side / Lr.side;
    p.box = c->box; p.off = c->off; p.pool = c->pool;
    p.alpha = part == 1 ? c->alphaA : c->alphaB;
    p.mu = Lr.mu; p.logmu = Lr.logmu; p.nu = Lr.nu;
    p.scratch = c->eval_scratch; p.scratch_off = d_scr_off;
    p.cell_res = c->eval_res;
    p.cr0 = cr0; p.cr1 = cr1;
    long long* d_coo_off = nullptr;
    int* dx = nullptr;
    int* dy = nullptr;
    double* dm = nullptr;
    const long long total = coo_off[ncells];
    if (coo) {
        if (coo_count) *coo_count = total;
        if (!cx) return DD_OK;   // size query
        CK(cudaMalloc(&d_coo_off, (ncells + 1) * sizeof(long long)));
        CK(cudaMalloc(&dx, std::max(1LL, total) * sizeof(int)));
        CK(cudaMalloc(&dy, std::max(1LL, total) * sizeof(int)));
        CK(cudaMalloc(&dm, std::max(1LL, total) * sizeof(double)));
        CK(cudaMemcpyAsync(d_coo_off, coo_off.data(), (ncells + 1) * sizeof(long long), cudaMemcpyHostToDevice, c->st));
        p.coo = 1; p.coo_off = d_coo_off; p.coo_x = dx; p.coo_y = dy; p.coo_m = dm;
    }
    CK(launch_eval(p, ncells, c->d_sums, c->st));
    CK(cudaMemcpyAsync(out3, c->d_sums, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    if (coo) {
        CK(cudaMemcpyAsync(cx, dx, total * sizeof(int), cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(cy, dy, total * sizeof(int), cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(cm, dm, total * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    if (coo) { cudaFree(d_coo_off); cudaFree(dx); cudaFree(dy); cudaFree(dm); }
    return DD_OK;
}

void fill_stats(const DevStats& d, dd_sweep_stats* s) {
    s->cells = d.cells;
    s->iters_sum = d.iters_sum;
    s->iters_max = d.iters_max;
    s->failed = d.failed;
    s->err_x_sum = d.err_sum;
    s->entries = d.entries;
    s->mufu_ops = d.mufu;
    s->big_cells = d.deferred + d.huge;
    s->max_box = d.max_box;
    s->reserved_i = (int)std::min<long long>(d.fallbacks, 2147483647LL);
    s->cluster_cells = d.cluster;
}

}  // namespace

// =================================================================== ABI ==
extern "C" {

const char* dd_version(void) { return "ddot-b200 0.1 (sm_100a)"; }

const char* dd_last_error(const dd_ctx* c) { return c ? c->err.c_str() : "null context"; }

int dd_build_schedule(int n_final, int coarsest_side, double kappa_final, double eps_start, int* side,
                      double* kappa, int* sweeps, int max) {
    return build_schedule(n_final, coarsest_side, kappa_final, eps_start, side, kappa, sweeps, max);
}

int dd_init(dd_ctx** out, int n, const double* mu, const double* nu, int cost, double eps, int cell_size,
            const dd_options* opt) {
    if (!out) return DD_EINVAL;
    *out = nullptr;
    dd_ctx* c = new (std::nothrow) dd_ctx();
    if (!c) return DD_ENOMEM;
    *out = c;
    if (opt) c->opt = *opt;
    if (c->opt.err_tol <= 0) c->opt.err_tol = 1e-6;
    if (c->opt.max_inner_iter <= 0) c->opt.max_inner_iter = 10000;
    if (c->opt.check_every <= 0) c->opt.check_every = 1;
    c->tau = c->opt.trunc_tau == 0.0 ? 1e-15 : (c->opt.trunc_tau < 0 ? 0.0 : c->opt.trunc_tau);
    if (c->opt.no_truncate) c->tau = 0.0;
    if (cost != DD_COST_SQEUCLID) { set_err(c, "only DD_COST_SQEUCLID is supported"); return DD_EINVAL; }
    if (!is_pow2(n) || n < 4) { set_err(c, "n=%d must be a power of two >= 4", n); return DD_EINVAL; }
    if (!is_pow2(cell_size) || cell_size > n / 2 || (n / cell_size) % 2) {
        set_err(c, "cell_size=%d must be a power of two with n/s even", cell_size);
        return DD_EINVAL;
    }
    if (!(eps > 0.0) || !std::isfinite(eps)) { set_err(c, "eps must be > 0"); return DD_EINVAL; }
    if (!mu || !nu) { set_err(c, "null marginal"); return DD_EINVAL; }
    // ---- device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_err(c, "no CUDA device: this library has no CPU fallback");
        return DD_ECUDA;
    }
    c->device = c->opt.device;
    CK(cudaSetDevice(c->device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major < 10) {
        set_err(c, "device %s (sm_%d%d) is not sm_100: this build targets B200 only", prop.name, prop.major, prop.minor);
        return DD_ECUDA;
    }
    c->grid_big = prop.multiProcessorCount;
    {
        const char* e = getenv("DD_SERIAL_TIERS");
        c->serial = e && e[0] == '1';
    }
    if (c->opt.stream) c->st = (cudaStream_t)c->opt.stream;
    else {
        CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    // ---- host validation (every basic cell of every layer has mass > 0)
    const size_t n2 = (size_t)n * n;
    std::vector<double> hmu(n2), hnu(n2);
    if (c->opt.flags & DD_FLAG_DEVICE_INPUT) {
        CK(cudaMemcpy(hmu.data(), mu, n2 * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hnu.data(), nu, n2 * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
        memcpy(hmu.data(), mu, n2 * sizeof(double));
        memcpy(hnu.data(), nu, n2 * sizeof(double));
    }
    // compensated (Neumaier) sums: a plain running sum of 4M masses drifts by
    // ~1e-12, the size of the equality tolerance itself
    double smu = 0, snu = 0, cmu = 0, cnu = 0;
    auto nadd = [](double& sum, double& comp, double x) {
        const double t = sum + x;
        comp += (std::fabs(sum) >= std::fabs(x)) ? (sum - t) + x : (x - t) + sum;
        sum = t;
    };
    for (size_t k = 0; k < n2; ++k) {
        if (!std::isfinite(hmu[k]) || hmu[k] < 0 || !std::isfinite(hnu[k]) || hnu[k] < 0) {
            set_err(c, "marginals must be finite and >= 0 (index %zu)", k);
            return DD_EINVAL;
        }
        nadd(smu, cmu, hmu[k]);
        nadd(snu, cnu, hnu[k]);
    }
    smu += cmu;
    snu += cnu;
    if (!(smu > 0) || std::fabs(smu - snu) > 1e-12 * smu) {
        set_err(c, "||mu|| = %.17g != ||nu|| = %.17g", smu, snu);
        return DD_EINVAL;
    }
    int coarsest = n;
    if (c->opt.schedule == DD_SCHED_LADDER) {
        coarsest = c->opt.coarsest_side > 0 ? c->opt.coarsest_side : 8;
        if (!is_pow2(coarsest) || coarsest < 4) { set_err(c, "bad coarsest_side"); return DD_EINVAL; }
        coarsest = std::min(coarsest, n);
    }
    int nl = 0;
    for (int sd = coarsest; sd <= n; sd *= 2) ++nl;
    if (nl > kMaxLayers) { set_err(c, "too many layers"); return DD_EINVAL; }
    c->n_layers = nl;
    c->cell_size = cell_size;
    {   // host-side basic-cell masses per layer (validation only)
        std::vector<double> m = hmu;
        int sd = n;
        for (int k = nl - 1; k >= 0; --k) {
            const int s = std::min(cell_size, sd / 2), nb = sd / s;
            std::vector<double> mass((size_t)nb * nb, 0.0);
            for (int i = 0; i < sd; ++i)
                for (int j = 0; j < sd; ++j) mass[(i / s) * nb + j / s] += m[(size_t)i * sd + j];
            for (int q = 0; q < nb * nb; ++q)
                if (!(mass[q] > 0)) {
                    set_err(c, "basic cell %d of layer side %d has zero mass (P:299)", q, sd);
                    return DD_EINVAL;
                }
            if (k > 0) {
                std::vector<double> cm((size_t)(sd / 2) * (sd / 2));
                for (int i = 0; i < sd / 2; ++i)
                    for (int j = 0; j < sd / 2; ++j) {
                        const size_t a = (size_t)(2 * i) * sd + 2 * j;
                        cm[(size_t)i * (sd / 2) + j] = (m[a] + m[a + 1]) + (m[a + sd] + m[a + sd + 1]);
                    }
                m.swap(cm);
                sd /= 2;
            }
        }
    }
    // ---- device layers: finest uploaded, coarser by 2x2 sum pooling (A20)
    for (int k = nl - 1; k >= 0; --k) {
        Layer& Lr = c->L[k];
        Lr.side = coarsest << k;
        Lr.s = std::min(cell_size, Lr.side / 2);
        Lr.nb = Lr.side / Lr.s;
        const size_t m2 = (size_t)Lr.side * Lr.side;
        CK(cudaMalloc(&Lr.mu, m2 * sizeof(double)));
        CK(cudaMalloc(&Lr.nu, m2 * sizeof(double)));
        CK(cudaMalloc(&Lr.logmu, m2 * sizeof(double)));
        CK(cudaMalloc(&Lr.mass, (size_t)Lr.nb * Lr.nb * sizeof(double)));
        if (k == nl - 1) {
            const cudaMemcpyKind kind = (c->opt.flags & DD_FLAG_DEVICE_INPUT) ? cudaMemcpyDeviceToDevice
                                                                              : cudaMemcpyHostToDevice;
            CK(cudaMemcpyAsync(Lr.mu, mu, m2 * sizeof(double), kind, c->st));
            CK(cudaMemcpyAsync(Lr.nu, nu, m2 * sizeof(double), kind, c->st));
        } else {
            CK(launch_pool2x2(c->L[k + 1].mu, Lr.mu, Lr.side, c->st));
            CK(launch_pool2x2(c->L[k + 1].nu, Lr.nu, Lr.side, c->st));
        }
        CK(launch_log(Lr.mu, Lr.logmu, (long long)m2, c->st));
        CK(launch_mass_i(Lr.mu, Lr.mass, Lr.side, Lr.s, Lr.nb, c->st));
    }
    // ---- state buffers (finest sizes)
    const Layer& F = c->L[nl - 1];
    const Layer& C0 = c->L[0];
    const int nbmax = F.nb;
    c->cap = c->opt.pool_capacity > 0 ? c->opt.pool_capacity : 64LL * (long long)n2 + (1LL << 22);
    c->cap = std::max(c->cap, (long long)C0.nb * C0.nb * C0.side * C0.side + 16);
    // multi-GPU: the last quarter of the pool holds two imported boundary
    // rows (a row of boxes is <= side^3 / s entries in the product state)
    c->halo_cap = (c->cap / 3) & ~7LL;   // 16-byte aligned slots
    c->cap += c->halo_cap;
    CK(cudaMalloc(&c->alphaA, n2 * sizeof(double)));
    CK(cudaMalloc(&c->alphaB, n2 * sizeof(double)));
    CK(cudaMalloc(&c->box, (size_t)nbmax * nbmax * sizeof(int4)));
    CK(cudaMalloc(&c->box2, (size_t)nbmax * nbmax * sizeof(int4)));
    CK(cudaMalloc(&c->off, (size_t)nbmax * nbmax * sizeof(long long)));
    CK(cudaMalloc(&c->off2, (size_t)nbmax * nbmax * sizeof(long long)));
    CK(cudaMalloc(&c->pool, (size_t)c->cap * sizeof(double)));
    CK(cudaMalloc(&c->scratch, (size_t)c->cap * sizeof(double)));
    CK(cudaMalloc(&c->bump, sizeof(unsigned long long)));
    c->ncell_max = (nbmax / 2 + 1) * (nbmax / 2 + 1);
    CK(cudaMalloc(&c->lists, (size_t)7 * c->ncell_max * sizeof(int)));
    CK(cudaMalloc(&c->bside, (size_t)c->ncell_max * sizeof(int)));
    CK(cudaMalloc(&c->ipred, (size_t)2 * c->ncell_max * sizeof(int)));
    CK(cudaMalloc(&c->counters, 16 * sizeof(int)));
    CK(cudaMemsetAsync(c->counters, 0, 16 * sizeof(int), c->st));
    // BIG tiers: one global slice per persistent CTA holding log nu_cell
    // (b^2 float2), the phase-A stabilisers (b^2 float) and the extraction partial sums (b^2 float4), sized for
    // the largest tier capacity over the layers (box sides never exceed the side)
    for (int k = 0; k < nl; ++k) {
        int b0, b1, b2;
        tier_caps(c->L[k].s, c->opt.reserved[0], c->opt.reserved[1], &b0, &b1, &b2);
        c->slice_cap[0] = std::max(c->slice_cap[0], std::min(b1, c->L[k].side));
        c->slice_cap[1] = std::max(c->slice_cap[1], std::min(b2, c->L[k].side));
    }
    c->grid_t[0] = kT1PerSM * prop.multiProcessorCount;
    c->grid_t[1] = kT2PerSM * prop.multiProcessorCount;
    for (int t = 0; t < 2; ++t) {
        const long long b = c->slice_cap[t];
        auto al = [](long long v) { return (v + 255) & ~255LL; };
        c->slice_bytes[t] = al(b * b * (long long)sizeof(float2)) + al(b * b * (long long)sizeof(float)) +
                            al(b * b * (long long)sizeof(float4));
        CK(cudaMalloc(&c->slices[t], (size_t)c->slice_bytes[t] * c->grid_t[t]));
    }
    for (int k = 0; k < 2; ++k) {
        CK(cudaStreamCreateWithFlags(&c->st_t[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming));
    }
    // cluster tier: reserved[3] = 0 / -1 off (default), 1 every big-path cell
    // (testing), 2 auto (the long poles); reserved[4] routing threshold theta in
    // % (default 300); reserved[5] clusters.  Off by default: measured, a
    // cluster of 8 SMs solves a long-pole cell only 1.3-1.7x faster than one
    // SM, and dd_run_schedule_batch fills the
    // SMs a latency-bound sweep leaves idle at far better efficiency.
    c->nsm = prop.multiProcessorCount;
    c->cl_mode = c->opt.reserved[3] == 1 ? 1 : 0;
    c->cl_theta = c->opt.reserved[4] > 0 ? 0.01f * (float)c->opt.reserved[4] : 3.0f;
    if ((c->opt.reserved[3] == 1 || c->opt.reserved[3] == 2) && prop.major >= 9) {
        size_t sm2 = 0;
        for (int k = 0; k < nl; ++k)
            sm2 = std::max(sm2, k1_smem_bytes_host(c->L[k].s, std::min(c->slice_cap[1], c->L[k].side), true,
                                                   kT2Threads / 32));
        const int want = c->opt.reserved[5] > 0 ? c->opt.reserved[5] : kDefaultClusters;
        c->ncl = std::min(want, k1_max_clusters(sm2));
    }
    if (c->ncl > 0) {
        CK(cudaMalloc(&c->cl_slices, (size_t)c->slice_bytes[1] * c->ncl));
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->st_cl, cudaStreamNonBlocking, hi));
        CK(cudaEventCreateWithFlags(&c->ev_join_cl, cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaMalloc(&c->cellout, (size_t)c->ncell_max * sizeof(CellOut)));
    CK(cudaMalloc(&c->d_total, 2 * sizeof(long long)));
    CK(cudaMalloc(&c->d_last, sizeof(DevStats)));
    CK(cudaMalloc(&c->d_tot, sizeof(DevStats)));
    CK(cudaMalloc(&c->d_sums, 4 * sizeof(double)));
    CK(cudaMalloc(&c->yacc, n2 * sizeof(unsigned long long)));
    CK(cudaMalloc(&c->partial, 256 * sizeof(double)));
    {   // K5 scratch for the largest coarse layer
        size_t g = 16;
        for (int k = 0; k + 1 < nl; ++k) g = std::max(g, glue_scratch_doubles(c->L[k].side, c->L[k].s));
        CK(cudaMalloc(&c->glue, g * sizeof(double)));
    }
    CK(cudaMemsetAsync(c->d_last, 0, sizeof(DevStats), c->st));
    CK(cudaMemsetAsync(c->d_tot, 0, sizeof(DevStats), c->st));
    CK(cudaMemsetAsync(c->d_total, 0, 2 * sizeof(long long), c->st));
    // DD_POISON=1 (testing): fill the state and scratch buffers with 0xFF
    // (NaN) bytes and have K1 poison its SMEM, so that a read of memory the
    // path did not write shows up as a result difference (tests/test_batch_gpu.py)
    if (getenv("DD_POISON")) {
        c->poison = 1;
        const size_t nbm = (size_t)nbmax * nbmax;
        CK(cudaMemsetAsync(c->pool, 0xFF, (size_t)c->cap * sizeof(double), c->st));
        CK(cudaMemsetAsync(c->scratch, 0xFF, (size_t)c->cap * sizeof(double), c->st));
        CK(cudaMemsetAsync(c->box, 0xFF, nbm * sizeof(int4), c->st));
        CK(cudaMemsetAsync(c->box2, 0xFF, nbm * sizeof(int4), c->st));
        CK(cudaMemsetAsync(c->off, 0xFF, nbm * sizeof(long long), c->st));
        CK(cudaMemsetAsync(c->off2, 0xFF, nbm * sizeof(long long), c->st));
        CK(cudaMemsetAsync(c->alphaA, 0xFF, n2 * sizeof(double), c->st));
        CK(cudaMemsetAsync(c->alphaB, 0xFF, n2 * sizeof(double), c->st));
        for (int t = 0; t < 2; ++t)
            CK(cudaMemsetAsync(c->slices[t], 0xFF, (size_t)c->slice_bytes[t] * c->grid_t[t], c->st));
        if (c->cl_slices) CK(cudaMemsetAsync(c->cl_slices, 0xFF, (size_t)c->slice_bytes[1] * c->ncl, c->st));
        CK(cudaMemsetAsync(c->cellout, 0xFF, (size_t)c->ncell_max * sizeof(CellOut), c->st));
        CK(cudaMemsetAsync(c->yacc, 0xFF, n2 * sizeof(unsigned long long), c->st));
    }
    // K1 needs > 48 KB dynamic SMEM on the big path: set the attribute once here
    choose_caps(c, F.s);
    c->cur = 0;
    c->eps_final = eps;
    c->eps = (c->opt.schedule == DD_SCHED_LADDER) ? 2.0 / ((double)coarsest * coarsest) : eps;
    int rc = product_init(c);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->st));
    return DD_OK;
}

int dd_reset(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    c->cur = 0;
    c->stripe_lo = c->stripe_hi = 0;
    c->eps = (c->opt.schedule == DD_SCHED_LADDER) ? 2.0 / ((double)c->L[0].side * c->L[0].side) : c->eps_final;
    return product_init(c);
}

int dd_set_cost(dd_ctx* c, int n_entries, const double* h1, const double* h2) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->st));
    if (c->d_h1) { CK(cudaFree(c->d_h1)); c->d_h1 = nullptr; }
    if (c->d_h2) { CK(cudaFree(c->d_h2)); c->d_h2 = nullptr; }
    if (!h1 && !h2) return DD_OK;
    const int n = c->L[c->n_layers - 1].side;
    if (!h1 || !h2 || n_entries != n) {
        set_err(c, "dd_set_cost: two tables of n = %d entries (finest-grid pixel differences) required", n);
        return DD_EINVAL;
    }
    for (int d = 0; d < n; ++d)
        if (!std::isfinite(h1[d]) || !std::isfinite(h2[d])) {
            set_err(c, "dd_set_cost: non-finite table entry at d = %d", d);
            return DD_EINVAL;
        }
    CK(cudaMalloc(&c->d_h1, n * sizeof(double)));
    CK(cudaMalloc(&c->d_h2, n * sizeof(double)));
    CK(cudaMemcpy(c->d_h1, h1, n * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_h2, h2, n * sizeof(double), cudaMemcpyHostToDevice));
    return DD_OK;
}

int dd_set_max_inner_iter(dd_ctx* c, int k) {
    if (!c || k < 1) return DD_EINVAL;
    c->opt.max_inner_iter = k;
    return DD_OK;
}

int dd_set_eps(dd_ctx* c, double eps) {
    if (!c || !(eps > 0.0)) return DD_EINVAL;
    c->eps = eps;   // alpha = eps log u kept constant
    return DD_OK;
}

int dd_iterate(dd_ctx* c, int k) {
    if (!c || k < 0) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    for (int i = 0; i < k; ++i) {
        int rc = sweep(c);
        if (rc) return rc;
    }
    return DD_OK;
}

int dd_refine(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    if (c->cur + 1 >= c->n_layers) { set_err(c, "already at the finest layer"); return DD_EINVAL; }
    Layer& Lc = c->L[c->cur];
    Layer& Lf = c->L[c->cur + 1];
    CK(launch_refine(c->box, c->off, c->pool, c->box2, c->off2, c->scratch, Lc.nu, Lf.nu, Lc.mass, Lf.mass,
                     Lc.nb, Lf.nb, Lc.side, Lf.side, c->cap - c->halo_cap, c->counters + 6, c->d_total,
                     c->d_total + 1, c->st));
    std::swap(c->box, c->box2);
    std::swap(c->off, c->off2);
    std::swap(c->pool, c->scratch);
    const size_t n2 = (size_t)Lf.side * Lf.side;
    const bool striped = c->stripe_hi > c->stripe_lo;   // another rank owns part of alpha
    if (c->opt.reserved[2] == 0 && !striped && c->last_part != 0) {
        // glue the coarse potentials (Helmholtz least squares,
        // P:1425-1452) and interpolate them in log space onto the fine layer
        CK(launch_glue_refine(c->alphaA, c->alphaB, Lc.mu, Lc.side, Lc.s, c->eps, c->glue, c->alphaA, c->alphaB,
                              c->st));
        c->launches_pending += 4;
    } else {
        CK(cudaMemsetAsync(c->alphaA, 0, n2 * sizeof(double), c->st));   // cold start (reading A14)
        CK(cudaMemsetAsync(c->alphaB, 0, n2 * sizeof(double), c->st));
    }
    c->launches_pending += 3;
    c->cur += 1;
    c->stripe_lo = c->stripe_hi = 0;     // the driver sets the fine layer's stripe
    c->last_part = 0;
    return DD_OK;
}

int dd_run_schedule(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    if (c->opt.schedule != DD_SCHED_LADDER) { set_err(c, "dd_run_schedule needs DD_SCHED_LADDER"); return DD_EINVAL; }
    const int nf = c->L[c->n_layers - 1].side;
    const double kf = c->eps_final * (double)nf * nf;
    int sides[256], sweeps[256];
    double kap[256];
    const int ns = std::min(256, build_schedule(nf, c->L[0].side, kf, c->opt.eps_start, sides, kap, sweeps, 256));
    for (int k = 0; k < ns; ++k) {
        while (c->L[c->cur].side < sides[k]) {
            int rc = dd_refine(c);
            if (rc) return rc;
        }
        const double h = 1.0 / sides[k];
        dd_set_eps(c, kap[k] * h * h);
        int rc = dd_iterate(c, sweeps[k]);
        if (rc) return rc;
    }
    // one wait at the end of the schedule: DD_ENOCONV if any cell hit max_inner_iter
    return dd_synchronize(c);
}

int dd_run_schedule_batch(dd_ctx* const* cs, int n) {
    if (!cs || n <= 0) return DD_EINVAL;
    dd_ctx* c = cs[0];
    if (!c) return DD_EINVAL;
    for (int i = 0; i < n; ++i) {
        dd_ctx* q = cs[i];
        if (!q || q->opt.schedule != DD_SCHED_LADDER || q->device != c->device || q->n_layers != c->n_layers ||
            q->L[q->n_layers - 1].side != c->L[c->n_layers - 1].side || q->cell_size != c->cell_size ||
            q->L[0].side != c->L[0].side || q->eps_final != c->eps_final || q->opt.eps_start != c->opt.eps_start) {
            set_err(c, "dd_run_schedule_batch: context %d differs (ladder, device, grid, cell size, eps)", i);
            return DD_EINVAL;
        }
        for (int j = 0; j < i; ++j)
            if (cs[j] == q || cs[j]->st == q->st) {
                set_err(c, "dd_run_schedule_batch: contexts %d and %d share a stream", j, i);
                return DD_EINVAL;
            }
    }
    CK(cudaSetDevice(c->device));
    // fork: every context's stream waits for the work already queued on ctxs[0]'s
    if (!c->ev_batch) CK(cudaEventCreateWithFlags(&c->ev_batch, cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_batch, c->st));
    for (int i = 1; i < n; ++i) CK(cudaStreamWaitEvent(cs[i]->st, c->ev_batch, 0));
    const int nf = c->L[c->n_layers - 1].side;
    const double kf = c->eps_final * (double)nf * nf;
    int sides[256], sweeps[256];
    double kap[256];
    const int ns = std::min(256, build_schedule(nf, c->L[0].side, kf, c->opt.eps_start, sides, kap, sweeps, 256));
    for (int k = 0; k < ns; ++k) {
        for (int i = 0; i < n; ++i) {
            dd_ctx* q = cs[i];
            while (q->L[q->cur].side < sides[k]) {
                int rc = dd_refine(q);
                if (rc) return rc;
            }
            const double h = 1.0 / sides[k];
            dd_set_eps(q, kap[k] * h * h);
        }
        for (int j = 0; j < sweeps[k]; ++j)
            for (int i = 0; i < n; ++i) {
                int rc = sweep(cs[i]);
                if (rc) return rc;
            }
    }
    // join: ctxs[0]'s stream waits for every context's last sweep
    for (int i = 1; i < n; ++i) {
        dd_ctx* q = cs[i];
        if (!q->ev_batch) CK(cudaEventCreateWithFlags(&q->ev_batch, cudaEventDisableTiming));
        CK(cudaEventRecord(q->ev_batch, q->st));
        CK(cudaStreamWaitEvent(c->st, q->ev_batch, 0));
    }
    int first = DD_OK;
    for (int i = 0; i < n; ++i) {
        const int rc = dd_synchronize(cs[i]);
        if (rc && !first) first = rc;
    }
    return first;
}

int dd_synchronize(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    // A6: cells that hit max_inner_iter since the last report (the sweeps
    // themselves never wait on the host)
    DevStats d;
    CK(cudaMemcpy(&d, c->d_tot, sizeof(DevStats), cudaMemcpyDeviceToHost));
    if (d.failed > c->failed_seen) {
        set_err(c, "%lld cells did not converge within max_inner_iter = %d (state stays Y-feasible)",
                (long long)d.failed - c->failed_seen, c->opt.max_inner_iter);
        c->failed_seen = d.failed;
        return DD_ENOCONV;
    }
    return DD_OK;
}

int dd_get_stats(dd_ctx* c, dd_sweep_stats* s) {
    if (!c || !s) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    DevStats d;
    CK(cudaMemcpy(&d, c->d_last, sizeof(DevStats), cudaMemcpyDeviceToHost));
    memset(s, 0, sizeof(*s));
    fill_stats(d, s);
    s->ms = c->ms_last;
    s->solve_ms = c->solve_ms_last;
    s->launches = 8;
    if (d.failed) {
        set_err(c, "%d cells did not converge within max_inner_iter", d.failed);
        return DD_ENOCONV;
    }
    return DD_OK;
}

int dd_get_totals(dd_ctx* c, dd_sweep_stats* s) {
    if (!c || !s) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    DevStats d;
    CK(cudaMemcpy(&d, c->d_tot, sizeof(DevStats), cudaMemcpyDeviceToHost));
    memset(s, 0, sizeof(*s));
    fill_stats(d, s);
    s->ms = c->ms_tot;
    s->solve_ms = c->solve_ms_tot;
    s->launches = c->launches_tot;
    return DD_OK;
}

int dd_set_stripe(dd_ctx* c, int row_lo, int row_hi) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row_lo == 0 && row_hi == 0) { c->stripe_lo = c->stripe_hi = 0; return DD_OK; }
    if (row_lo < 0 || row_hi > Lr.nb || row_lo >= row_hi || (row_lo & 1) || (row_hi & 1)) {
        set_err(c, "stripe [%d, %d) must be even basic-row bounds inside [0, %d)", row_lo, row_hi, Lr.nb);
        return DD_EINVAL;
    }
    c->stripe_lo = row_lo;
    c->stripe_hi = row_hi;
    // rows outside the stripe become empty (another rank owns them)
    if (row_lo > 0) CK(cudaMemsetAsync(c->box, 0, (size_t)row_lo * Lr.nb * sizeof(int4), c->st));
    if (row_hi < Lr.nb)
        CK(cudaMemsetAsync(c->box + (size_t)row_hi * Lr.nb, 0, (size_t)(Lr.nb - row_hi) * Lr.nb * sizeof(int4), c->st));
    return DD_OK;
}

int dd_clear_rows(dd_ctx* c, int row, int nrows) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row < 0 || nrows < 0 || row + nrows > Lr.nb) { set_err(c, "rows out of range"); return DD_EINVAL; }
    if (nrows) CK(cudaMemsetAsync(c->box + (size_t)row * Lr.nb, 0, (size_t)nrows * Lr.nb * sizeof(int4), c->st));
    return DD_OK;
}

namespace {
int ensure_xoff(dd_ctx* c, long long n) {
    if (n <= c->xoff_n) return DD_OK;
    if (c->d_xoff) cudaFree(c->d_xoff);
    c->d_xoff = nullptr;
    CK(cudaMalloc(&c->d_xoff, (size_t)n * sizeof(long long)));
    c->xoff_n = n;
    return DD_OK;
}
long long pad2(long long a) { return (a + 1) & ~1LL; }
}  // namespace

int dd_export_rows(dd_ctx* c, int row, int nrows, void* buf, size_t* bytes) {
    if (!c || !bytes) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row < 0 || nrows <= 0 || row + nrows > Lr.nb) { set_err(c, "rows out of range"); return DD_EINVAL; }
    int rc = sync_state(c);
    if (rc) return rc;
    const int n = nrows * Lr.nb;
    std::vector<int4> hb(n);
    CK(cudaMemcpy(hb.data(), c->box + (size_t)row * Lr.nb, n * sizeof(int4), cudaMemcpyDeviceToHost));
    std::vector<long long> pre(n);
    long long tot = 0;
    for (int i = 0; i < n; ++i) { pre[i] = tot; tot += pad2((long long)hb[i].z * hb[i].w); }
    const size_t need = (size_t)n * sizeof(int4) + 16 + (size_t)tot * sizeof(double);
    if (!buf) { *bytes = need; return DD_OK; }
    if (*bytes < need) { set_err(c, "export buffer too small (%zu < %zu)", *bytes, need); return DD_EINVAL; }
    char* b = (char*)buf;
    const long long hdr[2] = {tot, n};
    rc = ensure_xoff(c, n);
    if (rc) return rc;
    CK(cudaMemcpyAsync(b, c->box + (size_t)row * Lr.nb, n * sizeof(int4), cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(b + (size_t)n * sizeof(int4), hdr, sizeof(hdr), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->d_xoff, pre.data(), n * sizeof(long long), cudaMemcpyHostToDevice, c->st));
    CK(launch_copy_boxes(c->box + (size_t)row * Lr.nb, c->off + (size_t)row * Lr.nb, c->d_xoff, c->pool,
                         (double*)(b + (size_t)n * sizeof(int4) + 16), n, tot, c->st));
    CK(cudaStreamSynchronize(c->st));
    *bytes = need;
    return DD_OK;
}

int dd_import_rows(dd_ctx* c, int row, int nrows, const void* buf, size_t bytes) {
    if (!c || !buf) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row < 0 || nrows <= 0 || row + nrows > Lr.nb) { set_err(c, "rows out of range"); return DD_EINVAL; }
    int rc = sync_state(c);
    if (rc) return rc;
    const int n = nrows * Lr.nb;
    const char* b = (const char*)buf;
    if (bytes < (size_t)n * sizeof(int4) + 16) { set_err(c, "import buffer too small"); return DD_EINVAL; }
    std::vector<int4> hb(n);
    long long hdr[2];
    CK(cudaMemcpy(hb.data(), b, n * sizeof(int4), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hdr, b + (size_t)n * sizeof(int4), sizeof(hdr), cudaMemcpyDeviceToHost));
    std::vector<long long> pre(2 * (size_t)n);
    long long tot = 0;
    for (int i = 0; i < n; ++i) {
        if (hb[i].z < 0 || hb[i].w < 0 || hb[i].x < 0 || hb[i].y < 0 || hb[i].x + hb[i].z > Lr.side ||
            hb[i].y + hb[i].w > Lr.side) { set_err(c, "imported box %d out of range", i); return DD_EINVAL; }
        pre[i] = tot;
        tot += pad2((long long)hb[i].z * hb[i].w);
    }
    if (hdr[0] != tot || hdr[1] != n || bytes < (size_t)n * sizeof(int4) + 16 + (size_t)tot * sizeof(double)) {
        set_err(c, "import header mismatch");
        return DD_EINVAL;
    }
    // two halo slots: rows above the stripe (the B-cells' upper row) and the
    // stripe's own rows returned by the rank below (both may be live at once)
    const long long slot = c->halo_cap / 2;
    if (tot > slot) { set_err(c, "imported rows (%lld entries) exceed the halo slot %lld", tot, slot); return DD_ENOMEM; }
    const long long hbase = c->cap - c->halo_cap + ((row < c->stripe_lo) ? 0 : slot);
    for (int i = 0; i < n; ++i) pre[n + i] = hbase + pre[i];
    rc = ensure_xoff(c, 2LL * n);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->box + (size_t)row * Lr.nb, b, n * sizeof(int4), cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->d_xoff, pre.data(), 2 * (size_t)n * sizeof(long long), cudaMemcpyHostToDevice, c->st));
    CK(launch_copy_boxes(c->box + (size_t)row * Lr.nb, c->d_xoff, c->d_xoff + n,
                         (const double*)(b + (size_t)n * sizeof(int4) + 16), c->pool, n, c->cap, c->st));
    CK(cudaMemcpyAsync(c->off + (size_t)row * Lr.nb, c->d_xoff + n, n * sizeof(long long), cudaMemcpyDeviceToDevice,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    return DD_OK;
}

int dd_compact(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    const int nb2 = Lr.nb * Lr.nb;
    // K2 over the current pool: new basic-cell-order offsets, pool -> scratch, swap
    CK(launch_scan_areas(c->box, c->off2, c->d_total, nb2, c->d_total + 1, c->st));
    CK(launch_copy_boxes(c->box, c->off, c->off2, c->pool, c->scratch, nb2, c->cap - c->halo_cap, c->st));
    std::swap(c->off, c->off2);
    std::swap(c->pool, c->scratch);
    return DD_OK;
}

int dd_export_rows_slab(dd_ctx* c, int row, int nrows, void* slab, size_t slab_bytes) {
    if (!c || !slab) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row < 0 || nrows <= 0 || row + nrows > Lr.nb) { set_err(c, "rows out of range"); return DD_EINVAL; }
    const int n = nrows * Lr.nb;
    if (slab_bytes < (size_t)(64 + 16LL * n + 16)) { set_err(c, "slab smaller than its header"); return DD_EINVAL; }
    int rc = ensure_xoff(c, 2LL * n);
    if (rc) return rc;
    CK(launch_slab_export(c->box + (size_t)row * Lr.nb, c->off + (size_t)row * Lr.nb, c->pool, n, slab,
                          (long long)slab_bytes, c->d_xoff, c->counters + 6, c->st));
    return DD_OK;
}

int dd_import_rows_slab(dd_ctx* c, int row, int nrows, const void* slab, size_t slab_bytes) {
    if (!c || !slab) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row < 0 || nrows <= 0 || row + nrows > Lr.nb) { set_err(c, "rows out of range"); return DD_EINVAL; }
    const int n = nrows * Lr.nb;
    if (slab_bytes < (size_t)(64 + 16LL * n + 16)) { set_err(c, "slab smaller than its header"); return DD_EINVAL; }
    int rc = ensure_xoff(c, 2LL * n);
    if (rc) return rc;
    // the same two halo slots as dd_import_rows (rows above the stripe | the
    // stripe's own rows returned by the rank below)
    const long long slot = c->halo_cap / 2;
    const long long hbase = c->cap - c->halo_cap + ((row < c->stripe_lo) ? 0 : slot);
    CK(launch_slab_import(slab, n, Lr.side, hbase, slot, c->box + (size_t)row * Lr.nb, c->off + (size_t)row * Lr.nb,
                          c->pool, c->cap, c->d_xoff, c->counters + 6, c->st));
    return DD_OK;
}

int dd_copy_alpha(dd_ctx* c, int partition, int row0, int nrows, void* buf, int to_ctx) {
    if (!c || !buf || (partition != 1 && partition != 2)) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    if (row0 < 0 || nrows < 0 || row0 + nrows > Lr.side) { set_err(c, "alpha rows out of range"); return DD_EINVAL; }
    double* a = (partition == 1 ? c->alphaA : c->alphaB) + (size_t)row0 * Lr.side;
    const size_t bytes = (size_t)nrows * Lr.side * sizeof(double);
    if (to_ctx) CK(cudaMemcpyAsync(a, buf, bytes, cudaMemcpyDeviceToDevice, c->st));
    else CK(cudaMemcpyAsync(buf, a, bytes, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    return DD_OK;
}

int dd_y_accumulate(dd_ctx* c, unsigned long long* acc) {
    if (!c || !acc) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    CK(launch_scatter_y(c->box, c->off, c->pool, Lr.nb, acc, Lr.side, c->st));
    CK(cudaStreamSynchronize(c->st));
    return DD_OK;
}

int dd_y_l1(dd_ctx* c, const unsigned long long* acc, double* l1_y) {
    if (!c || !acc || !l1_y) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    const Layer& Lr = c->L[c->cur];
    CK(launch_l1y(acc, Lr.nu, Lr.side, c->partial, c->d_sums + 3, c->st));
    CK(cudaMemcpyAsync(l1_y, c->d_sums + 3, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return DD_OK;
}

int dd_phase_profile(dd_ctx* c, unsigned long long* out32) {
    if (!c || !out32) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = harvest(c);
    if (rc) return rc;
    CK(k1_phase_read(out32));
    return DD_OK;
}

int dd_get_cell_stats(dd_ctx* c, int* iters, int* box_side, double* mufu_ops, int* kcycles, int* flags,
                      float* err_x, int max_cells) {
    if (!c || max_cells < 0) return -DD_EINVAL;
    if (cudaSetDevice(c->device) != cudaSuccess) return -DD_ECUDA;
    int rc = harvest(c);
    if (rc) return -rc;
    const Layer& Lr = c->L[c->cur];
    const int part = c->last_part ? c->last_part : 1;
    const int nca = cells_axis(Lr.nb, part);
    const int ncells = c->last_part ? nca * nca : 0;
    const int m = std::min(ncells, max_cells);
    if (m > 0) {
        std::vector<CellOut> h(m);
        if (cudaMemcpy(h.data(), c->cellout, m * sizeof(CellOut), cudaMemcpyDeviceToHost) != cudaSuccess) {
            set_err(c, "dd_get_cell_stats: copy failed");
            return -DD_ECUDA;
        }
        for (int k = 0; k < m; ++k) {
            if (iters) iters[k] = h[k].iters;
            if (box_side) box_side[k] = h[k].box;
            if (mufu_ops) mufu_ops[k] = h[k].mufu;
            if (kcycles) kcycles[k] = h[k].pad;
            if (flags) flags[k] = h[k].flags;
            if (err_x) err_x[k] = h[k].err;
        }
    }
    return ncells;
}

int dd_reset_totals(dd_ctx* c) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = harvest(c);
    if (rc) return rc;
    CK(cudaMemsetAsync(c->d_tot, 0, sizeof(DevStats), c->st));
    CK(cudaStreamSynchronize(c->st));
    c->ms_tot = c->solve_ms_tot = 0;
    c->launches_tot = 0;
    c->failed_seen = 0;
    return DD_OK;
}

int dd_primal_cost(dd_ctx* c, double* transport_cost, double* entropic) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    double s[3];
    rc = evaluate(c, s, false, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    if (transport_cost) *transport_cost = s[0];
    if (entropic) *entropic = s[1];
    return DD_OK;
}

int dd_dual_gap(dd_ctx* c, double* primal, double* dual, double* rel_gap) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    if (c->stripe_hi > c->stripe_lo) { set_err(c, "dd_dual_gap needs the whole layer (no stripe)"); return DD_EINVAL; }
    double s3[3];
    rc = evaluate(c, s3, false, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    Layer& Lr = c->L[c->cur];
    const double P = s3[1] / c->eps;                     // KL(pi|K) - ||K|| (A15)
    // glue at the current layer (k_glue.cu, default stream), then the dense
    // Y-iteration against u_hat and the dual terms
    CK(cudaStreamSynchronize(c->st));
    const size_t gneed = glue_scratch_doubles(Lr.side, Lr.s);
    double* g = nullptr;
    CK(cudaMalloc(&g, gneed * sizeof(double)));
    double* phi = nullptr;
    CK(launch_glue_phi(c->alphaA, c->alphaB, Lr.mu, Lr.side, Lr.s, c->eps, g, &phi));
    CK(cudaDeviceSynchronize());
    const size_t n2 = (size_t)Lr.side * Lr.side;
    double* T = nullptr;
    CK(cudaMalloc(&T, 2 * n2 * sizeof(double)));
    const double kappa = c->eps * (double)Lr.side * Lr.side;
    CK(launch_dual_terms(phi, Lr.mu, Lr.logmu, Lr.nu, Lr.side, c->eps, kappa, T, T + n2, c->st,
                         c->d_h1, c->d_h2, c->L[c->n_layers - 1].side / Lr.side));
    // fixed-order sum of the n^2 terms
    std::vector<double> h(n2);
    CK(cudaMemcpyAsync(h.data(), T + n2, n2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    cudaFree(T);
    cudaFree(g);
    double D = 0.0, comp = 0.0;                              // Neumaier, host (n^2 doubles, once)
    for (size_t k = 0; k < n2; ++k) {
        const double t = D + h[k];
        comp += (std::fabs(D) >= std::fabs(h[k])) ? (D - t) + h[k] : (h[k] - t) + D;
        D = t;
    }
    D += comp;
    if (primal) *primal = P;
    if (dual) *dual = D;
    if (rel_gap) *rel_gap = (P - D) / P;
    return DD_OK;
}

int dd_marginal_error(dd_ctx* c, double* l1_x, double* l1_y) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    double s[3];
    rc = evaluate(c, s, false, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    Layer& Lr = c->L[c->cur];
    CK(launch_scatter_l1y(c->box, c->off, c->pool, Lr.nb, c->yacc, Lr.nu, Lr.side, c->partial, c->d_sums + 3, c->st));
    double ly = 0;
    CK(cudaMemcpyAsync(&ly, c->d_sums + 3, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (l1_x) *l1_x = s[2];
    if (l1_y) *l1_y = ly;
    return DD_OK;
}

int dd_get_state_info(dd_ctx* c, dd_state_info* info) {
    if (!c || !info) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    Layer& Lr = c->L[c->cur];
    info->side = Lr.side;
    info->s = Lr.s;
    info->nb = Lr.nb;
    info->last_partition = c->last_part;
    info->half_index = c->half_index;
    info->eps = c->eps;
    std::vector<int4> hb((size_t)Lr.nb * Lr.nb);
    CK(cudaMemcpy(hb.data(), c->box, hb.size() * sizeof(int4), cudaMemcpyDeviceToHost));
    long long e = 0;
    for (auto& b : hb) e += (long long)b.z * b.w;
    info->entries = e;
    return DD_OK;
}

int dd_get_state(dd_ctx* c, int* boxes, long long* offsets, double* values, double* alpha_A, double* alpha_B) {
    if (!c) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    Layer& Lr = c->L[c->cur];
    const int nb2 = Lr.nb * Lr.nb;
    std::vector<int4> hb(nb2);
    std::vector<long long> ho(nb2);
    CK(cudaMemcpy(hb.data(), c->box, nb2 * sizeof(int4), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho.data(), c->off, nb2 * sizeof(long long), cudaMemcpyDeviceToHost));
    long long o = 0;
    for (int i = 0; i < nb2; ++i) {
        const long long a = (long long)hb[i].z * hb[i].w;
        if (boxes) { boxes[4 * i] = hb[i].x; boxes[4 * i + 1] = hb[i].y; boxes[4 * i + 2] = hb[i].z; boxes[4 * i + 3] = hb[i].w; }
        if (offsets) offsets[i] = o;
        if (values && a) CK(cudaMemcpy(values + o, c->pool + ho[i], a * sizeof(double), cudaMemcpyDeviceToHost));
        o += a;
    }
    const size_t n2 = (size_t)Lr.side * Lr.side;
    if (alpha_A) CK(cudaMemcpy(alpha_A, c->alphaA, n2 * sizeof(double), cudaMemcpyDeviceToHost));
    if (alpha_B) CK(cudaMemcpy(alpha_B, c->alphaB, n2 * sizeof(double), cudaMemcpyDeviceToHost));
    return DD_OK;
}

int dd_set_state(dd_ctx* c, int side, long long half_index, int last_partition, const int* boxes,
                 const long long* offsets, const double* values, long long n_values, const double* alpha_A,
                 const double* alpha_B) {
    if (!c || !boxes || !offsets || !values) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int k = 0;
    while (k < c->n_layers && c->L[k].side != side) ++k;
    if (k == c->n_layers) { set_err(c, "no layer of side %d", side); return DD_EINVAL; }
    int rc = harvest(c);
    if (rc) return rc;
    Layer& Lr = c->L[k];
    const int nb2 = Lr.nb * Lr.nb;
    std::vector<int4> hb(nb2);
    std::vector<long long> ho(nb2);
    long long o = 0;
    for (int i = 0; i < nb2; ++i) {
        hb[i] = make_int4(boxes[4 * i], boxes[4 * i + 1], boxes[4 * i + 2], boxes[4 * i + 3]);
        if (hb[i].z < 0 || hb[i].w < 0 || hb[i].x < 0 || hb[i].y < 0 || hb[i].x + hb[i].z > side ||
            hb[i].y + hb[i].w > side) {
            set_err(c, "box %d out of range", i);
            return DD_EINVAL;
        }
        const long long a = (long long)hb[i].z * hb[i].w;
        if (offsets[i] < 0 || offsets[i] + a > n_values) { set_err(c, "offset %d out of range", i); return DD_EINVAL; }
        ho[i] = o;
        o += (a + 1) & ~1LL;
    }
    if (o > c->cap - c->halo_cap) { set_err(c, "state larger than the pool capacity"); return DD_ENOMEM; }
    std::vector<double> pool(std::max(1LL, o), 0.0);
    for (int i = 0; i < nb2; ++i) {
        const long long a = (long long)hb[i].z * hb[i].w;
        if (a) memcpy(pool.data() + ho[i], values + offsets[i], a * sizeof(double));
    }
    CK(cudaMemcpy(c->box, hb.data(), nb2 * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->off, ho.data(), nb2 * sizeof(long long), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->pool, pool.data(), pool.size() * sizeof(double), cudaMemcpyHostToDevice));
    const size_t n2 = (size_t)side * side;
    if (alpha_A) CK(cudaMemcpy(c->alphaA, alpha_A, n2 * sizeof(double), cudaMemcpyHostToDevice));
    else CK(cudaMemset(c->alphaA, 0, n2 * sizeof(double)));
    if (alpha_B) CK(cudaMemcpy(c->alphaB, alpha_B, n2 * sizeof(double), cudaMemcpyHostToDevice));
    else CK(cudaMemset(c->alphaB, 0, n2 * sizeof(double)));
    c->cur = k;
    c->half_index = half_index;
    c->last_part = last_partition;
    return DD_OK;
}

int dd_fetch_plan(dd_ctx* c, int format, void* buf, size_t* bytes) {
    if (!c || !bytes) return DD_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = sync_state(c);
    if (rc) return rc;
    Layer& Lr = c->L[c->cur];
    if (format == DD_PLAN_BASIC_MARGINALS) {
        dd_state_info info;
        rc = dd_get_state_info(c, &info);
        if (rc) return rc;
        const int nb2 = Lr.nb * Lr.nb;
        const size_t need = (size_t)nb2 * 4 * sizeof(int) + (size_t)nb2 * sizeof(long long) +
                            (size_t)info.entries * sizeof(double);
        if (!buf) { *bytes = need; return DD_OK; }
        if (*bytes < need) { set_err(c, "buffer too small (%zu < %zu)", *bytes, need); return DD_EINVAL; }
        char* p = (char*)buf;
        int* bx = (int*)p;
        long long* of = (long long*)(p + (size_t)nb2 * 4 * sizeof(int));
        double* v = (double*)(p + (size_t)nb2 * 4 * sizeof(int) + (size_t)nb2 * sizeof(long long));
        rc = dd_get_state(c, bx, of, v, nullptr, nullptr);
        *bytes = need;
        return rc;
    }
    if (format == DD_PLAN_COO) {
        long long cnt = 0;
        double s3[3];
        rc = evaluate(c, s3, true, &cnt, nullptr, nullptr, nullptr);
        if (rc) return rc;
        const size_t need = (size_t)cnt * (2 * sizeof(int) + sizeof(double));
        if (!buf) { *bytes = need; return DD_OK; }
        if (*bytes < need) { set_err(c, "buffer too small"); return DD_EINVAL; }
        char* p = (char*)buf;
        int* xs = (int*)p;
        int* ys = (int*)(p + cnt * sizeof(int));
        double* ms = (double*)(p + 2 * cnt * sizeof(int));
        rc = evaluate(c, s3, true, &cnt, xs, ys, ms);
        *bytes = need;
        return rc;
    }
    set_err(c, "unknown plan format %d", format);
    return DD_EINVAL;
}

int dd_measure_mufu_peak(int device, double* ops_per_s) {
    if (!ops_per_s) return DD_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return DD_ECUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DD_ECUDA;
    float* out = nullptr;
    if (cudaMalloc(&out, 65536 * sizeof(float)) != cudaSuccess) return DD_ECUDA;
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a, st);
        launch_mufu_bench(out, blocks, threads, iters, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * iters * 8.0;
        if (rep > 0) best = std::max(best, ops / (ms * 1e-3));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    cudaFree(out);
    *ops_per_s = best;
    return cudaGetLastError() == cudaSuccess ? DD_OK : DD_ECUDA;
}

void dd_free(dd_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->st) cudaStreamSynchronize(c->st);
    free_all(c);
    delete c;
}

}  // extern "C"
