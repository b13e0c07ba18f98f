// dd_aux.cuh -- host-visible declarations of the B200 path's kernels.
#pragma once
#include "dd_common.cuh"

namespace dd {

struct DevStats {
    long long cells, iters_sum;
    int iters_max, failed;
    double err_sum, mufu;
    long long fallbacks, deferred, huge;
    int max_box, overflow;
    long long entries;
    long long cluster;     // cells solved by the cluster tier
};

struct EvalParams {
    int part, side, s, nb, nca;
    int cr0, cr1;               // cell rows evaluated (multi-GPU stripe)
    double eps;
    const int4* box;
    const long long* off;
    const double* pool;
    const double* alpha;
    const double* mu;
    const double* logmu;
    const double* nu;
    double* scratch;            // per cell: nu_cell[ny], g[ny], f[nx] at scratch_off[cell]
    const long long* scratch_off;
    double* cell_res;           // 3 per cell
    int coo;
    const long long* coo_off;
    int* coo_x;
    int* coo_y;
    double* coo_m;
    const double* h1;           // general separable cost tables (nullptr: |x-y|^2), SweepParams::h1
    const double* h2;
    int hst;
};

// Ground cost between layer pixels (r1, c1) and (r2, c2), [0,1]^2 units.
__device__ __forceinline__ double ground_cost(const double* h1, const double* h2, int hst, int side,
                                              int r1, int c1, int r2, int c2) {
    if (h1) return h1[(long long)abs(r1 - r2) * hst] + h2[(long long)abs(c1 - c2) * hst];
    const double h = 1.0 / side;
    const double d1 = (r1 - r2) * h, d2 = (c1 - c2) * h;
    return d1 * d1 + d2 * d2;
}

cudaError_t k1_phase_read(unsigned long long* out32);
size_t k1_smem_bytes_host(int s, int bcap, bool big = false, int nwarps = 0, bool gc = false);
cudaError_t launch_k1(const SweepParams& p, int tier, int grid, size_t smem, cudaStream_t st);
int k1_max_clusters(size_t smem);
cudaError_t launch_k0_cluster(const int* sorted, int* counts, int ncap, const int* bside, float theta, int nsm,
                              int mode, int* list3, cudaStream_t st);
cudaError_t launch_k0(const SweepParams& p, int b0, int b1, int b2, int* lists, int* counts, int ncap, int* bside,
                      int* sorted, cudaStream_t st);
cudaError_t launch_slab_export(const int4* box, const long long* off, const double* pool, int n, void* slab,
                               long long cap_bytes, long long* scratch, int* flag, cudaStream_t st);
cudaError_t launch_slab_import(const void* slab, int n, int side, long long hbase, long long slot, int4* box,
                               long long* off, double* pool, long long pool_cap, long long* scratch, int* flag,
                               cudaStream_t st);
cudaError_t launch_pool2x2(const double* fine, double* coarse, int sc, cudaStream_t st);
cudaError_t launch_log(const double* x, double* lx, long long n, cudaStream_t st);
cudaError_t launch_mass_i(const double* mu, double* mass, int side, int s, int nb, cudaStream_t st);
cudaError_t launch_product_init(int4* box, long long* off, double* pool, const double* mass, const double* nu,
                                int side, int nb, cudaStream_t st);
cudaError_t launch_scan_areas(const int4* box, long long* newoff, long long* total, int n, long long* entries,
                              cudaStream_t st);
cudaError_t launch_copy_boxes(const int4* box, const long long* srcoff, const long long* dstoff, const double* src,
                              double* dst, int n, long long cap, cudaStream_t st);
cudaError_t launch_reduce_stats(const CellOut* out, int ncells, DevStats* last, DevStats* tot,
                                const long long* entries, const int* n_deferred, const int* overflow,
                                const int* n_huge, cudaStream_t st);
cudaError_t launch_refine(const int4* cbox, const long long* coff, const double* cpool, int4* fbox,
                          long long* foff, double* fpool, const double* cnu, const double* fnu,
                          const double* cmass, const double* fmass, int nbc, int nbf, int sidec, int sidef,
                          long long cap, int* overflow, long long* total, long long* entries, cudaStream_t st);
cudaError_t launch_scatter_l1y(const int4* box, const long long* off, const double* pool, int nb,
                               unsigned long long* acc, const double* nu, int side, double* partial,
                               double* out, cudaStream_t st);
cudaError_t launch_eval(const EvalParams& p, int ncells, double* sums, cudaStream_t st);
cudaError_t launch_scatter_y(const int4* box, const long long* off, const double* pool, int nb,
                             unsigned long long* acc, int side, cudaStream_t st);
cudaError_t launch_l1y(const unsigned long long* acc, const double* nu, int side, double* partial, double* out,
                       cudaStream_t st);
cudaError_t launch_glue_refine(const double* aA_c, const double* aB_c, const double* mu_c, int side_c, int s_c,
                               double eps, double* scratch, double* aA_f, double* aB_f, cudaStream_t st);
size_t glue_scratch_doubles(int side_c, int s_c);
cudaError_t launch_glue_phi(const double* aA, const double* aB, const double* mu, int side, int s, double eps,
                            double* scratch, double** phi_out);
cudaError_t launch_dual_terms(const double* phi, const double* mu, const double* logmu, const double* nu, int n,
                              double eps, double kappa, double* T, double* term, cudaStream_t st,
                              const double* h1 = nullptr, const double* h2 = nullptr, int hst = 1);
cudaError_t launch_mufu_bench(float* out, int blocks, int threads, int iters, cudaStream_t st);

}  // namespace dd
