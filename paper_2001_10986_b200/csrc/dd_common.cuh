// dd_common.cuh -- device-side types and helpers of the B200 entropic domain
// decomposition path (arXiv 2001.10986).  Product code: shares nothing with
// oracle/.  See DESIGN.md for the numerics (hi/lo split potentials, local
// affine gauge, speculative stabilisers).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dd {

// K1 tier 1 (fused big-cell path): threads per CTA and resident CTAs per SM
#ifndef DD_T1_NT
#define DD_T1_NT 256
#endif
#ifndef DD_T1_MINB
#define DD_T1_MINB 3
#endif
constexpr int kT1Threads = DD_T1_NT, kT1PerSM = DD_T1_MINB;
// K1 tier 2 (the largest boxes, 1 CTA/SM): threads per CTA
#ifndef DD_T2_NT
#define DD_T2_NT 768
#endif
#ifndef DD_T2_MINB
#define DD_T2_MINB 1
#endif
constexpr int kT2Threads = DD_T2_NT, kT2PerSM = DD_T2_MINB;
// K1 cluster tier (tier 3): tier 2's CTA shape, kClusterSize CTAs (SMs) per cell
#ifndef DD_CLUSTER
#define DD_CLUSTER 8
#endif
constexpr int kClusterSize = DD_CLUSTER;


// ------------------------------------------------------------ constants --
constexpr float kL2E = 1.4426950408889634f;   // log2(e)
constexpr float kLN2 = 0.6931471805599453f;
// hi parts of potentials live on the grid 2^-8: sums
// and differences of on-grid values of magnitude < 2^15 are exact in fp32.
constexpr float kGridMagic = 49152.0f;        // 1.5 * 2^15: (v + M) - M rounds v to 2^-8
constexpr int kThreads = 256;                 // K1 block size

// ------------------------------------------------------------- structs --
// Per composite cell result of one solve (K1 -> K3).
struct CellOut {
    int iters;        // Sinkhorn iterations (Y+X pairs)
    int flags;        // bit0 no-convergence, bit1 non-finite, bit2 deferred, bit3 overflow
    float err;        // L1 X-error of the returned plan
    int box;          // max(b_r, b_c) of the union Y box
    double mufu;      // MUFU ops executed (ex2 + lg2/rcp), without fallbacks
    int fallbacks;    // outputs recomputed with an exact max (speculative miss)
    int pad;          // solve time of the cell in units of 1024 SM cycles (diagnostic)
};

struct SweepParams {
    int part;             // 1 = A, 2 = B
    int side, s, nb, nca; // layer side, basic cell side, basic cells/axis, cells/axis of part
    int ncells;
    int cr0, cr1;         // cell rows of the partition this context solves (multi-GPU stripe)
    double eps;           // [0,1]^2 units
    double kappa;         // eps / h^2 (squared pixels)
    double tau;           // truncation threshold
    double err_tol;       // Err
    int max_iter;
    int check_every;     // stop test cadence (A5): tested when it % check_every == 0
    int bcap;             // max Y-box side this launch handles
    int mode;             // 0: one CTA per cell; 1: work list in SMEM; 2: work list in global scratch
    unsigned char* gscratch;    // mode 2: per-CTA slice of global memory replacing SMEM
    long long gslice;           // bytes per CTA slice
    long long sl_off, acc_off;  // BIG: byte offsets of the stabiliser and extraction arrays in a slice
    int4* box;            // nb*nb (y0r, y0c, hr, hc), updated in place
    long long* off;       // nb*nb offsets (in: pool_in, out: scratch)
    const double* pool_in;
    double* scratch;
    unsigned long long* bump;   // scratch allocation counter (entries)
    long long cap;              // scratch capacity (entries)
    double* alpha;        // alpha_C image, side*side
    const double* mu;     // layer mu
    const double* logmu;  // layer log mu (-inf where 0)
    const double* mass_i; // nb*nb
    CellOut* out;         // ncells
    int* list_in;         // modes 1/2: cells to solve
    int* n_in;
    int* list_out;        // modes 0/1: cells whose Y box exceeds bcap (next tier)
    int* n_out;
    int* work_counter;    // modes 1/2 dynamic work index
    int* overflow;        // set if scratch capacity exceeded
    int* ipred;           // this partition's iteration counts of the previous sweep (work predictor for the LPT order)
    int poison;           // testing (DD_POISON): K1 fills its dynamic SMEM with 0xFF bytes first
    size_t smem_bytes;    // dynamic SMEM of the launch (for the poison fill)
    // general separable cost (dd_set_cost): c = h1(|dr|) + h2(|dc|) in [0,1]^2 units,
    // tables over FINEST-grid pixel differences; a layer difference d is d * hst finest
    // pixels.  nullptr: |x - y|^2 (the shifted-gauge quadratic path)
    const double* h1;
    const double* h2;
    int hst;
    int safeguard;        // DD_FLAG_SAFEGUARD: eps-raising retry of failing cells (A29)
    // testing (env DD_FORCE_RESCUE="cell:it", read per sweep): composite cell `force_cell` leaves the
    // fp32 loop after `force_it` iterations and finishes in fp64 (rescue_fp64), as a stalled cell would
    int force_cell, force_it;
    // tier G (SMEM-tier kernel on a global-memory layout): the
    // cells beyond the largest on-chip tier; CTA b carves its K1Lay from
    // gbase + b * gbase_bytes instead of shared memory
    unsigned char* gbase;
    long long gbase_bytes;
};

// ------------------------------------------------------------- helpers --
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2f(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {   // FMNMX3 (sm_100)
    float y;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
    return y;
}
__device__ __forceinline__ float rcpf(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// ------------------------------------------------ bulk-copy engine (TMA) --
// 1D bulk global -> shared copies (cp.async.bulk) completing on an mbarrier:
// K1 stages a cell's X side (alpha, mu, log mu rows) this way.
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned a, unsigned parity) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    return ok != 0;
}

// ------------------------------------------- thread-block cluster (DSMEM) --
// The K1 cluster tier splits one composite cell
// over CS CTAs of a cluster: every CTA keeps a full replica of the O(a b)
// SMEM state and each output a CTA computes is stored to all replicas.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// address of the same SMEM location in the CTA of cluster rank r
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned r) {
    unsigned o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void st_cl(unsigned a, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cl(unsigned a, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cl(unsigned a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cl(unsigned a, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_cl(unsigned a, int v) {
    int o;
    asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}
// one lane's shared-memory counter fetch (no compiler warp-aggregation code around it)
__device__ __forceinline__ int atom_add_sh(unsigned a, int v) {
    int o;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ void atom_or_cl(unsigned a, int v) {
    asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// all threads of all CTAs of the cluster; release/acquire at cluster scope
// (orders the DSMEM stores and the global-slice writes of the iteration)
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Store v at p in this CTA and in the CS - 1 peer replicas.
template <int CS, typename T>
__device__ __forceinline__ void bcast(T* p, T v) {
    *p = v;
    if constexpr (CS > 1) {
        const unsigned a = smem_u32(p), me = cluster_rank();
#pragma unroll
        for (unsigned r = 0; r < (unsigned)CS; ++r)
            if (r != me) st_cl(mapa_u32(a, r), v);
    }
}
template <int CS>
__device__ __forceinline__ void cta_or_cluster_sync() {
    if constexpr (CS > 1) cluster_sync_all();
    else __syncthreads();
}

// Round to the 2^-8 grid without touching the XU pipe (two FADDs).
__device__ __forceinline__ float grid8(float v) {
    return __fsub_rn(__fadd_rn(v, kGridMagic), kGridMagic);
}
__host__ __device__ inline int odd_pitch(int n) { return n | 1; }

// Composite-cell geometry (A11): basic rows/cols of
// cell p along one axis of partition part.
__device__ __forceinline__ void cell_span(int nb, int part, int p, int& lo, int& hi) {
    if (part == 1) { lo = 2 * p; hi = 2 * p + 1; }
    else {
        lo = 2 * p - 1 < 0 ? 0 : 2 * p - 1;
        hi = 2 * p > nb - 1 ? nb - 1 : 2 * p;
    }
}

// Block-wide reductions (blockDim.x == kThreads).  red: >= 32 doubles of smem.
__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Fixed-order block sum: every thread returns the total.
__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    for (int k = 0; k < nw; ++k) t += red[k];
    return t;
}
// The same with one barrier: only valid when every thread's previous read of
// red[] is separated from this call by at least one other block barrier.
__device__ __forceinline__ double block_sum1(double v, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    for (int k = 0; k < nw; ++k) t += red[k];
    return t;
}
__device__ __forceinline__ double block_max(double v, double* red) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = -INFINITY;
    const int nw = blockDim.x >> 5;
    for (int k = 0; k < nw; ++k) t = fmax(t, red[k]);
    return t;
}

}  // namespace dd
