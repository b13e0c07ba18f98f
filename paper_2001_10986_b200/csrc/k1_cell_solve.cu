// k1_cell_solve.cu -- K1: fused composite-cell solve of one sweep of
// Algorithm 2 (arXiv 2001.10986), one CTA per cell.
//
//   line 8   nu_cell = sum_{i in J} nu_i          -> gather, log into SMEM
//   line 9   (pi_cell, u_{C,J}) = Sinkhorn(...)    -> separable log-domain
//            Sinkhorn, warm-started from alpha, starts with a Y-iteration,
//            stops when the L1 X-error <= ||mu_J|| Err (Sec. 6.2)
//   line 10  nu_i = P_Y(pi_cell restricted to X_i x Y) -> one final exact
//            Y-iteration from the plan's F that splits every row sum by
//            basic-cell quadrant (ratio form, A7)
//   line 11  BalanceMeasures (A8)
//   line 12  Truncate + tight bounding box -> scratch pool
//
// Numerics: potentials in a cell-local affine
// gauge as fp32 (hi, lo2) pairs, hi on a per-cell grid 2^-q chosen so that
// hi - C(d) - S is EXACT in fp32; exact per-axis cost table C(d) = d^2/kappa;
// ex2.approx of the reduced argument; accurate fp32 log of each row sum;
// fp64 staging, balance and marginal sums.  The grid cost is separable, so a
// half-iteration is two 1D log-sum-exp passes (a^2 b + a b^2 exps, not a^2 b^2).
//
// Work layout: each thread owns R = 4 consecutive outputs of a pass (one row
// o1 of the pass input P, outputs o2 .. o2+3), so one 8-byte SMEM load of
// P(o1, k) feeds 4 exponentials and the cost window slides by one table
// load per k.  Lanes of a warp own different rows (odd pitches: conflict-free)
// and read the same cost entries (broadcast).  When a pass has fewer tasks
// than threads, G lanes split the k-range of a task (shuffle-combined).
#include "dd_common.cuh"

#ifndef DD_T0_MINB
#define DD_T0_MINB 3
#endif
// phase A of the fused pass with 8-column quarter chunks for the narrow tails
// fused pass, per-group control (round 2, profiles/r02/r02_t2_lines.txt: the group fetch, the
// stabiliser prologue, the window check and the U epilogue were ~13 % of K1's instructions):
// inline atom.shared for the group counter, branch-free prologue / window check, the four U
// outputs of a (row, x2 quad) dealt over its YS lanes.  Same arithmetic, same bits.
#ifndef DD_FV2
#define DD_FV2 1
#endif
#ifndef DD_PA_Q
#define DD_PA_Q 1
#endif
namespace dd {

constexpr int kR = 4;   // outputs per thread-task

// the CTA's mbarrier of the X-side bulk copies (initialised at kernel start)
__shared__ unsigned long long g_k1_mbar;

// --------------------------------------------------------- SMEM layout --
struct K1Lay {
    float2* FX;   // [ar][pX]  X potential F (hi, lo2)
    float2* FXn;  // [ar][pX]  X-iteration output
    float2* LM;   // [ar][ac]  log mu (hi, lo2)
    float* MU;    // [ar][ac]  mu (fp32, error weights)
    float2* Tt;   // [bc][pT]  Y pass-1 output T(x1, y2), transposed
    float2* Ut;   // [ac][pU]  X pass-1 output U(y1, x2); final pass: split weights W [bc][pT]
    float2* G;    // [br][pG]  Y potential G (hi, lo2); final pass: ACC (float4 [br][bc]) over G+LNU
    float2* LNU;  // [br][bc]  log nu_cell (hi, lo2)
    float* CT;    // cost table C(d) = d^2 / kappa, d in [-OFF, OFF]
    double* red;  // reduction scratch (64)
    float2* gbuf; // BIG: per-warp G rows of the fused Y2+X1 pass [warp][kGbufPerWarp]
    float2* CP;   // BIG: cost pairs CP[k] = (CT[k], CT[k-1])
    int* WK;      // BIG: [0] row-group counter of the fused pass (dynamic LPT)
    float* FH;    // BIG: F (current) as separate hi / lo planes [a_r][a_c] for the Y1 pass
    float* FL;
    int2* RI;     // BIG: per Y row, the columns [lo, hi] where nu_cell > 0 (lo > hi: empty)
    int* GL;      // BIG: row groups of the fused pass, heaviest first (dynamic LPT)
    int2* GI;     // BIG: per row group, the union of its rows' non-zero column ranges
    double* errv; // BIG: per X point, the X-error term of the current iteration [a_r][a_c]
    float2* CG;   // general cost (tier 0 only): 4 tables [row+, row-, col+, col-][2 off + 8] of
                  // (hi on the cell grid, lo2) -- index semantics as CT, see cg_table()
};

// BIG mode (fused Y2+X1): G is never stored as
// a b^2 array; log nu_cell (b^2 float2) and the extraction partial sums
// (b^2 float4) live in an L2-resident global slice per CTA.
constexpr int kGbufPerWarp = 144;   // max over NQ (RG = 4) of RG * YS * (SUB + 1)

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }
__host__ __device__ inline int k1_ct_off(int s, int bcap) { return (2 * s > bcap ? 2 * s : bcap) + 24; }

__host__ __device__ inline void k1_sizes(int s, int bcap, size_t* sz, bool big = false, int nwarps = 0,
                                         bool gc = false) {
    const size_t A = 2 * s, pA = odd_pitch(2 * s), pB = odd_pitch(bcap), B = bcap;
    sz[0] = align16(A * pA * 8);                        // FX
    sz[1] = align16(A * pA * 8);                        // FXn
    sz[2] = align16(A * A * 8);                         // LM
    sz[3] = align16(A * A * 4);                         // MU
    sz[4] = align16(B * pA * 8);                        // Tt
    sz[5] = align16((A * pB > B * pA ? A * pB : B * pA) * 8);   // Ut / W
    sz[6] = big ? 0 : align16(B * pB * 8);              // G   } ACC (16 B per y) overlays
    sz[7] = big ? 0 : align16(B * B * 8);               // LNU }
    sz[8] = align16((2 * k1_ct_off(s, bcap) + 8) * 4);  // CT
    sz[9] = 64 * 8;                                     // red
    sz[10] = big ? (size_t)nwarps * kGbufPerWarp * 8 : 0;   // gbuf
    sz[11] = big ? align16((2 * k1_ct_off(s, bcap) + 8) * 8) : 0;   // CP
    sz[12] = big ? 16 : 0;                                           // WK [0] groups [1] npos [2] flags [3] fallbacks
    sz[13] = big ? (size_t)A * A * 4 : 0;                            // FH
    sz[14] = big ? (size_t)A * A * 4 : 0;                            // FL
    sz[15] = align16((size_t)A * A * 8);                             // errv (fp64 rescue, BIG loop)
    sz[16] = big ? align16((size_t)(bcap + 1) * 8) : 0;             // RI
    sz[17] = big ? align16((size_t)(bcap / 4 + 2) * 4) : 0;         // GL
    sz[18] = (gc && !big) ? align16((size_t)4 * (2 * k1_ct_off(s, bcap) + 8) * 8) : 0;   // CG
    sz[19] = big ? align16((size_t)(bcap / 4 + 2) * 8) : 0;         // GI
}

__host__ __device__ inline size_t k1_smem_bytes(int s, int bcap, bool big = false, int nwarps = 0,
                                                bool gc = false) {
    size_t sz[20], b = 0;
    k1_sizes(s, bcap, sz, big, nwarps, gc);
    for (int k = 0; k < 20; ++k) b += sz[k];
    return b;
}

__device__ inline K1Lay k1_carve(unsigned char* base, int s, int bcap, bool big = false, int nwarps = 0,
                                 bool gc = false) {
    size_t sz[20];
    k1_sizes(s, bcap, sz, big, nwarps, gc);
    K1Lay L;
    size_t o = 0;
    L.FX = (float2*)(base + o);  o += sz[0];
    L.FXn = (float2*)(base + o); o += sz[1];
    L.LM = (float2*)(base + o);  o += sz[2];
    L.MU = (float*)(base + o);   o += sz[3];
    L.Tt = (float2*)(base + o);  o += sz[4];
    L.Ut = (float2*)(base + o);  o += sz[5];
    L.G = (float2*)(base + o);   o += sz[6];
    L.LNU = (float2*)(base + o); o += sz[7];
    L.CT = (float*)(base + o);   o += sz[8];
    L.red = (double*)(base + o); o += sz[9];
    L.gbuf = (float2*)(base + o); o += sz[10];
    L.CP = (float2*)(base + o); o += sz[11];
    L.WK = (int*)(base + o); o += sz[12];

    L.FH = (float*)(base + o); o += sz[13];
    L.FL = (float*)(base + o); o += sz[14];
    L.errv = (double*)(base + o); o += sz[15];
    L.RI = (int2*)(base + o); o += sz[16];
    L.GL = (int*)(base + o); o += sz[17];
    L.CG = (float2*)(base + o); o += sz[18];
    L.GI = (int2*)(base + o);
    return L;
}

struct Dims {
    int ar, ac, br, bc, s;
    int pX, pT, pG, pU;
    int off;      // CT centre
};

// Per-cell hi grid 2^-q: all hi values, the cost table and every
// intermediate hi - C - S stay multiples of 2^-q below 2^(23-q) -> exact.
struct Grid {
    float magic;      // 1.5 * 2^(23-q): (v + magic) - magic rounds v to the grid
    double scale;     // 2^q
    double inv;       // 2^-q
};
__device__ __forceinline__ float gridq(float v, const Grid& g) {
    return __fsub_rn(__fadd_rn(v, g.magic), g.magic);
}

// Split an fp64 value into (hi on the grid, lo2 = (v - hi) * log2 e).
__device__ __forceinline__ float2 split_hl(double v, const Grid& g) {
    if (!(v > -1e30)) return make_float2(-INFINITY, 0.0f);
    const double h = rint(v * g.scale) * g.inv;
    return make_float2((float)h, (float)((v - h) * 1.4426950408889634));
}
__device__ __forceinline__ double join_hl(float2 p) {
    return (double)p.x + (double)p.y * 0.6931471805599453;
}

// ln(x) = hi + lo2 * ln 2 with hi on the grid; ~5e-8 absolute and ~1e-7
// RELATIVE near x = 1 (converged sums).  x > 0 normal.
__device__ __forceinline__ void ln_split(float x, const Grid& gq, float& hi, float& lo2) {
    const float LN2H = 0.693145751953125f;          // 0x3F317200 (e * LN2H exact)
    const float LN2L = 1.428606765330187e-06f;
    const int ix = __float_as_int(x);
    int e = ((ix >> 23) & 0xff) - 127;
    float m = __int_as_float((ix & 0x007fffff) | 0x3f800000);
    if (m > 1.41421356f) { m *= 0.5f; e += 1; }
    const float num = m - 1.0f;
    const float den = m + 1.0f;
    float r = rcpf(den);
    r = r * fmaf(-den, r, 2.0f);
    const float z = num * r;
    const float z2 = z * z;
    float p = 0.18181818f;
    p = fmaf(p, z2, 0.22222222f);
    p = fmaf(p, z2, 0.28571429f);
    p = fmaf(p, z2, 0.4f);
    p = fmaf(p, z2, 0.66666667f);
    p = fmaf(p, z2, 2.0f);
    const float lnm = z * p;
    const float eh = (float)e * LN2H;
    const float g = gridq(eh, gq);
    const float v = (eh - g) + lnm;
    const float gh = gridq(v, gq);
    hi = g + gh;
    lo2 = ((v - gh) + (float)e * LN2L) * kL2E;
}

enum { PY1 = 0, PY2 = 1, PX1 = 2, PX2 = 3, PY1S = 4, PY2S = 5 };


// Phase profile (build with -DDD_PHASE_PROF, tools/phase_profile.py): per-warp
// cycle counters summed over all warps of all cells of a launch, by BIG mode.
#ifdef DD_PHASE_PROF
__device__ unsigned long long g_phase[2][16];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(k, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase[BIG ? 1 : 0][k], (unsigned long long)(v)); } while (0)
#else
#define PROF_T(v) do {} while (0)
#define PROF_ADD(k, v) do {} while (0)
#endif

// One separable log-sum-exp pass.  A task is (o1, outputs o2 = 4j .. 4j+3).
//   out(o1, o2) = S + log sum_k exp(P(o1,k).hi - C(k - o2) - S + P(o1,k).lo2 ln 2)
// Y1 : o1 = x1, k = x2, o2 = y2 -> Tt[y2][x1]
// Y2 : o1 = y2, k = x1, o2 = y1 -> G[y1][y2] = LNU - out
// X1 : o1 = y1, k = y2, o2 = x2 -> Ut[x2][y1]
// X2 : o1 = x2, k = y1, o2 = x1 -> FXn[x1][x2] = LM - out, L1 X-error
// Y1S: as Y1 (exact), also the split weights W[y2][x1] of the two x2 halves
// Y2S: as Y2 (exact), writes the quadrant partial sums ACC[y1][y2] instead of G
// Lane groups of G (compile time) lanes split the k-range of a task.  Every
// lane of a warp runs the same number of tasks (ntask_pad) and the exact /
// speculative mode is decided per WARP for G > 1, so the group reductions are
// full-warp xor butterflies (offsets < G stay inside the aligned group; the
// summation order is that of the group) -- no divergent-mask shuffles.
template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ float gmax(float v) {
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int PASS, int NT, int G, bool GC>
__device__ __forceinline__ void lse_pass_g(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all,
                                           float2* Fcur, float2* Fout, double& err_acc, int& fallbacks,
                                           int& nonfinite);

template <int PASS, int NT, bool GC = false>
__device__ __forceinline__ void lse_pass(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all,
                                         float2* Fcur, float2* Fout, double& err_acc, int& fallbacks,
                                         int& nonfinite) {
    // NT threads take part (a larger block calls it with a smaller NT: the
    // lane-group split, hence the summation order, depends on NT only)
    if (threadIdx.x >= NT) return;
    int n1, n2;
    if (PASS == PY1 || PASS == PY1S) { n1 = d.ar; n2 = d.bc; }
    else if (PASS == PY2 || PASS == PY2S) { n1 = d.bc; n2 = d.br; }
    else if (PASS == PX1) { n1 = d.br; n2 = d.ac; }
    else { n1 = d.ac; n2 = d.ar; }
    const int ntask = n1 * ((n2 + kR - 1) / kR);
    int G = 1;
    while (G < 8 && ntask * G * 2 <= NT) G <<= 1;
    switch (G) {
    case 1: lse_pass_g<PASS, NT, 1, GC>(L, d, gq, exact_all, Fcur, Fout, err_acc, fallbacks, nonfinite); break;
    case 2: lse_pass_g<PASS, NT, 2, GC>(L, d, gq, exact_all, Fcur, Fout, err_acc, fallbacks, nonfinite); break;
    case 4: lse_pass_g<PASS, NT, 4, GC>(L, d, gq, exact_all, Fcur, Fout, err_acc, fallbacks, nonfinite); break;
    default: lse_pass_g<PASS, NT, 8, GC>(L, d, gq, exact_all, Fcur, Fout, err_acc, fallbacks, nonfinite); break;
    }
}

template <int PASS, int NT, int G, bool GC>
__device__ __forceinline__ void lse_pass_g(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all,
                                           float2* Fcur, float2* Fout, double& err_acc, int& fallbacks,
                                           int& nonfinite) {
    constexpr bool kY1 = (PASS == PY1 || PASS == PY1S);
    constexpr bool kY2 = (PASS == PY2 || PASS == PY2S);
    constexpr bool kSplit = (PASS == PY1S || PASS == PY2S);
    int n1, K, n2, pitchP, ksplit;
    const float2* P;
    if (kY1) { n1 = d.ar; K = d.ac; n2 = d.bc; P = Fcur; pitchP = d.pX; ksplit = min(d.s, K); }
    else if (kY2) { n1 = d.bc; K = d.ar; n2 = d.br; P = L.Tt; pitchP = d.pT; ksplit = min(d.s, K); }
    else if (PASS == PX1) { n1 = d.br; K = d.bc; n2 = d.ac; P = L.G; pitchP = d.pG; ksplit = K; }
    else { n1 = d.ac; K = d.br; n2 = d.ar; P = L.Ut; pitchP = d.pU; ksplit = K; }
    const float2* Wb = L.Ut;              // split weights (Y1S writes, Y2S reads), layout [y2][x1]
    float4* ACC = reinterpret_cast<float4*>(L.G);

    const int n2q = (n2 + kR - 1) / kR;
    const int ntask = n1 * n2q;
    const int lg = threadIdx.x & (G - 1);
    const int ntask_pad = ((ntask + (NT / G) - 1) / (NT / G)) * (NT / G);
    const float2 L2E2 = make_float2(kL2E, kL2E);

    for (int t = threadIdx.x / G; t < ntask_pad; t += NT / G) {
        const bool active = t < ntask;
        const int o1 = active ? t % n1 : 0;
        const int o2 = active ? (t / n1) * kR : 0;
        const float2* Prow = P + o1 * pitchP;
        bool valid[kR], skip[kR];
        float2 tg[kR];
        float S[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            valid[r] = active && (o2 + r < n2);
            skip[r] = !valid[r];
            tg[r] = make_float2(0.f, 0.f);
            if (valid[r]) {
                if (PASS == PY2) {
                    tg[r] = L.LNU[(o2 + r) * d.bc + o1];
                    skip[r] = (tg[r].x == -INFINITY);
                } else if (PASS == PX2) {
                    tg[r] = L.LM[(o2 + r) * d.ac + o1];
                    skip[r] = (tg[r].x == -INFINITY);
                }
            }
            S[r] = 0.f;
        }
        bool exact = exact_all || kSplit;
        if (!exact) {
            bool okS = true;
            float Sf = 0.f;
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                if (skip[r]) continue;
                const int o = o2 + r;
                float s;
                if (PASS == PY1) s = L.Tt[o * d.pT + o1].x;
                else if (PASS == PY2) s = tg[r].x - L.G[o * d.pG + o1].x;
                else if (PASS == PX1) s = L.Ut[o * d.pU + o1].x;
                else s = tg[r].x - Fcur[o * d.pX + o1].x;
                S[r] = s;
                Sf = s;
                okS = okS && (fabsf(s) < 1e30f);
            }
#pragma unroll
            for (int r = 0; r < kR; ++r) if (skip[r]) S[r] = Sf;
            exact = !okS;
            if (G > 1) exact = __any_sync(0xffffffffu, exact);   // one mode per warp (converged shuffles)
        }
        const float* ctp = L.CT + d.off - o2;   // C(k - o2 - r) = ctp[k - r]
        // general cost: the pass's (axis, orientation) table, same indexing,
        // entries (hi on the cell grid, lo2 = (C - hi) log2 e)
        constexpr int kTab = kY1 ? 2 : kY2 ? 0 : (PASS == PX1) ? 3 : 1;
        const float2* cgp = GC ? L.CG + kTab * (2 * d.off + 8) + d.off - o2 : nullptr;
        float acc[kR], acc1[kR], q[kR][4];
        bool done = false;
        for (int attempt = 0; attempt < 2 && !done; ++attempt) {
            if (exact) {
                float M[kR];
#pragma unroll
                for (int r = 0; r < kR; ++r) M[r] = -INFINITY;
                for (int k = lg; k < K; k += G) {
                    const float px = Prow[k].x;
#pragma unroll
                    for (int r = 0; r < kR; ++r) M[r] = fmaxf(M[r], px - (GC ? cgp[k - r].x : ctp[k - r]));
                }
#pragma unroll
                for (int r = 0; r < kR; ++r) {
                    if (G > 1) M[r] = gmax<G>(M[r]);
                    if (M[r] == -INFINITY) { skip[r] = true; S[r] = 0.f; }
                    else S[r] = M[r];
                }
            }
            const float2 nS01 = make_float2(-S[0], -S[1]), nS23 = make_float2(-S[2], -S[3]);
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                acc[r] = 0.f; acc1[r] = 0.f;
                q[r][0] = q[r][1] = q[r][2] = q[r][3] = 0.f;
            }
            // ---- the hot loop: 4 exps per 8-byte P load + 1 cost-table load
            auto body = [&](int k, float c0, float c1, float c2, float c3, float* A, int half) {
                const float2 pk = Prow[k];
                if constexpr (GC) {      // c_r = the hi parts; the lo parts join the lo term
                    const float2 g0 = cgp[k], g1 = cgp[k - 1], g2 = cgp[k - 2], g3 = cgp[k - 3];
                    c0 = g0.x; c1 = g1.x; c2 = g2.x; c3 = g3.x;
                    float2 t01 = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-c0, -c1));
                    float2 t23 = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-c2, -c3));
                    t01 = __fadd2_rn(t01, nS01);
                    t23 = __fadd2_rn(t23, nS23);
                    t01 = __ffma2_rn(t01, L2E2, make_float2(pk.y - g0.y, pk.y - g1.y));
                    t23 = __ffma2_rn(t23, L2E2, make_float2(pk.y - g2.y, pk.y - g3.y));
                    const float e0 = ex2f(t01.x), e1 = ex2f(t01.y), e2 = ex2f(t23.x), e3 = ex2f(t23.y);
                    if (PASS == PY2S) {
                        const float2 w = Wb[o1 * d.pT + k];
                        const int c = 2 * half;
                        q[0][c] = fmaf(e0, w.x, q[0][c]); q[0][c + 1] = fmaf(e0, w.y, q[0][c + 1]);
                        q[1][c] = fmaf(e1, w.x, q[1][c]); q[1][c + 1] = fmaf(e1, w.y, q[1][c + 1]);
                        q[2][c] = fmaf(e2, w.x, q[2][c]); q[2][c + 1] = fmaf(e2, w.y, q[2][c + 1]);
                        q[3][c] = fmaf(e3, w.x, q[3][c]); q[3][c + 1] = fmaf(e3, w.y, q[3][c + 1]);
                    } else {
                        float2 a01 = make_float2(A[0], A[1]), a23 = make_float2(A[2], A[3]);
                        a01 = __fadd2_rn(a01, make_float2(e0, e1));
                        a23 = __fadd2_rn(a23, make_float2(e2, e3));
                        A[0] = a01.x; A[1] = a01.y; A[2] = a23.x; A[3] = a23.y;
                    }
                    return;
                }
                float2 t01 = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-c0, -c1));
                float2 t23 = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-c2, -c3));
                t01 = __fadd2_rn(t01, nS01);
                t23 = __fadd2_rn(t23, nS23);
                t01 = __ffma2_rn(t01, L2E2, make_float2(pk.y, pk.y));
                t23 = __ffma2_rn(t23, L2E2, make_float2(pk.y, pk.y));
                const float e0 = ex2f(t01.x), e1 = ex2f(t01.y), e2 = ex2f(t23.x), e3 = ex2f(t23.y);
                if (PASS == PY2S) {
                    const float2 w = Wb[o1 * d.pT + k];
                    const int c = 2 * half;
                    q[0][c] = fmaf(e0, w.x, q[0][c]); q[0][c + 1] = fmaf(e0, w.y, q[0][c + 1]);
                    q[1][c] = fmaf(e1, w.x, q[1][c]); q[1][c + 1] = fmaf(e1, w.y, q[1][c + 1]);
                    q[2][c] = fmaf(e2, w.x, q[2][c]); q[2][c + 1] = fmaf(e2, w.y, q[2][c + 1]);
                    q[3][c] = fmaf(e3, w.x, q[3][c]); q[3][c + 1] = fmaf(e3, w.y, q[3][c + 1]);
                } else {
                    float2 a01 = make_float2(A[0], A[1]), a23 = make_float2(A[2], A[3]);
                    a01 = __fadd2_rn(a01, make_float2(e0, e1));
                    a23 = __fadd2_rn(a23, make_float2(e2, e3));
                    A[0] = a01.x; A[1] = a01.y; A[2] = a23.x; A[3] = a23.y;
                }
            };
            if (GC) {
                for (int k = lg; k < ksplit; k += G) body(k, 0.f, 0.f, 0.f, 0.f, acc, 0);
                const int k1 = ksplit + ((lg - ksplit % G) % G + G) % G;
                for (int k = k1; k < K; k += G) body(k, 0.f, 0.f, 0.f, 0.f, acc1, 1);
            } else if (G == 1) {
                // sliding cost window: c_r = C(k - o2 - r)
                float c1 = ctp[-1], c2 = ctp[-2], c3 = ctp[-3];
#pragma unroll 2
                for (int k = 0; k < ksplit; ++k) {
                    const float c0 = ctp[k];
                    body(k, c0, c1, c2, c3, acc, 0);
                    c3 = c2; c2 = c1; c1 = c0;
                }
#pragma unroll 2
                for (int k = ksplit; k < K; ++k) {
                    const float c0 = ctp[k];
                    body(k, c0, c1, c2, c3, acc1, 1);
                    c3 = c2; c2 = c1; c1 = c0;
                }
            } else {
                for (int k = lg; k < ksplit; k += G) body(k, ctp[k], ctp[k - 1], ctp[k - 2], ctp[k - 3], acc, 0);
                const int k1 = ksplit + ((lg - ksplit % G) % G + G) % G;   // first k >= ksplit with k = lg mod G
                for (int k = k1; k < K; k += G) body(k, ctp[k], ctp[k - 1], ctp[k - 2], ctp[k - 3], acc1, 1);
            }
            float tot[kR];
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                if (G > 1) {
                    acc[r] = gsum<G>(acc[r]);
                    acc1[r] = gsum<G>(acc1[r]);
                    if (PASS == PY2S)
#pragma unroll
                        for (int c = 0; c < 4; ++c) q[r][c] = gsum<G>(q[r][c]);
                }
                tot[r] = (PASS == PY2S) ? (q[r][0] + q[r][1]) + (q[r][2] + q[r][3]) : acc[r] + acc1[r];
            }
            if (exact) { done = true; break; }
            // speculative window: dominant terms must stay near t = 0 for the
            // exactness argument of the (hi, lo) arithmetic
            bool ok = true;
#pragma unroll
            for (int r = 0; r < kR; ++r) ok = ok && (skip[r] || (tot[r] >= 0.25f && tot[r] <= 4.0f));
            if (G > 1) ok = __all_sync(0xffffffffu, ok);
            if (ok) { done = true; break; }
            exact = true;
            if (lg == 0) ++fallbacks;
        }

        // ---- finalise the outputs (one lane per group)
        if (lg != 0) continue;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            if (!valid[r]) continue;
            const int o = o2 + r;
            const float tot = (PASS == PY2S) ? (q[r][0] + q[r][1]) + (q[r][2] + q[r][3]) : acc[r] + acc1[r];
            float Lhi = -INFINITY, Llo = 0.f;
            const bool empty = skip[r] || !(tot > 1e-37f);
            if (!empty) {
                float lh, ll;
                ln_split(tot, gq, lh, ll);
                Lhi = S[r] + lh;
                Llo = ll;
                if (!(fabsf(Lhi) < 1e30f)) nonfinite = 1;
            }
            if (kY1) {
                L.Tt[o * d.pT + o1] = make_float2(Lhi, empty ? 0.f : Llo);
                if (PASS == PY1S) {
                    float2 w = make_float2(0.f, 0.f);
                    if (!empty) {
                        const float rr = rcpf(tot);
                        w = make_float2(acc[r] * rr, acc1[r] * rr);
                    }
                    L.Ut[o * d.pT + o1] = w;
                }
            } else if (PASS == PY2) {
                if (skip[r]) {
                    L.G[o * d.pG + o1] = make_float2(-INFINITY, 0.f);
                } else {
                    if (empty) nonfinite = 1;     // nu_cell(y) > 0 unreachable
                    L.G[o * d.pG + o1] = make_float2(tg[r].x - Lhi, tg[r].y - Llo);
                }
            } else if (PASS == PY2S) {
                ACC[o * d.bc + o1] = make_float4(q[r][0], q[r][1], q[r][2], q[r][3]);
            } else if (PASS == PX1) {
                L.Ut[o * d.pU + o1] = make_float2(Lhi, empty ? 0.f : Llo);
            } else {
                const int ix = o * d.pX + o1;
                if (skip[r]) {
                    Fout[ix] = make_float2(-INFINITY, 0.f);
                } else {
                    if (empty) nonfinite = 1;
                    const float2 fn = make_float2(tg[r].x - Lhi, tg[r].y - Llo);
                    Fout[ix] = fn;
                    const float2 fo = Fcur[ix];
                    // P_X pi(x) = mu(x) exp(F - F_new)  (plan (F, G))
                    const float dF = (fo.x - fn.x) + (fo.y - fn.y) * kLN2;
                    err_acc += (double)L.MU[o * d.ac + o1] * (double)fabsf(expm1f(dF));
                }
            }
        }
    }
}

// ------------------------------------------------- BIG: fused Y2 + X1 pass --
// For every Y row y1 (row groups of RG = 8 rows per warp, no block barrier):
//   phase A (lane <-> y2 of a 32-column chunk):
//     G(y1, y2) = log nu_cell(y1, y2) - LSE_x1[T(x1, y2) - C(x1 - y1)]
//     with the speculative stabiliser S = this output's LSE of the previous
//     iteration (global slice SL, on the hi grid); rows are processed in
//     pairs so that one packed FADD2/FFMA2 serves two exps with T(x1, y2)
//     broadcast and the cost pair (C(x1-y1), C(x1-y1-1)) one LDS.64 from the
//     pair table CP; an output whose sum leaves [1/4, 4] is recomputed with
//     an exact max (first iteration: exact two-pass for all).
//   phase B (lane <-> (row r, x2 quad, y2 slice hB: columns hB + YS k)):
//     U(y1, x2) += sum_{y2 in chunk} exp(G(y1, y2) - C(y2 - x2) - S(y1, x2))
//     (S = previous U; cost pairs slide with period 2 over y2; exact two-pass
//     max on the first iteration or when the window check fails).
// G lives only in a per-warp buffer of one chunk; U is written to Ut[x2][y1]
// for the X2 pass.  Algorithmic exps: ar br bc (phase A) + br bc ac (phase B)
// = the Y2 and X1 passes of the separable scheme.
//
// Work units are whole row groups taken from a block-wide counter, heaviest
// first (dynamic LPT; cost ~ 32-column chunks, then width).  U of a group
// does not depend on which warp computed it, so the result is deterministic;
// the X2 pass runs after the block barrier (x2_finalize) over fixed row
// ranges.  (Measured: splitting a group's chunks over warps with a published
// partial-sum combine, and fusing X2 into this pass, were both slower.)

__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
template <bool B> struct BoolTag { static constexpr bool value = B; };

template <int NT, int AR, int NQ, int RG, int CS>
__device__ __forceinline__ void fused_y2x1(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all,
                                           const float2* __restrict__ LNUg, float* __restrict__ SLg,
                                           int& fallbacks, int& nonfinite) {
    constexpr int YS = 32 / (RG * NQ);      // phase-B lanes sharing one output (y2 split)
    constexpr int SUB = 32 / YS;            // y2 per phase-B lane slice of a chunk
    constexpr int PR = YS * (SUB + 1);      // gbuf row pitch (float2), conflict-free
    static_assert(RG * PR <= kGbufPerWarp, "gbuf");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* gb = L.gbuf + warp * kGbufPerWarp;
    const int rB = lane / (NQ * YS);
    const int qB = (lane / YS) % NQ;
    const int hB = lane % YS;
    const int x2b = 4 * qB;
    const bool qvalid = x2b < d.ac;       // NQ = 4 serves a_c = 16; NQ = 2 serves a_c = 8 and 4
    // phase-B lane hB owns the chunk columns hB, hB + YS, hB + 2 YS, ... (interleaved:
    // the YS slices of an output get equal work on partial chunks and read
    // conflict-free cost pairs); phase A stores column c at slot (c % YS, c / YS)
    const float2 L2E2 = make_float2(kL2E, kL2E);
    const float2* CP = L.CP;

    const int ng = (d.br + RG - 1) / RG;
    // the group counter lives in cluster rank 0 (CS > 1: groups are dealt
    // over all warps of the cluster)
#if DD_FV2
    const unsigned wk0 = CS > 1 ? mapa_u32(smem_u32(&L.WK[0]), 0) : smem_u32(&L.WK[0]);
#else
    const unsigned wk0 = CS > 1 ? mapa_u32(smem_u32(&L.WK[0]), 0) : 0u;
#endif
    while (true) {
        int u = 0;
#if DD_FV2
        if (lane == 0) u = CS > 1 ? atom_add_cl(wk0, 1) : atom_add_sh(wk0, 1);
#else
        if (lane == 0) u = CS > 1 ? atom_add_cl(wk0, 1) : atomicAdd(&L.WK[0], 1);
#endif
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= ng) break;
        const int grp = L.GL[u];
        const int y1b = grp * RG;
        const int y1B = y1b + rB;
        const bool rvalid = y1B < d.br;
        // the group's non-zero column range [glo, ghi] (union of its rows)
        const int2 gi = L.GI[grp];
        const int glo = gi.x, gend = gi.y + 1;        // exclusive end
        const int cpo = d.off - y1b;        // CP[cpo + x - r] = (C(x - y1b - r), C(x - y1b - r - 1))

        // ---------------------------------------------------------- phase A
        // Full chunk: lane <-> column c0 + lane, all RG rows (RG/2 row pairs).
        // Half chunk (the group's last <= 16 columns; typical row bands are
        // narrow): lane <-> (column c0 + lane % 16, row pair lane / 16), so no
        // lane idles on the missing columns.
        auto phaseA = [&](int c0, auto half_tag) {
            constexpr bool H = decltype(half_tag)::value;
            constexpr int NRL = H ? 2 : RG;             // rows per lane
            constexpr int NP = NRL / 2;                 // row pairs per lane
            const int cl = H ? (lane & 15) : lane;      // column within the chunk
            const int rb = H ? 2 * (lane >> 4) : 0;     // first row of this lane
            const int y2 = c0 + cl;
            const bool vy = y2 < gend;
            const int y2c = vy ? y2 : gend - 1;        // clamped: every lane runs the same code
            float2 ln[NRL];
            float sp[NRL];
#pragma unroll
            for (int q = 0; q < NRL; ++q) {
                const int r = rb + q;
                const bool v = vy && (y1b + r < d.br);
                const int idx = (y1b + r) * d.bc + y2;
                ln[q] = v ? LNUg[idx] : make_float2(-INFINITY, 0.f);
                sp[q] = v ? SLg[idx] : 0.f;
            }
            const float2* __restrict__ Tc = L.Tt + y2c * d.pT;
            // cpb[x - 2 i] = (C(x - r), C(x - r - 1)) for rows r = y1b + rb + 2 i, r + 1
            const float2* __restrict__ cpb = CP + cpo - rb;
            if (exact_all) {
                // exact two-pass: stabiliser = max_x1 (T.hi - C)
                float2 M[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) M[i] = make_float2(-INFINITY, -INFINITY);
#pragma unroll 4
                for (int x = 0; x < AR; ++x) {
                    float th = Tc[x].x;
                    if (AR == 8) th = (x < d.ar) ? th : -INFINITY;
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const float2 tt = __fadd2_rn(make_float2(th, th), neg2(cpb[x - 2 * i]));
                        M[i] = make_float2(fmaxf(M[i].x, tt.x), fmaxf(M[i].y, tt.y));
                    }
                }
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    sp[2 * i] = M[i].x > -INFINITY ? M[i].x : 0.f;
                    sp[2 * i + 1] = M[i].y > -INFINITY ? M[i].y : 0.f;
                }
            }
            float2 nS[NP], acc[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                nS[i] = make_float2(-sp[2 * i], -sp[2 * i + 1]);
                acc[i] = make_float2(0.f, 0.f);
            }
#pragma unroll 4
            for (int x = 0; x < AR; ++x) {
                float2 t = Tc[x];
                // s = 4 edge cells (a_r = 4): rows x >= a_r are past T's pitch
                // (stale SMEM): both halves replaced, so no NaN / inf leaks in
                if (AR == 8 && x >= d.ar) t = make_float2(-INFINITY, 0.f);
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const float2 cs = __fadd2_rn(cpb[x - 2 * i], neg2(nS[i]));   // C + S (exact)
                    float2 tt = __fadd2_rn(make_float2(t.x, t.x), neg2(cs));
                    tt = __ffma2_rn(tt, L2E2, make_float2(t.y, t.y));
                    acc[i] = __fadd2_rn(acc[i], make_float2(ex2f(tt.x), ex2f(tt.y)));
                }
            }
            bool anybad = false;
#pragma unroll
            for (int q = 0; q < NRL; ++q) {
                const float s = (q & 1) ? acc[q >> 1].y : acc[q >> 1].x;
                anybad |= ln[q].x != -INFINITY && (exact_all ? !(s > 0.f) : !(s >= 0.25f && s <= 4.0f));
            }
            anybad = __any_sync(0xffffffffu, anybad);
            const int gslot = (cl % YS) * (SUB + 1) + cl / YS;
#pragma unroll
            for (int q = 0; q < NRL; ++q) {
                const int r = rb + q;
                float2 g = make_float2(-INFINITY, 0.f);
                float s = (q & 1) ? acc[q >> 1].y : acc[q >> 1].x;
                float S = sp[q];
                const bool live = ln[q].x != -INFINITY;
                // exact recompute of an output whose speculative window failed
                // (rare after the first iterations of a solve)
                if (anybad) {
                    const bool bad = live && (exact_all ? !(s > 0.f) : !(s >= 0.25f && s <= 4.0f));
                    if (bad) {
                        float M = -INFINITY;
                        for (int x = 0; x < d.ar; ++x) M = fmaxf(M, Tc[x].x - cpb[x - q].x);
                        s = 0.f;
                        if (M > -INFINITY)
                            for (int x = 0; x < d.ar; ++x) {
                                const float2 t = Tc[x];
                                s += ex2f(((t.x - cpb[x - q].x) - M) * kL2E + t.y);
                            }
                        S = M;
                        if (!exact_all) ++fallbacks;
                    }
                }
                if (live) {
                    if (s > 1e-37f && S > -INFINITY) {
                        const float l2 = lg2f(s);
                        const float lh = gridq(l2 * kLN2, gq);
                        const float ll2 = fmaf(-lh, kL2E, l2);
                        const float Sn = S + lh;
                        SLg[(y1b + r) * d.bc + y2] = Sn;
                        g = make_float2(ln[q].x - Sn, ln[q].y - ll2);
                        if (!(fabsf(Sn) < 1e30f)) nonfinite = 1;
                    } else {
                        nonfinite = 1;       // nu_cell(y) > 0 unreachable from X
                    }
                }
                gb[r * PR + gslot] = g;
            }
        };

#if DD_PA_Q
        // Quarter chunk (8 columns at chunk offset co, the group's last <= 8
        // columns, or columns 16..23 after a half chunk): lane <-> (column
        // co + lane / 4, x1 quarter lane % 4).  Each lane sums its quarter of
        // the x1 range for all RG = 4 rows (the same packed body as above),
        // then a reduce-scatter over the four quarter lanes leaves row
        // lane % 4's sum in that lane, which runs the one-output epilogue.
        // Padding of phase A drops from 16/32 to 8 columns (K1).
        auto phaseQ = [&](int c0, int co) {
            static_assert(RG == 4, "quarter chunk: 4 rows");
            constexpr int XQ = AR / 4;                  // x1 per quarter
            const int qt = lane & 3;
            const int cl = co + (lane >> 2);
            const int y2 = c0 + cl;
            const bool vy = y2 < gend;
            const int y2c = vy ? y2 : gend - 1;
            const int xb = qt * XQ;
            float sp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool v = vy && (y1b + q < d.br);
                sp[q] = v ? SLg[(y1b + q) * d.bc + y2] : 0.f;
            }
            const bool vr = vy && (y1b + qt < d.br);
            const float2 lnr = vr ? LNUg[(y1b + qt) * d.bc + y2] : make_float2(-INFINITY, 0.f);
            const float2* __restrict__ Tc = L.Tt + y2c * d.pT;
            const float2* __restrict__ cpb = CP + cpo;
            if (exact_all) {
                float2 M[2] = {make_float2(-INFINITY, -INFINITY), make_float2(-INFINITY, -INFINITY)};
#pragma unroll
                for (int k = 0; k < XQ; ++k) {
                    const int x = xb + k;
                    float th = Tc[x].x;
                    if (AR == 8) th = (x < d.ar) ? th : -INFINITY;
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const float2 tt = __fadd2_rn(make_float2(th, th), neg2(cpb[x - 2 * i]));
                        M[i] = make_float2(fmaxf(M[i].x, tt.x), fmaxf(M[i].y, tt.y));
                    }
                }
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    for (int o = 1; o <= 2; o <<= 1) {
                        M[i].x = fmaxf(M[i].x, __shfl_xor_sync(0xffffffffu, M[i].x, o));
                        M[i].y = fmaxf(M[i].y, __shfl_xor_sync(0xffffffffu, M[i].y, o));
                    }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    sp[2 * i] = M[i].x > -INFINITY ? M[i].x : 0.f;
                    sp[2 * i + 1] = M[i].y > -INFINITY ? M[i].y : 0.f;
                }
            }
            const float2 nS0 = make_float2(-sp[0], -sp[1]), nS1 = make_float2(-sp[2], -sp[3]);
            float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < XQ; ++k) {
                const int x = xb + k;
                float2 t = Tc[x];
                if (AR == 8 && x >= d.ar) t = make_float2(-INFINITY, 0.f);
                const float2 cs0 = __fadd2_rn(cpb[x], neg2(nS0));
                const float2 cs1 = __fadd2_rn(cpb[x - 2], neg2(nS1));
                float2 t0 = __fadd2_rn(make_float2(t.x, t.x), neg2(cs0));
                float2 t1 = __fadd2_rn(make_float2(t.x, t.x), neg2(cs1));
                t0 = __ffma2_rn(t0, L2E2, make_float2(t.y, t.y));
                t1 = __ffma2_rn(t1, L2E2, make_float2(t.y, t.y));
                a0 = __fadd2_rn(a0, make_float2(ex2f(t0.x), ex2f(t0.y)));
                a1 = __fadd2_rn(a1, make_float2(ex2f(t1.x), ex2f(t1.y)));
            }
            // reduce-scatter: xor 2 exchanges row pairs, xor 1 the rows of a pair
            const bool b1 = (qt & 2) != 0, b0 = (qt & 1) != 0;
            float2 keep = b1 ? a1 : a0;
            const float2 send = b1 ? a0 : a1;
            keep = __fadd2_rn(keep, make_float2(__shfl_xor_sync(0xffffffffu, send.x, 2),
                                                __shfl_xor_sync(0xffffffffu, send.y, 2)));
            float s = b0 ? keep.y : keep.x;
            s += __shfl_xor_sync(0xffffffffu, b0 ? keep.x : keep.y, 1);
            float S = qt == 0 ? sp[0] : qt == 1 ? sp[1] : qt == 2 ? sp[2] : sp[3];
            const bool live = lnr.x != -INFINITY;
            const bool bad = live && (exact_all ? !(s > 0.f) : !(s >= 0.25f && s <= 4.0f));
            if (__any_sync(0xffffffffu, bad) && bad) {
                float M = -INFINITY;
                for (int x = 0; x < d.ar; ++x) M = fmaxf(M, Tc[x].x - cpb[x - qt].x);
                s = 0.f;
                if (M > -INFINITY)
                    for (int x = 0; x < d.ar; ++x) {
                        const float2 t = Tc[x];
                        s += ex2f(((t.x - cpb[x - qt].x) - M) * kL2E + t.y);
                    }
                S = M;
                if (!exact_all) ++fallbacks;
            }
            float2 g = make_float2(-INFINITY, 0.f);
            if (live) {
                if (s > 1e-37f && S > -INFINITY) {
                    const float l2 = lg2f(s);
                    const float lh = gridq(l2 * kLN2, gq);
                    const float ll2 = fmaf(-lh, kL2E, l2);
                    const float Sn = S + lh;
                    SLg[(y1b + qt) * d.bc + y2] = Sn;
                    g = make_float2(lnr.x - Sn, lnr.y - ll2);
                    if (!(fabsf(Sn) < 1e30f)) nonfinite = 1;
                } else {
                    nonfinite = 1;
                }
            }
            gb[qt * PR + (cl % YS) * (SUB + 1) + cl / YS] = g;
        };
#endif

        // ---------------------------------------------------------- phase B
        auto phaseB = [&](int c0, bool maxmode, const float* S, float* A) {
            const int yb0 = c0 + hB;                      // this lane's columns yb0 + YS k
            const int nk = max(0, min(SUB, (gend - yb0 + YS - 1) / YS));
            const float2* __restrict__ gp = gb + rB * PR + hB * (SUB + 1);
            // pair table: cp[YS k] = (C(y2 - x2b), C(y2 - x2b - 1)), y2 = yb0 + YS k;
            // cp[YS k - 2] the next two (x2b + 2, x2b + 3)
            const float2* __restrict__ cp = CP + d.off + yb0 - x2b;
            if (maxmode) {
                for (int k = 0; k < nk; ++k) {
                    const float gx = gp[k].x;
                    const float2 p0 = cp[YS * k], p1 = cp[YS * k - 2];
                    A[0] = fmaxf(A[0], gx - p0.x); A[1] = fmaxf(A[1], gx - p0.y);
                    A[2] = fmaxf(A[2], gx - p1.x); A[3] = fmaxf(A[3], gx - p1.y);
                }
                return;
            }
            const float2 nS01 = make_float2(-S[0], -S[1]), nS23 = make_float2(-S[2], -S[3]);
            float2 a01 = make_float2(A[0], A[1]), a23 = make_float2(A[2], A[3]);
            float2 b01 = make_float2(0.f, 0.f), b23 = make_float2(0.f, 0.f);   // second accumulator chain
            // (C + S) first (exact on the hi grid, independent of G): one dependent
            // FADD2 before the FFMA2, the same bits as (G - C) - S
            const float2 S01 = neg2(nS01), S23 = neg2(nS23);
            auto body = [&](float2 g, float2 p01, float2 p23, float2& s01, float2& s23) {
                const float2 cs01 = __fadd2_rn(p01, S01);
                const float2 cs23 = __fadd2_rn(p23, S23);
                float2 t01 = __fadd2_rn(make_float2(g.x, g.x), neg2(cs01));
                float2 t23 = __fadd2_rn(make_float2(g.x, g.x), neg2(cs23));
                t01 = __ffma2_rn(t01, L2E2, make_float2(g.y, g.y));
                t23 = __ffma2_rn(t23, L2E2, make_float2(g.y, g.y));
                s01 = __fadd2_rn(s01, make_float2(ex2f(t01.x), ex2f(t01.y)));
                s23 = __fadd2_rn(s23, make_float2(ex2f(t23.x), ex2f(t23.y)));
            };
            int k = 0;
            if constexpr (YS == 2) {
                // columns step by 2: the (j = 2, 3) pair at k is the (j = 0, 1) pair at k - 1
                float2 pa = cp[-2];
                for (; k + 4 <= nk; k += 4) {
                    const float2 p0 = cp[0], p1 = cp[2], p2 = cp[4], p3 = cp[6];
                    const float2 g0 = gp[0], g1 = gp[1], g2 = gp[2], g3 = gp[3];
                    body(g0, p0, pa, a01, a23);
                    body(g1, p1, p0, b01, b23);
                    body(g2, p2, p1, a01, a23);
                    body(g3, p3, p2, b01, b23);
                    pa = p3;
                    gp += 4;
                    cp += 8;
                }
                for (; k < nk; ++k) {
                    const float2 p0 = cp[0];
                    body(gp[0], p0, pa, a01, a23);
                    pa = p0;
                    ++gp;
                    cp += 2;
                }
            } else {
                for (; k + 2 <= nk; k += 2) {
                    const float2 g0 = gp[0], g1 = gp[1];
                    body(g0, cp[0], cp[-2], a01, a23);
                    body(g1, cp[YS], cp[YS - 2], b01, b23);
                    gp += 2;
                    cp += 2 * YS;
                }
                if (k < nk) body(gp[0], cp[0], cp[-2], a01, a23);
            }
            a01 = __fadd2_rn(a01, b01);
            a23 = __fadd2_rn(a23, b23);
            A[0] = a01.x; A[1] = a01.y; A[2] = a23.x; A[3] = a23.y;
        };

        // speculative stabilisers from the previous U (row y1B, x2 = x2b .. x2b+3)
        float S[4];
        bool empty[4];
        bool exact = exact_all;
#if DD_FV2
        {
            const bool ld = !exact && rvalid && qvalid;
            const float2* up = L.Ut + x2b * d.pU + y1B;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float u = ld ? up[j * d.pU].x : 0.f;
                const bool fin = fabsf(u) < 1e30f;
                empty[j] = (u == -INFINITY);
                S[j] = fin ? u : 0.f;
                exact = exact | (!fin & !empty[j]);       // +inf or NaN: exact two-pass
            }
        }
#else
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            empty[j] = false;
            S[j] = 0.f;
            if (!exact && rvalid && qvalid) {
                const float u = L.Ut[(x2b + j) * d.pU + y1B].x;
                if (u == -INFINITY) empty[j] = true;
                else if (fabsf(u) < 1e30f) S[j] = u;
                else exact = true;
            }
        }
#endif
        if (!exact_all) exact = __any_sync(0xffffffffu, exact);
        // passes: speculative -> one sum pass; exact -> max pass + sum pass.
        // A failed speculative window check restarts the group in exact mode.
        // (single call sites of phaseA / phaseB keep the code compact)
        float acc[4];
        int pass = exact ? 0 : 1;          // 0: max pass, 1: sum pass
        bool a_done = false;               // G of the (single) chunk still in gbuf
        while (true) {
            const bool maxmode = (pass == 0);
            float A[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) A[j] = maxmode ? -INFINITY : 0.f;
            for (int c0 = glo; c0 < gend; c0 += 32) {
                if (!a_done) {
#if DD_PA_Q
                    const int rem = gend - c0;
                    if (rem <= 8) {
                        phaseQ(c0, 0);
                    } else if (rem <= 24) {
                        phaseA(c0, BoolTag<true>());
                        if (rem > 16) phaseQ(c0, 16);
                    } else {
                        phaseA(c0, BoolTag<false>());
                    }
#else
                    if (gend - c0 <= 16) phaseA(c0, BoolTag<true>());
                    else phaseA(c0, BoolTag<false>());
#endif
                }
                __syncwarp();
                phaseB(c0, maxmode, S, A);
                __syncwarp();
            }
            a_done = (gend - glo <= 32);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                for (int o = YS >> 1; o > 0; o >>= 1) {
                    const float v = __shfl_xor_sync(0xffffffffu, A[j], o);
                    A[j] = maxmode ? fmaxf(A[j], v) : A[j] + v;
                }
            if (maxmode) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    empty[j] = !(A[j] > -INFINITY);
                    S[j] = empty[j] ? 0.f : A[j];
                }
                exact = true;
                pass = 1;
                continue;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = A[j];
            if (exact) break;
            bool ok = true;
#if DD_FV2
            {
                const bool nrq = !rvalid | !qvalid;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool win = (acc[j] >= 0.25f) & (acc[j] <= 4.0f);
                    const bool okj = empty[j] ? (acc[j] == 0.f) : win;
                    ok = ok & (nrq | okj);
                }
            }
#else
#pragma unroll
            for (int j = 0; j < 4; ++j)
                ok = ok && (!rvalid || !qvalid ||
                            (empty[j] ? acc[j] == 0.f : (acc[j] >= 0.25f && acc[j] <= 4.0f)));
#endif
            if (__all_sync(0xffffffffu, ok)) break;
            if (lane == 0) ++fallbacks;
            pass = 0;
        }
#if DD_FV2
        if (rvalid && qvalid) {
            // every lane of the YS-lane slice holds the four sums: lane hB finalises
            // outputs j = hB (4 / YS) .. (one or two of the four)
            constexpr int JO = 4 / YS;
#pragma unroll
            for (int jj = 0; jj < JO; ++jj) {
                float a, Sj;
                bool e;
                if constexpr (YS == 2) {
                    a = hB ? acc[2 + jj] : acc[jj];
                    Sj = hB ? S[2 + jj] : S[jj];
                    e = hB ? empty[2 + jj] : empty[jj];
                } else {
                    static_assert(YS == 2 || YS == 4, "phase-B slice");
                    a = hB == 0 ? acc[0] : hB == 1 ? acc[1] : hB == 2 ? acc[2] : acc[3];
                    Sj = hB == 0 ? S[0] : hB == 1 ? S[1] : hB == 2 ? S[2] : S[3];
                    e = hB == 0 ? empty[0] : hB == 1 ? empty[1] : hB == 2 ? empty[2] : empty[3];
                }
                const int j = hB * JO + jj;
                float2 u = make_float2(-INFINITY, 0.f);
                if (!e && a > 1e-37f) {
                    float lh, ll;
                    if (a >= 0.25f && a <= 4.0f) {
                        // the common (speculative) case: lg2.approx is within ~1e-7 here
                        const float l2 = lg2f(a);
                        lh = gridq(l2 * kLN2, gq);
                        ll = fmaf(-lh, kL2E, l2);
                    } else {
                        ln_split(a, gq, lh, ll);
                    }
                    u = make_float2(Sj + lh, ll);
                    if (!(fabsf(u.x) < 1e30f)) nonfinite = 1;
                }
                bcast<CS>(&L.Ut[(x2b + j) * d.pU + y1B], u);
            }
        }
#else
        if (hB == 0 && rvalid && qvalid) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 u = make_float2(-INFINITY, 0.f);
                if (!empty[j] && acc[j] > 1e-37f) {
                    float lh, ll;
                    if (acc[j] >= 0.25f && acc[j] <= 4.0f) {
                        // the common (speculative) case: lg2.approx is within ~1e-7 here
                        const float l2 = lg2f(acc[j]);
                        lh = gridq(l2 * kLN2, gq);
                        ll = fmaf(-lh, kL2E, l2);
                    } else {
                        ln_split(acc[j], gq, lh, ll);
                    }
                    u = make_float2(S[j] + lh, ll);
                    if (!(fabsf(u.x) < 1e30f)) nonfinite = 1;
                }
                bcast<CS>(&L.Ut[(x2b + j) * d.pU + y1B], u);
            }
        }
#endif
    }
}


// BIG: the first Y half-pass T(x1, y2) = LSE_x2[F(x1, x2) - C(x2 - y2)].
// Work units (32-column chunk, x1 pair) round-robin over warps (balanced:
// #units is a multiple of a_r/2); lane <-> y2; the F row pair is read as
// broadcast 128-bit loads from the hi/lo planes, the per-lane cost pair
// (C(x2 - y2), C(x2 + 1 - y2)) from CP; speculative stabiliser = previous T
// (exact two-pass on the first iteration or when the window check fails).
template <int NT, int CS>
__device__ void y1_big(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all, int& fallbacks,
                       int& nonfinite) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int npair = d.ar >> 1;
    const int nchunks = (d.bc + 31) >> 5;
    const int nunits = nchunks * npair;
    const float2 L2E2 = make_float2(kL2E, kL2E);
    const int rank = CS > 1 ? (int)cluster_rank() : 0;
    for (int u = warp * CS + rank; u < nunits; u += CS * (NT / 32)) {
        const int c = u / npair, pr = u % npair;
        const int y2 = 32 * c + lane;
        const bool vy = y2 < d.bc;
        const int y2c = vy ? y2 : d.bc - 1;
        const int x1 = 2 * pr;
        float2* Tc = L.Tt + y2c * d.pT;
        const float2* cpp = L.CP + d.off + y2c;           // cpp[-x2] = (C(x2 - y2), C(x2 + 1 - y2))
        const float* fh0 = L.FH + x1 * d.ac;
        const float* fh1 = fh0 + d.ac;
        const float* fl0 = L.FL + x1 * d.ac;
        const float* fl1 = fl0 + d.ac;
        float S0, S1;
        bool exact = exact_all;
        if (!exact) {
            S0 = Tc[x1].x;
            S1 = Tc[x1 + 1].x;
            exact = !(fabsf(S0) < 1e30f) || !(fabsf(S1) < 1e30f);
        }
        float s0 = 0.f, s1 = 0.f;
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (exact) {
                float M0 = -INFINITY, M1 = -INFINITY;
                for (int x2 = 0; x2 < d.ac; x2 += 2) {
                    const float2 cp = cpp[-x2];
                    const float2 a = __fadd2_rn(*reinterpret_cast<const float2*>(fh0 + x2), neg2(cp));
                    const float2 b = __fadd2_rn(*reinterpret_cast<const float2*>(fh1 + x2), neg2(cp));
                    M0 = fmax3f(M0, a.x, a.y);
                    M1 = fmax3f(M1, b.x, b.y);
                }
                S0 = M0 > -INFINITY ? M0 : 0.f;
                S1 = M1 > -INFINITY ? M1 : 0.f;
            }
            float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
            const float2 nS0 = make_float2(-S0, -S0), nS1 = make_float2(-S1, -S1);
#pragma unroll 2
            for (int x2 = 0; x2 < d.ac; x2 += 4) {
                const float4 h0 = *reinterpret_cast<const float4*>(fh0 + x2);
                const float4 h1 = *reinterpret_cast<const float4*>(fh1 + x2);
                const float4 l0 = *reinterpret_cast<const float4*>(fl0 + x2);
                const float4 l1 = *reinterpret_cast<const float4*>(fl1 + x2);
                const float2 cpa = cpp[-x2], cpb = cpp[-x2 - 2];
                float2 t;
                t = __ffma2_rn(__fadd2_rn(__fadd2_rn(make_float2(h0.x, h0.y), neg2(cpa)), nS0), L2E2, make_float2(l0.x, l0.y));
                a0 = __fadd2_rn(a0, make_float2(ex2f(t.x), ex2f(t.y)));
                t = __ffma2_rn(__fadd2_rn(__fadd2_rn(make_float2(h0.z, h0.w), neg2(cpb)), nS0), L2E2, make_float2(l0.z, l0.w));
                a0 = __fadd2_rn(a0, make_float2(ex2f(t.x), ex2f(t.y)));
                t = __ffma2_rn(__fadd2_rn(__fadd2_rn(make_float2(h1.x, h1.y), neg2(cpa)), nS1), L2E2, make_float2(l1.x, l1.y));
                a1 = __fadd2_rn(a1, make_float2(ex2f(t.x), ex2f(t.y)));
                t = __ffma2_rn(__fadd2_rn(__fadd2_rn(make_float2(h1.z, h1.w), neg2(cpb)), nS1), L2E2, make_float2(l1.z, l1.w));
                a1 = __fadd2_rn(a1, make_float2(ex2f(t.x), ex2f(t.y)));
            }
            s0 = a0.x + a0.y;
            s1 = a1.x + a1.y;
            if (exact) break;
            const bool ok = (s0 >= 0.25f && s0 <= 4.0f) && (s1 >= 0.25f && s1 <= 4.0f);
            if (ok) break;
            exact = true;
            ++fallbacks;
        }
        if (vy) {
            float2 t0 = make_float2(-INFINITY, 0.f), t1 = make_float2(-INFINITY, 0.f);
            if (s0 > 1e-37f) {
                const float l2 = lg2f(s0);
                const float lh = gridq(l2 * kLN2, gq);
                t0 = make_float2(S0 + lh, fmaf(-lh, kL2E, l2));
                if (!(fabsf(t0.x) < 1e30f)) nonfinite = 1;
            }
            if (s1 > 1e-37f) {
                const float l2 = lg2f(s1);
                const float lh = gridq(l2 * kLN2, gq);
                t1 = make_float2(S1 + lh, fmaf(-lh, kL2E, l2));
                if (!(fabsf(t1.x) < 1e30f)) nonfinite = 1;
            }
            bcast<CS>(&Tc[x1], t0);
            bcast<CS>(&Tc[x1 + 1], t1);
        }
    }
}

// BIG: the X2 half-pass and the X-iteration's finalisation, after the
// block (cluster) barrier of the fused pass:
//   F_new(x1, x2) = log mu - (S + ln sum_y1 exp(U(y1, x2) - C(y1 - x1) - S))
// with the speculative stabiliser S = LM - F (the previous X2 LSE).  A task
// is (x1 pair, x2); P = 4 threads split its rows (fixed ranges, xor-tree
// combine) whatever the CTA shape or cluster size, so the big-cell path's
// result does not depend on either (tiers 1, 2 and the cluster tier agree
// bit for bit).  Tasks go round-robin over the cluster's CTAs; per row one
// LDS.64 of U and one of the cost pair feed two exps.  An output whose sum
// leaves [1/4, 4] is recomputed with an exact max over y1.  Each output's
// term of the L1 X-error of the plan (F, G) goes to errv[x] (summed in a
// fixed order by err_sum after the barrier).
template <int CS>
__device__ __forceinline__ void x2_out(const K1Lay& L, const Dims& d, const Grid& gq, int h, int x1a, int x2,
                                       float2 lm0, float2 lm1, float2 fo0, float2 fo1, float S0, float S1,
                                       float2 a, const float2* __restrict__ Ur, float2* Fout,
                                       int& fallbacks, int& nonfinite);
// P threads per task (x1 pair, x2) split the y1 range in P fixed parts.  P is
// a constant (never the CTA shape), so every tier gives the same bits.
// Measured (profiles/r02/ab_x2_p4.log): P = 4 for the tier-2 cells (b_r > 120,
// 512 of 768 threads busy instead of 256) was 1.3-1.7 % SLOWER on cfg 5 than
// P = 2 everywhere, and P = 4 in tier 1 (two task rounds) 4 % slower.
#ifndef DD_X2P
#define DD_X2P 2
#endif
template <int NT, int CS, int P = DD_X2P>
__device__ void x2_finalize(const K1Lay& L, const Dims& d, const Grid& gq, const float2* Fcur, float2* Fout,
                            int& fallbacks, int& nonfinite) {
    constexpr int SLOTS = NT / P;          // task slots per CTA
    static_assert(NT % (32 * P) == 0 && (P == 2 || P == 4), "x2 split");
    const int rank = CS > 1 ? (int)cluster_rank() : 0;
    if (threadIdx.x == 0 && rank == 0) L.WK[0] = 0;     // row-group counter of the next fused pass
    const int ntask = (d.ar >> 1) * d.ac;
    const int h = threadIdx.x % P;
    const int R = (d.br + P - 1) / P;
    const float2 L2E2 = make_float2(kL2E, kL2E);
    for (int base = 0; base < ntask; base += CS * SLOTS) {
        const int t = base + (threadIdx.x / P) * CS + rank;
        const bool tv = t < ntask;
        const int x2 = tv ? t % d.ac : 0, x1a = tv ? 2 * (t / d.ac) : 0;
        const float2 lm0 = L.LM[x1a * d.ac + x2], lm1 = L.LM[(x1a + 1) * d.ac + x2];
        const float2 fo0 = Fcur[x1a * d.pX + x2], fo1 = Fcur[(x1a + 1) * d.pX + x2];
        const float S0 = (fo0.x > -INFINITY && lm0.x > -INFINITY) ? lm0.x - fo0.x : 0.f;
        const float S1 = (fo1.x > -INFINITY && lm1.x > -INFINITY) ? lm1.x - fo1.x : 0.f;
        const int ya = tv ? min(h * R, d.br) : 0, yb = tv ? min(ya + R, d.br) : 0;
        const float2* __restrict__ Ur = L.Ut + x2 * d.pU;
        const float2* __restrict__ cpr = L.CP + d.off - x1a;     // cpr[y1] = (C(x1a - y1), C(x1a + 1 - y1))
        const float2 nS = make_float2(-S0, -S1);
        float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
        auto row = [&](int yy, float2& acc) {
            const float2 u = Ur[yy], c = cpr[yy];
            float2 tt = __fadd2_rn(__fadd2_rn(make_float2(u.x, u.x), neg2(c)), nS);   // exact (hi grid)
            tt = __ffma2_rn(tt, L2E2, make_float2(u.y, u.y));
            acc = __fadd2_rn(acc, make_float2(ex2f(tt.x), ex2f(tt.y)));
        };
        int y = ya;
        for (; y + 4 <= yb; y += 4) {
            row(y, a); row(y + 1, b); row(y + 2, a); row(y + 3, b);
        }
        for (; y < yb; ++y) row(y, a);
        a = __fadd2_rn(a, b);
#pragma unroll
        for (int o = 1; o < P; o <<= 1) {
            a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
            a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        }
        // lane h < 2 finalises output (x1a + h, x2)
        if (tv && h < 2)
            x2_out<CS>(L, d, gq, h, x1a, x2, lm0, lm1, fo0, fo1, S0, S1, a, Ur, Fout, fallbacks, nonfinite);
    }
}

template <int CS>
__device__ __forceinline__ void x2_out(const K1Lay& L, const Dims& d, const Grid& gq, int h, int x1a, int x2,
                                       float2 lm0, float2 lm1, float2 fo0, float2 fo1, float S0, float S1,
                                       float2 a, const float2* __restrict__ Ur, float2* Fout,
                                       int& fallbacks, int& nonfinite) {
    const int x1 = x1a + h, o = x1 * d.ac + x2;
    const float2 lm = h ? lm1 : lm0;
    const float2 fo = h ? fo1 : fo0;
    float2* fp = &Fout[x1 * d.pX + x2];
    if (lm.x == -INFINITY) {
        bcast<CS>(fp, make_float2(-INFINITY, 0.f));
        bcast<CS>(&L.FH[o], -INFINITY);
        bcast<CS>(&L.FL[o], 0.f);
        bcast<CS>(&L.errv[o], 0.0);
        return;
    }
    float S = h ? S1 : S0;
    float s = h ? a.y : a.x;
    if (!(s >= 0.25f && s <= 4.0f)) {
        // exact recompute over y1 of U(y1, x2) - C(y1 - x1)
        const float* ctp = L.CT + d.off - x1;        // C(y1 - x1) = ctp[y1]
        float M = -INFINITY;
        for (int yy = 0; yy < d.br; ++yy) M = fmaxf(M, Ur[yy].x - ctp[yy]);
        s = 0.f;
        if (M > -INFINITY)
            for (int yy = 0; yy < d.br; ++yy) {
                const float2 u = Ur[yy];
                s += ex2f(((u.x - ctp[yy]) - M) * kL2E + u.y);
            }
        S = M;
        ++fallbacks;
    }
    if (!(s > 1e-37f) || !(S > -INFINITY)) {
        nonfinite = 1;
        bcast<CS>(fp, make_float2(-INFINITY, 0.f));
        bcast<CS>(&L.FH[o], -INFINITY);
        bcast<CS>(&L.FL[o], 0.f);
        bcast<CS>(&L.errv[o], 0.0);
        return;
    }
    float lh, ll;
    ln_split(s, gq, lh, ll);
    const float2 fn = make_float2(lm.x - (S + lh), lm.y - ll);
    bcast<CS>(fp, fn);
    bcast<CS>(&L.FH[o], fn.x);
    bcast<CS>(&L.FL[o], fn.y);
    if (!(fabsf(fn.x) < 1e30f)) nonfinite = 1;
    // P_X pi(x) = mu(x) exp(F - F_new)  (plan (F, G))
    const float dF = (fo.x - fn.x) + (fo.y - fn.y) * kLN2;
    bcast<CS>(&L.errv[o], (double)L.MU[o] * (double)fabsf(expm1f(dF)));
}

// Fixed-order sum of the per-output X-error terms (every warp computes it;
// the xor butterfly gives identical bits in every lane, warp and CTA).
__device__ __forceinline__ double err_sum(const double* ev, int n) {
    double v = 0.0;
    for (int k = threadIdx.x & 31; k < n; k += 32) v += ev[k];
    return warp_sum(v);
}

template <int NT, int CS>
__device__ void fused_dispatch(const K1Lay& L, const Dims& d, const Grid& gq, bool exact_all,
                               const float2* LNUg, float* SLg, int& fb, int& nf) {
    // row groups of RG = 4 (measured: RG = 2 loses more to per-group overhead
    // than it gains in last-round balance; RG = 8 the reverse)
    if (d.ar > 8) {
        if (d.ac > 8) fused_y2x1<NT, 16, 4, 4, CS>(L, d, gq, exact_all, LNUg, SLg, fb, nf);
        else fused_y2x1<NT, 16, 2, 4, CS>(L, d, gq, exact_all, LNUg, SLg, fb, nf);
    } else {
        if (d.ac > 8) fused_y2x1<NT, 8, 4, 4, CS>(L, d, gq, exact_all, LNUg, SLg, fb, nf);
        else fused_y2x1<NT, 8, 2, 4, CS>(L, d, gq, exact_all, LNUg, SLg, fb, nf);
    }
}

// BIG: the extraction's exact Y-iteration partial sums per basic-cell
// quadrant (x1 half, x2 half via the split weights W[y2][x1] of PY1S),
// one output y per thread, written to the global ACC slice.
template <int NT>
__device__ void final_split_big(const K1Lay& L, const Dims& d, float4* __restrict__ ACCg) {
    const int ny = d.br * d.bc;
    const int ks = min(d.s, d.ar);
    for (int y = threadIdx.x; y < ny; y += NT) {
        const int y1 = y / d.bc, y2 = y % d.bc;
        const float2* Tc = L.Tt + y2 * d.pT;
        const float2* Wc = L.Ut + y2 * d.pT;
        const float* ctp = L.CT + d.off - y1;      // C(x1 - y1) = ctp[x1]
        float M = -INFINITY;
        for (int x = 0; x < d.ar; ++x) M = fmaxf(M, Tc[x].x - ctp[x]);
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (M > -INFINITY) {
            for (int x = 0; x < d.ar; ++x) {
                const float2 t = Tc[x];
                const float e = ex2f(((t.x - ctp[x]) - M) * kL2E + t.y);
                const float2 w = Wc[x];
                if (x < ks) { q.x = fmaf(e, w.x, q.x); q.y = fmaf(e, w.y, q.y); }
                else { q.z = fmaf(e, w.x, q.z); q.w = fmaf(e, w.y, q.w); }
            }
        }
        ACCg[y] = q;
    }
}

// ------------------------------------------------------- fp64 rescue --
// A cell whose fp32 X-error stalls just above its tolerance (measured: the
// error floor of the fp32 passes can reach ~1.04 ||mu_J|| Err on cells of
// tiny mass next to the image border, where the fp64 oracle converges in a
// few hundred iterations) continues from its current potentials with the
// same four separable log-domain passes in fp64 (exact max stabilisers,
// libm exp/log) until err <= tol.  Every output is computed by one thread
// of a fixed set of 256 (NT-independent, deterministic); Y potentials and
// log nu_cell in fp64 live in G64 / LNU64.  Returns the iterations done;
// F holds the plan's F (F_old of the last iteration) as fp64 on return.
// (the paper's safeguard for cells the fast
// solver cannot finish is Sec. 7.3.)
constexpr int kRescueIters = 2048;

// Per-axis cost in eps units for a LOCAL index difference e of a pass, by
// table t (0 row+: e = x1 - y1, 1 row-: e = y1 - x1, 2 col+: e = x2 - y2,
// 3 col-: e = y2 - x2): the global pixel difference is +-e + D (D = X-box
// origin - Y-box origin).  Quadratic: e^2 / kappa in the shifted gauge
// (DESIGN.md), symmetric, so t does not matter.  General (dd_set_cost,
// P:1528): h1 (rows) / h2 (columns) at |+-e + D| * hst finest pixels.
struct CostF {
    double ik, ie;
    const double* h1;
    const double* h2;
    int hst, side, Dr, Dc;
    __device__ double operator()(int t, int e) const {
        if (!h1) { const double v = (double)e; return v * v * ik; }
        int g = (t & 1) ? -e : e;
        g += (t < 2) ? Dr : Dc;
        g = min(abs(g), side - 1);
        return ((t < 2) ? h1 : h2)[(long long)g * hst] * ie;
    }
};

template <int NT>
__device__ int rescue_fp64(const K1Lay& L, const Dims& d, double* F, double* Fn, double* G64, int gstr,
                           const double* LNU64, int lstr, const CostF& cf, double tol, int max_it, double& err) {
    constexpr int NR = 256;
    const int tid = threadIdx.x;
    const bool act = tid < NR;
    double* T = reinterpret_cast<double*>(L.Tt);     // [y2][pT]
    double* U = reinterpret_cast<double*>(L.Ut);     // [x2][pU]
    int n = 0;
    while (true) {
        // Y1: T(x1, y2) = LSE_x2 [F(x1, x2) - C(x2 - y2)]
        for (int o = tid; act && o < d.ar * d.bc; o += NR) {
            const int x1 = o % d.ar, y2 = o / d.ar;
            const double* Fr = F + x1 * d.pX;
            double M = -INFINITY;
            for (int x2 = 0; x2 < d.ac; ++x2) M = fmax(M, Fr[x2] - cf(2, x2 - y2));
            double sm = 0.0;
            if (M > -INFINITY)
                for (int x2 = 0; x2 < d.ac; ++x2) sm += exp(Fr[x2] - cf(2, x2 - y2) - M);
            T[y2 * d.pT + x1] = M > -INFINITY ? M + log(sm) : -INFINITY;
        }
        __syncthreads();
        // Y2: G(y1, y2) = log nu_cell - LSE_x1 [T(x1, y2) - C(x1 - y1)]
        for (int o = tid; act && o < d.br * d.bc; o += NR) {
            const int y1 = o / d.bc, y2 = o % d.bc;
            const double ln = LNU64[(size_t)o * lstr];
            double g = -INFINITY;
            if (ln > -INFINITY) {
                const double* Tc = T + y2 * d.pT;
                double M = -INFINITY;
                for (int x1 = 0; x1 < d.ar; ++x1) M = fmax(M, Tc[x1] - cf(0, x1 - y1));
                double sm = 0.0;
                for (int x1 = 0; x1 < d.ar; ++x1) sm += exp(Tc[x1] - cf(0, x1 - y1) - M);
                g = ln - (M + log(sm));
            }
            G64[(size_t)o * gstr] = g;
        }
        __syncthreads();
        // X1: U(y1, x2) = LSE_y2 [G(y1, y2) - C(y2 - x2)]
        for (int o = tid; act && o < d.br * d.ac; o += NR) {
            const int y1 = o % d.br, x2 = o / d.br;
            const double* Gr = G64 + (size_t)y1 * d.bc * gstr;
            double M = -INFINITY;
            for (int y2 = 0; y2 < d.bc; ++y2) M = fmax(M, Gr[(size_t)y2 * gstr] - cf(3, y2 - x2));
            double sm = 0.0;
            if (M > -INFINITY)
                for (int y2 = 0; y2 < d.bc; ++y2) sm += exp(Gr[(size_t)y2 * gstr] - cf(3, y2 - x2) - M);
            U[x2 * d.pU + y1] = M > -INFINITY ? M + log(sm) : -INFINITY;
        }
        __syncthreads();
        // X2: F_new = log mu - LSE_y1 [U(y1, x2) - C(y1 - x1)]; X-error of the plan (F, G)
        for (int o = tid; act && o < d.ar * d.ac; o += NR) {
            const int x1 = o / d.ac, x2 = o % d.ac;
            const float2 lmf = L.LM[o];
            const double lm = lmf.x == -INFINITY ? -INFINITY : join_hl(lmf);
            double fn = -INFINITY, e = 0.0;
            if (lm > -INFINITY) {
                const double* Ur = U + x2 * d.pU;
                double M = -INFINITY;
                for (int y1 = 0; y1 < d.br; ++y1) M = fmax(M, Ur[y1] - cf(1, y1 - x1));
                double sm = 0.0;
                if (M > -INFINITY)
                    for (int y1 = 0; y1 < d.br; ++y1) sm += exp(Ur[y1] - cf(1, y1 - x1) - M);
                fn = M > -INFINITY ? lm - (M + log(sm)) : -INFINITY;
                const double f = F[x1 * d.pX + x2];
                e = (fn > -INFINITY && f > -INFINITY) ? (double)L.MU[o] * fabs(expm1(f - fn)) : 0.0;
            }
            Fn[x1 * d.pX + x2] = fn;
            L.errv[o] = e;
        }
        __syncthreads();
        err = err_sum(L.errv, d.ar * d.ac);
        ++n;
        if (err <= tol || n >= max_it || !(err == err)) break;
        __syncthreads();      // every warp has read errv before the next X2 writes it
        double* t = F; F = Fn; Fn = t;
    }
    // the plan's F (F_old) into the first buffer for the caller
    if (n % 2 == 0) {
        for (int o = tid; o < d.ar * d.ac; o += NT) {
            const int i = (o / d.ac) * d.pX + o % d.ac;
            Fn[i] = F[i];
        }
        __syncthreads();
    }
    return n;
}

// ----------------------------------------------------------- the solve --
// CS > 1 (cluster tier, BIG only): the CS CTAs of a cluster solve the cell
// together: each keeps a replica of the SMEM state,
// Y1 units, fused row groups and X2 tasks are dealt over the cluster and
// every output is stored to all replicas (DSMEM); three cluster barriers per
// iteration.  Rank 0 alone runs the extraction and the epilogue.  gslice is
// the cluster's (shared) global slice.
template <int NT, bool BIG, int CS, bool GC, bool GM>
__device__ void solve_cell(const SweepParams& p, int cell, unsigned char* base, unsigned char* gslice,
                           unsigned& tma_phase) {
    static_assert(CS == 1 || BIG, "cluster tier = big-cell path");
    static_assert(!(GC && BIG), "general costs run on the SMEM tier only");
    // general costs (dd_set_cost) run on the SMEM tier only (DESIGN.md "general
    // costs"): a separate kernel instantiation, so the quadratic kernels carry no
    // general-cost code
    constexpr bool gc = GC;
    const K1Lay L = k1_carve(base, p.s, p.bcap, BIG, NT / 32, gc);
    const int rank = CS > 1 ? (int)cluster_rank() : 0;
    __shared__ int4 s_box[4];
    __shared__ long long s_off[4];
    __shared__ int s_q[4];          // quadrant of each member
    __shared__ int s_mem[4];        // basic cell index of each member
    __shared__ long long s_newoff[4];
    __shared__ int4 s_newbox[4];
    __shared__ double s_bal[8];
    __shared__ int s_flag;
    __shared__ int s_ired[(NT / 32) * 16];

    const int tid = threadIdx.x;
    const int cp = cell / p.nca, cq = cell % p.nca;
    int rlo, rhi, clo, chi;
    cell_span(p.nb, p.part, cp, rlo, rhi);
    cell_span(p.nb, p.part, cq, clo, chi);
    const int ncol = chi - clo + 1;
    const int nmem = (rhi - rlo + 1) * ncol;
    if (tid < nmem) {
        const int r = rlo + tid / ncol, c = clo + tid % ncol;
        const int i = r * p.nb + c;
        s_mem[tid] = i;
        s_q[tid] = (r - rlo) * 2 + (c - clo);
        s_box[tid] = p.box[i];
        s_off[tid] = p.off[i];
    }
    if (tid == 0) s_flag = 0;
    __syncthreads();

    Dims d;
    d.s = p.s;
    d.ar = (rhi - rlo + 1) * p.s;
    d.ac = ncol * p.s;
    const int R0 = rlo * p.s, C0 = clo * p.s;
    int y0 = 1 << 30, x0 = 1 << 30, y1 = -1, x1 = -1;
    for (int m = 0; m < nmem; ++m) {
        const int4 b = s_box[m];
        if (b.z <= 0 || b.w <= 0) continue;
        y0 = min(y0, b.x); x0 = min(x0, b.y);
        y1 = max(y1, b.x + b.z - 1); x1 = max(x1, b.y + b.w - 1);
    }
    d.br = y1 >= 0 ? y1 - y0 + 1 : 0;
    d.bc = x1 >= 0 ? x1 - x0 + 1 : 0;
    const int Y0 = y0, X0 = x0;
    CellOut co;
    co.iters = 0; co.flags = 0; co.err = 0.f; co.box = max(d.br, d.bc); co.mufu = 0.0;
    co.fallbacks = 0; co.pad = 0;
    const long long t_start = clock64();

    // BIG: solve in the transposed frame when the box is wider than tall, so
    // the fused Y2+X1 pass (parallel over Y rows) always runs over the longer
    // side (warp balance).  Local (r, c) = global (c, r); the MUFU work is
    // the same in both orientations.
    const bool tr = BIG && (d.bc > d.br);
    if (tr) {
        const int t1 = d.ar; d.ar = d.ac; d.ac = t1;
        const int t2 = d.br; d.br = d.bc; d.bc = t2;
    }
    // local <-> global offsets inside the X and Y boxes
    auto goff = [tr](int r, int c, int& gr, int& gc) { if (tr) { gr = c; gc = r; } else { gr = r; gc = c; } };
    auto qloc = [tr](int q) { return tr ? (((q & 1) << 1) | (q >> 1)) : q; };   // member quadrant, local frame
    if (d.br > p.bcap || d.bc > p.bcap || d.br == 0 || (BIG && (d.ac % 4 != 0 || d.ar > 16 || d.ac > 16)) ||
        (BIG && p.h1 != nullptr)) {
        if (tid == 0) {
            co.flags = 2;   // misrouted (tier classification) or empty support
            atomicOr(p.overflow, 2);
            p.out[cell] = co;
        }
        return;
    }
    d.pX = odd_pitch(d.ac); d.pT = odd_pitch(d.ar); d.pG = odd_pitch(d.bc); d.pU = odd_pitch(d.br);
    d.off = k1_ct_off(p.s, p.bcap);
    const int Dr = R0 - Y0, Dc = C0 - X0;          // local-frame offsets (DESIGN.md gauge)
    const double inv_kappa = 1.0 / p.kappa;
    const double inv_eps = 1.0 / p.eps;
    CostF cf;
    cf.ik = inv_kappa; cf.ie = inv_eps; cf.h1 = gc ? p.h1 : nullptr; cf.h2 = p.h2; cf.hst = p.hst;
    cf.side = p.side; cf.Dr = Dr; cf.Dc = Dc;

    // ---- cost table (exact for kappa = 2^k)
    for (int i = tid; i < 2 * d.off + 1; i += NT) {
        const double dd = (double)(i - d.off);
        L.CT[i] = (float)(dd * dd * inv_kappa);
    }
    if (BIG) {
        for (int i = tid; i < 2 * d.off + 1; i += NT) {
            const double a = (double)(i - d.off), b = (double)(i - 1 - d.off);
            L.CP[i] = make_float2((float)(a * a * inv_kappa), (float)(b * b * inv_kappa));
        }
    }
    // ---- X side: F = alpha/eps + log mu - shift(x~) - lambda (local affine gauge)
    const int nx = d.ar * d.ac;
    // ---- stage the X side in shared memory by the bulk-copy engine (TMA,
    // north_star): alpha, mu and log mu of the cell's a_r x a_c pixels, one
    // cp.async.bulk per image row and array (a_c * 8 bytes, 16-B aligned since
    // s >= 2), issued by one thread, completion on the CTA's mbarrier.  The
    // staging area is scratch the solve writes only later (BIG: Tt/Ut; SMEM
    // tier: G/LNU).  Tier G's layout is in global memory: direct loads there.
    const double* xA = p.alpha;
    const double* xM = p.mu;
    const double* xL = p.logmu;
    long long xbase = (long long)R0 * p.side + C0, xstr = p.side;     // (xr, xc) -> xbase + xr xstr + xc
    bool staged = false;
    if constexpr (!GM) {
        const int arg = (rhi - rlo + 1) * p.s, acg = ncol * p.s;        // the global (untransposed) frame
        double* stage = reinterpret_cast<double*>(BIG ? reinterpret_cast<unsigned char*>(L.Tt)
                                                      : reinterpret_cast<unsigned char*>(L.G));
        const unsigned need = 3u * (unsigned)nx * 8u;
        if ((size_t)need <= (size_t)(reinterpret_cast<unsigned char*>(L.CT) - reinterpret_cast<unsigned char*>(stage))) {
            const unsigned mb = smem_u32(&g_k1_mbar);
            if (tid == 0) {
                fence_proxy_async_smem();     // the previous cell's generic accesses of the area first
                mbar_expect_tx(mb, need);
                for (int r = 0; r < arg; ++r) {
                    const long long g = (long long)(R0 + r) * p.side + C0;
                    bulk_g2s(smem_u32(stage + r * acg), p.alpha + g, acg * 8, mb);
                    bulk_g2s(smem_u32(stage + nx + r * acg), p.mu + g, acg * 8, mb);
                    bulk_g2s(smem_u32(stage + 2 * nx + r * acg), p.logmu + g, acg * 8, mb);
                }
            }
            while (!mbar_try_wait(mb, tma_phase)) {}
            tma_phase ^= 1u;
            xA = stage; xM = stage + nx; xL = stage + 2 * nx;
            xbase = 0; xstr = acg;
            staged = true;
        }
    }
    double fmax_l = -INFINITY, fmin_l = INFINITY, muJ = 0.0;
    for (int x = tid; x < nx; x += NT) {
        int xr, xc;
        goff(x / d.ac, x % d.ac, xr, xc);
        const long long g = xbase + (long long)xr * xstr + xc;
        const double m = xM[g];
        muJ += m;
        if (m > 0.0) {
            const double sh = gc ? 0.0 : ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            const double F = xA[g] * inv_eps + xL[g] - sh;
            fmax_l = fmax(fmax_l, F);
            fmin_l = fmin(fmin_l, F);
        }
    }
    const double lambda = block_max(fmax_l, L.red);
    const double fmin_b = -block_max(-fmin_l, L.red + 16);
    const double frange = (lambda > fmin_b) ? lambda - fmin_b : 0.0;
    if (BIG) {
        // ||mu_J|| in a fixed order (one warp), so that the stop tolerance of
        // the big-cell path does not depend on the CTA shape
        if (tid < 32) {
            double v = 0.0;
            for (int x = tid; x < nx; x += 32) {
                int xr, xc;
                goff(x / d.ac, x % d.ac, xr, xc);
                v += xM[xbase + (long long)xr * xstr + xc];
            }
            v = warp_sum(v);
            if (tid == 0) L.red[60] = v;
        }
        __syncthreads();
        muJ = L.red[60];
    } else {
        muJ = block_sum(muJ, L.red + 32);
    }
    // ---- per-cell hi grid: magnitudes bounded by M = 2 Cmax + 2 |F| + 64
    Grid gq;
    {
        const double dmax = (double)max(d.ar + d.br, d.ac + d.bc);
        double cmax = dmax * dmax * inv_kappa;
        if (gc) {     // the largest entry of the cell's four general-cost tables
            double cm = 0.0;
            for (int i = tid; i < 4 * (2 * d.off + 1); i += NT) cm = fmax(cm, cf(i / (2 * d.off + 1), i % (2 * d.off + 1) - d.off));
            cmax = block_max(cm, L.red);
        }
        const double M = 2.0 * cmax + 2.0 * frange + 64.0;
        int q = 8;
        while (q > -4 && ldexp(M, q) >= 4194304.0) --q;      // 2 M 2^q < 2^23
        gq.magic = (float)ldexp(1.5, 23 - q);
        gq.scale = ldexp(1.0, q);
        gq.inv = ldexp(1.0, -q);
    }
    if (gc) {
        // general cost tables: hi on the cell grid (so hi - C - S stays exact,
        // as for the quadratic table), the remainder as lo2 joins the lo term
        const int tl = 2 * d.off + 8;
        for (int i = tid; i < 4 * tl; i += NT) {
            const int t = i / tl, k = i % tl;
            L.CG[i] = (k <= 2 * d.off) ? split_hl(cf(t, k - d.off), gq) : make_float2(0.f, 0.f);
        }
    }
    for (int x = tid; x < nx; x += NT) {
        int xr, xc;
        goff(x / d.ac, x % d.ac, xr, xc);
        const long long g = xbase + (long long)xr * xstr + xc;
        const double m = xM[g];
        float2 f = make_float2(-INFINITY, 0.f), lm = make_float2(-INFINITY, 0.f);
        if (m > 0.0) {
            const double sh = gc ? 0.0 : ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            f = split_hl(xA[g] * inv_eps + xL[g] - sh - lambda, gq);
            lm = split_hl(xL[g], gq);
        }
        L.FX[(x / d.ac) * d.pX + x % d.ac] = f;
        if (BIG) {
            L.FH[x] = f.x;
            L.FL[x] = f.y;
        }
        L.LM[x] = lm;
        L.MU[x] = (float)m;
    }
    if (!BIG && staged) __syncthreads();     // the staging area (G/LNU) is read before LNU is written
    // ---- line 8: nu_cell = sum_i nu_i on the union box; log nu_cell
    // (BIG: log nu_cell and the extraction sums live in the CTA's global slice)
    float2* LNU = BIG ? reinterpret_cast<float2*>(gslice) : L.LNU;
    const size_t b2 = (size_t)p.bcap * p.bcap;
    (void)b2;
    float* SLg = BIG ? reinterpret_cast<float*>(gslice + p.sl_off) : nullptr;
    float4* ACCp = BIG ? reinterpret_cast<float4*>(gslice + p.acc_off) : reinterpret_cast<float4*>(L.G);
    const int ny = d.br * d.bc;
    double npos = 0.0;
    for (int y = rank * NT + tid; y < ny; y += CS * NT) {
        int gy, gx;
        goff(y / d.bc, y % d.bc, gy, gx);
        gy += Y0;
        gx += X0;
        double v = 0.0;
        for (int m = 0; m < nmem; ++m) {
            const int4 b = s_box[m];
            const int ry = gy - b.x, rx = gx - b.y;
            if (ry >= 0 && ry < b.z && rx >= 0 && rx < b.w) v += p.pool_in[s_off[m] + (long long)ry * b.w + rx];
        }
        LNU[y] = (v > 0.0) ? split_hl(log(v), gq) : make_float2(-INFINITY, 0.f);
        npos += (v > 0.0) ? 1.0 : 0.0;
    }
    npos = block_sum(npos, L.red);     // (barrier: staging complete)
    if constexpr (CS > 1) {
        // the slice rows of the other CTAs; the non-zero count at rank 0
        if (tid == 0) atom_add_cl(mapa_u32(smem_u32(&L.WK[1]), 0), (int)npos);
        cluster_sync_all();
        npos = (double)L.WK[1];
    }
    if (BIG) {
        // per Y row: the non-zero columns of nu_cell.  The separable passes
        // only need those (G = -inf elsewhere); about half of a union box is
        // zero (basic-cell supports are bands inside their bounding boxes).
        const int lane = tid & 31;
        for (int r = tid >> 5; r < d.br; r += NT / 32) {
            int lo = 1 << 30, hi = -1;
            for (int c = lane; c < d.bc; c += 32)
                if (LNU[r * d.bc + c].x != -INFINITY) { lo = min(lo, c); hi = max(hi, c); }
            lo = warp_min_i(lo);
            hi = warp_max_i(hi);
            if (lane == 0) L.RI[r] = make_int2(lo, hi);
        }
        __syncthreads();
        // the 4-row groups of the fused pass, heaviest first (dynamic LPT): a
        // group costs about its 32-column chunks (phase A runs whole chunks),
        // then its non-zero span; fixed for the whole solve (nu_cell does not
        // change).  Rank sort on unique keys (group id in the low bits).
        const int ng = (d.br + 3) / 4;
        int* w = reinterpret_cast<int*>(L.gbuf);           // temp (gbuf is idle in the prologue)
        for (int g = tid; g < ng; g += NT) {
            int lo = 1 << 30, hi = -1;
            for (int r = 4 * g; r < min(4 * g + 4, d.br); ++r) { lo = min(lo, L.RI[r].x); hi = max(hi, L.RI[r].y); }
            const int len = hi >= lo ? hi - lo + 1 : 0;
            L.GI[g] = make_int2(lo, hi);
            w[g] = ((((len + 31) >> 5) * 1024 + len) << 12) | g;   // ng < 4096, len < 1024
        }
        if (tid == 0) L.WK[0] = 0;                         // group counter of the first fused pass
        __syncthreads();
        for (int g = tid; g < ng; g += NT) {
            const int v = w[g];
            int r = 0;
            for (int k = 0; k < ng; ++k) r += (w[k] > v);
            L.GL[r] = v & 0xfff;
        }
        __syncthreads();
    }

    // ---- line 9: Sinkhorn (Y-iteration first; stop test fused in the X-iteration)
    // stop at err <= (1 - 2^-7) ||mu_J|| Err: the test runs on the fp32
    // potentials; the margin keeps the fp64 re-evaluation of the plan's
    // X-error (dd_marginal_error) within P:1409's bound (A28)
    auto nucell = [&](int y) {
        int gy, gx;
        goff(y / d.bc, y % d.bc, gy, gx);
        gy += Y0;
        gx += X0;
        double v = 0.0;
        for (int m = 0; m < nmem; ++m) {
            const int4 b = s_box[m];
            const int ry = gy - b.x, rx = gx - b.y;
            if (ry >= 0 && ry < b.z && rx >= 0 && rx < b.w) v += p.pool_in[s_off[m] + (long long)ry * b.w + rx];
        }
        return v;
    };
    const double tol = muJ * p.err_tol * (1.0 - 0.0078125);
    float2* Fc = L.FX;
    float2* Fn = L.FXn;
    int it = 0, fallbacks = 0, nonfinite = 0;
    double err = 0.0;
    double err_ck = INFINITY;       // X-error at the last stall checkpoint
    bool rescue = false;
    bool safeguard = false;     // eps-raising safeguard (DD_FLAG_SAFEGUARD, A29)
    PROF_T(t_loop0);
    while (true) {
        const bool exact = (it == 0);
        double e_loc = 0.0;
        PROF_T(ta);
        if (BIG) y1_big<NT, CS>(L, d, gq, exact, fallbacks, nonfinite);
        else if (gc) lse_pass<PY1, NT, true>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        else lse_pass<PY1, NT>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        PROF_T(tb);
        cta_or_cluster_sync<CS>();
        PROF_T(tc);
        if (BIG) {
            fused_dispatch<NT, CS>(L, d, gq, exact, LNU, SLg, fallbacks, nonfinite);
        } else {
            if (gc) lse_pass<PY2, NT, true>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
            else lse_pass<PY2, NT>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
            __syncthreads();
            if (gc) lse_pass<PX1, NT, true>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
            else lse_pass<PX1, NT>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        }
        PROF_T(td);
        cta_or_cluster_sync<CS>();
        PROF_T(te);
        if (BIG) {
            x2_finalize<NT, CS>(L, d, gq, Fc, Fn, fallbacks, nonfinite);
        } else {
            if (gc) lse_pass<PX2, NT, true>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
            else lse_pass<PX2, NT>(L, d, gq, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        }
        PROF_T(tf);
        if (BIG) {
            cta_or_cluster_sync<CS>();
            err = err_sum(L.errv, nx);
        } else {
            // one barrier: the previous iteration's reads of red[] are two
            // barriers back (after Y1, after the Y2/X1 passes)
            err = block_sum1(e_loc, L.red);
        }
        PROF_T(tg);
        // per warp: busy time of the passes and barrier waits (phase profile build only)
        PROF_ADD(0, tb - ta); PROF_ADD(1, tc - tb); PROF_ADD(2, td - tc); PROF_ADD(3, te - td);
        PROF_ADD(4, tf - te); PROF_ADD(5, tg - tf);
        ++it;
        if (err <= tol && it % p.check_every == 0) break;
        if (it >= p.max_iter || !(err == err)) {
            if (p.safeguard) safeguard = true;
            else co.flags |= 1;
            break;
        }
        if (cell == p.force_cell && it >= p.force_it) { rescue = true; break; }    // DD_FORCE_RESCUE (testing)
        // stall at the fp32 error floor: < 2 % progress over 256 iterations
        // within 1.5x of the tolerance -> continue in fp64 (rescue_fp64)
        if ((it & 255) == 0) {
            if (it >= 512 && err < 1.5 * tol && err > 0.98 * err_ck) { rescue = true; break; }
            err_ck = err;
        }
        float2* t = Fc; Fc = Fn; Fn = t;
    }
    if (CS == 1 && p.safeguard) {
        // non-finite potentials (nu_cell(y) > 0 unreachable) also
        // trigger the safeguard; the retry recomputes them
        if (__syncthreads_or(nonfinite)) { safeguard = true; nonfinite = 0; }
    }
    PROF_T(t_loop1);
    PROF_ADD(6, t_loop1 - t_loop0);
    PROF_ADD(7, t_loop0 - t_start);
    int peer_fallbacks = 0;
    if constexpr (CS > 1) {
        // flags and fallback counts of the other CTAs to rank 0, which alone
        // runs the extraction and the epilogue (its replica is complete)
        const int fb = (int)block_sum((double)fallbacks, L.red + 32);
        if (rank != 0) {
            if (nonfinite) atom_or_cl(mapa_u32(smem_u32(&s_flag), 0), 2);
            if (tid == 0) atom_add_cl(mapa_u32(smem_u32(&L.WK[3]), 0), fb);
        }
        cluster_sync_all();
        if (rank != 0) return;
        peer_fallbacks = L.WK[3];
    }
    if (rescue || safeguard) {
        // fp64 continuation (rescue_fp64): potentials and Y-side arrays as fp64
        double* F64 = reinterpret_cast<double*>(Fc);
        double* Fn64 = reinterpret_cast<double*>(Fn);
        for (int x = tid; rescue && x < nx; x += NT) {
            const int i = (x / d.ac) * d.pX + x % d.ac;
            const float2 f = Fc[i];
            F64[i] = f.x == -INFINITY ? -INFINITY : join_hl(f);
        }
        double* G64;
        double* LNU64;
        int str;
        if (BIG) {
            G64 = reinterpret_cast<double*>(ACCp);
            LNU64 = G64 + 1;
            str = 2;
        } else {
            G64 = reinterpret_cast<double*>(L.G);
            LNU64 = reinterpret_cast<double*>(L.LNU);
            str = 1;
        }
        for (int y = tid; y < ny; y += NT) {
            const double v = nucell(y);
            LNU64[(size_t)y * str] = v > 0.0 ? log(v) : -INFINITY;
        }
        __syncthreads();
        double e64 = err;
        // at most kRescueIters fp64 iterations: a precision stall converges in a
        // few hundred (measured 257); a cell that is merely this slow in fp64
        // too (the oracle needs > 4e4 iterations on such cells) keeps its
        // Y-feasible plan and is flagged (reading A6)
        if (rescue) {
            const int n = rescue_fp64<NT>(L, d, F64, Fn64, G64, str, LNU64, str, cf, tol,
                                          max(1, min(kRescueIters, p.max_iter - it)), e64);
            it += n;
            err = e64;
            co.flags |= 16;                   // solved to the tolerance by the fp64 rescue
            if (!(err <= tol)) {
                if (p.safeguard) safeguard = true;
                else co.flags |= 1;
            }
        }
        if (safeguard) {
            // eps-raising safeguard ("temporarily increasing eps"; S:281,
            // S:323; A29): attempt k restarts from the cell's INPUT
            // alpha at eps_k = 2^k eps (absorbed F' = r (F0 - log mu) + log mu,
            // r = 2^-k, costs r C: alpha kept), then re-solves at eps
            // from the result, every stage to the same tolerance and cap
            bool ok = false;
            for (int k = 1; k <= 3 && !ok; ++k) {
                const double r = ldexp(1.0, -k);
                for (int x = tid; x < nx; x += NT) {
                    int xr, xc;
                    goff(x / d.ac, x % d.ac, xr, xc);
                    const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
                    double f = -INFINITY;
                    if (p.mu[g] > 0.0) {
                        const double sh = gc ? 0.0 : ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
                        const double F0 = p.alpha[g] * inv_eps + p.logmu[g] - sh - lambda;
                        f = r * (F0 - p.logmu[g]) + p.logmu[g];
                    }
                    F64[(x / d.ac) * d.pX + x % d.ac] = f;
                }
                __syncthreads();
                CostF ck = cf;
                ck.ik *= r;
                ck.ie *= r;
                double e1 = INFINITY;
                it += rescue_fp64<NT>(L, d, F64, Fn64, G64, str, LNU64, str, ck, tol, p.max_iter, e1);
                for (int x = tid; x < nx; x += NT) {
                    int xr, xc;
                    goff(x / d.ac, x % d.ac, xr, xc);
                    const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
                    const int i = (x / d.ac) * d.pX + x % d.ac;
                    if (F64[i] > -INFINITY) F64[i] = (F64[i] - p.logmu[g]) / r + p.logmu[g];
                }
                __syncthreads();
                it += rescue_fp64<NT>(L, d, F64, Fn64, G64, str, LNU64, str, cf, tol, p.max_iter, e64);
                ok = e64 <= tol;
            }
            err = e64;
            co.flags |= 32;
            if (!ok) co.flags |= 1;
        }
        for (int x = tid; x < nx; x += NT) {
            const int i = (x / d.ac) * d.pX + x % d.ac;
            const double f = F64[i];
            Fc[i] = split_hl(f, gq);
        }
        __syncthreads();
    }
    // ---- line 10: extraction from the plan (F, G): exact Y-iteration with
    // the row sums split by basic-cell quadrant (x1 half, x2 half)
    {
        double dummy = 0.0;
        // (the big-cell path: 256 threads, whatever the CTA shape)
        if (gc) lse_pass<PY1S, NT, true>(L, d, gq, true, Fc, Fn, dummy, fallbacks, nonfinite);
        else lse_pass<PY1S, BIG ? 256 : NT>(L, d, gq, true, Fc, Fn, dummy, fallbacks, nonfinite);
        __syncthreads();
        if (BIG) final_split_big<NT>(L, d, ACCp);
        else if (gc) lse_pass<PY2S, NT, true>(L, d, gq, true, Fc, Fn, dummy, fallbacks, nonfinite);
        else lse_pass<PY2S, NT>(L, d, gq, true, Fc, Fn, dummy, fallbacks, nonfinite);
    }
    if (nonfinite) atomicOr(&s_flag, 2);
    fallbacks = (int)block_sum((double)fallbacks, L.red + 32) + peer_fallbacks;
    co.flags |= s_flag;
    co.iters = it;
    if (tid == 0 && p.ipred) p.ipred[cell] = it;
    co.err = (float)err;
    co.fallbacks = fallbacks;
    {
        // algorithmic MUFU ops: one ex2 per term of the four 1D
        // passes + one log per pass output; + the extraction Y-iteration
        const double ar = d.ar, ac = d.ac, br = d.br, bc = d.bc;
        // Y1 a_r a_c b_c + Y2 a_r n_y + X1 n_y a_c + X2 a_c b_r a_r exps (terms
        // with nu_cell(y) = 0 are -inf and not algorithmic work) + one log per output
        const double per_it = ar * ac * bc + ar * npos + npos * ac + ac * br * ar
                              + ar * bc + npos + br * ac + ar * ac;
        co.mufu = per_it * it + (ar * ac * bc + ar * br * bc + ar * bc + br * bc);
    }

    // ---- epilogue (ACC over the G+LNU region; nu_cell re-gathered from pool_in)
    const float4* ACC = ACCp;
    // line 10: nu_i(y) = nu_cell(y) S_i(y) / S(y) (ratio form, A7); norms
    double nrm0 = 0.0, nrm1 = 0.0, nrm2 = 0.0, nrm3 = 0.0;
    // (the big-cell path: 256 threads in a fixed order, whatever the CTA shape)
    constexpr int NTN = BIG ? 256 : NT;
    for (int y = tid; y < ny && tid < NTN; y += NTN) {
        const float4 a = ACC[y];
        const double tot = (double)a.x + (double)a.y + (double)a.z + (double)a.w;
        if (!(tot > 0.0)) continue;
        const double sc = nucell(y) / tot;
        nrm0 += a.x * sc; nrm1 += a.y * sc; nrm2 += a.z * sc; nrm3 += a.w * sc;
    }
    nrm0 = block_sum(nrm0, L.red);
    nrm1 = block_sum(nrm1, L.red + 8);
    nrm2 = block_sum(nrm2, L.red + 16);
    nrm3 = block_sum(nrm3, L.red + 24);
    // line 11: BalanceMeasures (A8): donors give nu_i d_i/||nu_i|| T/Dsum,
    // receivers take r(y) (-d_j)/Psum, T = min(Dsum, Psum)
    if (tid == 0) {
        const double qn[4] = {nrm0, nrm1, nrm2, nrm3};
        double dsum = 0.0, psum = 0.0, dmax = 0.0, dv[4] = {0, 0, 0, 0}, nm[4] = {1, 1, 1, 1};
        for (int m = 0; m < nmem; ++m) {
            nm[m] = qn[qloc(s_q[m])];
            dv[m] = nm[m] - p.mass_i[s_mem[m]];
            dmax = fmax(dmax, fabs(dv[m]));
            if (dv[m] > 0) dsum += dv[m]; else psum += -dv[m];
        }
        const bool skip = (dmax <= 1e-18 || dsum <= 0.0 || psum <= 0.0);
        const double T = dsum < psum ? dsum : psum;
        for (int m = 0; m < 4; ++m) {
            double fd = 0.0, gr = 0.0;
            if (!skip && m < nmem) {
                if (dv[m] > 0) fd = (dv[m] / nm[m]) * (T / dsum);
                else if (dv[m] < 0) gr = -dv[m] / psum;
            }
            s_bal[2 * m] = fd;
            s_bal[2 * m + 1] = gr;
        }
    }
    __syncthreads();
    const double fd0 = s_bal[0], gr0 = s_bal[1], fd1 = s_bal[2], gr1 = s_bal[3];
    const double fd2 = s_bal[4], gr2 = s_bal[5], fd3 = s_bal[6], gr3 = s_bal[7];
    const int q0 = qloc(s_q[0]), q1 = nmem > 1 ? qloc(s_q[1]) : 0, q2 = nmem > 2 ? qloc(s_q[2]) : 0,
              q3 = nmem > 3 ? qloc(s_q[3]) : 0;
    auto pick = [](const float4& a, int qd) { return qd == 0 ? a.x : qd == 1 ? a.y : qd == 2 ? a.z : a.w; };
    // balanced value of member m at y
    auto balanced = [&](int y, int m) -> double {
        const float4 a = ACC[y];
        const double tot = (double)a.x + (double)a.y + (double)a.z + (double)a.w;
        if (!(tot > 0.0)) return 0.0;
        const double sc = nucell(y) / tot;
        const double v0 = pick(a, q0) * sc;
        const double v1 = nmem > 1 ? pick(a, q1) * sc : 0.0;
        const double v2 = nmem > 2 ? pick(a, q2) * sc : 0.0;
        const double v3 = nmem > 3 ? pick(a, q3) * sc : 0.0;
        const double r = v0 * fd0 + v1 * fd1 + v2 * fd2 + v3 * fd3;
        const double vm = m == 0 ? v0 : m == 1 ? v1 : m == 2 ? v2 : v3;
        const double fm = m == 0 ? fd0 : m == 1 ? fd1 : m == 2 ? fd2 : fd3;
        const double gm = m == 0 ? gr0 : m == 1 ? gr1 : m == 2 ? gr2 : gr3;
        return vm - vm * fm + r * gm;
    };
    // line 12: Truncate + tight bbox per member
    for (int m = 0; m < nmem; ++m) {
        int r0 = 1 << 30, r1 = -1, c0 = 1 << 30, c1 = -1;
        for (int y = tid; y < ny; y += NT) {
            const double v = balanced(y, m);
            if (v >= p.tau && v > 0.0) {
                int yr, yc;
                goff(y / d.bc, y % d.bc, yr, yc);
                r0 = min(r0, yr); r1 = max(r1, yr); c0 = min(c0, yc); c1 = max(c1, yc);
            }
        }
        r0 = warp_min_i(r0); r1 = warp_max_i(r1); c0 = warp_min_i(c0); c1 = warp_max_i(c1);
        if ((tid & 31) == 0) {
            const int w = tid >> 5;
            s_ired[(w * 4 + m) * 4 + 0] = r0; s_ired[(w * 4 + m) * 4 + 1] = r1;
            s_ired[(w * 4 + m) * 4 + 2] = c0; s_ired[(w * 4 + m) * 4 + 3] = c1;
        }
    }
    __syncthreads();
    if (tid == 0) {
        long long total = 0;
        long long area[4];
        for (int m = 0; m < nmem; ++m) {
            int r0 = 1 << 30, r1 = -1, c0 = 1 << 30, c1 = -1;
            for (int w = 0; w < NT / 32; ++w) {
                r0 = min(r0, s_ired[(w * 4 + m) * 4 + 0]); r1 = max(r1, s_ired[(w * 4 + m) * 4 + 1]);
                c0 = min(c0, s_ired[(w * 4 + m) * 4 + 2]); c1 = max(c1, s_ired[(w * 4 + m) * 4 + 3]);
            }
            const int hh = r1 >= 0 ? r1 - r0 + 1 : 0, ww = r1 >= 0 ? c1 - c0 + 1 : 0;
            s_newbox[m] = r1 >= 0 ? make_int4(Y0 + r0, X0 + c0, hh, ww) : make_int4(Y0, X0, 0, 0);
            area[m] = ((long long)hh * ww + 1) & ~1LL;       // 16-byte aligned boxes
            total += area[m];
        }
        const long long base = (long long)atomicAdd(p.bump, (unsigned long long)total);
        if (base + total > p.cap) {
            atomicOr(p.overflow, 1);
            for (int m = 0; m < nmem; ++m) s_newoff[m] = -1;
        } else {
            long long o = base;
            for (int m = 0; m < nmem; ++m) { s_newoff[m] = o; o += area[m]; }
        }
    }
    __syncthreads();
    for (int m = 0; m < nmem; ++m) {
        const int4 nb4 = s_newbox[m];
        const long long o = s_newoff[m];
        if (o < 0) continue;
        const int r0 = nb4.x - Y0, c0 = nb4.y - X0;
        const int area = nb4.z * nb4.w;
        for (int k = tid; k < area; k += NT) {
            const int gr = r0 + k / nb4.w, gc = c0 + k % nb4.w;
            const int y = tr ? gc * d.bc + gr : gr * d.bc + gc;
            const double val = balanced(y, m);
            p.scratch[o + k] = (val >= p.tau && val > 0.0) ? val : 0.0;
        }
    }
    if (tid < nmem) {
        p.box[s_mem[tid]] = s_newoff[tid] < 0 ? make_int4(Y0, X0, 0, 0) : s_newbox[tid];
        p.off[s_mem[tid]] = s_newoff[tid] < 0 ? 0 : s_newoff[tid];
    }
    // store u_{C,J}: alpha = eps (F + lambda + shift - log mu)  (plan's F, A4)
    for (int x = tid; x < nx; x += NT) {
        int xr, xc;
        goff(x / d.ac, x % d.ac, xr, xc);
        const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
        const float2 f = Fc[(x / d.ac) * d.pX + x % d.ac];
        double a = 0.0;
        if (f.x > -INFINITY && p.mu[g] > 0.0) {
            const double sh = gc ? 0.0 : ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            a = p.eps * (join_hl(f) + lambda + sh - p.logmu[g]);
        }
        p.alpha[g] = a;
    }
    if (tid == 0) {
        if (s_newoff[0] < 0) co.flags |= 8;
        co.pad = (int)min((clock64() - t_start) >> 10, (long long)0x7fffffff);   // solve time, kcycles
        PROF_ADD(8, clock64() - t_loop1);
        PROF_ADD(9, it);
        p.out[cell] = co;
    }
}

// Persistent CTAs pulling cells from a tier list (K0 classification).
// BIG = false: all per-cell arrays in SMEM (small Y boxes, 3 CTAs/SM);
// BIG = true: fused Y2+X1 path, O(a b) SMEM + a global slice per CTA;
// CS > 1: persistent clusters of CS CTAs, one cell per cluster at a time,
// one global slice per cluster.
template <int NT, bool BIG, int MINB, int CS, bool GC, bool GM>
__global__ void __launch_bounds__(NT, MINB) k1_cell_solve(SweepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_cell;
    // GM (tier G): the layout in a per-CTA global slice; otherwise shared
    // memory (a separate instantiation, so the on-chip tiers keep shared-window
    // addressing for every K1Lay array)
    unsigned char* base = GM ? p.gbase + (long long)blockIdx.x * p.gbase_bytes : smem;
    unsigned tma_phase = 0;
    if (!GM && threadIdx.x == 0) mbar_init(smem_u32(&g_k1_mbar), 1);
    const int slot = CS > 1 ? blockIdx.x / CS : blockIdx.x;
    unsigned char* gslice = BIG ? p.gscratch + (long long)slot * p.gslice : nullptr;
    if (p.poison) {     // testing: SMEM the path did not write reads as NaN
        for (size_t i = threadIdx.x; i < p.smem_bytes / 4; i += NT) reinterpret_cast<unsigned*>(smem)[i] = 0xFFFFFFFFu;
        __syncthreads();
    }
    if constexpr (CS == 1) {
        while (true) {
            if (threadIdx.x == 0) {
                const int k = atomicAdd(p.work_counter, 1);
                s_cell = (k < *p.n_in) ? p.list_in[k] : -1;
            }
            __syncthreads();
            const int cell = s_cell;
            if (cell < 0) return;
            solve_cell<NT, BIG, 1, GC, GM>(p, cell, base, gslice, tma_phase);
            __syncthreads();
        }
    } else {
        const K1Lay L = k1_carve(base, p.s, p.bcap, BIG, NT / 32);
        const unsigned rank = cluster_rank();
        while (true) {
            if (rank == 0 && threadIdx.x == 0) {
                const int k = atomicAdd(p.work_counter, 1);
                const int c = (k < *p.n_in) ? p.list_in[k] : -1;
                L.WK[1] = 0;          // the cell's cluster counters (non-zero count, fallbacks)
                L.WK[3] = 0;
                for (unsigned r = 0; r < (unsigned)CS; ++r) st_cl(mapa_u32(smem_u32(&s_cell), r), c);
            }
            cluster_sync_all();
            const int cell = s_cell;
            if (cell < 0) return;        // all CTAs of the cluster leave together
            solve_cell<NT, BIG, CS, false, false>(p, cell, base, gslice, tma_phase);
            cluster_sync_all();          // rank 0's epilogue done before the next cell's stores
        }
    }
}

// K0: route every cell of the sweep to a tier by its union Y-box side
// (tier 0 <= b0: SMEM path; tier 1 <= b1 and tier 2 (beyond): BIG path;
// cells beyond tier 2's capacity are flagged by the solve), and record the
// side for the LPT ordering of the big tiers.
__global__ void k0_classify(SweepParams p, int b0, int b1, int b2, int* lists, int* counts, int ncap, int* bside,
                            unsigned long long* wsum) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= p.ncells) return;
    const int cp = cell / p.nca, cq = cell % p.nca;
    if (cp < p.cr0 || cp >= p.cr1) {      // another rank's stripe: no solve, zero statistics
        CellOut z;
        z.iters = 0; z.flags = 0; z.err = 0.f; z.box = 0; z.mufu = 0.0; z.fallbacks = 0; z.pad = 0;
        p.out[cell] = z;
        bside[cell] = 0;
        return;
    }
    int rlo, rhi, clo, chi;
    cell_span(p.nb, p.part, cp, rlo, rhi);
    cell_span(p.nb, p.part, cq, clo, chi);
    int y0 = 1 << 30, x0 = 1 << 30, y1 = -1, x1 = -1;
    for (int r = rlo; r <= rhi; ++r)
        for (int c = clo; c <= chi; ++c) {
            const int4 b = p.box[r * p.nb + c];
            if (b.z <= 0 || b.w <= 0) continue;
            y0 = min(y0, b.x); x0 = min(x0, b.y);
            y1 = max(y1, b.x + b.z - 1); x1 = max(x1, b.y + b.w - 1);
        }
    const int bmax = y1 >= 0 ? max(y1 - y0 + 1, x1 - x0 + 1) : 0;
    const bool small_x = p.s < 4;       // the BIG path needs a_c % 4 == 0
    const int tier = bmax <= b0 ? 0 : small_x ? 3 : (bmax <= b1 ? 1 : (bmax <= b2 ? 2 : 3));
    // tier 3 here = tier G (beyond every on-chip tier): list 6, count counts[12]
    const int k = atomicAdd(&counts[tier == 3 ? 12 : tier], 1);
    lists[(tier == 3 ? 6 : tier) * ncap + k] = cell;
    // LPT key ~ predicted solve time: box area x the cell's iteration count in
    // this partition's previous sweep (1 before the first), log-binned
    const int ip = p.ipred ? max(1, p.ipred[cell]) : 1;
    const float w = (float)max(bmax, 1) * (float)max(bmax, 1) * (float)ip;
    bside[cell] = min(1023, (int)(32.f * __log2f(w)));
    atomicAdd(wsum, (unsigned long long)max(bmax, 1) * (unsigned long long)max(bmax, 1) * (unsigned long long)ip);
}

// K0c: route the long poles of the sweep to the cluster tier.  A cell whose
// predicted work w (box area x previous iterations, the K0 key) exceeds
// theta x (the sweep's total predicted work) / #SMs would run longer on one
// SM than the whole sweep takes when spread over the machine.  The big tiers'
// LPT lists are sorted by the key, so the long poles are their prefixes: the
// cluster list merges the two prefixes (largest first) and tiers 1 / 2 start
// their work counters behind them.  mode 1: every big-path cell (testing).
// The big-path result does not depend on the tier (x2_finalize), so the
// routing only affects timing.
__global__ void k0_cluster(const int* sorted, int* counts, int ncap, const int* bside,
                           const unsigned long long* wsum, float theta, int nsm, int mode, int* list3) {
    if (threadIdx.x != 0) return;
    const int n1 = counts[1], n2 = counts[2];
    const int* l1 = sorted;
    const int* l2 = sorted + ncap;
    int thr = 1 << 30;
    if (mode == 1) {
        thr = -1;
    } else {
        const double w = (double)*wsum * (double)theta / (double)nsm;
        if (w >= 1.0) thr = (int)(32.0 * log2(w));
    }
    int a = 0, b = 0;
    while (a < n1 && bside[l1[a]] >= thr) ++a;
    while (b < n2 && bside[l2[b]] >= thr) ++b;
    int i = 0, j = 0, k = 0;
    while (i < b || j < a) {      // merge, tier-2 (larger box) first on equal keys
        if (j >= a || (i < b && bside[l2[i]] >= bside[l1[j]])) list3[k++] = l2[i++];
        else list3[k++] = l1[j++];
    }
    counts[8] = k;                 // cluster tier: list length, work counter counts[9] (zeroed)
    counts[4] = a;                 // tier 1 starts behind its prefix
    counts[5] = b;                 // tier 2 likewise
}

// LPT order for the big tiers: counting sort of the tier-t list by the K0
// key (predicted work), descending: the slowest cells start first.  One
// block per tier.
__global__ void k0_sort(const int* lists, const int* counts, int ncap, const int* bside, int* sorted) {
    __shared__ int hist[1024];
    const int t = 1 + blockIdx.x;
    const int n = counts[t];
    const int* in = lists + (size_t)t * ncap;
    int* out = sorted + (size_t)blockIdx.x * ncap;
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) atomicAdd(&hist[1023 - min(bside[in[k]], 1023)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < 1024; ++k) { const int v = hist[k]; hist[k] = acc; acc += v; }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int c = in[k];
        out[atomicAdd(&hist[1023 - min(bside[c], 1023)], 1)] = c;
    }
}

// Read (and reset) the phase profile counters; zeros unless built with -DDD_PHASE_PROF.
cudaError_t k1_phase_read(unsigned long long* out32) {
#ifdef DD_PHASE_PROF
    cudaError_t e = cudaMemcpyFromSymbol(out32, g_phase, sizeof(g_phase));
    if (e != cudaSuccess) return e;
    unsigned long long z[32] = {0};
    return cudaMemcpyToSymbol(g_phase, z, sizeof(g_phase));
#else
    for (int k = 0; k < 32; ++k) out32[k] = 0;
    return cudaSuccess;
#endif
}

cudaError_t launch_k0_cluster(const int* sorted, int* counts, int ncap, const int* bside, float theta, int nsm,
                              int mode, int* list3, cudaStream_t st) {
    k0_cluster<<<1, 32, 0, st>>>(sorted, counts, ncap, bside, reinterpret_cast<const unsigned long long*>(counts + 10),
                                 theta, nsm, mode, list3);
    return cudaGetLastError();
}

size_t k1_smem_bytes_host(int s, int bcap, bool big, int nwarps, bool gc) { return k1_smem_bytes(s, bcap, big, nwarps, gc); }

cudaError_t launch_k0(const SweepParams& p, int b0, int b1, int b2, int* lists, int* counts, int ncap, int* bside,
                      int* sorted, cudaStream_t st) {
    k0_classify<<<(p.ncells + 255) / 256, 256, 0, st>>>(p, b0, b1, b2, lists, counts, ncap, bside,
                                                         reinterpret_cast<unsigned long long*>(counts + 10));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k0_sort<<<2, 1024, 0, st>>>(lists, counts, ncap, bside, sorted);
    return cudaGetLastError();
}

template <int NT, bool BIG, int MINB, int CS, bool GC = false, bool GM = false>
static cudaError_t launch_tier(const SweepParams& p, int grid, size_t smem, cudaStream_t st) {
    // the SMEM opt-in is a per-device function attribute: cache it per device
    static size_t attr[64] = {0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    // opt in whenever the request grows: the 48 KB default covers static +
    // dynamic SMEM together, so a dynamic size just under 48 KB can fail too
    if (smem > attr[dev]) {
        e = cudaFuncSetAttribute(k1_cell_solve<NT, BIG, MINB, CS, GC, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr[dev] = smem;
    }
    SweepParams q = p;
    q.smem_bytes = smem;
    if constexpr (CS == 1) {
        k1_cell_solve<NT, BIG, MINB, CS, GC, GM><<<grid, NT, smem, st>>>(q);
        return cudaGetLastError();
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid * CS);
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, k1_cell_solve<NT, BIG, MINB, CS, GC, GM>, q);
    }
}

// tier 0: 256 threads, all arrays in SMEM, 3 CTAs/SM;
// tier 1: BIG path, 256 threads, 3 CTAs/SM; tier 2: BIG path, 768 threads, 1 CTA/SM (both <= 80 registers);
// tier 3 (cluster tier): tier 2's CTA in clusters of kClusterSize, grid = number of clusters.
cudaError_t launch_k1(const SweepParams& p, int tier, int grid, size_t smem, cudaStream_t st) {
    if (tier == 0) {
        if (p.gbase) {          // tier G: the SMEM-tier kernel on global-memory layouts
            if (p.h1) return launch_tier<256, false, DD_T0_MINB, 1, true, true>(p, grid, 0, st);
            return launch_tier<256, false, DD_T0_MINB, 1, false, true>(p, grid, 0, st);
        }
        if (p.h1) return launch_tier<256, false, DD_T0_MINB, 1, true>(p, grid, smem, st);
        return launch_tier<256, false, DD_T0_MINB, 1>(p, grid, smem, st);
    }
    if (tier == 1) return launch_tier<kT1Threads, true, kT1PerSM, 1>(p, grid, smem, st);
    if (tier == 2) return launch_tier<kT2Threads, true, kT2PerSM, 1>(p, grid, smem, st);
    return launch_tier<kT2Threads, true, 1, kClusterSize>(p, grid, smem, st);
}

// Clusters of the cluster tier that can be resident at once (0: none).
int k1_max_clusters(size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClusterSize * 32);
    cfg.blockDim = dim3(kT2Threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterSize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaFuncSetAttribute(k1_cell_solve<kT2Threads, true, 1, kClusterSize, false, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k1_cell_solve<kT2Threads, true, 1, kClusterSize, false, false>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace dd
