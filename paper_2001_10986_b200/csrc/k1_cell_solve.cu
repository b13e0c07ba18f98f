// k1_cell_solve.cu -- K1: fused composite-cell solve of one sweep of
// Algorithm 2 (arXiv 2001.10986), one CTA per cell.
//
//   line 8   nu_cell = sum_{i in J} nu_i          -> gather into SMEM
//   line 9   (pi_cell, u_{C,J}) = Sinkhorn(...)    -> separable log-domain
//            Sinkhorn, warm-started from alpha, starts with a Y-iteration,
//            stops when the L1 X-error <= ||mu_J|| Err (Sec. 6.2)
//   line 10  nu_i = P_Y(pi_cell restricted to X_i x Y) -> ratio split from the
//            last Y-iteration (A7)
//   line 11  BalanceMeasures (A8)
//   line 12  Truncate + tight bounding box -> scratch pool
//
// Numerics: potentials in a cell-local affine
// gauge as fp32 (hi, lo2) pairs, hi on the 2^-8 grid so hi - C(d) - S is exact;
// exact per-axis cost table C(d) = d^2/kappa; ex2.approx of the reduced
// argument; accurate fp32 log of each row sum; fp64 staging, balance and
// marginal sums.  The grid cost is separable, so every half-iteration is two
// 1D log-sum-exp passes (a^2 b + a b^2 exps instead of a^2 b^2).
#include "dd_common.cuh"

namespace dd {

// --------------------------------------------------------- SMEM layout --
struct K1Lay {
    float2* FX;   // [ar][pX]  X potential F (hi, lo2)
    float2* FXn;  // [ar][pX]  X-iteration output
    float2* LM;   // [ar][ac]  log mu (hi, lo2)
    float* MU;    // [ar][ac]  mu (fp32, error weights)
    float2* Tt;   // [bc][pT]  Y pass-1 output T(x1, y2), transposed
    float2* W;    // [bc][pT]  split weights (w0, w1) of T over the x2 halves
    float2* G;    // [br][pG]  Y potential G (hi, lo2); epilogue: fp64 nu_cell
    float2* LNU;  // [br][bc]  log nu_cell (hi, lo2)
    float4* ACC;  // [br][bc]  per-quadrant partial sums of the last Y-iteration
    float2* Ut;   // [ac][pU]  X pass-1 output U(y1, x2), transposed
    float* CT;    // cost table C(d) = d^2 / kappa, d in [-OFF, OFF]
    double* red;  // reduction scratch (64)
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline int k1_ct_off(int s, int bcap) { return (2 * s > bcap ? 2 * s : bcap) + 2; }

__host__ __device__ inline size_t k1_smem_bytes(int s, int bcap) {
    const size_t A = 2 * s, pA = odd_pitch(2 * s), pB = odd_pitch(bcap), B = bcap;
    size_t b = 0;
    b += align16(A * pA * 8) * 2;          // FX, FXn
    b += align16(A * A * 8);               // LM
    b += align16(A * A * 4);               // MU
    b += align16(B * pA * 8) * 2;          // Tt, W
    b += align16(B * pB * 8);              // G
    b += align16(B * B * 8);               // LNU
    b += align16(B * B * 16);              // ACC
    b += align16(A * pB * 8);              // Ut
    b += align16((2 * k1_ct_off(s, bcap) + 4) * 4);  // CT
    b += 64 * 8;                           // red
    return b;
}

__device__ inline K1Lay k1_carve(unsigned char* base, int s, int bcap) {
    const size_t A = 2 * s, pA = odd_pitch(2 * s), pB = odd_pitch(bcap), B = bcap;
    K1Lay L;
    size_t o = 0;
    L.FX = (float2*)(base + o);  o += align16(A * pA * 8);
    L.FXn = (float2*)(base + o); o += align16(A * pA * 8);
    L.LM = (float2*)(base + o);  o += align16(A * A * 8);
    L.MU = (float*)(base + o);   o += align16(A * A * 4);
    L.Tt = (float2*)(base + o);  o += align16(B * pA * 8);
    L.W = (float2*)(base + o);   o += align16(B * pA * 8);
    L.G = (float2*)(base + o);   o += align16(B * pB * 8);
    L.LNU = (float2*)(base + o); o += align16(B * B * 8);
    L.ACC = (float4*)(base + o); o += align16(B * B * 16);
    L.Ut = (float2*)(base + o);  o += align16(A * pB * 8);
    L.CT = (float*)(base + o);   o += align16((2 * k1_ct_off(s, bcap) + 4) * 4);
    L.red = (double*)(base + o);
    return L;
}

struct Dims {
    int ar, ac, br, bc, s;
    int pX, pT, pG, pU;
    int off;      // CT centre
};

// Split an fp64 value into (hi on the 2^-8 grid, lo2 = (v - hi) * log2 e).
__device__ __forceinline__ float2 split_hl(double v) {
    if (!(v > -1e30)) return make_float2(-INFINITY, 0.0f);
    double h = rint(v * 256.0) * (1.0 / 256.0);
    return make_float2((float)h, (float)((v - h) * 1.4426950408889634));
}
__device__ __forceinline__ double join_hl(float2 p) {
    return (double)p.x + (double)p.y * 0.6931471805599453;
}

// ln(x) = hi + lo2 * ln 2 with hi on the 2^-8 grid, accurate to ~5e-8
// absolute and to ~1e-7 RELATIVE near x = 1 (converged sums), x > 0 normal.
__device__ __forceinline__ void ln_split(float x, float& hi, float& lo2) {
    const float LN2H = 0.693145751953125f;          // 0x3F317200 (exact e * LN2H)
    const float LN2L = 1.428606765330187e-06f;
    int ix = __float_as_int(x);
    int e = ((ix >> 23) & 0xff) - 127;
    float m = __int_as_float((ix & 0x007fffff) | 0x3f800000);
    if (m > 1.41421356f) { m *= 0.5f; e += 1; }
    const float num = m - 1.0f;
    const float den = m + 1.0f;
    float r = rcpf(den);
    r = r * fmaf(-den, r, 2.0f);
    const float z = num * r;
    const float z2 = z * z;
    float p = 0.18181818f;                          // 2/11
    p = fmaf(p, z2, 0.22222222f);                   // 2/9
    p = fmaf(p, z2, 0.28571429f);                   // 2/7
    p = fmaf(p, z2, 0.4f);                          // 2/5
    p = fmaf(p, z2, 0.66666667f);                   // 2/3
    p = fmaf(p, z2, 2.0f);
    const float lnm = z * p;
    const float eh = (float)e * LN2H;
    const float g = grid8(eh);
    const float v = (eh - g) + lnm;
    const float gh = grid8(v);
    hi = g + gh;
    lo2 = ((v - gh) + (float)e * LN2L) * kL2E;
}

enum { PY1 = 0, PY2 = 1, PX1 = 2, PX2 = 3 };

// One separable log-sum-exp pass.  Task = (o1, output pair o2a = 2j, 2j+1).
// out(o1, o2) = S + log sum_k exp(P(o1,k).hi - C(k - o2) - S + P(o1,k).lo2 ln2).
// Y1: o1 = x1, k = x2, o2 = y2 -> Tt[y2][x1], W   (split at x2 = s)
// Y2: o1 = y2, k = x1, o2 = y1 -> G[y1][y2] = LNU - out, ACC (quadrant sums)
// X1: o1 = y1, k = y2, o2 = x2 -> Ut[x2][y1]
// X2: o1 = x2, k = y1, o2 = x1 -> FXn[x1][x2] = LM - out; L1 X-error
template <int PASS>
__device__ __forceinline__ void lse_pass(const K1Lay& L, const Dims& d, bool exact_all,
                                         float2* Fcur, float2* Fout, double& err_acc,
                                         int& fallbacks, int& nonfinite) {
    int n1, K, n2, pitchP, ksplit;
    const float2* P;
    if (PASS == PY1) { n1 = d.ar; K = d.ac; n2 = d.bc; P = Fcur; pitchP = d.pX; ksplit = min(d.s, K); }
    else if (PASS == PY2) { n1 = d.bc; K = d.ar; n2 = d.br; P = L.Tt; pitchP = d.pT; ksplit = min(d.s, K); }
    else if (PASS == PX1) { n1 = d.br; K = d.bc; n2 = d.ac; P = L.G; pitchP = d.pG; ksplit = K; }
    else { n1 = d.ac; K = d.br; n2 = d.ar; P = L.Ut; pitchP = d.pU; ksplit = K; }

    const int n2h = (n2 + 1) >> 1;
    const int ntask = n1 * n2h;
    const float2 L2E2 = make_float2(kL2E, kL2E);

    for (int t = threadIdx.x; t < ntask; t += blockDim.x) {
        const int o1 = t % n1;
        const int j = t / n1;
        const int oa = 2 * j;
        const int ob = oa + 1;
        const bool vb = ob < n2;
        const float2* Prow = P + o1 * pitchP;

        // outputs that are -inf by definition (nu_cell(y) = 0 / mu(x) = 0)
        bool skipa = false, skipb = !vb;
        float2 tga = make_float2(0.f, 0.f), tgb = make_float2(0.f, 0.f);   // LNU / LM targets
        if (PASS == PY2) {
            tga = L.LNU[oa * d.bc + o1];
            tgb = vb ? L.LNU[ob * d.bc + o1] : tga;
            skipa = (tga.x == -INFINITY);
            skipb = skipb || (tgb.x == -INFINITY);
        } else if (PASS == PX2) {
            tga = L.LM[oa * d.ac + o1];
            tgb = vb ? L.LM[ob * d.ac + o1] : tga;
            skipa = (tga.x == -INFINITY);
            skipb = skipb || (tgb.x == -INFINITY);
        }

        // speculative stabilisers: hi part of the previous output of this pass
        float Sa = 0.f, Sb = 0.f;
        bool exact = exact_all;
        if (!exact) {
            if (PASS == PY1) { Sa = L.Tt[oa * d.pT + o1].x; Sb = vb ? L.Tt[ob * d.pT + o1].x : Sa; }
            else if (PASS == PY2) { Sa = tga.x - L.G[oa * d.pG + o1].x; Sb = vb ? tgb.x - L.G[ob * d.pG + o1].x : Sa; }
            else if (PASS == PX1) { Sa = L.Ut[oa * d.pU + o1].x; Sb = vb ? L.Ut[ob * d.pU + o1].x : Sa; }
            else { Sa = tga.x - Fcur[oa * d.pX + o1].x; Sb = vb ? tgb.x - Fcur[ob * d.pX + o1].x : Sa; }
            if (skipa) Sa = Sb;
            if (skipb) Sb = Sa;
            exact = !(fabsf(Sa) < 1e30f) || !(fabsf(Sb) < 1e30f);
        }

        const float* ctp = L.CT + d.off - oa;   // C(k - oa) = ctp[k]; C(k - ob) = ctp[k - 1]
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);   // halves (Y1) / totals
        float2 q00 = acc0, q01 = acc0, q10 = acc0, q11 = acc0;                // Y2 quadrants
        bool done = false;
        for (int attempt = 0; attempt < 2 && !done; ++attempt) {
            if (exact) {
                float Ma = -INFINITY, Mb = -INFINITY;
                float cb = ctp[-1];
                for (int k = 0; k < K; ++k) {
                    const float px = Prow[k].x;
                    const float ca = ctp[k];
                    Ma = fmaxf(Ma, px - ca);
                    Mb = fmaxf(Mb, px - cb);
                    cb = ca;
                }
                Sa = (Ma == -INFINITY) ? 0.f : Ma;
                Sb = (Mb == -INFINITY) ? 0.f : Mb;
                if (Ma == -INFINITY) skipa = true;
                if (Mb == -INFINITY) skipb = true;
            }
            const float2 nS = make_float2(-Sa, -Sb);
            acc0 = acc1 = q00 = q01 = q10 = q11 = make_float2(0.f, 0.f);
            float cb = ctp[-1];
            if (PASS == PY2) {
                const float2* Wrow = L.W + o1 * d.pT;
#pragma unroll 2
                for (int k = 0; k < ksplit; ++k) {
                    const float2 pk = Prow[k];
                    const float2 w = Wrow[k];
                    const float ca = ctp[k];
                    float2 tt = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-ca, -cb));
                    tt = __fadd2_rn(tt, nS);
                    tt = __ffma2_rn(tt, L2E2, make_float2(pk.y, pk.y));
                    const float2 e = make_float2(ex2f(tt.x), ex2f(tt.y));
                    q00 = __ffma2_rn(e, make_float2(w.x, w.x), q00);
                    q01 = __ffma2_rn(e, make_float2(w.y, w.y), q01);
                    cb = ca;
                }
#pragma unroll 2
                for (int k = ksplit; k < K; ++k) {
                    const float2 pk = Prow[k];
                    const float2 w = Wrow[k];
                    const float ca = ctp[k];
                    float2 tt = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-ca, -cb));
                    tt = __fadd2_rn(tt, nS);
                    tt = __ffma2_rn(tt, L2E2, make_float2(pk.y, pk.y));
                    const float2 e = make_float2(ex2f(tt.x), ex2f(tt.y));
                    q10 = __ffma2_rn(e, make_float2(w.x, w.x), q10);
                    q11 = __ffma2_rn(e, make_float2(w.y, w.y), q11);
                    cb = ca;
                }
                acc0 = __fadd2_rn(__fadd2_rn(q00, q01), __fadd2_rn(q10, q11));
            } else {
#pragma unroll 4
                for (int k = 0; k < ksplit; ++k) {
                    const float2 pk = Prow[k];
                    const float ca = ctp[k];
                    float2 tt = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-ca, -cb));
                    tt = __fadd2_rn(tt, nS);
                    tt = __ffma2_rn(tt, L2E2, make_float2(pk.y, pk.y));
                    acc0 = __fadd2_rn(acc0, make_float2(ex2f(tt.x), ex2f(tt.y)));
                    cb = ca;
                }
                if (PASS == PY1) {
#pragma unroll 4
                    for (int k = ksplit; k < K; ++k) {
                        const float2 pk = Prow[k];
                        const float ca = ctp[k];
                        float2 tt = __fadd2_rn(make_float2(pk.x, pk.x), make_float2(-ca, -cb));
                        tt = __fadd2_rn(tt, nS);
                        tt = __ffma2_rn(tt, L2E2, make_float2(pk.y, pk.y));
                        acc1 = __fadd2_rn(acc1, make_float2(ex2f(tt.x), ex2f(tt.y)));
                        cb = ca;
                    }
                }
            }
            const float ta = (PASS == PY1) ? acc0.x + acc1.x : acc0.x;
            const float tb = (PASS == PY1) ? acc0.y + acc1.y : acc0.y;
            if (exact) { done = true; break; }
            // speculative window: dominant terms must stay near t = 0 for the
            // exactness argument of the (hi, lo) arithmetic
            const bool oka = skipa || (ta >= 0.25f && ta <= 4.0f);
            const bool okb = skipb || (tb >= 0.25f && tb <= 4.0f);
            if (oka && okb) { done = true; break; }
            exact = true;
            ++fallbacks;
        }

        // ---- finalise the (up to) two outputs
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool valid = (h == 0) ? true : vb;
            if (!valid) continue;
            const int o2 = (h == 0) ? oa : ob;
            const bool skip = (h == 0) ? skipa : skipb;
            const float S = (h == 0) ? Sa : Sb;
            const float tot = (PASS == PY1) ? ((h == 0) ? acc0.x + acc1.x : acc0.y + acc1.y)
                                            : ((h == 0) ? acc0.x : acc0.y);
            float Lhi = -INFINITY, Llo = 0.f;
            const bool empty = skip || !(tot > 1e-37f);
            if (!empty) {
                float lh, ll;
                ln_split(tot, lh, ll);
                Lhi = S + lh;
                Llo = ll;
                if (!(fabsf(Lhi) < 1e30f)) nonfinite = 1;
            }
            if (PASS == PY1) {
                L.Tt[o2 * d.pT + o1] = make_float2(Lhi, empty ? 0.f : Llo);
                float2 w = make_float2(0.f, 0.f);
                if (!empty) {
                    const float s0 = (h == 0) ? acc0.x : acc0.y;
                    const float s1 = (h == 0) ? acc1.x : acc1.y;
                    const float r = rcpf(tot);
                    w = make_float2(s0 * r, s1 * r);
                }
                L.W[o2 * d.pT + o1] = w;
            } else if (PASS == PY2) {
                const float2 tg = (h == 0) ? tga : tgb;
                if (skip) {
                    L.G[o2 * d.pG + o1] = make_float2(-INFINITY, 0.f);
                    L.ACC[o2 * d.bc + o1] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    if (empty) nonfinite = 1;     // nu_cell(y) > 0 unreachable
                    L.G[o2 * d.pG + o1] = make_float2(tg.x - Lhi, tg.y - Llo);
                    L.ACC[o2 * d.bc + o1] = (h == 0) ? make_float4(q00.x, q01.x, q10.x, q11.x)
                                                     : make_float4(q00.y, q01.y, q10.y, q11.y);
                }
            } else if (PASS == PX1) {
                L.Ut[o2 * d.pU + o1] = make_float2(Lhi, empty ? 0.f : Llo);
            } else {
                const float2 tg = (h == 0) ? tga : tgb;
                const int ix = o2 * d.pX + o1;
                if (skip) {
                    Fout[ix] = make_float2(-INFINITY, 0.f);
                } else {
                    if (empty) nonfinite = 1;
                    const float2 fn = make_float2(tg.x - Lhi, tg.y - Llo);
                    Fout[ix] = fn;
                    const float2 fo = Fcur[ix];
                    // P_X pi(x) = mu(x) exp(F - F_new)  (plan (F, G))
                    const float dF = (fo.x - fn.x) + (fo.y - fn.y) * kLN2;
                    err_acc += (double)L.MU[o2 * d.ac + o1] * (double)fabsf(expm1f(dF));
                }
            }
        }
    }
}

// ----------------------------------------------------------- the solve --
__device__ void solve_cell(const SweepParams& p, int cell, unsigned char* smem) {
    const K1Lay L = k1_carve(smem, p.s, p.bcap);
    __shared__ int4 s_box[4];
    __shared__ long long s_off[4];
    __shared__ int s_q[4];          // quadrant of each member
    __shared__ int s_mem[4];        // basic cell index of each member
    __shared__ int s_nb[4 * 4];     // epilogue bbox (rmin, rmax, cmin, cmax) per member
    __shared__ long long s_newoff[4];
    __shared__ int4 s_newbox[4];
    __shared__ double s_bal[4 * 3];
    __shared__ int s_flag;

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

    if (d.br > p.bcap || d.bc > p.bcap || d.br == 0) {
        if (tid == 0) {
            if (p.mode == 0 && d.br > 0) {
                const int k = atomicAdd(p.n_deferred, 1);
                p.deferred[k] = cell;
                co.flags = 4;
            } else {
                co.flags = 2;   // cannot be handled: too large even for the big path / empty
                atomicOr(p.overflow, 2);
            }
            p.out[cell] = co;
        }
        return;
    }
    d.pX = odd_pitch(d.ac); d.pT = odd_pitch(d.ar); d.pG = odd_pitch(d.bc); d.pU = odd_pitch(d.br);
    d.off = k1_ct_off(p.s, p.bcap);
    const int Dr = R0 - Y0, Dc = C0 - X0;          // local-frame offsets (DESIGN.md gauge)
    const double inv_kappa = 1.0 / p.kappa;
    const double inv_eps = 1.0 / p.eps;

    // ---- cost table (exact for kappa = 2^k)
    for (int i = tid; i < 2 * d.off + 1; i += blockDim.x) {
        const double dd = (double)(i - d.off);
        L.CT[i] = (float)(dd * dd * inv_kappa);
    }
    // ---- line 8: nu_cell = sum_i nu_i on the union box; log nu_cell
    const int ny = d.br * d.bc;
    double npos = 0.0;
    for (int y = tid; y < ny; y += blockDim.x) {
        const int gy = Y0 + y / d.bc, gx = X0 + y % d.bc;
        double v = 0.0;
        for (int m = 0; m < nmem; ++m) {
            const int4 b = s_box[m];
            const int ry = gy - b.x, rx = gx - b.y;
            if (ry >= 0 && ry < b.z && rx >= 0 && rx < b.w) v += p.pool_in[s_off[m] + (long long)ry * b.w + rx];
        }
        L.LNU[y] = (v > 0.0) ? split_hl(log(v)) : make_float2(-INFINITY, 0.f);
        npos += (v > 0.0) ? 1.0 : 0.0;
    }
    // ---- X side: F = alpha/eps + log mu - shift(x~) - lambda (local gauge)
    const int nx = d.ar * d.ac;
    double fmax_l = -INFINITY, muJ = 0.0;
    for (int x = tid; x < nx; x += blockDim.x) {
        const int xr = x / d.ac, xc = x % d.ac;
        const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
        const double m = p.mu[g];
        muJ += m;
        if (m > 0.0) {
            const double sh = ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            const double F = p.alpha[g] * inv_eps + p.logmu[g] - sh;
            fmax_l = fmax(fmax_l, F);
        }
    }
    const double lambda = block_max(fmax_l, L.red);
    muJ = block_sum(muJ, L.red + 32);
    npos = block_sum(npos, L.red);
    for (int x = tid; x < nx; x += blockDim.x) {
        const int xr = x / d.ac, xc = x % d.ac;
        const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
        const double m = p.mu[g];
        float2 f = make_float2(-INFINITY, 0.f), lm = make_float2(-INFINITY, 0.f);
        if (m > 0.0) {
            const double sh = ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            f = split_hl(p.alpha[g] * inv_eps + p.logmu[g] - sh - lambda);
            lm = split_hl(p.logmu[g]);
        }
        L.FX[xr * d.pX + xc] = f;
        L.LM[x] = lm;
        L.MU[x] = (float)m;
    }
    __syncthreads();

    // ---- line 9: Sinkhorn (Y-iteration first; stop test fused in the X-iteration)
    const double tol = muJ * p.err_tol;
    float2* Fc = L.FX;
    float2* Fn = L.FXn;
    int it = 0, fallbacks = 0, nonfinite = 0;
    double err = 0.0;
    if (tid == 0) s_flag = 0;
    while (true) {
        const bool exact = (it == 0);
        double e_loc = 0.0;
        lse_pass<PY1>(L, d, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        __syncthreads();
        lse_pass<PY2>(L, d, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        __syncthreads();
        lse_pass<PX1>(L, d, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        __syncthreads();
        lse_pass<PX2>(L, d, exact, Fc, Fn, e_loc, fallbacks, nonfinite);
        err = block_sum(e_loc, L.red);      // includes the barrier
        ++it;
        if (err <= tol) break;
        if (it >= p.max_iter || !(err == err)) { co.flags |= 1; break; }
        float2* t = Fc; Fc = Fn; Fn = t;
    }
    if (nonfinite) atomicOr(&s_flag, 2);
    fallbacks = (int)block_sum((double)fallbacks, L.red + 32);
    __syncthreads();
    co.flags |= s_flag;
    co.iters = it;
    co.err = (float)err;
    co.fallbacks = fallbacks;
    {
        const double ar = d.ar, ac = d.ac, br = d.br, bc = d.bc;
        // algorithmic MUFU ops per iteration: one ex2 per term of
        // the four 1D passes + one log per pass output (skipped nu = 0 rows excluded)
        const double per_it = ar * ac * bc + ar * npos + br * bc * ac + ac * br * ar
                              + ar * bc + npos + br * ac + ar * ac;
        co.mufu = per_it * it;
    }

    // ---- epilogue: nu_cell (fp64) into the G region
    double* NUC = reinterpret_cast<double*>(L.G);
    for (int y = tid; y < ny; y += blockDim.x) {
        const int gy = Y0 + y / d.bc, gx = X0 + y % d.bc;
        double v = 0.0;
        for (int m = 0; m < nmem; ++m) {
            const int4 b = s_box[m];
            const int ry = gy - b.x, rx = gx - b.y;
            if (ry >= 0 && ry < b.z && rx >= 0 && rx < b.w) v += p.pool_in[s_off[m] + (long long)ry * b.w + rx];
        }
        NUC[y] = v;
    }
    __syncthreads();
    // line 10: nu_i(y) = nu_cell(y) S_i(y) / S(y)  (ratio form, A7) ; norms
    double nrm[4] = {0.0, 0.0, 0.0, 0.0};
    for (int y = tid; y < ny; y += blockDim.x) {
        const float4 a = L.ACC[y];
        const double tot = (double)a.x + (double)a.y + (double)a.z + (double)a.w;
        if (!(tot > 0.0)) continue;
        const double sc = NUC[y] / tot;
        const double q[4] = {a.x * sc, a.y * sc, a.z * sc, a.w * sc};
        for (int m = 0; m < nmem; ++m) nrm[m] += q[s_q[m]];
    }
    for (int m = 0; m < nmem; ++m) nrm[m] = block_sum(nrm[m], L.red + 8 * m);
    // line 11: BalanceMeasures (A8): donors give nu_i d_i/||nu_i|| T/Dsum, receivers
    // take r(y) (-d_j)/Psum, T = min(Dsum, Psum)
    if (tid == 0) {
        double dsum = 0.0, psum = 0.0, dmax = 0.0, dv[4];
        for (int m = 0; m < nmem; ++m) {
            dv[m] = nrm[m] - p.mass_i[s_mem[m]];
            dmax = fmax(dmax, fabs(dv[m]));
            if (dv[m] > 0) dsum += dv[m]; else psum += -dv[m];
        }
        const bool skip = (dmax <= 1e-18 || dsum <= 0.0 || psum <= 0.0);
        const double T = dsum < psum ? dsum : psum;
        for (int m = 0; m < 4; ++m) {
            double fd = 0.0, gr = 0.0;
            if (!skip && m < nmem) {
                if (dv[m] > 0) fd = (dv[m] / nrm[m]) * (T / dsum);
                else if (dv[m] < 0) gr = -dv[m] / psum;
            }
            s_bal[2 * m] = fd;
            s_bal[2 * m + 1] = gr;
        }
    }
    __syncthreads();
    double fd[4], gr[4];
    for (int m = 0; m < 4; ++m) { fd[m] = s_bal[2 * m]; gr[m] = s_bal[2 * m + 1]; }
    auto balanced = [&](int y, double* out) {
        const float4 a = L.ACC[y];
        const double tot = (double)a.x + (double)a.y + (double)a.z + (double)a.w;
        if (!(tot > 0.0)) { for (int m = 0; m < nmem; ++m) out[m] = 0.0; return; }
        const double sc = NUC[y] / tot;
        const double q[4] = {a.x * sc, a.y * sc, a.z * sc, a.w * sc};
        double v[4], r = 0.0;
        for (int m = 0; m < nmem; ++m) {
            v[m] = q[s_q[m]];
            const double take = v[m] * fd[m];
            r += take;
            v[m] -= take;
        }
        for (int m = 0; m < nmem; ++m) out[m] = v[m] + r * gr[m];
    };
    // line 12: Truncate + tight bbox per member
    int bb[4][4];
    for (int m = 0; m < 4; ++m) { bb[m][0] = 1 << 30; bb[m][1] = -1; bb[m][2] = 1 << 30; bb[m][3] = -1; }
    for (int y = tid; y < ny; y += blockDim.x) {
        double v[4];
        balanced(y, v);
        const int yr = y / d.bc, yc = y % d.bc;
        for (int m = 0; m < nmem; ++m)
            if (v[m] >= p.tau && v[m] > 0.0) {
                bb[m][0] = min(bb[m][0], yr); bb[m][1] = max(bb[m][1], yr);
                bb[m][2] = min(bb[m][2], yc); bb[m][3] = max(bb[m][3], yc);
            }
    }
    for (int m = 0; m < nmem; ++m) {
        int a0 = warp_min_i(bb[m][0]), a1 = warp_max_i(bb[m][1]);
        int a2 = warp_min_i(bb[m][2]), a3 = warp_max_i(bb[m][3]);
        bb[m][0] = a0; bb[m][1] = a1; bb[m][2] = a2; bb[m][3] = a3;
    }
    int* ired = reinterpret_cast<int*>(L.red);
    __syncthreads();
    if ((tid & 31) == 0) {
        const int w = tid >> 5;
        for (int m = 0; m < nmem; ++m)
            for (int k = 0; k < 4; ++k) ired[(w * 4 + m) * 4 + k] = bb[m][k];
    }
    __syncthreads();
    if (tid == 0) {
        const int nw = blockDim.x >> 5;
        long long total = 0;
        long long area[4];
        for (int m = 0; m < nmem; ++m) {
            int r0 = 1 << 30, r1 = -1, c0 = 1 << 30, c1 = -1;
            for (int w = 0; w < nw; ++w) {
                r0 = min(r0, ired[(w * 4 + m) * 4 + 0]); r1 = max(r1, ired[(w * 4 + m) * 4 + 1]);
                c0 = min(c0, ired[(w * 4 + m) * 4 + 2]); c1 = max(c1, ired[(w * 4 + m) * 4 + 3]);
            }
            s_nb[4 * m + 0] = r0; s_nb[4 * m + 1] = r1; s_nb[4 * m + 2] = c0; s_nb[4 * m + 3] = c1;
            const int hh = r1 >= 0 ? r1 - r0 + 1 : 0, ww = r1 >= 0 ? c1 - c0 + 1 : 0;
            s_newbox[m] = r1 >= 0 ? make_int4(Y0 + r0, X0 + c0, hh, ww) : make_int4(Y0, X0, 0, 0);
            area[m] = ((long long)hh * ww + 1) & ~1LL;       // 16-byte aligned boxes
            total += area[m];
        }
        const long long base = (long long)atomicAdd(p.bump, (unsigned long long)total);
        if (base + total > p.cap) {
            atomicOr(p.overflow, 1);
            co.flags |= 8;
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
        for (int k = tid; k < area; k += blockDim.x) {
            const int y = (r0 + k / nb4.w) * d.bc + (c0 + k % nb4.w);
            double v[4];
            balanced(y, v);
            const double val = v[m];
            p.scratch[o + k] = (val >= p.tau && val > 0.0) ? val : 0.0;
        }
    }
    if (tid < nmem) {
        p.box[s_mem[tid]] = s_newbox[tid];
        p.off[s_mem[tid]] = s_newoff[tid] < 0 ? 0 : s_newoff[tid];
        if (s_newoff[tid] < 0) p.box[s_mem[tid]] = make_int4(Y0, X0, 0, 0);
    }
    // store u_{C,J}: alpha = eps (F + lambda + shift - log mu)  (plan's F, A4)
    for (int x = tid; x < nx; x += blockDim.x) {
        const int xr = x / d.ac, xc = x % d.ac;
        const long long g = (long long)(R0 + xr) * p.side + (C0 + xc);
        const float2 f = Fc[xr * d.pX + xc];
        double a = 0.0;
        if (f.x > -INFINITY && p.mu[g] > 0.0) {
            const double sh = ((2.0 * xr + Dr) * Dr + (2.0 * xc + Dc) * Dc) * inv_kappa;
            a = p.eps * (join_hl(f) + lambda + sh - p.logmu[g]);
        }
        p.alpha[g] = a;
    }
    if (tid == 0) p.out[cell] = co;
}

__global__ void __launch_bounds__(kThreads) k1_cell_solve(SweepParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_cell;
    if (p.mode == 0) {
        solve_cell(p, blockIdx.x, smem);
        return;
    }
    while (true) {
        if (threadIdx.x == 0) {
            const int k = atomicAdd(p.work_counter, 1);
            s_cell = (k < *p.n_deferred) ? p.deferred[k] : -1;
        }
        __syncthreads();
        const int cell = s_cell;
        if (cell < 0) return;
        solve_cell(p, cell, smem);
        __syncthreads();
    }
}

size_t k1_smem_bytes_host(int s, int bcap) { return k1_smem_bytes(s, bcap); }

cudaError_t launch_k1(const SweepParams& p, int grid, size_t smem, cudaStream_t st) {
    static int attr_set_bytes = 0;
    if ((int)smem > attr_set_bytes) {
        cudaError_t e = cudaFuncSetAttribute(k1_cell_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set_bytes = (int)smem;
    }
    k1_cell_solve<<<grid, kThreads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace dd
