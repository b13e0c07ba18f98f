// k_glue.cu -- K5: coarse-to-fine refinement of the X-potentials (arXiv
// 2001.10986): "glue" the per-cell potentials of the coarse
// layer by the discrete Helmholtz least squares of Sec. 6.3,
// then interpolate linearly in log space (alpha = eps log u) onto the fine
// pixels.  Used as the warm start of both partitions on the new layer.
//
// Graph: vertices = composite cells J of partition A; for each
// B-cell J_B and two of its basic cells i1 != i2 (they lie in different A
// cells J1 = A(i1), J2 = A(i2)) an edge with
//   log q_(J1,J2) = log avg_{X_i1} exp((a_A - a_B)/eps) dmu + log avg_{X_i2} exp((a_B - a_A)/eps) dmu
// (J_A cap J_B is exactly one basic cell).  Least squares over all edges
//   min_V sum ((V(J2) - V(J1)) - log q_(J1,J2))^2
// taken in both orientations (antisymmetrised weights).  Sign (DESIGN.md
// reading A25): P:1447 prints (V(J1) - V(J2)) - log q, but the path product
// u_J = prod q u_{A,J} it approximates implies V(J2) - V(J1) =
// log q_(J1,J2); only this sign cancels the per-cell constants at
// convergence.  a_i = log avg_{X_i} e^{(aA-aB)/eps} dmu, b_i = log avg e^{(aB-aA)/eps} dmu.
// Normal equations L V = r (graph Laplacian, zero-sum r) by Jacobi-
// preconditioned CG in one CTA (fixed order: deterministic).  Then
// alpha_hat = alpha_A + eps V (cost units) and bilinear interpolation.
#include <algorithm>

#include "dd_aux.cuh"

namespace dd {

// a_i, b_i per basic cell (one warp per basic cell)
__global__ void k_glue_ab(const double* __restrict__ aA, const double* __restrict__ aB, const double* __restrict__ mu,
                          int side, int s, int nb, double eps, double* __restrict__ ab) {
    const int warps = blockDim.x >> 5;
    const int i = blockIdx.x * warps + (threadIdx.x >> 5);
    const int l = threadIdx.x & 31;
    if (i >= nb * nb) return;
    const int r0 = (i / nb) * s, c0 = (i % nb) * s;
    // pass 1: maxima of (aA - aB)/eps and its negative over mu > 0
    double mp = -INFINITY, mn = -INFINITY;
    for (int k = l; k < s * s; k += 32) {
        const long long g = (long long)(r0 + k / s) * side + (c0 + k % s);
        if (mu[g] > 0.0) {
            const double d = (aA[g] - aB[g]) / eps;
            mp = fmax(mp, d);
            mn = fmax(mn, -d);
        }
    }
    mp = warp_max(mp);
    mn = warp_max(mn);
    double sp = 0.0, sn = 0.0, sm = 0.0;
    for (int k = l; k < s * s; k += 32) {
        const long long g = (long long)(r0 + k / s) * side + (c0 + k % s);
        const double m = mu[g];
        if (m > 0.0) {
            const double d = (aA[g] - aB[g]) / eps;
            sp += m * exp(d - mp);
            sn += m * exp(-d - mn);
            sm += m;
        }
    }
    sp = warp_sum(sp);
    sn = warp_sum(sn);
    sm = warp_sum(sm);
    if (l == 0) {
        ab[2 * i] = (sm > 0.0) ? mp + log(sp / sm) : 0.0;
        ab[2 * i + 1] = (sm > 0.0) ? mn + log(sn / sm) : 0.0;
    }
}

// members of the B-cell containing basic cell (r, c); returns the count
__device__ __forceinline__ int bmembers(int nb, int r, int c, int* mr, int* mc) {
    const int q1 = (r + 1) / 2, q2 = (c + 1) / 2;      // B-cell row/col of basic row r: rows 2q-1, 2q
    int n = 0;
    for (int rr = 2 * q1 - 1; rr <= 2 * q1; ++rr)
        for (int cc = 2 * q2 - 1; cc <= 2 * q2; ++cc)
            if (rr >= 0 && rr < nb && cc >= 0 && cc < nb) { mr[n] = rr; mc[n] = cc; ++n; }
    return n;
}

// y = L x (or r = rhs when RHS) for the A-cell graph, gathered per A node.
template <bool RHS>
__device__ __forceinline__ double lap_row(int p, int na, int nb, const double* __restrict__ x,
                                          const double* __restrict__ ab, double* deg) {
    const int P = p / na, Q = p % na;
    double acc = 0.0, dg = 0.0;
    for (int k = 0; k < 4; ++k) {
        const int r = 2 * P + (k >> 1), c = 2 * Q + (k & 1);       // basic cell i of node p
        int mr[4], mc[4];
        const int m = bmembers(nb, r, c, mr, mc);
        const int i = r * nb + c;
        for (int t = 0; t < m; ++t) {
            if (mr[t] == r && mc[t] == c) continue;
            const int i2 = mr[t] * nb + mc[t];
            const int p2 = (mr[t] / 2) * na + (mc[t] / 2);
            dg += 1.0;
            // edge p -> p2 weight log q = a_i + b_i2; V(p2) - V(p) ~ log q (path product, see header)
            if (RHS) acc += 0.5 * ((ab[2 * i2] + ab[2 * i + 1]) - (ab[2 * i] + ab[2 * i2 + 1]));
            else acc += x[p] - x[p2];
        }
    }
    if (deg) *deg = dg;
    return acc;
}

__device__ __forceinline__ double bsum(double v, double* red) { return block_sum(v, red); }

// Jacobi-preconditioned CG on L V = r in one CTA; V -> eps V written to out.
// work: 4 * na^2 doubles (V, r, z/p, Ap).
__global__ void k_glue_cg(const double* __restrict__ ab, int nb, double eps, int max_it, double rtol,
                          double* __restrict__ work, double* __restrict__ outV) {
    __shared__ double red[32];
    const int na = nb / 2, n = na * na;
    double* V = work;
    double* R = work + n;
    double* Pv = work + 2 * n;
    double* AP = work + 3 * n;
    double rz = 0.0, rr0 = 0.0;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        double dg;
        const double r = lap_row<true>(p, na, nb, nullptr, ab, &dg);
        V[p] = 0.0;
        R[p] = r;
        const double z = dg > 0.0 ? r / dg : 0.0;
        Pv[p] = z;
        rz += r * z;
        rr0 += r * r;
    }
    rz = bsum(rz, red);
    rr0 = bsum(rr0, red);
    if (rr0 > 0.0) {
        for (int it = 0; it < max_it; ++it) {
            double pap = 0.0;
            for (int p = threadIdx.x; p < n; p += blockDim.x) {
                const double a = lap_row<false>(p, na, nb, Pv, ab, nullptr);
                AP[p] = a;
                pap += Pv[p] * a;
            }
            pap = bsum(pap, red);
            if (!(pap > 0.0)) break;
            const double alpha = rz / pap;
            double rzn = 0.0, rrn = 0.0;
            for (int p = threadIdx.x; p < n; p += blockDim.x) {
                V[p] += alpha * Pv[p];
                const double r = R[p] - alpha * AP[p];
                R[p] = r;
                double dg;
                lap_row<true>(p, na, nb, nullptr, ab, &dg);
                const double z = dg > 0.0 ? r / dg : 0.0;
                AP[p] = z;                              // z kept in AP until the direction update
                rzn += r * z;
                rrn += r * r;
            }
            rzn = bsum(rzn, red);
            rrn = bsum(rrn, red);
            if (rrn <= rtol * rtol * rr0) break;
            const double beta = rzn / rz;
            rz = rzn;
            for (int p = threadIdx.x; p < n; p += blockDim.x) Pv[p] = AP[p] + beta * Pv[p];
            __syncthreads();
        }
    }
    __syncthreads();
    // mean-zero gauge (the Laplacian's null space), cost units
    double mean = 0.0;
    for (int p = threadIdx.x; p < n; p += blockDim.x) mean += V[p];
    mean = bsum(mean, red) / (double)n;
    for (int p = threadIdx.x; p < n; p += blockDim.x) outV[p] = eps * (V[p] - mean);
}

// glued coarse potential alpha_hat = alpha_A + eps V(A(x))
__global__ void k_glue_apply(const double* __restrict__ aA, const double* __restrict__ epsV, int side, int s,
                             double* __restrict__ phi) {
    const int nb = side / s, na = nb / 2;
    const long long n2 = (long long)side * side;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n2; k += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(k / side), c = (int)(k % side);
        const int p = (r / s / 2) * na + (c / s / 2);
        phi[k] = aA[k] + epsV[p];
    }
}

// bilinear interpolation of the coarse phi (side sc) onto the fine pixel
// centres (side 2 sc), clamped at the border; written to both alpha images
__global__ void k_interp2x(const double* __restrict__ phi, int sc, double* __restrict__ aA, double* __restrict__ aB) {
    const int sf = 2 * sc;
    const long long n2 = (long long)sf * sf;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n2; k += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(k / sf), j = (int)(k % sf);
        // fine centre (i + 1/2) / sf in coarse index units: (i + 1/2)/2 - 1/2
        const double u = 0.5 * i - 0.25, v = 0.5 * j - 0.25;
        int i0 = (int)floor(u), j0 = (int)floor(v);
        double fu = u - i0, fv = v - j0;
        if (i0 < 0) { i0 = 0; fu = 0.0; }
        if (j0 < 0) { j0 = 0; fv = 0.0; }
        const int i1 = min(i0 + 1, sc - 1), j1 = min(j0 + 1, sc - 1);
        if (i0 >= sc - 1) fu = 0.0;
        if (j0 >= sc - 1) fv = 0.0;
        const double a00 = phi[(long long)i0 * sc + j0], a01 = phi[(long long)i0 * sc + j1];
        const double a10 = phi[(long long)i1 * sc + j0], a11 = phi[(long long)i1 * sc + j1];
        const double a = (1.0 - fu) * ((1.0 - fv) * a00 + fv * a01) + fu * ((1.0 - fv) * a10 + fv * a11);
        aA[k] = a;
        aB[k] = a;
    }
}

cudaError_t launch_glue_refine(const double* aA_c, const double* aB_c, const double* mu_c, int side_c, int s_c,
                               double eps, double* scratch, double* aA_f, double* aB_f, cudaStream_t st) {
    const int nb = side_c / s_c, na = nb / 2;
    double* ab = scratch;                                  // 2 nb^2
    double* work = ab + 2 * (size_t)nb * nb;               // 4 na^2
    double* epsV = work + 4 * (size_t)na * na;             // na^2
    double* phi = epsV + (size_t)na * na;                  // side_c^2
    k_glue_ab<<<(nb * nb + 7) / 8, 256, 0, st>>>(aA_c, aB_c, mu_c, side_c, s_c, nb, eps, ab);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_glue_cg<<<1, 1024, 0, st>>>(ab, nb, eps, 4 * nb + 64, 1e-10, work, epsV);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const long long n2 = (long long)side_c * side_c;
    k_glue_apply<<<(int)std::min<long long>((n2 + 255) / 256, 148 * 16), 256, 0, st>>>(aA_c, epsV, side_c, s_c, phi);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_interp2x<<<(int)std::min<long long>((4 * n2 + 255) / 256, 148 * 16), 256, 0, st>>>(phi, side_c, aA_f, aB_f);
    return cudaGetLastError();
}

// glued potential of the current layer only (the PD-gap dual candidate)
cudaError_t launch_glue_phi(const double* aA, const double* aB, const double* mu, int side, int s, double eps,
                            double* scratch, double** phi_out) {
    const int nb = side / s, na = nb / 2;
    double* ab = scratch;
    double* work = ab + 2 * (size_t)nb * nb;
    double* epsV = work + 4 * (size_t)na * na;
    double* phi = epsV + (size_t)na * na;
    k_glue_ab<<<(nb * nb + 7) / 8, 256>>>(aA, aB, mu, side, s, nb, eps, ab);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_glue_cg<<<1, 1024>>>(ab, nb, eps, 20 * nb * nb + 100, 1e-14, work, epsV);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const long long n2 = (long long)side * side;
    k_glue_apply<<<(int)std::min<long long>((n2 + 255) / 256, 148 * 16), 256>>>(aA, epsV, side, s, phi);
    *phi_out = phi;
    return cudaGetLastError();
}

size_t glue_scratch_doubles(int side_c, int s_c) {
    const size_t nb = side_c / s_c, na = nb / 2;
    return 2 * nb * nb + 5 * na * na + (size_t)side_c * side_c;
}

}  // namespace dd
