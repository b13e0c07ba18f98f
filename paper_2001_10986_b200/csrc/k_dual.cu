// k_dual.cu -- relative primal-dual gap of the current iterate, eq. RelPDGap
// (arXiv 2001.10986), with the dual candidate of Sec. 6.3
// (P:1416-1456): X-potentials glued by the Helmholtz least squares (k_glue.cu)
// and v_hat = the Y-iteration against u_hat (Remark Sinkhorn), so
//   J(u_hat, v_hat) - ||K|| = <log u_hat, mu> + <log v_hat, nu> - ||nu||.
// The Y-iteration is over the WHOLE grid (dense in x), done exactly as two
// separable fp64 log-sum-exp passes (c is separable): diagnostic, not timed.
#include <algorithm>

#include "dd_aux.cuh"

namespace dd {

// pass 1: T(x1, y2) = LSE_x2 [phi(x1,x2)/eps + log mu(x1,x2) - (x2 - y2)^2 / kappa]
// (general separable cost, dd_set_cost: h2(|x2 - y2|)/eps and h1(|x1 - y1|)/eps instead)
__device__ __forceinline__ double axis_cost(const double* h, int hst, int d, double inv_kappa, double inv_eps) {
    if (h) return h[(long long)abs(d) * hst] * inv_eps;
    const double v = (double)d;
    return v * v * inv_kappa;
}

__global__ void k_dual_pass1(const double* __restrict__ phi, const double* __restrict__ logmu, int n,
                             double inv_eps, double inv_kappa, double* __restrict__ T, const double* h2, int hst) {
    const long long n2 = (long long)n * n;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n2; o += (long long)gridDim.x * blockDim.x) {
        const int x1 = (int)(o / n), y2 = (int)(o % n);
        const double* ph = phi + (long long)x1 * n;
        const double* lm = logmu + (long long)x1 * n;
        double m = -INFINITY;
        for (int x2 = 0; x2 < n; ++x2) {
            if (lm[x2] == -INFINITY) continue;
            m = fmax(m, ph[x2] * inv_eps + lm[x2] - axis_cost(h2, hst, x2 - y2, inv_kappa, inv_eps));
        }
        double s = 0.0;
        if (m > -INFINITY)
            for (int x2 = 0; x2 < n; ++x2) {
                if (lm[x2] == -INFINITY) continue;
                s += exp(ph[x2] * inv_eps + lm[x2] - axis_cost(h2, hst, x2 - y2, inv_kappa, inv_eps) - m);
            }
        T[o] = (m > -INFINITY) ? m + log(s) : -INFINITY;
    }
}

// pass 2: log v_hat(y) = -LSE_x1 [T(x1, y2) - (x1 - y1)^2 / kappa]; per-y term
// nu(y) (log v_hat(y) - 1) for nu(y) > 0, and mu phi / eps per x
__global__ void k_dual_pass2(const double* __restrict__ T, const double* __restrict__ nu,
                             const double* __restrict__ mu, const double* __restrict__ phi, int n, double inv_eps,
                             double inv_kappa, double* __restrict__ term, const double* h1, int hst) {
    const long long n2 = (long long)n * n;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n2; o += (long long)gridDim.x * blockDim.x) {
        const int y1 = (int)(o / n), y2 = (int)(o % n);
        double t = (mu[o] > 0.0) ? mu[o] * phi[o] * inv_eps : 0.0;
        if (nu[o] > 0.0) {
            double m = -INFINITY;
            for (int x1 = 0; x1 < n; ++x1) {
                m = fmax(m, T[(long long)x1 * n + y2] - axis_cost(h1, hst, x1 - y1, inv_kappa, inv_eps));
            }
            double s = 0.0;
            for (int x1 = 0; x1 < n; ++x1) {
                s += exp(T[(long long)x1 * n + y2] - axis_cost(h1, hst, x1 - y1, inv_kappa, inv_eps) - m);
            }
            t += nu[o] * (-(m + log(s)) - 1.0);
        }
        term[o] = t;
    }
}

cudaError_t launch_dual_terms(const double* phi, const double* mu, const double* logmu, const double* nu, int n,
                              double eps, double kappa, double* T, double* term, cudaStream_t st,
                              const double* h1, const double* h2, int hst) {
    const long long n2 = (long long)n * n;
    const int grid = (int)std::min<long long>((n2 + 255) / 256, 148 * 32);
    k_dual_pass1<<<grid, 256, 0, st>>>(phi, logmu, n, 1.0 / eps, 1.0 / kappa, T, h2, hst);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_dual_pass2<<<grid, 256, 0, st>>>(T, nu, mu, phi, n, 1.0 / eps, 1.0 / kappa, term, h1, hst);
    return cudaGetLastError();
}

}  // namespace dd
