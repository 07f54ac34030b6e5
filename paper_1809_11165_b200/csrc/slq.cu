// slq.cu -- Lanczos tridiagonals from the mBCG coefficients (App. A display
// PAPER.md:468-475, reading R8) and stochastic Lanczos quadrature of
// log|Phat^{-1} Khat| (Eq. 5-6, runtime PAPER.md:521-528,
// weights by reading R12).  One block per probe: builds T_i (size m_i <= p),
// runs an implicit-shift QL eigensolve (Wilkinson shift) tracking only the
// first row of the eigenvector matrix (all that e_1^T log(T) e_1 needs,
// PAPER.md:525), then est_i = omega_i sum_j v0_j^2 log(lambda_j).
// fp64 throughout; O(t p^2) work -- latency-bound and negligible.
#include <cmath>

#include "bbmm_internal.cuh"

namespace bbmm {

namespace {

constexpr int kMaxP = 256;

// Implicit QL on (dg[0..m), e[0..m-1)) where e[i] couples i and i+1.
// z0 = first row of the accumulated rotations.  Returns false if it fails
// to converge.
__device__ bool tridiag_ql(int m, double *dg, double *e, double *z0) {
    for (int i = 0; i < m; i++) z0[i] = (i == 0) ? 1.0 : 0.0;
    if (m > 0) e[m - 1] = 0.0;
    for (int l = 0; l < m; l++) {
        int it = 0;
        while (true) {
            int mm = l;
            for (; mm < m - 1; mm++) {
                double dd = fabs(dg[mm]) + fabs(dg[mm + 1]);
                if (fabs(e[mm]) <= 2.220446049250313e-16 * dd) break;
            }
            if (mm == l) break;
            if (++it > 60) return false;
            // Wilkinson-type shift from the leading 2x2 block at l
            double g = (dg[l + 1] - dg[l]) / (2.0 * e[l]);
            double r = hypot(g, 1.0);
            g = dg[mm] - dg[l] + e[l] / (g + copysign(r, g));
            double s = 1.0, c = 1.0, p = 0.0;
            int i = mm - 1;
            bool early = false;
            for (; i >= l; i--) {
                double f = s * e[i], b = c * e[i];
                // T's entries are O(1/alpha) (no overflow): plain sqrt is enough and has a
                // much shorter dependency chain than hypot on this latency-bound path
                r = sqrt(fma(f, f, g * g));
                e[i + 1] = r;
                if (r == 0.0) {   // underflow: split and restart
                    dg[i + 1] -= p;
                    e[mm] = 0.0;
                    early = true;
                    break;
                }
                const double rinv = 1.0 / r;
                s = f * rinv;
                c = g * rinv;
                g = dg[i + 1] - p;
                r = (dg[i] - g) * s + 2.0 * c * b;
                p = s * r;
                dg[i + 1] = g + p;
                g = c * r - b;
                // rotate columns i, i+1 of the eigenvector matrix (row 0 only)
                double zf = z0[i + 1];
                z0[i + 1] = s * z0[i] + c * zf;
                z0[i] = c * z0[i] - s * zf;
            }
            if (early) continue;
            dg[l] -= p;
            e[l] = g;
            e[mm] = 0.0;
        }
    }
    return true;
}

// ahist/bhist: p x c (row j = iteration j); iters[c]; omega[c] (= rho0).
// One block per probe (thread 0 works): the QL sweeps of different probes take
// different paths, so running them as lanes of one warp would serialise them.
__global__ void k_slq(const double *__restrict__ ahist, const double *__restrict__ bhist,
                      const int *__restrict__ iters, const double *__restrict__ omega, int p,
                      int c, int col0, double *__restrict__ per_probe, int *status) {
    const int i = blockIdx.x;
    if (threadIdx.x != 0) return;
    const int col = col0 + i;
    const int m = min(iters[col], kMaxP);
    double dg[kMaxP], e[kMaxP], z0[kMaxP];
    for (int jj = 0; jj < m; jj++) {
        double a = ahist[(int64_t)jj * c + col];
        dg[jj] = 1.0 / a;
        if (jj > 0) dg[jj] += bhist[(int64_t)(jj - 1) * c + col] / ahist[(int64_t)(jj - 1) * c + col];
        if (jj < m - 1) e[jj] = sqrt(bhist[(int64_t)jj * c + col]) / a;
    }
    if (!tridiag_ql(m, dg, e, z0)) atomicExch(status, (int)BBMM_ERR_NUMERIC);
    double est = 0.0;
    for (int jj = 0; jj < m; jj++) {
        if (!(dg[jj] > 0.0)) {   // Ritz value <= 0: not positive definite
            atomicExch(status, (int)BBMM_ERR_NUMERIC);
            continue;
        }
        est += z0[jj] * z0[jj] * log(dg[jj]);
    }
    per_probe[i] = est * omega[col];
}

// (1/t) sum of the per-probe estimates, fixed order
__global__ void k_slq_sum(const double *__restrict__ per_probe, int t, double *__restrict__ out) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int q = 0; q < t; q++) s += per_probe[q];
    *out = s / (double)t;
}

}  // namespace

void slq_logdet(bbmm_ctx_s *ctx, const double *alpha_d, const double *beta_d, const int *iters_d,
                const double *omega_d, int p, int c, int col0, int t, double *out_d,
                int *status_d) {
    BBMM_REQUIRE(p <= kMaxP, "max_iter too large for the tridiagonal eigensolver (<= 256)");
    BBMM_REQUIRE(t <= 63, "too many probes");
    double *pp = (double *)ctx->ws.get("slq_per_probe", 64 * 8);
    k_slq<<<t, 32, 0, ctx->stream>>>(alpha_d, beta_d, iters_d, omega_d, p, c, col0, pp, status_d);
    k_slq_sum<<<1, 32, 0, ctx->stream>>>(pp, t, out_d);
    BBMM_LAUNCH_CHECK();
    ctx->launches += 2;
}

}  // namespace bbmm
