/*
 * bbmm_oracle.c -- plain, slow, fp64 CPU ORACLE for the BBMM mBCG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1809_11165_b200/, include/bbmm.h) never calls it,
 * and it shares no code, header, table or helper with the CUDA path.
 *
 * Source of truth: /root/reference/PAPER.md (arXiv 1809.11165), cited as
 * P:<line> with the section / algorithm / equation it falls in.  Where the
 * paper is garbled or ambiguous the reading taken is the one listed in
 * DESIGN.md "Readings" (R1..R26 = SURVEY.md §8c Q1..Q26).
 *
 * Everything is IEEE fp64, row-major, sequential sums in index order, no
 * blocking, no symmetry tricks, no expanded-distance tricks.  Compiled with
 * -ffp-contract=off so that a*b+c is two roundings, as written.  OpenMP is
 * used only to distribute independent output rows over host cores; every
 * output element is computed by one thread in the order written below, so
 * results do not depend on the thread count.
 *
 * Parity status of each function: see DESIGN.md "Oracle pins".  Every
 * function below is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_RBF 0
#define ORC_MATERN52 1

#define ORC_OK 0
#define ORC_ERR_ARG 2
#define ORC_ERR_NUMERIC 4

/* ------------------------------------------------------------------------ */
/* Kernel functions.                                                         */
/* P:612 (Background, "Popular kernels include the RBF kernel ... and the    */
/* Matern family"): the RBF formula is garbled in the paper; reading R1 uses */
/* the squared distance, k = s exp(-r^2/2), r^2 = sum_q (x_q-x'_q)^2/l_q^2    */
/* (ARD: one l_q per dimension).  Matern-5/2 (R2, not printed in the paper): */
/* k = s (1 + sqrt5 r + 5 r^2/3) exp(-sqrt5 r).                              */
/* ------------------------------------------------------------------------ */

static double sq_dist_scaled(int d, const double *xi, const double *xj,
                             const double *ls, int n_ls)
{
    double r2 = 0.0;
    for (int q = 0; q < d; q++) {
        double l = (n_ls == 1) ? ls[0] : ls[q];
        double diff = (xi[q] - xj[q]) / l;
        r2 += diff * diff;
    }
    return r2;
}

static double kernel_of_r2(int kind, double r2, double s)
{
    if (kind == ORC_RBF)
        return s * exp(-0.5 * r2);
    double r = sqrt(r2);
    double sr = sqrt(5.0) * r;
    return s * (1.0 + sr + (5.0 / 3.0) * r2) * exp(-sr);
}

double orc_kernel(int kind, int d, const double *xi, const double *xj,
                  int n_ls, const double *ls, double s)
{
    return kernel_of_r2(kind, sq_dist_scaled(d, xi, xj, ls, n_ls), s);
}

/* Derivatives w.r.t. theta = (log l_1..log l_{n_ls}, log s) of k(x_a,x_b),
 * reading R3 (log-parameterisation).  out has n_ls + 1 entries.
 *   RBF:    dk/dlog l_q = k * diff_q^2   (iso: k * r^2),   dk/dlog s = k
 *   Matern: dk/dlog l_q = s (5/3)(1 + sqrt5 r) exp(-sqrt5 r) * diff_q^2
 *           (iso: ... * r^2),                              dk/dlog s = k
 * (chain rule through r^2 = sum diff_q^2, diff_q = (x_aq - x_bq)/l_q).      */
void orc_kernel_grad(int kind, int d, const double *xa, const double *xb,
                     int n_ls, const double *ls, double s, double *out)
{
    double r2 = 0.0;
    double diff2[64];
    for (int q = 0; q < d; q++) {
        double l = (n_ls == 1) ? ls[0] : ls[q];
        double diff = (xa[q] - xb[q]) / l;
        diff2[q < 64 ? q : 63] = diff * diff;
        r2 += diff * diff;
    }
    double k = kernel_of_r2(kind, r2, s);
    double g;  /* common factor multiplying diff_q^2 */
    if (kind == ORC_RBF) {
        g = k;
    } else {
        double r = sqrt(r2);
        double sr = sqrt(5.0) * r;
        g = s * (5.0 / 3.0) * (1.0 + sr) * exp(-sr);
    }
    if (n_ls == 1) {
        out[0] = g * r2;
    } else {
        for (int q = 0; q < d; q++)
            out[q] = g * diff2[q];
    }
    out[n_ls] = k;
}

/* ------------------------------------------------------------------------ */
/* Hyperparameters                                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int kind, d, n_ls;
    double ls[64];
    double s, noise_var;
    const double *X;   /* n x d fp64 */
    int64_t n;
} hyper_t;

static int hyper_init(hyper_t *h, int kind, const double *X, int64_t n, int d,
                      int n_ls, const double *log_ls, double log_s,
                      double log_noise)
{
    if (d < 1 || d > 64 || n < 1 || (n_ls != 1 && n_ls != d) ||
        (kind != ORC_RBF && kind != ORC_MATERN52))
        return ORC_ERR_ARG;
    h->kind = kind; h->d = d; h->n_ls = n_ls; h->X = X; h->n = n;
    for (int q = 0; q < n_ls; q++) h->ls[q] = exp(log_ls[q]);
    h->s = exp(log_s);
    h->noise_var = exp(2.0 * log_noise);   /* sigma^2 = exp(2 log sigma), R3 */
    return ORC_OK;
}

static double *upcast_X(const float *X32, int64_t n, int d)
{
    double *X = (double *)malloc(sizeof(double) * (size_t)n * d);
    for (int64_t i = 0; i < n * d; i++) X[i] = (double)X32[i];
    return X;
}

/* ------------------------------------------------------------------------ */
/* Blackbox matmul with Khat = K_XX + sigma^2 I  ("only requires a     */
/* routine to perform matrix-multiplications with the kernel matrix";        */
/* P:706-708 "This multiplication takes O(n^2 t) time").  Matrix-free.       */
/* out[r][col] = sum_j k(x_{rows[r]}, x_j) M[j][col] + sigma^2 M[rows[r]][col]*/
/* ------------------------------------------------------------------------ */
static void khat_matmul_rows(const hyper_t *h, const double *M, int c,
                             const int64_t *rows, int64_t nrows, double *out)
{
    const int64_t n = h->n;
    const int d = h->d;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t i = rows ? rows[r] : r;
        double *o = out + r * c;
        for (int col = 0; col < c; col++) o[col] = 0.0;
        const double *xi = h->X + i * d;
        for (int64_t j = 0; j < n; j++) {
            double kij = orc_kernel(h->kind, d, xi, h->X + j * d, h->n_ls,
                                    h->ls, h->s);
            const double *mj = M + j * c;
            for (int col = 0; col < c; col++) o[col] += kij * mj[col];
        }
        for (int col = 0; col < c; col++) o[col] += h->noise_var * M[i * c + col];
    }
}

void orc_kernel_matmul(int kind, const float *X32, int64_t n, int d, int n_ls,
                       const double *log_ls, double log_s, double log_noise,
                       const double *M, int c, const int64_t *rows,
                       int64_t nrows, double *out)
{
    hyper_t h;
    double *X = upcast_X(X32, n, d);
    if (hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, log_noise) == ORC_OK)
        khat_matmul_rows(&h, M, c, rows, rows ? nrows : n, out);
    free(X);
}

/* Derivative matmuls dK/dtheta_q . M for q over (lengthscales, outputscale):
 * out[q][r][col] = sum_j dK_q[rows[r], j] M[j][col]   (P:515-516, P:683
 * "a single matrix multiply with the derivative").  sigma's derivative
 * 2 sigma^2 I is diagonal and handled by the caller.                        */
static void dk_matmul_rows(const hyper_t *h, const double *M, int c,
                           const int64_t *rows, int64_t nrows, double *out)
{
    const int64_t n = h->n;
    const int d = h->d;
    const int nq = h->n_ls + 1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t i = rows ? rows[r] : r;
        double g[65];
        for (int q = 0; q < nq; q++)
            for (int col = 0; col < c; col++)
                out[((int64_t)q * nrows + r) * c + col] = 0.0;
        const double *xi = h->X + i * d;
        for (int64_t j = 0; j < n; j++) {
            orc_kernel_grad(h->kind, d, xi, h->X + j * d, h->n_ls, h->ls, h->s, g);
            const double *mj = M + j * c;
            for (int q = 0; q < nq; q++) {
                double *o = out + ((int64_t)q * nrows + r) * c;
                for (int col = 0; col < c; col++) o[col] += g[q] * mj[col];
            }
        }
    }
}

void orc_dkernel_matmul(int kind, const float *X32, int64_t n, int d, int n_ls,
                        const double *log_ls, double log_s, const double *M,
                        int c, const int64_t *rows, int64_t nrows, double *out)
{
    hyper_t h;
    double *X = upcast_X(X32, n, d);
    if (hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, 0.0) == ORC_OK)
        dk_matmul_rows(&h, M, c, rows, rows ? nrows : n, out);
    free(X);
}

/* ------------------------------------------------------------------------ */
/* Pivoted Cholesky, App. B: greedy rank-one Schur updates with   */
/* the maximum remaining diagonal as pivot (Harbrecht's rule).        */
/* Without explicit permutations: diag <- diag(K); for m < k:                */
/*   p_m = argmax diag (ties -> lowest index, R14); stop if diag[p_m] <= tol */
/*   L[:,m] = (K[:,p_m] - L[:,:m] L[p_m,:m]^T) / sqrt(diag[p_m])             */
/*   diag  -= L[:,m]^2 ;  diag[p_m] = 0                                      */
/* L is n x k row-major (row i = L_{i,0..k-1}), original row order.          */
/* Complexity O(rho(K) k^2) with rho the cost of one row.        */
/* ------------------------------------------------------------------------ */
typedef void (*row_fn)(const void *ctx, int64_t i, double *out);

static int pivchol_generic(row_fn row, const void *ctx, const double *diag0,
                           int64_t n, int k, double stop_tol, double *L,
                           int64_t *piv, int *k_used, double *resid)
{
    double *diag = (double *)malloc(sizeof(double) * n);
    double *krow = (double *)malloc(sizeof(double) * n);
    memcpy(diag, diag0, sizeof(double) * n);
    for (int64_t i = 0; i < n * k; i++) L[i] = 0.0;
    int m;
    for (m = 0; m < k; m++) {
        int64_t p = 0;
        for (int64_t i = 1; i < n; i++)
            if (diag[i] > diag[p]) p = i;          /* strict > : lowest index on ties */
        if (!(diag[p] > stop_tol)) break;           /* numerical rank reached (R23) */
        piv[m] = p;
        double piv_val = diag[p];
        double sq = sqrt(piv_val);
        row(ctx, p, krow);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            double acc = krow[i];
            for (int mm = 0; mm < m; mm++)
                acc = acc - L[i * k + mm] * L[p * k + mm];
            L[i * k + m] = acc / sq;
        }
        for (int64_t i = 0; i < n; i++) {
            double lim = L[i * k + m];
            diag[i] = diag[i] - lim * lim;
        }
        diag[p] = 0.0;
    }
    for (int mm = m; mm < k; mm++) piv[mm] = -1;
    *k_used = m;
    double tr = 0.0;
    for (int64_t i = 0; i < n; i++) tr += diag[i];
    *resid = tr;
    free(diag);
    free(krow);
    return ORC_OK;
}

typedef struct { const double *K; int64_t n; } dense_ctx;
static void dense_row(const void *ctx, int64_t i, double *out)
{
    const dense_ctx *c = (const dense_ctx *)ctx;
    memcpy(out, c->K + i * c->n, sizeof(double) * c->n);
}

int orc_pivchol_dense(const double *K, int64_t n, int k, double *L,
                      int64_t *piv, int *k_used, double *resid)
{
    if (n < 1 || k < 0 || k > n) return ORC_ERR_ARG;
    double *diag = (double *)malloc(sizeof(double) * n);
    double dmax = 0.0;
    for (int64_t i = 0; i < n; i++) {
        diag[i] = K[i * n + i];
        if (diag[i] > dmax) dmax = diag[i];
    }
    dense_ctx ctx = {K, n};
    int st = pivchol_generic(dense_row, &ctx, diag, n, k, 1e-12 * dmax, L, piv,
                             k_used, resid);
    free(diag);
    return st;
}

static void kernel_row(const void *ctx, int64_t i, double *out)
{
    const hyper_t *h = (const hyper_t *)ctx;
    const double *xi = h->X + i * h->d;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < h->n; j++)
        out[j] = orc_kernel(h->kind, h->d, xi, h->X + j * h->d, h->n_ls, h->ls, h->s);
}

static int pivchol_kernel(const hyper_t *h, int k, double *L, int64_t *piv,
                          int *k_used, double *resid)
{
    double *diag = (double *)malloc(sizeof(double) * h->n);
    for (int64_t i = 0; i < h->n; i++)   /* stationary kernels: k(x,x) = s */
        diag[i] = orc_kernel(h->kind, h->d, h->X + i * h->d, h->X + i * h->d,
                             h->n_ls, h->ls, h->s);
    /* Pivchol is of K_XX without sigma^2 (R16); stop tol 1e-12 s.   */
    int st = pivchol_generic(kernel_row, h, diag, h->n, k, 1e-12 * h->s, L, piv,
                             k_used, resid);
    free(diag);
    return st;
}

int orc_pivchol_kernel(int kind, const float *X32, int64_t n, int d, int n_ls,
                       const double *log_ls, double log_s, int k, double *L,
                       int64_t *piv, int *k_used, double *resid)
{
    hyper_t h;
    if (k < 0 || k > n) return ORC_ERR_ARG;
    double *X = upcast_X(X32, n, d);
    int st = hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, 0.0);
    if (st == ORC_OK) st = pivchol_kernel(&h, k, L, piv, k_used, resid);
    free(X);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Preconditioner Phat = L L^T + sigma^2 I.                           */
/* Woodbury (App. B, sign corrected, R10):                         */
/*   Phat^{-1} R = (R - L C^{-1} L^T R) / sigma^2,  C = sigma^2 I_k + L^T L   */
/* Determinant lemma (sign corrected, R11):                        */
/*   log|Phat| = log|C| + (n - k) log sigma^2                                 */
/* k < 0 encodes "no preconditioner": P = I, log|P| = 0 (footnote P:197-200);*/
/* k = 0 columns (rank exhausted) is the valid limit P = sigma^2 I.          */
/* ------------------------------------------------------------------------ */

/* dense Cholesky of a k x k SPD matrix, lower factor in place (textbook).   */
static int chol_small(double *A, int k)
{
    for (int j = 0; j < k; j++) {
        double s = A[j * k + j];
        for (int m = 0; m < j; m++) s -= A[j * k + m] * A[j * k + m];
        if (!(s > 0.0)) return ORC_ERR_NUMERIC;
        double ljj = sqrt(s);
        A[j * k + j] = ljj;
        for (int i = j + 1; i < k; i++) {
            double t = A[i * k + j];
            for (int m = 0; m < j; m++) t -= A[i * k + m] * A[j * k + m];
            A[i * k + j] = t / ljj;
        }
        for (int i = 0; i < j; i++) A[i * k + j] = 0.0;
    }
    return ORC_OK;
}

/* L is n x ldl row-major, the first k columns used. */
int orc_precond_setup(const double *L, int64_t n, int ldl, int k,
                      double noise_var, double *cholC, double *logdet)
{
    if (k < 0) { *logdet = 0.0; return ORC_OK; }            /* identity */
    if (k == 0) { *logdet = (double)n * log(noise_var); return ORC_OK; }
    for (int a = 0; a < k; a++)
        for (int b = 0; b < k; b++) {
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += L[i * ldl + a] * L[i * ldl + b];
            cholC[a * k + b] = s + (a == b ? noise_var : 0.0);
        }
    int st = chol_small(cholC, k);
    if (st != ORC_OK) return st;
    double ld = 0.0;
    for (int a = 0; a < k; a++) ld += 2.0 * log(cholC[a * k + a]);
    *logdet = ld + (double)(n - k) * log(noise_var);
    return ORC_OK;
}

void orc_precond_solve(const double *L, int64_t n, int ldl, int k,
                       double noise_var, const double *cholC, const double *R,
                       int c, double *Z)
{
    if (k < 0) { memcpy(Z, R, sizeof(double) * n * c); return; }   /* identity */
    double *W = (double *)calloc((size_t)k * c, sizeof(double));
    /* W = L^T R  (k x c) */
    for (int a = 0; a < k; a++)
        for (int col = 0; col < c; col++) {
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += L[i * ldl + a] * R[i * c + col];
            W[a * c + col] = s;
        }
    /* S = C^{-1} W via forward then backward substitution with chol(C). */
    for (int col = 0; col < c; col++) {
        for (int a = 0; a < k; a++) {
            double s = W[a * c + col];
            for (int b = 0; b < a; b++) s -= cholC[a * k + b] * W[b * c + col];
            W[a * c + col] = s / cholC[a * k + a];
        }
        for (int a = k - 1; a >= 0; a--) {
            double s = W[a * c + col];
            for (int b = a + 1; b < k; b++) s -= cholC[b * k + a] * W[b * c + col];
            W[a * c + col] = s / cholC[a * k + a];
        }
    }
    /* Z = (R - L S) / sigma^2 */
    for (int64_t i = 0; i < n; i++)
        for (int col = 0; col < c; col++) {
            double s = R[i * c + col];
            for (int a = 0; a < k; a++) s -= L[i * ldl + a] * W[a * c + col];
            Z[i * c + col] = s / noise_var;
        }
    free(W);
}

/* ------------------------------------------------------------------------ */
/* Probe vectors.  The paper uses Rademacher probes with E[zz^T] = I */
/* (P:671).  Under the preconditioner (reading R13) z = L eps1 + sigma eps2,  */
/* eps Rademacher, so Cov(z) = Phat.  Counter-based splitmix64 generator      */
/* (DESIGN.md "Probe generator"): h(i,col) = mix(seed + (col (n+k) + i + 1)  */
/* * 0x9E3779B97F4A7C15); sign = +1 if bit 63 of h is 0 else -1; rows i < n   */
/* are eps2[i,col], rows n <= i < n+k are eps1[i-n,col].                      */
/* ------------------------------------------------------------------------ */
uint64_t orc_splitmix64_mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void orc_rademacher(uint64_t seed, int64_t n, int k, int t, int8_t *eps)
{
    for (int64_t i = 0; i < n + k; i++)
        for (int col = 0; col < t; col++) {
            uint64_t ctr = (uint64_t)col * (uint64_t)(n + k) + (uint64_t)i + 1ULL;
            uint64_t h = orc_splitmix64_mix(seed + ctr * 0x9E3779B97F4A7C15ULL);
            eps[i * t + col] = (h >> 63) ? (int8_t)-1 : (int8_t)1;
        }
}

/* Z[i][col] = sum_{m<k} L[i][m] eps1[m][col] + sigma eps2[i][col]           */
void orc_probes(const int8_t *eps, int64_t n, int kgen, int t, const double *L,
                int ldl, int k, double sigma, double *Z)
{
    for (int64_t i = 0; i < n; i++)
        for (int col = 0; col < t; col++) {
            double s = 0.0;
            for (int m = 0; m < k; m++)
                s += L[i * ldl + m] * (double)eps[(n + m) * t + col];
            Z[i * t + col] = s + sigma * (double)eps[i * t + col];
        }
    (void)kgen;
}

/* ------------------------------------------------------------------------ */
/* mBCG, Alg. S2 with the textbook signs and rTz beta of the     */
/* standard PCG it batches (Alg. S1; readings R5, R6, R7, R9):      */
/*   U = 0; R = B; Z = Phat^{-1} R; D = Z; rho_c = sum_i R_ic Z_ic            */
/*   for j = 0..p-1:                                                          */
/*     V = Khat D        */
/*     alpha_c = rho_c / sum_i D_ic V_ic        */
/*     U += diag(alpha) D ; R -= diag(alpha) V    */
/*     record alpha_j ; relres_c = ||R_c|| / ||B_c||                           */
/*     column converged (relres_c < tol, or rho'_c = 0 i.e. R_c = 0 exactly)  */
/*     -> frozen, no beta_j recorded                           (R9)    */
/*     Z = Phat^{-1} R ; rho'_c = sum R Z ; beta_c = rho'/rho    */
/*     record beta_j ; D = Z + diag(beta) D ; rho = rho'        */
/* Outputs: U (n x c), alpha/beta (p x c, row j = iteration j), iters[c] =    */
/* number of alphas recorded for column c, relres[c], rho0[c] = z^T P^-1 z.   */
/* ------------------------------------------------------------------------ */
typedef void (*op_fn)(const void *ctx, const double *M, int c, double *out);

typedef struct {
    const double *L; int64_t n; int ldl; int k; double noise_var;
    double *cholC;
} precond_t;

static int mbcg_generic(op_fn op, const void *opctx, const precond_t *P,
                        int64_t n, const double *B, int c, int p, double tol,
                        double *U, double *alpha, double *beta, int *iters,
                        double *relres, double *rho0, double *relres_hist)
{
    size_t nc = (size_t)n * c;
    double *R = (double *)malloc(sizeof(double) * nc);
    double *Z = (double *)malloc(sizeof(double) * nc);
    double *D = (double *)malloc(sizeof(double) * nc);
    double *V = (double *)malloc(sizeof(double) * nc);
    double *rho = (double *)malloc(sizeof(double) * c);
    double *bnorm = (double *)malloc(sizeof(double) * c);
    int *active = (int *)malloc(sizeof(int) * c);
    int st = ORC_OK;

    memset(U, 0, sizeof(double) * nc);
    memcpy(R, B, sizeof(double) * nc);
    orc_precond_solve(P->L, n, P->ldl, P->k, P->noise_var, P->cholC, R, c, Z);
    memcpy(D, Z, sizeof(double) * nc);
    for (int col = 0; col < c; col++) {
        double s = 0.0, b2 = 0.0;
        for (int64_t i = 0; i < n; i++) {
            s += R[i * c + col] * Z[i * c + col];
            b2 += B[i * c + col] * B[i * c + col];
        }
        rho[col] = s;
        rho0[col] = s;
        bnorm[col] = sqrt(b2);
        active[col] = bnorm[col] > 0.0;
        iters[col] = 0;
        relres[col] = active[col] ? 1.0 : 0.0;
    }
    for (int64_t i = 0; i < (int64_t)p * c; i++) {
        alpha[i] = 0.0; beta[i] = 0.0;
        if (relres_hist) relres_hist[i] = 0.0;
    }

    for (int j = 0; j < p; j++) {
        int any = 0;
        for (int col = 0; col < c; col++) any |= active[col];
        if (!any) break;
        op(opctx, D, c, V);
        for (int col = 0; col < c; col++) {
            if (!active[col]) continue;
            double dv = 0.0;
            for (int64_t i = 0; i < n; i++) dv += D[i * c + col] * V[i * c + col];
            double a = rho[col] / dv;
            if (!(a > 0.0) || !isfinite(a)) {
                /* reading R9/R24: a residual exhausted below fp64's range (rho <= 1e-250
                   rho_0, e.g. p far past convergence) is frozen like R = 0 exactly;
                   otherwise the operator is not positive definite: breakdown */
                if (rho[col] <= 1e-250 * rho0[col]) { active[col] = 0; continue; }
                st = ORC_ERR_NUMERIC; goto done;
            }
            double r2 = 0.0;
            for (int64_t i = 0; i < n; i++) {
                U[i * c + col] += a * D[i * c + col];
                R[i * c + col] -= a * V[i * c + col];
                r2 += R[i * c + col] * R[i * c + col];
            }
            alpha[(int64_t)j * c + col] = a;
            iters[col] = j + 1;
            relres[col] = sqrt(r2) / bnorm[col];
            if (relres_hist) relres_hist[(int64_t)j * c + col] = relres[col];
            if (relres[col] < tol) active[col] = 0;
        }
        orc_precond_solve(P->L, n, P->ldl, P->k, P->noise_var, P->cholC, R, c, Z);
        for (int col = 0; col < c; col++) {
            if (!active[col]) continue;
            double rz = 0.0;
            for (int64_t i = 0; i < n; i++) rz += R[i * c + col] * Z[i * c + col];
            if (rz == 0.0) { active[col] = 0; continue; }   /* exact convergence (R = 0) */
            double b = rz / rho[col];
            beta[(int64_t)j * c + col] = b;
            for (int64_t i = 0; i < n; i++)
                D[i * c + col] = Z[i * c + col] + b * D[i * c + col];
            rho[col] = rz;
        }
    }
done:
    free(R); free(Z); free(D); free(V); free(rho); free(bnorm); free(active);
    return st;
}

typedef struct { const double *A; int64_t n; } dense_op_ctx;
static void dense_op(const void *ctx, const double *M, int c, double *out)
{
    const dense_op_ctx *d = (const dense_op_ctx *)ctx;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < d->n; i++)
        for (int col = 0; col < c; col++) {
            double s = 0.0;
            for (int64_t j = 0; j < d->n; j++) s += d->A[i * d->n + j] * M[j * c + col];
            out[i * c + col] = s;
        }
}

static void khat_op(const void *ctx, const double *M, int c, double *out)
{
    khat_matmul_rows((const hyper_t *)ctx, M, c, NULL, ((const hyper_t *)ctx)->n, out);
}

/* mBCG on an explicit dense SPD A (tests), preconditioner L (n x k), sigma^2. */
int orc_mbcg_dense(const double *A, int64_t n, const double *L, int k,
                   double noise_var, const double *B, int c, int p, double tol,
                   double *U, double *alpha, double *beta, int *iters,
                   double *relres, double *rho0, double *relres_hist)
{
    /* k == 0 here means "no preconditioner" (P = I). */
    precond_t P = {L, n, k, k > 0 ? k : -1, noise_var, NULL};
    double ld;
    P.cholC = (double *)malloc(sizeof(double) * (k > 0 ? k * k : 1));
    int st = orc_precond_setup(L, n, k, P.k, noise_var, P.cholC, &ld);
    if (st == ORC_OK) {
        dense_op_ctx ctx = {A, n};
        st = mbcg_generic(dense_op, &ctx, &P, n, B, c, p, tol, U, alpha, beta,
                          iters, relres, rho0, relres_hist);
    }
    free(P.cholC);
    return st;
}

/* mBCG on Khat = K_XX + sigma^2 I (matrix-free) with preconditioner L. */
int orc_mbcg_kernel(int kind, const float *X32, int64_t n, int d, int n_ls,
                    const double *log_ls, double log_s, double log_noise,
                    const double *L, int k, const double *B, int c, int p,
                    double tol, double *U, double *alpha, double *beta,
                    int *iters, double *relres, double *rho0, double *relres_hist)
{
    hyper_t h;
    double *X = upcast_X(X32, n, d);
    int st = hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, log_noise);
    if (st == ORC_OK) {
        precond_t P = {L, n, k, k > 0 ? k : -1, h.noise_var, NULL};
        double ld;
        P.cholC = (double *)malloc(sizeof(double) * (k > 0 ? k * k : 1));
        st = orc_precond_setup(L, n, k, P.k, h.noise_var, P.cholC, &ld);
        if (st == ORC_OK)
            st = mbcg_generic(khat_op, &h, &P, n, B, c, p, tol, U, alpha, beta,
                              iters, relres, rho0, relres_hist);
        free(P.cholC);
    }
    free(X);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Lanczos tridiagonal from the CG coefficients, App. A observation matrix   */
/* display P:468-475 (reading R8, 0-based):                                   */
/*   diag_0 = 1/alpha_0 ; diag_j = 1/alpha_j + beta_{j-1}/alpha_{j-1}         */
/*   off_j  = sqrt(beta_j)/alpha_j      (j = 0..m-2)                           */
/* ------------------------------------------------------------------------ */
void orc_tridiag_from_cg(int m, const double *alpha, const double *beta,
                         int stride, double *diag, double *off)
{
    for (int j = 0; j < m; j++) {
        double a = alpha[(int64_t)j * stride];
        diag[j] = 1.0 / a;
        if (j > 0) {
            double ap = alpha[(int64_t)(j - 1) * stride];
            double bp = beta[(int64_t)(j - 1) * stride];
            diag[j] += bp / ap;
        }
        if (j < m - 1)
            off[j] = sqrt(beta[(int64_t)j * stride]) / a;
    }
}

/* Symmetric eigendecomposition of the m x m tridiagonal T ("we        */
/* eigendecompose T_i = V_i Lambda_i V_i^T").  Plain cyclic Jacobi on the     */
/* dense matrix (textbook; slow, robust, no tridiagonal-specific tricks).     */
/* Outputs eigenvalues (ascending) and the first row of V (V^T e_1).  */
int orc_tridiag_eig(int m, const double *diag, const double *off,
                    double *evals, double *v0)
{
    double *A = (double *)calloc((size_t)m * m, sizeof(double));
    double *Q = (double *)calloc((size_t)m * m, sizeof(double));
    for (int i = 0; i < m; i++) {
        A[i * m + i] = diag[i];
        if (i + 1 < m) { A[i * m + i + 1] = off[i]; A[(i + 1) * m + i] = off[i]; }
        Q[i * m + i] = 1.0;
    }
    int st = ORC_ERR_NUMERIC;
    for (int sweep = 0; sweep < 100; sweep++) {
        double offn = 0.0, tot = 0.0;
        for (int i = 0; i < m; i++)
            for (int j = 0; j < m; j++) {
                tot += A[i * m + j] * A[i * m + j];
                if (i != j) offn += A[i * m + j] * A[i * m + j];
            }
        if (offn <= 1e-30 * tot || offn == 0.0) { st = ORC_OK; break; }
        for (int pp = 0; pp < m - 1; pp++)
            for (int q = pp + 1; q < m; q++) {
                double apq = A[pp * m + q];
                if (apq == 0.0) continue;
                /* rotation zeroing A[p][q] (Golub & Van Loan, sym. Schur 2x2) */
                double tau = (A[q * m + q] - A[pp * m + pp]) / (2.0 * apq);
                double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double cs = 1.0 / sqrt(1.0 + tt * tt), sn = tt * cs;
                for (int r = 0; r < m; r++) {       /* A <- A J (columns p,q) */
                    double arp = A[r * m + pp], arq = A[r * m + q];
                    A[r * m + pp] = cs * arp - sn * arq;
                    A[r * m + q] = sn * arp + cs * arq;
                }
                for (int r = 0; r < m; r++) {       /* A <- J^T A (rows p,q) */
                    double apr = A[pp * m + r], aqr = A[q * m + r];
                    A[pp * m + r] = cs * apr - sn * aqr;
                    A[q * m + r] = sn * apr + cs * aqr;
                }
                for (int r = 0; r < m; r++) {       /* Q <- Q J */
                    double qrp = Q[r * m + pp], qrq = Q[r * m + q];
                    Q[r * m + pp] = cs * qrp - sn * qrq;
                    Q[r * m + q] = sn * qrp + cs * qrq;
                }
            }
    }
    /* sort ascending (selection sort), carry the first row of Q along. */
    int *idx = (int *)malloc(sizeof(int) * m);
    for (int i = 0; i < m; i++) idx[i] = i;
    for (int i = 0; i < m; i++)
        for (int j = i + 1; j < m; j++)
            if (A[idx[j] * m + idx[j]] < A[idx[i] * m + idx[i]]) {
                int tmp = idx[i]; idx[i] = idx[j]; idx[j] = tmp;
            }
    for (int i = 0; i < m; i++) {
        evals[i] = A[idx[i] * m + idx[i]];
        v0[i] = Q[0 * m + idx[i]];
    }
    free(idx); free(A); free(Q);
    return st;
}

/* SLQ (Eq. 5-6; runtime App. A) with the preconditioned */
/* log-det adjustment and reading R12 for the weights:            */
/*   log|Phat^{-1} Khat| ~= (1/t) sum_i omega_i sum_j V_i[0,j]^2 log lam_ij   */
/* omega_i = z_i^T Phat^{-1} z_i (= rho0 of probe column i).                  */
/* Columns col0..col0+t-1 of the (p x c) alpha/beta arrays are probes.        */
int orc_slq_logdet(int p, int c, int col0, int t, const int *iters,
                   const double *alpha, const double *beta, const double *omega,
                   double *logdet_ratio, double *per_probe)
{
    double *dg = (double *)malloc(sizeof(double) * (p + 1));
    double *of = (double *)malloc(sizeof(double) * (p + 1));
    double *ev = (double *)malloc(sizeof(double) * (p + 1));
    double *v0 = (double *)malloc(sizeof(double) * (p + 1));
    double acc = 0.0;
    int st = ORC_OK;
    for (int i = 0; i < t; i++) {
        int col = col0 + i;
        int m = iters[col];
        double est = 0.0;
        if (m > 0) {
            orc_tridiag_from_cg(m, alpha + col, beta + col, c, dg, of);
            int s2 = orc_tridiag_eig(m, dg, of, ev, v0);
            if (s2 != ORC_OK) st = s2;
            for (int j = 0; j < m; j++) {
                if (!(ev[j] > 0.0)) { st = ORC_ERR_NUMERIC; continue; }
                est += v0[j] * v0[j] * log(ev[j]);
            }
        }
        est *= omega[col];
        if (per_probe) per_probe[i] = est;
        acc += est;
    }
    *logdet_ratio = acc / (double)t;
    free(dg); free(of); free(ev); free(v0);
    return st;
}

/* ------------------------------------------------------------------------ */
/* One-call exact-GP marginal log likelihood and gradient (Eq. 2,  */
/* constants/signs by reading R4; "a single call to mBCG").         */
/*   mll  = -1/2 (y^T u0 + log|Khat| + n log 2 pi)                            */
/*   dmll/dtheta_q = 1/2 (u0^T dKhat_q u0 - tau_q)                            */
/*   tau_q = (1/t) sum_i (Khat^{-1} z_i)^T dKhat_q (Phat^{-1} z_i)  (Eq. 4,   */
/*           P:669-684, with the P^{-1} correction of reading R13)            */
/*   log|Khat| = SLQ(Phat^{-1}Khat) + log|Phat|                               */
/* theta = (log l_1..log l_{n_ls}, log s, log sigma); grad has n_ls + 2.      */
/* stats[0..7] = logdet_precond, logdet_ratio, quad_y (y^T u0), resid_trace,  */
/*               k_used, max iters, logdet, sum over probes of omega.         */
/* ------------------------------------------------------------------------ */
int orc_mll_and_grad(int kind, const float *X32, const float *y32, int64_t n,
                     int d, int n_ls, const double *log_ls, double log_s,
                     double log_noise, int t, int k, int p, double tol,
                     uint64_t seed, const int8_t *eps_opt, double *mll,
                     double *grad, double *stats, double *U_out,
                     int64_t *piv_out, double *alpha_out, double *beta_out,
                     int *iters_out)
{
    hyper_t h;
    if (t < 1 || p < 1 || k < 0 || k > n || tol < 0) return ORC_ERR_ARG;
    double *X = upcast_X(X32, n, d);
    int st = hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, log_noise);
    if (st != ORC_OK) { free(X); return st; }
    const int c = t + 1;
    const double sigma = exp(log_noise);
    double *L = (double *)malloc(sizeof(double) * (size_t)n * (k > 0 ? k : 1));
    int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int k_used = 0;
    double resid = 0.0;
    /* 1. pivoted Cholesky of K_XX */
    if (k > 0) st = pivchol_kernel(&h, k, L, piv, &k_used, &resid);
    else { for (int64_t i = 0; i < n; i++) resid += h.s; }
    /* 2. preconditioner (Woodbury / det lemma) */
    double *cholC = (double *)malloc(sizeof(double) * (k > 0 ? k * k : 1));
    double ld_pre = 0.0;
    /* k == 0: no preconditioner (P = I, footnote P:197-200) */
    const int kp = (k > 0) ? k_used : -1;
    if (st == ORC_OK) st = orc_precond_setup(L, n, k > 0 ? k : 1, kp, h.noise_var, cholC, &ld_pre);
    /* 3. probes z = L eps1 + sigma eps2 and B = [y | Z] */
    int8_t *eps = (int8_t *)malloc((size_t)(n + k) * t);
    if (eps_opt) memcpy(eps, eps_opt, (size_t)(n + k) * t);
    else orc_rademacher(seed, n, k, t, eps);
    double *Zp = (double *)malloc(sizeof(double) * (size_t)n * t);
    /* k == 0: plain Rademacher probes z = eps2 */
    orc_probes(eps, n, k, t, L, k > 0 ? k : 1, k_used, k > 0 ? sigma : 1.0, Zp);
    double *B = (double *)malloc(sizeof(double) * (size_t)n * c);
    for (int64_t i = 0; i < n; i++) {
        B[i * c] = (double)y32[i];
        for (int col = 0; col < t; col++) B[i * c + 1 + col] = Zp[i * t + col];
    }
    /* 4. one mBCG call on [y, z_1..z_t] */
    double *U = (double *)malloc(sizeof(double) * (size_t)n * c);
    double *al = (double *)malloc(sizeof(double) * (size_t)p * c);
    double *be = (double *)malloc(sizeof(double) * (size_t)p * c);
    int *it = (int *)malloc(sizeof(int) * c);
    double *rr = (double *)malloc(sizeof(double) * c);
    double *rho0 = (double *)malloc(sizeof(double) * c);
    if (st == ORC_OK) {
        precond_t P = {L, n, k > 0 ? k : 1, kp, h.noise_var, cholC};
        st = mbcg_generic(khat_op, &h, &P, n, B, c, p, tol, U, al, be, it, rr, rho0, NULL);
    }
    /* 5. SLQ log-det */
    double ld_ratio = 0.0;
    if (st == ORC_OK) st = orc_slq_logdet(p, c, 1, t, it, al, be, rho0, &ld_ratio, NULL);
    double logdet = ld_ratio + ld_pre;
    /* 6. derivative pass: dK_q [Phat^{-1} Z | u0] once */
    double *M = (double *)malloc(sizeof(double) * (size_t)n * c);
    double *Z0 = (double *)malloc(sizeof(double) * (size_t)n * t);
    const int nq = n_ls + 1;
    double *dKM = (double *)malloc(sizeof(double) * (size_t)nq * n * c);
    double quad_y = 0.0;
    if (st == ORC_OK) {
        precond_t P = {L, n, k > 0 ? k : 1, kp, h.noise_var, cholC};
        orc_precond_solve(P.L, n, P.ldl, P.k, P.noise_var, P.cholC, Zp, t, Z0);
        for (int64_t i = 0; i < n; i++) {
            for (int col = 0; col < t; col++) M[i * c + col] = Z0[i * t + col];
            M[i * c + t] = U[i * c + 0];
        }
        dk_matmul_rows(&h, M, c, NULL, n, dKM);
        for (int64_t i = 0; i < n; i++) quad_y += (double)y32[i] * U[i * c];
        for (int q = 0; q < nq; q++) {
            double tau = 0.0, quad = 0.0;
            const double *o = dKM + (int64_t)q * n * c;
            for (int col = 0; col < t; col++)
                for (int64_t i = 0; i < n; i++)
                    tau += U[i * c + 1 + col] * o[i * c + col];
            tau /= (double)t;
            for (int64_t i = 0; i < n; i++) quad += U[i * c] * o[i * c + t];
            grad[q] = 0.5 * (quad - tau);
        }
        /* log sigma: dKhat/dlog sigma = 2 sigma^2 I */
        double tau = 0.0, quad = 0.0;
        for (int col = 0; col < t; col++)
            for (int64_t i = 0; i < n; i++)
                tau += U[i * c + 1 + col] * Z0[i * t + col];
        tau = 2.0 * h.noise_var * tau / (double)t;
        for (int64_t i = 0; i < n; i++) quad += U[i * c] * U[i * c];
        quad *= 2.0 * h.noise_var;
        grad[nq] = 0.5 * (quad - tau);
        *mll = -0.5 * (quad_y + logdet + (double)n * log(2.0 * M_PI));
    }
    if (stats) {
        int mx = 0;
        double om = 0.0;
        for (int col = 0; col < c; col++) if (it[col] > mx) mx = it[col];
        for (int col = 1; col < c; col++) om += rho0[col];
        stats[0] = ld_pre; stats[1] = ld_ratio; stats[2] = quad_y; stats[3] = resid;
        stats[4] = k_used; stats[5] = mx; stats[6] = logdet; stats[7] = om;
    }
    if (U_out) memcpy(U_out, U, sizeof(double) * (size_t)n * c);
    if (piv_out) for (int m = 0; m < k; m++) piv_out[m] = m < k_used ? piv[m] : -1;
    if (alpha_out) memcpy(alpha_out, al, sizeof(double) * (size_t)p * c);
    if (beta_out) memcpy(beta_out, be, sizeof(double) * (size_t)p * c);
    if (iters_out) memcpy(iters_out, it, sizeof(int) * c);
    free(X); free(L); free(piv); free(cholC); free(eps); free(Zp); free(B);
    free(U); free(al); free(be); free(it); free(rr); free(rho0); free(M);
    free(Z0); free(dKM);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Predictions, Eq. 1 with zero prior mean (R19):                 */
/*   mean(x*) = k_{X x*}^T Khat^{-1} y                                        */
/*   var(x*)  = k(x*, x*) - k_{X x*}^T Khat^{-1} k_{X x*}   (pointwise, latent) */
/* All solves from ONE mBCG call on B = [y | k_{X x*_1} .. k_{X x*_ns}] with  */
/* the rank-k pivoted-Cholesky preconditioner and no probes (SPEC "predict":   */
/* "the n* solves performed as one batched mbcg call (probes absent)").       */
/* ------------------------------------------------------------------------ */
static int predict_core(int kind, const float *X32, const float *y32, int64_t n, int d,
                        const float *Xs32, int64_t ns, int n_ls, const double *log_ls,
                        double log_s, double log_noise, int k, int p, double tol,
                        double *mean, double *var, double *cov);

int orc_predict(int kind, const float *X32, const float *y32, int64_t n, int d,
                const float *Xs32, int64_t ns, int n_ls, const double *log_ls,
                double log_s, double log_noise, int k, int p, double tol,
                double *mean, double *var)
{
    return predict_core(kind, X32, y32, n, d, Xs32, ns, n_ls, log_ls, log_s, log_noise, k, p,
                        tol, mean, var, NULL);
}

/* The full predictive covariance between test points (Eq. 1, latent, R27):     */
/*   cov(x*_q, x*_r) = k(x*_q, x*_r) - k_{X x*_q}^T Khat^{-1} k_{X x*_r}                    */
/* from the same single mBCG call (u_r = the solve of column r); ns x ns row-major.       */
int orc_predict_cov(int kind, const float *X32, const float *y32, int64_t n, int d,
                    const float *Xs32, int64_t ns, int n_ls, const double *log_ls,
                    double log_s, double log_noise, int k, int p, double tol,
                    double *mean, double *cov)
{
    if (!cov) return ORC_ERR_ARG;
    return predict_core(kind, X32, y32, n, d, Xs32, ns, n_ls, log_ls, log_s, log_noise, k, p,
                        tol, mean, NULL, cov);
}

static int predict_core(int kind, const float *X32, const float *y32, int64_t n, int d,
                        const float *Xs32, int64_t ns, int n_ls, const double *log_ls,
                        double log_s, double log_noise, int k, int p, double tol,
                        double *mean, double *var, double *cov)
{
    hyper_t h;
    if (n < 1 || ns < 1 || p < 1 || k < 0 || k > n || tol < 0) return ORC_ERR_ARG;
    double *X = upcast_X(X32, n, d);
    double *Xs = upcast_X(Xs32, ns, d);
    int st = hyper_init(&h, kind, X, n, d, n_ls, log_ls, log_s, log_noise);
    if (st != ORC_OK) { free(X); free(Xs); return st; }
    const int64_t c = 1 + ns;
    double *L = (double *)malloc(sizeof(double) * (size_t)n * (k > 0 ? k : 1));
    int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int k_used = 0;
    double resid = 0.0;
    /* 1. preconditioner: pivoted Cholesky of K_XX, Woodbury (as for the MLL) */
    if (k > 0) st = pivchol_kernel(&h, k, L, piv, &k_used, &resid);
    double *cholC = (double *)malloc(sizeof(double) * (k > 0 ? k * k : 1));
    double ld_pre = 0.0;
    const int kp = (k > 0) ? k_used : -1;
    if (st == ORC_OK) st = orc_precond_setup(L, n, k > 0 ? k : 1, kp, h.noise_var, cholC, &ld_pre);
    /* 2. B = [y | k_{X x*_q}] */
    double *B = (double *)malloc(sizeof(double) * (size_t)n * c);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        B[i * c] = (double)y32[i];
        for (int64_t q = 0; q < ns; q++)
            B[i * c + 1 + q] = orc_kernel(kind, d, X + i * d, Xs + q * d, h.n_ls, h.ls, h.s);
    }
    /* 3. one mBCG call */
    double *U = (double *)malloc(sizeof(double) * (size_t)n * c);
    double *al = (double *)malloc(sizeof(double) * (size_t)p * c);
    double *be = (double *)malloc(sizeof(double) * (size_t)p * c);
    int *it = (int *)malloc(sizeof(int) * c);
    double *rr = (double *)malloc(sizeof(double) * c);
    double *rho0 = (double *)malloc(sizeof(double) * c);
    if (st == ORC_OK) {
        precond_t P = {L, n, k > 0 ? k : 1, kp, h.noise_var, cholC};
        st = mbcg_generic(khat_op, &h, &P, n, B, (int)c, p, tol, U, al, be, it, rr, rho0, NULL);
    }
    /* 4. mean_q = k_q . u_0 ; var_q = k(x*_q, x*_q) - k_q . u_q */
    if (st == ORC_OK) {
        for (int64_t q = 0; q < ns; q++) {
            double m = 0.0, v = 0.0;
            for (int64_t i = 0; i < n; i++) {
                m += B[i * c + 1 + q] * U[i * c];
                v += B[i * c + 1 + q] * U[i * c + 1 + q];
            }
            mean[q] = m;
            if (var)
                var[q] = orc_kernel(kind, d, Xs + q * d, Xs + q * d, h.n_ls, h.ls, h.s) - v;
        }
        if (cov) {
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < ns; q++)
                for (int64_t r = 0; r < ns; r++) {
                    double g = 0.0;
                    for (int64_t i = 0; i < n; i++) g += B[i * c + 1 + q] * U[i * c + 1 + r];
                    cov[q * ns + r] =
                        orc_kernel(kind, d, Xs + q * d, Xs + r * d, h.n_ls, h.ls, h.s) - g;
                }
        }
    }
    free(X); free(Xs); free(L); free(piv); free(cholC); free(B); free(U); free(al);
    free(be); free(it); free(rr); free(rho0);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Hyperparameter training ("All methods use the same optimizer        */
/* (Adam)"; settings unstated -> reading R26): `steps` Adam steps (Kingma &  */
/* Ba) on theta = (log l.., log s, log sigma) minimising -mll with the BBMM  */
/* gradient of orc_mll_and_grad, fresh probes each step (seed + step):       */
/*   g = -grad ; m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2                 */
/*   theta -= lr (m / (1 - b1^s)) / (sqrt(v / (1 - b2^s)) + eps)              */
/* trace (steps x (1 + ntheta), may be NULL): row s = [mll(theta_s), theta_s]. */
/* ------------------------------------------------------------------------ */
int orc_train_adam(int kind, const float *X32, const float *y32, int64_t n, int d,
                   int n_ls, const double *theta0, int t, int k, int p, double tol,
                   uint64_t seed, int steps, double lr, double b1, double b2,
                   double eps, double *theta_out, double *trace)
{
    const int nt = n_ls + 2;
    if (steps < 0 || !(lr > 0) || b1 < 0 || b1 >= 1 || b2 < 0 || b2 >= 1 || eps < 0)
        return ORC_ERR_ARG;
    double *th = (double *)malloc(sizeof(double) * nt);
    double *g = (double *)malloc(sizeof(double) * nt);
    double *m1 = (double *)calloc(nt, sizeof(double));
    double *m2 = (double *)calloc(nt, sizeof(double));
    memcpy(th, theta0, sizeof(double) * nt);
    int st = ORC_OK;
    for (int s = 0; s < steps && st == ORC_OK; s++) {
        double mll = 0.0;
        st = orc_mll_and_grad(kind, X32, y32, n, d, n_ls, th, th[n_ls], th[n_ls + 1], t, k, p,
                              tol, seed + (uint64_t)s, NULL, &mll, g, NULL, NULL, NULL, NULL,
                              NULL, NULL);
        if (st != ORC_OK) break;
        if (!isfinite(mll)) { st = ORC_ERR_NUMERIC; break; }
        if (trace) {
            trace[(int64_t)s * (1 + nt)] = mll;
            memcpy(trace + (int64_t)s * (1 + nt) + 1, th, sizeof(double) * nt);
        }
        const double c1 = 1.0 - pow(b1, s + 1), c2 = 1.0 - pow(b2, s + 1);
        for (int q = 0; q < nt; q++) {
            const double gq = -g[q];                   /* minimise -mll */
            m1[q] = b1 * m1[q] + (1.0 - b1) * gq;
            m2[q] = b2 * m2[q] + (1.0 - b2) * gq * gq;
            th[q] -= lr * (m1[q] / c1) / (sqrt(m2[q] / c2) + eps);
        }
    }
    memcpy(theta_out, th, sizeof(double) * nt);
    free(th); free(g); free(m1); free(m2);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Row f4: the Subset-of-Regressors (SGPR) operator through the same mBCG     */
/* ("Programmability"; row access for pivoted Cholesky, App. B      */
/* P:156-171):                                                                */
/*   K_SoR = K_XU (K_UU + j I)^{-1} K_UX ,  Khat_SoR = K_SoR + sigma^2 I       */
/* with m inducing points U and jitter j = 1e-6 s (reading R28).  The oracle  */
/* applies the definition: T = K_UX M, T = (K_UU + jI)^{-1} T (Cholesky       */
/* solve), out = K_XU T (+ sigma^2 M).                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
    hyper_t h;
    int64_t m;
    double *Kxu;   /* n x m */
    double *Luu;   /* m x m lower Cholesky factor of K_UU + j I */
} sor_t;

static int sor_init(sor_t *S, int kind, const double *X, int64_t n, int d, const double *U,
                    int64_t m, int n_ls, const double *log_ls, double log_s, double log_noise)
{
    int st = hyper_init(&S->h, kind, X, n, d, n_ls, log_ls, log_s, log_noise);
    if (st != ORC_OK) return st;
    S->m = m;
    S->Kxu = (double *)malloc(sizeof(double) * (size_t)n * m);
    S->Luu = (double *)malloc(sizeof(double) * (size_t)m * m);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        for (int64_t a = 0; a < m; a++)
            S->Kxu[i * m + a] = orc_kernel(kind, d, X + i * d, U + a * d, S->h.n_ls, S->h.ls, S->h.s);
    for (int64_t a = 0; a < m; a++)
        for (int64_t b = 0; b < m; b++)
            S->Luu[a * m + b] = orc_kernel(kind, d, U + a * d, U + b * d, S->h.n_ls, S->h.ls, S->h.s)
                                + (a == b ? 1e-6 * S->h.s : 0.0);
    return chol_small(S->Luu, (int)m);
}

static void sor_free(sor_t *S) { free(S->Kxu); free(S->Luu); }

/* x <- (L L^T)^{-1} x for the m x m factor L (c right-hand sides, x is m x c) */
static void chol_solve_mc(const double *L, int64_t m, double *x, int c)
{
    for (int col = 0; col < c; col++) {
        for (int64_t a = 0; a < m; a++) {
            double s = x[a * c + col];
            for (int64_t b = 0; b < a; b++) s -= L[a * m + b] * x[b * c + col];
            x[a * c + col] = s / L[a * m + a];
        }
        for (int64_t a = m - 1; a >= 0; a--) {
            double s = x[a * c + col];
            for (int64_t b = a + 1; b < m; b++) s -= L[b * m + a] * x[b * c + col];
            x[a * c + col] = s / L[a * m + a];
        }
    }
}

/* out = K_SoR M (+ sigma^2 M if with_noise), M n x c */
static void sor_apply(const sor_t *S, const double *M, int c, double *out, int with_noise)
{
    const int64_t n = S->h.n, m = S->m;
    double *T = (double *)calloc((size_t)m * c, sizeof(double));
    for (int64_t i = 0; i < n; i++)
        for (int64_t a = 0; a < m; a++)
            for (int col = 0; col < c; col++) T[a * c + col] += S->Kxu[i * m + a] * M[i * c + col];
    chol_solve_mc(S->Luu, m, T, c);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        for (int col = 0; col < c; col++) {
            double s = 0.0;
            for (int64_t a = 0; a < m; a++) s += S->Kxu[i * m + a] * T[a * c + col];
            out[i * c + col] = with_noise ? s + S->h.noise_var * M[i * c + col] : s;
        }
    free(T);
}

static void sor_op(const void *ctx, const double *M, int c, double *out)
{
    sor_apply((const sor_t *)ctx, M, c, out, 1);
}

/* row i of K_SoR: K_XU (K_UU + jI)^{-1} k_{U x_i} */
static void sor_row(const void *ctx, int64_t i, double *out)
{
    const sor_t *S = (const sor_t *)ctx;
    const int64_t m = S->m;
    double *w = (double *)malloc(sizeof(double) * m);
    memcpy(w, S->Kxu + i * m, sizeof(double) * m);
    chol_solve_mc(S->Luu, m, w, 1);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < S->h.n; j++) {
        double s = 0.0;
        for (int64_t a = 0; a < m; a++) s += S->Kxu[j * m + a] * w[a];
        out[j] = s;
    }
    free(w);
}

int orc_sor_matmul(int kind, const float *X32, int64_t n, int d, const float *U32, int64_t m,
                   int n_ls, const double *log_ls, double log_s, double log_noise,
                   const double *M, int c, int with_noise, double *out)
{
    if (n < 1 || m < 1 || c < 1) return ORC_ERR_ARG;
    double *X = upcast_X(X32, n, d), *U = upcast_X(U32, m, d);
    sor_t S;
    int st = sor_init(&S, kind, X, n, d, U, m, n_ls, log_ls, log_s, log_noise);
    if (st == ORC_OK) sor_apply(&S, M, c, out, with_noise);
    sor_free(&S); free(X); free(U);
    return st;
}

/* pivoted Cholesky of K_SoR through its rows (App. B): diag_i = row_i[i] */
static int pivchol_sor(const sor_t *S, int k, double *L, int64_t *piv, int *k_used, double *resid)
{
    const int64_t n = S->h.n, m = S->m;
    double *diag = (double *)malloc(sizeof(double) * n);
    double *w = (double *)malloc(sizeof(double) * m);
    for (int64_t i = 0; i < n; i++) {
        memcpy(w, S->Kxu + i * m, sizeof(double) * m);
        chol_solve_mc(S->Luu, m, w, 1);
        double s = 0.0;
        for (int64_t a = 0; a < m; a++) s += S->Kxu[i * m + a] * w[a];
        diag[i] = s;
    }
    int st = pivchol_generic(sor_row, S, diag, n, k, 1e-12 * S->h.s, L, piv, k_used, resid);
    free(diag); free(w);
    return st;
}

int orc_pivchol_sor(int kind, const float *X32, int64_t n, int d, const float *U32, int64_t m,
                    int n_ls, const double *log_ls, double log_s, int k, double *L,
                    int64_t *piv, int *k_used, double *resid)
{
    if (k < 0 || k > n) return ORC_ERR_ARG;
    double *X = upcast_X(X32, n, d), *U = upcast_X(U32, m, d);
    sor_t S;
    int st = sor_init(&S, kind, X, n, d, U, m, n_ls, log_ls, log_s, 0.0);
    if (st == ORC_OK) st = pivchol_sor(&S, k, L, piv, k_used, resid);
    sor_free(&S); free(X); free(U);
    return st;
}

/* mBCG on Khat_SoR with a preconditioner L (n x k, e.g. from orc_pivchol_sor) */
int orc_mbcg_sor(int kind, const float *X32, int64_t n, int d, const float *U32, int64_t m,
                 int n_ls, const double *log_ls, double log_s, double log_noise,
                 const double *L, int k, const double *B, int c, int p, double tol,
                 double *Uo, double *alpha, double *beta, int *iters, double *relres,
                 double *rho0, double *relres_hist)
{
    double *X = upcast_X(X32, n, d), *U = upcast_X(U32, m, d);
    sor_t S;
    int st = sor_init(&S, kind, X, n, d, U, m, n_ls, log_ls, log_s, log_noise);
    if (st == ORC_OK) {
        precond_t P = {L, n, k, k > 0 ? k : -1, S.h.noise_var, NULL};
        double ld;
        P.cholC = (double *)malloc(sizeof(double) * (k > 0 ? k * k : 1));
        st = orc_precond_setup(L, n, k, P.k, S.h.noise_var, P.cholC, &ld);
        if (st == ORC_OK)
            st = mbcg_generic(sor_op, &S, &P, n, B, c, p, tol, Uo, alpha, beta, iters, relres,
                              rho0, relres_hist);
        free(P.cholC);
    }
    sor_free(&S); free(X); free(U);
    return st;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
