/*
 * bbmm.h -- C-ABI of the B200-native BBMM hot path (arXiv 1809.11165).
 *
 * The library computes, for an exact Gaussian process with kernel matrix
 * Khat = K(X,X) + sigma^2 I, the three inference terms of the paper's Sec. 4
 * (Khat^{-1} y, log|Khat|, Tr(Khat^{-1} dKhat/dtheta)) with
 * ONE call of modified batched preconditioned conjugate gradients (mBCG,
 * Alg. S2) on the block [y, z_1..z_t],
 * preconditioned by a rank-k pivoted Cholesky factor applied through
 * Woodbury (App. B), and from them the
 * marginal log likelihood and its gradient (Eq. 2).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Pointers named *_d are DEVICE pointers on the context's device, owned by
 *    the caller; pointers named *_h are HOST pointers owned by the caller.
 *    The library owns only its workspace (inside the context).
 *  - Matrices are row-major.  X_d is n x d fp32 (every rank holds all n rows).
 *  - Work is enqueued on the context stream; a call returns after its _h
 *    outputs are written (it synchronises the stream only to deliver them).
 *  - Multi-GPU (bbmm_ctx_set_comm with nranks > 1): rank r owns the rows
 *    [r*nb, min(n, (r+1)*nb)) with nb = ceil(n / nranks) ("local rows").
 *    All ranks call collectively with identical scalar arguments; returned
 *    scalars are identical on all ranks.  Per iteration the library
 *    all-gathers the search directions and all-reduces per-column dot
 *    products over NCCL.
 *  - Hyperparameters theta = (log l_1..log l_{n_ls}, log s, log sigma):
 *    l = lengthscale(s) (n_ls = 1 isotropic, n_ls = d ARD), s = outputscale,
 *    sigma^2 = exp(2 log sigma) = noise variance (reading R3).
 *  - Kernels (readings R1/R2), r^2 = sum_q (x_q - x'_q)^2/l_q^2:
 *      BBMM_RBF:      k = s exp(-r^2 / 2)
 *      BBMM_MATERN52: k = s (1 + sqrt(5) r + 5 r^2 / 3) exp(-sqrt(5) r)
 *  - Errors: every function returns a bbmm_status_t; arguments are validated
 *    before anything is launched (BBMM_ERR_ARG); no exception crosses the
 *    ABI; bbmm_last_error() returns a text description of the last failure
 *    on that context.  Non-convergence within max_iter is NOT an error
 *    (iteration counts / residuals report it); pivoted Cholesky running out
 *    of positive pivots is NOT an error (k_used < k).
 */
#ifndef BBMM_H_
#define BBMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bbmm_ctx_s *bbmm_ctx_t;

typedef enum {
    BBMM_OK = 0,
    BBMM_ERR_ARG = 2,      /* invalid argument (shape, range, null pointer) */
    BBMM_ERR_DATA = 3,     /* non-finite input data */
    BBMM_ERR_NUMERIC = 4,  /* breakdown: alpha <= 0 / non-finite (indefinite
                              operator), Ritz value <= 0, chol(C) failed */
    BBMM_ERR_CUDA = 5,
    BBMM_ERR_NCCL = 6,
    BBMM_ERR_OOM = 7
} bbmm_status_t;

typedef enum { BBMM_RBF = 0, BBMM_MATERN52 = 1 } bbmm_kernel_t;

/* How the blackbox matmul Khat*M is performed:
 * ON-THE-FLY never materialises K (every kernel entry recomputed per matmul);
 * STORED materialises this rank's K row block (local rows x n fp32) once per
 * call and streams it from HBM every iteration. */
typedef enum { BBMM_ONTHEFLY = 0, BBMM_STORED = 1 } bbmm_kmode_t;

/* Arithmetic of the blackbox matmul Khat*D.
 * FP64ACC: kernel values in fp32 (MUFU ex2/sqrt), search directions
 *   D in fp64, products and sums in fp64.  Parity with the fp64 oracle holds
 *   whether or not mBCG has converged by max_iter (a per-iteration fp32
 *   rounding of D is amplified by an unconverged Krylov process).
 * FP32ACC: D rounded to fp32, products summed in fp32 over 16 terms then
 *   folded into fp64.  Faster; parity holds only where mBCG has converged
 *   (SURVEY.md §8c "regime A"). */
/* INT8EXACT (default): tcgen05 tensor cores, slice products summed EXACTLY in
 *   int32 (drained to fp64).  On the fly, RBF (isotropic or ARD): kernel values
 *   (fp32 MUFU ex2) on a 23- or 31-bit fixed-point grid -- 31 bits where the
 *   23-bit grid's per-entry error (5.3e-8 s rms) would put the solves near the
 *   1e-4 bar: sqrt(n) 5.3e-8 s / sigma^2 > 0.8e-4 (the error model of DESIGN.md
 *   §6a: ||du|| / ||u|| ~ sqrt(n) eps / sigma^2) -- D as 31-bit fixed point
 *   (per-column scale), the exponent from an fp16 hi/lo-split tensor-core
 *   distance; any t + 1 <= 33 (padded to the next instantiated column block) with
 *   any d <= 32, and max |x_scaled|^2 <= 16 (precision guard).  On the fly,
 *   Matern-5/2: distances from direct fp32 differences (the expanded form's
 *   ~1e-7 error breaks the parity bars there), kernel values on
 *   the 31-bit grid and 55-bit D (23-bit / 39-bit under INT8EXACT23, which
 *   misses the regime-B bars at full C2); t + 1 <= 64 (chunks of 17), d <= 14.
 *   Stored K (BBMM_STORED, t + 1 <= 33):
 *   K built in fp64 and stored as 30-bit fixed point, D as 55-bit fixed point.
 *   Everything else uses FP64ACC.
 * INT8EXACT31 / INT8EXACT23: INT8EXACT with the on-the-fly RBF grid forced to
 *   31 / 23 bits.  The 31-bit grid keeps the MUFU's kernel values exactly (a
 *   fourth, residual u8 slice of k~): per-entry error 3.3e-8 instead of 5.3e-8
 *   rms at C4 (the grid rounding removed, the MUFU's own error left), which the
 *   north-star solve bar needs at n = 1M; 1.18x the 23-bit
 *   kernel-matmul time.  The derivative pass and the Matern / stored operators
 *   are those of INT8EXACT. */
typedef enum {
    BBMM_MATMUL_FP64ACC = 0,
    BBMM_MATMUL_FP32ACC = 1,
    BBMM_MATMUL_INT8EXACT = 2,
    BBMM_MATMUL_INT8EXACT31 = 3,
    BBMM_MATMUL_INT8EXACT23 = 4
} bbmm_matmul_precision_t;

typedef struct {
    int32_t kind;            /* bbmm_kernel_t */
    int32_t n_ls;            /* 1 (isotropic) or d (ARD) */
    const double *log_ls_h;  /* host, n_ls entries */
    double log_outputscale;  /* log s */
    double log_noise;        /* log sigma */
} bbmm_hyper_t;

/* Diagnostics of one bbmm_mll_and_grad call (host struct). */
typedef struct {
    int32_t iters;           /* K-hat matmuls performed by mBCG */
    int32_t k_used;          /* pivoted-Cholesky rank actually used */
    double logdet_precond;   /* log|Phat| (determinant lemma) */
    double logdet_ratio;     /* SLQ estimate of log|Phat^{-1} Khat| */
    double logdet;           /* log|Khat| = sum of the two */
    double quad_y;           /* y^T Khat^{-1} y (y^T u_0) */
    double resid_trace;      /* tr(K - L L^T) after pivoted Cholesky */
    double relres_y;         /* ||r_y|| / ||y|| at exit */
    double ms_total;         /* device time of the whole call (CUDA events) */
    double ms_pivchol;       /* pivoted Cholesky + preconditioner setup */
    double ms_mbcg;          /* probes + mBCG loop (incl. collectives) */
    double ms_matmul;        /* sum over mBCG iterations of the K-hat*D kernel */
    double ms_slq;           /* tridiagonal eigensolves + SLQ */
    double ms_deriv;         /* derivative pass */
    int32_t matmul_launches; /* K-hat*D kernel launches inside ms_matmul */
    int32_t gpu_launches;    /* library kernels launched by the call */
    int32_t matmul_path;     /* 0 on-the-fly CUDA-core (FP64ACC/FP32ACC),
                                1 stored fp32 K (FP64ACC/FP32ACC), 2 tcgen05 exact on the
                                fly (INT8EXACT), 3 stored K as int8 slices on tcgen05
                                (INT8EXACT, BBMM_STORED) */
    int32_t unconverged;     /* 1 if mBCG had not converged at exit: with tol > 0, some column
                                still above tol after max_iter iterations; with tol == 0,
                                relres_max >= 1e-3 (SURVEY.md §8c "regime B": the Krylov iterate
                                is then sensitive to rounding); NOT an error */
    double relres_max;       /* max over the t + 1 columns of ||r_c|| / ||b_c|| at exit */
    double ms_comm;          /* device time inside the collectives (all-reduces, all-gathers)
                                on the context stream, incl. waiting for peers; 0 single-rank */
    int32_t kgrid_bits;      /* fixed-point grid of the on-the-fly kernel values (matmul_path
                                2): 23 or 31; 0 otherwise */
} bbmm_stats_t;

/* ---- context ----------------------------------------------------------- */

/* Create a context bound to CUDA `device`, enqueueing on `cuda_stream`
 * (a cudaStream_t; NULL = a stream the context creates and owns). */
bbmm_status_t bbmm_ctx_create(int device, void *cuda_stream, bbmm_ctx_t *out);
bbmm_status_t bbmm_ctx_destroy(bbmm_ctx_t ctx);
/* Text of the last error on `ctx` (static storage owned by ctx). */
const char *bbmm_last_error(bbmm_ctx_t ctx);
/* Library version string. */
const char *bbmm_version(void);

/* Multi-GPU: rank 0 calls bbmm_nccl_unique_id, broadcasts the 128 bytes to
 * all ranks (e.g. torch.distributed.broadcast), then every rank calls
 * bbmm_ctx_set_comm (collective; creates an NCCL communicator). */
bbmm_status_t bbmm_nccl_unique_id(void *out_128_bytes);
bbmm_status_t bbmm_ctx_set_comm(bbmm_ctx_t ctx, int nranks, int rank,
                                const void *nccl_unique_id_128_bytes);
/* In-process rank group (SURVEY.md §8e row partition without NCCL): nranks
 * contexts in ONE process, each driven by its own host thread, may share one
 * GPU.  Collectives are synchronous and host-staged (each rank synchronises its
 * stream; sums in rank order, so every rank gets identical bits); a rank that
 * waits more than 120 s for its peers fails with BBMM_ERR_NCCL.  For testing the
 * multi-rank data flow on one GPU -- not a performance path.  The group is owned
 * by the caller and must outlive the contexts that use it.  BBMM_ERR_ARG for
 * nranks < 1, rank outside [0, nranks) or NULL arguments. */
typedef struct bbmm_local_group_s *bbmm_local_group_t;
bbmm_status_t bbmm_local_group_create(int32_t nranks, bbmm_local_group_t *out);
bbmm_status_t bbmm_local_group_destroy(bbmm_local_group_t group);
bbmm_status_t bbmm_ctx_set_local_comm(bbmm_ctx_t ctx, bbmm_local_group_t group,
                                      int32_t rank);
/* Select the matmul arithmetic for subsequent calls on ctx (default INT8EXACT). */
bbmm_status_t bbmm_ctx_set_matmul_precision(bbmm_ctx_t ctx, bbmm_matmul_precision_t p);
/* Row partition of the multi-GPU path: rank owns
 * [*r0, *r1) with blocks of nb = ceil(ceil(n / nranks) / 128) * 128 rows (host
 * arithmetic only, no context or GPU needed; nb may be NULL).  BBMM_ERR_ARG for
 * n < 0, nranks < 1, rank outside [0, nranks) or NULL outputs. */
bbmm_status_t bbmm_row_partition(int64_t n, int32_t nranks, int32_t rank,
                                 int64_t *r0, int64_t *r1, int64_t *nb);
/* Local row range [*r0, *r1) of this rank for problem size n. */
bbmm_status_t bbmm_local_rows(bbmm_ctx_t ctx, int64_t n, int64_t *r0,
                              int64_t *r1);

/* ---- entry points ------------------------------------------------------ */

/* Blackbox matmul V = Khat * D (the K1/K2 kernel
 * alone -- the "kernel-matmul" of the metric).
 *   D_d: n x ncols fp64, leading dim ldd (all n rows, every rank).
 *   V_d: (local rows) x ncols fp64, leading dim ldv.
 *   1 <= ncols <= 64, 1 <= d <= 32. */
bbmm_status_t bbmm_kernel_matmul(bbmm_ctx_t ctx, const float *X_d, int64_t n,
                                 int32_t d, const bbmm_hyper_t *hyper,
                                 bbmm_kmode_t kmode, const double *D_d,
                                 int32_t ncols, int64_t ldd, double *V_d,
                                 int64_t ldv);

/* Rank-k pivoted Cholesky of K_XX (no noise term; App. B PAPER.md:80-135,
 * PAPER.md:729-735), fp64, pivots = argmax of the remaining Schur diagonal
 * with ties broken by the lowest index; stops early when the maximum is
 * <= 1e-12 * s (then k_used < k).  Replicated: every rank computes all n.
 *   L_d: k x n fp64 (row m = column m of the n x k factor, contiguous over
 *        the n points; rows >= k_used are zero).
 *   pivots_h: k int64 (entries >= k_used are -1). */
bbmm_status_t bbmm_pivchol(bbmm_ctx_t ctx, const float *X_d, int64_t n,
                           int32_t d, const bbmm_hyper_t *hyper, int32_t k,
                           double *L_d, int64_t *pivots_h, int32_t *k_used_h,
                           double *resid_trace_h);

/* mBCG (Alg. S2, textbook signs, R5-R9) on
 * Khat with preconditioner Phat = L L^T + sigma^2 I applied via Woodbury
 * (k >= 1) or no preconditioner (k == 0, L_d ignored).
 *   L_d: k x n fp64 as returned by bbmm_pivchol (full n on every rank).
 *   B_d, U_d: (local rows) x ncols fp64, leading dims ldb / ldu.
 *   Columns [ncols - n_tridiag, ncols) are probe columns whose Lanczos
 *   coefficients are returned (all columns' alpha/beta are returned anyway).
 *   tol: a column is frozen once ||r_c|| / ||b_c|| < tol; tol == 0 runs
 *   exactly max_iter iterations.  1 <= ncols <= 64.
 *   alpha_h, beta_h: max_iter x ncols host fp64 (row j = iteration j; 0 where
 *   not computed);  iters_h: ncols int32 (alphas recorded per column);
 *   relres_h: ncols fp64;  rho0_h: ncols fp64 (b^T Phat^{-1} b), may be NULL;
 *   relres_hist_h: max_iter x ncols fp64, row j = ||r_c|| / ||b_c|| after
 *   iteration j (0 once the column is frozen), may be NULL (row f3 study). */
bbmm_status_t bbmm_mbcg(bbmm_ctx_t ctx, const float *X_d, int64_t n, int32_t d,
                        const bbmm_hyper_t *hyper, bbmm_kmode_t kmode,
                        const double *L_d, int32_t k, const double *B_d,
                        int32_t ncols, int64_t ldb, int32_t max_iter,
                        double tol, double *U_d, int64_t ldu, double *alpha_h,
                        double *beta_h, int32_t *iters_h, double *relres_h,
                        double *rho0_h, double *relres_hist_h);

/* One-call exact-GP marginal log likelihood and gradient (north-star entry):
 *   pivchol(k) -> Phat -> probes z_i = L eps1_i + sigma eps2_i (k >= 1; plain
 *   Rademacher eps2_i when k == 0) -> one mBCG on [y, z_1..z_t] -> SLQ
 *   log|Khat| -> one derivative pass -> mll, grad.
 *   mll = -1/2 (y^T u_0 + log|Khat| + n log 2 pi)
 *   grad_q = 1/2 (u_0^T dKhat_q u_0 - (1/t) sum_i u_i^T dKhat_q Phat^{-1} z_i)
 * Inputs: X_d n x d fp32, y_d n fp32 (all rows on every rank).
 *   eps_d: NULL -> probe signs from the counter-based generator with `seed`
 *          (DESIGN.md "Probe generator"); else (n + k) x t int8 in {-1, +1}
 *          device array (rows < n: eps2, rows >= n: eps1).
 *   1 <= t <= 63, 0 <= k <= min(n, 128), max_iter >= 1, tol >= 0.
 * Outputs: mll_h (1), grad_h (n_ls + 2: d/dlog l_q..., d/dlog s,
 *   d/dlog sigma), stats_h (may be NULL).
 * Optional outputs (NULL to skip): U_d (local rows) x (t+1) fp64 solves
 *   [Khat^{-1} y, Khat^{-1} z_1..]; pivots_h (k int64). */
bbmm_status_t bbmm_mll_and_grad(bbmm_ctx_t ctx, const float *X_d,
                                const float *y_d, int64_t n, int32_t d,
                                const bbmm_hyper_t *hyper, bbmm_kmode_t kmode,
                                int32_t t, int32_t k, int32_t max_iter,
                                double tol, uint64_t seed, const int8_t *eps_d,
                                double *mll_h, double *grad_h,
                                bbmm_stats_t *stats_h, double *U_d,
                                int64_t *pivots_h);

/* GP predictions: predictive mean and pointwise latent
 * variance, Eq. 1, zero prior mean (R19):
 *   mean[q] = k_{X x*_q}^T Khat^{-1} y
 *   var[q]  = k(x*_q, x*_q) - k_{X x*_q}^T Khat^{-1} k_{X x*_q}
 * Every solve is an mBCG solve (bbmm_mbcg semantics, no probes) with the
 * rank-k pivoted-Cholesky preconditioner, 17 right-hand sides per call
 * ([y | first 16 test columns], then 17 test columns per call); the kernel
 * columns k_{X x*} are evaluated in fp64 from X and Xstar.
 * Inputs (device, fp32, all rows on every rank): X_d n x d, y_d n,
 *   Xstar_d nstar x d.  0 <= k <= min(n, 128), max_iter >= 1, tol >= 0.
 * Outputs (device, fp64, nstar each, identical on every rank): mean_d; var_d
 *   (NULL: mean only -- one solve of y, no solves of test columns).
 * Errors: BBMM_ERR_ARG (sizes, NULL), BBMM_ERR_DATA (non-finite input),
 *   BBMM_ERR_NUMERIC (mBCG breakdown). */
bbmm_status_t bbmm_predict(bbmm_ctx_t ctx, const float *X_d, const float *y_d,
                           int64_t n, int32_t d, const float *Xstar_d,
                           int64_t nstar, const bbmm_hyper_t *hyper,
                           bbmm_kmode_t kmode, int32_t k, int32_t max_iter,
                           double tol, double *mean_d, double *var_d);

/* The full predictive (latent) covariance between the test points, Eq. 1
 * with zero prior mean (reading R19):
 *   cov[q][r] = k(x*_q, x*_r) - k_{X x*_q}^T Khat^{-1} k_{X x*_r}
 * from the same batched mBCG solves as bbmm_predict (u_r = Khat^{-1} k_{X x*_r}); the
 * contraction K_{*X} U_* runs over this rank's rows and is all-reduced.  Its diagonal is
 * bbmm_predict's var.  Inputs as bbmm_predict, 1 <= nstar <= 8192.  Outputs (device, fp64,
 * identical on every rank): mean_d (nstar), cov_d (nstar x nstar row-major).
 * Errors: as bbmm_predict. */
bbmm_status_t bbmm_predict_cov(bbmm_ctx_t ctx, const float *X_d, const float *y_d,
                               int64_t n, int32_t d, const float *Xstar_d,
                               int64_t nstar, const bbmm_hyper_t *hyper,
                               bbmm_kmode_t kmode, int32_t k, int32_t max_iter,
                               double tol, double *mean_d, double *cov_d);

/* Hyperparameter training ("All methods use
 * the same optimizer (Adam)"; settings by DESIGN.md reading R26): `steps` Adam
 * steps on theta = (log l_1..l_{n_ls}, log s, log sigma) minimising -mll, with
 * the gradient of bbmm_mll_and_grad and fresh probes each step (seed + step):
 *   g = -grad ; m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2 ;
 *   theta -= lr (m / (1 - b1^s)) / (sqrt(v / (1 - b2^s)) + eps)
 * hyper: initial theta (host).  Outputs (host): theta_out_h (n_ls + 2, the
 *   trained theta); trace_h (steps x (n_ls + 3) fp64, may be NULL): row s =
 *   [mll(theta_s), theta_s].  Other arguments as bbmm_mll_and_grad.
 * Errors: as bbmm_mll_and_grad (the failing step is named); BBMM_ERR_ARG for
 *   steps < 0, lr <= 0, b1/b2 outside [0, 1), eps < 0. */
bbmm_status_t bbmm_train_adam(bbmm_ctx_t ctx, const float *X_d, const float *y_d,
                              int64_t n, int32_t d, const bbmm_hyper_t *hyper,
                              bbmm_kmode_t kmode, int32_t t, int32_t k,
                              int32_t max_iter, double tol, uint64_t seed,
                              int32_t steps, double lr, double beta1,
                              double beta2, double eps, double *theta_out_h,
                              double *trace_h);

/* Second operator through the same mBCG (PAPER.md:786-799
 * "Programmability", row access for pivoted Cholesky App. B): the
 * Subset-of-Regressors / SGPR kernel with m inducing points U,
 *   Khat_SoR = K_XU (K_UU + 1e-6 s I)^{-1} K_UX + sigma^2 I   (jitter: reading R28)
 * Builds Bs = Lu^{-1} K_UX (K_UU + jI = Lu Lu^T; m x n fp64, every rank), the
 * rank-k pivoted Cholesky of K_SoR = Bs^T Bs through its rows (k = 0: none), then
 * one mBCG call on B exactly as bbmm_mbcg (B_d, U_d: local rows x ncols fp64).
 * Xu_d: m x d fp32 device, 1 <= m <= 512.  piv_h (k int64), iters_h,
 * relres_h (ncols), relres_hist_h (max_iter x ncols): host, may be NULL.
 * Errors: BBMM_ERR_ARG (sizes / NULL), BBMM_ERR_DATA (non-finite X / Xu),
 *   BBMM_ERR_NUMERIC (K_UU + jI not PD, mBCG breakdown). */
bbmm_status_t bbmm_sor_mbcg(bbmm_ctx_t ctx, const float *X_d, int64_t n, int32_t d,
                            const float *Xu_d, int32_t m,
                            const bbmm_hyper_t *hyper, int32_t k, const double *B_d,
                            int32_t ncols, int64_t ldb, int32_t max_iter,
                            double tol, double *U_d, int64_t ldu, int64_t *piv_h,
                            int32_t *iters_h, double *relres_h,
                            double *relres_hist_h);

#ifdef __cplusplus
}
#endif

#endif /* BBMM_H_ */
