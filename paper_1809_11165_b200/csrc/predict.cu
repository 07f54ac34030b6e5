// predict.cu -- SURVEY §8 row f1: GP predictive mean and pointwise latent
// variance, Eq. 1, zero prior mean (reading R19):
//   mean(x*) = k_{X x*}^T Khat^{-1} y
//   var(x*)  = k(x*, x*) - k_{X x*}^T Khat^{-1} k_{X x*}
// Every solve is an mBCG solve (the same mbcg_run and blackbox matmul as the
// MLL path) with the rank-k pivoted-Cholesky preconditioner and no probes,
// batched PRED_COLS right-hand sides at a time: [y | k_{X x*_0..15}] first,
// then 17 test columns per batch (17 = a tensor-core-supported width; unused
// columns are zero and freeze at once).  The kernel columns k_{X x*} are
// evaluated in fp64 from the raw inputs, i.e. the definition, so only the
// solves carry the blackbox matmul's precision.
#include <algorithm>
#include <cmath>
#include <vector>

#include "bbmm_internal.cuh"

namespace bbmm {

namespace {

// B[i * ldb + col0 + q] = k(x_{r0+i}, x*_{q0+q}), fp64 (RBF or Matern-5/2)
__global__ void k_cross_cols(int kind, const float *__restrict__ X, int64_t r0, int64_t nloc,
                             int d, const float *__restrict__ Xs, int64_t q0, int m,
                             const double *__restrict__ inv_ls2, double s, double *__restrict__ B,
                             int ldb, int col0) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / m;
        const int q = (int)(e - i * m);
        const float *xi = X + (r0 + i) * d, *xs = Xs + (q0 + q) * d;
        double r2 = 0.0;
        for (int a = 0; a < d; a++) {
            const double df = (double)xi[a] - (double)xs[a];
            r2 += df * df * inv_ls2[a];
        }
        double kv;
        if (kind == BBMM_RBF) {
            kv = s * exp(-0.5 * r2);
        } else {
            const double r = sqrt(r2), sr = sqrt(5.0) * r;
            kv = s * (1.0 + sr + (5.0 / 3.0) * r2) * exp(-sr);
        }
        B[i * ldb + col0 + q] = kv;
    }
}

__global__ void k_y_col(const float *__restrict__ y, int64_t r0, int64_t nloc,
                        double *__restrict__ B, int ldb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x)
        B[i * ldb] = (double)y[r0 + i];
}

__global__ void k_take_col(const double *__restrict__ U, int ldu, int64_t nloc,
                           double *__restrict__ a) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = U[i * ldu];
}

// Per block: part[blk][q] = sum_i B[i][col0+q] a_i, part[blk][m+q] = sum_i B[i][col0+q] U[i][col0+q]
// (fixed-order warp then block reduction: deterministic).
constexpr int kPredMaxM = 17;
__global__ void __launch_bounds__(256)
k_pred_dots(const double *__restrict__ B, const double *__restrict__ U, int ld, int col0, int m,
            const double *__restrict__ a, int64_t nloc, double *__restrict__ part) {
    double sm_[kPredMaxM], sv_[kPredMaxM];
#pragma unroll
    for (int q = 0; q < kPredMaxM; q++) sm_[q] = sv_[q] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ai = a[i];
#pragma unroll
        for (int q = 0; q < kPredMaxM; q++) {
            if (q < m) {
                const double b = B[i * ld + col0 + q];
                sm_[q] = fma(b, ai, sm_[q]);
                if (U) sv_[q] = fma(b, U[i * ld + col0 + q], sv_[q]);
            }
        }
    }
    __shared__ double wp[8][2 * kPredMaxM];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kPredMaxM; q++) {
        double x = sm_[q], y = sv_[q];
        for (int o = 16; o > 0; o >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, o);
            y += __shfl_xor_sync(0xffffffffu, y, o);
        }
        if (lane == 0) { wp[warp][q] = x; wp[warp][kPredMaxM + q] = y; }
    }
    __syncthreads();
    if (threadIdx.x < 2 * m) {
        const int q = threadIdx.x < m ? threadIdx.x : kPredMaxM + threadIdx.x - m;
        double acc = 0.0;
        for (int w = 0; w < 8; w++) acc += wp[w][q];
        part[(int64_t)blockIdx.x * 2 * m + threadIdx.x] = acc;
    }
}

// mean[q0+q] = red[q];  var[q0+q] = s - red[m+q]  (k(x*, x*) = s: stationary kernels)
__global__ void k_pred_finish(const double *__restrict__ red, int m, double s, int64_t q0,
                              double *__restrict__ mean, double *__restrict__ var) {
    const int q = threadIdx.x;
    if (q < m) {
        mean[q0 + q] = red[q];
        if (var) var[q0 + q] = s - red[m + q];
    }
}

// dst[i * ldd + dcol0 + q] = src[i * lds + scol0 + q]  (q < m)
__global__ void k_copy_cols(const double *__restrict__ src, int lds, int scol0, int m,
                            int64_t nloc, double *__restrict__ dst, int64_t ldd, int64_t dcol0) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / m;
        const int q = (int)(e - i * m);
        dst[i * ldd + dcol0 + q] = src[i * lds + scol0 + q];
    }
}

// G[q][r] = sum_i Kq[i][q] U[i][r] over the local rows (ns x ns, fp64): 16 x 16 output tiles,
// 32-row chunks of both operands staged in shared memory, fixed summation order.
__global__ void __launch_bounds__(256)
k_gram(const double *__restrict__ Kq, const double *__restrict__ U, int64_t ns, int64_t nloc,
       double *__restrict__ G) {
    __shared__ double ka[32][17], ub[32][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t q = (int64_t)blockIdx.y * 16 + ty, r = (int64_t)blockIdx.x * 16 + tx;
    double acc = 0.0;
    for (int64_t i0 = 0; i0 < nloc; i0 += 32) {
        for (int e = threadIdx.x; e < 32 * 16; e += 256) {
            const int ii = e >> 4, c = e & 15;
            const int64_t i = i0 + ii;
            const int64_t qq = (int64_t)blockIdx.y * 16 + c, rr = (int64_t)blockIdx.x * 16 + c;
            ka[ii][c] = (i < nloc && qq < ns) ? Kq[i * ns + qq] : 0.0;
            ub[ii][c] = (i < nloc && rr < ns) ? U[i * ns + rr] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int ii = 0; ii < 32; ii++) acc = fma(ka[ii][ty], ub[ii][tx], acc);
        __syncthreads();
    }
    if (q < ns && r < ns) G[q * ns + r] = acc;
}

// cov[q][r] = k(x*_q, x*_r) - G[q][r], kernel values in fp64 from the raw inputs
__global__ void k_cov_finish(int kind, const float *__restrict__ Xs, int d, int64_t ns,
                             const double *__restrict__ inv_ls2, double s,
                             const double *__restrict__ G, double *__restrict__ cov) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ns * ns;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / ns, r = e - q * ns;
        const float *a = Xs + q * d, *b = Xs + r * d;
        double r2 = 0.0;
        for (int t = 0; t < d; t++) {
            const double df = (double)a[t] - (double)b[t];
            r2 += df * df * inv_ls2[t];
        }
        double kv;
        if (kind == BBMM_RBF) {
            kv = s * exp(-0.5 * r2);
        } else {
            const double rr = sqrt(r2), sr = sqrt(5.0) * rr;
            kv = s * (1.0 + sr + (5.0 / 3.0) * r2) * exp(-sr);
        }
        cov[e] = kv - G[e];
    }
}

int pgrid(int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 8 * kNumSMs));
}

}  // namespace

void predict_run(bbmm_ctx_s *ctx, const float *X, const float *y, int64_t n, int d,
                 const float *Xstar, int64_t nstar, const Hyper &h, bool stored, int k,
                 int max_iter, double tol, double *mean, double *var, double *cov) {
    cudaStream_t sm = ctx->stream;
    Workspace &ws = ctx->ws;
    constexpr int CW = kPredMaxM;                  // right-hand sides per mBCG call
    const RowRange rr = local_rows(ctx, n);
    const int64_t nloc = rr.count();
    const int dp = pad_dim(d), ds = (dp + 3) & ~3;
    float *Xs = (float *)ws.get("Xs", (size_t)n * ds * 4);
    scale_inputs(ctx, X, n, d, h, Xs, dp);

    // preconditioner (as for the MLL: pivoted Cholesky of K_XX, Woodbury)
    double *L = (double *)ws.get("L", (size_t)std::max(k, 1) * n * 8);
    int k_used = 0;
    double resid = 0.0;
    std::vector<int64_t> piv(std::max(k, 1), -1);
    if (k > 0) pivchol(ctx, X, n, d, h, k, L, piv.data(), &k_used, &resid);
    double *cholC = (double *)ws.get("cholC", (size_t)std::max(k, 1) * std::max(k, 1) * 8);
    double *ldp = (double *)ws.get("logdet_pre", 8);
    precond_setup(ctx, L, n, k > 0 ? k_used : 0, h.noise_var, cholC, ldp);
    float *Kst = nullptr;
    TcOperand tcop = prepare_operator(ctx, stored, X, Xs, dp, n, d, CW, h, rr.r0, nloc,
                                      rr.nb * ctx->nranks, &Kst);
    MbcgArgs a{Xs, dp, h.kind, h.s, tcop, Kst, n, rr.r0, nloc, rr.nb, h.noise_var, L,
               k > 0 ? k_used : 0, CW, max_iter, tol};

    double inv_ls2[kMaxDim];
    for (int q = 0; q < d; q++) {
        const double l = h.ls[h.n_ls == 1 ? 0 : q];
        inv_ls2[q] = 1.0 / (l * l);
    }
    double *inv_d = (double *)ws.get("pred_inv_ls2", sizeof(inv_ls2));
    BBMM_CUDA(cudaMemcpyAsync(inv_d, inv_ls2, sizeof(double) * d, cudaMemcpyHostToDevice, sm));
    const int64_t nl1 = std::max<int64_t>(nloc, 1);
    double *B = (double *)ws.get("pred_B", (size_t)nl1 * CW * 8);
    double *alpha = (double *)ws.get("pred_alpha", (size_t)nl1 * 8);
    const int nblk = pgrid(nl1);
    double *part = (double *)ws.get("pred_part", (size_t)nblk * 2 * CW * 8);
    double *red = (double *)ws.get("pred_red", 2 * CW * 8);
    auto cross = [&](int64_t q0, int m, int col0) {
        if (nloc > 0 && m > 0) {
            k_cross_cols<<<pgrid(nloc * m), 256, 0, sm>>>(h.kind, X, rr.r0, nloc, d, Xstar, q0,
                                                            m, inv_d, h.s, B, CW, col0);
            ctx->launches++;
        }
    };
    auto dots = [&](const double *U, int col0, int m, int64_t q0) {
        if (nloc > 0) {
            k_pred_dots<<<nblk, 256, 0, sm>>>(B, U, CW, col0, m, alpha, nloc, part);
            ctx->launches++;
            reduce_blocks(ctx, part, nblk, 2 * m, red);
        } else {
            BBMM_CUDA(cudaMemsetAsync(red, 0, 2 * m * 8, sm));
        }
        allreduce_sum(ctx, red, (size_t)2 * m);
        k_pred_finish<<<1, 32, 0, sm>>>(red, m, h.s, q0, mean, U ? var : nullptr);
        ctx->launches++;
    };

    // covariance: keep every test column k_{X x*_q} and its solve (local rows x nstar)
    const bool solves = var != nullptr || cov != nullptr;
    double *Kq = cov ? (double *)ws.get("pred_Kq", (size_t)nl1 * nstar * 8) : nullptr;
    double *Ust = cov ? (double *)ws.get("pred_Ust", (size_t)nl1 * nstar * 8) : nullptr;
    auto keep = [&](const double *U, int col0, int m, int64_t q0) {
        if (!cov || nloc == 0 || m == 0) return;
        k_copy_cols<<<pgrid(nloc * m), 256, 0, sm>>>(B, CW, col0, m, nloc, Kq, nstar, q0);
        k_copy_cols<<<pgrid(nloc * m), 256, 0, sm>>>(U, CW, col0, m, nloc, Ust, nstar, q0);
        ctx->launches += 2;
    };

    // batch 0: [y | first test columns] (variance / covariance) or [y] alone (mean only)
    BBMM_CUDA(cudaMemsetAsync(B, 0, (size_t)nl1 * CW * 8, sm));
    if (nloc > 0) {
        k_y_col<<<pgrid(nloc), 256, 0, sm>>>(y, rr.r0, nloc, B, CW);
        ctx->launches++;
    }
    const int m0 = solves ? (int)std::min<int64_t>(nstar, CW - 1) : 0;
    cross(0, m0, 1);
    MbcgOut o;
    mbcg_run(ctx, a, B, CW, cholC, o);
    if (nloc > 0) {
        k_take_col<<<pgrid(nloc), 256, 0, sm>>>(o.U_d, CW, nloc, alpha);
        ctx->launches++;
    }
    if (solves) {
        if (m0 > 0) {
            dots(o.U_d, 1, m0, 0);
            keep(o.U_d, 1, m0, 0);
        }
        // later batches: CW test columns each, solved together
        for (int64_t q0 = m0; q0 < nstar; q0 += CW) {
            const int m = (int)std::min<int64_t>(nstar - q0, CW);
            BBMM_CUDA(cudaMemsetAsync(B, 0, (size_t)nl1 * CW * 8, sm));
            cross(q0, m, 0);
            MbcgOut ob;
            mbcg_run(ctx, a, B, CW, cholC, ob);
            dots(ob.U_d, 0, m, q0);
            keep(ob.U_d, 0, m, q0);
        }
        if (cov) {
            double *G = (double *)ws.get("pred_G", (size_t)nstar * nstar * 8);
            if (nloc > 0) {
                const dim3 gg((unsigned)ceil_div(nstar, 16), (unsigned)ceil_div(nstar, 16));
                k_gram<<<gg, 256, 0, sm>>>(Kq, Ust, nstar, nloc, G);
                ctx->launches++;
            } else {
                BBMM_CUDA(cudaMemsetAsync(G, 0, (size_t)nstar * nstar * 8, sm));
            }
            allreduce_sum(ctx, G, (size_t)nstar * nstar);
            k_cov_finish<<<pgrid(nstar * nstar), 256, 0, sm>>>(h.kind, Xstar, d, nstar, inv_d,
                                                               h.s, G, cov);
            ctx->launches++;
        }
    } else {
        // mean only: k_{X x*}^T alpha, no further solves
        for (int64_t q0 = 0; q0 < nstar; q0 += CW) {
            const int m = (int)std::min<int64_t>(nstar - q0, CW);
            cross(q0, m, 0);
            dots(nullptr, 0, m, q0);
        }
    }
    BBMM_LAUNCH_CHECK();
}

}  // namespace bbmm
