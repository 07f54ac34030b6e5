// sor.cu -- SURVEY §8 row f4: the Subset-of-Regressors (SGPR) operator
// through the same mBCG ("Programmability"; row access for
// pivoted Cholesky, App. B):
//   K_SoR = K_XU (K_UU + j I)^{-1} K_UX,  j = 1e-6 s (reading R28),
//   Khat_SoR = K_SoR + sigma^2 I.
// With K_UU + jI = Lu Lu^T and Bs = Lu^{-1} K_UX (m x n; built as W K_UX with
// W = Lu^{-1}, a register-tiled fp64 product), K_SoR = Bs^T Bs, so
//   * the blackbox matmul is two skinny products: T = Bs D (m x c, summed over
//     rows, all-reduced across ranks) and V = Bs^T T (row-local) -- no
//     all-gather of D, HBM-bound on Bs (2 * 8 m n bytes per product);
//   * diag(K_SoR)_i = |Bs[:, i]|^2 and row p of K_SoR = Bs[:, p]^T Bs (O(nm)),
//     which is the row access the pivoted Cholesky needs.
// Bs is built once per call, replicated on every rank (like L).
#include <algorithm>
#include <cmath>

#include "bbmm_internal.cuh"

namespace bbmm {

namespace {

__device__ double kval64(int kind, const float *__restrict__ xa, const float *__restrict__ xb, int d,
                         const double *__restrict__ inv_ls2, double s) {
    double r2 = 0.0;
    for (int q = 0; q < d; q++) {
        const double df = (double)xa[q] - (double)xb[q];
        r2 += df * df * inv_ls2[q];
    }
    if (kind == BBMM_RBF) return s * exp(-0.5 * r2);
    const double r = sqrt(r2), sr = sqrt(5.0) * r;
    return s * (1.0 + sr + (5.0 / 3.0) * r2) * exp(-sr);
}

// Kuu[a][b] = k(u_a, u_b) + j delta_ab
__global__ void k_sor_kuu(int kind, const float *__restrict__ U, int64_t m, int d,
                          const double *__restrict__ inv_ls2, double s, double jit,
                          double *__restrict__ Kuu) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e / m, b = e - a * m;
        Kuu[e] = kval64(kind, U + a * d, U + b * d, d, inv_ls2, s) + (a == b ? jit : 0.0);
    }
}

// In-place lower Cholesky of the m x m row-major matrix (one block, left-looking by
// columns: column j's entries below the diagonal in parallel).  status = 1 if not PD.
__global__ void k_sor_chol(double *__restrict__ A, int m, int *status) {
    __shared__ double djj;
    for (int j = 0; j < m; j++) {
        if (threadIdx.x == 0) {
            double s = A[(int64_t)j * m + j];
            for (int q = 0; q < j; q++) s -= A[(int64_t)j * m + q] * A[(int64_t)j * m + q];
            if (!(s > 0.0)) *status = 1;
            djj = sqrt(fmax(s, 1e-300));
            A[(int64_t)j * m + j] = djj;
        }
        __syncthreads();
        for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) {
            double t = A[(int64_t)i * m + j];
            for (int q = 0; q < j; q++) t -= A[(int64_t)i * m + q] * A[(int64_t)j * m + q];
            A[(int64_t)i * m + j] = t / djj;
        }
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += blockDim.x)
        if (e % m > e / m) A[e] = 0.0;
}

// W = Lu^{-1} (lower triangular, m x m): thread j solves Lu w = e_j down its column.
__global__ void k_sor_trinv(const double *__restrict__ Lu, int m, double *__restrict__ W) {
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        for (int a = 0; a < m; a++) {
            double v = (a == j) ? 1.0 : 0.0;
            if (a >= j) {
                const double *La = Lu + (int64_t)a * m;
                for (int b = j; b < a; b++) v -= La[b] * W[(int64_t)b * m + j];
                v /= La[a];
            }
            W[(int64_t)a * m + j] = v;
        }
    }
}

// Bs = W K_UX (m x n): 64 x 64 output tile per block, 4 x 4 per thread (fp64 FMA),
// K-loop over 16-wide slices of the inducing points; the K_UX slice is evaluated on
// the fly from X and U (never stored), W is lower triangular so b runs to the tile's
// last row only.
__global__ void __launch_bounds__(256)
k_sor_bs(int kind, const float *__restrict__ X, int64_t n, int d, const float *__restrict__ U,
         int m, const double *__restrict__ inv_ls2, double s, const double *__restrict__ W,
         double *__restrict__ Bs) {
    __shared__ double Ws[64][17];
    __shared__ double Ks[16][65];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t I0 = (int64_t)blockIdx.x * 64;
    const int A0 = blockIdx.y * 64;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[r][q] = 0.0;
    const int bmax = min(m, A0 + 64);
    for (int B0 = 0; B0 < bmax; B0 += 16) {
        __syncthreads();
        for (int e = threadIdx.x; e < 64 * 16; e += 256) {
            const int aa = e >> 4, bb = e & 15;
            const int a = A0 + aa, b = B0 + bb;
            Ws[aa][bb] = (a < m && b < m) ? W[(int64_t)a * m + b] : 0.0;
        }
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int bb = e >> 6, ii = e & 63;
            const int b = B0 + bb;
            const int64_t i = I0 + ii;
            Ks[bb][ii] = (b < m && i < n) ? kval64(kind, X + i * d, U + (int64_t)b * d, d, inv_ls2, s)
                                          : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int bb = 0; bb < 16; bb++) {
            double w[4], kx[4];
#pragma unroll
            for (int r = 0; r < 4; r++) w[r] = Ws[ty * 4 + r][bb];
#pragma unroll
            for (int q = 0; q < 4; q++) kx[q] = Ks[bb][tx * 4 + q];
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int q = 0; q < 4; q++) acc[r][q] = fma(w[r], kx[q], acc[r][q]);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int a = A0 + ty * 4 + r;
        if (a >= m) continue;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t i = I0 + tx * 4 + q;
            if (i < n) Bs[(int64_t)a * n + i] = acc[r][q];
        }
    }
}

int sgrid(int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 8 * kNumSMs));
}

}  // namespace

void sor_setup(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const float *U, int m,
               const Hyper &h, double *Bs) {
    BBMM_REQUIRE(m >= 1 && m <= kMaxInducing, "m (inducing points) must be in [1, 512]");
    cudaStream_t sm = ctx->stream;
    Workspace &ws = ctx->ws;
    double inv_ls2[kMaxDim];
    for (int q = 0; q < d; q++) {
        const double l = h.ls[h.n_ls == 1 ? 0 : q];
        inv_ls2[q] = 1.0 / (l * l);
    }
    double *inv_d = (double *)ws.get("sor_inv_ls2", sizeof(inv_ls2));
    BBMM_CUDA(cudaMemcpyAsync(inv_d, inv_ls2, sizeof(double) * d, cudaMemcpyHostToDevice, sm));
    double *Lu = (double *)ws.get("sor_Lu", (size_t)m * m * 8);
    int *status = (int *)ws.get("sor_status", sizeof(int));
    BBMM_CUDA(cudaMemsetAsync(status, 0, sizeof(int), sm));
    k_sor_kuu<<<sgrid((int64_t)m * m), 256, 0, sm>>>(h.kind, U, m, d, inv_d, h.s, 1e-6 * h.s, Lu);
    k_sor_chol<<<1, 256, 0, sm>>>(Lu, m, status);
    double *W = (double *)ws.get("sor_W", (size_t)m * m * 8);
    k_sor_trinv<<<1, 512, 0, sm>>>(Lu, m, W);
    const dim3 grid((unsigned)ceil_div(n, 64), (unsigned)ceil_div(m, 64));
    k_sor_bs<<<grid, 256, 0, sm>>>(h.kind, X, n, d, U, m, inv_d, h.s, W, Bs);
    BBMM_LAUNCH_CHECK();
    ctx->launches += 4;
    int st_h = 0;
    BBMM_CUDA(cudaMemcpyAsync(&st_h, status, sizeof(int), cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaStreamSynchronize(sm));
    if (st_h) throw Error{BBMM_ERR_NUMERIC, "K_UU + jitter is not positive definite"};
}

}  // namespace bbmm
