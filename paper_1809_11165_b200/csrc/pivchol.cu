// pivchol.cu -- rank-k pivoted Cholesky of K_XX in fp64 (App. B,
// PAPER.md:80-135; complexity PAPER.md:141-154), the preconditioner factor of
// Sec. 4.1.
//
// Without explicit permutations (Harbrecht's greedy rule):
//   diag <- diag(K) = s ; for m < k:
//     p_m = argmax diag (ties -> lowest index, reading R14);
//     stop if diag[p_m] <= 1e-12 s (numerical rank reached, k_used = m);
//     L[m][:] = (K[p_m][:] - sum_{m'<m} L[m'][:] L[m'][p_m]) / sqrt(diag[p_m]);
//     diag -= L[m][:]^2 ; diag[p_m] = 0.
// Everything is fp64 with explicitly rounded operations (no FMA contraction)
// because pivots must match the fp64 oracle bit-for-bit (reading R15: fp32
// pivots diverge within 1-3 steps).  One kernel per step computes the pivot
// row of K on the fly, the Schur update of L and diag, and the block-partial
// argmax of the updated diagonal; a one-block kernel finishes the argmax.
// Every rank computes all n rows (replicated; no collectives needed).
#include <algorithm>
#include <cmath>

#include <cstdint>

#include "bbmm_internal.cuh"

namespace bbmm {

namespace {

constexpr int kThreads = 256;

struct PivState {
    int64_t piv[kMaxRank];
    double pivval;
    int k_used;
    int stop;
};

__device__ __forceinline__ void argmax_combine(double &v, int64_t &i, double v2, int64_t i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ void block_argmax(double v, int64_t i, double *pv, int64_t *pi) {
    __shared__ double sv[kThreads / 32];
    __shared__ int64_t si[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_down_sync(0xffffffffu, v, o);
        int64_t i2 = __shfl_down_sync(0xffffffffu, i, o);
        argmax_combine(v, i, v2, i2);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sv[w] = v; si[w] = i; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = sv[0];
        int64_t bi = si[0];
        for (int q = 1; q < kThreads / 32; q++) argmax_combine(bv, bi, sv[q], si[q]);
        *pv = bv;
        *pi = bi;
    }
}

// K(x_a, x_b) in fp64, evaluated exactly as written in the method's definition
// (reading R1/R2): diff_q = (x_aq - x_bq)/l_q ; r2 = sum diff_q^2 ;
//   RBF:    s * exp(-0.5 r2)
//   Matern: s * (1 + sqrt5 r + (5/3) r2) * exp(-sqrt5 r)
__device__ double kernel_fp64(int kind, const float *__restrict__ xa, const float *__restrict__ xb,
                              int d, const double *__restrict__ ls, int n_ls, double s) {
    double r2 = 0.0;
    for (int q = 0; q < d; q++) {
        double l = ls[n_ls == 1 ? 0 : q];
        double diff = __ddiv_rn(__dsub_rn((double)xa[q], (double)xb[q]), l);
        r2 = __dadd_rn(r2, __dmul_rn(diff, diff));
    }
    if (kind == BBMM_RBF) return __dmul_rn(s, exp(__dmul_rn(-0.5, r2)));
    double r = __dsqrt_rn(r2);
    double sr = __dmul_rn(__dsqrt_rn(5.0), r);
    double poly = __dadd_rn(__dadd_rn(1.0, sr), __dmul_rn(5.0 / 3.0, r2));
    return __dmul_rn(__dmul_rn(s, poly), exp(-sr));
}

__global__ void k_piv_init(double *__restrict__ diag, int64_t n, double s, double *__restrict__ L,
                           int64_t Ltotal, PivState *st, double *pv, int64_t *pi, int nblk) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Ltotal;
         i += (int64_t)gridDim.x * blockDim.x) {
        L[i] = 0.0;
        if (i < n) diag[i] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->k_used = 0;
        st->stop = 0;
        st->pivval = 0.0;
        for (int m = 0; m < kMaxRank; m++) st->piv[m] = -1;
    }
    // initial block partials: every diag entry equals s -> lowest index wins.
    if (threadIdx.x == 0 && blockIdx.x < nblk) {
        pv[blockIdx.x] = s;
        pi[blockIdx.x] = 0;
    }
}

// Finish the argmax over block partials; decide pivot m (or stop).
__global__ void k_piv_select(PivState *st, const double *__restrict__ pv,
                             const int64_t *__restrict__ pi, int nblk, int m, double stop_tol) {
    // one warp: (value, -index) is a total order, so the strided lane partials and the
    // butterfly give exactly the sequential argmax (ties -> lowest index)
    if (st->stop) return;
    const int lane = threadIdx.x;
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int b = lane; b < nblk; b += 32) argmax_combine(bv, bi, pv[b], pi[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_combine(bv, bi, v2, i2);
    }
    if (lane != 0) return;
    if (!(bv > stop_tol)) {
        st->stop = 1;
        st->k_used = m;
        return;
    }
    st->piv[m] = bi;
    st->pivval = bv;
    st->k_used = m + 1;
}

// Step m: L[m][:], diag update, block-partial argmax of the new diag.
__global__ void __launch_bounds__(kThreads)
k_piv_step(PivState *st, int m, int kind, const float *__restrict__ X, int64_t n, int d,
           const double *__restrict__ ls, int n_ls, double s, double *__restrict__ L,
           double *__restrict__ diag, double *pv, int64_t *pi) {
    if (st->stop) return;
    const int64_t p = st->piv[m];
    const double sq = __dsqrt_rn(st->pivval);
    const float *xp = X + p * d;
    double bv = -1.0;
    int64_t bi = n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = kernel_fp64(kind, xp, X + i * d, d, ls, n_ls, s);
        for (int mm = 0; mm < m; mm++)
            acc = __dsub_rn(acc, __dmul_rn(L[(int64_t)mm * n + i], L[(int64_t)mm * n + p]));
        double lim = __ddiv_rn(acc, sq);
        L[(int64_t)m * n + i] = lim;
        double dg = (i == p) ? 0.0 : __dsub_rn(diag[i], __dmul_rn(lim, lim));
        diag[i] = dg;
        argmax_combine(bv, bi, dg, i);
    }
    block_argmax(bv, bi, pv + blockIdx.x, pi + blockIdx.x);
}

// ---- SoR operator (row f4): rows of K_SoR = Bs^T Bs (Bs m x n, row-major)
__global__ void __launch_bounds__(kThreads)
k_piv_init_sor(double *__restrict__ diag, int64_t n, const double *__restrict__ Bs, int m,
               double *__restrict__ L, int64_t Ltotal, PivState *st, double *pv, int64_t *pi) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < Ltotal;
         e += (int64_t)gridDim.x * blockDim.x)
        L[e] = 0.0;
    double bv = -1.0;
    int64_t bi = n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int a = 0; a < m; a++) {
            const double b = Bs[(int64_t)a * n + i];
            s = __dadd_rn(s, __dmul_rn(b, b));
        }
        diag[i] = s;
        argmax_combine(bv, bi, s, i);
    }
    block_argmax(bv, bi, pv + blockIdx.x, pi + blockIdx.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->k_used = 0;
        st->stop = 0;
        st->pivval = 0.0;
        for (int q = 0; q < kMaxRank; q++) st->piv[q] = -1;
    }
}

__global__ void __launch_bounds__(kThreads)
k_piv_step_sor(PivState *st, int mstep, const double *__restrict__ Bs, int m, int64_t n,
               double *__restrict__ L, double *__restrict__ diag, double *pv, int64_t *pi) {
    if (st->stop) return;
    const int64_t p = st->piv[mstep];
    const double sq = __dsqrt_rn(st->pivval);
    double bv = -1.0;
    int64_t bi = n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // K_SoR[p][i] = Bs[:, p] . Bs[:, i], four partial sums (ILP over the strided loads)
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        int a = 0;
        for (; a + 4 <= m; a += 4)
#pragma unroll
            for (int u = 0; u < 4; u++)
                s4[u] = __dadd_rn(s4[u], __dmul_rn(Bs[(int64_t)(a + u) * n + p],
                                                   Bs[(int64_t)(a + u) * n + i]));
        for (; a < m; a++)
            s4[0] = __dadd_rn(s4[0], __dmul_rn(Bs[(int64_t)a * n + p], Bs[(int64_t)a * n + i]));
        double acc = __dadd_rn(__dadd_rn(s4[0], s4[1]), __dadd_rn(s4[2], s4[3]));
        for (int mm = 0; mm < mstep; mm++)
            acc = __dsub_rn(acc, __dmul_rn(L[(int64_t)mm * n + i], L[(int64_t)mm * n + p]));
        const double lim = __ddiv_rn(acc, sq);
        L[(int64_t)mstep * n + i] = lim;
        const double dg = (i == p) ? 0.0 : __dsub_rn(diag[i], __dmul_rn(lim, lim));
        diag[i] = dg;
        argmax_combine(bv, bi, dg, i);
    }
    block_argmax(bv, bi, pv + blockIdx.x, pi + blockIdx.x);
}

__global__ void k_sum(const double *__restrict__ x, int64_t n, double *out) {
    __shared__ double sh[kThreads];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

}  // namespace

void pivchol(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h, int k, double *L,
             int64_t *piv_h, int *k_used_h, double *resid_h) {
    BBMM_REQUIRE(k >= 0 && k <= kMaxRank && k <= n, "pivchol rank out of range");
    cudaStream_t sm = ctx->stream;
    Workspace &ws = ctx->ws;
    double *diag = (double *)ws.get("pv_diag", (size_t)n * 8);
    PivState *st = (PivState *)ws.get("pv_state", sizeof(PivState));
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), 4 * kNumSMs));
    double *pv = (double *)ws.get("pv_pv", (size_t)nblk * 8);
    int64_t *pi = (int64_t *)ws.get("pv_pi", (size_t)nblk * 8);
    double *ls_d = (double *)ws.get("pv_ls", kMaxDim * 8);
    double *res_d = (double *)ws.get("pv_res", 8);
    BBMM_CUDA(cudaMemcpyAsync(ls_d, h.ls, sizeof(double) * h.n_ls, cudaMemcpyHostToDevice, sm));
    const int64_t Ltot = (int64_t)std::max(k, 1) * n;
    k_piv_init<<<nblk, kThreads, 0, sm>>>(diag, n, h.s, L, k > 0 ? Ltot : 0, st, pv, pi, nblk);
    int launches = 1;
    const double stop_tol = 1e-12 * h.s;
    for (int m = 0; m < k; m++) {
        k_piv_select<<<1, 32, 0, sm>>>(st, pv, pi, nblk, m, stop_tol);
        k_piv_step<<<nblk, kThreads, 0, sm>>>(st, m, h.kind, X, n, d, ls_d, h.n_ls, h.s, L, diag,
                                               pv, pi);
        launches += 2;
    }
    k_sum<<<1, kThreads, 0, sm>>>(diag, n, res_d);
    launches++;
    BBMM_LAUNCH_CHECK();
    ctx->launches += launches;
    PivState st_h;
    BBMM_CUDA(cudaMemcpyAsync(&st_h, st, sizeof(PivState), cudaMemcpyDeviceToHost, sm));
    double res = 0.0;
    BBMM_CUDA(cudaMemcpyAsync(&res, res_d, 8, cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaStreamSynchronize(sm));
    if (k == 0) res = h.s * (double)n;
    if (piv_h)
        for (int m = 0; m < k; m++) piv_h[m] = m < st_h.k_used ? st_h.piv[m] : -1;
    if (k_used_h) *k_used_h = (k == 0) ? 0 : st_h.k_used;
    if (resid_h) *resid_h = res;
}

void pivchol_sor(bbmm_ctx_s *ctx, const double *Bs, int64_t n, int m, double s, int k, double *L,
                 int64_t *piv_h, int *k_used_h, double *resid_h) {
    BBMM_REQUIRE(k >= 0 && k <= kMaxRank && k <= n, "pivchol rank out of range");
    cudaStream_t sm = ctx->stream;
    Workspace &ws = ctx->ws;
    double *diag = (double *)ws.get("pv_diag", (size_t)n * 8);
    PivState *st = (PivState *)ws.get("pv_state", sizeof(PivState));
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), 4 * kNumSMs));
    double *pv = (double *)ws.get("pv_pv", (size_t)nblk * 8);
    int64_t *pi = (int64_t *)ws.get("pv_pi", (size_t)nblk * 8);
    double *res_d = (double *)ws.get("pv_res", 8);
    const int64_t Ltot = (int64_t)std::max(k, 1) * n;
    k_piv_init_sor<<<nblk, kThreads, 0, sm>>>(diag, n, Bs, m, L, k > 0 ? Ltot : 0, st, pv, pi);
    int launches = 1;
    const double stop_tol = 1e-12 * s;                 // as for the exact kernel (R23)
    for (int q = 0; q < k; q++) {
        k_piv_select<<<1, 32, 0, sm>>>(st, pv, pi, nblk, q, stop_tol);
        k_piv_step_sor<<<nblk, kThreads, 0, sm>>>(st, q, Bs, m, n, L, diag, pv, pi);
        launches += 2;
    }
    k_sum<<<1, kThreads, 0, sm>>>(diag, n, res_d);
    launches++;
    BBMM_LAUNCH_CHECK();
    ctx->launches += launches;
    PivState st_h;
    BBMM_CUDA(cudaMemcpyAsync(&st_h, st, sizeof(PivState), cudaMemcpyDeviceToHost, sm));
    double res = 0.0;
    BBMM_CUDA(cudaMemcpyAsync(&res, res_d, 8, cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaStreamSynchronize(sm));
    if (piv_h)
        for (int q = 0; q < k; q++) piv_h[q] = q < st_h.k_used ? st_h.piv[q] : -1;
    if (k_used_h) *k_used_h = (k == 0) ? 0 : st_h.k_used;
    if (resid_h) *resid_h = res;
}

}  // namespace bbmm
