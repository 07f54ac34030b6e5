// mbcg_fused.cu -- the mBCG vector work of one iteration in ONE cooperative
// kernel (north star item 3: "fused mBCG vector updates, where per-column
// alpha/beta dot products use warp-shuffle reductions and the Lanczos
// coefficients are recorded in the same pass").  Single rank, t + 1 <= 20
// columns, no SoR operator, n <= 65 536 (the launch-latency regime: C0-C2); otherwise
// mbcg.cu's per-step kernels run.
//
// Same arithmetic as mbcg.cu's k_passA .. k_passD (Alg. S2
// with readings R5-R9, Woodbury PAPER.md:173-179 / R10), between grid-wide
// barriers instead of kernel launches:
//   P1  V = sum_s Vpart_s + sigma^2 D, partial <D,V>                  | sync
//   P2  alpha = rho/<D,V> (every block, identical), record alpha_j;
//       U += alpha D, R -= alpha V, partial |R|^2, partial L^T R      | sync
//   P3  distributed cross-block sums of |R|^2 and W = L^T R           | sync
//   P4  relres, freeze (tol), S = C^-1 W (explicit C^-1, set up once);
//       Z = (R - L S)/sigma^2, partial <R,Z>                          | sync
//   P5  beta = rho'/rho, record beta_j; D = Z + beta D; matmul operand:
//       fp64/fp32 copy, or (tensor-core path) column max        | sync |
//       then the int8 slices of the block's own rows
// Every block holds the row range [blk * rpb, (blk + 1) * rpb) and a private
// copy of the per-column state; block 0 alone writes the state, histories and
// counters to global memory, so the blocks never race on them.  Cross-block
// sums use the fixed lane-strided + butterfly order of k_reduce_blocks.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"

namespace cg = cooperative_groups;

namespace bbmm {
namespace fz {

constexpr int kT = 512;          // threads per block (16 warps: enough loads in flight for HBM)
constexpr int kCW = 32;          // column lanes of the element-wise passes (c <= 20)
constexpr int kRB = kT / kCW;    // rows per sweep
constexpr int kCM = 20;          // max columns of the fused path

struct Args {
    MbcgState *st;
    const double *Vpart;
    int splits, cs, c, k;
    int64_t nloc, n, rpb;
    double noise_var, tol;
    double *D, *V, *U, *R, *Z;
    const double *L, *Cinv;
    double *ahist, *bhist, *rhist;
    double *partA, *partRR, *partW, *partRZ, *partMax, *red;
    void *Dm;
    int dm_f32;
    // tensor-core operand
    int use_tc, nd, blk_cols, nb_rows;
    uint8_t *Bp;
    double *Stc;
    int64_t pad_end;   // points covered by Bp (k1tc_pad_rows(n))
    int cb;            // instantiation columns: D in [0, c), zero D in [c, cb), constant at cb
    int KT;
};

struct Shared {
    int act[kMaxCols];
    double rho[kMaxCols], bn[kMaxCols], alpha[kMaxCols], beta[kMaxCols], colv[kMaxCols];
    double sred[kT];
    int j, any;
};

// per-thread value of column tx -> part[blk * c + tx] (rows of the block summed in ty order)
__device__ void block_cols(Shared &sh, double v, double *part, int c) {
    const int tx = threadIdx.x % kCW, ty = threadIdx.x / kCW;
    sh.sred[ty * kCW + tx] = v;
    __syncthreads();
    if (ty == 0 && tx < c) {
        double s = 0.0;
        for (int y = 0; y < kRB; y++) s += sh.sred[y * kCW + tx];
        part[(int64_t)blockIdx.x * c + tx] = s;
    }
    __syncthreads();
}

// out[e] = sum_b part[b * m + e] for e < m (every block; warp per output, fixed order)
__device__ void sum_parts(const double *part, int nblk, int m, double *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < m; e += kT / 32) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * m + e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[e] = s;
    }
}

template <int MPT>
__global__ void __launch_bounds__(kT, 1) k_mbcg_fused(Args a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double dyn[];
    __shared__ Shared sh;
    const int tid = threadIdx.x, tx = tid % kCW, ty = tid / kCW;
    const int c = a.c, k = a.k, G = gridDim.x;
    const bool b0 = blockIdx.x == 0;
    const int64_t i_beg = (int64_t)blockIdx.x * a.rpb;
    const int64_t i_end = min(a.nloc, i_beg + a.rpb);
    MbcgState *st = a.st;
    if (tid < c) {
        sh.act[tid] = st->active[tid];
        sh.rho[tid] = st->rho[tid];
        sh.bn[tid] = st->bnorm[tid];
    }
    if (tid == 0) sh.j = st->j;
    __syncthreads();
    const int j = sh.j;

    // ---------------- P1: V = sum_s Vpart + sigma^2 D ; <D, V>
    {
        double acc = 0.0;
        if (tx < c)
            for (int64_t i = i_beg + ty; i < i_end; i += kRB) {
                double v = 0.0;
                for (int s = 0; s < a.splits; s++) v += a.Vpart[((int64_t)s * a.nloc + i) * a.cs + tx];
                const double dv = a.D[i * c + tx];
                v += a.noise_var * dv;
                a.V[i * c + tx] = v;
                acc += dv * v;
            }
        block_cols(sh, acc, a.partA, c);
    }
    grid.sync();

    // ---------------- P2: alpha ; U, R update ; |R|^2 ; L^T R
    sum_parts(a.partA, G, c, sh.colv);
    __syncthreads();
    if (tid < c) {
        const int col = tid;
        double al = 0.0;
        if (sh.act[col]) {
            al = sh.rho[col] / sh.colv[col];
            if (!(al > 0.0) || !isfinite(al)) {
                // reading R9/R24: exhausted residual (rho <= 1e-250 rho_0) freezes like
                // R = 0; otherwise an indefinite operator: breakdown
                const bool exhausted = sh.rho[col] <= 1e-250 * st->rho0[col];
                al = 0.0;
                sh.act[col] = 0;
                if (b0) {
                    if (!exhausted) st->status = BBMM_ERR_NUMERIC;
                    st->active[col] = 0;
                }
            } else if (b0) {
                a.ahist[(int64_t)j * c + col] = al;
                st->iters[col] = j + 1;
            }
        }
        sh.alpha[col] = al;
        if (b0) st->alpha[col] = al;
    }
    __syncthreads();
    {
        double acc = 0.0;
        if (tx < c) {
            const double al = sh.alpha[tx];
            for (int64_t i = i_beg + ty; i < i_end; i += kRB) {
                double r = a.R[i * c + tx];
                if (al != 0.0) {
                    a.U[i * c + tx] += al * a.D[i * c + tx];
                    r -= al * a.V[i * c + tx];
                    a.R[i * c + tx] = r;
                }
                acc += r * r;
            }
        }
        block_cols(sh, acc, a.partRR, c);     // ends with __syncthreads: R rows visible
    }
    if (k > 0) {
        // W partial = L[:, own rows]^T R[own rows] (register-tiled as k_LtR2)
        double *Lt = dyn;                       // KT x k
        double *Rt = dyn + (size_t)a.KT * k;    // KT x c
        const int CGN = (c + 3) / 4, MLN = kT / CGN;
        const int g = tid % CGN, ml = tid / CGN;
        const bool act = ml < MLN;
        double acc[MPT][4];
#pragma unroll
        for (int q = 0; q < MPT; q++)
#pragma unroll
            for (int u = 0; u < 4; u++) acc[q][u] = 0.0;
        for (int64_t i0 = i_beg; i0 < i_end; i0 += a.KT) {
            const int rows = (int)min((int64_t)a.KT, i_end - i0);
            __syncthreads();
            for (int e = tid; e < k * a.KT; e += kT) {
                const int m = e / a.KT, kk = e - m * a.KT;
                Lt[kk * k + m] = kk < rows ? a.L[(int64_t)m * a.n + i0 + kk] : 0.0;
            }
            for (int e = tid; e < a.KT * c; e += kT) {
                const int kk = e / c;
                Rt[e] = kk < rows ? a.R[i0 * c + e] : 0.0;
            }
            __syncthreads();
            if (act)
                for (int kk = 0; kk < a.KT; kk++) {
                    double r[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) r[u] = (4 * g + u < c) ? Rt[kk * c + 4 * g + u] : 0.0;
#pragma unroll
                    for (int q = 0; q < MPT; q++) {
                        const int m = ml + q * MLN;
                        const double l = m < k ? Lt[kk * k + m] : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; u++) acc[q][u] = fma(l, r[u], acc[q][u]);
                    }
                }
        }
        if (act)
#pragma unroll
            for (int q = 0; q < MPT; q++) {
                const int m = ml + q * MLN;
                if (m < k)
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (4 * g + u < c)
                            a.partW[(int64_t)blockIdx.x * k * c + m * c + 4 * g + u] = acc[q][u];
            }
    }
    grid.sync();

    // ---------------- P3: red = [ |R|^2 (c) | W (k c) ], outputs spread over all warps
    {
        const int lane = tid & 31;
        const int m = c + k * c;
        for (int e = blockIdx.x * (kT / 32) + (tid >> 5); e < m; e += G * (kT / 32)) {
            const double *src = e < c ? a.partRR : a.partW;
            const int mm = e < c ? c : k * c, ee = e < c ? e : e - c;
            double s = 0.0;
            for (int b = lane; b < G; b += 32) s += src[(int64_t)b * mm + ee];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) a.red[e] = s;
        }
    }
    grid.sync();

    // ---------------- P4: relres / freeze ; S = C^-1 W ; Z = (R - L S)/sigma^2 ; <R, Z>
    double *S = dyn;                                       // k x c (reuses the L^T R tiles)
    if (tid < c && sh.act[tid]) {
        const int col = tid;
        const double rel = sqrt(a.red[col]) / sh.bn[col];
        if (b0) { st->relres[col] = rel; a.rhist[(int64_t)j * c + col] = rel; }
        if (rel < a.tol) { sh.act[col] = 0; if (b0) st->active[col] = 0; }
    }
    if (k > 0)
        for (int e = tid; e < k * c; e += kT) {
            const int m = e / c, col = e - m * c;
            double s = 0.0;
            for (int l = 0; l < k; l++) s = fma(a.Cinv[m * k + l], a.red[c + l * c + col], s);
            S[e] = s;
        }
    __syncthreads();
    {
        const double inv = 1.0 / a.noise_var;
        double rz[kCM];
#pragma unroll
        for (int u = 0; u < kCM; u++) rz[u] = 0.0;
        for (int64_t i = i_beg + tid; i < i_end; i += kT) {
            double acc[kCM];
#pragma unroll
            for (int u = 0; u < kCM; u++) acc[u] = 0.0;
            for (int m = 0; m < k; m++) {
                const double l = a.L[(int64_t)m * a.n + i];
#pragma unroll
                for (int u = 0; u < kCM; u++)
                    if (u < c) acc[u] = fma(l, S[m * c + u], acc[u]);
            }
#pragma unroll
            for (int u = 0; u < kCM; u++)
                if (u < c) {
                    const double r = a.R[i * c + u];
                    const double z = k > 0 ? (r - acc[u]) * inv : r;
                    a.Z[i * c + u] = z;
                    rz[u] += r * z;
                }
        }
        // block sum of rz[u] over threads: warp butterfly, then warps in order
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int u = 0; u < kCM; u++) {
            if (u >= c) break;
            double v = rz[u];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sh.sred[warp * kCM + u] = v;   // 8 warps x 20 <= 256
        }
        __syncthreads();
        if (tid < c) {
            double s = 0.0;
            for (int w = 0; w < kT / 32; w++) s += sh.sred[w * kCM + tid];
            a.partRZ[(int64_t)blockIdx.x * c + tid] = s;
        }
    }
    grid.sync();

    // ---------------- P5: beta ; D = Z + beta D ; matmul operand
    sum_parts(a.partRZ, G, c, sh.colv);
    if (tid == 0) sh.any = 0;
    __syncthreads();
    if (tid < c) {
        const int col = tid;
        double be = 0.0;
        if (sh.act[col]) {
            const double r = sh.colv[col];
            if (r == 0.0) {
                sh.act[col] = 0;                   // R = 0 exactly
                if (b0) st->active[col] = 0;
            } else {
                be = r / sh.rho[col];
                if (b0) { st->rho[col] = r; a.bhist[(int64_t)j * c + col] = be; }
            }
        }
        sh.beta[col] = be;
        if (b0) st->beta[col] = be;
        if (sh.act[col]) atomicOr(&sh.any, 1);
    }
    __syncthreads();
    if (b0 && tid == 0) st->any_active = sh.any;
    {
        double mx = 0.0;
        const bool act = tx < c && sh.act[tx];
        const double be = tx < c ? sh.beta[tx] : 0.0;
        if (tx < a.cs || (a.use_tc && tx < c))
            for (int64_t i = i_beg + ty; i < i_end; i += kRB) {
                double dn = 0.0;
                if (act) dn = a.Z[i * c + tx] + be * a.D[i * c + tx];
                if (tx < c) a.D[i * c + tx] = dn;
                if (a.use_tc) {
                    mx = fmax(mx, fabs(dn));
                } else if (tx < a.cs) {
                    if (a.dm_f32) reinterpret_cast<float *>(a.Dm)[i * a.cs + tx] = (float)dn;
                    else reinterpret_cast<double *>(a.Dm)[i * a.cs + tx] = dn;
                }
            }
        if (a.use_tc) {
            // block column max (order-free) -> partMax
            sh.sred[ty * kCW + tx] = mx;
            __syncthreads();
            if (ty == 0 && tx < c) {
                double m2 = 0.0;
                for (int y = 0; y < kRB; y++) m2 = fmax(m2, sh.sred[y * kCW + tx]);
                a.partMax[(int64_t)blockIdx.x * c + tx] = m2;
            }
        }
    }
    if (a.use_tc) {
        grid.sync();
        // column scales (every block; max is order-free) -> int8 slices of own rows
        if (tid < c) {
            double m2 = 0.0;
            for (int b = 0; b < G; b++) m2 = fmax(m2, a.partMax[(int64_t)b * c + tid]);
            sh.colv[tid] = m2 > 0.0 ? m2 : 1.0;
            if (b0) a.Stc[tid] = sh.colv[tid];
        }
        __syncthreads();
        const int T = 8 * a.nd - 2;
        const double scaleT = ldexp(1.0, T);
        const int64_t offT = 1LL << T;
        const int64_t q0 = i_beg / 16;
        const int64_t q1 = (i_end >= a.nloc) ? a.pad_end / 16 : i_end / 16;  // last block: padding
        const int64_t total = (q1 - q0) * a.nb_rows;
        for (int64_t e = tid; e < total; e += kT) {
            const int nn = (int)(e % a.nb_rows);
            const int64_t q = q0 + e / a.nb_rows;
            const int bi = nn / a.blk_cols, col = nn - bi * a.blk_cols;
            uint32_t wv[4] = {0, 0, 0, 0};
            if (bi < a.nd && col <= a.cb) {
                const int shift = 8 * (a.nd - 1 - bi);
#pragma unroll 4
                for (int p = 0; p < 16; p++) {
                    const int64_t jj = q * 16 + p;
                    uint32_t byte = 0;
                    if (jj < a.nloc) {
                        int64_t P = offT;
                        if (col < c) P = llrint(a.D[jj * c + col] / sh.colv[col] * scaleT) + offT;
                        byte = (uint32_t)((P >> shift) & 0xFF);
                    }
                    wv[p >> 2] |= byte << (8 * (p & 3));
                }
            }
            *reinterpret_cast<uint4 *>(a.Bp + q * (int64_t)a.nb_rows * 16 + (int64_t)nn * 16) =
                make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
    }
    if (b0 && tid == 0) st->j = j + 1;
}

// C^-1 (k x k) from the Cholesky factor, one warp per column of the identity.
__global__ void k_cinv(const double *__restrict__ cholC, int k, double *__restrict__ Cinv) {
    extern __shared__ double xs[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *x = xs + (size_t)warp * k;
    for (int col = warp; col < k; col += (int)(blockDim.x >> 5)) {
        for (int r = 0; r < k; r++) {
            double p = 0.0;
            for (int b = lane; b < r; b += 32) p = fma(cholC[r * k + b], x[b], p);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (lane == 0) x[r] = ((r == col ? 1.0 : 0.0) - p) / cholC[r * k + r];
            __syncwarp();
        }
        for (int r = k - 1; r >= 0; r--) {
            double p = 0.0;
            for (int b = r + 1 + lane; b < k; b += 32) p = fma(cholC[b * k + r], x[b], p);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (lane == 0) x[r] = (x[r] - p) / cholC[r * k + r];
            __syncwarp();
        }
        for (int r = lane; r < k; r += 32) Cinv[r * k + col] = x[r];
        __syncwarp();
    }
}

}  // namespace fz

// ======================================================================
// host side
// ======================================================================
namespace {
template <int MPT>
void *fused_fn() { return (void *)fz::k_mbcg_fused<MPT>; }
}

// Latency regime only: one 256-thread block per SM keeps 8 warps per SM in flight, too few
// to stream the HBM-bound vector work of large n (C4: 157 vs 70 ms per call on the per-step
// kernels; C2, n = 45 730: even; C1: 2.06 vs 2.9 ms).
constexpr int64_t kFusedMaxRows = 65536;
bool mbcg_fused_applicable(const bbmm_ctx_s *ctx, int c, int k, bool use_sor, int64_t nloc) {
    const char *mx = getenv("BBMM_FUSED_MAX_ROWS");      // experiment override
    const int64_t max_rows = mx ? atoll(mx) : kFusedMaxRows;
    if (ctx->nranks != 1 || use_sor || c > fz::kCM || k > kMaxRank || nloc > max_rows)
        return false;
    const char *env = getenv("BBMM_NO_FUSED_MBCG");
    return !(env && env[0] == '1');
}

// Plan + one-off setup for a call: grid, rows per block, C^-1.
FusedPlan mbcg_fused_plan(bbmm_ctx_s *ctx, int64_t nloc, int c, int k, const double *cholC,
                          double *Cinv) {
    FusedPlan p;
    const int CGN = (c + 3) / 4, MLN = fz::kT / CGN;
    const int need = std::max(1, (k + MLN - 1) / MLN);
    p.mpt = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 12 ? 12 : 16;
    p.KT = k <= 64 ? 32 : 16;
    p.smem = std::max((size_t)p.KT * (k + c), (size_t)k * c) * 8;
    void *fn = p.mpt == 1 ? fused_fn<1>() : p.mpt == 2 ? fused_fn<2>() : p.mpt == 4 ? fused_fn<4>()
             : p.mpt == 8 ? fused_fn<8>() : p.mpt == 12 ? fused_fn<12>() : fused_fn<16>();
    p.fn = fn;
    BBMM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(p.smem, 1)));
    int per_sm = 0;
    BBMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, fz::kT, p.smem));
    const int64_t gmax = (int64_t)std::max(per_sm, 1) * kNumSMs;
    int64_t G = std::max<int64_t>(1, std::min<int64_t>(gmax, ceil_div(std::max<int64_t>(nloc, 1), 64)));
    p.rpb = ceil_div(ceil_div(std::max<int64_t>(nloc, 1), G), 64) * 64;
    p.G = (int)ceil_div(std::max<int64_t>(nloc, 1), p.rpb);
    p.ok = per_sm > 0;
    if (k > 0) {
        fz::k_cinv<<<1, 1024, (size_t)32 * k * 8, ctx->stream>>>(cholC, k, Cinv);
        BBMM_LAUNCH_CHECK();
        ctx->launches++;
    }
    return p;
}

void mbcg_fused_iteration(bbmm_ctx_s *ctx, const FusedPlan &p, const FusedIo &io) {
    fz::Args a;
    a.st = io.st; a.Vpart = io.Vpart; a.splits = io.splits; a.cs = io.cs; a.c = io.c; a.k = io.k;
    a.nloc = io.nloc; a.n = io.n; a.rpb = p.rpb; a.noise_var = io.noise_var; a.tol = io.tol;
    a.D = io.D; a.V = io.V; a.U = io.U; a.R = io.R; a.Z = io.Z; a.L = io.L; a.Cinv = io.Cinv;
    a.ahist = io.ahist; a.bhist = io.bhist; a.rhist = io.rhist;
    a.partA = io.part; a.partRR = io.part + (size_t)p.G * io.c;
    a.partRZ = io.part + (size_t)2 * p.G * io.c; a.partMax = io.part + (size_t)3 * p.G * io.c;
    a.partW = io.partW; a.red = io.red;
    a.Dm = io.Dm; a.dm_f32 = io.dm_f32;
    a.use_tc = io.Bp != nullptr; a.nd = io.nd; a.blk_cols = io.nb_rows / std::max(io.nd, 1);
    a.nb_rows = io.nb_rows; a.Bp = io.Bp; a.Stc = io.Stc; a.pad_end = io.pad_end; a.KT = p.KT;
    a.cb = io.cb > 0 ? io.cb : io.c;
    void *args[] = {&a};
    BBMM_CUDA(cudaLaunchCooperativeKernel(p.fn, dim3(p.G), dim3(fz::kT), args, p.smem, ctx->stream));
    ctx->launches++;
}

}  // namespace bbmm
