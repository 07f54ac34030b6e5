// matmul.cu -- the blackbox matmul Khat*D of mBCG,
// the hot loop of the method (>95% of the time).
//
//   K1  k1_onthefly : V_i = s * sum_j k~(x_i, x_j) D_j   (never materialises K)
//   K2  k2_build    : Kst[i][j] = s * k~(x_i, x_j)        (stored variant, fp32)
//       k2_stored   : V_i = sum_j Kst[i][j] D_j            (HBM streaming)
//
// Both write fp64 partial sums Vpart[split][row][col]; the sigma^2 D term and
// the sum over j-splits are added by the mBCG pass-A kernel (mbcg.cu).
//
// Precision: kernel values and D in fp32, products
// accumulated in fp32 over at most 16 j-terms, then folded into fp64
// accumulators (long fp32 accumulation breaks the 1e-4 solve
// bar at large n).
#include <algorithm>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"

namespace bbmm {

// --------------------------------------------------------------------------
// Input scaling: Xs[i][q] = X[i][q] * scale_q, zero-padded to ds columns.
// --------------------------------------------------------------------------
__global__ void k_scale_inputs(const float *__restrict__ X, int64_t n, int d,
                               const float *__restrict__ scale, float *__restrict__ Xs, int ds) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = n * ds;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx / ds;
        int q = (int)(idx - i * ds);
        Xs[idx] = q < d ? X[i * d + q] * scale[q] : 0.0f;
    }
}

// --------------------------------------------------------------------------
// K1: on-the-fly kernel matmul, FFMA contraction.
// Block = 128 threads, each thread owns R rows (rows blockRow + tid + 128 r).
// j-range of the block = split blockIdx.y.  Tiles of BJ = 64 points of
// (xs_j, D_j) are staged in shared memory; every thread reads them as
// broadcasts.  Inner loop per (row, j): distance (2D FLOP), one ex2 (MUFU),
// CP FFMAs into fp32 accumulators, folded to fp64 every 16 j.
// --------------------------------------------------------------------------
template <int KIND, int D, int CP, int R>
__global__ void __launch_bounds__(128)
k1_onthefly(const float *__restrict__ Xs, const float *__restrict__ D32, int64_t n, int64_t r0,
            int64_t nloc, int64_t jchunk, double s, double *__restrict__ Vpart) {
    constexpr int DS = round4(D), CS = round4(CP);
    constexpr int BJ = 64, FOLD = 16;
    __shared__ __align__(16) float xs[BJ][DS];
    __shared__ __align__(16) float dsm[BJ][CS];

    const int tid = threadIdx.x;
    const int64_t rowbase = (int64_t)blockIdx.x * (128 * R);
    float xi[R][D];
#pragma unroll
    for (int r = 0; r < R; r++) {
        int64_t i = rowbase + tid + 128 * r;
#pragma unroll
        for (int q = 0; q < D; q++) xi[r][q] = (i < nloc) ? Xs[(r0 + i) * DS + q] : 0.0f;
    }
    double a64[R][CP];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int c = 0; c < CP; c++) a64[r][c] = 0.0;

    const int64_t j0 = (int64_t)blockIdx.y * jchunk;
    const int64_t j1 = min(n, j0 + jchunk);
    for (int64_t jt = j0; jt < j1; jt += BJ) {
        __syncthreads();
        {
            const float4 *X4 = reinterpret_cast<const float4 *>(Xs);
            const float4 *D4 = reinterpret_cast<const float4 *>(D32);
            float4 *xs4 = reinterpret_cast<float4 *>(&xs[0][0]);
            float4 *ds4 = reinterpret_cast<float4 *>(&dsm[0][0]);
            for (int e = tid; e < BJ * DS / 4; e += 128) {
                int jj = e / (DS / 4);
                int64_t j = jt + jj;
                xs4[e] = (j < j1) ? X4[j * (DS / 4) + (e - jj * (DS / 4))]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int e = tid; e < BJ * CS / 4; e += 128) {
                int jj = e / (CS / 4);
                int64_t j = jt + jj;
                ds4[e] = (j < j1) ? D4[j * (CS / 4) + (e - jj * (CS / 4))]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int jf = 0; jf < BJ; jf += FOLD) {
            float a32[R][CP];
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int c = 0; c < CP; c++) a32[r][c] = 0.0f;
#pragma unroll 2
            for (int jj = jf; jj < jf + FOLD; jj++) {
                float xj[D], dj[CP];
#pragma unroll
                for (int q = 0; q < D; q++) xj[q] = xs[jj][q];
#pragma unroll
                for (int c = 0; c < CP; c++) dj[c] = dsm[jj][c];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float rs2 = 0.0f;
#pragma unroll
                    for (int q = 0; q < D; q++) {
                        float df = xi[r][q] - xj[q];
                        rs2 = fmaf(df, df, rs2);
                    }
                    float kv = kval_scaled<KIND>(rs2);
#pragma unroll
                    for (int c = 0; c < CP; c++) a32[r][c] = fmaf(kv, dj[c], a32[r][c]);
                }
            }
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int c = 0; c < CP; c++) a64[r][c] += (double)a32[r][c];
        }
    }
    double *out = Vpart + (int64_t)blockIdx.y * nloc * CS;
#pragma unroll
    for (int r = 0; r < R; r++) {
        int64_t i = rowbase + tid + 128 * r;
        if (i < nloc) {
#pragma unroll
            for (int c = 0; c < CP; c++) out[i * CS + c] = s * a64[r][c];
#pragma unroll
            for (int c = CP; c < CS; c++) out[i * CS + c] = 0.0;
        }
    }
}

// --------------------------------------------------------------------------
// K2 build: Kst[i][j] = s * k~(x_{r0+i}, x_j), fp32, row-major nloc x n (ldk).
// --------------------------------------------------------------------------
template <int KIND, int D>
__global__ void __launch_bounds__(256)
k2_build(const float *__restrict__ Xs, int64_t n, int64_t r0, int64_t nloc, int64_t ldk, float s,
         float *__restrict__ Kst) {
    constexpr int DS = round4(D);
    constexpr int BI = 16, BJ = 256;
    __shared__ float xi_s[BI][DS];
    const int64_t i0 = (int64_t)blockIdx.y * BI;
    const int64_t j = (int64_t)blockIdx.x * BJ + threadIdx.x;
    for (int e = threadIdx.x; e < BI * DS; e += 256) {
        int ii = e / DS;
        xi_s[ii][e % DS] = (i0 + ii < nloc) ? Xs[(r0 + i0 + ii) * DS + e % DS] : 0.0f;
    }
    __syncthreads();
    if (j >= n) return;
    float xj[D];
#pragma unroll
    for (int q = 0; q < D; q++) xj[q] = Xs[j * DS + q];
    for (int ii = 0; ii < BI && i0 + ii < nloc; ii++) {
        float rs2 = 0.0f;
#pragma unroll
        for (int q = 0; q < D; q++) {
            float df = xi_s[ii][q] - xj[q];
            rs2 = fmaf(df, df, rs2);
        }
        Kst[(i0 + ii) * ldk + j] = s * kval_scaled<KIND>(rs2);
    }
}

// --------------------------------------------------------------------------
// K2 stream: V_i = sum_j Kst[i][j] D_j.  HBM-bound on the Kst read.
// Block = 16 warps; warp w owns rows blockRow + 4w .. +3 (R = 4); lane l owns
// j = jt + 4l..4l+3 of each BJ = 128 tile (one coalesced 16-byte load per row).
// The D tile is staged transposed (dT[c][j]) so each lane reads its 4 j's of
// column c with one conflict-free 16-byte shared load.  Per-lane fp32
// partials cover 16 terms (4 tiles), then a warp butterfly (fp32, 5 levels)
// folds them into an fp64 accumulator held by lane (r*CP + c) % 32.
// --------------------------------------------------------------------------
template <int CP>
__global__ void __launch_bounds__(512)
k2_stored(const float *__restrict__ Kst, int64_t n, int64_t nloc, int64_t ldk,
          const float *__restrict__ D32, int64_t jchunk, double *__restrict__ Vpart) {
    constexpr int CS = round4(CP);
    constexpr int R = 4, W = 16, BJ = 128, FOLD_TILES = 4;
    constexpr int NACC = (R * CP + 31) / 32;
    __shared__ __align__(16) float dT[CP][BJ];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rowbase = (int64_t)blockIdx.x * (W * R) + warp * R;
    const int64_t j0 = (int64_t)blockIdx.y * jchunk;
    const int64_t j1 = min(n, j0 + jchunk);

    double acc64[NACC];
#pragma unroll
    for (int a = 0; a < NACC; a++) acc64[a] = 0.0;
    float a32[R][CP];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int c = 0; c < CP; c++) a32[r][c] = 0.0f;

    int tile = 0;
    for (int64_t jt = j0; jt < j1; jt += BJ, tile++) {
        __syncthreads();
        for (int e = threadIdx.x; e < BJ * CP; e += 512) {
            int jj = e / CP, c = e - jj * CP;
            int64_t j = jt + jj;
            dT[c][jj] = (j < j1) ? D32[j * CS + c] : 0.0f;
        }
        __syncthreads();
        float4 kv[R];
        const int64_t jl = jt + 4 * lane;
#pragma unroll
        for (int r = 0; r < R; r++) {
            int64_t i = rowbase + r;
            if (i < nloc && jl + 3 < j1) {
                kv[r] = __ldcs(reinterpret_cast<const float4 *>(Kst + i * ldk + jl));
            } else {
                float t[4];
#pragma unroll
                for (int u = 0; u < 4; u++)
                    t[u] = (i < nloc && jl + u < j1) ? Kst[i * ldk + jl + u] : 0.0f;
                kv[r] = make_float4(t[0], t[1], t[2], t[3]);
            }
        }
#pragma unroll
        for (int c = 0; c < CP; c++) {
            float4 dv = *reinterpret_cast<const float4 *>(&dT[c][4 * lane]);
#pragma unroll
            for (int r = 0; r < R; r++) {
                float a = a32[r][c];
                a = fmaf(kv[r].x, dv.x, a);
                a = fmaf(kv[r].y, dv.y, a);
                a = fmaf(kv[r].z, dv.z, a);
                a = fmaf(kv[r].w, dv.w, a);
                a32[r][c] = a;
            }
        }
        if ((tile + 1) % FOLD_TILES == 0 || jt + BJ >= j1) {
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int c = 0; c < CP; c++) {
                    float v = a32[r][c];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    const int idx = r * CP + c;
                    if (lane == (idx & 31)) acc64[idx >> 5] += (double)v;
                    a32[r][c] = 0.0f;
                }
        }
    }
    double *out = Vpart + (int64_t)blockIdx.y * nloc * CS;
#pragma unroll
    for (int a = 0; a < NACC; a++) {
        int idx = a * 32 + lane;
        if (idx < R * CP) {
            int r = idx / CP, c = idx - r * CP;
            int64_t i = rowbase + r;
            if (i < nloc) out[i * CS + c] = acc64[a];
        }
    }
    if (lane < R) {
        int64_t i = rowbase + lane;
        if (i < nloc)
            for (int c = CP; c < CS; c++) out[i * CS + c] = 0.0;
    }
}

// ==========================================================================
// host side: shape dispatch
// ==========================================================================
static const int kDims[] = {1, 3, 4, 8, 9, 16, 19, 26, 32};
static const int kCols[] = {4, 8, 11, 12, 16, 17, 24, 32, 33, 48, 64};

int pad_dim(int d) {
    for (int v : kDims)
        if (v >= d) return v;
    return -1;
}
int pad_cols(int c) {
    for (int v : kCols)
        if (v >= c) return v;
    return -1;
}

void scale_inputs(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h, float *Xs,
                  int dp) {
    float sc[kMaxDim];
    const double base = (h.kind == BBMM_RBF) ? std::sqrt(0.5 / std::log(2.0)) : std::sqrt(5.0);
    for (int q = 0; q < d; q++) sc[q] = (float)(base / h.ls[h.n_ls == 1 ? 0 : q]);
    float *sc_d = (float *)ctx->ws.get("scale_vec", sizeof(sc));
    BBMM_CUDA(cudaMemcpyAsync(sc_d, sc, sizeof(float) * d, cudaMemcpyHostToDevice, ctx->stream));
    int ds = round4(dp);
    int64_t total = n * ds;
    int grid = (int)std::min<int64_t>(ceil_div(total, 256), 4096);
    k_scale_inputs<<<grid, 256, 0, ctx->stream>>>(X, n, d, sc_d, Xs, ds);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

template <int KIND, int D, int CP>
static void launch_k1(bbmm_ctx_s *ctx, const float *Xs, int64_t n, int64_t r0, int64_t nloc,
                      const float *D32, double s, double *Vpart, int splits) {
    constexpr int R = (CP <= 17) ? 2 : 1;
    dim3 grid((unsigned)ceil_div(nloc, 128 * R), (unsigned)splits);
    int64_t jchunk = ceil_div(ceil_div(n, splits), 64) * 64;
    k1_onthefly<KIND, D, CP, R><<<grid, 128, 0, ctx->stream>>>(Xs, D32, n, r0, nloc, jchunk, s,
                                                              Vpart);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

#define BBMM_DISPATCH_COLS(CPV, ...)                                                      \
    switch (CPV) {                                                                        \
        case 4: { constexpr int CP_ = 4; __VA_ARGS__; } break;                            \
        case 8: { constexpr int CP_ = 8; __VA_ARGS__; } break;                            \
        case 11: { constexpr int CP_ = 11; __VA_ARGS__; } break;                          \
        case 12: { constexpr int CP_ = 12; __VA_ARGS__; } break;                          \
        case 16: { constexpr int CP_ = 16; __VA_ARGS__; } break;                          \
        case 17: { constexpr int CP_ = 17; __VA_ARGS__; } break;                          \
        case 24: { constexpr int CP_ = 24; __VA_ARGS__; } break;                          \
        case 32: { constexpr int CP_ = 32; __VA_ARGS__; } break;                          \
        case 33: { constexpr int CP_ = 33; __VA_ARGS__; } break;                          \
        case 48: { constexpr int CP_ = 48; __VA_ARGS__; } break;                          \
        case 64: { constexpr int CP_ = 64; __VA_ARGS__; } break;                          \
        default: throw Error{BBMM_ERR_ARG, "unsupported column count"};                  \
    }

#define BBMM_DISPATCH_DIMS(DV, ...)                                                       \
    switch (DV) {                                                                         \
        case 1: { constexpr int D_ = 1; __VA_ARGS__; } break;                             \
        case 3: { constexpr int D_ = 3; __VA_ARGS__; } break;                             \
        case 4: { constexpr int D_ = 4; __VA_ARGS__; } break;                             \
        case 8: { constexpr int D_ = 8; __VA_ARGS__; } break;                             \
        case 9: { constexpr int D_ = 9; __VA_ARGS__; } break;                             \
        case 16: { constexpr int D_ = 16; __VA_ARGS__; } break;                           \
        case 19: { constexpr int D_ = 19; __VA_ARGS__; } break;                           \
        case 26: { constexpr int D_ = 26; __VA_ARGS__; } break;                           \
        case 32: { constexpr int D_ = 32; __VA_ARGS__; } break;                           \
        default: throw Error{BBMM_ERR_ARG, "unsupported input dimension"};               \
    }

static int choose_splits(int64_t n, int64_t nloc, int64_t rows_per_block, int target_blocks) {
    int64_t rb = ceil_div(nloc, rows_per_block);
    int64_t sp = ceil_div(target_blocks, rb);
    sp = std::max<int64_t>(1, std::min<int64_t>(sp, ceil_div(n, 256)));
    return (int)sp;
}

size_t vpart_elems(int64_t n, int64_t nloc, int cp, bool stored) {
    int cs = round4(cp);
    int splits = stored ? choose_splits(n, nloc, 64, 2 * kNumSMs)
                        : choose_splits(n, nloc, 128, 6 * kNumSMs);
    return (size_t)splits * (size_t)nloc * cs;
}

int kernel_matmul_onthefly(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n,
                           int64_t r0, int64_t nloc, const float *D32, int cp, double s,
                           double *Vpart, size_t cap, cudaEvent_t ev0, cudaEvent_t ev1) {
    int splits = choose_splits(n, nloc, 128, 6 * kNumSMs);
    BBMM_REQUIRE((size_t)splits * nloc * round4(cp) <= cap, "Vpart workspace too small");
    if (ev0) BBMM_CUDA(cudaEventRecord(ev0, ctx->stream));
    if (nloc == 0) {
        if (ev1) BBMM_CUDA(cudaEventRecord(ev1, ctx->stream));
        return splits;
    }
    if (kind == BBMM_RBF) {
        BBMM_DISPATCH_DIMS(dp, BBMM_DISPATCH_COLS(cp, launch_k1<0, D_, CP_>(
                                                        ctx, Xs, n, r0, nloc, D32, s, Vpart, splits)))
    } else {
        BBMM_DISPATCH_DIMS(dp, BBMM_DISPATCH_COLS(cp, launch_k1<1, D_, CP_>(
                                                        ctx, Xs, n, r0, nloc, D32, s, Vpart, splits)))
    }
    if (ev1) BBMM_CUDA(cudaEventRecord(ev1, ctx->stream));
    return splits;
}

void build_stored_k(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n, int64_t r0,
                    int64_t nloc, double s, float *Kst) {
    const int64_t ldk = ((n + 3) / 4) * 4;
    dim3 grid((unsigned)ceil_div(n, 256), (unsigned)ceil_div(nloc, 16));
    if (kind == BBMM_RBF) {
        BBMM_DISPATCH_DIMS(dp, (k2_build<0, D_><<<grid, 256, 0, ctx->stream>>>(Xs, n, r0, nloc,
                                                                              ldk, (float)s, Kst)))
    } else {
        BBMM_DISPATCH_DIMS(dp, (k2_build<1, D_><<<grid, 256, 0, ctx->stream>>>(Xs, n, r0, nloc,
                                                                              ldk, (float)s, Kst)))
    }
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

int kernel_matmul_stored(bbmm_ctx_s *ctx, const float *Kst, int64_t n, int64_t nloc,
                         const float *D32, int cp, double *Vpart, size_t cap,
                         cudaEvent_t ev0, cudaEvent_t ev1) {
    const int64_t ldk = ((n + 3) / 4) * 4;
    int splits = choose_splits(n, nloc, 64, 2 * kNumSMs);
    BBMM_REQUIRE((size_t)splits * nloc * round4(cp) <= cap, "Vpart workspace too small");
    int64_t jchunk = ceil_div(ceil_div(n, splits), 128) * 128;
    dim3 grid((unsigned)ceil_div(nloc, 64), (unsigned)splits);
    if (ev0) BBMM_CUDA(cudaEventRecord(ev0, ctx->stream));
    if (nloc == 0) {
        if (ev1) BBMM_CUDA(cudaEventRecord(ev1, ctx->stream));
        return splits;
    }
    BBMM_DISPATCH_COLS(cp, (k2_stored<CP_><<<grid, 512, 0, ctx->stream>>>(Kst, n, nloc, ldk, D32,
                                                                           jchunk, Vpart)))
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    if (ev1) BBMM_CUDA(cudaEventRecord(ev1, ctx->stream));
    return splits;
}

}  // namespace bbmm
