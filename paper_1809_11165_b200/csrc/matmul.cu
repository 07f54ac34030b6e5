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
#include <type_traits>

#include "bbmm_internal.cuh"
#include "k1_kernels.cuh"
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
// K2 stream: V_i = sum_j Kst[i][j] D_j.  Reads Kst (fp32) once per matmul.
// Block = W warps; warp w owns rows blockRow + R w .. + R-1; lane l owns
// j = jt + 4l..4l+3 of each BJ = 128 tile (one coalesced 16-byte load per
// row).  The D tile is staged transposed (dT[c][j]) so each lane reads its 4
// j's of column c with conflict-free shared loads.
//   ACC64: D fp64, fp64 products and per-lane fp64 sums (butterfly at the end)
//   !ACC64: D fp32, 16-term per-lane fp32 partials folded into fp64 through a
//           5-level fp32 butterfly into the lane owning (r, c).
// --------------------------------------------------------------------------
template <int CP, bool ACC64>
__global__ void __launch_bounds__(256)
k2_stored(const float *__restrict__ Kst, int64_t n, int64_t nloc, int64_t ldk,
          const void *__restrict__ Dm_, int64_t jchunk, double *__restrict__ Vpart) {
    using DT = typename std::conditional<ACC64, double, float>::type;
    constexpr int CS = round4(CP);
    constexpr int R = 4, W = 8, BJ = 128, FOLD_TILES = 4;
    constexpr int NACC = (R * CP + 31) / 32;
    extern __shared__ __align__(16) unsigned char k2_smem[];
    DT(*dT)[BJ] = reinterpret_cast<DT(*)[BJ]>(k2_smem);   // [CP][BJ]
    const DT *__restrict__ Dm = reinterpret_cast<const DT *>(Dm_);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rowbase = (int64_t)blockIdx.x * (W * R) + warp * R;
    const int64_t j0 = (int64_t)blockIdx.y * jchunk;
    const int64_t j1 = min(n, j0 + jchunk);

    using AT = typename std::conditional<ACC64, double, float>::type;
    AT acc[R][CP];
    double acc64[NACC];
#pragma unroll
    for (int a = 0; a < NACC; a++) acc64[a] = 0.0;
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int c = 0; c < CP; c++) acc[r][c] = AT(0);

    int tile = 0;
    for (int64_t jt = j0; jt < j1; jt += BJ, tile++) {
        __syncthreads();
        for (int e = threadIdx.x; e < BJ * CP; e += W * 32) {
            int jj = e / CP, c = e - jj * CP;
            int64_t j = jt + jj;
            dT[c][jj] = (j < j1) ? Dm[j * CS + c] : DT(0);
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
            DT d0 = dT[c][4 * lane], d1 = dT[c][4 * lane + 1], d2 = dT[c][4 * lane + 2],
               d3 = dT[c][4 * lane + 3];
#pragma unroll
            for (int r = 0; r < R; r++) {
                AT a = acc[r][c];
                a = fma((AT)kv[r].x, (AT)d0, a);
                a = fma((AT)kv[r].y, (AT)d1, a);
                a = fma((AT)kv[r].z, (AT)d2, a);
                a = fma((AT)kv[r].w, (AT)d3, a);
                acc[r][c] = a;
            }
        }
        if (!ACC64 && ((tile + 1) % FOLD_TILES == 0 || jt + BJ >= j1)) {
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int c = 0; c < CP; c++) {
                    float v = (float)acc[r][c];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    const int idx = r * CP + c;
                    if (lane == (idx & 31)) acc64[idx >> 5] += (double)v;
                    acc[r][c] = AT(0);
                }
        }
    }
    if (ACC64) {
#pragma unroll
        for (int r = 0; r < R; r++)
#pragma unroll
            for (int c = 0; c < CP; c++) {
                double v = (double)acc[r][c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                const int idx = r * CP + c;
                if (lane == (idx & 31)) acc64[idx >> 5] = v;
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

void launch_k1_rbf_f64(bbmm_ctx_s *, int, int, const float *, int64_t, int64_t, int64_t,
                       const void *, double, double *, int);
void launch_k1_rbf_f32(bbmm_ctx_s *, int, int, const float *, int64_t, int64_t, int64_t,
                       const void *, double, double *, int);
void launch_k1_matern_f64(bbmm_ctx_s *, int, int, const float *, int64_t, int64_t, int64_t,
                          const void *, double, double *, int);
void launch_k1_matern_f32(bbmm_ctx_s *, int, int, const float *, int64_t, int64_t, int64_t,
                          const void *, double, double *, int);

template <int CP, bool ACC64>
static void launch_k2(bbmm_ctx_s *ctx, dim3 grid, const float *Kst, int64_t n, int64_t nloc,
                      int64_t ldk, const void *Dm, int64_t jchunk, double *Vpart) {
    const size_t smem = (size_t)CP * 128 * (ACC64 ? 8 : 4);
    static DeviceOnce attr;
    if (smem > 48 * 1024)
        attr(ctx->device, [&] {
            BBMM_CUDA(cudaFuncSetAttribute(k2_stored<CP, ACC64>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
    k2_stored<CP, ACC64><<<grid, 256, smem, ctx->stream>>>(Kst, n, nloc, ldk, Dm, jchunk, Vpart);
}

static int choose_splits(int64_t n, int64_t nloc, int64_t rows_per_block, int target_blocks) {
    int64_t rb = ceil_div(nloc, rows_per_block);
    int64_t sp = ceil_div(target_blocks, rb);
    sp = std::max<int64_t>(1, std::min<int64_t>(sp, ceil_div(n, 256)));
    return (int)sp;
}

size_t vpart_elems(int64_t n, int64_t nloc, int cp, bool stored) {
    int cs = round4(cp);
    int splits = stored ? choose_splits(n, nloc, 32, 4 * kNumSMs)
                        : choose_splits(n, nloc, 128, 6 * kNumSMs);
    return (size_t)splits * (size_t)nloc * cs;
}

int kernel_matmul_onthefly(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n,
                           int64_t r0, int64_t nloc, const void *Dm, bool acc64, int cp, double s,
                           double *Vpart, size_t cap, cudaEvent_t ev0, cudaEvent_t ev1) {
    int splits = choose_splits(n, nloc, 128, 6 * kNumSMs);
    BBMM_REQUIRE((size_t)splits * nloc * round4(cp) <= cap, "Vpart workspace too small");
    if (ev0) record_event(ctx, ev0);
    if (nloc == 0) {
        if (ev1) record_event(ctx, ev1);
        return splits;
    }
    if (kind == BBMM_RBF) {
        if (acc64) launch_k1_rbf_f64(ctx, dp, cp, Xs, n, r0, nloc, Dm, s, Vpart, splits);
        else launch_k1_rbf_f32(ctx, dp, cp, Xs, n, r0, nloc, Dm, s, Vpart, splits);
    } else {
        if (acc64) launch_k1_matern_f64(ctx, dp, cp, Xs, n, r0, nloc, Dm, s, Vpart, splits);
        else launch_k1_matern_f32(ctx, dp, cp, Xs, n, r0, nloc, Dm, s, Vpart, splits);
    }
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    if (ev1) record_event(ctx, ev1);
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
                         const void *Dm, bool acc64, int cp, double *Vpart, size_t cap,
                         cudaEvent_t ev0, cudaEvent_t ev1) {
    const int64_t ldk = ((n + 3) / 4) * 4;
    int splits = choose_splits(n, nloc, 32, 4 * kNumSMs);
    BBMM_REQUIRE((size_t)splits * nloc * round4(cp) <= cap, "Vpart workspace too small");
    int64_t jchunk = ceil_div(ceil_div(n, splits), 128) * 128;
    dim3 grid((unsigned)ceil_div(nloc, 32), (unsigned)splits);
    if (ev0) record_event(ctx, ev0);
    if (nloc == 0) {
        if (ev1) record_event(ctx, ev1);
        return splits;
    }
    if (acc64) {
        BBMM_DISPATCH_COLS(cp, launch_k2<CP_, true>(ctx, grid, Kst, n, nloc, ldk, Dm, jchunk, Vpart))
    } else {
        BBMM_DISPATCH_COLS(cp, launch_k2<CP_, false>(ctx, grid, Kst, n, nloc, ldk, Dm, jchunk, Vpart))
    }
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    if (ev1) record_event(ctx, ev1);
    return splits;
}

}  // namespace bbmm
