// k1_kernels.cuh -- template of the on-the-fly kernel-matmul kernel (K1).
// Instantiated per (kernel kind, accumulation mode) in k1_*.cu so the many
// shape instantiations compile in parallel.
#pragma once

#include <type_traits>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"

namespace bbmm {

// --------------------------------------------------------------------------
// K1: on-the-fly kernel matmul.
// Block = 128 threads, each thread owns R rows (rows blockRow + tid + 128 r).
// j-range of the block = split blockIdx.y.  Tiles of BJ = 64 points of
// (xs_j, D_j) are staged in shared memory; every thread reads them as
// broadcasts.  Inner loop per (row, j): distance (2D FLOP), one ex2 (MUFU),
// then the contraction with the CP columns of D_j:
//   ACC64 (default): D fp64, k_ij converted to fp64,
//          CP DFMAs into fp64 accumulators (exact products, fp64 sums);
//   !ACC64 (fast):  D fp32, CP FFMAs into fp32 accumulators folded into fp64
//          every 16 j (valid only where the Krylov iteration has converged,
//          SURVEY.md §8c regime A).
// --------------------------------------------------------------------------
template <int KIND, int D, int CP, int R, bool ACC64>
__global__ void __launch_bounds__(128)
k1_onthefly(const float *__restrict__ Xs, const void *__restrict__ Dm_, int64_t n, int64_t r0,
            int64_t nloc, int64_t jchunk, double s, double *__restrict__ Vpart) {
    using DT = typename std::conditional<ACC64, double, float>::type;
    constexpr int DS = round4(D), CS = round4(CP);
    constexpr int BJ = 64, FOLD = 16;
    __shared__ __align__(16) float xs[BJ][DS];
    __shared__ __align__(16) DT dsm[BJ][CS];
    const DT *__restrict__ Dm = reinterpret_cast<const DT *>(Dm_);

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
            float4 *xs4 = reinterpret_cast<float4 *>(&xs[0][0]);
            for (int e = tid; e < BJ * DS / 4; e += 128) {
                int jj = e / (DS / 4);
                int64_t j = jt + jj;
                xs4[e] = (j < j1) ? X4[j * (DS / 4) + (e - jj * (DS / 4))]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            constexpr int V16 = 16 / sizeof(DT);   // elements per 16-byte vector
            const int4 *D4 = reinterpret_cast<const int4 *>(Dm);
            int4 *ds4 = reinterpret_cast<int4 *>(&dsm[0][0]);
            for (int e = tid; e < BJ * CS / V16; e += 128) {
                int jj = e / (CS / V16);
                int64_t j = jt + jj;
                ds4[e] = (j < j1) ? D4[j * (CS / V16) + (e - jj * (CS / V16))]
                                  : make_int4(0, 0, 0, 0);
            }
        }
        __syncthreads();
        if (ACC64) {
#pragma unroll 2
            for (int jj = 0; jj < BJ; jj++) {
                float xj[D];
#pragma unroll
                for (int q = 0; q < D; q++) xj[q] = xs[jj][q];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float rs2 = 0.0f;
#pragma unroll
                    for (int q = 0; q < D; q++) {
                        float df = xi[r][q] - xj[q];
                        rs2 = fmaf(df, df, rs2);
                    }
                    const double kv = (double)kval_scaled<KIND>(rs2);
#pragma unroll
                    for (int c = 0; c < CP; c++) a64[r][c] = fma(kv, (double)dsm[jj][c], a64[r][c]);
                }
            }
        } else {
#pragma unroll 1
            for (int jf = 0; jf < BJ; jf += FOLD) {
                float a32[R][CP];
#pragma unroll
                for (int r = 0; r < R; r++)
#pragma unroll
                    for (int c = 0; c < CP; c++) a32[r][c] = 0.0f;
#pragma unroll 2
                for (int jj = jf; jj < jf + FOLD; jj++) {
                    float xj[D];
#pragma unroll
                    for (int q = 0; q < D; q++) xj[q] = xs[jj][q];
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
                        for (int c = 0; c < CP; c++)
                            a32[r][c] = fmaf(kv, (float)dsm[jj][c], a32[r][c]);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; r++)
#pragma unroll
                    for (int c = 0; c < CP; c++) a64[r][c] += (double)a32[r][c];
            }
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


// (D, CP) shape dispatch shared by the pair kernels.
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

template <int KIND, bool ACC64>
void launch_k1_variant(bbmm_ctx_s *ctx, int dp, int cp, const float *Xs, int64_t n, int64_t r0,
                       int64_t nloc, const void *Dm, double s, double *Vpart, int splits) {
    BBMM_DISPATCH_DIMS(dp, BBMM_DISPATCH_COLS(cp, {
        constexpr int R = (CP_ <= 17) ? 2 : 1;
        dim3 grid((unsigned)ceil_div(nloc, 128 * R), (unsigned)splits);
        int64_t jchunk = ceil_div(ceil_div(n, splits), 64) * 64;
        k1_onthefly<KIND, D_, CP_, R, ACC64><<<grid, 128, 0, ctx->stream>>>(Xs, Dm, n, r0, nloc,
                                                                            jchunk, s, Vpart);
    }))
}

}  // namespace bbmm
