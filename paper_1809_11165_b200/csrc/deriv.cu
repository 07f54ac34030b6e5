// deriv.cu -- the derivative pass (K7): ONE matrix-free pass with the kernel
// derivatives after mBCG ("a single matrix multiply with the
// derivative", reading R17), fused into bilinear forms:
//
//   S_q = sum_{a,b} dK_q[a,b] W_ab,  W_ab = A_a . B_b,
//   A_a = [u_1..u_t, u_0](a)  (mBCG solves, local rows),
//   B_b = [(Phat^{-1} z_1..z_t)/t, -u_0](b)   (all rows),
// so S_q = tau_q - quad_q with tau_q = (1/t) sum_i u_i^T dK_q Phat^{-1} z_i
// (Hutchinson, Eq. 4 PAPER.md:669-684 with the P^{-1} correction, reading R13)
// and quad_q = u_0^T dK_q u_0 (Eq. 2), hence dmll/dtheta_q = -S_q / 2.
//
// dK_q for q over input dimensions (lengthscales; the isotropic gradient is
// the sum over q) and the outputscale (dK/dlog s = K):
//   RBF:    dK/dlog l_q = K * dx_q^2/l_q^2       = s k~ * dxs_q^2 * 2 ln 2
//   Matern: dK/dlog l_q = s (5/3)(1+rh) e^-rh dx_q^2/l_q^2 = s (1/3) g~ dxs_q^2
// (dxs = difference of the scaled inputs; host multiplies the constants).
#include <algorithm>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"

namespace bbmm {

namespace {

template <int KIND, int D, int CP>
__global__ void __launch_bounds__(128)
k7_deriv(const float *__restrict__ Xs, const float *__restrict__ A32,
         const float *__restrict__ B32, int64_t n, int64_t r0, int64_t nloc, int64_t jchunk,
         double *__restrict__ part) {
    constexpr int DS = round4(D), CS = round4(CP);
    constexpr int BJ = 64, FOLD = 16;
    __shared__ __align__(16) float xs[BJ][DS];
    __shared__ __align__(16) float bs[BJ][CS];
    __shared__ double red[128];

    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.x * 128 + tid;
    const bool valid = i < nloc;
    float xi[D], ai[CP];
#pragma unroll
    for (int q = 0; q < D; q++) xi[q] = valid ? Xs[(r0 + i) * DS + q] : 0.0f;
#pragma unroll
    for (int c = 0; c < CP; c++) ai[c] = valid ? A32[i * CS + c] : 0.0f;
    double s64[D + 1];
#pragma unroll
    for (int q = 0; q <= D; q++) s64[q] = 0.0;

    const int64_t j0 = (int64_t)blockIdx.y * jchunk;
    const int64_t j1 = min(n, j0 + jchunk);
    for (int64_t jt = j0; jt < j1; jt += BJ) {
        __syncthreads();
        {
            const float4 *X4 = reinterpret_cast<const float4 *>(Xs);
            const float4 *B4 = reinterpret_cast<const float4 *>(B32);
            float4 *xs4 = reinterpret_cast<float4 *>(&xs[0][0]);
            float4 *bs4 = reinterpret_cast<float4 *>(&bs[0][0]);
            for (int e = tid; e < BJ * DS / 4; e += 128) {
                int jj = e / (DS / 4);
                int64_t j = jt + jj;
                xs4[e] = (j < j1) ? X4[j * (DS / 4) + (e - jj * (DS / 4))]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int e = tid; e < BJ * CS / 4; e += 128) {
                int jj = e / (CS / 4);
                int64_t j = jt + jj;
                bs4[e] = (j < j1) ? B4[j * (CS / 4) + (e - jj * (CS / 4))]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int jf = 0; jf < BJ; jf += FOLD) {
            float s32[D + 1];
#pragma unroll
            for (int q = 0; q <= D; q++) s32[q] = 0.0f;
#pragma unroll 2
            for (int jj = jf; jj < jf + FOLD; jj++) {
                // four independent partial sums each for r^2 and W (instruction-level
                // parallelism: the single chains were latency-bound at low occupancy)
                float dq[D];
                float r4[4] = {0.0f, 0.0f, 0.0f, 0.0f}, w4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int q = 0; q < D; q++) {
                    float df = xi[q] - xs[jj][q];
                    dq[q] = df * df;
                    r4[q & 3] += dq[q];
                }
                const float rs2 = (r4[0] + r4[1]) + (r4[2] + r4[3]);
#pragma unroll
                for (int c = 0; c < CP; c++) w4[c & 3] = fmaf(ai[c], bs[jj][c], w4[c & 3]);
                const float w = (w4[0] + w4[1]) + (w4[2] + w4[3]);
                float kv, g;
                kval_and_dfac<KIND>(rs2, kv, g);
                float gw = g * w;
#pragma unroll
                for (int q = 0; q < D; q++) s32[q] = fmaf(gw, dq[q], s32[q]);
                s32[D] = fmaf(kv, w, s32[D]);
            }
#pragma unroll
            for (int q = 0; q <= D; q++) s64[q] += (double)s32[q];
        }
    }
    // block reduction of the D+1 accumulators (fixed order); fully unrolled so that s64
    // stays in registers (a runtime index would move it to local memory)
    const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
#pragma unroll
    for (int q = 0; q <= D; q++) {
        __syncthreads();
        red[tid] = s64[q];
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int u = 0; u < 128; u++) s += red[u];
            part[blk * (D + 1) + q] = s;
        }
    }
}

}  // namespace

#define BBMM_D7_COLS(CPV, ...)                                                            \
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

#define BBMM_D7_DIMS(DV, ...)                                                             \
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

template <int KIND, int D, int CP>
static void launch_k7(bbmm_ctx_s *ctx, const float *Xs, int64_t n, int64_t r0, int64_t nloc,
                      const float *A32, const float *B32, double *part, int *nblocks) {
    int64_t rb = ceil_div(nloc, 128);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(6 * kNumSMs, rb), ceil_div(n, 256)));
    int64_t jchunk = ceil_div(ceil_div(n, sp), 64) * 64;
    sp = ceil_div(n, jchunk);
    dim3 grid((unsigned)rb, (unsigned)sp);
    k7_deriv<KIND, D, CP><<<grid, 128, 0, ctx->stream>>>(Xs, A32, B32, n, r0, nloc, jchunk, part);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    *nblocks = (int)(rb * sp);
}

size_t derivative_part_elems(int64_t n, int64_t nloc, int dp) {
    int64_t rb = ceil_div(nloc, 128);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(6 * kNumSMs, rb), ceil_div(n, 256)));
    return (size_t)(rb * sp) * (dp + 1);
}

void derivative_pass(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n, int64_t r0,
                     int64_t nloc, const float *A32, const float *B32, int cp, int nq_out,
                     bool ard, int d, double *part, int *nblocks_out) {
    (void)nq_out; (void)ard; (void)d;
    if (kind == BBMM_RBF) {
        BBMM_D7_DIMS(dp, BBMM_D7_COLS(cp, launch_k7<0, D_, CP_>(ctx, Xs, n, r0, nloc, A32, B32,
                                                                 part, nblocks_out)))
    } else {
        BBMM_D7_DIMS(dp, BBMM_D7_COLS(cp, launch_k7<1, D_, CP_>(ctx, Xs, n, r0, nloc, A32, B32,
                                                                 part, nblocks_out)))
    }
}

}  // namespace bbmm
