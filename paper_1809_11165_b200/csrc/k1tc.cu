// k1tc.cu -- operand preparation shared by the tensor-core kernel-matmul
// (k1tc2.cu): per-column scales of the search directions and their packing
// into the int8 slice tiles the tcgen05 MMAs consume, plus the input mean.
//
// Packed operand:
//   D_jc  -> P'_jc = round(D_jc / S_c 2^30) + 2^30 in [0, 2^31], four u8
//            slices p3 p2 p1 p0 (S_c = max_j |D_jc|); one extra constant
//            column with P' = 2^30 removes the offset exactly.
#include <algorithm>
#include <cmath>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"

namespace bbmm {

namespace tc {

constexpr int BK = 64;                        // points per packed chunk group (16-point chunks)

__global__ void k_col_mean(const float *__restrict__ X, int64_t n, int d, double *__restrict__ mean) {
    const int q = blockIdx.x;
    __shared__ double sh[256];
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += (double)X[j * d + q];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) mean[q] = sh[0] / (double)n;
}

// per-block partial max |D_c| over rows (threadIdx.x = column)
__global__ void k_colmax_part(const double *__restrict__ D, int64_t ldd, int64_t rows, int c,
                              double *__restrict__ part) {
    const int col = threadIdx.x;
    __shared__ double sh[256];
    double m = 0.0;
    if (col < c)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < rows;
             i += (int64_t)gridDim.x * blockDim.y)
            m = fmax(m, fabs(D[i * ldd + col]));
    sh[threadIdx.y * blockDim.x + col] = m;
    __syncthreads();
    if (threadIdx.y == 0 && col < c) {
        for (int y = 1; y < blockDim.y; y++) m = fmax(m, sh[y * blockDim.x + col]);
        part[(int64_t)blockIdx.x * c + col] = m;
    }
}
// one warp per column (max is order-independent)
__global__ void k_colmax_final(const double *__restrict__ part, int nblk, int c, double *__restrict__ S) {
    const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (col >= c) return;
    double m = 0.0;
    for (int b = lane; b < nblk; b += 32) m = fmax(m, part[(int64_t)b * c + col]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    // raw maximum (0 for an all-zero column or a rank without rows): the caller may all-reduce
    // it (max) across ranks, so no substitute value here -- a rank with no rows must not
    // contribute 1.0 (that coarsened every rank's fixed-point D to a 2^-31 grid of 1.0 once
    // mBCG had converged: stagnation at relres ~5e-9 and an alpha breakdown on 4 ranks)
    if (lane == 0) S[col] = m;
}

// Pack rows [row0, row0 + rows) of D (fp64) into the K-major slice layout
// [16-point chunk][NB rows][16 bytes] (linear in the chunk index, so any
// multiple-of-16 j-tile is contiguous): row n = b_idx * BLK + col, b_idx
// 0..ND-1 = bytes ND-1..0 of P' = round(D/S 2^T) + 2^T with T = 8 ND - 2
// (ND = 4: 31-bit, K1-TC; ND = 5 / 7: Matern / stored K).  The operand is laid out for a
// kernel instantiated for cb >= c columns: columns c..cb-1 are zero D (P' = 2^T), column cb
// is the constant 2^T that removes the offset, columns > cb zero padding.  One thread writes
// the 16 bytes of one (chunk, n).
__global__ void k_pack_bslices(const double *__restrict__ D, int64_t ldd, int64_t row0,
                               int64_t rows, int64_t n, int c, int cb, int BLK, int NB, int ND,
                               const double *__restrict__ S, uint8_t *__restrict__ Bpack,
                               int64_t tile0, int64_t tiles) {
    const int T = 8 * ND - 2;
    const double scaleT = ldexp(1.0, T);
    const int64_t offT = 1LL << T;
    const int64_t total = tiles * (BK / 16) * NB;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int nn = (int)(e % NB);
        const int64_t rest = e / NB;
        const int kc = (int)(rest % (BK / 16));
        const int64_t tt = tile0 + rest / (BK / 16);
        const int bi = nn / BLK, col = nn - bi * BLK;
        uint32_t wv[4] = {0, 0, 0, 0};
        if (bi < ND && col <= cb) {
            const int shift = 8 * (ND - 1 - bi);
#pragma unroll
            for (int p = 0; p < 16; p++) {
                const int64_t j = tt * BK + kc * 16 + p;       // global point index
                uint32_t byte = 0;
                if (j < n && j >= row0 && j < row0 + rows) {
                    int64_t P;
                    if (col < c) {
                        const double sc = S[col] > 0.0 ? S[col] : 1.0;   // all-zero column
                        double q = D[(j - row0) * ldd + col] / sc * scaleT;
                        P = llrint(q) + offT;                  // in [0, 2^(T+1)]
                    } else {
                        P = offT;                              // constant column
                    }
                    byte = (uint32_t)((P >> shift) & 0xFF);
                }
                wv[p >> 2] |= byte << (8 * (p & 3));
            }
        }
        uint8_t *dst = Bpack + tt * (int64_t)NB * BK + (int64_t)kc * NB * 16 + (int64_t)nn * 16;
        *reinterpret_cast<uint4 *>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
}

}  // namespace tc

// ======================================================================
// host side
// ======================================================================
// rows of the packed D-slice operand: 4 blocks of BLK = round4(c + 1)
// columns (matching k1tc2's accumulator blocks)
int k1tc_bslice_rows(int c) { return 4 * ((c + 1 + 3) & ~3); }
// ND = 5 (K2-TC): the MMA N = 5 BLK must be a multiple of 16, so BLK = round16(c + 1)
int tc_bslice_rows(int c, int nd) { return nd == 4 ? k1tc_bslice_rows(c) : nd * ((c + 1 + 15) & ~15); }
int tc_dslices(const TcOperand &op) { return op.nd; }

void k1tc_col_mean(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, double *mean) {
    tc::k_col_mean<<<d, 256, 0, ctx->stream>>>(X, n, d, mean);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

// rows covered by the tensor-core operands: a multiple of 384 = lcm(128-row
// partitions, 96-point j-tiles)
int64_t k1tc_pad_rows(int64_t n) { return ceil_div(n, 384) * 384; }

// S (c doubles, device): column max |D| over the rows given (local rows);
// caller all-reduces (max) across ranks if needed.
void k1tc_colmax(bbmm_ctx_s *ctx, const double *D, int64_t ldd, int64_t rows, int c, double *S) {
    // columns c.. of S (padding columns of a wider kernel instantiation) read as 0
    if (c < kMaxCols) BBMM_CUDA(cudaMemsetAsync(S + c, 0, (size_t)(kMaxCols - c) * 8, ctx->stream));
    const int cw = c <= 32 ? 32 : 64, rb = 256 / cw;
    int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, rb), 2 * kNumSMs));
    double *part = (double *)ctx->ws.get("tc_cmax", (size_t)nblk * c * 8);
    tc::k_colmax_part<<<nblk, dim3(cw, rb), 0, ctx->stream>>>(D, ldd, rows, c, part);
    tc::k_colmax_final<<<(int)ceil_div(c, 8), 256, 0, ctx->stream>>>(part, nblk, c, S);
    BBMM_LAUNCH_CHECK();
    ctx->launches += 2;
}

// Pack local rows [row0, row0 + rows) into Bpack (tiles covering them).
void k1tc_pack(bbmm_ctx_s *ctx, const double *D, int64_t ldd, int64_t row0, int64_t rows,
               int64_t n, int c, const double *S, uint8_t *Bpack, int nd, int cb) {
    if (cb < c) cb = c;
    const int NB = tc_bslice_rows(cb, nd), BLK = NB / nd;
    // the rank holding the last rows also writes the zero padding up to
    // k1tc_pad_rows(n) (the j-tiles read past n); the layout is linear in
    // 16-point chunks, [chunk][NB][16 B], so any tile width reads it
    const int64_t end = (row0 + rows >= n) ? k1tc_pad_rows(n) : row0 + rows;
    const int64_t tile0 = row0 / tc::BK;
    const int64_t tiles = ceil_div(end, tc::BK) - tile0;
    const int64_t total = tiles * (tc::BK / 16) * NB;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 8 * kNumSMs));
    tc::k_pack_bslices<<<grid, 256, 0, ctx->stream>>>(D, ldd, row0, rows, n, c, cb, BLK, NB, nd, S,
                                                      Bpack, tile0, tiles);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

}  // namespace bbmm
