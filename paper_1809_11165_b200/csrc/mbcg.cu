// mbcg.cu -- modified batched preconditioned CG (Alg. S2)
// on the GPU: the per-iteration vector updates, the Woodbury preconditioner
// apply (App. B, sign-corrected: DESIGN.md R10), the
// per-column fp64 dot products, and the Lanczos coefficient record
// (PAPER.md:342-344 / display PAPER.md:468-475).
//
// Data layout (local rows of this rank, row-major, fp64):
//   U, R, Z, D, V : nloc x c        (ld = c)
//   Dm            : n_pad x CS fp64/fp32 matmul copy of D (all rows; this rank writes r0..r1;
//                                    the all-gather fills the rest)
//   L             : k x n fp64      (row m = pivoted-Cholesky column m)
// One iteration j (textbook signs, reading R5/R6):
//   V = Khat D ; alpha = rho / <D,V> ; U += alpha D ; R -= alpha V ;
//   relres = |R| / |B| (freeze if < tol) ; S = C^{-1} L^T R ;
//   Z = (R - L S)/sigma^2 ; rho' = <R,Z> ; beta = rho'/rho ; D = Z + beta D.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "bbmm_internal.cuh"

namespace bbmm {

namespace {

constexpr int kRedBlocks = 2 * kNumSMs;   // persistent reduction grid

// Column-major thread layout for the O(n c) passes: threadIdx.x = column
// (blockDim.x = CW, a multiple of 32 >= c), threadIdx.y = row within block.
struct PassGeom {
    int cw, rb;
    dim3 block, grid;
};

PassGeom pass_geom(int64_t nloc, int c) {
    PassGeom g;
    g.cw = c <= 32 ? 32 : 64;
    g.rb = 256 / g.cw;
    g.block = dim3(g.cw, g.rb);
    int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, g.rb), kRedBlocks));
    g.grid = dim3((unsigned)blocks);
    return g;
}

// Block-level reduction over threadIdx.y of a per-thread fp64 value for the
// thread's column, written to part[blockIdx.x * m + col].
__device__ void block_reduce_cols(double v, double *part, int m, int col_offset) {
    __shared__ double sred[256];
    const int tx = threadIdx.x, ty = threadIdx.y, cw = blockDim.x, rb = blockDim.y;
    sred[ty * cw + tx] = v;
    __syncthreads();
    if (ty == 0) {
        double s = 0.0;
        for (int y = 0; y < rb; y++) s += sred[y * cw + tx];
        if (col_offset + tx < m) part[(int64_t)blockIdx.x * m + col_offset + tx] = s;
    }
    __syncthreads();
}

// --------------------------------------------------------------- kernels
// red[e] = sum_b part[b][e]: one warp per output, lane l sums b = l, l + 32, ..
// in order, then a fixed xor-butterfly (every lane ends with the same value):
// deterministic, and ~nblk/32 dependent loads instead of nblk.
__global__ void k_reduce_blocks(const double *__restrict__ part, int nblk, int m,
                                double *__restrict__ red) {
    const int lane = threadIdx.x & 31;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m;
         e += (gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * m + e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[e] = s;
    }
}
inline int reduce_grid(int m) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 8), 8 * kNumSMs));
}

// R = B, U = 0, D = 0 ; partial sum of B^2 per column.
__global__ void k_init_vectors(const double *__restrict__ B, int64_t ldb, int64_t nloc, int c,
                               double *__restrict__ U, double *__restrict__ R,
                               double *__restrict__ D, double *__restrict__ part) {
    const int col = threadIdx.x;
    double acc = 0.0;
    if (col < c) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < nloc;
             i += (int64_t)gridDim.x * blockDim.y) {
            double b = B[i * ldb + col];
            R[i * c + col] = b;
            U[i * c + col] = 0.0;
            D[i * c + col] = 0.0;
            acc += b * b;
        }
    }
    block_reduce_cols(acc, part, c, 0);
}

// W partial = L^T R over this block's rows: part[blk][m*c + col].
// HBM-bound skinny product (L: k x n fp64 read once).  Block = 8 warps; per
// chunk of kLtrRows rows the R rows are staged in shared memory, then warp w
// takes m = w, w + 8, ..: each lane walks rows lane, lane + 32, .. of the
// chunk (L[m][row] reads coalesced across the warp), keeps the c products in
// registers, and one shuffle reduction per (m, chunk) adds them into the
// block's k x c accumulator (each m owned by one warp: deterministic).
constexpr int kLtrRows = 256;
template <int CMAX>
__global__ void __launch_bounds__(256)
k_LtR(const double *__restrict__ L, int64_t n, int64_t r0, int k, const double *__restrict__ R,
      int64_t nloc, int c, double *__restrict__ part) {
    extern __shared__ double sm_ltr[];
    double *Rt = sm_ltr;                          // kLtrRows x c
    double *acc = Rt + kLtrRows * c;              // k x c block accumulator
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < k * c; e += 256) acc[e] = 0.0;
    for (int64_t i0 = (int64_t)blockIdx.x * kLtrRows; i0 < nloc;
         i0 += (int64_t)gridDim.x * kLtrRows) {
        const int rows = (int)(nloc - i0 < kLtrRows ? nloc - i0 : kLtrRows);
        __syncthreads();
        for (int e = tid; e < rows * c; e += 256) Rt[e] = R[i0 * c + e];
        __syncthreads();
        for (int m = warp; m < k; m += 8) {
            const double *Lm = L + (int64_t)m * n + r0 + i0;
            double v[CMAX];
#pragma unroll
            for (int q = 0; q < CMAX; q++) v[q] = 0.0;
            for (int r = lane; r < rows; r += 32) {
                const double l = Lm[r];
                const double *rr = Rt + r * c;
#pragma unroll
                for (int q = 0; q < CMAX; q++)
                    if (q < c) v[q] = fma(l, rr[q], v[q]);
            }
#pragma unroll
            for (int q = 0; q < CMAX; q++) {
                if (q < c) {
                    double s = v[q];
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (lane == 0) acc[m * c + q] += s;
                }
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < k * c; e += 256) part[(int64_t)blockIdx.x * k * c + e] = acc[e];
}

// Split-K register-tiled version of the same product (used when it fits): block b
// owns a contiguous range of rows and ALL k x c outputs; thread t owns the column
// group g = t % CGN (4 columns) and the rows m = t / CGN + j * MLN (j < MPT) of W,
// accumulated in registers over the whole range -- one write per output, no
// shuffles.  Per 16/32-row step the L tile (k x KT, stored transposed) and the
// R tile are staged in shared memory; L reads are coalesced along the rows.
template <int MPT>
__global__ void __launch_bounds__(256, 2)
k_LtR2(const double *__restrict__ L, int64_t n, int64_t r0, int k, const double *__restrict__ R,
       int64_t nloc, int c, int64_t rows_per_blk, int KT, double *__restrict__ part) {
    extern __shared__ double sm_l2[];
    double *Lt = sm_l2;                           // KT x k  (Lt[kk * k + m])
    double *Rt = Lt + (size_t)KT * k;             // KT x c
    const int CGN = (c + 3) / 4, MLN = 256 / CGN;
    const int g = threadIdx.x % CGN, ml = threadIdx.x / CGN;
    const bool act = ml < MLN;
    double acc[MPT][4];
#pragma unroll
    for (int j = 0; j < MPT; j++)
#pragma unroll
        for (int u = 0; u < 4; u++) acc[j][u] = 0.0;
    const int64_t i_beg = (int64_t)blockIdx.x * rows_per_blk;
    const int64_t i_end = min(nloc, i_beg + rows_per_blk);
    // The next chunk's L / R values are loaded into registers while the current chunk is
    // multiplied (one chunk of loads in flight per thread instead of none): up to
    // kPF elements per thread, else the loads are issued just before the stores.
    constexpr int kPF = MPT <= 4 ? 24 : 0;
    double lr[kPF > 0 ? kPF : 1];
    const int nl = (k * KT + 255) / 256, nr = (KT * c + 255) / 256;
    const bool pf = kPF > 0 && nl + nr <= kPF;
    // fully unrolled over kPF with runtime predicates, so lr[] stays in registers
    auto fetch = [&](int64_t i0, double *dst) {
        const int rows = (int)min((int64_t)KT, i_end - i0);
#pragma unroll
        for (int q = 0; q < (kPF > 0 ? kPF : 1); q++) {
            double v = 0.0;
            if (q < nl) {
                const int e = threadIdx.x + 256 * q;
                const int m = e / KT, kk = e - m * KT;
                if (e < k * KT && kk < rows) v = L[(int64_t)m * n + r0 + i0 + kk];
            } else if (q < nl + nr) {
                const int e = threadIdx.x + 256 * (q - nl);
                if (e < KT * c && e / c < rows) v = R[i0 * c + e];
            }
            dst[q] = v;
        }
    };
    if (pf && i_beg < i_end) fetch(i_beg, lr);
    for (int64_t i0 = i_beg; i0 < i_end; i0 += KT) {
        const int rows = (int)min((int64_t)KT, i_end - i0);
        __syncthreads();
        if (pf) {
#pragma unroll
            for (int q = 0; q < (kPF > 0 ? kPF : 1); q++) {
                if (q < nl) {
                    const int e = threadIdx.x + 256 * q;
                    if (e < k * KT) Lt[(e % KT) * k + e / KT] = lr[q];
                } else if (q < nl + nr) {
                    const int e = threadIdx.x + 256 * (q - nl);
                    if (e < KT * c) Rt[e] = lr[q];
                }
            }
        } else {
            for (int e = threadIdx.x; e < k * KT; e += 256) {
                const int m = e / KT, kk = e - m * KT;
                Lt[kk * k + m] = kk < rows ? L[(int64_t)m * n + r0 + i0 + kk] : 0.0;
            }
            for (int e = threadIdx.x; e < KT * c; e += 256) {
                const int kk = e / c;
                Rt[e] = kk < rows ? R[i0 * c + e] : 0.0;
            }
        }
        __syncthreads();
        if (pf && i0 + KT < i_end) fetch(i0 + KT, lr);
        if (act) {
            for (int kk = 0; kk < KT; kk++) {
                double r[4];
#pragma unroll
                for (int u = 0; u < 4; u++) r[u] = (4 * g + u < c) ? Rt[kk * c + 4 * g + u] : 0.0;
#pragma unroll
                for (int j = 0; j < MPT; j++) {
                    const int m = ml + j * MLN;
                    const double l = m < k ? Lt[kk * k + m] : 0.0;
#pragma unroll
                    for (int u = 0; u < 4; u++) acc[j][u] = fma(l, r[u], acc[j][u]);
                }
            }
        }
    }
    if (act) {
#pragma unroll
        for (int j = 0; j < MPT; j++) {
            const int m = ml + j * MLN;
            if (m < k)
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (4 * g + u < c) part[(int64_t)blockIdx.x * k * c + m * c + 4 * g + u] = acc[j][u];
        }
    }
}

// The same product for a tall L (K >= 128 rows: the SoR operator's Bs, m x n) with the tiles
// streamed through a 3-stage cp.async ring instead of registers: one 256-thread block per SM,
// each owning a contiguous row range; per 16-row step the K x 16 tile of L (row-major, rows
// padded to 18 doubles: the 7 rows a warp reads at one kk fall in distinct banks) and the
// 16 x c tile of R land in shared memory while the two previous steps are multiplied -- two
// 45 KB steps in flight per SM instead of one register-staged step (k_LtR2 reached ~1.1 TB/s
// on the 2.4 GB Bs of n = 1M, m = 300).  Thread = MPT rows of L x 4 columns of R, as k_LtR2.
// Requires n, r0 and the rows per block even (16-byte chunks); the caller checks.
namespace {
__device__ __forceinline__ void cp16(void *dst, const void *src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
}  // namespace
#ifndef BBMM_LTR3_T
#define BBMM_LTR3_T 16
#endif
#ifndef BBMM_LTR3_ST
#define BBMM_LTR3_ST 3
#endif
constexpr int kL3T = BBMM_LTR3_T, kL3Ld = BBMM_LTR3_T + 2, kL3St = BBMM_LTR3_ST;
template <int MPT, int NT = 256>
__global__ void __launch_bounds__(NT, 1)
k_LtR3(const double *__restrict__ L, int64_t n, int64_t r0, int k, const double *__restrict__ R,
       int64_t nloc, int c, int64_t rows_per_blk, double *__restrict__ part) {
    extern __shared__ __align__(16) double sm_l3[];
    const int stage_d = k * kL3Ld + kL3T * c + 2;      // doubles per stage (keep 16-B alignment)
    const int stage = (stage_d + 1) & ~1;
    BBMM_DCHECK((size_t)kL3St * stage * 8 <= dyn_smem_bytes());
    const int CGN = (c + 3) / 4, MLN = NT / CGN;
    const int g = threadIdx.x % CGN, ml = threadIdx.x / CGN;
    const bool act = ml < MLN;
    double acc[MPT][4];
#pragma unroll
    for (int j = 0; j < MPT; j++)
#pragma unroll
        for (int u = 0; u < 4; u++) acc[j][u] = 0.0;
    const int64_t i_beg = (int64_t)blockIdx.x * rows_per_blk;
    const int64_t i_end = min(nloc, i_beg + rows_per_blk);
    const int nsteps = i_beg < i_end ? (int)((i_end - i_beg + kL3T - 1) / kL3T) : 0;
    auto load = [&](int st) {
        double *Ls = sm_l3 + (size_t)(st % kL3St) * stage;
        double *Rs = Ls + (size_t)k * kL3Ld;
        const int64_t i0 = i_beg + (int64_t)st * kL3T;
        const int rows = (int)min((int64_t)kL3T, i_end - i0);
        // L: k rows x 8 chunks of 2 doubles
        for (int e = threadIdx.x; e < k * (kL3T / 2); e += NT) {
            const int m = e / (kL3T / 2), q = e % (kL3T / 2);
            const bool ok = 2 * q < rows;            // rows is even except at the very end
            const double *src = L + (int64_t)m * n + r0 + i0 + (ok ? 2 * q : 0);
            BBMM_DCHECK(m < k && r0 + i0 + (ok ? 2 * q + (2 * q + 1 < rows ? 2 : 1) : 0) <= n);
            cp16(Ls + m * kL3Ld + 2 * q, src, ok ? (2 * q + 1 < rows ? 16 : 8) : 0);
        }
        // R: rows x c doubles, contiguous
        const int rd = rows * c, rchunks = (kL3T * c + 1) / 2;
        for (int e = threadIdx.x; e < rchunks; e += NT) {
            const int o = 2 * e;
            const int nb = o + 1 < rd ? 16 : (o < rd ? 8 : 0);
            BBMM_DCHECK(i0 * c + (nb ? o + nb / 8 : 0) <= nloc * c);
            cp16(Rs + o, R + i0 * c + (nb ? o : 0), nb);
        }
    };
    for (int st = 0; st < kL3St - 1; st++) {
        if (st < nsteps) load(st);
        cp_commit();
    }
    for (int st = 0; st < nsteps; st++) {
        if (st + kL3St - 1 < nsteps) load(st + kL3St - 1);
        cp_commit();
        cp_wait<kL3St - 1>();
        __syncthreads();
        const double *Ls = sm_l3 + (size_t)(st % kL3St) * stage;
        const double *Rs = Ls + (size_t)k * kL3Ld;
        if (act) {
            // two kk per step: the L pair (kk, kk + 1) of a row is one 16-byte shared load
#pragma unroll 2
            for (int kk = 0; kk < kL3T; kk += 2) {
                double r0[4], r1[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    r0[u] = (4 * g + u < c) ? Rs[kk * c + 4 * g + u] : 0.0;
                    r1[u] = (4 * g + u < c) ? Rs[(kk + 1) * c + 4 * g + u] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < MPT; j++) {
                    const int m = ml + j * MLN;
                    const double2 l = m < k ? *reinterpret_cast<const double2 *>(Ls + m * kL3Ld + kk)
                                            : make_double2(0.0, 0.0);
#pragma unroll
                    for (int u = 0; u < 4; u++) acc[j][u] = fma(l.y, r1[u], fma(l.x, r0[u], acc[j][u]));
                }
            }
        }
        __syncthreads();            // the stage is refilled by the next iteration's load
    }
    cp_wait<0>();
    if (act) {
#pragma unroll
        for (int j = 0; j < MPT; j++) {
            const int m = ml + j * MLN;
            if (m < k)
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (4 * g + u < c) part[(int64_t)blockIdx.x * k * c + m * c + 4 * g + u] = acc[j][u];
        }
    }
}
size_t ltr3_smem(int k, int c) {
    const int stage_d = k * kL3Ld + kL3T * c + 2;
    return (size_t)kL3St * ((stage_d + 1) & ~1) * 8;
}

// S = C^{-1} W (k x c), C = chol factor (lower, k x k row-major).  One warp per
// column (warp w takes columns w, w + 32, ..): forward then backward
// substitution with the column kept in shared memory and each inner product
// split over the lanes (fixed lane order + xor butterfly: deterministic).
// Launch: one block of kSolveThreads threads, dynamic smem kSolveThreads/32 * k doubles.
constexpr int kSolveThreads = 1024;
__device__ void chol_solve_warps(const double *__restrict__ cholC, int k, const double *W,
                                 double *__restrict__ S, int c) {
    extern __shared__ double sol_sh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *x = sol_sh + (size_t)warp * k;
    for (int col = warp; col < c; col += (int)(blockDim.x >> 5)) {
        for (int a = 0; a < k; a++) {
            double p = 0.0;
            for (int b = lane; b < a; b += 32) p = fma(cholC[a * k + b], x[b], p);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (lane == 0) x[a] = (W[a * c + col] - p) / cholC[a * k + a];
            __syncwarp();
        }
        for (int a = k - 1; a >= 0; a--) {
            double p = 0.0;
            for (int b = a + 1 + lane; b < k; b += 32) p = fma(cholC[b * k + a], x[b], p);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (lane == 0) x[a] = (x[a] - p) / cholC[a * k + a];
            __syncwarp();
        }
        for (int a = lane; a < k; a += 32) S[a * c + col] = x[a];
        __syncwarp();
    }
}

// SoR operator (row f4): Vpart[i][col] = sum_a Bs[a][r0 + i] T[a][col] (= K_SoR D on the
// local rows; k_passA adds sigma^2 D).  Thread = one row, all columns in registers (Bs
// read once, coalesced across the warp); T from shared memory (broadcast).
template <int CMAX>
__global__ void __launch_bounds__(256)
k_sor_expand(const double *__restrict__ Bs, int64_t n, int64_t r0, int m,
             const double *__restrict__ T, int64_t nloc, int c, int cs, double *__restrict__ Vpart) {
    extern __shared__ double Tsm[];   // m x c
    for (int e = threadIdx.x; e < m * c; e += blockDim.x) Tsm[e] = T[e];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc[CMAX];
#pragma unroll
        for (int u = 0; u < CMAX; u++) acc[u] = 0.0;
        for (int a = 0; a < m; a++) {
            const double b = Bs[(int64_t)a * n + r0 + i];
#pragma unroll
            for (int u = 0; u < CMAX; u++)
                if (u < c) acc[u] = fma(b, Tsm[a * c + u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < CMAX; u++)
            if (u < c) Vpart[i * cs + u] = acc[u];
    }
}

// k_sor_expand with two rows per thread (i and i + 256 within a 512-row block slab) and T read as
// 16-byte pairs (rows padded to an even count): half the shared-memory loads per Bs element and
// twice the loads in flight (k_sor_expand reached ~2 TB/s on n = 1M, m = 300).
template <int CMAX>
__global__ void __launch_bounds__(256)
k_sor_expand2(const double *__restrict__ Bs, int64_t n, int64_t r0, int m,
              const double *__restrict__ T, int64_t nloc, int c, int cs, double *__restrict__ Vpart) {
    constexpr int CP = (CMAX + 1) & ~1;
    extern __shared__ __align__(16) double Tp[];   // m x CP (zero padded)
    BBMM_DCHECK((uint32_t)m * CP * 8 <= dyn_smem_bytes());
    for (int e = threadIdx.x; e < m * CP; e += blockDim.x) {
        const int a = e / CP, u = e - a * CP;
        Tp[e] = u < c ? T[a * c + u] : 0.0;
    }
    __syncthreads();
    for (int64_t base = (int64_t)blockIdx.x * 512; base < nloc; base += (int64_t)gridDim.x * 512) {
        const int64_t i0 = base + threadIdx.x, i1 = i0 + 256;
        const bool v0 = i0 < nloc, v1 = i1 < nloc;
        double a0[CP], a1[CP];
#pragma unroll
        for (int u = 0; u < CP; u++) a0[u] = a1[u] = 0.0;
        const double *B0 = Bs + r0 + (v0 ? i0 : 0), *B1 = Bs + r0 + (v1 ? i1 : 0);
#pragma unroll 2
        for (int a = 0; a < m; a++) {
            const double b0 = v0 ? __ldg(B0 + (int64_t)a * n) : 0.0;
            const double b1 = v1 ? __ldg(B1 + (int64_t)a * n) : 0.0;
            const double2 *tr = reinterpret_cast<const double2 *>(Tp + a * CP);
#pragma unroll
            for (int u2 = 0; u2 < CP / 2; u2++) {
                if (2 * u2 < c) {
                    const double2 t = tr[u2];
                    a0[2 * u2] = fma(b0, t.x, a0[2 * u2]);
                    a0[2 * u2 + 1] = fma(b0, t.y, a0[2 * u2 + 1]);
                    a1[2 * u2] = fma(b1, t.x, a1[2 * u2]);
                    a1[2 * u2 + 1] = fma(b1, t.y, a1[2 * u2 + 1]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < CP; u++) {
            if (u < c) {
                if (v0) Vpart[i0 * cs + u] = a0[u];
                if (v1) Vpart[i1 * cs + u] = a1[u];
            }
        }
    }
}

// Z = (R - L S)/sigma^2  (k >= 1) or Z = R (no preconditioner); partial <R,Z>.
// Thread = one row x a chunk of 8 columns (blockIdx.y): L[m][row] loads are
// coalesced across the warp, S comes from shared memory (broadcast).  The
// per-column partials are reduced warp -> block in a fixed order.
__global__ void __launch_bounds__(256)
k_precond_apply(const double *__restrict__ L, int64_t n, int64_t r0, int k,
                const double *__restrict__ S, double noise_var, const double *__restrict__ R,
                int64_t nloc, int c, double *__restrict__ Z, double *__restrict__ part) {
    extern __shared__ double Ssm[];   // k x c, then 8 x 8 warp partials
    double *wp = Ssm + k * c;
    for (int e = threadIdx.x; e < k * c; e += blockDim.x) Ssm[e] = S[e];
    __syncthreads();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c0 = blockIdx.y * 8;
    const double inv = 1.0 / noise_var;
    double rz[8];
#pragma unroll
    for (int u = 0; u < 8; u++) rz[u] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = 0.0;
        if (k > 0) {
            for (int mm = 0; mm < k; mm++) {
                const double l = L[(int64_t)mm * n + r0 + i];
#pragma unroll
                for (int u = 0; u < 8; u++)
                    if (c0 + u < c) acc[u] += l * Ssm[mm * c + c0 + u];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (c0 + u < c) {
                const double r = R[i * c + c0 + u];
                const double z = k > 0 ? (r - acc[u]) * inv : r;
                Z[i * c + c0 + u] = z;
                rz[u] += r * z;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
        double v = rz[u];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) wp[warp * 8 + u] = v;
    }
    __syncthreads();
    if (tid < 8 && c0 + tid < c) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += wp[w * 8 + tid];
        part[(int64_t)blockIdx.x * c + c0 + tid] = s;
    }
}

// Initial state after R = B, Z = P^{-1} B.  red: [bb (c) | rz (c)].
__global__ void k_init_state(MbcgState *st, const double *__restrict__ bb,
                             const double *__restrict__ rz, int c) {
    const int col = threadIdx.x;
    if (col == 0) { st->j = 0; st->status = 0; st->any_active = 0; }
    __syncthreads();
    if (col < c) {
        double bn = sqrt(bb[col]);
        st->bnorm[col] = bn;
        st->rho[col] = rz[col];
        st->rho0[col] = rz[col];
        st->active[col] = bn > 0.0;
        st->iters[col] = 0;
        st->relres[col] = bn > 0.0 ? 1.0 : 0.0;
        st->alpha[col] = 0.0;
        st->beta[col] = 0.0;
        if (bn > 0.0) atomicOr(&st->any_active, 1);
    }
}

// Pass A: V = sum_s Vpart[s] + sigma^2 D ; partial <D, V>.
__global__ void k_passA(const double *__restrict__ Vpart, int splits, int cs, int64_t nloc, int c,
                        double noise_var, const double *__restrict__ D, double *__restrict__ V,
                        double *__restrict__ part) {
    const int col = threadIdx.x;
    double acc = 0.0;
    if (col < c) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < nloc;
             i += (int64_t)gridDim.x * blockDim.y) {
            double v = 0.0;
            for (int s = 0; s < splits; s++) v += Vpart[((int64_t)s * nloc + i) * cs + col];
            double dv = D[i * c + col];
            v += noise_var * dv;
            V[i * c + col] = v;
            acc += dv * v;
        }
    }
    block_reduce_cols(acc, part, c, 0);
}

// alpha = rho / <D,V> for active columns; record alpha_j; breakdown check.
__global__ void k_alpha(MbcgState *st, const double *__restrict__ dv, double *__restrict__ ahist,
                        int c) {
    const int col = threadIdx.x;
    if (col >= c) return;
    const int j = st->j;
    double a = 0.0;
    if (st->active[col]) {
        a = st->rho[col] / dv[col];
        if (!(a > 0.0) || !isfinite(a)) {
            // reading R9/R24: a residual exhausted below fp64's range (rho <= 1e-250 rho_0,
            // p far past convergence) freezes like R = 0; else indefinite operator: breakdown
            if (!(st->rho[col] <= 1e-250 * st->rho0[col])) st->status = BBMM_ERR_NUMERIC;
            a = 0.0;
            st->active[col] = 0;
        } else {
            ahist[(int64_t)j * c + col] = a;
            st->iters[col] = j + 1;
        }
    }
    st->alpha[col] = a;
}

// Pass B: U += alpha D ; R -= alpha V ; partial |R|^2.
__global__ void k_passB(const MbcgState *__restrict__ st, const double *__restrict__ D,
                        const double *__restrict__ V, int64_t nloc, int c, double *__restrict__ U,
                        double *__restrict__ R, double *__restrict__ part) {
    const int col = threadIdx.x;
    double acc = 0.0;
    if (col < c) {
        const double a = st->alpha[col];
        for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < nloc;
             i += (int64_t)gridDim.x * blockDim.y) {
            double r = R[i * c + col];
            if (a != 0.0) {
                U[i * c + col] += a * D[i * c + col];
                r -= a * V[i * c + col];
                R[i * c + col] = r;
            }
            acc += r * r;
        }
    }
    block_reduce_cols(acc, part, c, 0);
}

// relres, freezing (relres < tol, reading R9), then S = C^{-1} W.
// red layout: [rr (c) | W (k*c)].
__global__ void k_after_B(MbcgState *st, const double *__restrict__ red, const double *cholC,
                          int k, int c, double tol, double *__restrict__ S,
                          double *__restrict__ rhist) {
    const int col = threadIdx.x;
    if (col < c && st->active[col]) {
        double rel = sqrt(red[col]) / st->bnorm[col];
        st->relres[col] = rel;
        rhist[(int64_t)st->j * c + col] = rel;          // relres after iteration j (row f3)
        if (rel < tol) st->active[col] = 0;
    }
    if (k > 0) chol_solve_warps(cholC, k, red + c, S, c);
}

// S = C^{-1} W at initialisation (red = W).
__global__ void k_solve_S(const double *__restrict__ W, const double *cholC, int k, int c,
                          double *__restrict__ S) {
    if (k > 0) chol_solve_warps(cholC, k, W, S, c);
}

// beta = rho'/rho ; record beta_j ; rho = rho' ; exact convergence freezes.
__global__ void k_beta(MbcgState *st, const double *__restrict__ rz, double *__restrict__ bhist,
                       int c) {
    const int col = threadIdx.x;
    __shared__ int any;
    if (col == 0) any = 0;
    __syncthreads();
    if (col < c) {
        const int j = st->j;
        double b = 0.0;
        if (st->active[col]) {
            double r = rz[col];
            if (r == 0.0) {
                st->active[col] = 0;   // R = 0 exactly
            } else {
                b = r / st->rho[col];
                st->rho[col] = r;
                bhist[(int64_t)j * c + col] = b;
            }
        }
        st->beta[col] = b;
        if (st->active[col]) atomicOr(&any, 1);
    }
    __syncthreads();
    if (col == 0) st->any_active = any;
}

// Pass D: D = Z + beta D (active), 0 (frozen); the matmul copy Dm of the local
// rows (fp64 or fp32, stride cs, at global row positions r0..); block 0
// advances the iteration counter.
template <typename DT>
__global__ void k_passD(MbcgState *st, const double *__restrict__ Z, int64_t nloc, int c,
                        int64_t r0, int cs, double *__restrict__ D, DT *__restrict__ Dm,
                        int advance) {
    const int col = threadIdx.x;
    if (col < cs) {
        const bool act = col < c && st->active[col];
        const double b = col < c ? st->beta[col] : 0.0;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < nloc;
             i += (int64_t)gridDim.x * blockDim.y) {
            double dn = 0.0;
            if (act) dn = Z[i * c + col] + b * D[i * c + col];
            if (col < c) D[i * c + col] = dn;
            Dm[(r0 + i) * cs + col] = (DT)dn;
        }
    }
    if (advance && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) {
        // j is only read by kernels that follow in stream order
        st->j += 1;
    }
}

__global__ void k_copy(const double *__restrict__ a, double *__restrict__ b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

__global__ void k_copy_U(const double *__restrict__ U, int64_t nloc, int c, double *__restrict__ out,
                         int64_t ldo) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * c;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / c;
        out[i * ldo + (e - i * c)] = U[e];
    }
}

// ------------------------------------------------- preconditioner setup
// C = sigma^2 I + L^T L (k x k).  Register-tiled L^T L over a row range (split-K): block b
// sums rows [i_beg, i_end) of its share; thread (ta, tb) of a 16 x 16 grid owns C[a][b] for
// a = ta + 16 p, b = tb + 16 q (p, q < KPT), accumulated in registers; L tiles (KT rows x k,
// transposed) in shared memory.
template <int KPT>
__global__ void __launch_bounds__(256)
k_LtL2(const double *__restrict__ L, int64_t n, int64_t r0, int64_t nrows, int k,
       int64_t rows_per_blk, double *__restrict__ part) {
    constexpr int KT = 16;
    extern __shared__ double Lt[];            // KT x k
    const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
    double acc[KPT][KPT];
#pragma unroll
    for (int p = 0; p < KPT; p++)
#pragma unroll
        for (int q = 0; q < KPT; q++) acc[p][q] = 0.0;
    const int64_t i_beg = (int64_t)blockIdx.x * rows_per_blk;
    const int64_t i_end = min(nrows, i_beg + rows_per_blk);
    for (int64_t i0 = i_beg; i0 < i_end; i0 += KT) {
        const int rows = (int)min((int64_t)KT, i_end - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < k * KT; e += 256) {
            const int m = e / KT, kk = e - m * KT;
            Lt[kk * k + m] = kk < rows ? L[(int64_t)m * n + r0 + i0 + kk] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < KT; kk++) {
            double va[KPT], vb[KPT];
#pragma unroll
            for (int p = 0; p < KPT; p++) {
                const int a = ta + 16 * p, b = tb + 16 * p;
                va[p] = a < k ? Lt[kk * k + a] : 0.0;
                vb[p] = b < k ? Lt[kk * k + b] : 0.0;
            }
#pragma unroll
            for (int p = 0; p < KPT; p++)
#pragma unroll
                for (int q = 0; q < KPT; q++) acc[p][q] = fma(va[p], vb[q], acc[p][q]);
        }
    }
#pragma unroll
    for (int p = 0; p < KPT; p++)
#pragma unroll
        for (int q = 0; q < KPT; q++) {
            const int a = ta + 16 * p, b = tb + 16 * q;
            if (a < k && b < k) part[(int64_t)blockIdx.x * k * k + a * k + b] = acc[p][q];
        }
}

// In-place Cholesky of C (k x k, lower) + log|P| = log|C| + (n-k) log sigma^2.
__global__ void k_chol_small(double *C, const double *__restrict__ red, int k, double noise_var,
                             int64_t n, double *logdet, int *status) {
    // single thread: k <= 128, O(k^3/3) = 0.7 MFLOP
    if (threadIdx.x != 0) return;
    for (int a = 0; a < k; a++)
        for (int b = 0; b <= a; b++) {
            double v = red[a * k + b] + (a == b ? noise_var : 0.0);
            C[a * k + b] = v;
            C[b * k + a] = v;
        }
    for (int jj = 0; jj < k; jj++) {
        double s = C[jj * k + jj];
        for (int m = 0; m < jj; m++) s -= C[jj * k + m] * C[jj * k + m];
        if (!(s > 0.0)) { *status = BBMM_ERR_NUMERIC; return; }
        double l = sqrt(s);
        C[jj * k + jj] = l;
        for (int i = jj + 1; i < k; i++) {
            double t = C[i * k + jj];
            for (int m = 0; m < jj; m++) t -= C[i * k + m] * C[jj * k + m];
            C[i * k + jj] = t / l;
        }
        for (int i = 0; i < jj; i++) C[i * k + jj] = 0.0;
    }
    double ld = 0.0;
    for (int a = 0; a < k; a++) ld += 2.0 * log(C[a * k + a]);
    *logdet = ld + (double)(n - k) * log(noise_var);
}

// ------------------------------------------------------------ probes
// Counter-based splitmix64 Rademacher signs.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double rsign(uint64_t seed, int64_t n, int kgen, int col, int64_t row) {
    uint64_t ctr = (uint64_t)col * (uint64_t)(n + kgen) + (uint64_t)row + 1ULL;
    return (mix64(seed + ctr * 0x9E3779B97F4A7C15ULL) >> 63) ? -1.0 : 1.0;
}

// B[i][0] = y_{r0+i} ; B[i][1+col] = sum_m L[m][r0+i] eps1[m][col] + sig eps2[r0+i][col]
__global__ void k_probes(const int8_t *__restrict__ eps, uint64_t seed, int64_t n, int kgen, int t,
                         const double *__restrict__ L, int k_used, double sig, int64_t r0,
                         int64_t nloc, const float *__restrict__ y, double *__restrict__ B) {
    const int c = t + 1;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * c;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / c;
        int col = (int)(e - i * c);
        int64_t gi = r0 + i;
        double v;
        if (col == 0) {
            v = (double)y[gi];
        } else {
            int pc = col - 1;
            double acc = 0.0;
            for (int m = 0; m < k_used; m++) {
                double e1 = eps ? (double)eps[(n + m) * t + pc] : rsign(seed, n, kgen, pc, n + m);
                acc += L[(int64_t)m * n + gi] * e1;
            }
            double e2 = eps ? (double)eps[gi * t + pc] : rsign(seed, n, kgen, pc, gi);
            v = acc + sig * e2;
        }
        B[e] = v;
    }
}

}  // namespace

// ======================================================================
// host side
// ======================================================================
void reduce_blocks(bbmm_ctx_s *ctx, const double *part, int nblk, int m, double *red) {
    k_reduce_blocks<<<reduce_grid(m), 256, 0, ctx->stream>>>(part, nblk, m, red);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

void precond_setup(bbmm_ctx_s *ctx, const double *L, int64_t n, int k, double noise_var,
                   double *cholC, double *logdet_d) {
    int *status = (int *)ctx->ws.get("pc_status", sizeof(int));
    BBMM_CUDA(cudaMemsetAsync(status, 0, sizeof(int), ctx->stream));
    if (k == 0) {
        BBMM_CUDA(cudaMemsetAsync(logdet_d, 0, sizeof(double), ctx->stream));
        return;
    }
    // L^T L over this rank's rows (register-tiled split-K), then an all-reduce of the k x k sum
    const RowRange rr = local_rows(ctx, n);
    const int64_t nl = rr.count();
    int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(2 * kNumSMs, ceil_div(std::max<int64_t>(nl, 1), 512)));
    double *part = (double *)ctx->ws.get("pc_part", sizeof(double) * nblk * k * k);
    double *red = (double *)ctx->ws.get("pc_red", sizeof(double) * k * k);
    const int kpt = (k + 15) / 16;
    const int64_t rpb = ceil_div(ceil_div(std::max<int64_t>(nl, 1), nblk), 16) * 16;
    const size_t smem = (size_t)16 * k * 8;
    if (nl > 0) {
        auto f = kpt <= 2 ? k_LtL2<2> : kpt <= 4 ? k_LtL2<4> : kpt <= 6 ? k_LtL2<6> : k_LtL2<8>;
        f<<<nblk, 256, smem, ctx->stream>>>(L, n, rr.r0, nl, k, rpb, part);
        k_reduce_blocks<<<reduce_grid(k * k), 256, 0, ctx->stream>>>(part, nblk, k * k, red);
    } else {
        BBMM_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * k * k, ctx->stream));
    }
    allreduce_sum(ctx, red, (size_t)k * k);
    k_chol_small<<<1, 32, 0, ctx->stream>>>(cholC, red, k, noise_var, n, logdet_d, status);
    BBMM_LAUNCH_CHECK();
    ctx->launches += 3;
    int st_h = 0;
    BBMM_CUDA(cudaMemcpyAsync(&st_h, status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    if (st_h != 0) throw Error{BBMM_ERR_NUMERIC, "Cholesky of C = sigma^2 I + L^T L failed"};
}

void make_probes(bbmm_ctx_s *ctx, const int8_t *eps, uint64_t seed, int64_t n, int kgen, int t,
                 const double *L, int k_used, double sigma, int64_t r0, int64_t nloc,
                 const float *y, double *B, int c) {
    (void)c;
    int64_t total = nloc * (t + 1);
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 8 * kNumSMs));
    k_probes<<<grid, 256, 0, ctx->stream>>>(eps, seed, n, kgen, t, L, k_used, sigma, r0, nloc, y,
                                            B);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

void comm_events_reserve(bbmm_ctx_s *ctx, size_t n) {
    while (ctx->comm_events.size() < n) {
        cudaEvent_t e;
        BBMM_CUDA(cudaEventCreate(&e));
        ctx->comm_events.push_back(e);
    }
}

cudaEvent_t mm_event(bbmm_ctx_s *ctx, size_t i) {
    while (ctx->mm_events.size() <= i) {
        cudaEvent_t e;
        BBMM_CUDA(cudaEventCreate(&e));
        ctx->mm_events.push_back(e);
    }
    return ctx->mm_events[i];
}

void mbcg_run(bbmm_ctx_s *ctx, const MbcgArgs &a, const double *B, int64_t ldb,
              const double *cholC, MbcgOut &out) {
    const int c = a.c, k = a.k;
    const int cp = pad_cols(c);
    BBMM_REQUIRE(cp > 0, "too many columns");
    const int cs = (cp + 3) & ~3;
    const int64_t nloc = a.nloc;
    const size_t nc = (size_t)std::max<int64_t>(nloc, 1) * c;
    Workspace &ws = ctx->ws;
    cudaStream_t sm = ctx->stream;

    double *U = (double *)ws.get("cg_U", nc * 8);
    double *R = (double *)ws.get("cg_R", nc * 8);
    double *Z = (double *)ws.get("cg_Z", nc * 8);
    double *D = (double *)ws.get("cg_D", nc * 8);
    double *V = (double *)ws.get("cg_V", nc * 8);
    const int64_t npad = a.nb * ctx->nranks;
    const bool acc64 = ctx->matmul_acc64;
    const size_t esz = acc64 ? 8 : 4;
    void *Dm = ws.get("cg_Dm", (size_t)npad * cs * esz);
    const bool use_sor = a.sor_B != nullptr;
    const bool use_tc = a.tc.version != 0 && !use_sor;
    size_t vcap = use_sor ? (size_t)std::max<int64_t>(nloc, 1) * cs
                 : use_tc ? tc_vpart_elems(a.tc, a.n, nloc, a.tc.cb) : vpart_elems(a.n, nloc, cp, a.Kst != nullptr);
    const int64_t npad_tc = use_tc ? k1tc_pad_rows(npad) : 0;
    const int tc_nd = use_tc ? tc_dslices(a.tc) : 4;
    const int cb = use_tc ? a.tc.cb : c;              // columns of the tensor-core instantiation
    const int tc_rows = tc_bslice_rows(cb, tc_nd);
    const int vs = use_tc ? tc_vstride(a.tc) : cs;    // Vpart row stride
    BBMM_REQUIRE(!use_tc || a.tc.npad == npad_tc, "tc operand rows");
    uint8_t *Bp = use_tc ? (uint8_t *)ws.get("tc_B", tc_bp_bytes(a.tc)) : nullptr;
    double *Stc = use_tc ? (double *)ws.get("tc_S", kMaxCols * 8) : nullptr;
    if (use_tc) BBMM_CUDA(cudaMemsetAsync(Bp, 0, tc_bp_bytes(a.tc), sm));
    double *Vpart = (double *)ws.get("cg_Vpart", std::max<size_t>(vcap, 1) * 8);
    const PassGeom g = pass_geom(nloc, c);
    const int nblk = (int)g.grid.x;
    const int kk = std::max(k, 1);
    double *part = (double *)ws.get("cg_part", (size_t)nblk * (size_t)(kk + 1) * c * 8);
    double *red = (double *)ws.get("cg_red", (size_t)(kk + 2) * c * 8);
    double *S = (double *)ws.get("cg_S", (size_t)kk * c * 8);
    MbcgState *st = (MbcgState *)ws.get("cg_state", sizeof(MbcgState));
    double *ahist = (double *)ws.get("cg_ahist", (size_t)a.max_iter * c * 8);
    double *rhist = (double *)ws.get("cg_rhist", (size_t)a.max_iter * c * 8);
    BBMM_CUDA(cudaMemsetAsync(rhist, 0, (size_t)a.max_iter * c * 8, sm));
    double *bhist = (double *)ws.get("cg_bhist", (size_t)a.max_iter * c * 8);
    BBMM_CUDA(cudaMemsetAsync(ahist, 0, (size_t)a.max_iter * c * 8, sm));
    BBMM_CUDA(cudaMemsetAsync(bhist, 0, (size_t)a.max_iter * c * 8, sm));
    BBMM_CUDA(cudaMemsetAsync(Dm, 0, (size_t)npad * cs * esz, sm));
    const size_t smem_S = (size_t)kk * c * 8 + 64 * 8;
    if (smem_S > 48 * 1024)
        BBMM_CUDA(cudaFuncSetAttribute(k_precond_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_S));
    const bool multi = has_comm(ctx);
    int launches = 0;

    auto reduce = [&](int m, double *dst) {
        k_reduce_blocks<<<reduce_grid(m), 256, 0, sm>>>(part, nblk, m, dst);
        launches++;
    };
    // W = L^T R (+ |R|^2 already in red[0..c) when with_rr) -> red[c..c+kc)
    // >= one block per 64 rows so that small problems are not latency-bound on a few blocks
    const int ltr_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 64),
                                                                        2 * kNumSMs));
    const size_t smem_ltr = ((size_t)kLtrRows * c + (size_t)kk * c) * 8;
    auto ltr_kernel = c <= 8 ? k_LtR<8> : (c <= 17 ? k_LtR<17> : (c <= 33 ? k_LtR<33> : k_LtR<kMaxCols>));
    if (smem_ltr > 48 * 1024)
        BBMM_CUDA(cudaFuncSetAttribute(ltr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_ltr));
    double *part_ltr = (double *)ws.get("cg_part_ltr", (size_t)ltr_blocks * kk * c * 8);
    // part_out[blk][K x c] = Lp[:, rows of blk]^T R: the register-tiled split-K kernel when
    // its per-thread tile fits (c <= 20, <= 16 rows of Lp per thread), else k_LtR
    auto launch_ltr = [&](const double *Lp, int K, const double *Rp, double *part_out,
                          size_t smem_fallback) {
        const int CGN = (c + 3) / 4, MLN = 256 / CGN;
        const int need = (K + MLN - 1) / MLN;
        // tall L (the SoR operator's Bs): the cp.async-pipelined variant
        static const bool no_ltr3 = std::getenv("BBMM_NO_LTR3") != nullptr;
        if (!no_ltr3 && K >= 128 && c <= 20 && need <= 16 && a.n % 2 == 0 && a.r0 % 2 == 0 &&
            ltr3_smem(K, c) <= 200 * 1024) {
            const int64_t rpb = ceil_div(ceil_div(std::max<int64_t>(nloc, 1), ltr_blocks), kL3T) * kL3T;
            static DeviceOnce attr3;
            attr3(ctx->device, [] {
                for (auto f : {k_LtR3<4>, k_LtR3<8>, k_LtR3<12>, k_LtR3<16>})
                    BBMM_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   200 * 1024));
            });
            // (512-thread blocks with half the rows per thread measured slower: 1.40 vs 1.15 ms)
            auto f = need <= 4 ? k_LtR3<4> : need <= 8 ? k_LtR3<8> : need <= 12 ? k_LtR3<12>
                                                                               : k_LtR3<16>;
            f<<<ltr_blocks, 256, ltr3_smem(K, c), sm>>>(Lp, a.n, a.r0, K, Rp, nloc, c, rpb, part_out);
            return;
        }
        if (c <= 20 && need <= 16) {
            const int KT = K <= 256 ? 32 : 16;
            const int64_t rpb = ceil_div(ceil_div(std::max<int64_t>(nloc, 1), ltr_blocks), KT) * KT;
            const size_t smem2 = ((size_t)KT * K + (size_t)KT * c) * 8;
            static DeviceOnce attr2;
            attr2(ctx->device, [] {
                for (auto f : {k_LtR2<1>, k_LtR2<2>, k_LtR2<4>, k_LtR2<8>, k_LtR2<12>, k_LtR2<16>})
                    BBMM_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   100 * 1024));
            });
            auto f = need <= 1 ? k_LtR2<1> : need <= 2 ? k_LtR2<2> : need <= 4 ? k_LtR2<4>
                   : need <= 8 ? k_LtR2<8> : need <= 12 ? k_LtR2<12> : k_LtR2<16>;
            f<<<ltr_blocks, 256, smem2, sm>>>(Lp, a.n, a.r0, K, Rp, nloc, c, rpb, KT, part_out);
        } else {
            ltr_kernel<<<ltr_blocks, 256, smem_fallback, sm>>>(Lp, a.n, a.r0, K, Rp, nloc, c, part_out);
        }
    };
    auto LtR = [&](double *dst) {
        if (k == 0) return;
        launch_ltr(a.L, k, R, part_ltr, smem_ltr);
        k_reduce_blocks<<<reduce_grid(k * c), 256, 0, sm>>>(part_ltr, ltr_blocks, k * c, dst);
        launches += 2;
    };
    // SoR operator (row f4): T = Bs[:, local] D (the L^T R kernel with L = Bs), all-reduced,
    // then Vpart = Bs[:, local]^T T; splits = 1
    const int msor = use_sor ? a.sor_m : 1;
    auto sor_expand = c <= 8 ? k_sor_expand<8> : (c <= 17 ? k_sor_expand<17>
                    : (c <= 33 ? k_sor_expand<33> : k_sor_expand<kMaxCols>));
    const size_t smem_sor = ((size_t)kLtrRows * c + (size_t)msor * c) * 8;
    double *part_sor = use_sor ? (double *)ws.get("cg_part_sor", (size_t)ltr_blocks * msor * c * 8)
                               : nullptr;
    double *Tsor = use_sor ? (double *)ws.get("cg_Tsor", (size_t)msor * c * 8) : nullptr;
    if (use_sor) {
        if (smem_sor > 48 * 1024)
            BBMM_CUDA(cudaFuncSetAttribute(ltr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)std::max(smem_sor, smem_ltr)));
        if ((size_t)msor * c * 8 > 48 * 1024)
            BBMM_CUDA(cudaFuncSetAttribute(sor_expand, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)((size_t)msor * c * 8)));
    }
    auto sor_matmul = [&](cudaEvent_t e0, cudaEvent_t e1) {
        if (e0) record_event(ctx, e0);
        if (nloc > 0) {
            launch_ltr(a.sor_B, msor, D, part_sor, smem_sor);
            k_reduce_blocks<<<reduce_grid(msor * c), 256, 0, sm>>>(part_sor, ltr_blocks, msor * c,
                                                                    Tsor);
            launches += 2;
        } else {
            BBMM_CUDA(cudaMemsetAsync(Tsor, 0, (size_t)msor * c * 8, sm));
        }
        if (multi) allreduce_sum(ctx, Tsor, (size_t)msor * c);
        if (nloc > 0) {
            static const bool no_sor2 = std::getenv("BBMM_NO_SOR2") != nullptr;
            const size_t sm2 = (size_t)msor * (c <= 8 ? 8 : 18) * 8;   // m x CP of the instantiation
            if (!no_sor2 && c <= 17 && sm2 <= 48 * 1024) {
                const int eg = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 512), 4 * kNumSMs));
                if (c <= 8)
                    k_sor_expand2<8><<<eg, 256, sm2, sm>>>(a.sor_B, a.n, a.r0, msor, Tsor, nloc, c, cs, Vpart);
                else
                    k_sor_expand2<17><<<eg, 256, sm2, sm>>>(a.sor_B, a.n, a.r0, msor, Tsor, nloc, c, cs, Vpart);
            } else {
                const int eg = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 256), 4 * kNumSMs));
                sor_expand<<<eg, 256, (size_t)msor * c * 8, sm>>>(a.sor_B, a.n, a.r0, msor, Tsor, nloc, c,
                                                                 cs, Vpart);
            }
            launches++;
        }
        if (e1) record_event(ctx, e1);
        return 1;
    };
    // precondition apply: grid (row blocks, column chunks of 8); partials nblk x c
    const dim3 pa_grid((unsigned)nblk, (unsigned)ceil_div(c, 8));
    auto precond_apply = [&](double *dst) {
        k_precond_apply<<<pa_grid, 256, smem_S, sm>>>(a.L, a.n, a.r0, k, S, a.noise_var, R, nloc,
                                                      c, Z, part);
        reduce(c, dst);
        launches++;
    };
    // ---------------- initialisation: R = B, Z = P^{-1} R, D = Z
    k_init_vectors<<<g.grid, g.block, 0, sm>>>(B, ldb, nloc, c, U, R, D, part);
    launches++;
    reduce(c, red);                           // red[0..c) = |B|^2
    LtR(red + c);                             // red[c..c+kc) = L^T B
    if (multi) allreduce_sum(ctx, red, (size_t)(k + 1) * c);
    if (k > 0) {
        k_solve_S<<<1, kSolveThreads, (size_t)(kSolveThreads / 32) * k * 8, sm>>>(red + c, cholC,
                                                                                k, c, S);
        launches++;
    }
    double *red_rz = red + (size_t)(kk + 1) * c;
    precond_apply(red_rz);
    if (multi) allreduce_sum(ctx, red_rz, c);
    k_init_state<<<1, 64, 0, sm>>>(st, red, red_rz, c);
    launches++;
    if (out.Z0) {
        k_copy<<<256, 256, 0, sm>>>(Z, out.Z0, (int64_t)nc);
        launches++;
    }
    auto passD = [&](int advance) {
        dim3 blk(cs <= 32 ? 32 : 64, g.rb);
        if (acc64)
            k_passD<double><<<g.grid, blk, 0, sm>>>(st, Z, nloc, c, a.r0, cs, D, (double *)Dm,
                                                    advance);
        else
            k_passD<float><<<g.grid, blk, 0, sm>>>(st, Z, nloc, c, a.r0, cs, D, (float *)Dm,
                                                   advance);
        launches++;
        if (use_tc) {
            // tensor-core operand: global column scales, then int8 slices
            k1tc_colmax(ctx, D, c, nloc, c, Stc);
            if (multi) allreduce_max(ctx, Stc, c);
            if (nloc > 0) tc_pack(ctx, a.tc, D, c, a.r0, nloc, a.n, c, Stc, Bp);
            if (multi)      // each column chunk's operand holds the ranks' row blocks in order
                for (int z = 0; z < a.tc.nch; z++)
                    allgather_rows(ctx, Bp + (size_t)z * npad_tc * tc_rows, (size_t)a.nb * tc_rows);
        } else if (multi && !use_sor) {          // SoR needs only local rows of D
            allgather_rows(ctx, Dm, (size_t)a.nb * cs * esz);
        }
    };
    passD(0);
    BBMM_LAUNCH_CHECK();

    // fused vector work (one cooperative kernel per iteration) where it applies
    bool fused = mbcg_fused_applicable(ctx, c, k, use_sor, nloc) && (!use_tc || a.tc.nch == 1);
    FusedPlan fplan;
    double *Cinv = nullptr, *fpart = nullptr, *fpartW = nullptr, *fred = nullptr;
    if (fused) {
        Cinv = (double *)ws.get("cg_Cinv", (size_t)kk * kk * 8);
        fplan = mbcg_fused_plan(ctx, nloc, c, k, cholC, Cinv);
        fused = fplan.ok;
        if (fused) {
            fpart = (double *)ws.get("cg_fpart", (size_t)4 * fplan.G * c * 8);
            fpartW = (double *)ws.get("cg_fpartW", (size_t)fplan.G * kk * c * 8);
            fred = (double *)ws.get("cg_fred", (size_t)(kk + 1) * c * 8);
        }
    }

    // ---------------- iterations
    // pinned flag for convergence polling, allocated once per context and only when needed
    // (cudaMallocHost costs tens of ms; with tol == 0 nothing is polled)
    if (a.tol > 0.0 && !ctx->pinned_flag) BBMM_CUDA(cudaMallocHost(&ctx->pinned_flag, sizeof(int)));
    int *any_h = ctx->pinned_flag;
    int iters_run = 0;
    // one mBCG iteration (Alg. S2 body); false = stop (every column converged, tol > 0)
    auto iterate = [&](int j) -> bool {
        cudaEvent_t e0 = mm_event(ctx, 2 * (size_t)j), e1 = mm_event(ctx, 2 * (size_t)j + 1);
        int splits;
        if (use_sor)
            splits = sor_matmul(e0, e1);
        else if (use_tc)
            splits = tc_matmul(ctx, a.tc, Bp, Stc, cb, a.n, a.r0, nloc, a.s, Vpart, vcap, e0, e1);
        else if (a.Kst)
            splits = kernel_matmul_stored(ctx, a.Kst, a.n, nloc, Dm, acc64, cp, Vpart, vcap, e0,
                                          e1);
        else
            splits = kernel_matmul_onthefly(ctx, a.kind, a.Xs, a.dp, a.n, a.r0, nloc, Dm, acc64,
                                            cp, a.s, Vpart, vcap, e0, e1);
        if (fused) {
            FusedIo io{st, Vpart, splits, vs, c, k, nloc, a.n, a.noise_var, a.tol, D, V, U, R, Z,
                       a.L, Cinv, ahist, bhist, rhist, fpart, fpartW, fred, Dm, acc64 ? 0 : 1,
                       use_tc ? Bp : nullptr, tc_nd, tc_rows, Stc,
                       use_tc ? k1tc_pad_rows(a.n) : 0, cb};
            mbcg_fused_iteration(ctx, fplan, io);
        } else {
            k_passA<<<g.grid, g.block, 0, sm>>>(Vpart, splits, vs, nloc, c, a.noise_var, D, V, part);
            reduce(c, red);
            if (multi) allreduce_sum(ctx, red, c);
            k_alpha<<<1, 64, 0, sm>>>(st, red, ahist, c);
            k_passB<<<g.grid, g.block, 0, sm>>>(st, D, V, nloc, c, U, R, part);
            reduce(c, red);
            LtR(red + c);
            if (multi) allreduce_sum(ctx, red, (size_t)(k + 1) * c);
            k_after_B<<<1, kSolveThreads, (size_t)(kSolveThreads / 32) * std::max(k, 1) * 8, sm>>>(
                st, red, cholC, k, c, a.tol, S, rhist);
            // rho' = <R, Z> reduced directly.  (The Woodbury identity
            // (|R|^2 - W^T C^-1 W) / sigma^2 would spare this all-reduce but cancels
            // catastrophically once R reaches rounding level -- measured: alpha <= 0
            // breakdowns at n = 300, k = 100 on 4 ranks.)
            precond_apply(red_rz);
            if (multi) allreduce_sum(ctx, red_rz, c);
            k_beta<<<1, 64, 0, sm>>>(st, red_rz, bhist, c);
            launches += 7;
            passD(1);
        }
        BBMM_LAUNCH_CHECK();
        iters_run = j + 1;
        if (a.tol > 0.0) {
            BBMM_CUDA(cudaMemcpyAsync(any_h, &st->any_active, sizeof(int), cudaMemcpyDeviceToHost,
                                      sm));
            BBMM_CUDA(cudaStreamSynchronize(sm));
            if (!*any_h) return false;
        }
        return true;
    };
    // With tol == 0 the iteration count is fixed, so the per-step path (large n, multi-rank over
    // NCCL) captures iterations 1..p-1 -- kernels, collectives and the timing events -- into ONE
    // CUDA graph and launches it once: no per-kernel launch gaps between the ~12 kernels and
    // 4 collectives of an iteration.  Iteration 0 runs eagerly (first-use workspace and kernel
    // attributes are set up outside the capture).  The in-process rank group is host-staged and
    // cannot be captured; BBMM_NO_GRAPH=1 turns the capture off (A/B tests).
    const bool graph = !fused && a.tol == 0.0 && !ctx->local && a.max_iter >= 2 &&
                       !std::getenv("BBMM_NO_GRAPH");
    if (ctx->graph_exec) {            // the previous call's graph (that call has synchronised)
        cudaGraphExecDestroy(ctx->graph_exec);
        ctx->graph_exec = nullptr;
    }
    if (graph) {
        iterate(0);
        mm_event(ctx, 2 * (size_t)a.max_iter - 1);            // create the events outside the capture
        comm_events_reserve(ctx, ctx->n_comm_ev + 8 * (size_t)a.max_iter + 8);
        BBMM_CUDA(cudaStreamBeginCapture(sm, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        cudaGraph_t gr = nullptr;
        try {
            for (int j = 1; j < a.max_iter; j++) iterate(j);
        } catch (...) {
            ctx->capturing = false;
            if (cudaStreamEndCapture(sm, &gr) == cudaSuccess && gr) cudaGraphDestroy(gr);
            throw;
        }
        ctx->capturing = false;
        BBMM_CUDA(cudaStreamEndCapture(sm, &gr));
        const cudaError_t ie = cudaGraphInstantiate(&ctx->graph_exec, gr, 0);
        cudaGraphDestroy(gr);
        BBMM_CUDA(ie);
        BBMM_CUDA(cudaGraphLaunch(ctx->graph_exec, sm));
    } else {
        for (int j = 0; j < a.max_iter; j++)
            if (!iterate(j)) break;
    }
    // ---------------- outputs
    if (out.U) {
        k_copy_U<<<256, 256, 0, sm>>>(U, nloc, c, out.U, out.ldu);
        launches++;
    }
    out.matmul_launches = iters_run;
    out.iters_run = iters_run;
    out.U_d = U;
    out.R_d = R;
    out.ahist_d = ahist;
    out.bhist_d = bhist;
    out.state_d = st;
    out.rhist_d_ = rhist;
    out.c_ = c;
    out.max_iter_ = a.max_iter;
    out.n_ev_ = 2 * iters_run;
    ctx->launches += launches;   // matmul launches are counted by the matmul functions
    // host-side results: now, or (defer_host) by the caller's mbcg_finish after its own
    // stream synchronisation -- a latency-bound call then pays one host round trip less
    if (!out.defer_host) mbcg_finish(ctx, out);
}

void mbcg_finish(bbmm_ctx_s *ctx, MbcgOut &out) {
    cudaStream_t sm = ctx->stream;
    const int c = out.c_, p = out.max_iter_;
    MbcgState st_h;
    out.alpha.assign((size_t)p * c, 0.0);
    out.beta.assign((size_t)p * c, 0.0);
    out.relres_hist.assign((size_t)p * c, 0.0);
    BBMM_CUDA(cudaMemcpyAsync(out.relres_hist.data(), out.rhist_d_, (size_t)p * c * 8,
                              cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaMemcpyAsync(out.alpha.data(), out.ahist_d, (size_t)p * c * 8,
                              cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaMemcpyAsync(out.beta.data(), out.bhist_d, (size_t)p * c * 8,
                              cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaMemcpyAsync(&st_h, out.state_d, sizeof(MbcgState), cudaMemcpyDeviceToHost, sm));
    BBMM_CUDA(cudaStreamSynchronize(sm));
    BBMM_LAUNCH_CHECK();
    float ms_tot = 0.f;
    for (int q = 0; q + 1 < out.n_ev_; q += 2) {
        float ms = 0.f;
        BBMM_CUDA(cudaEventElapsedTime(&ms, ctx->mm_events[q], ctx->mm_events[q + 1]));
        ms_tot += ms;
    }
    out.n_ev_ = 0;
    out.ms_matmul = ms_tot;
    out.iters.assign(st_h.iters, st_h.iters + c);
    out.relres.assign(st_h.relres, st_h.relres + c);
    out.rho0.assign(st_h.rho0, st_h.rho0 + c);
    if (st_h.status != 0)
        throw Error{BBMM_ERR_NUMERIC,
                    "mBCG breakdown: alpha <= 0 or non-finite (operator not positive definite)"};
}

}  // namespace bbmm
