// k1tc2.cu -- Blackwell tensor-core kernel-matmul (K1-TC): V = s K~ D on the fly.
//
// The exact int8 contraction of DESIGN.md §6: kernel values k~ in [0, 1] as
// 23-bit fixed point in three u8 slices (the low bytes of the fp32 q = 2 + 2 k~),
// D as 31-bit (RBF) or 39-bit (Matern) fixed point per column (k1tc.cu), all
// slice products on the int8 tensor cores with exact integer accumulation in
// TMEM, drained to fp64.  Per 128 x 128 tile:
//   * RBF (MODE 0 / 1 / 3): the exponent S_ij = -|xs_i - xs_j|^2 is itself a
//     tcgen05 MMA (3-product hi/lo split in fp16 with operands scaled by 2^5:
//     at d <= 6 the three products packed along K into two kind::f16 MMAs,
//     above that kind::f16 per product -- half the MMAs of kind::tf32) of augmented vectors
//       A_i = [2 xs_i, -|xs_i|^2, 1] (shared memory),  B_j = [xs_j, 1, -|xs_j|^2]
//     (streamed [hi | lo] tiles) into a TMEM buffer; compute warps tcgen05.ld S,
//     run ex2 on the MUFU (MODE 1: times r^2, the isotropic lengthscale
//     derivative), quantise, and tcgen05.st the A slices over their S columns;
//   * Matern-5/2 (MODE 2): distances from direct fp32 differences of x tiles
//     streamed through the same ring (two points per FADD2 / FFMA2), then
//     sqrt + ex2 on the MUFU -- the expanded form's ~1e-7 error breaks the
//     parity bars for Matern.
// The int8 MMAs read the A slices from TMEM and the packed D slices from
// shared memory.
//
// CTA = 128 rows, 1 CTA per SM, 18 warps:
//   warps 0-15: compute; warp w serves TMEM lanes 32 (w % 4).. and the j-group
//               h = w / 4 (32 of the 128 j) of every tile
//   warp 16   : producer (bulk copies of the distance / x tile and the packed
//               D slices, two rings)
//   warp 17   : MMA issuer: int8 contraction of tile t, then the distance
//               MMA of tile t + NBUF into the TMEM buffer just consumed
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cuda_fp16.h>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"
#include "sm100_ptx.cuh"

namespace bbmm {
namespace tc2 {

// j-tile BK = JW NPS (default 32 x 4 = 128); 4 NPS compute warps (NPS per SM
// sub-partition, so that one warp's barrier / TMEM latency is covered by the
// others' MUFU work), warp (sub, h) serves TMEM lanes 32 sub.. and the j-group
// h (JW j) of every tile.  Each of the NBUF TMEM buffers (BK columns) first
// receives S (fp32, from the distance MMA); every warp then overwrites 24 of
// ITS OWN 32 S columns (JW = 32) with the three int8 slices of its quantised
// kernel values, which the int8 MMAs read as A.  With three buffers the MMA
// side runs two tiles ahead of the slowest warp.
//
// JW = 16 (a timing variant) column maps inside the 32-column group ks = h / 2
// of a buffer (eo = h % 2, u, v in 0..3, j' = 16 eo + 4 u + v the point's index
// within the group):
//   S  of j'          -> column 8 u + 4 eo + v      (order of the B' rows)
//   A  slice a, 4 j'  -> column 8 a + 4 eo + u      (K order = j', natural)
// so the A columns a warp writes (u = 0..2 quarters) are among its own S
// columns, and each slice's 8 columns hold the 32 j of the group in order.
#ifndef BBMM_TC2_NPS
#define BBMM_TC2_NPS 4
#endif
#ifndef BBMM_TC2_JW
#define BBMM_TC2_JW 32
#endif
#ifndef BBMM_TC2_F16DIST
#define BBMM_TC2_F16DIST 1
#endif
#ifndef BBMM_TC2_F16_MIN_DA
#define BBMM_TC2_F16_MIN_DA 16
#endif
// DA = 8 (d <= 6): the three hi/lo products packed along K into ONE fp16 operand pair,
// A' = [hi | hi | lo | 0], B' = [hi | lo | hi | 0] (K = 32 halves): 2 kind::f16 MMAs per tile
// instead of 3 kind::tf32 (same 11 + 11-bit split; a third less tensor time and TMEM
// accumulator traffic for the distance)
#ifndef BBMM_TC2_F16PACK
#define BBMM_TC2_F16PACK 1
#endif
// Trim the int8 MMAs of the low k~ slices to the products that carry weight (ND = 4):
// 0 = all twelve slice products; 1 (default) = q0 x [p3 p2 p1] (drops q0 p0: weight 2^0 of the
// 2^54 product scale, < 2^-38 relative -- 64x below the rounding of the 31-bit D itself);
// 2 = also q1 x [p3 p2 p1], q0 x [p3 p2] (drops the weight-2^8 products q1 p0, q0 p1: ~2^-29,
// i.e. above D's rounding -- timing experiments only).  The MMA N is rounded up to 16, so a few
// dropped-block columns are still added -- at their correct weight (the blocks are
// weight-ordered), never elsewhere.  Measured (B200): C4 289.0 -> 288.5 ms, C3 16.29 -> 15.93 ms.
// timing ablations of MODE 3 (results wrong by construction): 1 = no residual MMA,
// 2 = no residual TMEM stores, 3 = no residual arithmetic (zero slice)
#ifndef BBMM_TC2_ABL
#define BBMM_TC2_ABL 0
#endif
// S loaded in two tcgen05.ld.x16 halves, the second issued after the first half's quantisation
// (a shorter TMEM load occupying the warp's MIO queue, where its MUFU ops also queue; measured:
// MODE 3 339.6 -> 335.7 ms alone, but 336.9 with the store burst; MODE 0 +0.3 %) -- off
#ifndef BBMM_TC2_SPLITLD
#define BBMM_TC2_SPLITLD 0
#endif
// MODE 3: all A-slice stores of a tile as four tcgen05.st.x8 after the second half instead of
// eight .x4 spread over the tile (measured: MODE 3 339.6 -> 332.3 ms at C4; MODE 0, whose
// three slices are stored per half, gets slower with a burst: 289.0 -> 295.8 ms)
#ifndef BBMM_TC2_STBURST
#define BBMM_TC2_STBURST 1
#endif
#ifndef BBMM_TC2_TRIM
#define BBMM_TC2_TRIM 1
#endif
// fp16 distance operands are scaled by 2^5 (|xs|^2 by 2^10) so that the lo halves of the
// split stay normal fp16 numbers down to |xs| ~ 2^-8 (the precision guard keeps |xs|^2 <= 16,
// so 2^10 |xs|^2 <= 16384 < 65504); the MMA then yields 2^10 S, rescaled before ex2
constexpr float kF16Scale = 32.0f;
constexpr int NPS = BBMM_TC2_NPS;              // compute warps per lane quarter
constexpr int JW = BBMM_TC2_JW;                // j per warp per tile (16 or 32)
constexpr int BM = 128, BK = JW * NPS;         // j tile
constexpr int NCW = 4 * NPS;
static_assert((JW == 32 || (JW == 16 && NPS % 2 == 0)) && 32 * (NCW + 2) <= 1024, "CTA shape");
// j per TMEM drain.  All slice bytes are unsigned (q2 <= 0x40, p3 <= 0x80),
// so the accumulators are read as uint32; the largest per-j block sum is
// block 3: q2 p0 + q1 p1 + q0 p2 <= 128*255 + 2*255*255 = 162690 (q2 <= 0x80: k~ = 1
// exactly), hence < 2^32 / 162690 = 26399 j per window.
constexpr int WINDOW = (int)(4294967295ull / 162690ull) / BK * BK;
static_assert((double)WINDOW * 162690.0 < 4294967296.0, "uint32 window bound");
// MODE 3 (31-bit k~ grid) adds the residual slice r <= 255 at weight 2^-8 below q0, whose
// products r p3, r p2 (and r p1 for 8 columns) join blocks 3-5: the largest per-j block sum
// becomes block 3's q2 p0 + q1 p1 + q0 p2 + r p3 <= 128*255 + 2*255*255 + 255*128 = 195330
constexpr int WINDOW31 = (int)(4294967295ull / 195330ull) / BK * BK;
static_assert((double)WINDOW31 * 195330.0 < 4294967296.0, "uint32 window bound (MODE 3)");
// MODE 4 (Matern, four k~ slices x seven D slices): at most four products of <= 255^2 per block
constexpr int WINDOW4 = (int)(4294967295ull / 260100ull) / BK * BK;
static_assert((double)WINDOW4 * 260100.0 < 4294967296.0, "uint32 window bound (MODE 4)");
constexpr int kThreads = 32 * (NCW + 2);
constexpr int PRODUCER_WARP = NCW, MMA_WARP = NCW + 1;
static_assert(NCW * JW == 4 * BK, "4 lane quarters x BK columns");
static_assert(BK % 32 == 0, "int8 K-steps of 32");
// B' row (S column) of point jl in 0..BK-1 of a tile (see the column maps)
__host__ __device__ constexpr int s_col_of(int jl) {
    return JW == 32 ? jl : (jl & ~31) + 8 * ((jl >> 2) & 3) + 4 * ((jl >> 4) & 1) + (jl & 3);
}
constexpr __host__ __device__ int r16(int x) { return (x + 15) & ~15; }
constexpr __host__ __device__ int r32(int x) { return (x + 31) & ~31; }

// Accumulator layout: the slice products are merged by weight.  The D-slice
// operand holds four column blocks [p3 | p2 | p1 | p0] of BLK = round4(C + 1)
// columns (C real columns, 1 constant offset column, zero padding); the three
// int8 MMAs of a K-step multiply q2, q1, q0 by the whole operand (N = 4 BLK;
// q0's N trimmed to round16(3 BLK), BBMM_TC2_TRIM) into accumulator blocks 0-3,
// 1-4 and 2-5, so block k collects every product of weight 2^(8 (5 - k))
// (q_a p_b with a + b = 5 - k) -- the twelve slice products but q0 p0 -- in 6 BLK
// TMEM columns.  The MMAs always
// accumulate; the draining warps zero the columns they read.
// ND = number of D slices: 4 (31-bit D, RBF) or 5 (39-bit D, Matern, whose
// C2 shape is not converged at p: DESIGN.md §6 / reading R29); with 5 slices
// the MMA N = 5 BLK must be a multiple of 16.
template <int C, int DA, int ND = 4>
struct Cfg {
    static constexpr int C1 = C + 1;
    static_assert(C1 <= 48, "too many columns");
    static_assert(ND == 4 || ND == 5 || ND == 7, "D slices");
    static constexpr int BLK = ND == 4 ? (C1 + 3) & ~3 : (C1 + 15) & ~15;
    static constexpr int NB = ND * BLK;                        // D-slice rows (MMA N)
    static_assert(NB % 16 == 0 && NB <= 256, "MMA N");
    // accumulator blocks: ND + 2 (three k~ slices); ND = 7 (MODE 4: four k~ slices x 55-bit D)
    // keeps the 7 blocks of weight 2^64 .. 2^16 (the dropped products are < 2^-52 of the scale)
    static constexpr int NBLK = ND == 7 ? 7 : ND + 2;
    static constexpr int ACC_COLS = NBLK * BLK;
    static constexpr int ACC_END = r32(ACC_COLS);
    static constexpr int NBUF_FIT = (512 - ACC_END) / BK;
    static constexpr int NBUF = NBUF_FIT < 4 ? NBUF_FIT : 4;     // S/A TMEM buffers
    static_assert(NBUF >= 2, "TMEM budget");

    static constexpr int BUF_OFF = ACC_END;                    // NBUF x BK columns
    static constexpr int END = BUF_OFF + NBUF * BK;
    static_assert(END <= 512, "TMEM budget exceeded");
    // Distance MMA operand type: kind::f16 (fp16 hi/lo split, K = 16 per MMA) when DA > 8 --
    // half the MMAs of kind::tf32 (K = 8) at the same 11-bit split precision; at DA = 8 both
    // take one MMA per product and tf32 stays (no operand scaling).  ND == 5 is Matern (MODE 2:
    // plain fp32 x tiles, no distance MMA).
    static constexpr bool F16 = BBMM_TC2_F16DIST && ND == 4 && DA >= BBMM_TC2_F16_MIN_DA;
    static constexpr bool PK = BBMM_TC2_F16PACK && ND == 4 && DA == 8;   // packed fp16, K = 32
    static constexpr bool H16 = F16 || PK;                     // fp16 operands (scaled by 2^5)
    static constexpr int DH = F16 ? r16(DA) : DA;              // K per product group
    static constexpr int EB = H16 ? 2 : 4;                     // operand element bytes
    static constexpr int B8_BYTES = NB * BK;                   // int8 D slices per tile
    // B' per tile: [hi | lo] (2 DH), packed: [hi | lo | hi | 0] (32 halves = 2 DH x 2 bytes)
    static constexpr int XB_BYTES = 2 * DH * BK * (PK ? 4 : EB);
    static constexpr int AP_BYTES = BM * (PK ? 32 : 3 * DH) * EB;   // row operand A' (smem)
    // int8 MMA N of the q1 / q0 slices (BBMM_TC2_TRIM)
    static constexpr int N1 = (ND == 4 && BBMM_TC2_TRIM >= 2 && r16(3 * BLK) < NB) ? r16(3 * BLK) : NB;
    static constexpr int N0 = (ND == 4 && BBMM_TC2_TRIM >= 1)
                                  ? (BBMM_TC2_TRIM >= 2 ? r16(2 * BLK) : (r16(3 * BLK) < NB ? r16(3 * BLK) : NB))
                                  : NB;
    static constexpr int STATIC_BYTES = (C + 1) * BM * 8 + 512;   // acc_sm + barriers
    // Two shared-memory rings, each refilled as soon as its consumer MMA completes:
    // XB (read by the distance MMA of tile t, issued NBUF tiles before tile t's
    // int8 MMAs) and B8 (read by the int8 MMAs).  Depths as the budget allows.
    static constexpr int BUDGET = 227 * 1024 - STATIC_BYTES - AP_BYTES - 1024;
    static constexpr int XS = (3 * XB_BYTES + (NBUF + 3) * B8_BYTES <= BUDGET) ? 3 : 2;
    static constexpr int QS_FIT = (BUDGET - XS * XB_BYTES) / B8_BYTES;
    static constexpr int QS = QS_FIT < NBUF + 3 ? QS_FIT : NBUF + 3;
    static_assert(QS >= 2, "shared-memory ring too shallow");
    static constexpr int Q_OFF = XS * XB_BYTES;                // B8 ring after the XB ring
    static constexpr int AP_OFF = Q_OFF + QS * B8_BYTES;       // then the row operand
    static constexpr int RAW = AP_OFF + AP_BYTES + 1024;
    static_assert(RAW + STATIC_BYTES <= 227 * 1024, "shared memory budget exceeded");
    // >= 120 KB so that a single CTA (which owns all 512 TMEM columns) is resident per SM
    static constexpr int SMEM = RAW > 122880 ? RAW : 122880;
};

// Drain one window's int32 accumulators of this thread's row (TMEM lane)
// into the fp64 sums acc_sm[c][rl] (c == C: constant offset column):
// accumulator block k (BLK columns) carries weight 2^(8 (5 - k)).  The NPS
// warps of a lane quarter share the work: warp h sums the columns cc with
// cc % NPS == h (so no two warps touch one acc_sm entry) and zeroes the
// 32-column chunks q with q % NPS == h for the next window (caller waits for
// the stores).
template <int C, int BLK, int ACC_END, int ND>
__device__ __noinline__ void drain_window(uint32_t lane_base, double (*acc_sm)[BM], int rl, int h) {
    constexpr int NBLK = ND == 7 ? 7 : ND + 2;
    // weight of block 0: q2 (2^16 in k~ 2^23 units) times the top D slice (2^(8 (ND - 1)))
    constexpr double W0 = ND == 4 ? 0x1p40 : ND == 5 ? 0x1p48 : 0x1p64;
    constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    constexpr int M = (C + NPS) / NPS;             // columns cc = h + NPS m <= C per warp
    uint32_t v[M][NBLK];
#pragma unroll
    for (int m = 0; m < M; m++)
#pragma unroll
        for (int k = 0; k < NBLK; k++)
            v[m][k] = (h + NPS * m <= C) ? ptx::tmem_ld1(lane_base + k * BLK + h + NPS * m) : 0u;
    ptx::tmem_ld_wait();
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int cc = h + NPS * m;
        if (cc <= C) {
            double a = acc_sm[cc][rl];
#pragma unroll
            for (int k = 0; k < NBLK; k++) a = fma(W0 / (double)(1ull << (8 * k)), (double)v[m][k], a);
            acc_sm[cc][rl] = a;
        }
    }
    // every warp has read all columns before any is zeroed: the zeroing
    // targets only this warp's chunks, read above by all four warps, so
    // wait for the lane quarter (named barrier over its NPS warps)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (rl >> 5)), "n"(32 * NPS) : "memory");
#pragma unroll 1
    for (int q = 32 * h; q < ACC_END; q += 32 * NPS) {
#pragma unroll
        for (int o = 0; o < 32; o += 8) ptx::tmem_st8(lane_base + q + o, z);
    }
}

// MODE 0: value k~ = K/s (the blackbox matmul) on the 23-bit grid;  MODE 3: the same on a
// 31-bit grid (a fourth, residual slice; BBMM_MATMUL_INT8EXACT31);  MODE 1: value k~ r^2
// (= (dK/dlog l)/s for the isotropic RBF, used by the derivative pass);
// MODE 2: Matern-5/2 k~ = (1 + rh + rh^2/3) e^{-rh}, rh = sqrt(-S) (inputs
// scaled by sqrt5/l; two MUFU ops per pair: sqrt, ex2), 39-bit D (ND = 5).
// MODE 2 computes the distances directly on the FP32 pipes from plain x tiles
// ([BK][DA] fp32 in the XB ring, zero-padded past d) -- the 3xTF32 expanded form's
// ~1e-7 absolute error in r^2 is too large for Matern; DM = the
// dimensions those loops run over (a compile-time bound, zero padding past d).
template <int C, int DA, int MODE, int DM = DA>
__global__ void __launch_bounds__(kThreads, 1)
k1tc2_rbf(const float *__restrict__ Xa, const float *__restrict__ XB,
          const uint8_t *__restrict__ Bpack, const double *__restrict__ Sc, int64_t r0,
          int64_t nloc, int64_t tiles_per_split, int64_t ntiles, double s,
          double *__restrict__ Vpart, int ldv, int coff) {
    constexpr bool MAT = MODE == 2 || MODE == 4;     // Matern: direct distances, no distance MMA
    constexpr bool G31 = MODE == 3 || MODE == 4;     // k~ on the 31-bit grid (four A slices)
    constexpr int ND = MODE == 2 ? 5 : MODE == 4 ? 7 : 4;
    using K = Cfg<C, DA, ND>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_x[K::XS], free_x[K::XS], full_q[K::QS], free_q[K::QS];
    __shared__ __align__(8) uint64_t s_full[K::NBUF], a_full[K::NBUF];
    __shared__ __align__(8) uint64_t acc_full, acc_empty, init_done;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double acc_sm[C + 1][BM];   // fp64 accumulators (+ constant column)

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
    const int ntl = (int)(min(ntiles, t0 + tiles_per_split) - t0);
    constexpr int TPW = (MODE == 4 ? WINDOW4 : MODE == 3 ? WINDOW31 : WINDOW) / BK;

    if (tid == 0) {
        for (int q = 0; q < K::XS; q++) {
            ptx::mbar_init(&full_x[q], 1);
            // MODE 2 reads the x tile on the compute warps (direct distances), not in an MMA
            ptx::mbar_init(&free_x[q], MAT ? NCW : 1);
        }
        for (int q = 0; q < K::QS; q++) {
            ptx::mbar_init(&full_q[q], 1);
            ptx::mbar_init(&free_q[q], 1);
        }
        for (int q = 0; q < K::NBUF; q++) {
            ptx::mbar_init(&s_full[q], 1);
            ptx::mbar_init(&a_full[q], NCW);        // one elected lane per warp
        }
        ptx::mbar_init(&acc_full, 1);
        ptx::mbar_init(&acc_empty, NCW);
        ptx::mbar_init(&init_done, 128);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tmem_base_sh);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    BBMM_DCHECK((uint32_t)K::SMEM <= dyn_smem_bytes() && K::END <= 512);

    if (warp == PRODUCER_WARP) {
        // ------------------------------------------------------- producer
        // loads in the order the MMA issuer consumes them: XB of tiles 0..NBUF-1,
        // then per tile t: B8(t), XB(t + NBUF)
        if (ptx::elect_one()) {
            auto load_x = [&](int t) {
                const int xi = t % K::XS;
                ptx::mbar_wait(&free_x[xi], (uint32_t)(((t / K::XS) & 1) ^ 1));
                ptx::mbar_arrive_expect_tx(&full_x[xi], K::XB_BYTES);
                ptx::bulk_g2s(smem + xi * K::XB_BYTES,
                              reinterpret_cast<const uint8_t *>(XB) + (t0 + t) * K::XB_BYTES,
                              K::XB_BYTES, &full_x[xi]);
            };
            auto load_q = [&](int t) {
                const int qi = t % K::QS;
                ptx::mbar_wait(&free_q[qi], (uint32_t)(((t / K::QS) & 1) ^ 1));
                ptx::mbar_arrive_expect_tx(&full_q[qi], K::B8_BYTES);
                ptx::bulk_g2s(smem + K::Q_OFF + qi * K::B8_BYTES, Bpack + (t0 + t) * K::B8_BYTES,
                              K::B8_BYTES, &full_q[qi]);
            };
            for (int t = 0; t < K::NBUF && t < ntl; t++) load_x(t);
            for (int t = 0; t < ntl; t++) {
                load_q(t);
                if (t + K::NBUF < ntl) load_x(t + K::NBUF);
            }
        }
        __syncwarp();
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------ MMA issuer
        // One thread issues both MMA kinds.  tcgen05.mma ops of one thread
        // execute in issue order, so the distance MMA of tile t + K::NBUF, issued
        // right after the int8 MMAs of tile t that read the same TMEM buffer,
        // cannot overwrite it early: no buffer-free round trip is needed.
        constexpr uint32_t IDS = K::H16 ? ptx::idesc_f16(BM, BK) : ptx::idesc_tf32(BM, BK);
        constexpr uint32_t IDQ = ptx::idesc_i8(BM, K::NB, false, false);
        // MODE 4 (ND = 7, blocks of weight 2^64 .. 2^16): q2 x [p6..p0], q1 x [p6..p1],
        // q0 x [p6..p2], r x [p6..p3] -- N = 7, 6, 5, 4 BLK, every product of the kept weights
        constexpr uint32_t IDQ1 = ptx::idesc_i8(BM, ND == 7 ? 6 * K::BLK : K::N1, false, false);
        constexpr uint32_t IDQ0 = ptx::idesc_i8(BM, ND == 7 ? 5 * K::BLK : K::N0, false, false);
        // MODE 3 residual slice r x [p3 p2 (p1)]: N = round16(2 BLK) -- the extra columns land
        // in blocks of their own weight (r p1 -> block 5) or, at BLK = 4, in the padding
        // column block 6 that is never drained (ACC_END >= 7 BLK there)
        constexpr int NR = r16(2 * K::BLK);   // (r x p3 alone, N = round16(BLK): no faster)
        static_assert(MODE != 3 || NR <= 3 * K::BLK || 7 * K::BLK <= K::ACC_END, "residual N");
        constexpr uint32_t IDQR = ptx::idesc_i8(BM, ND == 7 ? 4 * K::BLK : NR, false, false);
        const bool leader = ptx::elect_one();
        ptx::mbar_wait(&init_done, 0);
        ptx::tc_fence_after();
        auto wait_x = [&](int t) {
            ptx::mbar_wait(&full_x[t % K::XS], (uint32_t)((t / K::XS) & 1));
        };
        // 3-product split: A' = [hi | hi | lo] (3 DH), B' = [hi | lo] (2 DH): K groups
        // (A hi, B hi), (A hi, B lo), (A lo, B hi); one MMA = 32 bytes of K per row
        // (8 tf32 or 16 fp16), the same core-matrix geometry for both kinds
        auto issue_dist = [&](int t) {
            const int xi = t % K::XS;
            const int b = t % K::NBUF;
            ptx::tc_fence_after();
            if (MAT) {
                // no distance MMA: only signal that buffer b is free again once the int8
                // MMAs issued so far (the last readers of b) have completed
                if (leader) ptx::mma_commit(&s_full[b]);
                __syncwarp();
                return;
            }
            if (leader) {
                const uint32_t xb = ptx::smem_u32(smem + xi * K::XB_BYTES);
                const uint32_t ap = ptx::smem_u32(smem + K::AP_OFF);
                if constexpr (K::PK) {
                    // packed: A' = [hi | hi | lo | 0] x B' = [hi | lo | hi | 0], two K = 16 MMAs
#pragma unroll
                    for (int ks = 0; ks < 2; ks++) {
                        const uint64_t bd = ptx::smem_desc_kmajor(xb + ks * 2 * BK * 16, BK * 16, 128);
                        const uint64_t ad = ptx::smem_desc_kmajor(ap + ks * 2 * BM * 16, BM * 16, 128);
                        ptx::mma_f16_ss(tmem + K::BUF_OFF + b * BK, ad, bd, IDS, ks > 0 ? 1u : 0u);
                    }
                } else {
                    constexpr int KS = K::DH * K::EB / 32;     // MMAs per product group
#pragma unroll
                    for (int ks = 0; ks < 3 * KS; ks++) {
                        const int g = ks / KS, kk = ks % KS;
                        const int kb = (g == 1 ? KS : 0) + kk;
                        const uint64_t bd = ptx::smem_desc_kmajor(xb + kb * 2 * BK * 16, BK * 16, 128);
                        const uint64_t ad = ptx::smem_desc_kmajor(ap + ks * 2 * BM * 16, BM * 16, 128);
                        if constexpr (K::F16)
                            ptx::mma_f16_ss(tmem + K::BUF_OFF + b * BK, ad, bd, IDS, ks > 0 ? 1u : 0u);
                        else
                            ptx::mma_tf32_ss(tmem + K::BUF_OFF + b * BK, ad, bd, IDS, ks > 0 ? 1u : 0u);
                    }
                }
                ptx::mma_commit(&s_full[b]);
                ptx::mma_commit(&free_x[xi]);
            }
            __syncwarp();
        };
        for (int t = 0; t < K::NBUF && t < ntl; t++) {
            if (!MAT) wait_x(t);
            issue_dist(t);
        }
        for (int t = 0; t < ntl; t++) {
            const int qi = t % K::QS;
            const int b = t % K::NBUF;
            const int win = t / TPW;
            const bool first = (t % TPW) == 0;
            // operands of the next distance MMA: normally resident long ago, so
            // this check overlaps the wait for the compute warps below
            if (!MAT && t + K::NBUF < ntl) wait_x(t + K::NBUF);
            if (first && win > 0) ptx::mbar_wait(&acc_empty, (uint32_t)((win - 1) & 1));
            ptx::mbar_wait(&a_full[b], (uint32_t)((t / K::NBUF) & 1));
            ptx::mbar_wait(&full_q[qi], (uint32_t)((t / K::QS) & 1));
            ptx::tc_fence_after();
            if (leader) {
                const uint32_t b8 = ptx::smem_u32(smem + K::Q_OFF + qi * K::B8_BYTES);
                const uint32_t aq = tmem + K::BUF_OFF + b * BK;
#pragma unroll
                for (int ks = 0; ks < BK / 32; ks++) {
                    const uint64_t bd = ptx::smem_desc_kmajor(b8 + ks * 2 * K::NB * 16, K::NB * 16, 128);
                    ptx::mma_i8_ts(tmem + 0, aq + 32 * ks + 16, bd, IDQ, 1u);              // q2
                    ptx::mma_i8_ts(tmem + K::BLK, aq + 32 * ks + 8, bd, IDQ1, 1u);         // q1
                    ptx::mma_i8_ts(tmem + 2 * K::BLK, aq + 32 * ks + 0, bd, IDQ0, 1u);     // q0
                    if constexpr (G31 && BBMM_TC2_ABL != 1)
                        ptx::mma_i8_ts(tmem + 3 * K::BLK, aq + 32 * ks + 24, bd, IDQR, 1u);  // r
                }
                ptx::mma_commit(&free_q[qi]);
                if (((t + 1) % TPW) == 0 || t + 1 == ntl) ptx::mma_commit(&acc_full);
            }
            __syncwarp();
            if (t + K::NBUF < ntl) issue_dist(t + K::NBUF);
        }
    } else {
        // -------------------------------------------------------- compute
        const int sub = warp & 3, h = warp >> 2;
        const int64_t row = (int64_t)blockIdx.x * BM + sub * 32 + lane;
        const bool valid = row < nloc;
        // MODE 2: this row's scaled inputs (plain layout of its XB tile)
        float xrow[MAT ? DM : 1];
        if constexpr (MAT) {
            const int64_t rg = r0 + row;
            const int jr = (int)(rg % BK);
            const float *src = XB + (rg / BK) * (int64_t)(2 * DA * BK) + (jr >> 1) * (2 * DA) + (jr & 1);
#pragma unroll
            for (int q = 0; q < DM; q++) xrow[q] = valid ? src[2 * q] : 0.0f;
        }
        const uint32_t lane_base = tmem + ((uint32_t)(sub * 32) << 16);
        if (h == 0) {
            // A_i = [2 xs_i, -|xs_i|^2, 1, 0..] split as [hi | hi | lo] (3xTF32), written to
            // shared memory K-major: [3 DA / 4 chunks][128 rows][4 floats]
            // (F16: fp16 [3 DH / 8 chunks][128 rows][8 halves], entries scaled as in k_prep_tc2)
            const int rl = sub * 32 + lane;
            if constexpr (K::PK) {
                // packed: fp16 [4 chunks][128 rows][8 halves], K = [hi | hi | lo | 0] of DA = 8
                uint16_t *ap = reinterpret_cast<uint16_t *>(smem + K::AP_OFF);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const float v = valid ? kF16Scale * Xa[(r0 + row) * DA + q] : 0.0f;
                    const __half vh = __float2half_rn(v);
                    const __half vl = __float2half_rn(v - __half2float(vh));
                    ap[0 * (BM * 8) + rl * 8 + q] = __half_as_ushort(vh);
                    ap[1 * (BM * 8) + rl * 8 + q] = __half_as_ushort(vh);
                    ap[2 * (BM * 8) + rl * 8 + q] = __half_as_ushort(vl);
                    ap[3 * (BM * 8) + rl * 8 + q] = 0;
                }
            } else if constexpr (K::F16) {
                uint16_t *ap = reinterpret_cast<uint16_t *>(smem + K::AP_OFF);
#pragma unroll
                for (int q = 0; q < K::DH; q++) {
                    const float v = (valid && q < DA) ? kF16Scale * Xa[(r0 + row) * DA + q] : 0.0f;
                    const __half vh = __float2half_rn(v);
                    const __half vl = __float2half_rn(v - __half2float(vh));
                    const __half parts[3] = {vh, vh, vl};
#pragma unroll
                    for (int pt = 0; pt < 3; pt++) {
                        const int k = pt * K::DH + q;
                        ap[(k >> 3) * (BM * 8) + rl * 8 + (k & 7)] = __half_as_ushort(parts[pt]);
                    }
                }
            } else {
                float *ap = reinterpret_cast<float *>(smem + K::AP_OFF);
#pragma unroll
                for (int q = 0; q < DA; q++) {
                    const float v = valid ? Xa[(r0 + row) * DA + q] : 0.0f;
                    const float vh = tf32_rn(v);
                    const float vl = tf32_rn(v - vh);
                    const float parts[3] = {vh, vh, vl};
#pragma unroll
                    for (int pt = 0; pt < 3; pt++) {
                        const int k = pt * DA + q;
                        ap[(k >> 2) * (BM * 4) + rl * 4 + (k & 3)] = parts[pt];
                    }
                }
            }
            // zero this lane quarter's accumulator columns (the MMAs only add)
            {
                constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int q = 0; q < K::ACC_END; q += 8) ptx::tmem_st8(lane_base + q, z);
                ptx::tmem_st_wait();
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&init_done);
        }
        // each warp zeroes the fp64 sums it alone accumulates (columns cc = h mod NPS of its
        // rows, drain_window): no cross-warp order needed before the first drain
        for (int cc = h; cc <= C; cc += NPS) acc_sm[cc][sub * 32 + lane] = 0.0;
        const uint32_t a_sfull = ptx::smem_u32(&s_full[0]);
        const uint32_t a_afull = ptx::smem_u32(&a_full[0]);
        const uint32_t a_accf = ptx::smem_u32(&acc_full), a_acce = ptx::smem_u32(&acc_empty);
        const uint32_t my_col = lane_base + K::BUF_OFF +
                                (JW == 32 ? 32 * h : 32 * (h >> 1) + 4 * (h & 1));
        int win = 0;
        // With only two S/A buffers the MMA side is one tile ahead, so a deferred publish
        // would sit on the critical path: publish each tile right after its stores then.
        constexpr bool DEFER = K::NBUF >= 3;
        // Per tile: S = LDTM, A slices = quantise(ex2(S)), STTM over the same
        // columns, arrive a_full.  The TMEM stores land slowly while the int8
        // MMAs of the previous tile stream through TMEM, so the arrive for
        // tile t (and its tcgen05.wait::st) is deferred to the middle of tile
        // t + 1's MUFU work instead of stalling the warp (K1-TC).
        static_assert(MODE != 3 || JW == 32, "MODE 3 stores four slices over the 32 S columns");
        auto quant4 = [&](const uint32_t *sv, int u, uint32_t &a0, uint32_t &a1, uint32_t &a2,
                          uint32_t &a3) {
            uint32_t q[4];
            uint32_t sw[4] = {sv[4 * u], sv[4 * u + 1], sv[4 * u + 2], sv[4 * u + 3]};
            if constexpr (K::H16) {   // the MMA gave 2^10 S: rescale, two points per FMUL2
#pragma unroll
                for (int v = 0; v < 4; v += 2) {
                    unsigned long long ps;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(ps) : "r"(sw[v]), "r"(sw[v + 1]));
                    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(ps) : "l"(0x3A8000003A800000ull));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(sw[v]), "=r"(sw[v + 1]) : "l"(ps));
                }
            }
            if constexpr (MAT) {
                // sv holds +rh'^2 with rh' = log2(e) rh (a sum of squares: no clamp);
                // k~ = (1 + rh + rh^2/3) 2^(-rh') with rh = ln2 rh'; the polynomial and the
                // product for two points per FFMA2 / FMUL2
#pragma unroll
                for (int v = 0; v < 4; v += 2) {
                    const float rh0 = sqrt_approx(__uint_as_float(sw[v]));
                    const float rh1 = sqrt_approx(__uint_as_float(sw[v + 1]));
                    const float e0 = ex2_approx(-rh0), e1 = ex2_approx(-rh1);
                    unsigned long long prh, prs, pe, pp;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(prh) : "f"(rh0), "f"(rh1));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(prs) : "r"(sw[v]), "r"(sw[v + 1]));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(pe) : "f"(e0), "f"(e1));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(prh), "l"(0x3F3172183F317218ull),
                        "l"(0x3F8000003F800000ull));                         // 1 + ln2 rh'
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(pp) : "l"(prs), "l"(0x3E23FEA03E23FEA0ull));
                    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(pp) : "l"(pe));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(q[v]), "=r"(q[v + 1]) : "l"(pp));
                }
            }
            if constexpr (!MAT) {
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sj = __uint_as_float(sw[v]);
                float kv = ex2_approx(sj);
                // r^2 = -2 ln2 S (S = -(log2 e / 2) r^2), clamped at 0 (S may be
                // +eps by rounding near the diagonal).  The factor 2 ln 2 is applied in the
                // epilogue, so the quantised value is k~ (-S) <= 1/(e ln 2)/2 ~= 0.53 (not
                // k~ r^2 <= 2/e ~= 0.74): the 2^-23 grid step is 1.39x coarser relative to
                // the derivative value (about half a bit), measured inside the gradient bar
                // (MODE 1 margin)
                // (one FMUL.SAT: the [0, 1] saturation clamps the rounding-positive S near the
                //  diagonal to 0 like max(-S, 0) did, and never binds above: k~ (-S) <= 0.53)
                if (MODE == 1) kv = __saturatef(kv * -sj);
                q[v] = __float_as_uint(kv);
            }
            }
            if constexpr (G31 && BBMM_TC2_ABL != 3) {
                // 31-bit grid: the fixed-point value F = k~ 2^31 (exact for k~ >= 2^-8, where the
                // fp32 k~ has no bits below 2^-31; floor below) as two 16-bit halves, F = H 2^16 + L:
                //   h = rz(2^15 k~ + 2^23)              = 2^23 + H,  H = floor(2^15 k~) <= 2^15
                //   u = 2^39 + 2^23 - 2^16 h             = 2^23 - 2^16 H (exact: a multiple of 2^16)
                //   m = rz(2^31 k~ + u)                  = 2^23 + L,  L = floor(2^31 k~ - 2^16 H) < 2^16
                // (each FMA's exact result is representable or truncated at ulp 1); the low two
                // bytes of h and m are the four u8 slices, k~ = (H.b1 2^24 + H.b0 2^16 + L.b1 2^8 +
                // L.b0) 2^-31 -- the weights of INT8EXACT's q2 q1 q0 plus the residual slot below q0,
                // 8 byte permutes per 4 pairs (INT8EXACT31)
                uint32_t hw[4], mw[4];
#pragma unroll
                for (int v = 0; v < 4; v += 2) {
                    unsigned long long pk, ph, pu, pm;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(pk) : "r"(q[v]), "r"(q[v + 1]));
                    asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(ph) : "l"(pk), "l"(0x4700000047000000ull),
                        "l"(0x4B0000004B000000ull));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pu) : "l"(ph), "l"(0xC7800000C7800000ull),
                        "l"(0x5300008053000080ull));
                    asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(pm) : "l"(pk), "l"(0x4F0000004F000000ull),
                        "l"(pu));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(hw[v]), "=r"(hw[v + 1]) : "l"(ph));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(mw[v]), "=r"(mw[v + 1]) : "l"(pm));
                }
                const uint32_t t01 = __byte_perm(hw[0], hw[1], 0x5140);
                const uint32_t t23 = __byte_perm(hw[2], hw[3], 0x5140);
                const uint32_t l01 = __byte_perm(mw[0], mw[1], 0x5140);
                const uint32_t l23 = __byte_perm(mw[2], mw[3], 0x5140);
                a2 = __byte_perm(t01, t23, 0x7632);      // H.b1: weight 2^24 (q2's)
                a1 = __byte_perm(t01, t23, 0x5410);      // H.b0: 2^16 (q1's)
                a0 = __byte_perm(l01, l23, 0x7632);      // L.b1: 2^8  (q0's)
                a3 = __byte_perm(l01, l23, 0x5410);      // L.b0: 2^0  (residual slot)
            } else {
                // q = 2 + 2 k~ in [2, 4]: for k~ < 1 the exponent is 128 (bit 23 = 0) and the
                // mantissa is k~ 2^23 rounded to nearest; k~ = 1 gives 4.0 = exponent 129, whose
                // low bit lands on bit 23 = 2^23 = k~ 2^23 again.  So the three low bytes are
                // exactly the 23-bit fixed-point k~ 2^23 for every k~ in [0, 1] (grid 2^-23: half
                // the rounding of the q = 2 + k~ form).  Two points per instruction (FFMA2).
    #pragma unroll
                for (int v = 0; v < 4; v += 2) {
                    unsigned long long pq;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(pq) : "r"(q[v]), "r"(q[v + 1]));
                    asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(pq) : "l"(0x4000000040000000ull));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(q[v]), "=r"(q[v + 1]) : "l"(pq));
                }
                const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240);
                const uint32_t t23 = __byte_perm(q[2], q[3], 0x6240);
                const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351);
                const uint32_t u23 = __byte_perm(q[2], q[3], 0x7351);
                a0 = __byte_perm(t01, t23, 0x5410);
                a2 = __byte_perm(t01, t23, 0x7632);
                a1 = __byte_perm(u01, u23, 0x5410);
                a3 = 0u;
            }
        };
        // publish tile tp's A slices (stores issued earlier), then drain the
        // accumulators if tp closed a window
        auto publish = [&](int tp) {
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_a(a_afull + 8 * (tp % K::NBUF));
            const bool last_of_window = ((tp + 1) % TPW) == 0 || tp + 1 == ntl;
            if (last_of_window) {
                ptx::mbar_wait_a(a_accf, (uint32_t)(win & 1));
                ptx::tc_fence_after();
                drain_window<C, K::BLK, K::ACC_END, ND>(lane_base, acc_sm, sub * 32 + lane, h);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_a(a_acce);
                win++;
            }
        };
        for (int t = 0; t < ntl; t++) {
            const int b = t % K::NBUF;
            ptx::mbar_wait_a(a_sfull + 8 * b, (uint32_t)((t / K::NBUF) & 1));
            ptx::tc_fence_after();
            uint32_t sv[JW];
            const uint32_t col = my_col + b * BK;
            if constexpr (MAT) {
                // S = -r^2 from direct differences with the tile's x_j (broadcast loads)
                const int xs = t % K::XS;
                ptx::mbar_wait(&full_x[xs], (uint32_t)((t / K::XS) & 1));
                // two points at a time on the paired FP32 pipe (FADD2 / FFMA2): the tile stores
                // (x_j0q, x_j1q) adjacent, so one 128-bit shared load gives two packed pairs
                const uint32_t xt = ptx::smem_u32(smem + xs * K::XB_BYTES) + (JW * h / 2) * (2 * DA) * 4;
                unsigned long long xr2[DM];
#pragma unroll
                for (int q = 0; q < DM; q++)
                    asm("mov.b64 %0, {%1, %1};" : "=l"(xr2[q]) : "f"(xrow[q]));
#pragma unroll
                for (int jp = 0; jp < JW / 2; jp++) {
                    unsigned long long acc2[2] = {0ull, 0ull};
#pragma unroll
                    for (int q2 = 0; q2 < (DM + 1) / 2; q2++) {
                        unsigned long long x2[2];
                        asm volatile("ld.shared.v2.b64 {%0,%1}, [%2];"
                                     : "=l"(x2[0]), "=l"(x2[1])
                                     : "r"(xt + (jp * 2 * DA + 4 * q2) * 4));
#pragma unroll
                        for (int u = 0; u < 2; u++) {
                            const int q = 2 * q2 + u;
                            if (q < DM) {
                                unsigned long long df;
                                asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(df) : "l"(xr2[q]), "l"(x2[u]));
                                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc2[u]) : "l"(df));
                            }
                        }
                    }
                    // the two partial sums of the pair, added in one FADD2
                    unsigned long long ssum;
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(ssum) : "l"(acc2[0]), "l"(acc2[1]));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(sv[2 * jp]), "=r"(sv[2 * jp + 1]) : "l"(ssum));
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&free_x[xs]);
            } else if constexpr (JW == 32 && BBMM_TC2_SPLITLD) {
                ptx::tmem_ld16(col, *reinterpret_cast<uint32_t(*)[16]>(sv));
            } else if constexpr (JW == 32) {
                ptx::tmem_ld32(col, *reinterpret_cast<uint32_t(*)[32]>(sv));
            } else {
#pragma unroll
                for (int u = 0; u < 4; u++) ptx::tmem_ld4(col + 8 * u, sv + 4 * u);
            }
            if constexpr (!MAT) ptx::tmem_ld_wait();
            uint32_t w0[JW / 4], w1[JW / 4], w2[JW / 4], w3[JW / 4];
#pragma unroll
            for (int u = 0; u < JW / 8; u++) quant4(sv, u, w0[u], w1[u], w2[u], w3[u]);
            if constexpr (JW == 32 && BBMM_TC2_SPLITLD && !MAT)
                ptx::tmem_ld16(col + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
            if (DEFER && t > 0) publish(t - 1);
            // (the first half's stores overwrite S columns 16-19 / 24-27 of the second half)
            if constexpr (JW == 32 && BBMM_TC2_SPLITLD && !MAT) ptx::tmem_ld_wait();
            // overwrite own S columns with the A slices q0 | q1 | q2 (column maps
            // above), each half as soon as it is quantised: spreading the stores
            // over the tile measured 3 % faster than one burst at its end
            if constexpr (JW == 32 && !(BBMM_TC2_STBURST && G31)) {
                ptx::tmem_st4(col + 0, *reinterpret_cast<const uint32_t(*)[4]>(w0));
                ptx::tmem_st4(col + 8, *reinterpret_cast<const uint32_t(*)[4]>(w1));
                ptx::tmem_st4(col + 16, *reinterpret_cast<const uint32_t(*)[4]>(w2));
                if constexpr (G31 && BBMM_TC2_ABL != 2) ptx::tmem_st4(col + 24, *reinterpret_cast<const uint32_t(*)[4]>(w3));
            }
#pragma unroll
            for (int u = JW / 8; u < JW / 4; u++) quant4(sv, u, w0[u], w1[u], w2[u], w3[u]);
            if constexpr (JW == 32 && (BBMM_TC2_STBURST && G31)) {
                ptx::tmem_st8(col + 0, *reinterpret_cast<const uint32_t(*)[8]>(w0));
                ptx::tmem_st8(col + 8, *reinterpret_cast<const uint32_t(*)[8]>(w1));
                ptx::tmem_st8(col + 16, *reinterpret_cast<const uint32_t(*)[8]>(w2));
                if constexpr (G31) ptx::tmem_st8(col + 24, *reinterpret_cast<const uint32_t(*)[8]>(w3));
            } else if constexpr (JW == 32) {
                ptx::tmem_st4(col + 4, *reinterpret_cast<const uint32_t(*)[4]>(w0 + 4));
                ptx::tmem_st4(col + 12, *reinterpret_cast<const uint32_t(*)[4]>(w1 + 4));
                ptx::tmem_st4(col + 20, *reinterpret_cast<const uint32_t(*)[4]>(w2 + 4));
                if constexpr (G31 && BBMM_TC2_ABL != 2) ptx::tmem_st4(col + 28, *reinterpret_cast<const uint32_t(*)[4]>(w3 + 4));
            } else {
                ptx::tmem_st4(col + 0, *reinterpret_cast<const uint32_t(*)[4]>(w0));
                ptx::tmem_st4(col + 8, *reinterpret_cast<const uint32_t(*)[4]>(w1));
                ptx::tmem_st4(col + 16, *reinterpret_cast<const uint32_t(*)[4]>(w2));
            }
            if (!DEFER) publish(t);
        }
        if (DEFER && ntl > 0) publish(ntl - 1);
        if (h == 0 && valid) {
            // Vpart rows of ldv columns, this launch's block at column coff (column chunks)
            constexpr int CS = (C + 3) & ~3;
            const int rl = sub * 32 + lane;
            double *out = Vpart + ((int64_t)blockIdx.y * nloc + row) * ldv + coff;
            BBMM_DCHECK(coff + C <= ldv);
            const double base = s * (ND == 4 ? 0x1p-53 : ND == 5 ? 0x1p-61 : 0x1p-77) *
                                (MODE == 1 ? 1.3862943611198906 : 1.0);   // MODE 1: r^2 = -2 ln2 S
            const double cacc = acc_sm[C][rl];
#pragma unroll
            for (int c = 0; c < C; c++) out[c] = base * Sc[c] * (acc_sm[c][rl] - cacc);
            if (coff + CS <= ldv)
#pragma unroll
                for (int c = C; c < CS; c++) out[c] = 0.0;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------- operand prep
// Per point: xs = (x - mean) scale (fp32), e = -|xs|^2.
//   Xa[i]  = [2 xs_i (d), e_i, 1, 0..]            (DA floats, row operand)
//   XB tile tt (BK points): B'_j = [xs_j, 1, e_j, 0..] split [hi | lo]
//   stored K-major for the MMA: [2 DA / 4 chunks][BK rows][4 floats] (tf32), or for
//   DA > 8 (Cfg::F16) times kF16Scale as fp16 [2 DH / 8 chunks][BK rows][8 halves].
__global__ void k_prep_tc2(const float *__restrict__ X, int64_t n, int64_t npad, int d, int DA,
                           const float *__restrict__ scale, const double *__restrict__ mean,
                           float *__restrict__ Xa, float *__restrict__ XB,
                           unsigned int *__restrict__ max_sq_bits, int plain) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npad;
         j += (int64_t)gridDim.x * blockDim.x) {
        float xs[kMaxDim];
        float e = 0.0f;
        for (int q = 0; q < d; q++) {
            xs[q] = (j < n) ? (float)((double)X[j * d + q] - mean[q]) * scale[q] : 0.0f;
            e = fmaf(xs[q], xs[q], e);
        }
        if (j < n) atomicMax(max_sq_bits, __float_as_uint(e));   // e >= 0: bits are ordered
        const bool f16 = BBMM_TC2_F16DIST && !plain && DA >= BBMM_TC2_F16_MIN_DA;   // Cfg::F16
        const bool pk = BBMM_TC2_F16PACK && !plain && DA == 8;                       // Cfg::PK
        const int DH = f16 ? (DA + 15) & ~15 : DA;
        e = -e;
        const bool ok = j < n;
        for (int q = 0; q < DA; q++) {
            float a = 0.0f, b = 0.0f;
            if (ok) {
                if (q < d) { a = 2.0f * xs[q]; b = xs[q]; }
                else if (q == d) { a = e; b = 1.0f; }
                else if (q == d + 1) { a = 1.0f; b = e; }
            }
            Xa[j * DA + q] = a;
            if (plain) {   // MODE 2: x_j fp32, point pairs interleaved: [BK/2][DA][2], zero past d
                const int jj = (int)(j % BK);
                XB[(j / BK) * (int64_t)(2 * DA * BK) + (jj >> 1) * (2 * DA) + 2 * q + (jj & 1)] =
                    (ok && q < d) ? xs[q] : 0.0f;
                continue;
            }
            const int64_t tt = j / BK;
            const int jj = s_col_of((int)(j - tt * BK));
            if (pk) {    // packed fp16 [4 chunks][BK rows][8 halves] = [hi | lo | hi | 0], times kF16Scale
                const float bs = kF16Scale * b;
                const __half bh = __float2half_rn(bs);
                const __half bl = __float2half_rn(bs - __half2float(bh));
                uint16_t *tile = reinterpret_cast<uint16_t *>(XB) + tt * (int64_t)(32 * BK);
                tile[0 * (BK * 8) + jj * 8 + q] = __half_as_ushort(bh);
                tile[1 * (BK * 8) + jj * 8 + q] = __half_as_ushort(bl);
                tile[2 * (BK * 8) + jj * 8 + q] = __half_as_ushort(bh);
                tile[3 * (BK * 8) + jj * 8 + q] = 0;
                continue;
            }
            if (f16) {   // fp16 [2 DH / 8 chunks][BK rows][8 halves], times kF16Scale
                const float bs = kF16Scale * b;
                const __half bh = __float2half_rn(bs);
                const __half bl = __float2half_rn(bs - __half2float(bh));
                uint16_t *tile = reinterpret_cast<uint16_t *>(XB) + tt * (int64_t)(2 * DH * BK);
                const __half parts[2] = {bh, bl};
                for (int pt = 0; pt < 2; pt++) {
                    const int k = pt * DH + q;         // K index in [0, 2 DH)
                    tile[(k >> 3) * (BK * 8) + jj * 8 + (k & 7)] = __half_as_ushort(parts[pt]);
                }
                continue;
            }
            const float bh = tf32_rn(b);
            const float bl = tf32_rn(b - bh);
            float *tile = XB + tt * (int64_t)(2 * DA * BK);
            const float parts[2] = {bh, bl};
            for (int pt = 0; pt < 2; pt++) {
                const int k = pt * DA + q;             // K index in [0, 2 DA)
                tile[(k >> 2) * (BK * 4) + jj * 4 + (k & 3)] = parts[pt];
            }
        }
        // F16: zero K padding DA..DH-1 of both halves
        if (f16) {
            const int64_t tt = j / BK;
            const int jj = s_col_of((int)(j - tt * BK));
            uint16_t *tile = reinterpret_cast<uint16_t *>(XB) + tt * (int64_t)(2 * DH * BK);
            for (int q = DA; q < DH; q++)
                for (int pt = 0; pt < 2; pt++) {
                    const int k = pt * DH + q;
                    tile[(k >> 3) * (BK * 8) + jj * 8 + (k & 7)] = 0;
                }
        }
    }
}

}  // namespace tc2

// ======================================================================
// host side
// ======================================================================
static int tc2_da(int d) { return ((d + 2 + 7) / 8) * 8; }

// The instantiated shapes (column block C, da): RBF C in {1, 2, 4, 8} with da <= 24 and
// {11, 17, 33} with da <= 40 (every d <= kMaxDim = 32); Matern-5/2 C in {11, 17} with da <= 16.  Any c up to the largest
// runs on the next instantiation with zero-padded columns (the padded columns add no work to the
// MUFU-bound pair loop, only to the int8 MMAs).
int k1tc2_cols(int kind, int d, int c) {
    const int da = tc2_da(d);
    if (kind == BBMM_MATERN52) return da > 16 ? 0 : c <= 11 ? 11 : c <= 17 ? 17 : 0;
    if (kind != BBMM_RBF || da > 40) return 0;
    if (da <= 24)
        for (int v : {1, 2, 4, 8})
            if (c <= v) return v;
    return c <= 11 ? 11 : c <= 17 ? 17 : c <= 33 ? 33 : 0;
}
bool k1tc2_supported(int kind, int d, int c) { return k1tc2_cols(kind, d, c) > 0; }
// More columns than the largest instantiation (c + 1 > 33 RBF / 17 Matern, up to the C-ABI's 64):
// ceil(c / cb) column chunks of the largest block, one launch each.  Every chunk recomputes the
// kernel values (the MUFU-bound pair loop runs nch times) -- still well under the CUDA-core
// FP64ACC path, whose cost grows with c (VERDICT r1 "next" 7).
int k1tc2_chunks(int kind, int d, int c, int *cb) {
    const int big = kind == BBMM_MATERN52 ? 17 : 33;
    if (c <= big || k1tc2_cols(kind, d, big) != big) return 0;
    *cb = big;
    return (c + big - 1) / big;
}
// isotropic-RBF derivative (MODE 1) instantiations: C in {11, 17, 33}, any da <= 40
int k1tc2_deriv_cols(int d, int c) {
    if (tc2_da(d) > 40) return 0;
    return c <= 11 ? 11 : c <= 17 ? 17 : c <= 33 ? 33 : 0;
}

int64_t k1tc2_xa_floats(int64_t npad, int d) { return npad * tc2_da(d); }
int64_t k1tc2_xb_floats(int64_t npad, int d) { return npad * 2 * tc2_da(d); }

float k1tc2_prep_inputs(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h,
                        float *Xa, float *XB, int64_t npad) {
    double *mean = (double *)ctx->ws.get("tc_mean", kMaxDim * 8);
    float *sc_d = (float *)ctx->ws.get("tc_scale", kMaxDim * 4);
    float sc[kMaxDim];
    // RBF: S = -|xs_i - xs_j|^2 = -(log2 e / 2) r^2 -> k~ = 2^S;  Matern: |xs_i - xs_j|^2 = rh'^2
    // Matern: inputs scaled by sqrt5 log2(e) / l, so rh' = log2(e) rh feeds ex2 directly
    const double base = h.kind == BBMM_RBF ? std::sqrt(0.5 / std::log(2.0))
                                           : std::sqrt(5.0) / std::log(2.0);
    for (int q = 0; q < d; q++) sc[q] = (float)(base / h.ls[h.n_ls == 1 ? 0 : q]);
    BBMM_CUDA(cudaMemcpyAsync(sc_d, sc, sizeof(float) * d, cudaMemcpyHostToDevice, ctx->stream));
    k1tc_col_mean(ctx, X, n, d, mean);
    unsigned int *mx = (unsigned int *)ctx->ws.get("tc_maxsq", 4);
    BBMM_CUDA(cudaMemsetAsync(mx, 0, 4, ctx->stream));
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npad, 256), 4 * kNumSMs));
    tc2::k_prep_tc2<<<grid, 256, 0, ctx->stream>>>(X, n, npad, d, tc2_da(d), sc_d, mean, Xa, XB,
                                                   mx, h.kind == BBMM_MATERN52 ? 1 : 0);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    unsigned int mh = 0;
    BBMM_CUDA(cudaMemcpyAsync(&mh, mx, 4, cudaMemcpyDeviceToHost, ctx->stream));
    BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    float mf;
    std::memcpy(&mf, &mh, 4);
    return mf;
}

template <int C, int DA, int MODE, int DM = DA>
static int launch_tc2(bbmm_ctx_s *ctx, const float *Xa, const float *XB, const uint8_t *Bp,
                      const double *S, int64_t n, int64_t r0, int64_t nloc, double s,
                      double *Vpart, size_t cap, int ldv, int coff) {
    using K = tc2::Cfg<C, DA, MODE == 2 ? 5 : MODE == 4 ? 7 : 4>;
    const int64_t ntiles = ceil_div(n, tc2::BK);
    const int64_t rb = ceil_div(nloc, tc2::BM);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * kNumSMs, rb), ntiles));
    const int64_t tps = ceil_div(ntiles, sp);
    sp = ceil_div(ntiles, tps);
    if (ldv == 0) ldv = (C + 3) & ~3;
    BBMM_REQUIRE(coff + C <= ldv && (size_t)sp * nloc * ldv <= cap, "Vpart workspace too small (k1tc2)");
    static DeviceOnce attr;
    attr(ctx->device, [] {
        BBMM_CUDA(cudaFuncSetAttribute(tc2::k1tc2_rbf<C, DA, MODE, DM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
    });
    dim3 grid((unsigned)rb, (unsigned)sp);
    tc2::k1tc2_rbf<C, DA, MODE, DM><<<grid, tc2::kThreads, K::SMEM, ctx->stream>>>(
        Xa, XB, Bp, S, r0, nloc, tps, ntiles, s, Vpart, ldv, coff);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    return (int)sp;
}

size_t k1tc2_vpart_elems(int64_t n, int64_t nloc, int c) {
    const int64_t ntiles = ceil_div(n, tc2::BK);
    const int64_t rb = ceil_div(std::max<int64_t>(nloc, 1), tc2::BM);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * kNumSMs, rb), ntiles));
    return (size_t)sp * std::max<int64_t>(nloc, 1) * ((c + 3) & ~3);
}

bool k1tc2_deriv_supported(int kind, int n_ls, int d, int c) {
    int cb;
    return n_ls == 1 && kind == BBMM_RBF &&
           (k1tc2_deriv_cols(d, c) > 0 || k1tc2_chunks(kind, d, c, &cb) > 0);   // chunks: MODE 1 at 33
}

int k1tc2_matmul(bbmm_ctx_s *ctx, const float *Xa, const float *XB, const uint8_t *Bp,
                 const double *S, int d, int c, int64_t n, int64_t r0, int64_t nloc, double s,
                 double *Vpart, size_t cap, cudaEvent_t ev0, cudaEvent_t ev1, int mode, int ldv,
                 int coff) {
    if (ev0) record_event(ctx, ev0);
    int sp = 1;
    const int da = tc2_da(d);
    if (mode == 1) {
        BBMM_REQUIRE(k1tc2_deriv_cols(d, c) == c, "k1tc2: derivative mode shape");
        if (nloc > 0) {
#define BBMM_TC2D(CC, DD) \
    if (c == CC && da == DD) sp = launch_tc2<CC, DD, 1>(ctx, Xa, XB, Bp, S, n, r0, nloc, s, Vpart, cap, ldv, coff); else
            BBMM_TC2D(11, 8) BBMM_TC2D(11, 16) BBMM_TC2D(11, 24) BBMM_TC2D(11, 32)
            BBMM_TC2D(17, 8) BBMM_TC2D(17, 16) BBMM_TC2D(17, 24) BBMM_TC2D(17, 32)
            BBMM_TC2D(33, 8) BBMM_TC2D(33, 16) BBMM_TC2D(33, 24) BBMM_TC2D(33, 32)
            BBMM_TC2D(11, 40) BBMM_TC2D(17, 40) BBMM_TC2D(33, 40)
            throw Error{BBMM_ERR_ARG, "k1tc2: unsupported derivative shape"};
#undef BBMM_TC2D
        }
        if (ev1) record_event(ctx, ev1);
        return sp;
    }
    if (mode == 2 || mode == 4) {   // Matern-5/2: 23-bit grid, 39-bit D / 31-bit grid, 55-bit D
#define BBMM_TC2M(CC, DD, DMM) \
    (mode == 4 ? launch_tc2<CC, DD, 4, DMM>(ctx, Xa, XB, Bp, S, n, r0, nloc, s, Vpart, cap, ldv, coff) \
               : launch_tc2<CC, DD, 2, DMM>(ctx, Xa, XB, Bp, S, n, r0, nloc, s, Vpart, cap, ldv, coff))
        if (nloc > 0) {
            if (c == 17 && d == 9) sp = BBMM_TC2M(17, 16, 9);
            else if (c == 17 && da == 16) sp = BBMM_TC2M(17, 16, 16);
            else if (c == 17 && da == 8) sp = BBMM_TC2M(17, 8, 8);
            else if (c == 11 && da == 16) sp = BBMM_TC2M(11, 16, 16);
            else if (c == 11 && da == 8) sp = BBMM_TC2M(11, 8, 8);
            else throw Error{BBMM_ERR_ARG, "k1tc2: unsupported Matern shape"};
        }
#undef BBMM_TC2M
        if (ev1) record_event(ctx, ev1);
        return sp;
    }
#define BBMM_TC2(CC, DD) \
    if (c == CC && da == DD) sp = g31 ? launch_tc2<CC, DD, 3>(ctx, Xa, XB, Bp, S, n, r0, nloc, s, Vpart, cap, ldv, coff) \
                                      : launch_tc2<CC, DD, 0>(ctx, Xa, XB, Bp, S, n, r0, nloc, s, Vpart, cap, ldv, coff); else
    const bool g31 = mode == 3;   // the 31-bit k~ grid (TcOperand::grid31): MODE 3
    if (nloc > 0) {
        BBMM_TC2(1, 8) BBMM_TC2(2, 8) BBMM_TC2(4, 8) BBMM_TC2(8, 8) BBMM_TC2(11, 8)
        BBMM_TC2(17, 8) BBMM_TC2(1, 16) BBMM_TC2(2, 16) BBMM_TC2(4, 16) BBMM_TC2(8, 16)
        BBMM_TC2(11, 16) BBMM_TC2(17, 16) BBMM_TC2(1, 24) BBMM_TC2(2, 24) BBMM_TC2(4, 24)
        BBMM_TC2(8, 24) BBMM_TC2(11, 24) BBMM_TC2(17, 24) BBMM_TC2(11, 32) BBMM_TC2(17, 32)
        BBMM_TC2(33, 8) BBMM_TC2(33, 16) BBMM_TC2(33, 24) BBMM_TC2(33, 32)
        BBMM_TC2(11, 40) BBMM_TC2(17, 40) BBMM_TC2(33, 40)
        throw Error{BBMM_ERR_ARG, "k1tc2: unsupported (c, d)"};
    }
#undef BBMM_TC2
    if (ev1) record_event(ctx, ev1);
    return sp;
}

// ------------------------------------------------ INT8EXACT dispatch
TcOperand tc_prepare(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, int c, const Hyper &h,
                     int64_t npad_rows) {
    TcOperand op;
    if (!ctx->matmul_tc) return op;
    const int64_t npad = k1tc_pad_rows(npad_rows);
    op.d = d;
    int cbk = 0;
    const int nch = k1tc2_chunks(h.kind, d, c, &cbk);
    if (k1tc2_supported(h.kind, d, c) || nch > 0) {
        float *xa = (float *)ctx->ws.get("tc2_Xa", (size_t)k1tc2_xa_floats(npad, d) * 4);
        float *xb = (float *)ctx->ws.get("tc2_XB", (size_t)k1tc2_xb_floats(npad, d) * 4);
        const float max_sq = k1tc2_prep_inputs(ctx, X, n, d, h, xa, xb, npad);
        // The expanded distance 2 xs_i.xs_j - |xs_i|^2 - |xs_j|^2 loses ~eps32 max|xs|^2
        // absolutely; beyond max|xs|^2 = 16 (kernel-value error > ~1e-6) fall back to
        // the direct-difference FP64ACC path.
        // (Matern computes direct differences: no expanded-form error, no guard)
        if (h.kind == BBMM_RBF && !(max_sq <= 16.0f)) return op;
        op.version = 2;
        op.kind = h.kind;
        op.cb = nch > 0 ? cbk : k1tc2_cols(h.kind, d, c);
        op.nch = nch > 0 ? nch : 1;
        op.npad = npad;
        // k~ grid: the 23-bit grid's per-entry error (5.3e-8 s rms at C4, the
        // MUFU's 2.8e-8 random part plus the grid's 4.2e-8) moves the solves by about
        // sqrt(n) eps s / sigma^2; where that would pass 0.8e-4 (a 20 % margin under the 1e-4
        // bar) the 31-bit grid (MUFU error only, 3.3e-8) is used -- C4 at n = 1M: 1.77e-4 -> 31 bits
        // Matern-5/2 on the fly keeps the 31-bit grid (with 55-bit D, MODE 4) unless the 23-bit
        // grid is forced: most of its kernel values are small (k~ ~ e^-rh), where the 23-bit
        // grid's ABSOLUTE 2^-24 error is large relative to the fp32 value, and the C2 shape is not
        // converged at p -- full C2 on the 23-bit grid with 39-bit D (MODE 2) missed the regime-B
        // bars (solve 3.2e-3 vs the fp64 oracle; the fp32-valued FP64ACC operator: 4.1e-4)
        const double est23 = std::sqrt((double)n) * 5.3e-8 * h.s / h.noise_var;
        op.grid31 = h.kind == BBMM_RBF
                        ? (ctx->matmul_grid == 31 || (ctx->matmul_grid == 0 && est23 > 0.8e-4))
                        : ctx->matmul_grid != 23;
        op.nd = h.kind == BBMM_MATERN52 ? (op.grid31 ? 7 : 5) : 4;
        op.Xa = xa;
        op.XB = xb;
    }
    return op;
}

size_t tc_vpart_elems(const TcOperand &op, int64_t n, int64_t nloc, int cb) {
    if (op.version == 3) return k2tc_vpart_elems(n, nloc, cb);
    return k1tc2_vpart_elems(n, nloc, cb == op.cb ? op.nch * op.cb : cb);   // all chunks' columns
}

size_t tc_bp_bytes(const TcOperand &op) {
    return (size_t)op.nch * op.npad * tc_bslice_rows(op.cb, tc_dslices(op));
}

void tc_pack(bbmm_ctx_s *ctx, const TcOperand &op, const double *D, int64_t ldd, int64_t row0,
             int64_t rows, int64_t n, int c, const double *S, uint8_t *Bp) {
    const int nd = tc_dslices(op);
    const size_t stride = (size_t)op.npad * tc_bslice_rows(op.cb, nd);
    for (int z = 0; z < op.nch; z++) {
        const int c0 = z * op.cb, cz = std::min(op.cb, c - c0);
        k1tc_pack(ctx, D + c0, ldd, row0, rows, n, cz, S + c0, Bp + z * stride, nd, op.cb);
    }
}

int tc_matmul(bbmm_ctx_s *ctx, const TcOperand &op, const uint8_t *Bp, const double *S, int c,
              int64_t n, int64_t r0, int64_t nloc, double s, double *Vpart, size_t cap,
              cudaEvent_t ev0, cudaEvent_t ev1, int mode) {
    // c = the column block (instantiation) to run; Bp packed for it
    if (op.version == 3) {
        BBMM_REQUIRE(mode == 0, "k2tc: stored K has no derivative mode");
        return k2tc_matmul(ctx, op.Kq, Bp, S, c, n, nloc, s, Vpart, cap, ev0, ev1);
    }
    if (op.kind == BBMM_MATERN52) {
        BBMM_REQUIRE(mode == 0, "k1tc2: no Matern derivative mode");
        mode = op.grid31 ? 4 : 2;
    }
    if (mode == 0 && op.grid31) mode = 3;   // the blackbox matmul on the 31-bit k~ grid
    if (op.nch > 1 && c == op.cb) {      // column chunks (tc_pack layout; mbcg and derivative)
        const size_t stride = (size_t)op.npad * tc_bslice_rows(op.cb, tc_dslices(op));
        int sp = 0;
        for (int z = 0; z < op.nch; z++)
            sp = k1tc2_matmul(ctx, op.Xa, op.XB, Bp + z * stride, S + z * op.cb, op.d, c, n, r0,
                              nloc, s, Vpart, cap, z == 0 ? ev0 : nullptr,
                              z + 1 == op.nch ? ev1 : nullptr, mode, tc_vstride(op), z * op.cb);
        return sp;
    }
    return k1tc2_matmul(ctx, op.Xa, op.XB, Bp, S, op.d, c, n, r0, nloc, s, Vpart, cap, ev0, ev1,
                        mode);
}

}  // namespace bbmm
