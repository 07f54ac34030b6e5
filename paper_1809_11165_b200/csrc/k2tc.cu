// k2tc.cu -- stored-K kernel-matmul on the int8 tensor cores (K2-TC).
//
// The stored variant of the blackbox matmul V = K D (north
// star item 2: "a stored-K variant for n where K fits in HBM, with vectorised,
// coalesced streaming of K per iteration"; PAPER.md:706-708 counts one MMM
// with K per mBCG iteration).  K is materialised ONCE per call, already in the
// exact fixed-point form of the K1-TC contraction, with one
// more slice because K is built once (and the fp32 kernel values then keep all
// their bits):
//   k~ = K/s in [0, 1]  ->  round(k~ 2^30), four u8 slices q0 (low) .. q3
// i.e. 4 bytes per entry like fp32, laid out tile by tile exactly as the
// tcgen05 MMA reads its A operand from shared memory.  (Three slices, i.e.
// 22-bit k~ as on the fly, measured 1.4e-4 solve error against the oracle at
// the C2 shape, n = 3000: over the 1e-4 bar where mBCG is not converged.)  Every mBCG
// iteration then streams the slices from HBM with bulk copies (TMA engine) and
// contracts them with the packed search directions (k1tc.cu format with seven
// u8 slices p6..p0: D as 55-bit fixed point per column) on the int8 tensor
// cores with exact uint32 accumulation in TMEM.  The kernel is bound by HBM
// (4 n_loc n bytes per K D); the tensor work (28 slice products) stays below
// the HBM time.  Why 55 bits of D (K1-TC uses 31): where mBCG is not yet
// converged at p ("regime B") the iterates amplify per-iteration
// rounding of D -- an fp64 emulation at the C2 shape (n = 3000, p = 20) moves the
// solves by 1.3e-4 with 31-bit D and by 2.9e-6 with 39-bit D, and at n = 12 000
// (relres 0.04) even 47-bit D moves them by 2.2e-4: 55 bits put the
// rounding of D at the level of an fp64 product (2^-55 of the column maximum).
//
// CTA (persistent, one per SM, 192 threads):
//   warps 0-3: epilogue -- drain a unit's accumulators (TMEM lane quarter w),
//              fold the six weighted blocks into fp64, write Vpart
//   warp 4   : producer -- bulk copies of the K-slice tile (32 KB) and the
//              D-slice tile (NB x 64 B) of each 64-point stage
//   warp 5   : MMA issuer -- tcgen05.mma.kind::i8 of q3 .. q0 times the
//              [p6|..|p0] operand (one MMA per slice group of N <= 256) per
//              32-point K-step
// Work unit = (128-row block, j-split); a split never exceeds the uint32
// accumulation window, so each unit is drained exactly once, into one of two
// TMEM accumulator sets (the MMAs of unit u+1 overlap the drain of unit u).
#include <algorithm>
#include <cmath>

#include "bbmm_internal.cuh"
#include "k1_kernels.cuh"
#include "pair_common.cuh"
#include "sm100_ptx.cuh"

namespace bbmm {
namespace k2tc {

constexpr int BM = 128;                    // rows per unit (TMEM lanes)
constexpr int SK = 64;                     // j points per pipeline stage
constexpr int NQ = 4;                      // K slices (30-bit fixed point)
constexpr int ND = 7;                      // D slices (55-bit fixed point, k1tc_pack nd = 7)
constexpr int SLICE_BYTES = BM * SK;       // one u8 slice of a tile: [SK/16][BM][16 B]
constexpr int A_BYTES = NQ * SLICE_BYTES;  // q0 | q1 | q2 | q3
// uint32 accumulation bound: block k collects q_a p_b with a + b = NBLK - 1 - k
// (at most NQ = 4 pairs); all bytes <= 255, q3 <= 0x40, p6 <= 0x80, so the
// largest per-point block sum is 64*255 + 3*255*255 = 211395 -> < 20317 points
// per window.
constexpr int BLOCK_MAX = 211395;
constexpr int WINDOW = (int)(4294967295ull / BLOCK_MAX) / SK * SK;
static_assert((double)WINDOW * BLOCK_MAX < 4294967296.0, "uint32 window bound");
constexpr int kThreads = 192;
constexpr int PRODUCER_WARP = 4, MMA_WARP = 5;

constexpr __host__ __device__ int r32(int x) { return (x + 31) & ~31; }
constexpr __host__ __device__ int pow2_cols(int x) {
    return x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : x <= 256 ? 256 : 512;
}

template <int C>
struct Cfg {
    static constexpr int C1 = C + 1;            // + constant offset column
    static_assert(C1 <= 48, "too many columns");
    static constexpr int BLK = (C1 + 15) & ~15; // N = ND BLK must be a multiple of 16
    static constexpr int NB = ND * BLK;         // B rows: [p6 | p5 | .. | p0]
    static constexpr int G = (256 / BLK) < ND ? (256 / BLK) : ND;   // D slices per MMA (N <= 256)
    static_assert((G * BLK) % 16 == 0 && ((ND % G) * BLK) % 16 == 0, "MMA N");
    static constexpr int NBLK = NQ + ND - 1;    // accumulator blocks
    static constexpr int ACC_COLS = NBLK * BLK; // block k has weight 2^(8 (NBLK - 1 - k))
    static constexpr int ACC_END = r32(ACC_COLS);
    static constexpr int NSET = 2 * ACC_END <= 512 ? 2 : 1;
    static constexpr int TMEM_COLS = pow2_cols(NSET * ACC_END);
    static constexpr int B_BYTES = NB * SK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES_FIT = (227 * 1024 - 2048) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT < 8 ? STAGES_FIT : 8;
    static_assert(STAGES >= 3, "shared-memory ring too shallow");
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;
};

// --------------------------------------------------------------------------
// Build: Kq tile (rb, t) = the four u8 slices of round(k~ 2^30) for rows
// rb*128.. and points t*SK.. (zeros past n_loc / n), K-major core-matrix
// layout [slice][SK/16 chunks][128 rows][16 B].  Thread = row.  The kernel
// values are evaluated in fp64 from the fp32 inputs (the method's definition,
// readings R1/R2: r^2 = sum_q ((x_iq - x_jq)/l_q)^2, k~ = exp(-r^2/2) or
// (1 + sqrt5 r + 5r^2/3) exp(-sqrt5 r)), so the 2^-31 fixed-point rounding is
// the only error of the stored operator: an fp32 distance alone perturbs K by
// ~1e-7 relative, which an unconverged mBCG amplifies past the 1e-4 solve bar
// (C2 full size: 4.1e-4 with fp32 distances).  K is built once
// per call, so the fp64 work (about 60 DFMA-pipe ops per entry) is paid once,
// not per iteration.
// --------------------------------------------------------------------------
struct InvLs {
    double v[kMaxDim];   // 1 / l_q (ARD) or 1 / l repeated, 0 past d
};

// exp(x) for x <= 0 in fp64 without libdevice's special-case paths: x = k ln2 + r (Cody-Waite,
// |r| <= ln2 / 2), exp(r) by its Taylor polynomial of degree 10 (truncation < 3e-13 relative),
// times 2^k through the exponent field; 0 below -708 (far under the 2^-30 grid of the stored K).
// The stored kernel values are rounded to 30-bit fixed point, so this keeps them exact to the
// grid while costing ~13 fp64 FMA-pipe ops instead of the general exp's range checks.
__device__ __forceinline__ double exp_nonpos(double x) {
    if (x < -708.0) return 0.0;
    const double kd = rint(x * 1.4426950408889634);
    double r = fma(kd, -6.93147180369123816490e-01, x);
    r = fma(kd, -1.90821492927058770002e-10, r);
    double p = 2.7557319223985893e-07;                 // 1/10!
    p = fma(p, r, 2.7557319223985888e-06);             // 1/9!
    p = fma(p, r, 2.4801587301587302e-05);             // 1/8!
    p = fma(p, r, 1.9841269841269841e-04);             // 1/7!
    p = fma(p, r, 1.3888888888888889e-03);             // 1/6!
    p = fma(p, r, 8.3333333333333332e-03);             // 1/5!
    p = fma(p, r, 4.1666666666666664e-02);             // 1/4!
    p = fma(p, r, 1.6666666666666666e-01);             // 1/3!
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    return p * __longlong_as_double((long long)((int)kd + 1023) << 52);
}

template <int KIND, int D>
__global__ void __launch_bounds__(BM)
k_build_kq64(const float *__restrict__ X, int d, InvLs il, int64_t n, int64_t r0, int64_t nloc,
             int64_t ntiles, uint8_t *__restrict__ Kq) {
    __shared__ double xj_s[SK][D];
    const int64_t t = blockIdx.x, rb = blockIdx.y;
    const int rl = threadIdx.x;
    const int64_t i = rb * BM + rl;
    for (int e = threadIdx.x; e < SK * D; e += BM) {
        const int jj = e / D, q = e % D;
        const int64_t j = t * SK + jj;
        xj_s[jj][q] = (j < n && q < d) ? (double)X[j * d + q] * il.v[q] : 0.0;
    }
    double xi[D];
    const bool vi = i < nloc;
#pragma unroll
    for (int q = 0; q < D; q++) xi[q] = (vi && q < d) ? (double)X[(r0 + i) * d + q] * il.v[q] : 0.0;
    __syncthreads();
    uint8_t *tile = Kq + (rb * ntiles + t) * (int64_t)A_BYTES;
#pragma unroll 1
    for (int ch = 0; ch < SK / 16; ch++) {
        uint32_t w[NQ][4];
#pragma unroll
        for (int g = 0; g < 4; g++) {
            uint32_t q[4];
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const int jj = ch * 16 + 4 * g + v;
                const int64_t j = t * SK + jj;
                double r2 = 0.0;
#pragma unroll
                for (int qd = 0; qd < D; qd++) {
                    const double df = xi[qd] - xj_s[jj][qd];
                    r2 = fma(df, df, r2);
                }
                double kv = 0.0;
                if (vi && j < n) {
                    if (r0 + i == j) {
                        kv = 1.0;                        // K_ii = s exactly
                    } else if (KIND == 0) {
                        kv = exp_nonpos(-0.5 * r2);
                    } else {
                        const double sr = sqrt(5.0 * r2);
                        kv = (1.0 + sr + (5.0 / 3.0) * r2) * exp_nonpos(-sr);
                    }
                }
                q[v] = __double2uint_rn(kv * 1073741824.0);
            }
#pragma unroll
            for (int a = 0; a < NQ; a++) {
                // byte a of each of the four words, in point order
                const uint32_t lo = __byte_perm(q[0], q[1], a | ((a + 4) << 4));
                const uint32_t hi = __byte_perm(q[2], q[3], a | ((a + 4) << 4));
                w[a][g] = __byte_perm(lo, hi, 0x5410);
            }
        }
#pragma unroll
        for (int a = 0; a < NQ; a++) {
            uint4 *dst = reinterpret_cast<uint4 *>(tile + a * SLICE_BYTES + (ch * BM + rl) * 16);
            *dst = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
        }
    }
}

// --------------------------------------------------------------------------
// V (split s of unit u) = s_out * S_c * sum_j k~_ij (P'_jc - 2^54) 2^-84
// --------------------------------------------------------------------------
template <int C>
__global__ void __launch_bounds__(kThreads, 1)
k2tc_stored(const uint8_t *__restrict__ Kq, const uint8_t *__restrict__ Bpack,
            const double *__restrict__ Sc, int64_t nloc, int64_t rbs, int64_t ntiles, int sp,
            int64_t tps, double s, double *__restrict__ Vpart) {
    using K = Cfg<C>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_b[K::STAGES], free_b[K::STAGES];
    __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2], init_done;
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t U = rbs * sp;

    if (tid == 0) {
        for (int q = 0; q < K::STAGES; q++) {
            ptx::mbar_init(&full_b[q], 1);
            ptx::mbar_init(&free_b[q], 1);
        }
        for (int q = 0; q < 2; q++) {
            ptx::mbar_init(&acc_full[q], 1);
            ptx::mbar_init(&acc_empty[q], 4);     // one elected lane per epilogue warp
        }
        ptx::mbar_init(&init_done, 4);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<K::TMEM_COLS>(&tmem_base_sh);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == PRODUCER_WARP) {
        // ------------------------------------------------------------ producer
        if (ptx::elect_one()) {
            const uint64_t pol = ptx::policy_evict_first();   // K slices are read once
            int64_t it = 0;
            for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
                const int64_t rb = u / sp, t0 = (u % sp) * tps, t1 = min(ntiles, t0 + tps);
                for (int64_t t = t0; t < t1; t++, it++) {
                    const int st = (int)(it % K::STAGES);
                    ptx::mbar_wait(&free_b[st], (uint32_t)(((it / K::STAGES) & 1) ^ 1));
                    uint8_t *sb = smem + st * K::STAGE_BYTES;
                    ptx::mbar_arrive_expect_tx(&full_b[st], K::STAGE_BYTES);
                    ptx::bulk_g2s_hint(sb, Kq + (rb * ntiles + t) * (int64_t)A_BYTES, A_BYTES,
                                       &full_b[st], pol);
                    ptx::bulk_g2s(sb + A_BYTES, Bpack + t * (int64_t)K::B_BYTES, K::B_BYTES,
                                  &full_b[st]);
                }
            }
        }
        __syncwarp();
    } else if (warp == MMA_WARP) {
        // --------------------------------------------------------- MMA issuer
        constexpr uint32_t IDQ = ptx::idesc_i8(BM, K::G * K::BLK, false, false);
        constexpr int GR = ND % K::G;                 // slices of the last, partial group
        constexpr uint32_t IDR = ptx::idesc_i8(BM, (GR ? GR : 1) * K::BLK, false, false);
        const bool leader = ptx::elect_one();
        ptx::mbar_wait(&init_done, 0);
        ptx::tc_fence_after();
        int64_t it = 0;
        int uc = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, uc++) {
            const int64_t t0 = (u % sp) * tps, t1 = min(ntiles, t0 + tps);
            const int set = uc % K::NSET;
            if (uc >= K::NSET) ptx::mbar_wait(&acc_empty[set], (uint32_t)(((uc / K::NSET) - 1) & 1));
            ptx::tc_fence_after();
            const uint32_t acc = tmem + set * K::ACC_END;
            for (int64_t t = t0; t < t1; t++, it++) {
                const int st = (int)(it % K::STAGES);
                ptx::mbar_wait(&full_b[st], (uint32_t)((it / K::STAGES) & 1));
                ptx::tc_fence_after();
                if (leader) {
                    const uint32_t sa = ptx::smem_u32(smem + st * K::STAGE_BYTES);
                    const uint32_t sbb = sa + A_BYTES;
#pragma unroll
                    for (int ks = 0; ks < SK / 32; ks++) {
                        const uint32_t kb = sbb + ks * 2 * K::NB * 16;
                        const uint32_t ka = sa + ks * 2 * BM * 16;
                        // q_a (weight 2^(8a)) times D-slice group [p_(ND-1-g0) ..] ->
                        // blocks (NQ - 1 - a) + g0 ..
#pragma unroll
                        for (int a = NQ - 1; a >= 0; a--) {
                            const uint64_t ad = ptx::smem_desc_kmajor(ka + a * SLICE_BYTES, BM * 16, 128);
#pragma unroll
                            for (int g0 = 0; g0 < ND; g0 += K::G)
                                ptx::mma_i8_ss(acc + (NQ - 1 - a + g0) * K::BLK, ad,
                                               ptx::smem_desc_kmajor(kb + g0 * K::BLK * 16,
                                                                     K::NB * 16, 128),
                                               g0 + K::G <= ND ? IDQ : IDR, 1u);
                        }
                    }
                    ptx::mma_commit(&free_b[st]);
                }
                __syncwarp();
            }
            if (leader) ptx::mma_commit(&acc_full[set]);
            __syncwarp();
        }
    } else {
        // ----------------------------------------------------------- epilogue
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        {
            constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 1
            for (int q = 0; q < K::NSET * K::ACC_END; q += 8) ptx::tmem_st8(lane_base + q, z);
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&init_done);
        }
        constexpr int CS = (C + 3) & ~3;
        int uc = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, uc++) {
            const int64_t rb = u / sp;
            const int split = (int)(u % sp);
            const int set = uc % K::NSET;
            ptx::mbar_wait(&acc_full[set], (uint32_t)((uc / K::NSET) & 1));
            ptx::tc_fence_after();
            const uint32_t base = lane_base + set * K::ACC_END;
            double a[C + 1];
#pragma unroll
            for (int c = 0; c <= C; c++) a[c] = 0.0;
#pragma unroll
            for (int q0 = 0; q0 < K::ACC_END; q0 += 32) {
                uint32_t v[32];
                ptx::tmem_ld32(base + q0, v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; e++) {
                    const int col = q0 + e, k = col / K::BLK, c = col % K::BLK;
                    if (col < K::ACC_COLS && c <= C)
                        a[c] = fma(ldexp(1.0, 8 * (K::NBLK - 1 - k)), (double)v[e], a[c]);
                }
            }
            // zero the set for its next unit, then hand it back to the issuer
            {
                constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int q = 0; q < K::ACC_END; q += 8) ptx::tmem_st8(base + q, z);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty[set]);
            }
            const int64_t row = rb * BM + warp * 32 + lane;
            if (row < nloc) {
                double *out = Vpart + ((int64_t)split * nloc + row) * CS;
                const double bs = s * 0x1p-84;     // 2^-30 (k~) x 2^-54 (D)
#pragma unroll
                for (int c = 0; c < C; c++) out[c] = bs * Sc[c] * (a[c] - a[C]);
#pragma unroll
                for (int c = C; c < CS; c++) out[c] = 0.0;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<K::TMEM_COLS>(tmem);
    }
}

struct Plan {
    int64_t rbs, ntiles, tps;
    int sp, grid;
};

// Split the j range so that (a) a split never exceeds the accumulation window
// and (b) the persistent CTAs get balanced work: minimise the tiles of the
// busiest CTA, ceil(units / grid) * tiles_per_split (ties: fewer splits).
static Plan plan(int64_t nloc, int64_t npad) {
    Plan p;
    p.rbs = ceil_div(std::max<int64_t>(nloc, 1), BM);
    p.ntiles = npad / SK;
    const int64_t sp_min = std::max<int64_t>(1, ceil_div(p.ntiles, WINDOW / SK));
    int64_t best = -1, best_sp = sp_min;
    for (int64_t sp = sp_min; sp <= sp_min + 64 && sp <= p.ntiles; sp++) {
        const int64_t tps = ceil_div(p.ntiles, sp);
        const int64_t spr = ceil_div(p.ntiles, tps);          // non-empty splits
        const int64_t U = p.rbs * spr;
        const int64_t g = std::min<int64_t>(U, kNumSMs);
        const int64_t cost = ceil_div(U, g) * tps + 2 * ceil_div(U, g);   // + per-unit drain
        if (best < 0 || cost < best) { best = cost; best_sp = sp; }
    }
    p.tps = ceil_div(p.ntiles, best_sp);
    p.sp = (int)ceil_div(p.ntiles, p.tps);
    p.grid = (int)std::min<int64_t>(p.rbs * p.sp, kNumSMs);
    return p;
}

template <int C>
static int launch(bbmm_ctx_s *ctx, const uint8_t *Kq, const uint8_t *Bp, const double *S,
                  int64_t nloc, int64_t npad, double s, double *Vpart, size_t cap) {
    using K = Cfg<C>;
    const Plan p = plan(nloc, npad);
    BBMM_REQUIRE((size_t)p.sp * nloc * ((C + 3) & ~3) <= cap, "Vpart workspace too small (k2tc)");
    static DeviceOnce attr;
    attr(ctx->device, [] {
        BBMM_CUDA(cudaFuncSetAttribute(k2tc_stored<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       K::SMEM));
    });
    k2tc_stored<C><<<p.grid, kThreads, K::SMEM, ctx->stream>>>(Kq, Bp, S, nloc, p.rbs, p.ntiles,
                                                                p.sp, p.tps, s, Vpart);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    return p.sp;
}

}  // namespace k2tc

// ======================================================================
// host side
// ======================================================================
// instantiated column counts; any c up to 33 runs on the next one (zero-padded columns)
int k2tc_cols(int c) {
    for (int v : {1, 2, 4, 8, 11, 16, 17, 32, 33})
        if (c <= v) return v;
    return 0;
}
bool k2tc_supported(int c) { return k2tc_cols(c) > 0; }

size_t k2tc_vpart_elems(int64_t n, int64_t nloc, int c) {
    const k2tc::Plan p = k2tc::plan(nloc, k1tc_pad_rows(n));
    return (size_t)p.sp * std::max<int64_t>(nloc, 1) * ((c + 3) & ~3);
}

size_t k2tc_kq_bytes(int64_t n, int64_t nloc) {
    return (size_t)ceil_div(std::max<int64_t>(nloc, 1), k2tc::BM) * k2tc::BM *
           (size_t)k1tc_pad_rows(n) * k2tc::NQ;
}

void k2tc_build(bbmm_ctx_s *ctx, const float *X, int d, const Hyper &h, int64_t n, int64_t r0,
                int64_t nloc, uint8_t *Kq) {
    if (nloc <= 0) return;
    const int64_t npad = k1tc_pad_rows(n);
    const int64_t ntiles = npad / k2tc::SK;
    dim3 grid((unsigned)ntiles, (unsigned)ceil_div(nloc, k2tc::BM));
    k2tc::InvLs il{};
    for (int q = 0; q < d; q++) il.v[q] = 1.0 / h.ls[h.n_ls == 1 ? 0 : q];
    const int dp = pad_dim(d);
    if (h.kind == BBMM_RBF) {
        BBMM_DISPATCH_DIMS(dp, (k2tc::k_build_kq64<0, D_><<<grid, k2tc::BM, 0, ctx->stream>>>(
                                   X, d, il, n, r0, nloc, ntiles, Kq)))
    } else {
        BBMM_DISPATCH_DIMS(dp, (k2tc::k_build_kq64<1, D_><<<grid, k2tc::BM, 0, ctx->stream>>>(
                                   X, d, il, n, r0, nloc, ntiles, Kq)))
    }
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
}

TcOperand prepare_operator(bbmm_ctx_s *ctx, bool stored, const float *X, const float *Xs, int dp,
                           int64_t n, int d, int c, const Hyper &h, int64_t r0, int64_t nloc,
                           int64_t npad_rows, float **Kst) {
    *Kst = nullptr;
    if (!stored) return tc_prepare(ctx, X, n, d, c, h, npad_rows);
    TcOperand op;
    if (ctx->matmul_tc && k2tc_supported(c)) {
        uint8_t *kq = (uint8_t *)ctx->ws.get("Kq", k2tc_kq_bytes(n, nloc));
        k2tc_build(ctx, X, d, h, n, r0, nloc, kq);
        op.version = 3;
        op.d = d;
        op.kind = h.kind;
        op.nd = k2tc::ND;
        op.cb = k2tc_cols(c);
        op.npad = k1tc_pad_rows(npad_rows);
        op.Kq = kq;
        return op;
    }
    if (nloc > 0) {
        const int64_t ldk = ((n + 3) / 4) * 4;
        *Kst = (float *)ctx->ws.get("Kst", (size_t)nloc * ldk * 4);
        build_stored_k(ctx, h.kind, Xs, dp, n, r0, nloc, h.s, *Kst);
    }
    return op;
}

int k2tc_matmul(bbmm_ctx_s *ctx, const uint8_t *Kq, const uint8_t *Bp, const double *S, int c,
                int64_t n, int64_t nloc, double s, double *Vpart, size_t cap, cudaEvent_t ev0,
                cudaEvent_t ev1) {
    if (ev0) record_event(ctx, ev0);
    int sp = 1;
    const int64_t npad = k1tc_pad_rows(n);
    if (nloc > 0) {
        switch (c) {
            case 1: sp = k2tc::launch<1>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 2: sp = k2tc::launch<2>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 4: sp = k2tc::launch<4>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 8: sp = k2tc::launch<8>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 11: sp = k2tc::launch<11>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 16: sp = k2tc::launch<16>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 17: sp = k2tc::launch<17>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 32: sp = k2tc::launch<32>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            case 33: sp = k2tc::launch<33>(ctx, Kq, Bp, S, nloc, npad, s, Vpart, cap); break;
            default: throw Error{BBMM_ERR_ARG, "k2tc: unsupported column count"};
        }
    }
    if (ev1) record_event(ctx, ev1);
    return sp;
}

}  // namespace bbmm
