// deriv_tc2.cu -- the RBF-ARD derivative pass (row a9, reading R17)
// as tensor-core matrix products: one pass over the pairs, ~2.5 tf32 MMAs per pair-tile and
// one exp + five FP32 ops per pair on the CUDA cores (deriv_tc.cu: ~110 FP32 ops per pair).
//
// For every input dimension q the derivative sums are (scaled inputs x~, k~ = K / s,
// W_ab = A_a . B_b the rank-c weight of deriv.cu's header)
//   S_q = sum_{a,b} k~_ab W_ab (x~_aq - x~_bq)^2 ,   S_s = sum_{a,b} k~_ab W_ab .
// With M = k~ o W (elementwise) the square expands:
//   S_q = sum_a x~_aq^2 (M 1)_a  -  2 sum_a x~_aq (M x~)_aq  +  sum_b x~_bq^2 (M^T 1)_b .
// The first two terms come from ONE contraction of M with the augmented inputs
// b_j = [x~_j, 1, -|x~_j|^2] -- exactly K1-TC's distance operand (the B' tiles), read
// here MN-major as the B of a kind::tf32 MMA whose A is M itself, written to TMEM by the
// compute warps (3xTF32: M_hi x [b_hi | b_lo] + M_lo x b_hi).  The third needs the column
// sums M^T 1 = B o (K~ A), and K A = K U (columns permuted) = B_blk - sigma^2 U - R by the
// mBCG residual identity (reading R25): an O(n c) pass, no pair work.
//
// Per 128-row x 64-point stage: S = the 3xTF32 distance MMA (K1-TC's A' / B'), W = the
// 3xTF32 weight MMA (deriv_tc.cu's A' / B'), both into TMEM; compute warps: k~ = ex2(S),
// m = k~ W, split m -> (m_hi, m_lo) over the S / W columns; then the M x b MMAs accumulate
// (fp32, TMEM) into 64 columns drained to fp64 every 32 stages.
// CTA = 128 rows (TMEM lanes), 10 warps: 8 compute (lane quarter w % 4, 32-point half w / 4
// of a stage), 1 producer (bulk copies of the stage's b and B tiles), 1 MMA issuer.
// TMEM: 2 stage buffers x (64 S + 64 W) columns + 64 accumulator columns.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"
#include "sm100_ptx.cuh"

namespace bbmm {
namespace dtc2 {

constexpr int BM = 128, BJ = 64;               // rows per CTA, points per stage
constexpr int NCW = 8, kThreads = 32 * (NCW + 2);
constexpr int PRODUCER_WARP = NCW, MMA_WARP = NCW + 1;
constexpr int NBUF = 2;                        // TMEM stage buffers (64 S + 64 W columns each)
constexpr int RA = 3, RB = 3;                  // shared-memory ring stages: (b, B) and b^T
constexpr int ACC_OFF = NBUF * 2 * BJ;         // 64 accumulator columns
constexpr int AS_TM = ACC_OFF + 64;            // A'_S in TMEM: 3 DA columns
constexpr int WST = 32;                        // stages per accumulator window (2048 points)

template <int DA, int CA>
struct Cfg {
    static constexpr int XB_BYTES = 2 * DA * BJ * 4;     // b  [hi | lo], K = dims: [2DA/4][64 j][4]
    static constexpr int WB_BYTES = 2 * CA * BJ * 4;     // B  [hi | lo], K = columns
    static constexpr int XT_BYTES = 2 * DA * BJ * 4;     // b^T, K = points: [64 j/4][2DA rows][4]
    static constexpr int STAGE_A = XB_BYTES + WB_BYTES;
    static constexpr int AW_BYTES = BM * 3 * CA * 4;     // A'_W = [hi | hi | lo] of A_i
    static constexpr int RB_OFF = RA * STAGE_A, AW_OFF = RB_OFF + RB * XT_BYTES;
    static constexpr int SMEM = AW_OFF + AW_BYTES + 1024;
    static_assert(SMEM <= 227 * 1024, "shared memory budget");
    static_assert(2 * DA <= 64 && AS_TM + 3 * DA <= 512, "TMEM budget");
};

// Per 64-point stage st: b_j = [x~_j (d), 1, e_j = -|x~_j|^2, 0..] split [hi | lo] (from K1-TC's
// row operand Xa_j = [2 x~_j, e_j, 1, 0..]; zero past n) in two layouts -- XB: K = dims (the
// distance MMA's B), XT: K = points (the B of M x b) -- and W's B tile from B32.
__global__ void k_prep_stage64(const float *__restrict__ Xa, int DA, int d, const float *__restrict__ B32,
                               int cs, int c, int CA, int64_t n, int64_t nstages,
                               float *__restrict__ XB, float *__restrict__ XT, float *__restrict__ WB) {
    const int64_t total = nstages * BJ;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t st = j / BJ;
        const int jj = (int)(j - st * BJ);
        float *xb = XB + st * (int64_t)(2 * DA * BJ), *xt = XT + st * (int64_t)(2 * DA * BJ);
        for (int q = 0; q < DA; q++) {
            float b = 0.0f;
            if (j < n) b = q < d ? 0.5f * Xa[j * DA + q] : q == d ? 1.0f : q == d + 1 ? Xa[j * DA + d] : 0.0f;
            const float bh = tf32_rn(b), bl = tf32_rn(b - bh);
            xb[(q >> 2) * (BJ * 4) + jj * 4 + (q & 3)] = bh;
            xb[((DA + q) >> 2) * (BJ * 4) + jj * 4 + (q & 3)] = bl;
            xt[(jj >> 2) * (2 * DA * 4) + q * 4 + (jj & 3)] = bh;
            xt[(jj >> 2) * (2 * DA * 4) + (DA + q) * 4 + (jj & 3)] = bl;
        }
        float *wb = WB + st * (int64_t)(2 * CA * BJ);
        for (int q = 0; q < CA; q++) {
            const float b = (j < n && q < c) ? B32[j * cs + q] : 0.0f;
            const float bh = tf32_rn(b), bl = tf32_rn(b - bh);
            wb[(q >> 2) * (BJ * 4) + jj * 4 + (q & 3)] = bh;
            wb[((CA + q) >> 2) * (BJ * 4) + jj * 4 + (q & 3)] = bl;
        }
    }
}

template <int D, int DA, int CA>
__global__ void __launch_bounds__(kThreads, 1)
k_deriv_tc2(const float *__restrict__ Xa, const float *__restrict__ A32, int csa,
            const float *__restrict__ XB, const float *__restrict__ XT, const float *__restrict__ WB,
            int64_t r0, int64_t nloc, int64_t stages_per_split, int64_t nstages,
            double *__restrict__ part) {
    using K = Cfg<DA, CA>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_a[RA], free_a[RA], full_b[RB], free_b[RB];
    __shared__ __align__(8) uint64_t s_full[NBUF], m_full[NBUF], acc_full, acc_empty, init_done;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double red_sh[NCW * 32];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t s0 = (int64_t)blockIdx.y * stages_per_split;
    const int ns = (int)(min(nstages, s0 + stages_per_split) - s0);

    if (tid == 0) {
        for (int q = 0; q < RA; q++) {
            ptx::mbar_init(&full_a[q], 1);
            ptx::mbar_init(&free_a[q], 1);
        }
        for (int q = 0; q < RB; q++) {
            ptx::mbar_init(&full_b[q], 1);
            ptx::mbar_init(&free_b[q], 1);
        }
        for (int q = 0; q < NBUF; q++) {
            ptx::mbar_init(&s_full[q], 1);
            ptx::mbar_init(&m_full[q], NCW);
        }
        ptx::mbar_init(&acc_full, 1);
        ptx::mbar_init(&acc_empty, NCW);
        ptx::mbar_init(&init_done, NCW);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tmem_base_sh);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    double out[D + 1];
#pragma unroll
    for (int q = 0; q <= D; q++) out[q] = 0.0;

    if (warp == PRODUCER_WARP) {
        // two rings in consumption order: (b, B) of stage s feeds the distance / weight MMAs
        // (issued NBUF stages ahead), b^T of stage s the M x b MMAs
        if (ptx::elect_one()) {
            auto load_a = [&](int s) {
                const int st = s % RA;
                ptx::mbar_wait(&free_a[st], (uint32_t)(((s / RA) & 1) ^ 1));
                uint8_t *sb = smem + st * K::STAGE_A;
                const int64_t sg = s0 + s;
                ptx::mbar_arrive_expect_tx(&full_a[st], K::STAGE_A);
                ptx::bulk_g2s(sb, reinterpret_cast<const uint8_t *>(XB) + sg * K::XB_BYTES,
                              K::XB_BYTES, &full_a[st]);
                ptx::bulk_g2s(sb + K::XB_BYTES, reinterpret_cast<const uint8_t *>(WB) + sg * K::WB_BYTES,
                              K::WB_BYTES, &full_a[st]);
            };
            auto load_b = [&](int s) {
                const int st = s % RB;
                ptx::mbar_wait(&free_b[st], (uint32_t)(((s / RB) & 1) ^ 1));
                ptx::mbar_arrive_expect_tx(&full_b[st], K::XT_BYTES);
                ptx::bulk_g2s(smem + K::RB_OFF + st * K::XT_BYTES,
                              reinterpret_cast<const uint8_t *>(XT) + (s0 + s) * K::XT_BYTES,
                              K::XT_BYTES, &full_b[st]);
            };
            for (int s = 0; s < NBUF && s < ns; s++) load_a(s);
            for (int s = 0; s < ns; s++) {
                load_b(s);
                if (s + NBUF < ns) load_a(s + NBUF);
            }
        }
        __syncwarp();
    } else if (warp == MMA_WARP) {
        constexpr uint32_t IDSW = ptx::idesc_tf32(BM, BJ);
        constexpr uint32_t IDX = ptx::idesc_tf32(BM, 2 * DA);
        constexpr uint32_t IDXH = ptx::idesc_tf32(BM, DA);
        const bool leader = ptx::elect_one();
        ptx::mbar_wait(&init_done, 0);
        ptx::tc_fence_after();
        const uint32_t aw = ptx::smem_u32(smem + K::AW_OFF);
        // distance + weight MMAs of stage s into buffer s % NBUF
        auto issue_sw = [&](int s) {
            const int st = s % RA, b = s % NBUF;
            ptx::mbar_wait(&full_a[st], (uint32_t)((s / RA) & 1));
            ptx::tc_fence_after();
            if (leader) {
                const uint32_t xb = ptx::smem_u32(smem + st * K::STAGE_A), wb = xb + K::XB_BYTES;
#pragma unroll
                for (int ks = 0; ks < 3 * DA / 8; ks++) {   // S = A'_S (TMEM) x b^T
                    const int g = ks / (DA / 8), kk = ks % (DA / 8);
                    const int kb = (g == 1 ? DA / 8 : 0) + kk;
                    ptx::mma_tf32_ts(tmem + b * 2 * BJ, tmem + AS_TM + 8 * ks,
                                     ptx::smem_desc_kmajor(xb + kb * 2 * BJ * 16, BJ * 16, 128), IDSW,
                                     ks > 0 ? 1u : 0u);
                }
#pragma unroll
                for (int ks = 0; ks < 3 * CA / 8; ks++) {   // W = A'_W x B^T
                    const int g = ks / (CA / 8), kk = ks % (CA / 8);
                    const int kb = (g == 1 ? CA / 8 : 0) + kk;
                    ptx::mma_tf32_ss(tmem + b * 2 * BJ + BJ,
                                     ptx::smem_desc_kmajor(aw + ks * 2 * BM * 16, BM * 16, 128),
                                     ptx::smem_desc_kmajor(wb + kb * 2 * BJ * 16, BJ * 16, 128), IDSW,
                                     ks > 0 ? 1u : 0u);
                }
                ptx::mma_commit(&s_full[b]);
                ptx::mma_commit(&free_a[st]);
            }
            __syncwarp();
        };
        for (int s = 0; s < NBUF && s < ns; s++) issue_sw(s);
        for (int s = 0; s < ns; s++) {
            const int st = s % RB, b = s % NBUF, win = s / WST;
            if (s % WST == 0 && win > 0) ptx::mbar_wait(&acc_empty, (uint32_t)((win - 1) & 1));
            ptx::mbar_wait(&m_full[b], (uint32_t)((s / NBUF) & 1));
            ptx::mbar_wait(&full_b[st], (uint32_t)((s / RB) & 1));
            ptx::tc_fence_after();
            if (leader) {
                // acc[:, 0:2DA] += M_hi x [b_hi | b_lo] ; acc[:, 0:DA] += M_lo x b_hi (b^T tile:
                // K = points, 4-point core-matrix chunks 2 DA x 16 bytes apart)
                const uint32_t xt = ptx::smem_u32(smem + K::RB_OFF + st * K::XT_BYTES);
                const uint32_t mh = tmem + b * 2 * BJ, ml = mh + BJ;
#pragma unroll
                for (int kk = 0; kk < BJ / 8; kk++) {
                    const uint64_t bd = ptx::smem_desc_kmajor(xt + kk * 2 * (2 * DA * 16), 2 * DA * 16, 128);
                    ptx::mma_tf32_ts(tmem + ACC_OFF, mh + 8 * kk, bd, IDX, 1u);
                    ptx::mma_tf32_ts(tmem + ACC_OFF, ml + 8 * kk, bd, IDXH, 1u);
                }
                ptx::mma_commit(&free_b[st]);
                if ((s + 1) % WST == 0 || s + 1 == ns) ptx::mma_commit(&acc_full);
            }
            __syncwarp();
            if (s + NBUF < ns) issue_sw(s + NBUF);   // in order: after the MMAs that read b
        }
    } else {
        // ----------------------------------------------------------- compute
        const int sub = warp & 3, h = warp >> 2;
        const int rl = sub * 32 + lane;
        const int64_t row = (int64_t)blockIdx.x * BM + rl;
        const bool valid = row < nloc;
        const uint32_t lane_base = tmem + ((uint32_t)(sub * 32) << 16);
        if (h == 0) {
            // A'_S = [hi | hi | lo] of a_i = Xa row -> TMEM columns AS_TM.. (this lane quarter)
            uint32_t av[32];
#pragma unroll 1
            for (int k0 = 0; k0 < 3 * DA; k0 += 32) {
#pragma unroll
                for (int u = 0; u < 32; u++) {
                    const int k = k0 + u, q = k % DA, pt = k / DA;
                    const float v = valid ? Xa[(r0 + row) * DA + q] : 0.0f;
                    const float vh = tf32_rn(v);
                    av[u] = __float_as_uint(pt < 2 ? vh : tf32_rn(v - vh));
                }
#pragma unroll
                for (int q = 0; q < 32; q += 8)
                    ptx::tmem_st8(lane_base + AS_TM + k0 + q, *reinterpret_cast<const uint32_t(*)[8]>(av + q));
            }
            float *awp = reinterpret_cast<float *>(smem + K::AW_OFF);
            for (int q = 0; q < CA; q++) {
                const float v = (valid && q < csa) ? A32[row * csa + q] : 0.0f;
                const float vh = tf32_rn(v), vl = tf32_rn(v - vh);
                const float parts[3] = {vh, vh, vl};
#pragma unroll
                for (int pt = 0; pt < 3; pt++) {
                    const int k = pt * CA + q;
                    awp[(k >> 2) * (BM * 4) + rl * 4 + (k & 3)] = parts[pt];
                }
            }
            ptx::fence_proxy_async_smem();
        }
        {   // zero this warp's 32 accumulator columns
            constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int q = 0; q < 32; q += 8) ptx::tmem_st8(lane_base + ACC_OFF + 32 * h + q, z);
            ptx::tmem_st_wait();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&init_done);
        float xr[D];                                   // this row's x~ (zero past d)
#pragma unroll
        for (int q = 0; q < D; q++) xr[q] = valid ? 0.5f * Xa[(r0 + row) * DA + q] : 0.0f;
        int win = 0;
        for (int s = 0; s < ns; s++) {
            const int b = s % NBUF;
            ptx::mbar_wait(&s_full[b], (uint32_t)((s / NBUF) & 1));
            ptx::tc_fence_after();
            uint32_t sv[32], wv[32];
            const uint32_t cs_ = lane_base + b * 2 * BJ + 32 * h;
            ptx::tmem_ld32(cs_, sv);
            ptx::tmem_ld32(cs_ + BJ, wv);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const float m = ex2_approx(__uint_as_float(sv[j])) * __uint_as_float(wv[j]);
                const float mh = tf32_rn(m);
                sv[j] = __float_as_uint(mh);
                wv[j] = __float_as_uint(tf32_rn(m - mh));
            }
#pragma unroll
            for (int q = 0; q < 32; q += 8) {
                ptx::tmem_st8(cs_ + q, *reinterpret_cast<const uint32_t(*)[8]>(sv + q));
                ptx::tmem_st8(cs_ + BJ + q, *reinterpret_cast<const uint32_t(*)[8]>(wv + q));
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&m_full[b]);
            if ((s + 1) % WST == 0 || s + 1 == ns) {
                // drain: warp h owns accumulator columns [32 h, 32 h + 32) = the hi (h = 0) or
                // lo (h = 1) part of every b entry; the fold is linear, so each half adds
                //   S_q += x~_q^2 a_d - 2 x~_q a_q  (q < d),   S_s += a_d
                ptx::mbar_wait(&acc_full, (uint32_t)(win & 1));
                ptx::tc_fence_after();
                uint32_t av[32];
                ptx::tmem_ld32(lane_base + ACC_OFF + 32 * h, av);
                ptx::tmem_ld_wait();
                const double ad = (double)__uint_as_float(av[D]);
#pragma unroll
                for (int q = 0; q < D; q++) {
                    const double x = (double)xr[q];
                    out[q] += x * (x * ad - 2.0 * (double)__uint_as_float(av[q]));
                }
                out[D] += ad;
                constexpr uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int q = 0; q < 32; q += 8) ptx::tmem_st8(lane_base + ACC_OFF + 32 * h + q, z);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty);
                win++;
            }
        }
        if (!valid)
#pragma unroll
            for (int q = 0; q <= D; q++) out[q] = 0.0;
    }
    // fixed-order block reduction of the D + 1 sums over the compute threads
    __syncthreads();
#pragma unroll
    for (int q = 0; q <= D; q++) {
        if (warp < NCW) red_sh[warp * 32 + lane] = out[q];
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int u = 0; u < NCW * 32; u++) s += red_sh[u];
            part[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (D + 1) + q] = s;
        }
        __syncthreads();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

__global__ void k_add_vec(double *__restrict__ a, const double *__restrict__ b, int m) {
    for (int i = threadIdx.x; i < m; i += blockDim.x) a[i] += b[i];
}

// Third term: per local row b, (M^T 1)_b = sum_c B_bc (K~ A)_bc with K A = K U = B_blk -
// sigma^2 U - R (residual identity R25; A = [U_1..U_t, U_0], B = [Z0_1..Z0_t / t, -U_0]);
// out[q] = sum_b x~_bq^2 (M^T 1)_b for q < D (block partials, fixed order).
template <int D>
__global__ void k_term2(const double *__restrict__ U, const double *__restrict__ R,
                        const double *__restrict__ Bblk, const double *__restrict__ Z0,
                        const float *__restrict__ Xa, int DA, int64_t r0, double noise_var,
                        double inv_s, int64_t nloc, int t, double *__restrict__ part) {
    const int c = t + 1;
    const double inv_t = 1.0 / (double)t;
    double acc[D];
#pragma unroll
    for (int q = 0; q < D; q++) acc[q] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double *u = U + i * c, *r = R + i * c, *b = Bblk + i * c, *z = Z0 + i * c;
        double m = 0.0;
        for (int q = 1; q <= t; q++) m += (b[q] - noise_var * u[q] - r[q]) * z[q];
        m = (m * inv_t - u[0] * (b[0] - noise_var * u[0] - r[0])) * inv_s;
#pragma unroll
        for (int q = 0; q < D; q++) {
            const double x = 0.5 * (double)Xa[(r0 + i) * DA + q];
            acc[q] += x * x * m;
        }
    }
    __shared__ double sh[256];
#pragma unroll 1
    for (int q = 0; q < D; q++) {
        sh[threadIdx.x] = acc[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int u = 0; u < (int)blockDim.x; u++) s += sh[u];
            part[(int64_t)blockIdx.x * D + q] = s;
        }
        __syncthreads();
    }
}

}  // namespace dtc2

// ======================================================================
// host side
// ======================================================================
namespace {
struct Dtc2Plan { int64_t rb, sp, sps, nstages; };
Dtc2Plan dtc2_plan(int64_t n, int64_t nloc) {
    Dtc2Plan p;
    p.nstages = ceil_div(n, dtc2::BJ);
    p.rb = ceil_div(std::max<int64_t>(nloc, 1), dtc2::BM);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * kNumSMs, p.rb), p.nstages));
    p.sps = ceil_div(p.nstages, sp);
    p.sp = ceil_div(p.nstages, p.sps);
    return p;
}
int dtc2_ca(int c) { return ((c + 7) / 8) * 8; }
}  // namespace

bool deriv_tc2_supported(int kind, int n_ls, int d, int dp, int c, int64_t n) {
    if (std::getenv("BBMM_NO_DERIV_TC2") || std::getenv("BBMM_NO_DERIV_TC")) return false;
    const char *mn = std::getenv("BBMM_DERIV_TC_MIN_N");
    if (n < (mn ? atoll(mn) : 16384)) return false;
    // instantiated: d = 26 (C3), c <= 40 columns of the weight operand
    return kind == BBMM_RBF && n_ls == d && n_ls > 1 && dp == 26 && d == 26 && dtc2_ca(c) <= 40;
}

size_t deriv_tc2_part_elems(int64_t n, int64_t nloc, int dp) {
    const Dtc2Plan p = dtc2_plan(n, nloc);
    const int nb2 = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(nloc, 1), 256), 2 * kNumSMs));
    return std::max<size_t>((size_t)(p.rb * p.sp) * (dp + 1), (size_t)nb2 * dp);
}

// S_q (q < dp) and S_s (at dp) of the RBF-ARD derivative pass into red[0..dp] (summed over
// this rank's rows; the caller all-reduces).  Xa: K1-TC's row operand (DA = 32), U, R, Bblk, Z0:
// the mBCG solves, recurrence residuals, right-hand sides and P^-1 B (local rows).
void derivative_pass_tc2(bbmm_ctx_s *ctx, const float *Xa, int d, int dp, int64_t n, int64_t r0,
                         int64_t nloc, const float *A32, const float *B32, int cs, int c,
                         const double *U, const double *R, const double *Bblk, const double *Z0,
                         double noise_var, double s, double *part, double *red) {
    constexpr int D = 26, DA = 32, CA = 40;
    using K = dtc2::Cfg<DA, CA>;
    BBMM_REQUIRE(dp == D && d == D && dtc2_ca(c) <= CA, "deriv_tc2: unsupported shape");
    const Dtc2Plan p = dtc2_plan(n, nloc);
    float *XB = (float *)ctx->ws.get("dtc2_XB", (size_t)p.nstages * K::XB_BYTES);
    float *XT = (float *)ctx->ws.get("dtc2_XT", (size_t)p.nstages * K::XT_BYTES);
    float *WB = (float *)ctx->ws.get("dtc2_WB", (size_t)p.nstages * K::WB_BYTES);
    const int pg = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.nstages * dtc2::BJ, 256),
                                                               8 * kNumSMs));
    dtc2::k_prep_stage64<<<pg, 256, 0, ctx->stream>>>(Xa, DA, d, B32, cs, c, CA, n, p.nstages, XB,
                                                      XT, WB);
    ctx->launches++;
    const int nblk = (int)(p.rb * p.sp);
    if (nloc > 0) {
        static DeviceOnce attr;
        attr(ctx->device, [] {
            BBMM_CUDA(cudaFuncSetAttribute(dtc2::k_deriv_tc2<D, DA, CA>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
        });
        dim3 grid((unsigned)p.rb, (unsigned)p.sp);
        dtc2::k_deriv_tc2<D, DA, CA><<<grid, dtc2::kThreads, K::SMEM, ctx->stream>>>(
            Xa, A32, cs, XB, XT, WB, r0, nloc, p.sps, p.nstages, part);
        BBMM_LAUNCH_CHECK();
        ctx->launches++;
        reduce_blocks(ctx, part, nblk, dp + 1, red);
        // + sum_b x~_bq^2 (M^T 1)_b from the residual identity
        const int nb2 = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 256), 2 * kNumSMs));
        double *part2 = (double *)ctx->ws.get("dtc2_part2", (size_t)nb2 * dp * 8);
        double *red2 = (double *)ctx->ws.get("dtc2_red2", (size_t)dp * 8);
        dtc2::k_term2<D><<<nb2, 256, 0, ctx->stream>>>(U, R, Bblk, Z0, Xa, DA, r0, noise_var,
                                                       1.0 / s, nloc, c - 1, part2);
        reduce_blocks(ctx, part2, nb2, dp, red2);
        dtc2::k_add_vec<<<1, 64, 0, ctx->stream>>>(red, red2, dp);
        ctx->launches += 2;
        BBMM_LAUNCH_CHECK();
    } else {
        BBMM_CUDA(cudaMemsetAsync(red, 0, (size_t)(dp + 1) * 8, ctx->stream));
    }
}

}  // namespace bbmm
