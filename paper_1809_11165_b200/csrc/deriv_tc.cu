// deriv_tc.cu -- the ARD / Matern derivative pass (row a9, PAPER.md:509-519,
// :683, reading R17) with the rank-c bilinear weights on the tensor cores.
//
// Same sums as deriv.cu's k7_deriv (read its header for the algebra):
//   S_q = sum_{a,b} g(r_ab) W_ab dxs_abq^2   (q < d),   S_d = sum_{a,b} k~(r_ab) W_ab
// with W_ab = A_a . B_b (c columns).  k7_deriv spends c FFMA + c shared loads per
// pair on W; here W for a 128 x 128 tile is one tcgen05 MMA (kind::tf32, 3xTF32:
// (A hi, B hi) + (A hi, B lo) + (A lo, B hi), fp32-level products) into TMEM,
// and the compute warps only form the distances, the kernel value and the d + 1
// weighted sums (4 FP32 ops per input dimension per pair).
//
// CTA = 128 rows (TMEM lanes), 10 warps: 8 compute (lane quarter sub = w % 4,
// j-half h = w / 4 of every 128-point tile), 1 producer (bulk copies of the
// B-operand tile and the tile's scaled inputs), 1 MMA issuer.  Two TMEM W
// buffers; a ring of shared-memory stages freed by the MMA (B) and by the
// compute warps (x_j).  fp32 sums per tile, folded into fp64 registers.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "bbmm_internal.cuh"
#include "pair_common.cuh"
#include "sm100_ptx.cuh"

namespace bbmm {
namespace dtc {

constexpr int BM = 128, BK = 128;
#ifndef BBMM_DTC_NCW
#define BBMM_DTC_NCW 8
#endif
constexpr int NCW = BBMM_DTC_NCW;              // compute warps (4 or 8)
constexpr int JPW = BK / (NCW / 4);            // points of a tile per compute warp
constexpr int kThreads = 32 * (NCW + 2);
constexpr int PRODUCER_WARP = NCW, MMA_WARP = NCW + 1;
constexpr int NBUF = 2;                        // TMEM W buffers (128 fp32 columns each)

template <int D, int CA>
struct Cfg {
    static constexpr int DS = round4(D);
    static constexpr int WB_BYTES = 2 * CA * BK * 4;       // B' tile [hi | lo], K-major
    static constexpr int XJ_BYTES = BK * DS * 4;           // scaled inputs of the tile
    static constexpr int STAGE = WB_BYTES + XJ_BYTES;
    static constexpr int AW_BYTES = BM * 3 * CA * 4;       // A' = [hi | hi | lo] (resident)
    static constexpr int STAGES_FIT = (227 * 1024 - 2048 - AW_BYTES) / STAGE;
    static constexpr int STAGES = STAGES_FIT < 3 ? STAGES_FIT : 3;
    static_assert(STAGES >= 2, "shared-memory ring too shallow");
    static constexpr int SMEM = STAGES * STAGE + AW_BYTES + 1024;
};

// B' tiles from B32 (all n points, stride cs): per 128-point tile, K-major
// [2 CA / 4 chunks][128 points][4 floats] of [hi(B_j) | lo(B_j)], and the tile's
// scaled inputs Xs (zero rows past n).
template <int D, int CA>
__global__ void k_prep_deriv_tc(const float *__restrict__ B32, int cs, int c,
                                const float *__restrict__ Xs, int64_t n, int64_t ntiles,
                                float *__restrict__ WB, float *__restrict__ XJ) {
    constexpr int DS = round4(D);
    const int64_t total = ntiles * BK;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tt = j / BK;
        const int jj = (int)(j - tt * BK);
        float *tile = WB + tt * (int64_t)(2 * CA * BK);
        for (int q = 0; q < CA; q++) {
            const float b = (j < n && q < c) ? B32[j * cs + q] : 0.0f;
            const float bh = tf32_rn(b);
            const float bl = tf32_rn(b - bh);
            tile[(q >> 2) * (BK * 4) + jj * 4 + (q & 3)] = bh;
            tile[((CA + q) >> 2) * (BK * 4) + jj * 4 + (q & 3)] = bl;
        }
        for (int q = 0; q < DS; q++) XJ[j * DS + q] = j < n ? Xs[j * DS + q] : 0.0f;
    }
}

template <int KIND, int D, int CA>
__global__ void __launch_bounds__(kThreads, 1)
k_deriv_tc(const float *__restrict__ Xs, const float *__restrict__ A32, int csa,
           const float *__restrict__ WB, const float *__restrict__ XJ, int64_t r0, int64_t nloc,
           int64_t tiles_per_split, int64_t ntiles, double *__restrict__ part) {
    using K = Cfg<D, CA>;
    constexpr int DS = K::DS;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_b[K::STAGES], free_b[K::STAGES];
    __shared__ __align__(8) uint64_t w_full[NBUF], w_empty[NBUF], init_done;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double red_sh[NCW * 32];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
    const int ntl = (int)(min(ntiles, t0 + tiles_per_split) - t0);
    uint8_t *aw_sm = smem + K::STAGES * K::STAGE;

    if (tid == 0) {
        for (int q = 0; q < K::STAGES; q++) {
            ptx::mbar_init(&full_b[q], 1);
            ptx::mbar_init(&free_b[q], 1 + NCW);     // MMA commit (B) + compute warps (x_j)
        }
        for (int q = 0; q < NBUF; q++) {
            ptx::mbar_init(&w_full[q], 1);
            ptx::mbar_init(&w_empty[q], NCW);
        }
        ptx::mbar_init(&init_done, NCW);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<NBUF * BK>(&tmem_base_sh);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    double out[D + 1];
#pragma unroll
    for (int q = 0; q <= D; q++) out[q] = 0.0;

    if (warp == PRODUCER_WARP) {
        if (ptx::elect_one()) {
            for (int t = 0; t < ntl; t++) {
                const int st = t % K::STAGES;
                ptx::mbar_wait(&free_b[st], (uint32_t)(((t / K::STAGES) & 1) ^ 1));
                uint8_t *sb = smem + st * K::STAGE;
                const int64_t tg = t0 + t;
                ptx::mbar_arrive_expect_tx(&full_b[st], K::STAGE);
                ptx::bulk_g2s(sb, reinterpret_cast<const uint8_t *>(WB) + tg * K::WB_BYTES,
                              K::WB_BYTES, &full_b[st]);
                ptx::bulk_g2s(sb + K::WB_BYTES, reinterpret_cast<const uint8_t *>(XJ) + tg * K::XJ_BYTES,
                              K::XJ_BYTES, &full_b[st]);
            }
        }
        __syncwarp();
    } else if (warp == MMA_WARP) {
        constexpr uint32_t IDW = ptx::idesc_tf32(BM, BK);
        const bool leader = ptx::elect_one();
        ptx::mbar_wait(&init_done, 0);
        ptx::tc_fence_after();
        const uint32_t aw = ptx::smem_u32(aw_sm);
        for (int t = 0; t < ntl; t++) {
            const int st = t % K::STAGES, b = t % NBUF;
            ptx::mbar_wait(&full_b[st], (uint32_t)((t / K::STAGES) & 1));
            if (t >= NBUF) ptx::mbar_wait(&w_empty[b], (uint32_t)(((t / NBUF) - 1) & 1));
            ptx::tc_fence_after();
            if (leader) {
                const uint32_t wb = ptx::smem_u32(smem + st * K::STAGE);
#pragma unroll
                for (int ks = 0; ks < 3 * CA / 8; ks++) {
                    const int g = ks / (CA / 8), kk = ks % (CA / 8);
                    const int kb = (g == 1 ? CA / 8 : 0) + kk;
                    const uint64_t bd = ptx::smem_desc_kmajor(wb + kb * 2 * BK * 16, BK * 16, 128);
                    const uint64_t ad = ptx::smem_desc_kmajor(aw + ks * 2 * BM * 16, BM * 16, 128);
                    ptx::mma_tf32_ss(tmem + b * BK, ad, bd, IDW, ks > 0 ? 1u : 0u);
                }
                ptx::mma_commit(&w_full[b]);
                ptx::mma_commit(&free_b[st]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ compute
        const int sub = warp & 3, h = warp >> 2;
        const int rl = sub * 32 + lane;
        const int64_t row = (int64_t)blockIdx.x * BM + rl;
        const bool valid = row < nloc;
        if (h == 0) {
            // A' = [hi | hi | lo] of A_row, K-major [3 CA / 4][128][4]
            float *ap = reinterpret_cast<float *>(aw_sm);
            for (int q = 0; q < CA; q++) {
                const float v = (valid && q < csa) ? A32[row * csa + q] : 0.0f;
                const float vh = tf32_rn(v);
                const float parts[3] = {vh, vh, tf32_rn(v - vh)};
#pragma unroll
                for (int pt = 0; pt < 3; pt++) {
                    const int k = pt * CA + q;
                    ap[(k >> 2) * (BM * 4) + rl * 4 + (k & 3)] = parts[pt];
                }
            }
            ptx::fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&init_done);
        float xi[D];
#pragma unroll
        for (int q = 0; q < D; q++) xi[q] = valid ? Xs[(r0 + row) * DS + q] : 0.0f;
        const uint32_t lane_base = tmem + ((uint32_t)(sub * 32) << 16);
        for (int t = 0; t < ntl; t++) {
            const int st = t % K::STAGES, b = t % NBUF;
            ptx::mbar_wait(&full_b[st], (uint32_t)((t / K::STAGES) & 1));
            ptx::mbar_wait(&w_full[b], (uint32_t)((t / NBUF) & 1));
            ptx::tc_fence_after();
            const float *xj = reinterpret_cast<const float *>(smem + st * K::STAGE + K::WB_BYTES);
#pragma unroll 1
            for (int quarter = 0; quarter < JPW / 16; quarter++) {
                // fp32 sums over 16 pairs, then folded into fp64 (as k7_deriv's FOLD = 16)
                float acc[D + 1];
#pragma unroll
                for (int q = 0; q <= D; q++) acc[q] = 0.0f;
                const int jb = h * JPW + quarter * 16;
                uint32_t wv[16];
                ptx::tmem_ld16(lane_base + b * BK + jb, wv);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int jj = 0; jj < 16; jj++) {     // full unroll: wv stays in registers
                    const float4 *x4 = reinterpret_cast<const float4 *>(xj + (jb + jj) * DS);
                    float dq[D];
                    float r4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                    for (int q4 = 0; q4 < DS / 4; q4++) {
                        const float4 x = x4[q4];
                        const float xs4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int q = 4 * q4 + u;
                            if (q < D) {
                                const float df = xi[q] - xs4[u];
                                dq[q] = df * df;
                                r4[u] += dq[q];
                            }
                        }
                    }
                    const float rs2 = (r4[0] + r4[1]) + (r4[2] + r4[3]);
                    float kv, g;
                    kval_and_dfac<KIND>(rs2, kv, g);
                    const float w = __uint_as_float(wv[jj]);
                    const float gw = g * w;
#pragma unroll
                    for (int q = 0; q < D; q++) acc[q] = fmaf(gw, dq[q], acc[q]);
                    acc[D] = fmaf(kv, w, acc[D]);
                }
#pragma unroll
                for (int q = 0; q <= D; q++) out[q] += (double)acc[q];
            }
            // W buffer and the x_j of this stage are no longer needed
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&w_empty[b]);
                ptx::mbar_arrive(&free_b[st]);
            }
        }
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
        ptx::tmem_dealloc<NBUF * BK>(tmem);
    }
}

}  // namespace dtc

// ======================================================================
// host side
// ======================================================================
namespace {
struct DtcPlan { int64_t rb, sp, tps, ntiles; };
DtcPlan dtc_plan(int64_t n, int64_t nloc) {
    DtcPlan p;
    p.ntiles = ceil_div(n, dtc::BK);
    p.rb = ceil_div(std::max<int64_t>(nloc, 1), dtc::BM);
    int64_t sp = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * kNumSMs, p.rb), p.ntiles));
    p.tps = ceil_div(p.ntiles, sp);
    p.sp = ceil_div(p.ntiles, p.tps);
    return p;
}

template <int KIND, int D, int CA>
int launch_dtc(bbmm_ctx_s *ctx, const float *Xs, int64_t n, int64_t r0, int64_t nloc,
               const float *A32, const float *B32, int cs, int c, double *part) {
    using K = dtc::Cfg<D, CA>;
    const DtcPlan p = dtc_plan(n, nloc);
    float *WB = (float *)ctx->ws.get("dtc_WB", (size_t)p.ntiles * K::WB_BYTES);
    float *XJ = (float *)ctx->ws.get("dtc_XJ", (size_t)p.ntiles * K::XJ_BYTES);
    const int pg = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.ntiles * dtc::BK, 256),
                                                               8 * kNumSMs));
    dtc::k_prep_deriv_tc<D, CA><<<pg, 256, 0, ctx->stream>>>(B32, cs, c, Xs, n, p.ntiles, WB, XJ);
    static DeviceOnce attr;
    attr(ctx->device, [] {
        BBMM_CUDA(cudaFuncSetAttribute(dtc::k_deriv_tc<KIND, D, CA>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
    });
    dim3 grid((unsigned)p.rb, (unsigned)p.sp);
    dtc::k_deriv_tc<KIND, D, CA><<<grid, dtc::kThreads, K::SMEM, ctx->stream>>>(
        Xs, A32, cs, WB, XJ, r0, nloc, p.tps, p.ntiles, part);
    BBMM_LAUNCH_CHECK();
    ctx->launches += 2;
    return (int)(p.rb * p.sp);
}
}  // namespace

bool deriv_tc_supported(int kind, int dp, int cp, int64_t n) {
    // small n: the per-tile pipeline costs more than it saves (C1: 0.15 vs 0.11 ms)
    const char *mn = getenv("BBMM_DERIV_TC_MIN_N");      // tests force small n through it
    if (getenv("BBMM_NO_DERIV_TC") || n < (mn ? atoll(mn) : 16384)) return false;
    if (kind == BBMM_RBF) return (dp == 26 && cp == 33) || (dp == 9 && cp == 17) || (dp == 19 && cp == 11);
    return dp == 9 && cp == 17;
}

size_t deriv_tc_part_elems(int64_t n, int64_t nloc, int dp) {
    const DtcPlan p = dtc_plan(n, nloc);
    return (size_t)(p.rb * p.sp) * (dp + 1);
}

int derivative_pass_tc(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n, int64_t r0,
                       int64_t nloc, const float *A32, const float *B32, int cp, int c,
                       double *part) {
    const int cs = round4(cp);
    if (kind == BBMM_RBF) {
        if (dp == 26 && cp == 33) return launch_dtc<0, 26, 40>(ctx, Xs, n, r0, nloc, A32, B32, cs, c, part);
        if (dp == 9 && cp == 17) return launch_dtc<0, 9, 24>(ctx, Xs, n, r0, nloc, A32, B32, cs, c, part);
        if (dp == 19 && cp == 11) return launch_dtc<0, 19, 16>(ctx, Xs, n, r0, nloc, A32, B32, cs, c, part);
    } else if (dp == 9 && cp == 17) {
        return launch_dtc<1, 9, 24>(ctx, Xs, n, r0, nloc, A32, B32, cs, c, part);
    }
    throw Error{BBMM_ERR_ARG, "deriv_tc: unsupported shape"};
}

}  // namespace bbmm
