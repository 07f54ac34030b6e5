// bbmm_api.cu -- the C-ABI of include/bbmm.h: argument validation, context
// and workspace management, NCCL plumbing, and the orchestration of the
// one-call MLL + gradient ("a single call to mBCG").
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>

#include "bbmm_internal.cuh"

namespace bbmm {

// ------------------------------------------------------------- workspace
void *Workspace::get(const std::string &name, size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    auto it = bufs.find(name);
    if (it != bufs.end()) {
        if (it->second.second >= bytes) return it->second.first;
        BBMM_CUDA(cudaFree(it->second.first));
        bufs.erase(it);
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error{BBMM_ERR_OOM, "cudaMalloc of workspace '" + name + "' (" +
                                      std::to_string(bytes) + " bytes) failed"};
    }
    bufs[name] = {p, bytes};
    return p;
}

void Workspace::release_all() {
    for (auto &kv : bufs) cudaFree(kv.second.first);
    bufs.clear();
}

// row blocks are multiples of 128 so rank boundaries align with the j-tiles of
// the tensor-core operand (k1tc) and the all-gathers.
static RowRange row_partition(int64_t n, int nranks, int rank) {
    RowRange r;
    r.nb = ceil_div(ceil_div(n, nranks), 128) * 128;
    r.r0 = std::min<int64_t>(n, (int64_t)rank * r.nb);
    r.r1 = std::min<int64_t>(n, r.r0 + r.nb);
    return r;
}

RowRange local_rows(const bbmm_ctx_s *ctx, int64_t n) { return row_partition(n, ctx->nranks, ctx->rank); }

Hyper make_hyper(const bbmm_hyper_t *hp, int d) {
    BBMM_REQUIRE(hp != nullptr, "hyper is NULL");
    BBMM_REQUIRE(hp->kind == BBMM_RBF || hp->kind == BBMM_MATERN52, "unknown kernel kind");
    BBMM_REQUIRE(hp->n_ls == 1 || hp->n_ls == d, "n_ls must be 1 or d");
    BBMM_REQUIRE(hp->log_ls_h != nullptr, "log_ls_h is NULL");
    Hyper h;
    h.kind = hp->kind;
    h.n_ls = hp->n_ls;
    for (int q = 0; q < hp->n_ls; q++) {
        BBMM_REQUIRE(std::isfinite(hp->log_ls_h[q]), "non-finite log lengthscale");
        h.ls[q] = std::exp(hp->log_ls_h[q]);
    }
    BBMM_REQUIRE(std::isfinite(hp->log_outputscale) && std::isfinite(hp->log_noise),
                 "non-finite hyperparameter");
    h.s = std::exp(hp->log_outputscale);
    h.noise_var = std::exp(2.0 * hp->log_noise);
    h.sigma = std::exp(hp->log_noise);
    return h;
}

// ------------------------------------------------------------------ comm
namespace {
struct CommSpan {   // pool events bracketing one collective on the context stream
    bbmm_ctx_s *ctx;
    explicit CommSpan(bbmm_ctx_s *c) : ctx(c) { record(); }
    ~CommSpan() {
        try { record(); } catch (...) {}
    }
    void record() {
        comm_events_reserve(ctx, ctx->n_comm_ev + 1);
        record_event(ctx, ctx->comm_events[ctx->n_comm_ev++]);
    }
};
}  // namespace

void comm_timing_reset(bbmm_ctx_s *ctx) { ctx->n_comm_ev = 0; }

double comm_timing_ms(bbmm_ctx_s *ctx) {
    double tot = 0.0;
    for (size_t q = 0; q + 1 < ctx->n_comm_ev; q += 2) {
        float ms = 0.f;
        BBMM_CUDA(cudaEventElapsedTime(&ms, ctx->comm_events[q], ctx->comm_events[q + 1]));
        tot += ms;
    }
    return tot;
}

void allreduce_sum(bbmm_ctx_s *ctx, double *buf, size_t count) {
    if (!has_comm(ctx)) return;
    CommSpan span(ctx);
    if (ctx->local) return local_allreduce_sum(ctx, buf, count);
    BBMM_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
}

void allreduce_max(bbmm_ctx_s *ctx, double *buf, size_t count) {
    if (!has_comm(ctx)) return;
    CommSpan span(ctx);
    if (ctx->local) return local_allreduce_max(ctx, buf, count);
    BBMM_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclMax, ctx->comm, ctx->stream));
}

void allgather_rows(bbmm_ctx_s *ctx, void *buf, size_t bytes_per_rank) {
    if (!has_comm(ctx)) return;
    CommSpan span(ctx);
    if (ctx->local) return local_allgather(ctx, buf, bytes_per_rank);
    char *b = (char *)buf;
    BBMM_NCCL(ncclAllGather(b + (size_t)ctx->rank * bytes_per_rank, b, bytes_per_rank, ncclChar,
                            ctx->comm, ctx->stream));
}

namespace {

// D (fp64, rows [0, rows) of an n x c block, ld) -> the matmul operand Dm
// (fp64 or fp32, stride cs, zero padding columns).
template <typename DT>
__global__ void k_pack_dm(const double *__restrict__ D, int64_t ldd, int64_t rows, int c, int cs,
                          DT *__restrict__ Dm) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cs;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / cs;
        int col = (int)(e - i * cs);
        Dm[i * cs + col] = col < c ? (DT)D[i * ldd + col] : DT(0);
    }
}

// V[i][col] = sum_s Vpart[s][i][col] + sigma^2 D[r0+i][col]
__global__ void k_matmul_finish(const double *__restrict__ Vpart, int splits, int cs, int64_t nloc,
                                int c, double noise_var, const double *__restrict__ D,
                                int64_t ldd, int64_t r0, double *__restrict__ V, int64_t ldv) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * c;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / c;
        int col = (int)(e - i * c);
        double v = 0.0;
        for (int s = 0; s < splits; s++) v += Vpart[((int64_t)s * nloc + i) * cs + col];
        V[i * ldv + col] = v + noise_var * D[(r0 + i) * ldd + col];
    }
}

// Derivative-pass operands: A32 = [U_1..U_t, U_0] (local rows),
// B32 rows at global positions = [Z0_1..Z0_t / t, -U_0] ; stride cs.
__global__ void k_pack_deriv(const double *__restrict__ U, const double *__restrict__ Z0,
                             int64_t nloc, int t, int cs, int64_t r0, float *__restrict__ A32,
                             float *__restrict__ B32) {
    const int c = t + 1;
    const double inv_t = 1.0 / (double)t;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * cs;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / cs;
        int col = (int)(e - i * cs);
        float a = 0.0f, b = 0.0f;
        if (col < t) {
            a = (float)U[i * c + 1 + col];
            b = (float)(Z0[i * c + 1 + col] * inv_t);
        } else if (col == t) {
            a = (float)U[i * c];
            b = (float)(-U[i * c]);
        }
        A32[i * cs + col] = a;
        B32[(r0 + i) * cs + col] = b;
    }
}

// Local scalar terms: out[0] = y^T u0, out[1] = u0^T u0, out[2] = sum_i u_i^T Z0_i
__global__ void k_scalar_terms(const double *__restrict__ U, const double *__restrict__ Z0,
                               const float *__restrict__ y, int64_t r0, int64_t nloc, int t,
                               double *__restrict__ part) {
    const int c = t + 1;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        double u0 = U[i * c];
        a0 += (double)y[r0 + i] * u0;
        a1 += u0 * u0;
        for (int q = 1; q <= t; q++) a2 += U[i * c + q] * Z0[i * c + q];
    }
    __shared__ double sh[3][256];
    sh[0][threadIdx.x] = a0;
    sh[1][threadIdx.x] = a1;
    sh[2][threadIdx.x] = a2;
    __syncthreads();
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int u = 0; u < 256; u++) s += sh[threadIdx.x][u];
        part[blockIdx.x * 3 + threadIdx.x] = s;
    }
}

// Outputscale term without a kernel-matmul (reading R25): with
// Khat = K + sigma^2 I and the mBCG residuals R = B - Khat U (maintained by
// the recurrence), K U = B - sigma^2 U - R, so by symmetry of K
//   S_s = sum_a A_a . (K Bd)_a = (1/t) sum_i (K u_i) . Z0_i - u_0 . (K u_0).
__global__ void k_outputscale_term(const double *__restrict__ U, const double *__restrict__ R,
                                   const double *__restrict__ B, const double *__restrict__ Z0,
                                   double noise_var, int64_t nloc, int t, double *__restrict__ part) {
    const int c = t + 1;
    const double inv_t = 1.0 / (double)t;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double *u = U + i * c, *r = R + i * c, *b = B + i * c, *z = Z0 + i * c;
        double s = 0.0;
        for (int q = 1; q <= t; q++) s += (b[q] - noise_var * u[q] - r[q]) * z[q];
        acc += s * inv_t - u[0] * (b[0] - noise_var * u[0] - r[0]);
    }
    __shared__ double sh[256];
    sh[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < (int)blockDim.x; q++) s += sh[q];
        part[blockIdx.x] = s;
    }
}

// Derivative-pass operand for the tensor-core path: Bd = [Z0_1..Z0_t / t, -u0] (fp64).
__global__ void k_build_bd(const double *__restrict__ U, const double *__restrict__ Z0,
                           int64_t nloc, int t, double *__restrict__ Bd) {
    const int c = t + 1;
    const double inv_t = 1.0 / (double)t;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * c;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / c;
        const int col = (int)(e - i * c);
        Bd[e] = col < t ? Z0[i * c + 1 + col] * inv_t : -U[i * c];
    }
}

// part[blk] = sum over this block's rows a of A_a . V_a, V = sum of split partials,
// A_a = [u_1..u_t, u_0](a) (so that sum_a A_a . (dK B)_a = S = tau - quad).
__global__ void k_deriv_dot(const double *__restrict__ Vpart, int splits, int cs, int64_t nloc,
                            int t, const double *__restrict__ U, double *__restrict__ part) {
    const int c = t + 1;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int col = 0; col < c; col++) {
            double v = 0.0;
            for (int s = 0; s < splits; s++) v += Vpart[((int64_t)s * nloc + i) * cs + col];
            const double av = col < t ? U[i * c + 1 + col] : U[i * c];
            acc += av * v;
        }
    }
    __shared__ double sh[256];
    sh[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int u = 0; u < (int)blockDim.x; u++) s += sh[u];
        part[blockIdx.x] = s;
    }
}

__global__ void k_check_finite(const float *__restrict__ x, int64_t n, int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) atomicExch(bad, 1);
}

int grid_for(int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 8 * kNumSMs));
}

void check_finite(bbmm_ctx_s *ctx, const float *x, int64_t n, const char *what) {
    int *bad = (int *)ctx->ws.get("finite_flag", sizeof(int));
    BBMM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    k_check_finite<<<grid_for(n), 256, 0, ctx->stream>>>(x, n, bad);
    BBMM_LAUNCH_CHECK();
    ctx->launches++;
    int h = 0;
    BBMM_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) throw Error{BBMM_ERR_DATA, std::string("non-finite values in ") + what};
}

struct Timer {
    cudaEvent_t e;
    explicit Timer(cudaStream_t s) {
        BBMM_CUDA(cudaEventCreate(&e));
        BBMM_CUDA(cudaEventRecord(e, s));
    }
    ~Timer() { cudaEventDestroy(e); }
    float since(const Timer &o) const {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, o.e, e);
        return ms;
    }
};

void validate_common(bbmm_ctx_s *ctx, const float *X, int64_t n, int d) {
    BBMM_REQUIRE(ctx != nullptr, "ctx is NULL");
    BBMM_REQUIRE(X != nullptr, "X is NULL");
    BBMM_REQUIRE(n >= 1, "n must be >= 1");
    BBMM_REQUIRE(d >= 1 && d <= kMaxDim, "d must be in [1, 32]");
}

template <typename F>
bbmm_status_t guarded(bbmm_ctx_s *ctx, F &&f) {
    try {
        if (ctx) BBMM_CUDA(cudaSetDevice(ctx->device));
        f();
        return BBMM_OK;
    } catch (const Error &e) {
        if (ctx) ctx->err = e.msg;
        return e.st;
    } catch (const std::exception &e) {
        if (ctx) ctx->err = e.what();
        return BBMM_ERR_CUDA;
    }
}

}  // namespace
}  // namespace bbmm

using namespace bbmm;

extern "C" {

const char *bbmm_version(void) { return "bbmm-b200 0.1 (sm_100a)"; }

bbmm_status_t bbmm_ctx_create(int device, void *cuda_stream, bbmm_ctx_t *out) {
    if (!out) return BBMM_ERR_ARG;
    *out = nullptr;
    bbmm_ctx_s *ctx = new bbmm_ctx_s();
    ctx->device = device;
    bbmm_status_t st = guarded(ctx, [&] {
        if (cuda_stream) {
            ctx->stream = (cudaStream_t)cuda_stream;
        } else {
            BBMM_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
    });
    if (st != BBMM_OK) {
        delete ctx;
        return st;
    }
    *out = ctx;
    return BBMM_OK;
}

bbmm_status_t bbmm_ctx_destroy(bbmm_ctx_t ctx) {
    if (!ctx) return BBMM_ERR_ARG;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->ws.release_all();
    if (ctx->pinned_flag) cudaFreeHost(ctx->pinned_flag);
    for (cudaEvent_t e : ctx->mm_events) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->comm_events) cudaEventDestroy(e);
    if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return BBMM_OK;
}

const char *bbmm_last_error(bbmm_ctx_t ctx) { return ctx ? ctx->err.c_str() : "ctx is NULL"; }

bbmm_status_t bbmm_nccl_unique_id(void *out) {
    if (!out) return BBMM_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return BBMM_ERR_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return BBMM_OK;
}

bbmm_status_t bbmm_ctx_set_comm(bbmm_ctx_t ctx, int nranks, int rank, const void *uid) {
    return guarded(ctx, [&] {
        BBMM_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
        if (ctx->comm) {
            ncclCommDestroy(ctx->comm);
            ctx->comm = nullptr;
        }
        ctx->local = nullptr;
        ctx->nranks = nranks;
        ctx->rank = rank;
        // nranks == 1 with an id: a 1-rank communicator, every collective still issued
        if (nranks > 1 || uid != nullptr) {
            BBMM_REQUIRE(uid != nullptr, "unique id is NULL");
            ncclUniqueId id;
            std::memcpy(&id, uid, sizeof(id));
            BBMM_NCCL(ncclCommInitRank(&ctx->comm, nranks, id, rank));
        }
    });
}

bbmm_status_t bbmm_ctx_set_matmul_precision(bbmm_ctx_t ctx, bbmm_matmul_precision_t p) {
    if (!ctx || (p != BBMM_MATMUL_FP64ACC && p != BBMM_MATMUL_FP32ACC &&
                 p != BBMM_MATMUL_INT8EXACT && p != BBMM_MATMUL_INT8EXACT31 &&
                 p != BBMM_MATMUL_INT8EXACT23))
        return BBMM_ERR_ARG;
    ctx->matmul_acc64 = (p != BBMM_MATMUL_FP32ACC);
    ctx->matmul_tc = (p == BBMM_MATMUL_INT8EXACT || p == BBMM_MATMUL_INT8EXACT31 ||
                      p == BBMM_MATMUL_INT8EXACT23);
    ctx->matmul_grid = p == BBMM_MATMUL_INT8EXACT31 ? 31 : p == BBMM_MATMUL_INT8EXACT23 ? 23 : 0;
    return BBMM_OK;
}

bbmm_status_t bbmm_row_partition(int64_t n, int32_t nranks, int32_t rank, int64_t *r0,
                                 int64_t *r1, int64_t *nb) {
    if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || !r0 || !r1) return BBMM_ERR_ARG;
    const RowRange rr = row_partition(n, nranks, rank);
    *r0 = rr.r0;
    *r1 = rr.r1;
    if (nb) *nb = rr.nb;
    return BBMM_OK;
}

bbmm_status_t bbmm_local_rows(bbmm_ctx_t ctx, int64_t n, int64_t *r0, int64_t *r1) {
    if (!ctx || !r0 || !r1 || n < 0) return BBMM_ERR_ARG;
    RowRange rr = local_rows(ctx, n);
    *r0 = rr.r0;
    *r1 = rr.r1;
    return BBMM_OK;
}

bbmm_status_t bbmm_kernel_matmul(bbmm_ctx_t ctx, const float *X, int64_t n, int32_t d,
                                 const bbmm_hyper_t *hyper, bbmm_kmode_t kmode, const double *D,
                                 int32_t ncols, int64_t ldd, double *V, int64_t ldv) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_kernel_matmul");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(D && V, "D / V is NULL");
        BBMM_REQUIRE(ncols >= 1 && ncols <= kMaxCols, "ncols must be in [1, 64]");
        BBMM_REQUIRE(ldd >= ncols && ldv >= ncols, "leading dimension < ncols");
        BBMM_REQUIRE(kmode == BBMM_ONTHEFLY || kmode == BBMM_STORED, "bad kmode");
        RowRange rr = local_rows(ctx, n);
        const int64_t nloc = rr.count();
        const int dp = pad_dim(d), cp = pad_cols(ncols), cs = (cp + 3) & ~3, ds = (dp + 3) & ~3;
        float *Xs = (float *)ctx->ws.get("Xs", (size_t)n * ds * 4);
        scale_inputs(ctx, X, n, d, h, Xs, dp);
        const bool acc64 = ctx->matmul_acc64;
        void *Dm = ctx->ws.get("mm_Dm", (size_t)n * cs * (acc64 ? 8 : 4));
        if (acc64)
            k_pack_dm<double><<<grid_for(n * cs), 256, 0, ctx->stream>>>(D, ldd, n, ncols, cs,
                                                                         (double *)Dm);
        else
            k_pack_dm<float><<<grid_for(n * cs), 256, 0, ctx->stream>>>(D, ldd, n, ncols, cs,
                                                                        (float *)Dm);
        BBMM_LAUNCH_CHECK();
        ctx->launches++;
        if (nloc == 0) return;
        const bool stored = kmode == BBMM_STORED;
        float *Kst = nullptr;
        TcOperand op = prepare_operator(ctx, stored, X, Xs, dp, n, d, ncols, h, rr.r0, nloc, n, &Kst);
        if (op.version != 0) {
            const int64_t npad = k1tc_pad_rows(n);
            double *S = (double *)ctx->ws.get("tc_S", kMaxCols * 8);
            k1tc_colmax(ctx, D, ldd, n, ncols, S);
            BBMM_REQUIRE(op.npad == npad, "tc operand rows");
            uint8_t *Bp = (uint8_t *)ctx->ws.get("tc_B", tc_bp_bytes(op));
            tc_pack(ctx, op, D, ldd, 0, n, n, ncols, S, Bp);
            size_t cap = tc_vpart_elems(op, n, nloc, op.cb);
            double *Vpart = (double *)ctx->ws.get("mm_Vpart", cap * 8);
            int splits = tc_matmul(ctx, op, Bp, S, op.cb, n, rr.r0, nloc, h.s, Vpart, cap, nullptr,
                                   nullptr);
            k_matmul_finish<<<grid_for(nloc * ncols), 256, 0, ctx->stream>>>(
                Vpart, splits, tc_vstride(op), nloc, ncols, h.noise_var, D, ldd, rr.r0, V, ldv);
            BBMM_LAUNCH_CHECK();
            ctx->launches++;
            BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        size_t cap = vpart_elems(n, nloc, cp, stored);
        double *Vpart = (double *)ctx->ws.get("mm_Vpart", cap * 8);
        int splits;
        if (stored) {
            splits = kernel_matmul_stored(ctx, Kst, n, nloc, Dm, acc64, cp, Vpart, cap, nullptr,
                                          nullptr);
        } else {
            splits = kernel_matmul_onthefly(ctx, h.kind, Xs, dp, n, rr.r0, nloc, Dm, acc64, cp,
                                            h.s, Vpart, cap, nullptr, nullptr);
        }
        k_matmul_finish<<<grid_for(nloc * ncols), 256, 0, ctx->stream>>>(
            Vpart, splits, cs, nloc, ncols, h.noise_var, D, ldd, rr.r0, V, ldv);
        BBMM_LAUNCH_CHECK();
        ctx->launches++;
        BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

bbmm_status_t bbmm_pivchol(bbmm_ctx_t ctx, const float *X, int64_t n, int32_t d,
                           const bbmm_hyper_t *hyper, int32_t k, double *L, int64_t *piv_h,
                           int32_t *k_used_h, double *resid_h) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_pivchol");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(k == 0 || L != nullptr, "L is NULL");
        int ku = 0;
        double res = 0.0;
        std::vector<int64_t> piv(std::max(k, 1));
        pivchol(ctx, X, n, d, h, k, L, piv.data(), &ku, &res);
        if (piv_h) std::copy(piv.begin(), piv.begin() + k, piv_h);
        if (k_used_h) *k_used_h = ku;
        if (resid_h) *resid_h = res;
    });
}

bbmm_status_t bbmm_mbcg(bbmm_ctx_t ctx, const float *X, int64_t n, int32_t d,
                        const bbmm_hyper_t *hyper, bbmm_kmode_t kmode, const double *L, int32_t k,
                        const double *B, int32_t ncols, int64_t ldb, int32_t max_iter, double tol,
                        double *U, int64_t ldu, double *alpha_h, double *beta_h, int32_t *iters_h,
                        double *relres_h, double *rho0_h, double *relres_hist_h) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_mbcg");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(k == 0 || L != nullptr, "L is NULL");
        BBMM_REQUIRE(B && U, "B / U is NULL");
        BBMM_REQUIRE(ncols >= 1 && ncols <= kMaxCols, "ncols must be in [1, 64]");
        BBMM_REQUIRE(ldb >= ncols && ldu >= ncols, "leading dimension < ncols");
        BBMM_REQUIRE(max_iter >= 1 && max_iter <= 256, "max_iter must be in [1, 256]");
        BBMM_REQUIRE(tol >= 0.0 && std::isfinite(tol), "tol must be >= 0");
        RowRange rr = local_rows(ctx, n);
        const int64_t nloc = rr.count();
        const int dp = pad_dim(d), cp = pad_cols(ncols), ds = (dp + 3) & ~3;
        float *Xs = (float *)ctx->ws.get("Xs", (size_t)n * ds * 4);
        scale_inputs(ctx, X, n, d, h, Xs, dp);
        double *cholC = (double *)ctx->ws.get("cholC", (size_t)std::max(k, 1) * std::max(k, 1) * 8);
        double *ldp = (double *)ctx->ws.get("logdet_pre", 8);
        precond_setup(ctx, L, n, k, h.noise_var, cholC, ldp);
        float *Kst = nullptr;
        TcOperand tcop = prepare_operator(ctx, kmode == BBMM_STORED, X, Xs, dp, n, d, ncols, h,
                                          rr.r0, nloc, rr.nb * ctx->nranks, &Kst);
        MbcgArgs a{Xs, dp, h.kind, h.s, tcop, Kst, n, rr.r0, nloc, rr.nb, h.noise_var, L, k, ncols,
                   max_iter, tol};
        MbcgOut o;
        o.U = U;
        o.ldu = ldu;
        mbcg_run(ctx, a, B, ldb, cholC, o);
        if (alpha_h) std::copy(o.alpha.begin(), o.alpha.end(), alpha_h);
        if (beta_h) std::copy(o.beta.begin(), o.beta.end(), beta_h);
        if (iters_h) std::copy(o.iters.begin(), o.iters.end(), iters_h);
        if (relres_h) std::copy(o.relres.begin(), o.relres.end(), relres_h);
        if (rho0_h) std::copy(o.rho0.begin(), o.rho0.end(), rho0_h);
        if (relres_hist_h) std::copy(o.relres_hist.begin(), o.relres_hist.end(), relres_hist_h);
    });
}

bbmm_status_t bbmm_mll_and_grad(bbmm_ctx_t ctx, const float *X, const float *y, int64_t n,
                                int32_t d, const bbmm_hyper_t *hyper, bbmm_kmode_t kmode,
                                int32_t t, int32_t k, int32_t max_iter, double tol, uint64_t seed,
                                const int8_t *eps, double *mll_h, double *grad_h,
                                bbmm_stats_t *stats_h, double *U_out, int64_t *pivots_h) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_mll_and_grad");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(y != nullptr, "y is NULL");
        BBMM_REQUIRE(t >= 1 && t + 1 <= kMaxCols, "t must be in [1, 63]");
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(max_iter >= 1 && max_iter <= 256, "max_iter must be in [1, 256]");
        BBMM_REQUIRE(tol >= 0.0 && std::isfinite(tol), "tol must be >= 0");
        BBMM_REQUIRE(mll_h && grad_h, "mll_h / grad_h is NULL");
        BBMM_REQUIRE(kmode == BBMM_ONTHEFLY || kmode == BBMM_STORED, "bad kmode");
        cudaStream_t sm = ctx->stream;
        const int launches0 = ctx->launches;
        check_finite(ctx, X, n * d, "X");
        check_finite(ctx, y, n, "y");
        comm_timing_reset(ctx);
        Timer t_start(sm);
        nv.next("pivchol");
        const int c = t + 1;
        RowRange rr = local_rows(ctx, n);
        const int64_t nloc = rr.count();
        const int dp = pad_dim(d), cp = pad_cols(c), cs = (cp + 3) & ~3, ds = (dp + 3) & ~3;
        Workspace &ws = ctx->ws;
        float *Xs = (float *)ws.get("Xs", (size_t)n * ds * 4);
        scale_inputs(ctx, X, n, d, h, Xs, dp);

        // 1. pivoted Cholesky + preconditioner (Sec. 4.1, App. B)
        double *L = (double *)ws.get("L", (size_t)std::max(k, 1) * n * 8);
        int k_used = 0;
        double resid = 0.0;
        std::vector<int64_t> piv(std::max(k, 1), -1);
        if (k > 0) pivchol(ctx, X, n, d, h, k, L, piv.data(), &k_used, &resid);
        else resid = h.s * (double)n;
        double *cholC = (double *)ws.get("cholC", (size_t)std::max(k, 1) * std::max(k, 1) * 8);
        double *scal = (double *)ws.get("scalars", 16 * 8);   // [logdet_pre, logdet_ratio, ...]
        int *status = (int *)ws.get("status", sizeof(int));
        BBMM_CUDA(cudaMemsetAsync(status, 0, sizeof(int), sm));
        precond_setup(ctx, L, n, k > 0 ? k_used : 0, h.noise_var, cholC, scal + 0);
        Timer t_pc(sm);
        nv.next("mbcg");

        // 2. probes and B = [y | Z] (Eq. 3)
        double *B = (double *)ws.get("B", (size_t)std::max<int64_t>(nloc, 1) * c * 8);
        double *Z0 = (double *)ws.get("Z0", (size_t)std::max<int64_t>(nloc, 1) * c * 8);
        if (nloc > 0)
            make_probes(ctx, eps, seed, n, k, t, L, k > 0 ? k_used : 0, k > 0 ? h.sigma : 1.0,
                        rr.r0, nloc, y, B, c);
        // 3. one mBCG call on [y, z_1..z_t]
        float *Kst = nullptr;
        TcOperand tcop = prepare_operator(ctx, kmode == BBMM_STORED, X, Xs, dp, n, d, c, h, rr.r0,
                                          nloc, rr.nb * ctx->nranks, &Kst);
        MbcgArgs a{Xs, dp, h.kind, h.s, tcop, Kst, n, rr.r0, nloc, rr.nb, h.noise_var, L,
                   k > 0 ? k_used : 0, c, max_iter, tol};
        MbcgOut o;
        o.Z0 = Z0;
        o.defer_host = true;                 // mbcg_finish after the final sync below
        mbcg_run(ctx, a, B, c, cholC, o);
        Timer t_cg(sm);
        nv.next("slq");

        // 4. SLQ log-det (probe columns 1..t)
        const char *stb = reinterpret_cast<const char *>(o.state_d);
        slq_logdet(ctx, o.ahist_d, o.bhist_d,
                   reinterpret_cast<const int *>(stb + offsetof(MbcgState, iters)),
                   reinterpret_cast<const double *>(stb + offsetof(MbcgState, rho0)), max_iter, c,
                   1, t, scal + 1, status);
        Timer t_slq(sm);
        nv.next("deriv");

        // 5. derivative pass (once)
        const int nq = dp + 1;
        double *dred = (double *)ws.get("d_red", (size_t)(nq + 3) * 8);
        BBMM_CUDA(cudaMemsetAsync(dred, 0, (size_t)(nq + 3) * 8, sm));
        const int sblk = grid_for(std::max<int64_t>(nloc, 1));
        double *spart = (double *)ws.get("s_part", (size_t)sblk * 3 * 8);
        const bool tc_deriv = tcop.version == 2 && k1tc2_deriv_supported(h.kind, h.n_ls, d, c);
        if (tc_deriv) {
            // isotropic RBF: S_l = sum_a A_a . (s K~ o R^2 Bd)_a by one exact tensor-core
            // kernel-matmul of the packed Bd = [P^-1 Z / t | -u0]; S_s = sum_a A_a . (s K~ Bd)_a
            // from K U = B - sigma^2 U - R (k_outputscale_term)
            double *Bd = (double *)ws.get("d_Bd", (size_t)std::max<int64_t>(nloc, 1) * c * 8);
            double *Sd = (double *)ws.get("d_S", kMaxCols * 8);
            const int64_t npad_tc = k1tc_pad_rows(rr.nb * ctx->nranks);
            // MODE-1 instantiation (>= c), or the operand's column chunks of 33 (c + 1 > 33)
            const bool chunked = tcop.nch > 1;
            const int cbd = chunked ? tcop.cb : k1tc2_deriv_cols(d, c);
            const int vsd = chunked ? tc_vstride(tcop) : (cbd + 3) & ~3;
            const int nchd = chunked ? tcop.nch : 1;
            BBMM_REQUIRE(!chunked || tcop.npad == npad_tc, "tc operand rows");
            uint8_t *Bp = (uint8_t *)ws.get("tc_B", (size_t)nchd * npad_tc * k1tc_bslice_rows(cbd));
            if (nloc > 0) {
                k_build_bd<<<grid_for(nloc * c), 256, 0, sm>>>(o.U_d, Z0, nloc, t, Bd);
                ctx->launches++;
            }
            k1tc_colmax(ctx, Bd, c, nloc, c, Sd);
            allreduce_max(ctx, Sd, c);
            if (nloc > 0) {
                if (chunked) tc_pack(ctx, tcop, Bd, c, rr.r0, nloc, n, c, Sd, Bp);
                else k1tc_pack(ctx, Bd, c, rr.r0, nloc, n, c, Sd, Bp, 4, cbd);
            }
            for (int z = 0; z < nchd; z++)
                allgather_rows(ctx, Bp + (size_t)z * npad_tc * k1tc_bslice_rows(cbd),
                               (size_t)rr.nb * k1tc_bslice_rows(cbd));
            const size_t cap = tc_vpart_elems(tcop, n, nloc, cbd);
            double *Vp = (double *)ws.get("d_Vpart", std::max<size_t>(cap, 1) * 8);
            double *dpart = (double *)ws.get("d_part", (size_t)sblk * 8);
            if (nloc > 0) {
                // S_l at dred[0]: the k~ r^2 kernel-matmul (mode 1)
                const int sp = tc_matmul(ctx, tcop, Bp, Sd, cbd, n, rr.r0, nloc, h.s, Vp, cap,
                                         nullptr, nullptr, 1);
                k_deriv_dot<<<sblk, 256, 0, sm>>>(Vp, sp, vsd, nloc, t, o.U_d, dpart);
                reduce_blocks(ctx, dpart, sblk, 1, dred);
                // S_s at dred[dp]: from the solves' residual identity (no matmul)
                k_outputscale_term<<<sblk, 256, 0, sm>>>(o.U_d, o.R_d, B, Z0, h.noise_var, nloc,
                                                         t, dpart);
                reduce_blocks(ctx, dpart, sblk, 1, dred + dp);
                ctx->launches += 2;
            }
            if (nloc > 0) {
                k_scalar_terms<<<sblk, 256, 0, sm>>>(o.U_d, Z0, y, rr.r0, nloc, t, spart);
                ctx->launches++;
                reduce_blocks(ctx, spart, sblk, 3, dred + nq);
            }
        } else {
            float *A32 = (float *)ws.get("A32", (size_t)std::max<int64_t>(nloc, 1) * cs * 4);
            float *B32 = (float *)ws.get("B32", (size_t)rr.nb * ctx->nranks * cs * 4);
            BBMM_CUDA(cudaMemsetAsync(B32, 0, (size_t)rr.nb * ctx->nranks * cs * 4, sm));
            if (nloc > 0) {
                k_pack_deriv<<<grid_for(nloc * cs), 256, 0, sm>>>(o.U_d, Z0, nloc, t, cs, rr.r0,
                                                                 A32, B32);
                ctx->launches++;
            }
            allgather_rows(ctx, B32, (size_t)rr.nb * cs * 4);
            const bool dtc = ctx->matmul_tc && deriv_tc_supported(h.kind, dp, cp, n);
            // RBF ARD with the K1-TC operand: the expanded-square tensor-core pass
            const bool dtc2 = ctx->matmul_tc && tcop.version == 2 &&
                              deriv_tc2_supported(h.kind, h.n_ls, d, dp, c, n);
            double *dpart = (double *)ws.get(
                "d_part", std::max({derivative_part_elems(n, std::max<int64_t>(nloc, 1), dp),
                                    deriv_tc_part_elems(n, std::max<int64_t>(nloc, 1), dp),
                                    deriv_tc2_part_elems(n, std::max<int64_t>(nloc, 1), dp)}) * 8);
            if (dtc2) {
                derivative_pass_tc2(ctx, tcop.Xa, d, dp, n, rr.r0, nloc, A32, B32, cs, c, o.U_d,
                                    o.R_d, B, Z0, h.noise_var, h.s, dpart, dred);
                if (nloc > 0) {
                    k_scalar_terms<<<sblk, 256, 0, sm>>>(o.U_d, Z0, y, rr.r0, nloc, t, spart);
                    ctx->launches++;
                    reduce_blocks(ctx, spart, sblk, 3, dred + nq);
                }
            } else if (nloc > 0) {
                int nblk = 0;
                if (dtc)   // W tiles on the tensor cores (deriv_tc.cu)
                    nblk = derivative_pass_tc(ctx, h.kind, Xs, dp, n, rr.r0, nloc, A32, B32, cp, c,
                                              dpart);
                else
                    derivative_pass(ctx, h.kind, Xs, dp, n, rr.r0, nloc, A32, B32, cp, nq,
                                    h.n_ls > 1, d, dpart, &nblk);
                reduce_blocks(ctx, dpart, nblk, nq, dred);
                k_scalar_terms<<<sblk, 256, 0, sm>>>(o.U_d, Z0, y, rr.r0, nloc, t, spart);
                ctx->launches++;
                reduce_blocks(ctx, spart, sblk, 3, dred + nq);
            }
        }
        allreduce_sum(ctx, dred, (size_t)nq + 3);
        BBMM_LAUNCH_CHECK();
        Timer t_end(sm);

        // 6. assemble (fp64, host): Eq. 2 with reading R4
        std::vector<double> hred(nq + 3);
        double hs[2];
        int st_h = 0;
        BBMM_CUDA(cudaMemcpyAsync(hred.data(), dred, (size_t)(nq + 3) * 8, cudaMemcpyDeviceToHost, sm));
        BBMM_CUDA(cudaMemcpyAsync(hs, scal, 2 * 8, cudaMemcpyDeviceToHost, sm));
        BBMM_CUDA(cudaMemcpyAsync(&st_h, status, sizeof(int), cudaMemcpyDeviceToHost, sm));
        BBMM_CUDA(cudaStreamSynchronize(sm));
        mbcg_finish(ctx, o);                 // mBCG host results + breakdown check (throws first)
        if (st_h) throw Error{BBMM_ERR_NUMERIC, "non-positive Ritz value in SLQ (Khat not PD?)"};
        const double logdet = hs[0] + hs[1];
        const double quad_y = hred[nq + 0], uu = hred[nq + 1], uz = hred[nq + 2];
        *mll_h = -0.5 * (quad_y + logdet + (double)n * std::log(2.0 * M_PI));
        // lengthscale / outputscale components: grad = -S/2
        if (tc_deriv) {
            grad_h[0] = -0.5 * hred[0];          // S_l (includes s)
            grad_h[1] = -0.5 * hred[dp];         // S_s (includes s)
        } else {
            // CUDA-core pass accumulates per input dimension in scaled units
            const double lfac = (h.kind == BBMM_RBF) ? h.s * 2.0 * std::log(2.0) : h.s / 3.0;
            if (h.n_ls == 1) {
                double sl = 0.0;
                for (int q = 0; q < d; q++) sl += hred[q];
                grad_h[0] = -0.5 * lfac * sl;
            } else {
                for (int q = 0; q < d; q++) grad_h[q] = -0.5 * lfac * hred[q];
            }
            grad_h[h.n_ls] = -0.5 * h.s * hred[dp];
        }
        // log sigma: dKhat = 2 sigma^2 I
        const double tau_s = 2.0 * h.noise_var * uz / (double)t;
        const double quad_s = 2.0 * h.noise_var * uu;
        grad_h[h.n_ls + 1] = 0.5 * (quad_s - tau_s);

        if (U_out && nloc > 0)
            BBMM_CUDA(cudaMemcpyAsync(U_out, o.U_d, (size_t)nloc * c * 8, cudaMemcpyDeviceToDevice, sm));
        if (pivots_h) std::copy(piv.begin(), piv.begin() + k, pivots_h);
        if (stats_h) {
            bbmm_stats_t s{};
            s.iters = o.iters_run;
            s.k_used = k_used;
            s.logdet_precond = hs[0];
            s.logdet_ratio = hs[1];
            s.logdet = logdet;
            s.quad_y = quad_y;
            s.resid_trace = resid;
            s.relres_y = o.relres.empty() ? 0.0 : o.relres[0];
            s.ms_total = t_end.since(t_start);
            s.ms_pivchol = t_pc.since(t_start);
            s.ms_mbcg = t_cg.since(t_pc);
            s.ms_matmul = o.ms_matmul;
            s.ms_slq = t_slq.since(t_cg);
            s.ms_deriv = t_end.since(t_slq);
            s.matmul_launches = o.matmul_launches;
            s.gpu_launches = ctx->launches - launches0;
            s.matmul_path = tcop.version == 3 ? 3 : tcop.version == 2 ? 2 : (Kst ? 1 : 0);
            s.kgrid_bits = tcop.version == 2 ? (tcop.grid31 ? 31 : 23) : 0;
            s.relres_max = 0.0;
            bool active = false;
            for (int col = 0; col < c && col < (int)o.relres.size(); col++) {
                s.relres_max = std::max(s.relres_max, o.relres[col]);
                active |= tol > 0.0 && o.iters[col] >= max_iter && o.relres[col] >= tol;
            }
            s.unconverged = (tol > 0.0 ? active : s.relres_max >= kUnconvergedRelres) ? 1 : 0;
            s.ms_comm = comm_timing_ms(ctx);
            *stats_h = s;
        }
        BBMM_CUDA(cudaStreamSynchronize(sm));
    });
}

bbmm_status_t bbmm_predict(bbmm_ctx_t ctx, const float *X, const float *y, int64_t n, int32_t d,
                           const float *Xstar, int64_t nstar, const bbmm_hyper_t *hyper,
                           bbmm_kmode_t kmode, int32_t k, int32_t max_iter, double tol,
                           double *mean, double *var) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_predict");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(y != nullptr && Xstar != nullptr && mean != nullptr, "y / Xstar / mean is NULL");
        BBMM_REQUIRE(nstar >= 1, "nstar must be >= 1");
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(max_iter >= 1 && max_iter <= 256, "max_iter must be in [1, 256]");
        BBMM_REQUIRE(tol >= 0.0 && std::isfinite(tol), "tol must be >= 0");
        BBMM_REQUIRE(kmode == BBMM_ONTHEFLY || kmode == BBMM_STORED, "bad kmode");
        check_finite(ctx, X, n * d, "X");
        check_finite(ctx, y, n, "y");
        check_finite(ctx, Xstar, nstar * d, "Xstar");
        predict_run(ctx, X, y, n, d, Xstar, nstar, h, kmode == BBMM_STORED, k, max_iter, tol, mean,
                    var);
        BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

bbmm_status_t bbmm_predict_cov(bbmm_ctx_t ctx, const float *X, const float *y, int64_t n,
                               int32_t d, const float *Xstar, int64_t nstar,
                               const bbmm_hyper_t *hyper, bbmm_kmode_t kmode, int32_t k,
                               int32_t max_iter, double tol, double *mean, double *cov) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_predict_cov");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(y != nullptr && Xstar != nullptr && mean != nullptr && cov != nullptr,
                     "y / Xstar / mean / cov is NULL");
        BBMM_REQUIRE(nstar >= 1 && nstar <= kMaxPredCov, "nstar must be in [1, 8192]");
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(max_iter >= 1 && max_iter <= 256, "max_iter must be in [1, 256]");
        BBMM_REQUIRE(tol >= 0.0 && std::isfinite(tol), "tol must be >= 0");
        BBMM_REQUIRE(kmode == BBMM_ONTHEFLY || kmode == BBMM_STORED, "bad kmode");
        check_finite(ctx, X, n * d, "X");
        check_finite(ctx, y, n, "y");
        check_finite(ctx, Xstar, nstar * d, "Xstar");
        predict_run(ctx, X, y, n, d, Xstar, nstar, h, kmode == BBMM_STORED, k, max_iter, tol, mean,
                    nullptr, cov);
        BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

bbmm_status_t bbmm_train_adam(bbmm_ctx_t ctx, const float *X, const float *y, int64_t n,
                              int32_t d, const bbmm_hyper_t *hyper, bbmm_kmode_t kmode, int32_t t,
                              int32_t k, int32_t max_iter, double tol, uint64_t seed, int32_t steps,
                              double lr, double beta1, double beta2, double eps,
                              double *theta_out_h, double *trace_h) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_train_adam");
        validate_common(ctx, X, n, d);
        BBMM_REQUIRE(hyper != nullptr && hyper->log_ls_h != nullptr, "hyper is NULL");
        BBMM_REQUIRE(hyper->n_ls == 1 || hyper->n_ls == d, "n_ls must be 1 or d");
        BBMM_REQUIRE(steps >= 0, "steps must be >= 0");
        BBMM_REQUIRE(lr > 0.0 && beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0 &&
                         eps >= 0.0,
                     "Adam settings out of range");
        BBMM_REQUIRE(theta_out_h != nullptr, "theta_out_h is NULL");
        const int nls = hyper->n_ls, nt = nls + 2;
        // theta = (log l.., log s, log sigma); Adam on -mll (reading R26)
        std::vector<double> th(nt), g(nt), m1(nt, 0.0), m2(nt, 0.0);
        std::copy(hyper->log_ls_h, hyper->log_ls_h + nls, th.begin());
        th[nls] = hyper->log_outputscale;
        th[nls + 1] = hyper->log_noise;
        for (int s = 0; s < steps; s++) {
            bbmm_hyper_t hs{hyper->kind, nls, th.data(), th[nls], th[nls + 1]};
            double mll = 0.0;
            const bbmm_status_t st = bbmm_mll_and_grad(ctx, X, y, n, d, &hs, kmode, t, k, max_iter,
                                                       tol, seed + (uint64_t)s, nullptr, &mll,
                                                       g.data(), nullptr, nullptr, nullptr);
            if (st != BBMM_OK) throw Error{st, "training step " + std::to_string(s) + ": " + ctx->err};
            if (!std::isfinite(mll)) throw Error{BBMM_ERR_NUMERIC, "non-finite mll during training"};
            if (trace_h) {
                trace_h[(size_t)s * (1 + nt)] = mll;
                std::copy(th.begin(), th.end(), trace_h + (size_t)s * (1 + nt) + 1);
            }
            const double c1 = 1.0 - std::pow(beta1, s + 1), c2 = 1.0 - std::pow(beta2, s + 1);
            for (int q = 0; q < nt; q++) {
                const double gq = -g[q];
                m1[q] = beta1 * m1[q] + (1.0 - beta1) * gq;
                m2[q] = beta2 * m2[q] + (1.0 - beta2) * gq * gq;
                th[q] -= lr * (m1[q] / c1) / (std::sqrt(m2[q] / c2) + eps);
            }
        }
        std::copy(th.begin(), th.end(), theta_out_h);
    });
}

bbmm_status_t bbmm_sor_mbcg(bbmm_ctx_t ctx, const float *X, int64_t n, int32_t d, const float *Xu,
                            int32_t m, const bbmm_hyper_t *hyper, int32_t k, const double *B,
                            int32_t ncols, int64_t ldb, int32_t max_iter, double tol, double *U,
                            int64_t ldu, int64_t *piv_h, int32_t *iters_h, double *relres_h,
                            double *relres_hist_h) {
    return guarded(ctx, [&] {
        NvtxPhase nv("bbmm_sor_mbcg");
        validate_common(ctx, X, n, d);
        Hyper h = make_hyper(hyper, d);
        BBMM_REQUIRE(Xu != nullptr && B != nullptr && U != nullptr, "Xu / B / U is NULL");
        BBMM_REQUIRE(m >= 1 && m <= kMaxInducing, "m must be in [1, 512]");
        BBMM_REQUIRE(k >= 0 && k <= n && k <= kMaxRank, "k must be in [0, min(n, 128)]");
        BBMM_REQUIRE(ncols >= 1 && ncols <= kMaxCols, "ncols must be in [1, 64]");
        BBMM_REQUIRE(ldb >= ncols && ldu >= ncols, "leading dimension < ncols");
        BBMM_REQUIRE(max_iter >= 1 && max_iter <= 256, "max_iter must be in [1, 256]");
        BBMM_REQUIRE(tol >= 0.0 && std::isfinite(tol), "tol must be >= 0");
        check_finite(ctx, X, n * d, "X");
        check_finite(ctx, Xu, (int64_t)m * d, "Xu");
        RowRange rr = local_rows(ctx, n);
        const int64_t nloc = rr.count();
        double *Bs = (double *)ctx->ws.get("sor_Bs", (size_t)m * n * 8);
        sor_setup(ctx, X, n, d, Xu, m, h, Bs);
        double *L = (double *)ctx->ws.get("L", (size_t)std::max(k, 1) * n * 8);
        int k_used = 0;
        double resid = 0.0;
        std::vector<int64_t> piv(std::max(k, 1), -1);
        if (k > 0) pivchol_sor(ctx, Bs, n, m, h.s, k, L, piv.data(), &k_used, &resid);
        double *cholC = (double *)ctx->ws.get("cholC", (size_t)std::max(k, 1) * std::max(k, 1) * 8);
        double *ldp = (double *)ctx->ws.get("logdet_pre", 8);
        precond_setup(ctx, L, n, k > 0 ? k_used : 0, h.noise_var, cholC, ldp);
        MbcgArgs a{nullptr, 0, h.kind, h.s, TcOperand{}, nullptr, n, rr.r0, nloc, rr.nb,
                   h.noise_var, L, k > 0 ? k_used : 0, ncols, max_iter, tol};
        a.sor_B = Bs;
        a.sor_m = m;
        MbcgOut o;
        o.U = U;
        o.ldu = ldu;
        mbcg_run(ctx, a, B, ldb, cholC, o);
        if (piv_h) std::copy(piv.begin(), piv.begin() + k, piv_h);
        if (iters_h) std::copy(o.iters.begin(), o.iters.end(), iters_h);
        if (relres_h) std::copy(o.relres.begin(), o.relres.end(), relres_h);
        if (relres_hist_h) std::copy(o.relres_hist.begin(), o.relres_hist.end(), relres_hist_h);
    });
}

}  // extern "C"
