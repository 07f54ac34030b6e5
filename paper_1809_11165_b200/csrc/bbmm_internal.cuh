// bbmm_internal.cuh -- shared declarations of the CUDA path (sm_100a).
// Nothing here is shared with oracle/ (independent implementations).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/bbmm.h"

namespace bbmm {

constexpr int kMaxCols = 64;     // ncols = t + 1 <= 64
constexpr int kMaxInducing = 512;  // SoR operator: inducing points m (row f4)
constexpr int kMaxRank = 128;    // preconditioner rank k
constexpr int kMaxDim = 32;      // input dimension d
constexpr int64_t kMaxPredCov = 8192;   // test points of bbmm_predict_cov (cov is nstar^2)
constexpr int kNumSMs = 148;
// bbmm_stats_t.unconverged: relres at exit above which mBCG counts as unconverged (SURVEY.md §8c
// regime B; regime A runs end at <= 1e-6, the regime-B configs at 1e-2..0.2)
constexpr double kUnconvergedRelres = 1e-3;

// ---------------------------------------------------------------- status
struct Error {
    bbmm_status_t st;
    std::string msg;
};

#define BBMM_CUDA(x)                                                              \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess)                                                    \
            throw ::bbmm::Error{BBMM_ERR_CUDA, std::string(#x) + ": " +           \
                                                 cudaGetErrorString(e_)};         \
    } while (0)

#define BBMM_NCCL(x)                                                              \
    do {                                                                          \
        ncclResult_t r_ = (x);                                                    \
        if (r_ != ncclSuccess)                                                    \
            throw ::bbmm::Error{BBMM_ERR_NCCL, std::string(#x) + ": " +           \
                                                 ncclGetErrorString(r_)};         \
    } while (0)

#define BBMM_REQUIRE(cond, msg)                                                   \
    do {                                                                          \
        if (!(cond)) throw ::bbmm::Error{BBMM_ERR_ARG, msg};                      \
    } while (0)

#define BBMM_LAUNCH_CHECK() BBMM_CUDA(cudaGetLastError())

// Device-side bounds checks of the newer kernels (a build with -DBBMM_BOUNDS_CHECK traps on a
// violated index; compute-sanitizer is not available on the GPU pool): off in the product build.
#ifdef BBMM_BOUNDS_CHECK
#define BBMM_DCHECK(cond)                                                                   \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("BBMM_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,  \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                            \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define BBMM_DCHECK(cond) ((void)0)
#endif
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

// ------------------------------------------------------- kernel parameters
// Input-space scaling so the pair kernels evaluate k from a scaled distance:
//   RBF:    xs = x * sqrt(log2(e)/2) / l   ->  k = s * 2^(-|xs_i - xs_j|^2)
//   Matern: xs = x * sqrt(5) / l           ->  rh = |xs_i - xs_j| = sqrt5 r,
//                                              k = s (1 + rh + rh^2/3) e^{-rh}
struct Hyper {
    int kind;
    int n_ls;
    double ls[kMaxDim];  // lengthscales (host exp of log_ls)
    double s;            // outputscale
    double noise_var;    // sigma^2
    double sigma;
};

// NVTX ranges around the host-side phases of a call (visible to nsys / ncu --nvtx): one
// range per entry point, next() closes the current phase and opens the following one.
struct NvtxPhase {
    int depth = 0;
    explicit NvtxPhase(const char *call) { push(call); }
    void next(const char *phase) {
        if (depth > 1) { nvtxRangePop(); depth--; }
        push(phase);
    }
    ~NvtxPhase() {
        while (depth-- > 0) nvtxRangePop();
    }
  private:
    void push(const char *name) { nvtxRangePushA(name); depth++; }
};

// ------------------------------------------------------------- workspace
struct Workspace {
    std::unordered_map<std::string, std::pair<void *, size_t>> bufs;
    void *get(const std::string &name, size_t bytes);
    void release_all();
};

// mBCG device state (one per context; lives in device memory).
struct MbcgState {
    int j;                        // current iteration
    int status;                   // 0 ok, BBMM_ERR_NUMERIC on breakdown
    int any_active;
    int pad_;
    int active[kMaxCols];
    int iters[kMaxCols];
    double rho[kMaxCols];         // r^T Phat^{-1} r of the current iterate
    double rho0[kMaxCols];
    double bnorm[kMaxCols];
    double alpha[kMaxCols];       // alpha of the current iteration
    double beta[kMaxCols];
    double relres[kMaxCols];
    double red[4 * kMaxCols];     // reduced sums: [dv | rr | rz | misc]
};

}  // namespace bbmm

namespace bbmm {
struct LocalGroup;
void local_allreduce_sum(bbmm_ctx_s *ctx, double *buf, size_t count);
void local_allreduce_max(bbmm_ctx_s *ctx, double *buf, size_t count);
void local_allgather(bbmm_ctx_s *ctx, void *buf, size_t bytes_per_rank);
}  // namespace bbmm

struct bbmm_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    std::string err;
    bbmm::Workspace ws;
    int launches = 0;   // library kernel launches since last reset
    bool matmul_acc64 = true;   // FP64ACC / INT8EXACT fallback: fp64 accumulation
    bool matmul_tc = true;      // BBMM_MATMUL_INT8EXACT (default): tcgen05 exact contraction
    int matmul_grid = 0;        // on-the-fly RBF k~ grid: 0 auto (INT8EXACT), 31 or 23 (forced)
    int *pinned_flag = nullptr; // pinned host int for per-iteration convergence polling (lazy)
    bbmm::LocalGroup *local = nullptr;   // in-process rank group (comm_local.cu) instead of NCCL
    // timing events of the mBCG matmuls, reused across calls (created on first use, destroyed
    // with the context): no per-call event creation, nothing to leak when a call throws
    std::vector<cudaEvent_t> mm_events;
    // collective timing (bbmm_stats_t.ms_comm): event pairs around every collective since the
    // last comm_timing_reset, reused across calls like mm_events
    std::vector<cudaEvent_t> comm_events;
    size_t n_comm_ev = 0;
    bool capturing = false;   // the context stream is being captured into a CUDA graph (mBCG)
    cudaGraphExec_t graph_exec = nullptr;   // the last call's captured mBCG iterations
};

namespace bbmm {

// Timing events on the context stream.  While the mBCG iterations are captured into a CUDA
// graph the record must be an external event-record node (a plain record on a capturing stream
// is only a dependency marker and would leave the event unrecorded).
inline void record_event(bbmm_ctx_s *ctx, cudaEvent_t ev) {
    cudaError_t e = ctx->capturing ? cudaEventRecordWithFlags(ev, ctx->stream, cudaEventRecordExternal)
                                   : cudaEventRecord(ev, ctx->stream);
    if (e != cudaSuccess) throw Error{BBMM_ERR_CUDA, std::string("event record: ") + cudaGetErrorString(e)};
}

// --------------------------------------------------------------- helpers
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Function attributes (cudaFuncSetAttribute) are per device: a call site runs its setup once
// per device it launches on (several contexts / devices may share the process).  Racing
// threads may both run the idempotent setup.
struct DeviceOnce {
    std::atomic<uint64_t> mask{0};
    template <typename F>
    void operator()(int dev, F &&f) {
        const uint64_t bit = 1ull << (dev & 63);
        if (mask.load(std::memory_order_acquire) & bit) return;
        f();
        mask.fetch_or(bit, std::memory_order_acq_rel);
    }
};

struct RowRange {
    int64_t r0, r1, nb;
    int64_t count() const { return r1 > r0 ? r1 - r0 : 0; }
};
RowRange local_rows(const bbmm_ctx_s *ctx, int64_t n);

Hyper make_hyper(const bbmm_hyper_t *h, int d);

// ------------------------------------------------ pair kernels (matmul.cu)
// X scaled for the fp32 pair kernels: n x dp fp32 (dp = padded d).
int pad_dim(int d);
int pad_cols(int c);
void scale_inputs(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h,
                  float *Xs, int dp);

// Kernel-matmul: Vpart[s][i][cp] (fp64) = sum_{j in split s} k(x_{r0+i}, x_j) D32[j][.]
// (outputscale applied, no sigma^2 term).  Returns number of splits used.
// Dm: the search directions as the matmul reads them: n_pad x round4(cp),
// fp64 when acc64 (default precision) else fp32.
int kernel_matmul_onthefly(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n,
                           int64_t r0, int64_t nloc, const void *Dm, bool acc64, int cp, double s,
                           double *Vpart, size_t vpart_cap_elems, cudaEvent_t ev0,
                           cudaEvent_t ev1);
int kernel_matmul_stored(bbmm_ctx_s *ctx, const float *Kst, int64_t n, int64_t nloc,
                         const void *Dm, bool acc64, int cp, double *Vpart,
                         size_t vpart_cap_elems, cudaEvent_t ev0, cudaEvent_t ev1);
void build_stored_k(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n, int64_t r0,
                    int64_t nloc, double s, float *Kst);
size_t vpart_elems(int64_t n, int64_t nloc, int cp, bool stored);

// ------------------------------------------- tensor-core matmul (k1tc.cu)
int64_t k1tc_pad_rows(int64_t n);
int k1tc_bslice_rows(int c);
void k1tc_col_mean(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, double *mean);
void k1tc_colmax(bbmm_ctx_s *ctx, const double *D, int64_t ldd, int64_t rows, int c, double *S);
void k1tc_pack(bbmm_ctx_s *ctx, const double *D, int64_t ldd, int64_t row0, int64_t rows,
               int64_t n, int c, const double *S, uint8_t *Bpack, int nd = 4, int cb = -1);
int tc_bslice_rows(int c, int nd);   // bytes per point of the packed D operand (nd slices)
void allreduce_max(bbmm_ctx_s *ctx, double *buf, size_t count);
bool k1tc2_supported(int kind, int d, int c);
// the K1-TC instantiation (column count, >= c) that runs c columns, 0 if none; the
// derivative (MODE 1) instantiation for c (isotropic RBF), 0 if none
int k1tc2_cols(int kind, int d, int c);
int k1tc2_deriv_cols(int d, int c);
int64_t k1tc2_xa_floats(int64_t npad, int d);
int64_t k1tc2_xb_floats(int64_t npad, int d);
float k1tc2_prep_inputs(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h,
                        float *Xa, float *XB, int64_t npad);
size_t k1tc2_vpart_elems(int64_t n, int64_t nloc, int c);
int k1tc2_matmul(bbmm_ctx_s *ctx, const float *Xa, const float *XB, const uint8_t *Bp,
                 const double *S, int d, int c, int64_t n, int64_t r0, int64_t nloc, double s,
                 double *Vpart, size_t cap, cudaEvent_t ev0, cudaEvent_t ev1, int mode = 0,
                 int ldv = 0, int coff = 0);
// column chunking of K1-TC for c above the largest instantiation (cb, nch; nch = 0: none)
int k1tc2_chunks(int kind, int d, int c, int *cb);
bool k1tc2_deriv_supported(int kind, int n_ls, int d, int c);

// Tensor-core operand of one mBCG call (prepared once per call).
struct TcOperand {
    int version = 0;            // 0: none (FP64ACC path), 2: k1tc2 (on the fly), 3: k2tc (stored)
    int d = 0;
    const float *Xa = nullptr;  // v2 row operand
    const float *XB = nullptr;  // v2 distance tiles
    const uint8_t *Kq = nullptr;  // v3 stored K slices (this rank's rows)
    int kind = 0;               // kernel family of the operand
    int nd = 4;                 // D slices of the packed operand (k1tc_pack nd)
    int cb = 0;                 // columns of the kernel instantiation (>= c; zero-padded)
    // v2 with more columns than the largest instantiation: nch column chunks of cb columns, each
    // its own packed operand (npad rows apart) and launch, writing Vpart columns [z cb, z cb + cb)
    int nch = 1;
    int64_t npad = 0;           // rows of one chunk's packed operand (k1tc_pad_rows)
    bool grid31 = false;        // v2 RBF: kernel values on the 31-bit grid (K1-TC MODE 3)
};
// Vpart row stride of a tensor-core operand's matmul (round4 of all chunks' columns)
inline int tc_vstride(const TcOperand &op) { return (op.nch * op.cb + 3) & ~3; }
// bytes of the packed D operand of all chunks (k1tc_pack layout per chunk)
size_t tc_bp_bytes(const TcOperand &op);
// pack D (c columns, rows [row0, row0 + rows) of n) into the operand's chunks (k1tc_pack each)
void tc_pack(bbmm_ctx_s *ctx, const TcOperand &op, const double *D, int64_t ldd, int64_t row0,
             int64_t rows, int64_t n, int c, const double *S, uint8_t *Bp);
int tc_dslices(const TcOperand &op);   // D slices of the operand's packed format (4 or 5)
// Prepare the tensor-core inputs for (kind, d, c) if the INT8EXACT mode applies.
TcOperand tc_prepare(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, int c, const Hyper &h,
                     int64_t npad_rows);
size_t tc_vpart_elems(const TcOperand &op, int64_t n, int64_t nloc, int c);
// cb: the column count of the instantiation to run (op.cb for the mBCG operand; the
// derivative block for mode 1); Bp packed for cb, Vpart rows of round4(cb)
int tc_matmul(bbmm_ctx_s *ctx, const TcOperand &op, const uint8_t *Bp, const double *S, int cb,
              int64_t n, int64_t r0, int64_t nloc, double s, double *Vpart, size_t cap,
              cudaEvent_t ev0, cudaEvent_t ev1, int mode = 0);

// stored K on the int8 tensor cores (k2tc.cu)
bool k2tc_supported(int c);
int k2tc_cols(int c);   // instantiated column count >= c, 0 if none
size_t k2tc_vpart_elems(int64_t n, int64_t nloc, int c);
size_t k2tc_kq_bytes(int64_t n, int64_t nloc);
void k2tc_build(bbmm_ctx_s *ctx, const float *X, int d, const Hyper &h, int64_t n, int64_t r0,
                int64_t nloc, uint8_t *Kq);
int k2tc_matmul(bbmm_ctx_s *ctx, const uint8_t *Kq, const uint8_t *Bp, const double *S, int c,
                int64_t n, int64_t nloc, double s, double *Vpart, size_t cap, cudaEvent_t ev0,
                cudaEvent_t ev1);
// The operator of one call: on the fly -> tc_prepare; stored -> the int8 K slices (k2tc) when
// INT8EXACT applies to c columns, else the fp32 stored K (*Kst, this rank's rows; null if none).
TcOperand prepare_operator(bbmm_ctx_s *ctx, bool stored, const float *X, const float *Xs, int dp,
                           int64_t n, int d, int c, const Hyper &h, int64_t r0, int64_t nloc,
                           int64_t npad_rows, float **Kst);

// ------------------------------------------------------- pivchol.cu
void pivchol(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const Hyper &h, int k,
             double *L, int64_t *piv_h, int *k_used_h, double *resid_h);

// ----------------------------------------------------------- mbcg.cu
struct MbcgArgs {
    const float *Xs; int dp; int kind; double s;   // on-the-fly operator
    TcOperand tc;                                   // tensor-core operand (version 0: none)
    const float *Kst;                               // stored operator (or null)
    int64_t n; int64_t r0; int64_t nloc; int64_t nb;
    double noise_var;
    const double *L; int k;                         // k x n (full), k == 0: no precond
    int c;                                          // columns
    int max_iter; double tol;
    const double *sor_B = nullptr; int sor_m = 0;   // SoR operator Bs (m x n), row f4
};
struct MbcgOut {
    double *U = nullptr; int64_t ldu = 0;   // optional copy of the solves
    double *Z0 = nullptr;  // optional: initial Phat^{-1} B (nloc x c), may be null
    // device-resident results (workspace; valid until the next library call)
    const double *U_d = nullptr;       // nloc x c solves
    const double *R_d = nullptr;       // nloc x c recurrence residuals B - Khat U
    const double *ahist_d = nullptr;   // max_iter x c
    const double *bhist_d = nullptr;
    const MbcgState *state_d = nullptr;
    std::vector<double> alpha, beta, relres, rho0;
    std::vector<double> relres_hist;   // max_iter x c: relres after each iteration (0: frozen)
    std::vector<int> iters;
    int iters_run = 0;
    float ms_matmul = 0.f;
    int matmul_launches = 0;
    // defer_host: mbcg_run returns without the host copies / stream sync; the caller runs
    // mbcg_finish after its own synchronisation (alpha, beta, relres, iters, ms_matmul and the
    // breakdown check are valid only after that)
    bool defer_host = false;
    const double *rhist_d_ = nullptr;
    int c_ = 0, max_iter_ = 0;
    int n_ev_ = 0;   // ctx->mm_events[0, n_ev_) bracket the matmuls of this run (pairs)
};
cudaEvent_t mm_event(bbmm_ctx_s *ctx, size_t i);
void comm_events_reserve(bbmm_ctx_s *ctx, size_t n);
void precond_setup(bbmm_ctx_s *ctx, const double *L, int64_t n, int k, double noise_var,
                   double *cholC, double *logdet_d);
// sor.cu: Bs = Lu^{-1} K_UX (m x n fp64, replicated), K_SoR = Bs^T Bs
void sor_setup(bbmm_ctx_s *ctx, const float *X, int64_t n, int d, const float *U, int m,
               const Hyper &h, double *Bs);
// pivchol.cu: rank-k pivoted Cholesky of K_SoR = Bs^T Bs through its rows
void pivchol_sor(bbmm_ctx_s *ctx, const double *Bs, int64_t n, int m, double s, int k, double *L,
                 int64_t *piv_h, int *k_used_h, double *resid_h);
// predict.cu: mean and pointwise variance (var may be null)
void predict_run(bbmm_ctx_s *ctx, const float *X, const float *y, int64_t n, int d,
                 const float *Xstar, int64_t nstar, const Hyper &h, bool stored, int k,
                 int max_iter, double tol, double *mean, double *var, double *cov = nullptr);
// mbcg_fused.cu: one cooperative kernel per iteration for the vector work (single rank)
struct FusedPlan {
    bool ok = false;
    void *fn = nullptr;
    int G = 0, mpt = 1, KT = 32;
    int64_t rpb = 0;
    size_t smem = 0;
};
struct FusedIo {
    MbcgState *st;
    const double *Vpart;
    int splits, cs, c, k;
    int64_t nloc, n;
    double noise_var, tol;
    double *D, *V, *U, *R, *Z;
    const double *L, *Cinv;
    double *ahist, *bhist, *rhist, *part, *partW, *red;
    void *Dm;
    int dm_f32;
    uint8_t *Bp;   // null: no tensor-core operand
    int nd, nb_rows;
    double *Stc;
    int64_t pad_end;
    int cb;        // columns of the tensor-core instantiation (constant column at cb)
};
bool mbcg_fused_applicable(const bbmm_ctx_s *ctx, int c, int k, bool use_sor, int64_t nloc);
FusedPlan mbcg_fused_plan(bbmm_ctx_s *ctx, int64_t nloc, int c, int k, const double *cholC,
                          double *Cinv);
void mbcg_fused_iteration(bbmm_ctx_s *ctx, const FusedPlan &p, const FusedIo &io);

void mbcg_finish(bbmm_ctx_s *ctx, MbcgOut &out);
void mbcg_run(bbmm_ctx_s *ctx, const MbcgArgs &a, const double *B, int64_t ldb,
              const double *cholC, MbcgOut &out);
void make_probes(bbmm_ctx_s *ctx, const int8_t *eps, uint64_t seed, int64_t n, int kgen,
                 int t, const double *L, int k_used, double sigma, int64_t r0, int64_t nloc,
                 const float *y, double *B, int c);

// -------------------------------------------------------------- slq.cu
void slq_logdet(bbmm_ctx_s *ctx, const double *alpha_d, const double *beta_d,
                const int *iters_d, const double *omega_d, int p, int c, int col0, int t,
                double *out_d, int *status_d);

// ------------------------------------------------------------ deriv.cu
void derivative_pass(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n,
                     int64_t r0, int64_t nloc, const float *A32, const float *B32, int cp,
                     int nq_out, bool ard, int d, double *part, int *nblocks_out);
size_t derivative_part_elems(int64_t n, int64_t nloc, int dp);
// deriv_tc.cu: the same pass with the bilinear weights W = A B^T on the tensor cores
bool deriv_tc_supported(int kind, int dp, int cp, int64_t n);
size_t deriv_tc_part_elems(int64_t n, int64_t nloc, int dp);
int derivative_pass_tc(bbmm_ctx_s *ctx, int kind, const float *Xs, int dp, int64_t n, int64_t r0,
                       int64_t nloc, const float *A32, const float *B32, int cp, int c,
                       double *part);
void reduce_blocks(bbmm_ctx_s *ctx, const double *part, int nblk, int m, double *red);
// deriv_tc2.cu: the RBF-ARD derivative as tensor-core products (expanded square, M = k~ o W)
bool deriv_tc2_supported(int kind, int n_ls, int d, int dp, int c, int64_t n);
size_t deriv_tc2_part_elems(int64_t n, int64_t nloc, int dp);
void derivative_pass_tc2(bbmm_ctx_s *ctx, const float *Xa, int d, int dp, int64_t n, int64_t r0,
                         int64_t nloc, const float *A32, const float *B32, int cs, int c,
                         const double *U, const double *R, const double *Bblk, const double *Z0,
                         double noise_var, double s, double *part, double *red);

// ------------------------------------------------------------- comm
// A context communicates when it has an NCCL communicator (also a 1-rank one, which issues
// every collective as on G ranks) or an in-process rank group.
inline bool has_comm(const bbmm_ctx_s *ctx) { return ctx->comm != nullptr || ctx->local != nullptr; }
void allreduce_sum(bbmm_ctx_s *ctx, double *buf, size_t count);
void allgather_rows(bbmm_ctx_s *ctx, void *buf, size_t bytes_per_rank);
void comm_timing_reset(bbmm_ctx_s *ctx);
double comm_timing_ms(bbmm_ctx_s *ctx);   // after a stream sync

}  // namespace bbmm
