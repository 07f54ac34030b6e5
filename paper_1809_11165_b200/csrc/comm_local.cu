// comm_local.cu -- in-process rank group: the collectives of the row partition
// (all-gather of the packed search directions, all-reduces of
// the per-column dots) between contexts that live in ONE process and are
// driven by one host thread each.  It exists so the multi-rank data flow --
// row ranges, all-gather layouts, which sums are reduced where -- runs on real
// GPU kernels with a single GPU (the NCCL path needs one GPU per rank).
// Collectives are synchronous and host-staged: every rank synchronises its
// stream, meets the others at a barrier, reads the peers' device buffers
// (same process: plain cudaMemcpy between device pointers), sums in rank
// order on the host (deterministic), and meets again before returning so no
// buffer is overwritten while a peer still reads it.  Not a performance path.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "bbmm_internal.cuh"

namespace bbmm {

struct LocalGroup {
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<void *> ptr;

    explicit LocalGroup(int nranks) : n(nranks), ptr(nranks, nullptr) {}

    // all n ranks arrive; times out (-> error instead of a hang) if a peer failed
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; }))
            throw Error{BBMM_ERR_NCCL, "local rank group: barrier timed out (a peer failed?)"};
    }
};

namespace {
void publish(bbmm_ctx_s *ctx, void *buf) {
    BBMM_CUDA(cudaStreamSynchronize(ctx->stream));
    {
        std::lock_guard<std::mutex> lk(ctx->local->m);
        ctx->local->ptr[ctx->rank] = buf;
    }
    ctx->local->barrier();
}

template <typename Op>
void local_allreduce(bbmm_ctx_s *ctx, double *buf, size_t count, Op op) {
    LocalGroup *g = ctx->local;
    publish(ctx, buf);
    std::vector<double> acc(count), tmp(count);
    for (int r = 0; r < g->n; r++) {            // rank order: identical result on every rank
        BBMM_CUDA(cudaMemcpy(r == 0 ? acc.data() : tmp.data(), g->ptr[r], count * 8,
                             cudaMemcpyDeviceToHost));
        if (r > 0)
            for (size_t e = 0; e < count; e++) acc[e] = op(acc[e], tmp[e]);
    }
    g->barrier();                                // every rank has read every buffer
    BBMM_CUDA(cudaMemcpy(buf, acc.data(), count * 8, cudaMemcpyHostToDevice));
    g->barrier();
}
}  // namespace

void local_allreduce_sum(bbmm_ctx_s *ctx, double *buf, size_t count) {
    local_allreduce(ctx, buf, count, [](double a, double b) { return a + b; });
}
void local_allreduce_max(bbmm_ctx_s *ctx, double *buf, size_t count) {
    local_allreduce(ctx, buf, count, [](double a, double b) { return std::max(a, b); });
}
void local_allgather(bbmm_ctx_s *ctx, void *buf, size_t bytes_per_rank) {
    LocalGroup *g = ctx->local;
    publish(ctx, buf);
    char *mine = (char *)buf;
    for (int r = 0; r < g->n; r++) {
        if (r == ctx->rank) continue;
        const char *src = (const char *)g->ptr[r] + (size_t)r * bytes_per_rank;
        BBMM_CUDA(cudaMemcpy(mine + (size_t)r * bytes_per_rank, src, bytes_per_rank,
                             cudaMemcpyDeviceToDevice));
    }
    g->barrier();                                // peers' own segments no longer read
}

}  // namespace bbmm

using namespace bbmm;

extern "C" {

bbmm_status_t bbmm_local_group_create(int32_t nranks, bbmm_local_group_t *out) {
    if (!out || nranks < 1) return BBMM_ERR_ARG;
    *out = reinterpret_cast<bbmm_local_group_t>(new LocalGroup(nranks));
    return BBMM_OK;
}

bbmm_status_t bbmm_local_group_destroy(bbmm_local_group_t group) {
    delete reinterpret_cast<LocalGroup *>(group);
    return BBMM_OK;
}

bbmm_status_t bbmm_ctx_set_local_comm(bbmm_ctx_t ctx, bbmm_local_group_t group, int32_t rank) {
    if (!ctx || !group) return BBMM_ERR_ARG;
    LocalGroup *g = reinterpret_cast<LocalGroup *>(group);
    if (rank < 0 || rank >= g->n) return BBMM_ERR_ARG;
    if (ctx->comm) {
        ncclCommDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
    ctx->local = g;
    ctx->nranks = g->n;
    ctx->rank = rank;
    return BBMM_OK;
}

}  // extern "C"
