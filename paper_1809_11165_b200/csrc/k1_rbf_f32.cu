// k1_rbf_f32.cu -- instantiations of K1 (RBF, fp32-chunked accumulation).
#include "k1_kernels.cuh"

namespace bbmm {
void launch_k1_rbf_f32(bbmm_ctx_s *ctx, int dp, int cp, const float *Xs, int64_t n, int64_t r0,
                      int64_t nloc, const void *Dm, double s, double *Vpart, int splits) {
    launch_k1_variant<0, false>(ctx, dp, cp, Xs, n, r0, nloc, Dm, s, Vpart, splits);
}
}  // namespace bbmm
