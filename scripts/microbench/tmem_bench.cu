// microbenchmark: tcgen05.ld / tcgen05.st throughput on one SM (16 warps, 1 CTA/SM)
#include <cstdio>
#include <cstdint>
#include "../../paper_1809_11165_b200/csrc/sm100_ptx.cuh"
using namespace bbmm;
template <int MODE>
__global__ void __launch_bounds__(512, 1) kt(int iters, uint32_t *out) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&tb);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + 32 * (warp >> 2);
    uint32_t r[32], acc = 0;
    for (int i = 0; i < 32; i++) r[i] = i * threadIdx.x;
    for (int it = 0; it < iters; it++) {
        const uint32_t col = base + 128 * (it & 3);
        if (MODE == 0 || MODE == 2) { ptx::tmem_ld32(col, r); ptx::tmem_ld_wait(); acc += r[0] ^ r[17] ^ r[31]; }
        if (MODE == 1 || MODE == 2) {
            uint32_t w[8];
            for (int q = 0; q < 8; q++) w[q] = r[q] + acc;
            ptx::tmem_st8(col, w); ptx::tmem_st8(col + 8, w); ptx::tmem_st8(col + 16, w);
            if (MODE == 1) ptx::tmem_st_wait();
        }
        if (MODE == 2) ptx::tmem_st_wait();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tb); }
}
template <int M> void run(uint32_t *o, int warps, int iters) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kt<M><<<148, warps * 32>>>(iters, o); cudaDeviceSynchronize();
    cudaEventRecord(a); kt<M><<<148, warps * 32>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes_ld = (M == 0 || M == 2) ? 4096.0 : 0, bytes_st = (M >= 1) ? 3072.0 : 0;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("mode %d warps %2d: %.3f ms  LD %.1f B/clk/SM  ST %.1f B/clk/SM  (per warp-iter %.0f clk)  err %s\n", M, warps, ms,
           bytes_ld * warps * iters / cyc, bytes_st * warps * iters / cyc, cyc / iters, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    uint32_t *o; cudaMalloc(&o, 148 * 1024 * 4);
    for (int w : {4, 8, 16}) { run<0>(o, w, 20000); run<1>(o, w, 20000); run<2>(o, w, 20000); }
    return 0;
}
