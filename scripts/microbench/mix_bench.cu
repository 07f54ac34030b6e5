// microbenchmark: the K1-TC per-tile warp body (LDTM.x32 -> ex2/quantise -> STTM) without MMAs/barriers
#include <cstdio>
#include <cstdint>
#include "../../paper_1809_11165_b200/csrc/sm100_ptx.cuh"
using namespace bbmm;
__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// MODE 0: no TMEM (registers only)  1: LDTM + STTM x8 x3 + wait::st   2: LDTM + STTM (wait deferred one iter)
// 3: LDTM only   4: STTM x32 single + wait   5: STTM x8 x3, no wait at all
template <int MODE>
__global__ void __launch_bounds__(512, 1) km(int iters, uint32_t *out) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&tb);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + 32 * (warp >> 2);
    uint32_t sv[32], acc = 0;
    for (int i = 0; i < 32; i++) sv[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
    if (MODE != 0) for (int b = 0; b < 4; b++) { ptx::tmem_st8(base + 128 * b, *reinterpret_cast<uint32_t(*)[8]>(sv)); ptx::tmem_st8(base + 128 * b + 8, *reinterpret_cast<uint32_t(*)[8]>(sv)); ptx::tmem_st8(base + 128 * b + 16, *reinterpret_cast<uint32_t(*)[8]>(sv)); ptx::tmem_st8(base + 128 * b + 24, *reinterpret_cast<uint32_t(*)[8]>(sv)); }
    ptx::tmem_st_wait();
    for (int it = 0; it < iters; it++) {
        const uint32_t col = base + 128 * (it & 3);
        if (MODE != 0) { ptx::tmem_ld32(col, sv); ptx::tmem_ld_wait(); }
        uint32_t w0[8], w1[8], w2[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            uint32_t q[4];
#pragma unroll
            for (int v = 0; v < 4; v++) q[v] = __float_as_uint(ex2a(__uint_as_float(sv[4 * u + v] & 0xBFFFFFFFu)) + 2.0f);
            const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240), t23 = __byte_perm(q[2], q[3], 0x6240);
            const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351), u23 = __byte_perm(q[2], q[3], 0x7351);
            w0[u] = __byte_perm(t01, t23, 0x5410); w2[u] = __byte_perm(t01, t23, 0x7632); w1[u] = __byte_perm(u01, u23, 0x5410);
        }
        if (MODE == 0 || MODE == 3) { for (int u = 0; u < 8; u++) acc ^= w0[u] + w1[u] + w2[u]; if (MODE == 0) for (int i = 0; i < 32; i++) sv[i] ^= (acc & 1); continue; }
        if (MODE == 2) ptx::tmem_st_wait();
        if (MODE == 4) {
            uint32_t w[32];
            for (int u = 0; u < 8; u++) { w[u] = w0[u]; w[8 + u] = w1[u]; w[16 + u] = w2[u]; w[24 + u] = 0; }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                         ::"r"(col), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
                           "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]) : "memory");
            ptx::tmem_st_wait();
            continue;
        }
        ptx::tmem_st8(col, w0); ptx::tmem_st8(col + 8, w1); ptx::tmem_st8(col + 16, w2);
        if (MODE == 1) ptx::tmem_st_wait();
    }
    ptx::tmem_st_wait();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tb); }
}
template <int M> void run(uint32_t *o, int warps, int iters) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    km<M><<<148, warps * 32>>>(iters, o); cudaDeviceSynchronize();
    cudaEventRecord(a); km<M><<<148, warps * 32>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("mode %d warps %2d: %.3f ms  %.2f elem/clk/SM  (%.0f clk per 128x128 tile)  %s\n", M, warps, ms,
           32.0 * 32 * warps * iters / cyc / 148 * 148, 16384.0 / (32.0 * 32 * warps * iters / cyc), cudaGetErrorString(cudaGetLastError()));
}
int main() {
    uint32_t *o; cudaMalloc(&o, 148 * 1024 * 4);
    printf("0 regs only | 1 ld+st+wait | 2 ld+st (wait next iter) | 3 ld only | 4 st.x32+wait | 5 st no wait\n");
    run<0>(o, 16, 20000); run<1>(o, 16, 20000); run<2>(o, 16, 20000); run<3>(o, 16, 20000); run<4>(o, 16, 20000); run<5>(o, 16, 20000);
    return 0;
}
