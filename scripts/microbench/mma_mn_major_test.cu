// Probe: kind::tf32 MMA with A from TMEM and B from shared memory in the MN-major SWIZZLE_NONE
// ("interleave") layout -- does it compute D = A B, and with which LBO / SBO reading?
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1809_11165_b200/csrc \
//        -o /tmp/mnt scripts/microbench/mma_mn_major_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "sm100_ptx.cuh"
using namespace bbmm;

constexpr int M = 128, N = 64, K = 8;
// B element (n, k) at: (n / 4) * SBO + k * 16 + (n % 4) * 4   (k < 8: one K group)
__global__ void probe(const float *A, const float *B, float *D, int variant) {
    __shared__ __align__(1024) float bs[N * K];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ __align__(1024) float as_[M * K];
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int n = e / K, k = e % K;
        if (variant == 3)   // K-major: [k / 4][n][4]
            bs[(k / 4) * (N * 4) + n * 4 + (k % 4)] = B[n * K + k];
        else                // MN-major: [n / 4][k][4]
            bs[(n / 4) * (8 * 4) + k * 4 + (n % 4)] = B[n * K + k];
    }
    for (int e = tid; e < M * K; e += blockDim.x) {   // A K-major in smem: [k / 4][m][4]
        const int m = e / K, k = e % K;
        as_[(k / 4) * (M * 4) + m * 4 + (k % 4)] = A[m * K + k];
    }
    if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc<128>(&tb);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = tb;
    // A rows -> TMEM lanes (warp w: lanes 32w..), columns 0..7 ; zero D columns 64..127
    {
        uint32_t r[8];
        for (int k = 0; k < 8; k++) r[k] = __float_as_uint(A[(warp * 32 + lane) * K + k]);
        ptx::tmem_st8(t + ((uint32_t)(warp * 32) << 16), r);
        uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int q = 0; q < 64; q += 8) ptx::tmem_st8(t + ((uint32_t)(warp * 32) << 16) + 64 + q, z);
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) {
        // v0: both 128 (either reading works); v1: SBO = the MN-chunk stride; v2: LBO = it
        uint32_t lbo = 128, sbo = 128;
        if (variant == 1) { lbo = 4096; sbo = 128; }
        if (variant == 2) { lbo = 128; sbo = 4096; }
        const uint32_t idesc = ptx::idesc_tf32(M, N) | (variant == 3 ? 0u : (1u << 16));
        if (variant == 3) { lbo = N * 16; sbo = 128; }
        if (ptx::elect_one()) {
            const uint64_t bd = ptx::smem_desc_kmajor(ptx::smem_u32(bs), lbo, sbo);
            if (variant == 4)
                ptx::mma_tf32_ss(t + 64, ptx::smem_desc_kmajor(ptx::smem_u32(as_), M * 16, 128), bd, idesc, 1u);
            else
                ptx::mma_tf32_ts(t + 64, t, bd, idesc, 1u);
            ptx::mma_commit(&bar);
        }
        __syncwarp();
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    if (warp < 4) {
        uint32_t v[32];
        for (int h = 0; h < 2; h++) {
            ptx::tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + 64 + 32 * h, v);
            ptx::tmem_ld_wait();
            for (int q = 0; q < 32; q++) D[(warp * 32 + lane) * N + 32 * h + q] = __uint_as_float(v[q]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<128>(t); }
}

int main() {
    float *A, *B, *D;
    cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&B, N * K * 4); cudaMallocManaged(&D, M * N * 4);
    for (int i = 0; i < M * K; i++) A[i] = (float)((i * 7) % 13 - 6);
    for (int i = 0; i < N * K; i++) B[i] = (float)((i * 5) % 11 - 5);
    for (int v = 0; v < 5; v++) {
        for (int i = 0; i < M * N; i++) D[i] = -999.f;
        probe<<<1, 128>>>(A, B, D, v);
        cudaError_t e = cudaDeviceSynchronize();
        double err = 0, mx = 0;
        for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
                double r = 0;
                for (int k = 0; k < K; k++) r += (double)A[m * K + k] * B[n * K + k];
                err = fmax(err, fabs(r - D[m * N + n]));
                mx = fmax(mx, fabs(r));
            }
        printf("variant %d: %s max|err| %.3g (max|ref| %.3g) D[0]=%g D[1]=%g\n", v, cudaGetErrorString(e), err, mx,
               D[0], D[1]);
    }
    return 0;
}
