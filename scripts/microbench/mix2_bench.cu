// microbenchmark (round 2): MUFU ex2 throughput under per-pair ALU mixes that K1-TC designs need.
// Per group of 4 pairs (one per lane, 8 groups per iteration):
//   0  ex2 only                         5  ex2 + FADD + 5 PRMT (two mixed-slice + one pure cell)
//   1  ex2 + FADD                        6  ex2 + FADD2 + 7 PRMT
//   2  ex2 + FADD2 (pairs of points)     7  ex2.f16x2 only (2 results per op)
//   3  ex2 + FADD + 4 PRMT               8  ex2 + FADD + 7 PRMT, 2 warps' worth of ILP (32 regs)
//   4  ex2 + FADD + 7 PRMT (round 1)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb2 mix2_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

template <int MODE>
__global__ void kb(uint32_t *out, int iters, float seed) {
    uint32_t acc = 0;
    float sv[32];
#pragma unroll
    for (int i = 0; i < 32; i++) sv[i] = -seed * (threadIdx.x + i) * 1e-3f;
    unsigned long long two2;
    asm("mov.b64 %0, {%1, %1};" : "=l"(two2) : "f"(2.0f));
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            uint32_t q[4];
            if (MODE == 7) {
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    uint32_t h = ex2h2(__float_as_uint(sv[4 * u + 2 * v]) ^ (it & 1));
                    q[2 * v] = h;
                    q[2 * v + 1] = h >> 3;
                }
            } else if (MODE == 2 || MODE == 6) {
#pragma unroll
                for (int v = 0; v < 4; v += 2) {
                    const float k0 = ex2a(sv[4 * u + v]), k1 = ex2a(sv[4 * u + v + 1]);
                    unsigned long long kk, r;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(kk) : "f"(k0), "f"(k1));
                    r = fadd2(kk, two2);
                    q[v] = (uint32_t)r;
                    q[v + 1] = (uint32_t)(r >> 32);
                }
            } else {
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const float k = ex2a(sv[4 * u + v]);
                    q[v] = MODE == 0 ? __float_as_uint(k) : __float_as_uint(k + 2.0f);
                }
            }
            if (MODE <= 2 || MODE == 7) {
                acc += q[0] ^ q[1] ^ q[2] ^ q[3];
                continue;
            }
            if (MODE == 3) {
                const uint32_t t01 = __byte_perm(q[0], q[1], 0x5140), t23 = __byte_perm(q[2], q[3], 0x5140);
                acc ^= __byte_perm(t01, t23, 0x5410) + __byte_perm(t01, t23, 0x7632);
                continue;
            }
            if (MODE == 5) {
                const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240), t23 = __byte_perm(q[2], q[3], 0x6240);
                const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351), u23 = __byte_perm(q[2], q[3], 0x7351);
                acc ^= t01 + t23 + __byte_perm(u01, u23, 0x5410);
                continue;
            }
            const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240), t23 = __byte_perm(q[2], q[3], 0x6240);
            const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351), u23 = __byte_perm(q[2], q[3], 0x7351);
            acc ^= __byte_perm(t01, t23, 0x5410) + __byte_perm(t01, t23, 0x7632) +
                   __byte_perm(u01, u23, 0x5410);
        }
#pragma unroll
        for (int i = 0; i < 32; i++) sv[i] = __uint_as_float(__float_as_uint(sv[i]) ^ (acc & 1));
    }
    if (acc == 0x12345) out[threadIdx.x] = 1;
}

template <int M>
void run(uint32_t *o, int warps, int iters, const char *what) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kb<M><<<148, warps * 32>>>(o, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    kb<M><<<148, warps * 32>>>(o, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ex = 148.0 * warps * 32 * 32.0 * iters;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("mode %d %-34s warps/SM %2d: %.3f ms, %.2f pairs/clk/SM (at %d MHz)\n", M, what, warps, ms,
           ex / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
}

int main() {
    uint32_t *o;
    cudaMalloc(&o, 4096 * 4);
    for (int w : {16, 32}) {
        run<0>(o, w, 20000, "ex2");
        run<1>(o, w, 20000, "ex2+FADD");
        run<2>(o, w, 20000, "ex2+FADD2");
        run<3>(o, w, 20000, "ex2+FADD+4PRMT");
        run<5>(o, w, 20000, "ex2+FADD+5PRMT");
        run<4>(o, w, 20000, "ex2+FADD+7PRMT (r1 kernel)");
        run<6>(o, w, 20000, "ex2+FADD2+7PRMT");
        run<7>(o, w, 20000, "ex2.f16x2 (pairs = 2 per op)");
    }
    return 0;
}
