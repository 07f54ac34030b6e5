// microbenchmark (round 2, re-entry): where does K1-TC's per-entry kernel-value error come from, and
// what does a finer k~ grid cost?
// (A) precision over C4-shaped pairs (x ~ N(0, I_3), l = 2 sqrt 3, s = 1): per pair the exact
//     k = exp(-r^2/2) (fp64) against
//       e_in   : 2^S32 with S32 = fp32(S) (the exponent rounded to fp32 only)
//       e_mufu : ex2.approx.ftz.f32(S32) (the MUFU, given the fp32-rounded exponent)
//       e_q23  : the MUFU value on the kernel's 23-bit grid (q = 2 + 2k, low 3 bytes)
//       e_q31  : the MUFU value on a 31-bit grid (23-bit truncated part + a residual byte)
//       e_f32d : fp32 direct-difference distance (the CUDA-core operator's S) then MUFU, no grid
//     rms / max absolute error and the mean (bias), relative to s.
// (B) MUFU throughput with the per-pair mixes: current (FFMA2 + 7 PRMT per 4 pairs) and the
//     31-bit grid (rz FFMA2 q, FFMA2 -k^, FADD2 r, FFMA2 byte, + 3 PRMT per 4 pairs).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pb prec_bench.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef unsigned long long u64;
__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(u64 v, uint32_t &a, uint32_t &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
}

// ---------------------------------------------------------------- (A) precision
struct Acc {
    double s2[5], mx[5], s1[5];
};
__global__ void kprec(const double *X, int n, double scl, int64_t npairs, uint64_t seed, double *out) {
    double s2[5] = {0}, mx[5] = {0}, s1[5] = {0};
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = seed + p * 0x9E3779B97F4A7C15ull;
        h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
        h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
        h ^= h >> 31;
        const int i = (int)(h % n), j = (int)((h >> 32) % n);
        double r2 = 0.0;
        float r2f = 0.0f;
        for (int q = 0; q < 3; q++) {
            const double dx = (X[3 * i + q] - X[3 * j + q]) * scl;
            r2 += dx * dx;
            const float df = (float)(X[3 * i + q] * scl) - (float)(X[3 * j + q] * scl);
            r2f = fmaf(df, df, r2f);
        }
        const double k = exp(-0.5 * r2);
        const double S = -0.5 * r2 / log(2.0);
        const float S32 = (float)S;
        const double e_in = exp2((double)S32) - k;
        const float km = ex2a(S32);
        const double e_mufu = (double)km - k;
        const double q23 = rint((double)km * 8388608.0) / 8388608.0;
        const double e_q23 = q23 - k;
        // 31-bit grid as the kernel would form it: q = fma.rz(k, 2, 2); -k^ = 1 - q/2; r = k - k^;
        // byte = floor(r 2^31)
        const float qz = __fmaf_rz(km, 2.0f, 2.0f);
        const float nk = fmaf(-0.5f, qz, 1.0f);
        const float rr = nk + km;
        const float bz = __fmaf_rz(rr, 2147483648.0f, 8388608.0f);
        const uint32_t byte = __float_as_uint(bz) & 0xFFu;
        const uint32_t hi = __float_as_uint(qz) & 0x7FFFFFu;
        const uint32_t hi24 = (__float_as_uint(qz) >> 23) == 129 ? 0x800000u : hi;   // q = 4: k = 1
        const double q31 = (double)hi24 / 8388608.0 + (double)byte / 2147483648.0;
        const double e_q31 = q31 - k;
        const float S32d = -0.72134752044448170f * r2f;   // -(log2 e / 2) r^2 in fp32
        const double e_f32d = (double)ex2a(S32d) - k;
        const double e[5] = {e_in, e_mufu, e_q23, e_q31, e_f32d};
        for (int m = 0; m < 5; m++) {
            s2[m] += e[m] * e[m];
            s1[m] += e[m];
            mx[m] = fmax(mx[m], fabs(e[m]));
        }
    }
    for (int m = 0; m < 5; m++) {
        atomicAdd(&out[m], s2[m]);
        atomicAdd(&out[5 + m], s1[m]);
        // max: via bits of a non-negative double
        atomicMax(reinterpret_cast<unsigned long long *>(&out[10 + m]), __double_as_longlong(mx[m]));
    }
}

// also the bare MUFU error over a dense grid of exponents in [-8, 0]
__global__ void kgrid(int64_t m, double *out) {
    double s2 = 0, s1 = 0, mx = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const float x = -8.0f * (float)((double)p / (double)m);
        const double ex = exp2((double)x);
        const double rel = ((double)ex2a(x) - ex) / ex;
        s2 += rel * rel;
        s1 += rel;
        mx = fmax(mx, fabs(rel));
    }
    atomicAdd(&out[0], s2);
    atomicAdd(&out[1], s1);
    atomicMax(reinterpret_cast<unsigned long long *>(&out[2]), __double_as_longlong(mx));
}

// ---------------------------------------------------------------- (B) throughput
template <int MODE>
__global__ void kb(uint32_t *out, int iters, float seed) {
    uint32_t acc = 0;
    float sv[32];
#pragma unroll
    for (int i = 0; i < 32; i++) sv[i] = -seed * (threadIdx.x + i) * 1e-3f;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            uint32_t q[4], rb[4];
#pragma unroll
            for (int v = 0; v < 4; v += 2) {
                const float k0 = ex2a(sv[4 * u + v]), k1 = ex2a(sv[4 * u + v + 1]);
                u64 kk = pk(k0, k1), qq;
                if (MODE == 0) {
                    asm("fma.rn.f32x2 %0, %1, %2, %2;" : "=l"(qq) : "l"(kk), "l"(0x4000000040000000ull));
                } else {
                    asm("fma.rz.f32x2 %0, %1, %2, %2;" : "=l"(qq) : "l"(kk), "l"(0x4000000040000000ull));
                    u64 nk, rr, bb;
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(nk) : "l"(qq), "l"(0xBF000000BF000000ull),
                        "l"(0x3F8000003F800000ull));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(nk), "l"(kk));
                    asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(bb) : "l"(rr), "l"(0x4F0000004F000000ull),
                        "l"(0x4B0000004B000000ull));
                    upk(bb, rb[v], rb[v + 1]);
                }
                upk(qq, q[v], q[v + 1]);
            }
            const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240), t23 = __byte_perm(q[2], q[3], 0x6240);
            const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351), u23 = __byte_perm(q[2], q[3], 0x7351);
            acc ^= __byte_perm(t01, t23, 0x5410) + __byte_perm(t01, t23, 0x7632) +
                   __byte_perm(u01, u23, 0x5410);
            if (MODE == 1) {
                const uint32_t r01 = __byte_perm(rb[0], rb[1], 0x0040), r23 = __byte_perm(rb[2], rb[3], 0x0040);
                acc += __byte_perm(r01, r23, 0x5410);
            }
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
    printf("{\"bench\": \"mix\", \"mode\": %d, \"what\": \"%s\", \"warps\": %d, \"ms\": %.3f, "
           "\"pairs_per_clk_sm_at_1965\": %.3f}\n", M, what, warps, ms, ex / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    // C4-shaped points
    const int n = 1 << 20;
    std::vector<double> X(3 * (size_t)n);
    srand(1);
    for (auto &v : X) {
        double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
        v = sqrt(-2 * log(u1)) * cos(2 * M_PI * u2);
    }
    double *Xd, *out;
    cudaMalloc(&Xd, X.size() * 8);
    cudaMemcpy(Xd, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 32 * 8);
    cudaMemset(out, 0, 32 * 8);
    const int64_t np = 1ll << 28;
    kprec<<<148 * 8, 256>>>(Xd, n, 1.0 / (2.0 * sqrt(3.0)), np, 12345, out);
    double h[32];
    cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
    const char *nm[5] = {"e_in (fp32 exponent, exact exp)", "e_mufu (ex2.approx of fp32 S)",
                         "e_q23 (MUFU on the 23-bit grid)", "e_q31 (MUFU on a 31-bit grid)",
                         "e_f32d (fp32 direct distance + MUFU)"};
    for (int m = 0; m < 5; m++)
        printf("{\"bench\": \"prec\", \"what\": \"%s\", \"rms\": %.3e, \"mean\": %.3e, \"max\": %.3e}\n", nm[m],
               sqrt(h[m] / np), h[5 + m] / np, h[10 + m]);
    cudaMemset(out, 0, 32 * 8);
    const int64_t mg = 1ll << 26;
    kgrid<<<148 * 8, 256>>>(mg, out);
    cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"mufu_rel_grid\", \"range\": \"[-8, 0]\", \"rms\": %.3e, \"mean\": %.3e, \"max\": %.3e}\n",
           sqrt(h[0] / mg), h[1] / mg, h[2]);
    uint32_t *o;
    cudaMalloc(&o, 4096 * 4);
    for (int w : {16}) {
        run<0>(o, w, 20000, "ex2 + FFMA2 q + 7 PRMT (kernel now)");
        run<1>(o, w, 20000, "31-bit grid: + 3 f32x2 + 3 PRMT");
    }
    return 0;
}
