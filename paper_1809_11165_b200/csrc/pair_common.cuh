// pair_common.cuh -- device helpers for the pairwise kernel-evaluation kernels
// (kernel matmul K1, stored-K build K2, derivative pass K7).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bbmm {

// Compile-time shapes of the fp32 pair kernels.  D = input dims handled by an
// instantiation (inputs padded with zero coordinates up to D), CP = columns
// (padded with zero columns up to CP).  Row strides in memory are rounded up
// to a multiple of 4 floats so tiles move with 16-byte loads.
__host__ __device__ constexpr int round4(int x) { return (x + 3) & ~3; }

// ex2.approx: 2^x on the MUFU pipe (~2 ulp), flush-to-zero for tiny results.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Round an fp32 value to the nearest tf32 (10 explicit mantissa bits) for the 3xTF32 splits
// x = hi + lo: hi rounded (|lo| <= 2^-11 |x|) and lo rounded too (the MMA would truncate its
// low 13 bits), so hi + lo matches x to ~2^-22 |x| -- truncating both left ~2^-20.
__host__ __device__ __forceinline__ float tf32_rn(float x) {
#ifdef __CUDA_ARCH__
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
#else
    uint32_t u;
    __builtin_memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    __builtin_memcpy(&r, &u, 4);
    return r;
#endif
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Kernel value from the scaled squared distance (see bbmm_internal.cuh Hyper):
//   RBF:    xs = x sqrt(log2 e / 2)/l :  k/s = 2^(-rs2)
//   Matern: xs = x sqrt(5)/l, rh = sqrt(rs2) :  k/s = (1 + rh + rh^2/3) 2^(-rh log2 e)
template <int KIND>
__device__ __forceinline__ float kval_scaled(float rs2) {
    if (KIND == 0) {
        return ex2_approx(-rs2);
    } else {
        float rh = sqrt_approx(rs2);
        float e = ex2_approx(-1.4426950408889634f * rh);
        return fmaf(rs2, 0.33333333333333333f, rh + 1.0f) * e;
    }
}

// Matern derivative factor g/s = (5/3)(1 + rh) e^{-rh}; with xs scaled by
// sqrt5/l, dK/dlog l_q = s g * diff_q^2/l_q^2 = s * (1/3)(1 + rh) e^{-rh} * dxs_q^2.
template <int KIND>
__device__ __forceinline__ void kval_and_dfac(float rs2, float &k, float &g) {
    if (KIND == 0) {
        k = ex2_approx(-rs2);
        g = k;   // RBF: dK/dlog l_q = K * diff_q^2/l_q^2 = K * dxs_q^2 / (log2e/2)
    } else {
        float rh = sqrt_approx(rs2);
        float e = ex2_approx(-1.4426950408889634f * rh);
        k = fmaf(rs2, 0.33333333333333333f, rh + 1.0f) * e;
        g = (rh + 1.0f) * e;   // times (1/3) applied on the host side
    }
}

}  // namespace bbmm
