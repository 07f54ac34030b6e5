// Relative error of ex2.approx.ftz.f32 over x in [-1, 0) on a 2^22-point grid (every fp32 value of
// the grid's spacing), written to gpurun_out/mufu_err.bin as float32 for offline analysis:
// how much of the MUFU's error is a smooth function of the fractional part (correctable) and how
// much is point-to-point noise.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/me mufu_err_map.cu
#include <cmath>
#include <cstdio>
#include <vector>
__global__ void k(float *out, int m) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        const float x = -(float)p / (float)m;
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        out[p] = (float)((double)y / exp2((double)x) - 1.0);
    }
}
int main() {
    const int m = 1 << 22;
    float *d;
    cudaMalloc(&d, m * 4);
    k<<<148 * 8, 256>>>(d, m);
    std::vector<float> h(m);
    cudaMemcpy(h.data(), d, m * 4, cudaMemcpyDeviceToHost);
    FILE *f = fopen("gpurun_out/mufu_err.bin", "wb");
    fwrite(h.data(), 4, m, f);
    fclose(f);
    printf("ok\n");
}
