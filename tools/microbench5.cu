// MUFU.EX2 throughput on one B200: independent ex2.approx.ftz.f32 chains,
// fp32 and packed f16x2, 148 x 512 threads.
#include <cstdio>
__global__ void ex2_f32(float* out, int iters) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ex2_f16x2(unsigned* out, int iters) {
    unsigned x[8];
    for (int i = 0; i < 8; ++i) x[i] = 0xB800B800u + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
    unsigned s = 0;
    for (int i = 0; i < 8; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 512 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        ex2_f32<<<148, 512>>>(o, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double n = 148.0 * 512 * 8 * iters;
        printf("ex2.f32: %.3f ms, %.1f per clk per SM at 1.9 GHz\n", ms, n / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(a);
        ex2_f16x2<<<148, 512>>>((unsigned*)o, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ex2.f16x2: %.3f ms, %.1f instr per clk per SM (x2 values)\n", ms, n / (ms * 1e-3) / 148 / 1.9e9);
    }
    return 0;
}
