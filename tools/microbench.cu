// microbench.cu -- issue-rate probes that decide the decode kernel's design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu && ./mb
// HMMA (mma.sync m16n8k16 f16->f32), FADD2, LOP3+SHF code extraction.
#include <cstdio>
#include <cuda_fp16.h>

__global__ void hmma_loop(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x3800;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void hmma16_loop(float* out, int iters) {  // f16 accumulate
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x3800;
    unsigned c[8][2] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                : "+r"(c[k][0]), "+r"(c[k][1])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= c[k][0] ^ c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

__global__ void fadd2_loop(float* out, int iters) {
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x + k, k);
    const float2 y = make_float2(1e-7f, -1e-7f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fadd2_rn(x[k], y);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps = 4; warps <= 32; warps *= 2) {
        float ms;
        hmma_loop<<<148, warps * 32>>>(out, 16);
        cudaEventRecord(e0);
        hmma_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double macs = 148.0 * 2 * warps * iters * 8 * 16 * 8 * 16;
        printf("HMMA f32acc warps/CTA %2d: %.1f TMAC/s (%.1f TFLOP/s)\n", warps, macs / ms / 1e9, 2 * macs / ms / 1e9);
        hmma16_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e0);
        hmma16_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("HMMA f16acc warps/CTA %2d: %.1f TMAC/s\n", warps, macs / ms / 1e9);
        fadd2_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e0);
        fadd2_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double adds = 148.0 * 2 * warps * 32 * iters * 8 * 2;
        printf("FADD2 warps/CTA %2d: %.1f T adds/s\n", warps, adds / ms / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
