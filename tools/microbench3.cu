// microbench3.cu -- mixed-precision FHFMA/FHADD issue rates and fp16-subnormal
// handling of FHFMA and HMMA (the decode kernel feeds 2-bit codes as fp16
// subnormals c * 2^(2e-24)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb3 tools/microbench3.cu && ./mb3
#include <cstdio>
#include <cuda_fp16.h>

#define CHAINS 8

__device__ __forceinline__ float fhfma(unsigned ab, float c) {  // lo(ab) * hi(ab) + c
    float r;
    asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; fma.rn.f32.f16 %0, lo, hi, %2;}" : "=f"(r) : "r"(ab), "f"(c));
    return r;
}
__device__ __forceinline__ float fhadd(unsigned a, float c) {  // lo(a) + c
    float r;
    asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; add.rn.f32.f16 %0, lo, %2;}" : "=f"(r) : "r"(a), "f"(c));
    return r;
}

template <int OP>
__global__ void loop(float* out, int iters) {
    float x[CHAINS];
    unsigned u[CHAINS];
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
        x[k] = threadIdx.x * 1e-3f + k;
        u[k] = 0x3C003C01u + k;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) {
            if (OP == 0) x[k] = fhfma(u[k], x[k]);
            if (OP == 1) x[k] = fhadd(u[k], x[k]);
        }
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void subnormal_probe(float* out) {
    // FHFMA: 1.5 (fp16) * (3 * 2^-24, subnormal) + 0
    const unsigned ab = (0x0003u << 16) | 0x3E00u;
    out[0] = fhfma(ab, 0.0f);
    // HMMA m16n8k16: A = all 1.5, B = all 3 * 2^-24 (subnormal); D[0] = 16 * 4.5 * 2^-24
    const unsigned a = 0x3E003E00u, b = 0x00030003u;
    float d0 = 0, d1 = 0, d2 = 0, d3 = 0;
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
                 : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
    if (threadIdx.x == 0) out[1] = d0;
    // HMMA with subnormal codes of magnitude 2^-24 * 1 and larger weights 1000
    const unsigned a2 = 0x63D063D0u /* 1000 */, b2 = 0x00010001u;
    d0 = d1 = d2 = d3 = 0;
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
                 : "r"(a2), "r"(a2), "r"(a2), "r"(a2), "r"(b2), "r"(b2));
    if (threadIdx.x == 0) out[2] = d0;
}

template <int OP>
void run(const char* name, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048, threads = 512, blocks = 148 * 4;
    loop<OP><<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    loop<OP><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double instr = double(blocks) * threads * iters * CHAINS;
    printf("%-8s %6.1f thread-instr/clk/SM\n", name, instr / (ms * 1e-3) / (148.0 * clk * 1e3));
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    run<0>("FHFMA", out);
    run<1>("FHADD", out);
    subnormal_probe<<<1, 32>>>(out);
    float h[3];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("FHFMA 1.5 * 3*2^-24 = %.9g (exact %.9g)\n", h[0], 4.5 * 5.9604644775390625e-08);
    printf("HMMA sum16 1.5 * 3*2^-24 = %.9g (exact %.9g)\n", h[1], 16 * 4.5 * 5.9604644775390625e-08);
    printf("HMMA sum16 1000 * 2^-24 = %.9g (exact %.9g)\n", h[2], 16 * 1000 * 5.9604644775390625e-08);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
