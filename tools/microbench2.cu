// microbench2.cu -- per-SM issue rates of the scalar/paired ops the decode
// kernel is built from (lane-ops per clock per SM, 8 independent chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 tools/microbench2.cu && ./mb2
#include <cstdio>
#include <cuda_fp16.h>

#define CHAINS 8

template <int OP>
__global__ void loop(float* out, int iters, float a, float b) {
    float x[CHAINS], y[CHAINS];
    unsigned u[CHAINS];
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
        x[k] = threadIdx.x * 1e-3f + k;
        y[k] = k * 0.5f;
        u[k] = threadIdx.x * 2654435761u + k;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) {
            if (OP == 0) x[k] = fmaf(x[k], a, b);  // FFMA
            if (OP == 1) {                          // FFMA2
                float2 r = __ffma2_rn(make_float2(x[k], y[k]), make_float2(a, a), make_float2(b, b));
                x[k] = r.x;
                y[k] = r.y;
            }
            if (OP == 2) x[k] = x[k] + a;  // FADD
            if (OP == 3) {                 // FADD2
                float2 r = __fadd2_rn(make_float2(x[k], y[k]), make_float2(a, b));
                x[k] = r.x;
                y[k] = r.y;
            }
            if (OP == 4) {  // HFMA2
                __half2 h = *reinterpret_cast<__half2*>(&u[k]);
                h = __hfma2(h, __floats2half2_rn(a, a), __floats2half2_rn(b, b));
                u[k] = *reinterpret_cast<unsigned*>(&h);
            }
            if (OP == 5) {  // LOP3
                unsigned r;
                asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(u[k]), "r"(0x600000u), "r"(0x3F800000u));
                u[k] = r ^ i;
            }
            if (OP == 6) {  // cvt.rn.f16x2.f32 (F2FP)
                unsigned r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[k]), "f"(y[k]));
                x[k] = __uint_as_float(r);
            }
            if (OP == 7) {  // cvt.f32.f16
                float r;
                asm volatile("{.reg .b16 lo; mov.b32 {lo, _}, %1; cvt.f32.f16 %0, lo;}" : "=f"(r) : "r"(u[k]));
                u[k] = __float_as_uint(r);
            }
            if (OP == 8) {  // PRMT
                unsigned r;
                asm volatile("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(u[k]), "r"(u[(k + 1) % CHAINS]));
                u[k] = r;
            }
            if (OP == 9) {  // SHF (funnel)
                u[k] = __funnelshift_l(u[k], u[(k + 1) % CHAINS], 7);
            }
            if (OP == 10) {  // IMAD
                u[k] = u[k] * 2654435761u + 12345u;
            }
            if (OP == 11) {  // FMUL2
                float2 r = __fmul2_rn(make_float2(x[k], y[k]), make_float2(a, b));
                x[k] = r.x;
                y[k] = r.y;
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) s += x[k] + y[k] + __uint_as_float(u[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048, threads = 512, blocks = 148 * 4;
    loop<OP><<<blocks, threads>>>(out, 16, 1.0001f, 1e-7f);
    cudaEventRecord(e0);
    loop<OP><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double instr = double(blocks) * threads * iters * CHAINS;  // thread-instructions
    const double per_clk_sm = instr / (ms * 1e-3) / (148.0 * clk * 1e3);
    printf("%-8s %6.1f thread-instr/clk/SM  (%.1f T/s)\n", name, per_clk_sm, instr / ms / 1e9);
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    run<0>("FFMA", out);
    run<1>("FFMA2", out);
    run<2>("FADD", out);
    run<3>("FADD2", out);
    run<11>("FMUL2", out);
    run<4>("HFMA2", out);
    run<5>("LOP3", out);
    run<6>("F2FP", out);
    run<7>("cvt.f32.f16", out);
    run<8>("PRMT", out);
    run<9>("SHF", out);
    run<10>("IMAD", out);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
