// microbench4.cu -- is mma.sync with an fp16 accumulator (C = 0) the correctly
// rounded fp16 of the exact H_16 . X?  Compares against the fp32-accumulated
// result rounded to nearest, over random fp16 inputs with mixed exponents.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb4 tools/microbench4.cu && ./mb4
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void probe(unsigned* mism, unsigned* total, float* maxrel) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    uint32_t a[4];
    auto h = [](int m, int k) -> uint32_t { return (__popc(m & k) & 1) ? 0xBC00u : 0x3C00u; };
    const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
    for (int r = 0; r < 4; ++r) a[r] = h(rows[r], cols[r]) | (h(rows[r], cols[r] + 1) << 16);
    unsigned mm = 0, tot = 0;
    float mr = 0.f;
    for (int it = 0; it < 4096; ++it) {
        uint32_t b[2];
        for (int r = 0; r < 2; ++r) {
            uint32_t v = 0;
            for (int hh = 0; hh < 2; ++hh) {
                const uint32_t x = hash((blockIdx.x * 4096 + it) * 64 + lane * 2 + r * 64 * 4096 + hh * 7919);
                const float s = (float)((x >> 20) & 7) - 3.0f;           // c - z in [-3, 4]
                const float sc = __uint_as_float(((x >> 4) & 0x7fff) | 0x3f800000u) * exp2f((float)((x >> 23) & 15) - 8.0f);
                const __half hv = __float2half_rn(s * sc);
                v |= (uint32_t)__half_as_ushort(hv) << (16 * hh);
            }
            b[r] = v;
        }
        float d[4] = {0, 0, 0, 0};
        uint32_t e[2] = {0, 0};
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                     : "+r"(e[0]), "+r"(e[1])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        for (int k = 0; k < 4; ++k) {
            const __half want = __float2half_rn(d[k]);
            const uint16_t got = (uint16_t)(e[k >> 1] >> (16 * (k & 1)));
            tot++;
            if (got != __half_as_ushort(want)) {
                mm++;
                const float rel = fabsf(__half2float(__ushort_as_half(got)) - d[k]) / fmaxf(fabsf(d[k]), 1e-30f);
                mr = fmaxf(mr, rel);
            }
        }
    }
    atomicAdd(mism, mm);
    atomicAdd(total, tot);
    atomicMax(reinterpret_cast<unsigned*>(maxrel), __float_as_uint(mr));
}

int main() {
    unsigned *m, *t;
    float* r;
    cudaMalloc(&m, 4);
    cudaMalloc(&t, 4);
    cudaMalloc(&r, 4);
    cudaMemset(m, 0, 4);
    cudaMemset(t, 0, 4);
    cudaMemset(r, 0, 4);
    probe<<<64, 32>>>(m, t, r);
    unsigned hm, ht;
    float hr;
    cudaMemcpy(&hm, m, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ht, t, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hr, r, 4, cudaMemcpyDeviceToHost);
    printf("f16-accumulate vs RN(f32 result): %u of %u differ, max rel err of differing %.3g (fp16 half-ulp = %.3g)\n",
           hm, ht, hr, 1.0 / 2048);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
