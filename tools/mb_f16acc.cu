// mb_f16acc.cu -- can the tensor core produce the fp16 hi/lo split of an
// H_16 product itself?
//   hi = mma.m16n8k16.f16.f16.f16.f16(H16, X, 0)        (fp16 accumulator)
//   lo = mma.m16n8k16.f16.f16.f16.f16(H16, X, -hi)
// If the unit rounds the exact A.B + C once to fp16, hi = RN16(Y) and
// lo = RN16(Y - hi), the split the decode kernel now builds with F2FP + FHADD
// (2 instructions per element).  Checks both against exact products (host,
// double) on dequantised-K-like inputs, and times f16- vs f32-accumulate HMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_f16acc tools/mb_f16acc.cu && tools/mb_f16acc
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <cuda_fp16.h>
#include <vector>

__device__ __forceinline__ void hfrag(uint32_t (&a)[4], int lane) {
    const int g = lane >> 2, t = lane & 3;
    auto h = [](int m, int k) -> uint32_t { return (__popc(m & k) & 1) ? 0xBC00u : 0x3C00u; };
    const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
    for (int r = 0; r < 4; ++r) a[r] = h(rows[r], cols[r]) | (h(rows[r], cols[r] + 1) << 16);
}

__device__ __forceinline__ void mma_f16(uint32_t (&d)[2], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                        uint32_t c0, uint32_t c1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%9};"
                 : "=r"(d[0]), "=r"(d[1])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c0), "r"(c1));
}
__device__ __forceinline__ void mma_f32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%10,%10,%10,%10};"
                 : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
}

// X: [tiles][16 k][8 n] fp16.  out: per tile, [16 m][8 n] hi, lo (fp16 bits), y32 (float)
__global__ void split_kernel(const uint16_t* X, int tiles, uint16_t* hi, uint16_t* lo, float* y32) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int tile = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (tile >= tiles) return;
    uint32_t a[4];
    hfrag(a, lane);
    const uint16_t* x = X + tile * 128;
    auto xv = [&](int k, int n) -> uint32_t { return x[k * 8 + n]; };
    const uint32_t b0 = xv(2 * t, g) | (xv(2 * t + 1, g) << 16), b1 = xv(2 * t + 8, g) | (xv(2 * t + 9, g) << 16);
    uint32_t h[2], l[2];
    mma_f16(h, a, b0, b1, 0u, 0u);
    mma_f16(l, a, b0, b1, h[0] ^ 0x80008000u, h[1] ^ 0x80008000u);
    float y[4];
    mma_f32(y, a, b0, b1);
    uint16_t* H = hi + tile * 128;
    uint16_t* L = lo + tile * 128;
    float* Y = y32 + tile * 128;
    const int rr[2] = {g, g + 8};
    for (int r = 0; r < 2; ++r) {
        H[rr[r] * 8 + 2 * t] = h[r] & 0xffff;
        H[rr[r] * 8 + 2 * t + 1] = h[r] >> 16;
        L[rr[r] * 8 + 2 * t] = l[r] & 0xffff;
        L[rr[r] * 8 + 2 * t + 1] = l[r] >> 16;
        Y[rr[r] * 8 + 2 * t] = y[2 * r];
        Y[rr[r] * 8 + 2 * t + 1] = y[2 * r + 1];
    }
}

template <bool F16>
__global__ void rate_kernel(float* out, int iters) {
    uint32_t a[4];
    hfrag(a, threadIdx.x & 31);
    uint32_t b0 = 0x3C003C00u + threadIdx.x, b1 = 0x3C00BC00u;
    uint32_t h[4][2] = {};
    float f[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (F16) {
                uint32_t d[2];
                mma_f16(d, a, b0 + c, b1, h[c][0], h[c][1]);
                h[c][0] = d[0];
                h[c][1] = d[1];
            } else {
                float d[4];
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                             "{%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(f[c][0]), "+f"(f[c][1]), "+f"(f[c][2]), "+f"(f[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0 + c), "r"(b1));
                (void)d;
            }
        }
    }
    float s = 0;
    for (int c = 0; c < 4; ++c) s += f[c][0] + __half2float(__ushort_as_half(h[c][0] & 0xffff));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

int main() {
    const int tiles = 1 << 16;
    std::vector<uint16_t> X(tiles * 128);
    srand(7);
    auto urand = []() { return (rand() + 0.5) / (RAND_MAX + 1.0); };
    for (size_t i = 0; i < X.size(); ++i) {
        // dequantised K: s * (c - z), s spanning ~2^-4 .. 2^4 per element (channels of different groups)
        const double s = std::exp2(-4.0 + 8.0 * urand()) * (1.0 + urand());
        const int cz = (rand() % 7) - 3;
        X[i] = __half_as_ushort(__float2half_rn(static_cast<float>(s * cz)));
    }
    uint16_t *dX, *dH, *dL;
    float* dY;
    cudaMalloc(&dX, X.size() * 2);
    cudaMalloc(&dH, X.size() * 2);
    cudaMalloc(&dL, X.size() * 2);
    cudaMalloc(&dY, X.size() * 4);
    cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
    split_kernel<<<tiles / 8, 256>>>(dX, tiles, dH, dL, dY);
    std::vector<uint16_t> H(X.size()), L(X.size());
    std::vector<float> Y(X.size());
    cudaMemcpy(H.data(), dH, H.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(L.data(), dL, L.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(Y.data(), dY, Y.size() * 4, cudaMemcpyDeviceToHost);
    long hi_rn = 0, hi_off = 0, lo_rn = 0, lo_off = 0, y32_exact = 0, n = 0;
    double max_rel_split = 0, max_rel_hi = 0;
    for (int tile = 0; tile < tiles; ++tile)
        for (int m = 0; m < 16; ++m)
            for (int c = 0; c < 8; ++c) {
                double y = 0;
                for (int k = 0; k < 16; ++k)
                    y += ((__builtin_popcount(m & k) & 1) ? -1.0 : 1.0) * h2f(X[tile * 128 + k * 8 + c]);
                const int i = tile * 128 + m * 8 + c;
                const double h = h2f(H[i]), l = h2f(L[i]);
                const uint16_t rn = __half_as_ushort(__float2half_rn(static_cast<float>(y)));
                // the float cast can double-round; compare in double via the neighbours
                (h2f(rn) == h ? hi_rn : hi_off)++;
                const double r = y - h;
                const uint16_t rnl = __half_as_ushort(__float2half_rn(static_cast<float>(r)));
                (h2f(rnl) == l ? lo_rn : lo_off)++;
                if (static_cast<double>(Y[i]) == y) ++y32_exact;
                if (y != 0) {
                    max_rel_split = std::fmax(max_rel_split, std::fabs(h + l - y) / std::fabs(y));
                    max_rel_hi = std::fmax(max_rel_hi, std::fabs(h - y) / std::fabs(y));
                }
                ++n;
            }
    printf("elements %ld: hi == RN16(Y) %ld (off %ld); lo == RN16(Y - hi) %ld (off %ld); f32 acc exact %ld\n", n,
           hi_rn, hi_off, lo_rn, lo_off, y32_exact);
    printf("max rel |hi + lo - Y| / |Y| = %.3e   (hi alone %.3e)\n", max_rel_split, max_rel_hi);

    float* dO;
    cudaMalloc(&dO, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int f16 = 0; f16 < 2; ++f16) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (f16)
                rate_kernel<true><<<148 * 8, 256>>>(dO, iters);
            else
                rate_kernel<false><<<148 * 8, 256>>>(dO, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = 148.0 * 8 * 8 * iters * 4;  // warps x iters x chains
            if (rep) printf("%s accumulate: %.1f HMMA.16816 / clk / SM (at 1.965 GHz)\n", f16 ? "f16" : "f32",
                            mmas / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
