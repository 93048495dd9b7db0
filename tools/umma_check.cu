// Stand-alone check of the tcgen05 wrappers in csrc/rkv_umma.cuh: one CTA
// computes D[128 x N] = A[128 x K] . B[N x K]^T (fp16 in, fp32 out) from
// K-major SWIZZLE_128B shared-memory operands and compares with the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2501_16383_b200/csrc tools/umma_check.cu -o tools/mb_umma
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rkv_umma.cuh"

using namespace rkv;

template <int N, int K>
__global__ void __launch_bounds__(128) umma_gemm(const __half* A, const __half* B, float* D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kSlabs = K / 64;
    unsigned char* sa = smem;                       // kSlabs x [128][128 B]
    unsigned char* sb = sa + kSlabs * 128 * 128;    // kSlabs x [N][128 B]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sb + kSlabs * N * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // fill: 16-byte chunks (8 K elements)
    for (int i = tid; i < 128 * K / 8; i += 128) {
        const int r = i / (K / 8), c = i % (K / 8);
        *reinterpret_cast<uint4*>(sa + (c / 8) * 128 * 128 + umma::sw128(r, c % 8)) =
            *reinterpret_cast<const uint4*>(A + r * K + 8 * c);
    }
    for (int i = tid; i < N * K / 8; i += 128) {
        const int r = i / (K / 8), c = i % (K / 8);
        *reinterpret_cast<uint4*>(sb + (c / 8) * N * 128 + umma::sw128(r, c % 8)) =
            *reinterpret_cast<const uint4*>(B + r * K + 8 * c);
    }
    umma::fence_proxy_async();
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) umma::alloc<128>(tslot);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t taddr = *tslot;
    if (warp == 1 && umma::elect_one()) {
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
        for (int ks = 0; ks < K / 16; ++ks) {
            const int slab = ks / 4, kk = ks % 4;
            umma::mma_f16(taddr, umma::sdesc(a0 + slab * 128 * 128 + kk * 32), umma::sdesc(b0 + slab * N * 128 + kk * 32),
                          umma::idesc_f16(128, N), ks > 0);
        }
        umma::commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    umma::fence_after();
    const int row = 32 * warp + lane;
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        umma::ld16(taddr + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
        umma::wait_ld();
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::dealloc<128>(taddr);
}

// same product with A in tensor memory: thread r (warp r / 32) writes row r
// of A as fp16 pairs into columns [256, 256 + K / 2) with tcgen05.st
template <int N, int K>
__global__ void __launch_bounds__(128) umma_gemm_ts(const __half* A, const __half* B, float* D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kSlabs = K / 64;
    unsigned char* sb = smem;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sb + kSlabs * N * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N * K / 8; i += 128) {
        const int r = i / (K / 8), c = i % (K / 8);
        *reinterpret_cast<uint4*>(sb + (c / 8) * N * 128 + umma::sw128(r, c % 8)) =
            *reinterpret_cast<const uint4*>(B + r * K + 8 * c);
    }
    umma::fence_proxy_async();
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) umma::alloc<512>(tslot);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t taddr = *tslot;
    const uint32_t lane_base = static_cast<uint32_t>(32 * warp) << 16;
    const uint32_t* arow = reinterpret_cast<const uint32_t*>(A + tid * K);
#pragma unroll
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = arow[c0 + j];
        umma::st16(taddr + lane_base + 256 + c0, v);
    }
    umma::wait_st();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (warp == 1 && umma::elect_one()) {
        const uint32_t b0 = smem_u32(sb);
#pragma unroll
        for (int ks = 0; ks < K / 16; ++ks) {
            const int slab = ks / 4, kk = ks % 4;
            umma::mma_f16_ts(taddr, taddr + 256 + 8 * ks, umma::sdesc(b0 + slab * N * 128 + kk * 32),
                             umma::idesc_f16(128, N), ks > 0);
        }
        umma::commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    umma::fence_after();
    const int row = 32 * warp + lane;
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        umma::ld16(taddr + lane_base + c0, v);
        umma::wait_ld(v);
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::dealloc<512>(taddr);
}

template <int N, int K>
int run(bool ts = false) {
    std::vector<__half> a(128 * K), b(N * K);
    std::vector<float> af(128 * K), bf(N * K), d(128 * N);
    srand(N * 7 + K);
    for (int i = 0; i < 128 * K; ++i) af[i] = __half2float(a[i] = __float2half((rand() % 17 - 8) / 8.0f));
    for (int i = 0; i < N * K; ++i) bf[i] = __half2float(b[i] = __float2half((rand() % 13 - 6) / 4.0f));
    __half *da, *db;
    float* dd;
    cudaMalloc(&da, a.size() * 2);
    cudaMalloc(&db, b.size() * 2);
    cudaMalloc(&dd, d.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dd, 0xff, d.size() * 4);
    const int smem = (K / 64) * (128 + N) * 128 + 64 + 1024;
    if (ts) {
        cudaFuncSetAttribute(umma_gemm_ts<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        umma_gemm_ts<N, K><<<1, 128, smem>>>(da, db, dd);
    } else {
        cudaFuncSetAttribute(umma_gemm<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        umma_gemm<N, K><<<1, 128, smem>>>(da, db, dd);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += double(af[i * K + k]) * bf[j * K + k];
            const double err = std::fabs(ref - d[i * N + j]);
            maxerr = std::max(maxerr, err);
            if (err > 1e-3 && bad++ < 5) printf("  D[%d][%d] = %f, want %f\n", i, j, d[i * N + j], ref);
        }
    printf("%s N=%d K=%d: %s (max err %.3g, %d bad)\n", ts ? "TS" : "SS", N, K, bad ? "FAIL" : "ok", maxerr, bad);
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<64, 64>();
    f |= run<64, 128>();
    f |= run<128, 64>();
    f |= run<128, 128>();
    f |= run<64, 128>(true);
    f |= run<128, 64>(true);
    return f;
}
