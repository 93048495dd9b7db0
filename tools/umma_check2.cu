// Stand-alone check of the 2-SM (cta_group::2) tcgen05 wrappers in
// csrc/rkv_umma.cuh: a cluster of two CTAs computes D[256 x N] = A[256 x K] .
// B[N x K]^T, A in tensor memory (CTA r: rows 128 r ..), B split by rows
// (CTA r: rows N/2 r ..) in each CTA's shared memory, D rows in each CTA's
// tensor memory; the leader issues, commit2 signals both CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2501_16383_b200/csrc tools/umma_check2.cu -o tools/mb_umma2
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rkv_umma.cuh"

using namespace rkv;

template <int N, int K>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) umma2_gemm(const __half* A, const __half* B, float* D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kSlabs = K / 64, NH = N / 2;
    unsigned char* sb = smem;  // kSlabs x [N/2][128 B]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sb + kSlabs * NH * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = umma::cluster_rank();
    for (int i = tid; i < NH * K / 8; i += 128) {
        const int r = i / (K / 8), c = i % (K / 8);
        *reinterpret_cast<uint4*>(sb + (c / 8) * NH * 128 + umma::sw128(r, c % 8)) =
            *reinterpret_cast<const uint4*>(B + (rank * NH + r) * K + 8 * c);
    }
    umma::fence_proxy_async();
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) umma::alloc2<512>(tslot);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t taddr = *tslot;
    const uint32_t lane_base = static_cast<uint32_t>(32 * warp) << 16;
    const uint32_t* arow = reinterpret_cast<const uint32_t*>(A + (rank * 128 + tid) * K);
#pragma unroll
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = arow[c0 + j];
        umma::st16(taddr + lane_base + 256 + c0, v);
    }
    umma::wait_st();
    umma::fence_before();
    umma::cluster_sync();  // both CTAs' B halves and A rows are in place
    umma::fence_after();
    if (rank == 0 && warp == 1 && umma::elect_one()) {
        const uint32_t b0 = smem_u32(sb);
#pragma unroll
        for (int ks = 0; ks < K / 16; ++ks) {
            const int slab = ks / 4, kk = ks % 4;
            umma::mma2_f16_ts(taddr, taddr + 256 + 8 * ks, umma::sdesc(b0 + slab * NH * 128 + kk * 32),
                              umma::idesc_f16(256, N), ks > 0);
        }
        umma::commit2(bar);
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
        for (int j = 0; j < 16; ++j) D[(rank * 128 + row) * N + c0 + j] = __uint_as_float(v[j]);
    }
    umma::fence_before();
    umma::cluster_sync();
    if (warp == 0) umma::dealloc2<512>(taddr);
}

template <int N, int K>
int run() {
    std::vector<__half> a(256 * K), b(N * K);
    std::vector<float> af(256 * K), bf(N * K), d(256 * N);
    srand(N * 11 + K);
    for (int i = 0; i < 256 * K; ++i) af[i] = __half2float(a[i] = __float2half((rand() % 17 - 8) / 8.0f));
    for (int i = 0; i < N * K; ++i) bf[i] = __half2float(b[i] = __float2half((rand() % 13 - 6) / 4.0f));
    __half *da, *db;
    float* dd;
    cudaMalloc(&da, a.size() * 2);
    cudaMalloc(&db, b.size() * 2);
    cudaMalloc(&dd, d.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dd, 0xff, d.size() * 4);
    const int smem = (K / 64) * (N / 2) * 128 + 64 + 1024;
    cudaFuncSetAttribute(umma2_gemm<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma2_gemm<N, K><<<2, 128, smem>>>(da, db, dd);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int i = 0; i < 256; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += double(af[i * K + k]) * bf[j * K + k];
            const double err = std::fabs(ref - d[i * N + j]);
            maxerr = std::max(maxerr, err);
            if (err > 1e-3 && bad++ < 5) printf("  D[%d][%d] = %f, want %f\n", i, j, d[i * N + j], ref);
        }
    printf("2SM TS N=%d K=%d: %s (max err %.3g, %d bad)\n", N, K, bad ? "FAIL" : "ok", maxerr, bad);
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<64, 128>();
    f |= run<128, 64>();
    return f;
}
