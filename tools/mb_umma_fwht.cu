// Throughput of tcgen05.mma (kind::f16, cta_group::1, M = 128) at the small
// N / K shapes a tensor-core FWHT factor would use (H_16: N = K = 16), with
// the data operand A in tensor memory (ts) or shared memory (ss), against the
// large-N shape -- the measurement behind DESIGN.md §3's "tcgen05 rotation"
// paragraph.  One CTA per SM, one elected thread issues R independent MMAs
// (D rotates over the 256 low TMEM columns), one commit, clock64 around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2501_16383_b200/csrc -I include tools/mb_umma_fwht.cu -o tools/mb_umma_fwht
#include <cuda_fp16.h>

#include <cstdio>
#include <vector>

#include "rkv_umma.cuh"

using namespace rkv;

template <int N, bool TS>
__global__ void __launch_bounds__(128) umma_rate(int reps, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sa = smem;              // A: 128 rows x 128 B (K = 64 max), SW128
    unsigned char* sb = smem + 128 * 128;  // B: N rows x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sb + 256 * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + 256) * 8; i += 128)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0xbc003c00u, 0x3c00bc00u, 0x3c003c00u);
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
    {  // A rows into TMEM columns [384, 392)
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = 0x3c003c00u;
        umma::st16(taddr + (static_cast<uint32_t>(32 * warp) << 16) + 384, v);
        umma::wait_st();
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (warp == 1 && umma::elect_one()) {
        const uint32_t id = umma::idesc_f16(128, N);
        const uint64_t bd = umma::sdesc(smem_u32(sb));
        const uint64_t ad = umma::sdesc(smem_u32(sa));
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t d = taddr + static_cast<uint32_t>((r * N) & 255);
            if (TS) umma::mma_f16_ts(d, taddr + 384, bd, id, 0u);
            else umma::mma_f16(d, ad, bd, id, 0u);
        }
        umma::commit(bar);
        mbar_wait(bar, 0);
        const long long t1 = clock64();
        cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::dealloc<512>(taddr);
}

template <int N, bool TS>
void run(int sms) {
    const int reps = 8192;
    unsigned long long* dc;
    cudaMalloc(&dc, sms * sizeof(unsigned long long));
    const size_t smem = (128 + 256) * 128 + 64;
    cudaFuncSetAttribute(umma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    umma_rate<N, TS><<<sms, 128, smem>>>(reps, dc);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    umma_rate<N, TS><<<sms, 128, smem>>>(reps, dc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> c(sms);
    cudaMemcpy(c.data(), dc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : c) avg += static_cast<double>(x);
    avg /= sms;
    const double macs = 128.0 * N * 16 * reps;  // per CTA
    std::printf("{\"N\": %d, \"K\": 16, \"A\": \"%s\", \"clk_per_mma\": %.2f, \"mac_per_clk_sm\": %.0f, "
                "\"tflops\": %.1f, \"err\": \"%s\"}\n",
                N, TS ? "tmem" : "smem", avg / reps, macs / avg, 2.0 * macs * sms / (ms * 1e-3) / 1e12,
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(dc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<16, true>(sms);
    run<16, false>(sms);
    run<32, true>(sms);
    run<32, false>(sms);
    run<64, true>(sms);
    run<128, true>(sms);
    run<256, true>(sms);
    run<256, false>(sms);
    return 0;
}
