// Cross-CTA hand-off latency inside a 2-CTA cluster: CTA 0 and CTA 1 bounce
// a token through mbarriers in each other's shared memory (remote
// mbarrier.arrive.release.cluster, local try_wait.acquire.cluster).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2501_16383_b200/csrc tools/cluster_pingpong.cu -o tools/mb_ping
#include <cstdio>

#include "rkv_umma.cuh"

using namespace rkv;

__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, long long* out, int relaxed_wait) {
    __shared__ uint64_t bar;
    const uint32_t rank = umma::cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    umma::cluster_sync();
    if (threadIdx.x == 0) {
        const uint32_t peer = umma::peer_addr(&bar, rank ^ 1u);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                umma::mbar_arrive_cluster(peer);
                if (relaxed_wait) mbar_wait(&bar, i & 1);
                else umma::mbar_wait_cluster(&bar, i & 1);
            } else {
                if (relaxed_wait) mbar_wait(&bar, i & 1);
                else umma::mbar_wait_cluster(&bar, i & 1);
                umma::mbar_arrive_cluster(peer);
            }
        }
        if (rank == 0) out[0] = (clock64() - t0) / iters;
    }
    umma::cluster_sync();
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    for (int rw = 0; rw < 2; ++rw) {
        pingpong<<<2, 32>>>(1000, d, rw);
        cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("round trip (2 hand-offs), %s wait: %lld cycles\n", rw ? "cta-scope" : "cluster-acquire", h);
    }
    return 0;
}
