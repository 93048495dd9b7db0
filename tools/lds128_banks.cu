// Shared-memory wavefronts of one warp-wide LDS.128 for several per-lane
// address patterns (profile with ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/lds128_banks.cu -o tools/mb_lds
#include <cstdio>

template <int PAT>
__global__ void lds(float4* out, int iters) {
    __shared__ __align__(16) unsigned char buf[16384];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(buf)[i] = i;
    __syncthreads();
    int off;
    if (PAT == 0) off = lane * 16;                                        // contiguous
    else if (PAT == 1) off = lane * 32 + 16 * ((lane >> 2) & 1);          // GQA K fragments (N = 256), jc = 0
    else if (PAT == 2) off = lane * 64 + 16 * ((lane >> 1) & 3);          // MHA K fragments (N = 512), jc = 0
    else if (PAT == 3) off = lane * 32 + 16 * ((lane >> 3) & 1);          // candidate
    else if (PAT == 4) off = lane * 32 + 16 * (((lane >> 2) ^ (lane >> 3)) & 1);  // candidate
    else off = lane * 32;                                                  // unswizzled 32-byte stride
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(static_cast<unsigned>(__cvta_generic_to_shared(buf + ((off + it * 0) & 16383)))));
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    out[threadIdx.x] = acc;
}

int main() {
    float4* d;
    cudaMalloc(&d, 32 * sizeof(float4));
    lds<0><<<1, 32>>>(d, 100);
    lds<1><<<1, 32>>>(d, 100);
    lds<2><<<1, 32>>>(d, 100);
    lds<3><<<1, 32>>>(d, 100);
    lds<4><<<1, 32>>>(d, 100);
    lds<5><<<1, 32>>>(d, 100);
    cudaDeviceSynchronize();
    printf("done\n");
    return 0;
}
