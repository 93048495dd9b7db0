// e2e_cpp.cu -- the decode step end to end through the C++ API
// (include/rotatekv/rotatekv.hpp, DeviceLayerCache), the path a reference
// caller switching over would take.  bench.py runs it for the
// `e2e_cpp` key.
//
//   e2e_cpp --batch B --q-heads Hq --kv-heads Hkv --group G --tokens T
//           [--steps K] [--warmup W] [--device D] [--seed S] [--rope-base R]
//
// Fills T tokens per sequence through DeviceLayerCache::append (seeded
// N(0,1) fp16 K/V generated on the device, token 0 a sink), then times K
// decode steps, each: H2D of the step's queries from pinned host memory,
// DeviceLayerCache::decode_attention, D2H of the fp32 output -- all inside
// the CUDA-event-timed region.  As in bench.py's e2e (the serving pattern),
// the copies run on a copy stream, double buffered, so step i+1's upload and
// step i-1's download overlap step i's kernels.  Prints one JSON line.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "rotatekv/rotatekv.hpp"

namespace {

__global__ void fill_normal(uint16_t* out, int64_t n, uint64_t seed, float gain_stride_mask) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // counter-based Box-Muller (splitmix64 of the index)
    auto mix = [](uint64_t z) {
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    const uint64_t a = mix(seed ^ (2 * static_cast<uint64_t>(i))), b = mix(seed ^ (2 * static_cast<uint64_t>(i) + 1));
    const float u1 = (static_cast<float>(a >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>(b >> 40) * (1.0f / 16777216.0f);
    float x = sqrtf(-2.0f * logf(u1)) * cosf(6.2831853f * u2);
    (void)gain_stride_mask;
    out[i] = __half_as_ushort(__float2half_rn(x));
}

int64_t arg(int argc, char** argv, const char* name, int64_t dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (std::strcmp(argv[i], name) == 0) return std::atoll(argv[i + 1]);
    return dflt;
}

}  // namespace

int main(int argc, char** argv) {
    using namespace rotatekv_b200;
    const int B = static_cast<int>(arg(argc, argv, "--batch", 8));
    const int Hq = static_cast<int>(arg(argc, argv, "--q-heads", 32));
    const int Hkv = static_cast<int>(arg(argc, argv, "--kv-heads", 32));
    const int G = static_cast<int>(arg(argc, argv, "--group", 4));
    const int64_t T = arg(argc, argv, "--tokens", 32768);
    const int steps = static_cast<int>(arg(argc, argv, "--steps", 20));
    const int warmup = static_cast<int>(arg(argc, argv, "--warmup", 3));
    const int dev = static_cast<int>(arg(argc, argv, "--device", 0));
    const uint64_t seed = static_cast<uint64_t>(arg(argc, argv, "--seed", 46));
    const double base = static_cast<double>(arg(argc, argv, "--rope-base", 10000));
    try {
        check_cuda(cudaSetDevice(dev), "cudaSetDevice");
        cudaStream_t s;
        check_cuda(cudaStreamCreate(&s), "stream");
        rkv_layer_desc d{};
        d.batch = B;
        d.num_q_heads = Hq;
        d.num_kv_heads = Hkv;
        d.head_dim = 128;
        d.heads_per_group = G;
        d.group_size = 128;
        d.bits = 2;
        d.scale_format = RKV_SCALE_FP16_CEIL;
        d.max_tokens = T;
        d.max_sinks = 4;
        d.rope_base = base;
        const int C = Hkv * 128;
        std::vector<int32_t> perm(static_cast<size_t>(C));
        std::iota(perm.begin(), perm.end(), 0);
        std::shuffle(perm.begin(), perm.end(), std::mt19937(static_cast<unsigned>(seed)));
        DeviceLayerCache cache(d, perm, s);
        // fill: chunks of tokens through append (token 0 of every sequence a sink)
        const int64_t chunk = 2048;
        uint16_t *dk = nullptr, *dv = nullptr;
        check_cuda(cudaMalloc(&dk, static_cast<size_t>(B) * chunk * C * 2), "k");
        check_cuda(cudaMalloc(&dv, static_cast<size_t>(B) * chunk * C * 2), "v");
        for (int64_t t0 = 0; t0 < T; t0 += chunk) {
            const int64_t n = std::min<int64_t>(chunk, T - t0);
            const int64_t cnt = static_cast<int64_t>(B) * n * C;
            fill_normal<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(dk, cnt, seed + 17 * t0, 0.f);
            fill_normal<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(dv, cnt, seed + 31 * t0 + 7, 0.f);
            std::vector<uint8_t> flags(static_cast<size_t>(B) * n, 0);
            if (t0 == 0)
                for (int b = 0; b < B; ++b) flags[static_cast<size_t>(b) * n] = 1;
            cache.append(dk, dv, n, flags);
        }
        // per-step queries (4 distinct sets, pinned host), pinned output buffers
        const size_t qn = static_cast<size_t>(B) * Hq * 128, on = qn;
        uint16_t* hq = nullptr;
        float* hout = nullptr;
        check_cuda(cudaMallocHost(&hq, 4 * qn * 2), "pinned q");
        check_cuda(cudaMallocHost(&hout, on * 4), "pinned out");
        std::mt19937 rng(static_cast<unsigned>(seed) + 1);
        std::normal_distribution<float> nd;
        for (size_t i = 0; i < 4 * qn; ++i) hq[i] = __half_as_ushort(__float2half_rn(nd(rng)));
        uint16_t* dq[2] = {nullptr, nullptr};
        float* dout[2] = {nullptr, nullptr};
        for (int j = 0; j < 2; ++j) {
            check_cuda(cudaMalloc(&dq[j], qn * 2), "q");
            check_cuda(cudaMalloc(&dout[j], on * 4), "out");
        }
        cudaStream_t cs;
        check_cuda(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
        cudaEvent_t up[2], comp[2], down[2];
        for (int j = 0; j < 2; ++j) {
            cudaEventCreateWithFlags(&up[j], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&comp[j], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&down[j], cudaEventDisableTiming);
        }
        auto upload = [&](int i) {
            const int j = i & 1;
            check_cuda(cudaStreamWaitEvent(cs, comp[j], 0), "wait comp");  // step i-2 done reading q buffer j
            check_cuda(cudaMemcpyAsync(dq[j], hq + (i % 4) * qn, qn * 2, cudaMemcpyHostToDevice, cs), "H2D q");
            cudaEventRecord(up[j], cs);
        };
        auto step = [&](int i, int n) {
            const int j = i & 1;
            if (i == 0) upload(0);
            if (i + 1 < n) upload(i + 1);
            check_cuda(cudaStreamWaitEvent(s, up[j], 0), "wait up");
            check_cuda(cudaStreamWaitEvent(s, down[j], 0), "wait down");  // out buffer j downloaded (step i-2)
            cache.decode_attention(dq[j], dout[j]);
            cudaEventRecord(comp[j], s);
            check_cuda(cudaStreamWaitEvent(cs, comp[j], 0), "wait comp");
            check_cuda(cudaMemcpyAsync(hout, dout[j], on * 4, cudaMemcpyDeviceToHost, cs), "D2H out");
            cudaEventRecord(down[j], cs);
        };
        for (int i = 0; i < warmup; ++i) step(i, warmup);
        check_cuda(cudaDeviceSynchronize(), "warmup");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        check_cuda(cudaStreamWaitEvent(cs, e0, 0), "start");
        for (int i = 0; i < steps; ++i) step(i, steps);
        cudaEvent_t last;
        cudaEventCreateWithFlags(&last, cudaEventDisableTiming);
        cudaEventRecord(last, cs);
        check_cuda(cudaStreamWaitEvent(s, last, 0), "last download");  // inside the timed region
        cudaEventRecord(e1, s);
        check_cuda(cudaEventSynchronize(e1), "timed");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double checksum = 0;
        for (size_t i = 0; i < on; ++i) checksum += hout[i];
        std::printf("{\"impl\": \"cpp\", \"batch\": %d, \"tokens\": %lld, \"steps\": %d, \"ms\": %.6f, "
                    "\"ms_per_step\": %.6f, \"tokens_per_s\": %.3f, \"h2d_bytes_per_step\": %zu, "
                    "\"d2h_bytes_per_step\": %zu, \"finite\": %s}\n",
                    B, static_cast<long long>(T), steps, ms, ms / steps, B * steps / (ms / 1e3), qn * 2, on * 4,
                    std::isfinite(checksum) ? "true" : "false");
        cudaFree(dk);
        cudaFree(dv);
        for (int j = 0; j < 2; ++j) {
            cudaFree(dq[j]);
            cudaFree(dout[j]);
        }
        cudaStreamDestroy(cs);
        cudaFreeHost(hq);
        cudaFreeHost(hout);
        cudaStreamDestroy(s);
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "e2e_cpp: %s\n", ex.what());
        return 1;
    }
    return 0;
}
