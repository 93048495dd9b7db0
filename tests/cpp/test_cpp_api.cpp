// C++ parity test of the B200 library through its C++ API (rotatekv.hpp),
// written in the style of the reference's doctest suites
// (proj/tests/test_kv_cache.cpp, test_pipeline.cpp): the device cache is
// filled through DeviceLayerCache::append and read back; codes must equal the
// CPU oracle (oracle/rkv_oracle.c) bit for bit, decode must match it within
// 2e-3, and argument errors must throw the reference's exception classes.
// Built and run by tests/test_gpu_parity.py::test_cpp_api_program.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "rkv_oracle.h"
#include "rotatekv/rotatekv.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                            \
    do {                                                                    \
        if (c) ++g_pass;                                                    \
        else { ++g_fail; std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); } \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                            \
    do {                                                                    \
        bool thrown = false;                                                \
        try { expr; } catch (const E&) { thrown = true; } catch (...) {}    \
        CHECK(thrown);                                                      \
    } while (0)

namespace {

struct Lcg {  // seeded synthetic data (CounterRng-style determinism)
    uint64_t s;
    double uniform() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return static_cast<double>((s >> 11) & ((1ULL << 53) - 1)) * 0x1.0p-53;
    }
    double normal() {
        double u1 = uniform(), u2 = uniform();
        if (u1 < 1e-300) u1 = 1e-300;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
    }
};

}  // namespace

int main() {
    const int B = 2, H = 8, D = 128, G = 4, T = 40;
    const int C = H * D;
    rkv_layer_desc desc{};
    desc.batch = B;
    desc.num_q_heads = H;
    desc.num_kv_heads = H;
    desc.head_dim = D;
    desc.heads_per_group = G;
    desc.group_size = 128;
    desc.bits = 2;
    desc.scale_format = RKV_SCALE_FP16_CEIL;
    desc.max_tokens = 48;
    desc.max_sinks = 4;
    desc.rope_base = 10000.0;

    Lcg rng{42};
    std::vector<int32_t> perm(C);
    for (int i = 0; i < C; ++i) perm[static_cast<size_t>(i)] = i;
    for (int i = C - 1; i > 0; --i) std::swap(perm[static_cast<size_t>(i)], perm[static_cast<size_t>(rng.uniform() * (i + 1))]);
    std::vector<uint16_t> k(static_cast<size_t>(B) * T * C), v(k.size()), q(static_cast<size_t>(B) * H * D);
    for (size_t i = 0; i < k.size(); ++i) {
        const double gain = (i % static_cast<size_t>(C)) % 97 == 3 ? 20.0 : 1.0;  // outlier channels
        k[i] = rkvo_float_to_half_rn(static_cast<float>(rng.normal() * gain));
        v[i] = rkvo_float_to_half_rn(static_cast<float>(rng.normal()));
    }
    for (auto& x : q) x = rkvo_float_to_half_rn(static_cast<float>(rng.normal()));
    std::vector<uint8_t> flags(static_cast<size_t>(B) * T, 0);
    flags[0] = 1;
    flags[static_cast<size_t>(T) + 7] = 1;

    uint16_t *dk = nullptr, *dv = nullptr, *dq = nullptr;
    float* dout = nullptr;
    cudaMalloc(&dk, k.size() * 2);
    cudaMalloc(&dv, v.size() * 2);
    cudaMalloc(&dq, q.size() * 2);
    cudaMalloc(&dout, q.size() * 4);
    cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);

    {
        rotatekv_b200::DeviceLayerCache cache(desc, perm);
        // decode on an empty cache: position must equal current cache length
        CHECK_THROWS_AS(cache.decode_attention(dq, dout), std::invalid_argument);
        cache.append(dk, dv, T, flags);
        CHECK(cache.size(0) == T && cache.size(1) == T);
        CHECK(cache.sink_count(0) == 1 && cache.sink_count(1) == 1);
        // capacity: 48 tokens, 40 used -> 9 more is out of range
        CHECK_THROWS_AS(cache.append(dk, dv, 9), std::out_of_range);

        // bit-exact codes vs the oracle
        const auto& view = cache.view();
        const int W = C / 16, MG = C / 128;
        std::vector<uint32_t> kc(static_cast<size_t>(B) * desc.max_tokens * W), km(static_cast<size_t>(B) * desc.max_tokens * MG);
        std::vector<uint32_t> vc(kc.size()), vm(km.size());
        cudaMemcpy(kc.data(), view.k_codes, kc.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(km.data(), view.k_meta, km.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(vc.data(), view.v_codes, vc.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(vm.data(), view.v_meta, vm.size() * 4, cudaMemcpyDeviceToHost);
        cache.decode_attention(dq, dout);
        std::vector<float> out(q.size());
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);

        for (int b = 0; b < B; ++b) {
            std::vector<uint32_t> okc(static_cast<size_t>(T) * W), okm(static_cast<size_t>(T) * MG), ovc(okc.size()), ovm(okm.size());
            rkvo_quantize_kv_rows(k.data() + static_cast<size_t>(b) * T * C, v.data() + static_cast<size_t>(b) * T * C, T, H, D,
                                  G, perm.data(), RKVO_SCALE_FP16_CEIL, okc.data(), okm.data(), ovc.data(), ovm.data());
            bool same = true;
            for (int t = 0; t < T; ++t) {
                const bool sink = flags[static_cast<size_t>(b * T + t)] != 0;
                for (int w = 0; w < W; ++w) {
                    const size_t g = (static_cast<size_t>(b) * desc.max_tokens + t) * W + w;
                    const uint32_t want_k = sink ? 0u : okc[static_cast<size_t>(t) * W + w];
                    const uint32_t want_v = sink ? 0u : ovc[static_cast<size_t>(t) * W + w];
                    same = same && kc[g] == want_k && vc[g] == want_v;
                }
                for (int m = 0; m < MG; ++m) {
                    const size_t g = (static_cast<size_t>(b) * desc.max_tokens + t) * MG + m;
                    same = same && km[g] == (sink ? 0u : okm[static_cast<size_t>(t) * MG + m]) &&
                           vm[g] == (sink ? 0u : ovm[static_cast<size_t>(t) * MG + m]);
                }
            }
            CHECK(same);

            // decode vs the oracle over the same codes
            std::vector<float> want(static_cast<size_t>(H) * D);
            std::vector<uint32_t> bkc(okc.size()), bkm(okm.size()), bvc(ovc.size()), bvm(ovm.size());
            for (int t = 0; t < T; ++t) {
                for (int w = 0; w < W; ++w) {
                    bkc[static_cast<size_t>(t) * W + w] = kc[(static_cast<size_t>(b) * desc.max_tokens + t) * W + w];
                    bvc[static_cast<size_t>(t) * W + w] = vc[(static_cast<size_t>(b) * desc.max_tokens + t) * W + w];
                }
                for (int m = 0; m < MG; ++m) {
                    bkm[static_cast<size_t>(t) * MG + m] = km[(static_cast<size_t>(b) * desc.max_tokens + t) * MG + m];
                    bvm[static_cast<size_t>(t) * MG + m] = vm[(static_cast<size_t>(b) * desc.max_tokens + t) * MG + m];
                }
            }
            rkvo_decode_attention(bkc.data(), bkm.data(), bvc.data(), bvm.data(), flags.data() + static_cast<size_t>(b) * T,
                                  k.data() + static_cast<size_t>(b) * T * C, v.data() + static_cast<size_t>(b) * T * C, T,
                                  q.data() + static_cast<size_t>(b) * H * D, H, H, D, G, perm.data(), 10000.0, want.data());
            double mx = 0, err = 0;
            for (size_t i = 0; i < want.size(); ++i) {
                mx = std::fmax(mx, std::fabs(want[i]));
                err = std::fmax(err, std::fabs(static_cast<double>(want[i]) - out[static_cast<size_t>(b) * H * D + i]));
            }
            std::printf("sequence %d: decode rel err %.3g\n", b, err / mx);
            CHECK(err / mx < 2e-3);
        }

        // prefill attention half: the last prompt row (position T-1) with the decode query
        // must reproduce the decode output; rows past the cache are refused
        {
            const size_t row = static_cast<size_t>(H) * D;
            std::vector<uint16_t> qp(static_cast<size_t>(B) * T * row);
            for (size_t i = 0; i < qp.size(); ++i) qp[i] = q[i % q.size()];
            for (int b = 0; b < B; ++b)
                std::copy(q.begin() + static_cast<long>(b * row), q.begin() + static_cast<long>((b + 1) * row),
                          qp.begin() + static_cast<long>((static_cast<size_t>(b) * T + T - 1) * row));
            uint16_t* dqp = nullptr;
            float* dpo = nullptr;
            cudaMalloc(&dqp, qp.size() * 2);
            cudaMalloc(&dpo, qp.size() * 4);
            cudaMemcpy(dqp, qp.data(), qp.size() * 2, cudaMemcpyHostToDevice);
            cache.prefill_attention(dqp, T, std::vector<int64_t>(static_cast<size_t>(B), 0), dpo);
            std::vector<float> po(qp.size());
            cudaMemcpy(po.data(), dpo, po.size() * 4, cudaMemcpyDeviceToHost);
            for (int b = 0; b < B; ++b) {
                double mx = 0, err = 0;
                for (size_t i = 0; i < row; ++i) {
                    const double d = out[static_cast<size_t>(b) * row + i];
                    mx = std::fmax(mx, std::fabs(d));
                    err = std::fmax(err, std::fabs(d - po[(static_cast<size_t>(b) * T + T - 1) * row + i]));
                }
                std::printf("sequence %d: prefill last row vs decode rel err %.3g\n", b, err / mx);
                CHECK(err / mx < 2e-3);
            }
            CHECK_THROWS_AS(cache.prefill_attention(dqp, T, std::vector<int64_t>(static_cast<size_t>(B), 1), dpo),
                            std::out_of_range);
            cudaFree(dqp);
            cudaFree(dpo);
        }

        // LayerKVCache::append in the fused frame (fuse_weights, proj/src/pipeline.cpp:88-99):
        // the oracle's K' = reorder(H_G k) and V' = H_128 v as fp32 rows give the same words
        {
            std::vector<float> kr(k.size()), kf(k.size()), vf(v.size());
            for (size_t i = 0; i < k.size(); ++i) {
                kr[i] = rkvo_half_to_float(k[i]);
                vf[i] = rkvo_half_to_float(v[i]);
            }
            rkvo_rotate_rows(kr.data(), static_cast<int64_t>(B) * T, D, G, H);
            rkvo_apply_reorder(kr.data(), static_cast<int64_t>(B) * T, C, perm.data(), 0, kf.data());
            rkvo_rotate_rows(vf.data(), static_cast<int64_t>(B) * T, D, 1, H);
            float *dkf = nullptr, *dvf = nullptr;
            cudaMalloc(&dkf, kf.size() * 4);
            cudaMalloc(&dvf, vf.size() * 4);
            cudaMemcpy(dkf, kf.data(), kf.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dvf, vf.data(), vf.size() * 4, cudaMemcpyHostToDevice);
            rotatekv_b200::DeviceLayerCache fused(desc, perm);
            fused.append_fused(dkf, dvf, RKV_ROWS_F32, T, flags);
            CHECK(fused.size(0) == T && fused.sink_count(1) == 1);
            const auto& fv = fused.view();
            std::vector<uint32_t> fkc(kc.size()), fkm(km.size()), fvc(vc.size()), fvm(vm.size());
            cudaMemcpy(fkc.data(), fv.k_codes, fkc.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(fkm.data(), fv.k_meta, fkm.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(fvc.data(), fv.v_codes, fvc.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(fvm.data(), fv.v_meta, fvm.size() * 4, cudaMemcpyDeviceToHost);
            bool same = true;
            for (int b = 0; b < B; ++b)
                for (int t = 0; t < T; ++t) {
                    const size_t r = static_cast<size_t>(b) * desc.max_tokens + t;
                    for (int w = 0; w < W; ++w) same = same && fkc[r * W + w] == kc[r * W + w] && fvc[r * W + w] == vc[r * W + w];
                    for (int m = 0; m < MG; ++m) same = same && fkm[r * MG + m] == km[r * MG + m] && fvm[r * MG + m] == vm[r * MG + m];
                }
            CHECK(same);
            CHECK_THROWS_AS(fused.append_fused(dkf, dvf, RKV_ROWS_F32, 9), std::out_of_range);
            CHECK_THROWS_AS(fused.append_fused(dkf, dvf, static_cast<rkv_rows_dtype>(7), 1), std::invalid_argument);
            cudaFree(dkf);
            cudaFree(dvf);
        }

        // LayerKVCache::serialize / deserialize round trip (fp16-scale wire format)
        const std::vector<uint8_t> blob = cache.serialize(1, RKV_WIRE_FP16_SCALE);
        rotatekv_b200::DeviceLayerCache other(desc, perm);
        other.deserialize(blob, 0);
        CHECK(other.size(0) == T && other.sink_count(0) == 1);
        CHECK(other.serialize(0, RKV_WIRE_FP16_SCALE) == blob);
        std::vector<uint8_t> truncated(blob.begin(), blob.end() - 5);
        CHECK_THROWS_AS(other.deserialize(truncated, 1), std::runtime_error);
    }

    // rotate_rows + calibrate_reorder on the device == the oracle's on the host
    {
        const int R = 64;
        std::vector<int32_t> dperm, dinv, operm(C), oinv(C);
        rotatekv_b200::calibrate_reorder_device(desc, dk, R, RKV_STAT_MEAN_ABS, dperm, dinv);
        std::vector<float> rows(static_cast<size_t>(R) * C);
        for (size_t i = 0; i < rows.size(); ++i) rows[i] = rkvo_half_to_float(k[i]);
        rkvo_rotate_rows(rows.data(), R, D, G, H);
        rkvo_calibrate_reorder(rows.data(), R, C, RKVO_STAT_MEAN_ABS, operm.data(), oinv.data());
        CHECK(dperm == operm);
    }
    // RotationPlan::make validation (proj/tests/test_hadamard.cpp:57-61)
    rkv_layer_desc bad = desc;
    bad.heads_per_group = 3;
    CHECK_THROWS_AS(rotatekv_b200::DeviceLayerCache(bad, perm), std::invalid_argument);
    // calibrate_reorder KAT (proj/tests/test_reorder.cpp:22-30)
    auto plan = rotatekv_b200::calibrate_reorder({{3.0f, -5.0f, 1.0f}}, 3);
    CHECK(plan.perm[0] == (std::vector<int32_t>{1, 2, 0}));
    CHECK_THROWS_AS(rotatekv_b200::calibrate_reorder({}, 3), std::invalid_argument);

    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dq);
    cudaFree(dout);
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
