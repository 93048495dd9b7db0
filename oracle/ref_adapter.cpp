// ref_adapter.cpp -- extern "C" shims over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/librotatekv_ref.so.  Nothing here re-implements reference
// arithmetic: every function only marshals plain arrays into the reference's
// own types (Tensor, ReorderPlan, LayerKVCache, ...) and calls its public API
// (proj/include/rotatekv/*.hpp).  Used to pin oracle/rkv_oracle.c, to generate
// tests/golden/ fixtures, and as bench.py's CPU reference arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "rotatekv/fp8.hpp"
#include "rotatekv/hadamard.hpp"
#include "rotatekv/kv_cache.hpp"
#include "rotatekv/pipeline.hpp"
#include "rotatekv/quant.hpp"
#include "rotatekv/reorder.hpp"
#include "rotatekv/rng.hpp"
#include "rotatekv/rope.hpp"
#include "rotatekv/sink.hpp"

using namespace rotatekv;

namespace {

ReorderPlan plan_from_perm(const int32_t* perm, int64_t channels) {
    ReorderPlan plan;
    std::vector<int32_t> p(perm, perm + channels), inv(static_cast<size_t>(channels));
    for (int64_t i = 0; i < channels; ++i) inv[static_cast<size_t>(p[static_cast<size_t>(i)])] = static_cast<int32_t>(i);
    plan.perm.push_back(std::move(p));
    plan.inverse.push_back(std::move(inv));
    return plan;
}

Tensor eye(int64_t n) {
    Tensor t({n, n});
    for (int64_t i = 0; i < n; ++i) t.at2(i, i) = 1.0f;
    return t;
}

}  // namespace

// ---------------------------------------------------------------- CPU bench
// bench.py's reference arm: nseq independent sequences, each a LayerKVCache
// of T tokens built through the reference's own append path, then decode
// steps through decode_step.  Harness-level parallelism: one std::thread per
// sequence slice (the reference itself is single-threaded).
struct RefBench {
    int64_t c = 0, h = 0, d = 0, g = 0;
    PipelineConfig cfg;
    AttentionWeights w;
    std::vector<LayerKVCache> caches;
    std::vector<DecodeMemo> memos;  // the reference's own memoisation of reconstructed keys (pipeline.hpp:78-81)
    bool use_memo = true;
    std::vector<int64_t> position;
    uint64_t seed = 0;
};

static Tensor synth_rows(int64_t rows, int64_t c, uint64_t seed) {
    Tensor t({rows, c});
    CounterRng rng(seed);
    for (int64_t i = 0; i < t.numel(); ++i) t[i] = static_cast<float>(rng.normal(static_cast<uint64_t>(i)));
    return t;
}

template <class F>
static void parallel_for(int64_t n, int nthreads, F&& f) {
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
        th.emplace_back([&, w] {
            for (int64_t i = w; i < n; i += nthreads) f(i);
        });
    for (auto& t : th) t.join();
}


extern "C" {

int ref_fwht(float* v, int64_t n) {
    try {
        fwht_inplace(std::span<float>(v, static_cast<size_t>(n)));
        return 0;
    } catch (const std::exception&) { return -1; }
}

int ref_rotate_rows(float* x, int64_t rows, int64_t head_dim, int64_t hpg, int64_t num_heads) {
    try {
        RotationPlan plan = RotationPlan::make(head_dim, hpg, num_heads);
        int64_t c = head_dim * num_heads;
        Tensor t({rows, c}, std::vector<float>(x, x + rows * c));
        Tensor r = rotate_rows(t, plan, false);
        std::memcpy(x, r.data(), sizeof(float) * static_cast<size_t>(rows * c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

int ref_apply_reorder(const float* x, int64_t rows, int64_t channels, const int32_t* perm,
                      int inverse, float* out) {
    try {
        ReorderPlan plan = plan_from_perm(perm, channels);
        Tensor t({rows, channels}, std::vector<float>(x, x + rows * channels));
        Tensor r = apply_reorder(t, plan, 0, inverse != 0);
        std::memcpy(out, r.data(), sizeof(float) * static_cast<size_t>(rows * channels));
        return 0;
    } catch (const std::exception&) { return -1; }
}

int ref_calibrate_reorder(const float* x, int64_t rows, int64_t channels, int32_t* perm,
                          int32_t* inv) {
    try {
        Tensor t({rows, channels}, std::vector<float>(x, x + rows * channels));
        ReorderPlan plan = calibrate_reorder({t});
        std::memcpy(perm, plan.perm[0].data(), sizeof(int32_t) * static_cast<size_t>(channels));
        std::memcpy(inv, plan.inverse[0].data(), sizeof(int32_t) * static_cast<size_t>(channels));
        return 0;
    } catch (const std::exception&) { return -1; }
}

float ref_e4m3_decode(uint8_t c) { return e4m3_decode(c); }
uint8_t ref_e4m3_encode(float x) { return e4m3_encode(x); }
uint8_t ref_e4m3_encode_ceil(float x) { return e4m3_encode_ceil(x); }

// quantize_group (proj/src/quant.cpp:53-97).  codes: unpacked [n]; packed:
// the reference's own LSB-first bytes [(n*bits+7)/8].
int ref_quantize_group(const float* x, int64_t n, int bits, int64_t group_size, uint8_t* codes,
                       uint8_t* packed, uint8_t* scale_e4m3, uint8_t* zero) {
    try {
        QuantConfig cfg;
        cfg.bits = bits;
        cfg.group_size = group_size;
        QuantizedBlock b = quantize_group(std::span<const float>(x, static_cast<size_t>(n)), cfg);
        auto u = unpack_codes(b.codes, bits, b.count);
        std::memcpy(codes, u.data(), u.size());
        std::memcpy(packed, b.codes.data(), b.codes.size());
        *scale_e4m3 = b.scale_e4m3;
        *zero = b.zero_point;
        return 0;
    } catch (const std::exception&) { return -1; }
}

int ref_apply_rope_rows(float* x, int64_t rows, int64_t num_heads, int64_t head_dim, double base,
                        const int64_t* positions, int inverse) {
    try {
        RopeConfig cfg{head_dim, base};
        int64_t c = num_heads * head_dim;
        Tensor t({rows, c}, std::vector<float>(x, x + rows * c));
        Tensor r = apply_rope_rows(t, cfg, num_heads,
                                   std::span<const int64_t>(positions, static_cast<size_t>(rows)),
                                   inverse != 0);
        std::memcpy(x, r.data(), sizeof(float) * static_cast<size_t>(rows * c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

int64_t ref_detect_sinks(const float* hidden, int64_t b, int64_t s, int64_t h, double rel,
                         double abs_floor, uint8_t* flags) {
    try {
        Tensor t({b, s, h}, std::vector<float>(hidden, hidden + b * s * h));
        SinkSet set = detect_massive_activations(t, rel, abs_floor);
        std::memset(flags, 0, static_cast<size_t>(s));
        for (int64_t tok : set.tokens) flags[tok] = 1;
        return static_cast<int64_t>(set.tokens.size());
    } catch (const std::exception&) { return -1; }
}

// The north-star quantize chain through the reference's own functions:
// rotate_rows(K,G) -> apply_reorder -> quantize_token; rotate_rows(V,1) ->
// quantize_token (proj/src/pipeline.cpp:317-324, :120).  Outputs the GPU
// word/meta layout with meta = (e4m3-decoded scale as fp16, zero as fp16).
int ref_quantize_kv_rows(const float* k_raw, const float* v_raw, int64_t rows, int64_t num_heads,
                         int64_t head_dim, int64_t hpg, const int32_t* perm, uint32_t* k_codes,
                         uint8_t* k_scale_e4m3, uint8_t* k_zero, uint32_t* v_codes,
                         uint8_t* v_scale_e4m3, uint8_t* v_zero) {
    try {
        int64_t c = num_heads * head_dim;
        RotationPlan kr = RotationPlan::make(head_dim, hpg, num_heads);
        RotationPlan vr = RotationPlan::make(head_dim, 1, num_heads);
        ReorderPlan plan = plan_from_perm(perm, c);
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        Tensor k({rows, c}, std::vector<float>(k_raw, k_raw + rows * c));
        Tensor v({rows, c}, std::vector<float>(v_raw, v_raw + rows * c));
        Tensor kt = apply_reorder(rotate_rows(k, kr, false), plan, 0, false);
        Tensor vt = rotate_rows(v, vr, false);
        for (int64_t r = 0; r < rows; ++r) {
            auto kb = quantize_token(std::span<const float>(kt.data() + r * c, static_cast<size_t>(c)), q);
            auto vb = quantize_token(std::span<const float>(vt.data() + r * c, static_cast<size_t>(c)), q);
            for (size_t g = 0; g < kb.size(); ++g) {
                std::memcpy(k_codes + r * (c / 16) + g * 8, kb[g].codes.data(), 32);
                std::memcpy(v_codes + r * (c / 16) + g * 8, vb[g].codes.data(), 32);
                k_scale_e4m3[r * (c / 128) + static_cast<int64_t>(g)] = kb[g].scale_e4m3;
                k_zero[r * (c / 128) + static_cast<int64_t>(g)] = kb[g].zero_point;
                v_scale_e4m3[r * (c / 128) + static_cast<int64_t>(g)] = vb[g].scale_e4m3;
                v_zero[r * (c / 128) + static_cast<int64_t>(g)] = vb[g].zero_point;
            }
        }
        return 0;
    } catch (const std::exception&) { return -1; }
}

// LayerKVCache::serialize (proj/src/kv_cache.cpp:119-139) of a cache the
// reference fills from raw rows as prefill does: fused-frame rows (rotate +
// reorder for K, per-head rotate for V), sinks in the fp32 sidecar.  Returns
// the byte count (copies at most cap bytes), -1 on error.
int64_t ref_cache_serialize(const float* k_raw, const float* v_raw, const uint8_t* sink, int64_t rows,
                            int64_t num_heads, int64_t head_dim, int64_t hpg, const int32_t* perm, uint8_t* out,
                            int64_t cap) {
    try {
        int64_t c = num_heads * head_dim;
        RotationPlan kr = RotationPlan::make(head_dim, hpg, num_heads);
        RotationPlan vr = RotationPlan::make(head_dim, 1, num_heads);
        ReorderPlan plan = plan_from_perm(perm, c);
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        Tensor k({rows, c}, std::vector<float>(k_raw, k_raw + rows * c));
        Tensor v({rows, c}, std::vector<float>(v_raw, v_raw + rows * c));
        Tensor kt = apply_reorder(rotate_rows(k, kr, false), plan, 0, false);
        Tensor vt = rotate_rows(v, vr, false);
        LayerKVCache cache(q, c);
        for (int64_t r = 0; r < rows; ++r)
            cache.append(std::span<const float>(kt.data() + r * c, static_cast<size_t>(c)),
                         std::span<const float>(vt.data() + r * c, static_cast<size_t>(c)), sink[r] != 0);
        std::vector<uint8_t> bytes = cache.serialize();
        std::memcpy(out, bytes.data(), std::min<size_t>(bytes.size(), static_cast<size_t>(cap)));
        return static_cast<int64_t>(bytes.size());
    } catch (const std::exception&) { return -1; }
}

// LayerKVCache::deserialize then serialize again (the reference accepts the
// bytes and reproduces them); returns the byte count or -1 if it throws.
int64_t ref_cache_reserialize(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap) {
    try {
        LayerKVCache cache = LayerKVCache::deserialize(std::span<const uint8_t>(in, static_cast<size_t>(n)));
        std::vector<uint8_t> bytes = cache.serialize();
        std::memcpy(out, bytes.data(), std::min<size_t>(bytes.size(), static_cast<size_t>(cap)));
        return static_cast<int64_t>(bytes.size());
    } catch (const std::exception&) { return -1; }
}

// One decode step through the reference's own decode_step
// (proj/src/pipeline.cpp:193-263) with identity projections, so the decode
// token's raw row x is simultaneously its key, value and query.  The prefix
// cache is filled exactly as prefill does (proj/src/pipeline.cpp:171-176):
// fused-frame rows (rotate+reorder for K, per-head rotate for V), sinks kept
// in the fp32 sidecar.  out = decode_step's [C] output (V rotation undone by
// W_o_f).  MHA only: the reference has no GQA.
int ref_decode_step(int64_t num_heads, int64_t head_dim, int64_t hpg, const float* k_raw,
                    const float* v_raw, const uint8_t* sink, int64_t T, const int32_t* perm,
                    double rope_base, const float* x, float* out) {
    try {
        int64_t c = num_heads * head_dim;
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        PipelineConfig cfg = PipelineConfig::make(PipelineMode::RotateKV, num_heads, head_dim, hpg, q, true);
        cfg.reorder = plan_from_perm(perm, c);
        cfg.rope.base = rope_base;
        AttentionWeights w;
        w.wq = eye(c);
        w.wk = eye(c);
        w.wv = eye(c);
        w.wo = eye(c);
        fuse_weights(w, cfg.key_rotation, cfg.reorder, cfg.value_rotation);
        LayerKVCache cache(q, c);
        if (T > 0) {
            Tensor k({T, c}, std::vector<float>(k_raw, k_raw + T * c));
            Tensor v({T, c}, std::vector<float>(v_raw, v_raw + T * c));
            Tensor kt = apply_reorder(rotate_rows(k, cfg.key_rotation, false), cfg.reorder, 0, false);
            Tensor vt = rotate_rows(v, cfg.value_rotation, false);
            for (int64_t t = 0; t < T; ++t)
                cache.append(std::span<const float>(kt.data() + t * c, static_cast<size_t>(c)),
                             std::span<const float>(vt.data() + t * c, static_cast<size_t>(c)),
                             sink[t] != 0);
        }
        Tensor row({1, c}, std::vector<float>(x, x + c));
        Tensor o = decode_step(row, cache, w, cfg, T, nullptr);
        std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

// The reference's own prefill (proj/src/pipeline.cpp:156-191) with identity
// projections: x [T][C] is each token's key, value and query; token 0 and the
// flagged tokens are sinks; out = prefill's attention output [T][C] (after the
// fused W_o, i.e. V's rotation undone).  MHA only (the reference has no GQA).
int ref_prefill(int64_t num_heads, int64_t head_dim, int64_t hpg, const float* x, const uint8_t* sink, int64_t T,
                const int32_t* perm, double rope_base, float* out) {
    try {
        int64_t c = num_heads * head_dim;
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        PipelineConfig cfg = PipelineConfig::make(PipelineMode::RotateKV, num_heads, head_dim, hpg, q, true);
        cfg.reorder = plan_from_perm(perm, c);
        cfg.rope.base = rope_base;
        AttentionWeights w;
        w.wq = eye(c);
        w.wk = eye(c);
        w.wv = eye(c);
        w.wo = eye(c);
        fuse_weights(w, cfg.key_rotation, cfg.reorder, cfg.value_rotation);
        SinkSet extra;
        extra.tokens.push_back(0);  // token 0 is always a member (proj/include/rotatekv/sink.hpp:18-19)
        for (int64_t t = 1; t < T; ++t)
            if (sink[t]) extra.tokens.push_back(t);
        Tensor xt({1, T, c}, std::vector<float>(x, x + T * c));
        PrefillResult r = prefill(xt, w, cfg, &extra);
        std::memcpy(out, r.output.data(), sizeof(float) * static_cast<size_t>(T * c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

void* ref_bench_create(int64_t num_heads, int64_t head_dim, int64_t hpg, int64_t T, int64_t nseq,
                       const int32_t* perm, double rope_base, uint64_t seed, int nthreads) {
    try {
        auto* b = new RefBench();
        b->h = num_heads;
        b->d = head_dim;
        b->g = hpg;
        b->c = num_heads * head_dim;
        b->seed = seed;
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        b->cfg = PipelineConfig::make(PipelineMode::RotateKV, num_heads, head_dim, hpg, q, true);
        b->cfg.reorder = plan_from_perm(perm, b->c);
        b->cfg.rope.base = rope_base;
        b->w.wq = eye(b->c);
        b->w.wk = eye(b->c);
        b->w.wv = eye(b->c);
        b->w.wo = eye(b->c);
        fuse_weights(b->w, b->cfg.key_rotation, b->cfg.reorder, b->cfg.value_rotation);
        b->caches.assign(static_cast<size_t>(nseq), LayerKVCache(q, b->c));
        b->memos.assign(static_cast<size_t>(nseq), DecodeMemo{});
        b->position.assign(static_cast<size_t>(nseq), T);
        parallel_for(nseq, nthreads, [&](int64_t s) {
            Tensor k = synth_rows(T, b->c, seed ^ (0x1000ULL + static_cast<uint64_t>(s)));
            Tensor v = synth_rows(T, b->c, seed ^ (0x2000ULL + static_cast<uint64_t>(s)));
            Tensor kt = apply_reorder(rotate_rows(k, b->cfg.key_rotation, false), b->cfg.reorder, 0, false);
            Tensor vt = rotate_rows(v, b->cfg.value_rotation, false);
            auto& cache = b->caches[static_cast<size_t>(s)];
            for (int64_t t = 0; t < T; ++t)
                cache.append(std::span<const float>(kt.data() + t * b->c, static_cast<size_t>(b->c)),
                             std::span<const float>(vt.data() + t * b->c, static_cast<size_t>(b->c)),
                             t == 0);
        });
        return b;
    } catch (const std::exception&) { return nullptr; }
}

// One decode step (append + attention) for every sequence; returns seconds.
double ref_bench_step(void* handle, int nthreads) {
    auto* b = static_cast<RefBench*>(handle);
    auto t0 = std::chrono::steady_clock::now();
    parallel_for(static_cast<int64_t>(b->caches.size()), nthreads, [&](int64_t s) {
        auto& pos = b->position[static_cast<size_t>(s)];
        Tensor x = synth_rows(1, b->c, b->seed ^ (0x3000ULL + static_cast<uint64_t>(s) * 7919ULL + static_cast<uint64_t>(pos)));
        Tensor o = decode_step(x, b->caches[static_cast<size_t>(s)], b->w, b->cfg, pos,
                               b->use_memo ? &b->memos[static_cast<size_t>(s)] : nullptr);
        (void)o;
        ++pos;
    });
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

void ref_bench_destroy(void* handle) { delete static_cast<RefBench*>(handle); }

// LayerKVCache::keys() / values() (proj/src/kv_cache.cpp:68-85) of a cache
// filled like ref_decode_step: the stored fused-frame rows (dequantised
// blocks, fp32 sidecar rows for sinks), [T][C] each.
int ref_cache_rows(int64_t num_heads, int64_t head_dim, int64_t hpg, const float* k_raw, const float* v_raw,
                   const uint8_t* sink, int64_t T, const int32_t* perm, float* k_out, float* v_out) {
    try {
        int64_t c = num_heads * head_dim;
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        PipelineConfig cfg = PipelineConfig::make(PipelineMode::RotateKV, num_heads, head_dim, hpg, q, true);
        cfg.reorder = plan_from_perm(perm, c);
        LayerKVCache cache(q, c);
        Tensor k({T, c}, std::vector<float>(k_raw, k_raw + T * c));
        Tensor v({T, c}, std::vector<float>(v_raw, v_raw + T * c));
        Tensor kt = apply_reorder(rotate_rows(k, cfg.key_rotation, false), cfg.reorder, 0, false);
        Tensor vt = rotate_rows(v, cfg.value_rotation, false);
        for (int64_t t = 0; t < T; ++t)
            cache.append(std::span<const float>(kt.data() + t * c, static_cast<size_t>(c)),
                         std::span<const float>(vt.data() + t * c, static_cast<size_t>(c)), sink[t] != 0);
        Tensor ks = cache.keys(), vs = cache.values();
        std::memcpy(k_out, ks.data(), sizeof(float) * static_cast<size_t>(T * c));
        std::memcpy(v_out, vs.data(), sizeof(float) * static_cast<size_t>(T * c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

// memo = 1 (default): decode_step memoises the reconstructed post-RoPE keys
// across steps (the reference's DecodeMemo; the first step after creation
// reconstructs the whole cache once); memo = 0: every step reconstructs it.
void ref_bench_set_memo(void* handle, int memo) { static_cast<RefBench*>(handle)->use_memo = memo != 0; }

// route_sinks after the fact (proj/src/sink.cpp:47-63 -> kv_cache.cpp:43-55):
// the cache is filled like ref_decode_step (sinks flagged at append time in
// `sink`), then the tokens `promote[0..np)` are routed to the fp32 sidecar with
// their fused-frame rows, then one decode_step with x.  Returns -1 on an
// exception (e.g. an out-of-range token), -2 if promote_to_sink did not make
// the tokens sinks.
int ref_decode_step_routed(int64_t num_heads, int64_t head_dim, int64_t hpg, const float* k_raw, const float* v_raw,
                           const uint8_t* sink, int64_t T, const int64_t* promote, int64_t np, const int32_t* perm,
                           double rope_base, const float* x, float* out) {
    try {
        int64_t c = num_heads * head_dim;
        QuantConfig q;
        q.bits = 2;
        q.group_size = 128;
        PipelineConfig cfg = PipelineConfig::make(PipelineMode::RotateKV, num_heads, head_dim, hpg, q, true);
        cfg.reorder = plan_from_perm(perm, c);
        cfg.rope.base = rope_base;
        AttentionWeights w;
        w.wq = eye(c);
        w.wk = eye(c);
        w.wv = eye(c);
        w.wo = eye(c);
        fuse_weights(w, cfg.key_rotation, cfg.reorder, cfg.value_rotation);
        LayerKVCache cache(q, c);
        Tensor k({T, c}, std::vector<float>(k_raw, k_raw + T * c));
        Tensor v({T, c}, std::vector<float>(v_raw, v_raw + T * c));
        Tensor kt = apply_reorder(rotate_rows(k, cfg.key_rotation, false), cfg.reorder, 0, false);
        Tensor vt = rotate_rows(v, cfg.value_rotation, false);
        for (int64_t t = 0; t < T; ++t)
            cache.append(std::span<const float>(kt.data() + t * c, static_cast<size_t>(c)),
                         std::span<const float>(vt.data() + t * c, static_cast<size_t>(c)), sink[t] != 0);
        SinkSet set;
        for (int64_t i = 0; i < np; ++i) set.tokens.push_back(promote[i]);
        route_sinks(cache, set, kt, vt);
        for (int64_t i = 0; i < np; ++i)
            if (!cache.is_sink(promote[i])) return -2;
        Tensor row({1, c}, std::vector<float>(x, x + c));
        Tensor o = decode_step(row, cache, w, cfg, T, nullptr);
        std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(c));
        return 0;
    } catch (const std::exception&) { return -1; }
}

}  // extern "C"
