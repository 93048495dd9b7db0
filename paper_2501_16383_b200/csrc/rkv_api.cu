// rkv_api.cu -- the extern "C" boundary (include/rotatekv/rotatekv.h).
//
// Validation mirrors the reference's exceptions: RotationPlan::make
// (proj/src/hadamard.cpp:18-33), QuantConfig::validate (proj/src/quant.cpp:
// 15-23), rope check_cfg (proj/src/rope.cpp:8-12), calibrate_reorder
// (proj/src/reorder.cpp:91-93), detect_massive_activations
// (proj/src/sink.cpp:16-24).  Messages keep the reference's wording where
// one exists.  Host-only entry points (validate, carve, calibrate, detect)
// run without a GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "rkv_internal.h"
#include "rkv_layout.h"

namespace {

thread_local std::string g_err;

rkv_status fail(rkv_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

rkv_status cuda_fail(cudaError_t e, const char* where) {
    return fail(RKV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct CacheSizes {
    size_t codes, meta, sink, sink_pos, sink_count, mask;
};

CacheSizes cache_sizes(const rkv_layer_desc& d) {
    const size_t C = static_cast<size_t>(d.num_kv_heads) * d.head_dim;
    const size_t B = static_cast<size_t>(d.batch), T = static_cast<size_t>(d.max_tokens);
    CacheSizes s{};
    s.codes = al256(B * T * (C / 16) * 4);
    s.meta = al256(B * T * (C / 128) * 4);
    s.sink = al256(B * static_cast<size_t>(d.max_sinks) * C * 2);
    s.sink_pos = al256(B * static_cast<size_t>(d.max_sinks) * 4);
    s.sink_count = al256(B * 4);
    s.mask = al256(B * ((T + 31) / 32) * 4);
    return s;
}

rkv_status validate(const rkv_layer_desc* d) {
    if (!d) return fail(RKV_ERR_INVALID_ARGUMENT, "layer descriptor is null");
    if (d->batch < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1 || d->head_dim < 1 || d->heads_per_group < 1)
        return fail(RKV_ERR_INVALID_ARGUMENT, "rotation plan dimensions must be positive");
    if (d->num_kv_heads % d->heads_per_group != 0)
        return fail(RKV_ERR_INVALID_ARGUMENT, "heads_per_group must divide num_heads");
    const int64_t n = static_cast<int64_t>(d->heads_per_group) * d->head_dim;
    if (!is_pow2(n)) return fail(RKV_ERR_INVALID_ARGUMENT, "rotation matrix dimension must be a power of two");
    if (n > (int64_t{1} << 13)) return fail(RKV_ERR_INVALID_ARGUMENT, "rotation matrix dimension exceeds 2^13");
    if (d->bits < 1 || d->bits > 8) return fail(RKV_ERR_INVALID_ARGUMENT, "quant bits must be in [1,8]");
    if (d->group_size < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "quant group_size must be >= 1");
    if (!(d->rope_base > 1.0)) return fail(RKV_ERR_INVALID_ARGUMENT, "rope: base must be > 1");
    if (d->head_dim % 2 != 0) return fail(RKV_ERR_INVALID_ARGUMENT, "rope: head_dim must be even and >= 2");
    if (d->num_q_heads % d->num_kv_heads != 0)
        return fail(RKV_ERR_INVALID_ARGUMENT, "num_q_heads must be a multiple of num_kv_heads");
    if (d->max_tokens < 1 || d->max_tokens > (int64_t{1} << 30))
        return fail(RKV_ERR_INVALID_ARGUMENT, "max_tokens must be in [1, 2^30]");
    if (d->max_sinks < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "max_sinks must be >= 0");
    if (d->scale_format != RKV_SCALE_FP16_CEIL && d->scale_format != RKV_SCALE_E4M3_CEIL)
        return fail(RKV_ERR_INVALID_ARGUMENT, "unknown scale_format");
    if (d->reserved != 0) return fail(RKV_ERR_INVALID_ARGUMENT, "reserved field must be 0");
    // sm_100a kernel specialisation limits (documented in DESIGN.md)
    if (d->head_dim != 128) return fail(RKV_ERR_INVALID_ARGUMENT, "the sm_100a kernels need head_dim == 128");
    if (d->bits != 2 || d->group_size != 128)
        return fail(RKV_ERR_INVALID_ARGUMENT, "the sm_100a kernels implement bits == 2, group_size == 128");
    const int64_t C = static_cast<int64_t>(d->num_kv_heads) * d->head_dim;
    if (C > 8192) return fail(RKV_ERR_INVALID_ARGUMENT, "num_kv_heads*head_dim must be <= 8192");
    // every power-of-two rotation size up to 2^13 and every head ratio has a kernel
    // (the generic one where the specialised ones do not tile); it keeps a row and
    // the per-head state in shared memory
    if (rkv::decode_kind(*d) == rkv::kDecodeGeneric && rkv::generic_decode_smem(*d) > 227 * 1024)
        return fail(RKV_ERR_INVALID_ARGUMENT, "too many query heads for the generic decode kernel's shared memory");
    return RKV_OK;
}

// stable ascending argsort of the per-channel statistic (proj/src/reorder.cpp:105-109)
void sort_channels(const std::vector<double>& key, int32_t* perm_out, int32_t* inverse_out) {
    std::vector<int32_t> order(key.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return key[static_cast<size_t>(a)] < key[static_cast<size_t>(b)]; });
    std::memcpy(perm_out, order.data(), order.size() * sizeof(int32_t));
    if (inverse_out)
        for (size_t j = 0; j < order.size(); ++j) inverse_out[order[j]] = static_cast<int32_t>(j);
}


// ---------------------------------------------------------------- wire format
// Host helpers for rkv_cache_export / rkv_cache_import.

float half_bits_to_float(uint16_t h) {
    const uint32_t sgn = static_cast<uint32_t>(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
    uint32_t bits;
    if (e == 0) {
        if (m == 0) {
            bits = sgn;
        } else {  // subnormal: normalise
            int sh = 0;
            while (!(m & 0x400u)) {
                m <<= 1;
                ++sh;
            }
            bits = sgn | ((113u - static_cast<uint32_t>(sh)) << 23) | ((m & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        bits = sgn | 0x7f800000u | (m << 13);
    } else {
        bits = sgn | ((e + 112u) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
}

uint16_t float_to_half_bits(float f) {  // round to nearest even
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sgn = (x >> 16) & 0x8000u;
    const int32_t e = static_cast<int32_t>((x >> 23) & 0xffu) - 127 + 15;
    uint32_t m = x & 0x7fffffu;
    if (((x >> 23) & 0xffu) == 0xffu) return static_cast<uint16_t>(sgn | 0x7c00u | (m ? 0x200u : 0u));
    if (e >= 31) return static_cast<uint16_t>(sgn | 0x7c00u);
    if (e <= 0) {
        if (e < -10) return static_cast<uint16_t>(sgn);
        m |= 0x800000u;
        const int sh = 14 - e;
        uint32_t hm = m >> sh;
        const uint32_t rem = m & ((1u << sh) - 1), half = 1u << (sh - 1);
        if (rem > half || (rem == half && (hm & 1u))) ++hm;
        return static_cast<uint16_t>(sgn | hm);
    }
    uint32_t hm = m >> 13;
    const uint32_t rem = m & 0x1fffu;
    uint32_t he = static_cast<uint32_t>(e);
    if (rem > 0x1000u || (rem == 0x1000u && (hm & 1u))) {
        if (++hm == 0x400u) {
            hm = 0;
            ++he;
        }
    }
    if (he >= 31) return static_cast<uint16_t>(sgn | 0x7c00u);
    return static_cast<uint16_t>(sgn | (he << 10) | hm);
}

float e4m3_value(uint8_t c) {  // OCP e4m3fn, positive codes
    const int e = (c >> 3) & 0xf, m = c & 7;
    return e == 0 ? std::ldexp(static_cast<float>(m), -9) : std::ldexp(1.0f + m * 0.125f, e - 7);
}

bool e4m3_code_of(float v, uint8_t* code) {  // exact inverse on e4m3 values
    for (int c = 0; c <= 0x7e; ++c)
        if (e4m3_value(static_cast<uint8_t>(c)) == v) {
            *code = static_cast<uint8_t>(c);
            return true;
        }
    return false;
}

// In-place grouped FWHT of one row (rotate_rows, proj/src/hadamard.cpp:47-84):
// stages half = 1, 2, ..., n/2 in fp32, then x 1/sqrtf(n).
void fwht_row(float* x, int64_t C, int64_t n) {
    const float norm = 1.0f / std::sqrt(static_cast<float>(n));
    for (int64_t base = 0; base < C; base += n) {
        float* v = x + base;
        for (int64_t h = 1; h < n; h <<= 1)
            for (int64_t i = 0; i < n; i += 2 * h)
                for (int64_t j = i; j < i + h; ++j) {
                    const float a = v[j], b = v[j + h];
                    v[j] = a + b;
                    v[j + h] = a - b;
                }
        for (int64_t j = 0; j < n; ++j) v[j] *= norm;
    }
}

void put_u64(std::vector<uint8_t>& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_f32(std::vector<uint8_t>& o, float f) {
    uint32_t b;
    std::memcpy(&b, &f, 4);
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(b >> (8 * i)));
}

rkv_status check_cache(const rkv_cache* c) {
    if (!c || !c->k_codes || !c->v_codes || !c->k_meta || !c->v_meta || !c->sink_count || !c->sink_mask)
        return fail(RKV_ERR_INVALID_ARGUMENT, "cache arrays must be non-null");
    return RKV_OK;
}

}  // namespace

extern "C" {

const char* rkv_last_error(void) { return g_err.c_str(); }

const char* rkv_version(void) { return "rotatekv-b200 0.1 (sm_100a)"; }

rkv_status rkv_layer_validate(const rkv_layer_desc* desc) { return validate(desc); }

size_t rkv_cache_bytes(const rkv_layer_desc* desc) {
    if (validate(desc) != RKV_OK) return 0;
    CacheSizes s = cache_sizes(*desc);
    return 2 * s.codes + 2 * s.meta + 2 * s.sink + s.sink_pos + s.sink_count + s.mask;
}

rkv_status rkv_cache_carve(const rkv_layer_desc* desc, void* base, size_t bytes, rkv_cache* out) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if (!base || !out) return fail(RKV_ERR_INVALID_ARGUMENT, "cache_carve: null pointer");
    if (reinterpret_cast<uintptr_t>(base) % 256 != 0)
        return fail(RKV_ERR_INVALID_ARGUMENT, "cache_carve: base must be 256-byte aligned");
    if (bytes < rkv_cache_bytes(desc)) return fail(RKV_ERR_INVALID_ARGUMENT, "cache_carve: buffer too small");
    CacheSizes s = cache_sizes(*desc);
    char* p = static_cast<char*>(base);
    out->k_codes = reinterpret_cast<uint32_t*>(p), p += s.codes;
    out->v_codes = reinterpret_cast<uint32_t*>(p), p += s.codes;
    out->k_meta = reinterpret_cast<uint32_t*>(p), p += s.meta;
    out->v_meta = reinterpret_cast<uint32_t*>(p), p += s.meta;
    out->sink_k = reinterpret_cast<uint16_t*>(p), p += s.sink;
    out->sink_v = reinterpret_cast<uint16_t*>(p), p += s.sink;
    out->sink_pos = reinterpret_cast<int32_t*>(p), p += s.sink_pos;
    out->sink_count = reinterpret_cast<int32_t*>(p), p += s.sink_count;
    out->sink_mask = reinterpret_cast<uint32_t*>(p);
    return RKV_OK;
}

rkv_status rkv_cache_reset(const rkv_layer_desc* desc, const rkv_cache* cache, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    CacheSizes s = cache_sizes(*desc);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(cache->sink_count, 0, static_cast<size_t>(desc->batch) * 4, cs);
    if (e == cudaSuccess) e = cudaMemsetAsync(cache->sink_mask, 0, s.mask, cs);
    if (e == cudaSuccess && cache->sink_pos) e = cudaMemsetAsync(cache->sink_pos, 0, s.sink_pos, cs);
    if (e != cudaSuccess) return cuda_fail(e, "cache_reset");
    return RKV_OK;
}

size_t rkv_rope_table_bytes(const rkv_layer_desc* desc, int64_t max_pos) {
    if (validate(desc) != RKV_OK || max_pos < 1) return 0;
    // per position pair 128 float4: section 1 (cos p0, cos p1, sin p0, sin p1) x 64
    // frequencies, section 2 two [32] frequency-pair rows (decode_attention.cu)
    const size_t npairs = static_cast<size_t>((max_pos + 1) / 2);
    return 2 * npairs * (desc->head_dim / 2) * 4 * sizeof(float);
}

rkv_status rkv_rope_table_init(const rkv_layer_desc* desc, float* table, int64_t max_pos, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if (!table || max_pos < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "rope_table_init: null table or max_pos < 1");
    cudaError_t e = rkv::launch_rope_table(*desc, reinterpret_cast<float4*>(table), max_pos,
                                           static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rope_table_init");
    return RKV_OK;
}

rkv_status rkv_quantize_kv(const rkv_layer_desc* desc, const uint16_t* k_new, const uint16_t* v_new,
                           const int32_t* perm, const uint8_t* sink_flags, const int64_t* start_pos,
                           int64_t num_new, const rkv_cache* cache, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (num_new < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv: num_new must be >= 0");
    if (num_new == 0) return RKV_OK;
    if (!k_new || !v_new || !perm || !start_pos)
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv: k_new, v_new, perm and start_pos must be non-null");
    if (num_new > desc->max_tokens) return fail(RKV_ERR_OUT_OF_RANGE, "quantize_kv: num_new exceeds max_tokens");
    if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new) | reinterpret_cast<uintptr_t>(perm)) &
        15u)
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv: k_new, v_new and perm must be 16-byte aligned");
    if (sink_flags && (!cache->sink_k || !cache->sink_v || !cache->sink_pos))
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv: sink flags need the sidecar arrays");
    rkv::QuantParams p{};
    p.k_new = k_new;
    p.v_new = v_new;
    p.perm = perm;
    p.sink_flags = sink_flags;
    p.start_pos = start_pos;
    p.num_new = num_new;
    p.max_tokens = desc->max_tokens;
    p.C = desc->num_kv_heads * desc->head_dim;
    p.max_sinks = desc->max_sinks;
    p.scale_format = desc->scale_format;
    p.k_norm = 1.0f / std::sqrt(static_cast<float>(desc->heads_per_group * desc->head_dim));
    p.v_norm = 1.0f / std::sqrt(static_cast<float>(desc->head_dim));
    p.cache = *cache;
    cudaError_t e = rkv::launch_quantize(*desc, p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "quantize_kv");
    return RKV_OK;
}

rkv_status rkv_quantize_kv_fused(const rkv_layer_desc* desc, const void* k_rows, const void* v_rows, int32_t dtype,
                                 const int32_t* perm, const uint8_t* sink_flags, const int64_t* start_pos,
                                 int64_t num_new, const rkv_cache* cache, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (dtype != RKV_ROWS_F32 && dtype != RKV_ROWS_F16)
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv_fused: dtype must be RKV_ROWS_F32 or RKV_ROWS_F16");
    if (num_new < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv_fused: num_new must be >= 0");
    if (num_new == 0) return RKV_OK;
    if (!k_rows || !v_rows || !perm || !start_pos)
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv_fused: k_rows, v_rows, perm and start_pos must be non-null");
    if (num_new > desc->max_tokens) return fail(RKV_ERR_OUT_OF_RANGE, "quantize_kv_fused: num_new exceeds max_tokens");
    if ((reinterpret_cast<uintptr_t>(k_rows) | reinterpret_cast<uintptr_t>(v_rows)) & 15u)
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv_fused: k_rows and v_rows must be 16-byte aligned");
    if (sink_flags && (!cache->sink_k || !cache->sink_v || !cache->sink_pos))
        return fail(RKV_ERR_INVALID_ARGUMENT, "quantize_kv_fused: sink flags need the sidecar arrays");
    rkv::QuantParams p{};
    p.perm = perm;
    p.sink_flags = sink_flags;
    p.start_pos = start_pos;
    p.num_new = num_new;
    p.max_tokens = desc->max_tokens;
    p.C = desc->num_kv_heads * desc->head_dim;
    p.max_sinks = desc->max_sinks;
    p.scale_format = desc->scale_format;
    p.k_norm = 1.0f / std::sqrt(static_cast<float>(desc->heads_per_group * desc->head_dim));
    p.v_norm = 1.0f / std::sqrt(static_cast<float>(desc->head_dim));
    p.cache = *cache;
    cudaError_t e = rkv::launch_quantize_fused(*desc, p, k_rows, v_rows, dtype, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "quantize_kv_fused");
    return RKV_OK;
}

rkv_status rkv_promote_sinks(const rkv_layer_desc* desc, const rkv_cache* cache, const int64_t* tokens,
                             int64_t num_tokens, const uint16_t* k_rows, const uint16_t* v_rows, int32_t* promoted,
                             void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (num_tokens < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "promote_sinks: num_tokens must be >= 0");
    if (num_tokens == 0) return RKV_OK;
    if (num_tokens > rkv::promote_sinks_max())
        return fail(RKV_ERR_INVALID_ARGUMENT, "promote_sinks: at most 256 tokens per sequence and call");
    if (!tokens || !k_rows || !v_rows) return fail(RKV_ERR_INVALID_ARGUMENT, "promote_sinks: null argument");
    if (!cache->sink_k || !cache->sink_v || !cache->sink_pos)
        return fail(RKV_ERR_INVALID_ARGUMENT, "promote_sinks: the cache has no sidecar arrays");
    rkv::QuantParams p{};
    p.k_new = k_rows;
    p.v_new = v_rows;
    p.max_tokens = desc->max_tokens;
    p.C = desc->num_kv_heads * desc->head_dim;
    p.max_sinks = desc->max_sinks;
    p.cache = *cache;
    cudaError_t e = rkv::launch_promote_sinks(*desc, p, tokens, static_cast<int>(num_tokens), promoted,
                                              static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "promote_sinks");
    return RKV_OK;
}

rkv_status rkv_cache_read(const rkv_layer_desc* desc, const rkv_cache* cache, const int32_t* perm, int64_t seq,
                          int64_t t0, int64_t num_tokens, int32_t frame, float* k_out, float* v_out, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (frame != RKV_FRAME_STORED && frame != RKV_FRAME_RAW)
        return fail(RKV_ERR_INVALID_ARGUMENT, "cache_read: frame must be RKV_FRAME_STORED or RKV_FRAME_RAW");
    if (seq < 0 || seq >= desc->batch || t0 < 0 || num_tokens < 0 || t0 + num_tokens > desc->max_tokens)
        return fail(RKV_ERR_OUT_OF_RANGE, "cache: token index out of range");
    if (num_tokens == 0) return RKV_OK;
    if (!perm || !k_out || !v_out) return fail(RKV_ERR_INVALID_ARGUMENT, "cache_read: null argument");
    cudaError_t e = rkv::launch_cache_read(*desc, *cache, perm, static_cast<int>(seq), t0, num_tokens, frame, k_out,
                                           v_out, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cache_read");
    return RKV_OK;
}

size_t rkv_layer_plan_bytes(const rkv_layer_desc* desc) {
    if (validate(desc) != RKV_OK) return 0;
    const int W = desc->num_kv_heads * desc->head_dim / 16;
    return static_cast<size_t>(rkv::plan_words(W)) * 4;
}

rkv_status rkv_layer_plan_build(const rkv_layer_desc* desc, const int32_t* perm, uint32_t* plan_host,
                                size_t bytes, int32_t* cost_out) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if (!perm || !plan_host) return fail(RKV_ERR_INVALID_ARGUMENT, "layer_plan: null argument");
    const int C = desc->num_kv_heads * desc->head_dim;
    std::vector<int32_t> inv(static_cast<size_t>(C), -1);
    for (int j = 0; j < C; ++j) {
        if (perm[j] < 0 || perm[j] >= C || inv[static_cast<size_t>(perm[j])] != -1)
            return fail(RKV_ERR_INVALID_ARGUMENT, "reorder plan: perm must be a permutation of the channel count");
        inv[static_cast<size_t>(perm[j])] = j;
    }
    std::vector<uint32_t> words;
    int cost = 0;
    if (!rkv::build_decode_plan(*desc, perm, words, cost)) return fail(RKV_ERR_RUNTIME, "layer_plan: build failed");
    if (bytes < words.size() * 4) return fail(RKV_ERR_INVALID_ARGUMENT, "layer_plan: buffer too small");
    std::memcpy(plan_host, words.data(), words.size() * 4);
    if (cost_out) *cost_out = cost;
    return RKV_OK;
}

rkv_status rkv_layer_plan_init(const rkv_layer_desc* desc, const int32_t* perm, void* plan_dev, size_t bytes,
                               void* stream) {
    std::vector<uint32_t> host(bytes / 4);
    rkv_status st = rkv_layer_plan_build(desc, perm, host.data(), bytes, nullptr);
    if (st != RKV_OK) return st;
    if (!plan_dev) return fail(RKV_ERR_INVALID_ARGUMENT, "layer_plan: null device buffer");
    const size_t used = rkv_layer_plan_bytes(desc);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(plan_dev, host.data(), used, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);  // host staging buffer dies on return
    if (e != cudaSuccess) return cuda_fail(e, "layer_plan_init");
    return RKV_OK;
}

namespace {
rkv::DecodeParams decode_params(const rkv_layer_desc* desc, const rkv::DecodePlan& pl, const uint16_t* q,
                                const int64_t* seq_len, const rkv_cache* cache, const void* layer_plan,
                                const float* rope_table, float* out, void* workspace) {
    const size_t rows = static_cast<size_t>(desc->batch) * pl.NP * desc->num_q_heads;
    rkv::DecodeParams p{};
    p.q = q;
    p.seq_len = seq_len;
    p.plan = static_cast<const uint32_t*>(layer_plan);
    p.rope = reinterpret_cast<const float4*>(rope_table);
    p.cache = *cache;
    if (workspace) {
        p.ws_ml = static_cast<float*>(workspace);
        p.ws_o = reinterpret_cast<float*>(static_cast<char*>(workspace) + al256(rows * 2 * sizeof(float)));
    }
    p.out = out;
    p.max_tokens = desc->max_tokens;
    p.B = desc->batch;
    p.Hq = desc->num_q_heads;
    p.Hkv = desc->num_kv_heads;
    p.C = desc->num_kv_heads * desc->head_dim;
    p.S = pl.S;
    p.NP = pl.NP;
    p.max_sinks = desc->max_sinks;
    p.chunk = pl.chunk;
    p.P = pl.P;
    p.P_pairs = pl.PP;
    p.stages = pl.stages;
    p.k_norm = 1.0f / std::sqrt(static_cast<float>(desc->heads_per_group * desc->head_dim));
    p.qscale = rkv::kLog2eHost / std::sqrt(static_cast<float>(desc->head_dim));
    return p;
}
}  // namespace

size_t rkv_decode_workspace_bytes(const rkv_layer_desc* desc, int64_t max_seq_len) {
    if (validate(desc) != RKV_OK) return 0;
    const rkv::DecodePlan& pl = rkv::cached_plan(*desc, max_seq_len);
    const size_t rows = static_cast<size_t>(desc->batch) * pl.NP * desc->num_q_heads;
    return al256(rows * 2 * sizeof(float)) + al256(rows * 128 * sizeof(float));
}

rkv_status rkv_decode_attention(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len,
                                int64_t max_seq_len, const rkv_cache* cache, const void* layer_plan,
                                const float* rope_table, float* out, void* workspace, size_t ws_bytes,
                                void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (!q || !seq_len || !layer_plan || !rope_table || !out || !workspace)
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention: null argument");
    if (max_seq_len < 0 || max_seq_len > desc->max_tokens)
        return fail(RKV_ERR_OUT_OF_RANGE, "decode_attention: max_seq_len exceeds max_tokens");
    if (max_seq_len == 0) max_seq_len = desc->max_tokens;
    if (ws_bytes < rkv_decode_workspace_bytes(desc, max_seq_len))
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention: workspace too small");
    const rkv::DecodePlan& pl = rkv::cached_plan(*desc, max_seq_len);
    if (!pl.ok)
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention: layer shape exceeds the sm_100a kernel's tile budget");
    rkv::DecodeParams p = decode_params(desc, pl, q, seq_len, cache, layer_plan, rope_table, out, workspace);
    cudaError_t e = rkv::launch_decode(*desc, pl, p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "decode_attention");
    return RKV_OK;
}

rkv_status rkv_decode_attention_partial(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len,
                                        const int64_t* tok_begin, const int64_t* tok_end, int64_t max_span,
                                        const rkv_cache* cache, const void* layer_plan, const float* rope_table,
                                        float* part_ml, float* part_o, void* workspace, size_t ws_bytes,
                                        void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (!q || !seq_len || !tok_begin || !tok_end || !layer_plan || !rope_table || !part_ml || !part_o || !workspace)
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention_partial: null argument");
    if (max_span < 1 || max_span > desc->max_tokens)
        return fail(RKV_ERR_OUT_OF_RANGE, "decode_attention_partial: max_span must be in [1, max_tokens]");
    if (ws_bytes < rkv_decode_workspace_bytes(desc, max_span))
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention_partial: workspace too small");
    const rkv::DecodePlan& pl = rkv::cached_plan(*desc, max_span);
    if (!pl.ok)
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_attention_partial: layer shape exceeds the kernel's tile budget");
    rkv::DecodeParams p = decode_params(desc, pl, q, seq_len, cache, layer_plan, rope_table, part_o, workspace);
    p.tok_begin = tok_begin;
    p.tok_end = tok_end;
    p.partial_ml = part_ml;
    cudaError_t e = rkv::launch_decode(*desc, pl, p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "decode_attention_partial");
    return RKV_OK;
}

rkv_status rkv_decode_merge(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len, int32_t num_parts,
                            const float* parts_ml, const float* parts_o, const rkv_cache* cache,
                            const float* rope_table, float* out, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (!q || !seq_len || !parts_ml || !parts_o || !rope_table || !out)
        return fail(RKV_ERR_INVALID_ARGUMENT, "decode_merge: null argument");
    if (num_parts < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "decode_merge: num_parts must be >= 1");
    rkv::DecodePlan pl{};
    pl.NP = num_parts;
    rkv::DecodeParams p = decode_params(desc, pl, q, seq_len, cache, nullptr, rope_table, out, nullptr);
    p.ws_ml = const_cast<float*>(parts_ml);  // [B][num_parts][Hq][2]
    p.ws_o = const_cast<float*>(parts_o);    // [B][num_parts][Hq][d]
    cudaError_t e = rkv::launch_decode_combine(p, desc->batch, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "decode_merge");
    return RKV_OK;
}

namespace {
// reconstructed K (hi, lo) + V tiles: 48 KB per (sequence, KV head, 64 keys)
size_t prefill_tile_bytes(const rkv_layer_desc& d) {
    const size_t nt = static_cast<size_t>((d.max_tokens + rkv::kPrefillKT - 1) / rkv::kPrefillKT);
    return static_cast<size_t>(d.batch) * d.num_kv_heads * nt * rkv::kPrefillTileBytes;
}
}  // namespace

size_t rkv_prefill_workspace_bytes(const rkv_layer_desc* desc, int64_t num_q, int64_t max_seq_len) {
    if (validate(desc) != RKV_OK || num_q < 0 || max_seq_len < 0) return 0;
    const size_t rows = static_cast<size_t>(desc->batch) * static_cast<size_t>(rkv::prefill_q_pad(num_q)) *
                        static_cast<size_t>(desc->num_q_heads);
    return al256(prefill_tile_bytes(*desc)) + al256(rows * 512);
}

rkv_status rkv_prefill_attention(const rkv_layer_desc* desc, const uint16_t* q, int64_t num_q, const int64_t* q_start,
                                 const int64_t* seq_len, int64_t max_seq_len, const rkv_cache* cache,
                                 const void* layer_plan, const float* rope_table, float* out, void* workspace,
                                 size_t ws_bytes, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (num_q < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "prefill: negative query count");
    if (num_q == 0) return RKV_OK;
    if (!q || !q_start || !seq_len || !layer_plan || !rope_table || !out || !workspace)
        return fail(RKV_ERR_INVALID_ARGUMENT, "prefill: null argument");
    if (max_seq_len < 1 || max_seq_len > desc->max_tokens)
        return fail(RKV_ERR_OUT_OF_RANGE, "prefill: max_seq_len must be in [1, max_tokens]");
    if (rkv::decode_kind(*desc) != rkv::kDecodeMma)
        return fail(RKV_ERR_INVALID_ARGUMENT,
                    "prefill: the tensor-core path covers Hq == Hkv with G = 1, 2, 4 and C a multiple of 512 "
                    "up to 8192, and GQA (any Hq / Hkv >= 2) with G = 2 or 4 and Hkv <= 16");
    if (desc->max_sinks > rkv::kPrefillMaxSinks)
        return fail(RKV_ERR_INVALID_ARGUMENT, "prefill: at most 16 sink rows per sequence (max_sinks <= 16)");
    if (ws_bytes < rkv_prefill_workspace_bytes(desc, num_q, max_seq_len))
        return fail(RKV_ERR_INVALID_ARGUMENT, "prefill: workspace too small");
    const size_t C = static_cast<size_t>(desc->num_kv_heads) * desc->head_dim;
    const size_t tiles = al256(prefill_tile_bytes(*desc));
    char* w = static_cast<char*>(workspace);
    rkv::PrefillParams p{};
    p.q = q;
    p.q_start = q_start;
    p.seq_len = seq_len;
    p.plan = static_cast<const uint32_t*>(layer_plan);
    p.rope = reinterpret_cast<const float4*>(rope_table);
    p.cache = *cache;
    p.kv_tiles = reinterpret_cast<unsigned char*>(w);
    p.kv_tiles_per_seq = (desc->max_tokens + rkv::kPrefillKT - 1) / rkv::kPrefillKT;
    p.q_rows = reinterpret_cast<unsigned char*>(w + tiles);
    p.num_q_pad = rkv::prefill_q_pad(num_q);
    p.out = out;
    p.max_tokens = desc->max_tokens;
    p.num_q = num_q;
    p.B = desc->batch;
    p.Hq = desc->num_q_heads;
    p.Hkv = desc->num_kv_heads;
    p.C = static_cast<int>(C);
    p.max_sinks = desc->max_sinks;
    p.k_norm = 1.0f / std::sqrt(static_cast<float>(desc->heads_per_group * desc->head_dim));
    p.qscale = rkv::kLog2eHost / std::sqrt(static_cast<float>(desc->head_dim));
    cudaError_t e = rkv::launch_prefill(*desc, p, max_seq_len, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "prefill_attention");
    return RKV_OK;
}

rkv_status rkv_rotate_keys(const rkv_layer_desc* desc, const uint16_t* k, int64_t rows, float* out, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if (!k || !out || rows < 0) return fail(RKV_ERR_INVALID_ARGUMENT, "rotate_keys: null argument");
    if (rows == 0) return RKV_OK;
    cudaError_t e = rkv::launch_rotate_keys(*desc, k, rows, out, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rotate_keys");
    return RKV_OK;
}

rkv_status rkv_calibrate_reorder(const float* rotated_keys, int64_t rows, int64_t channels, int32_t stat,
                                 int32_t* perm_out, int32_t* inverse_out) {
    if (!rotated_keys || !perm_out) return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: null argument");
    if (rows < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: empty calibration set");
    if (channels < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: channels must be >= 1");
    if (stat != RKV_STAT_SUM && stat != RKV_STAT_MEAN_ABS)
        return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: unknown statistic");
    // per-channel statistic accumulated sequentially over rows in double
    std::vector<double> key(static_cast<size_t>(channels), 0.0);
    for (int64_t i = 0; i < rows; ++i) {
        const float* r = rotated_keys + i * channels;
        for (int64_t j = 0; j < channels; ++j) {
            const double v = r[j];
            key[static_cast<size_t>(j)] += stat == RKV_STAT_MEAN_ABS ? std::fabs(v) : v;
        }
    }
    if (stat == RKV_STAT_MEAN_ABS)
        for (double& k : key) k /= static_cast<double>(rows);
    sort_channels(key, perm_out, inverse_out);
    return RKV_OK;
}

size_t rkv_calibrate_workspace_bytes(const rkv_layer_desc* desc, int64_t rows) {
    if (validate(desc) != RKV_OK || rows < 1) return 0;
    const size_t C = static_cast<size_t>(desc->num_kv_heads) * desc->head_dim;
    return al256(static_cast<size_t>(rows) * C * sizeof(float)) + al256(C * sizeof(double));
}

rkv_status rkv_calibrate_reorder_device(const rkv_layer_desc* desc, const uint16_t* k_rows, int64_t rows,
                                        int32_t stat, void* workspace, size_t workspace_bytes, int32_t* perm_out,
                                        int32_t* inverse_out, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if (rows < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: empty calibration set");
    if (!k_rows || !workspace || !perm_out) return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: null argument");
    if (stat != RKV_STAT_SUM && stat != RKV_STAT_MEAN_ABS)
        return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: unknown statistic");
    if (workspace_bytes < rkv_calibrate_workspace_bytes(desc, rows))
        return fail(RKV_ERR_INVALID_ARGUMENT, "calibrate_reorder: workspace too small");
    const int64_t C = static_cast<int64_t>(desc->num_kv_heads) * desc->head_dim;
    float* rotated = static_cast<float*>(workspace);
    double* stats = reinterpret_cast<double*>(static_cast<char*>(workspace) +
                                              al256(static_cast<size_t>(rows) * C * sizeof(float)));
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    cudaError_t e = rkv::launch_rotate_keys(*desc, k_rows, rows, rotated, cs);
    if (e == cudaSuccess) e = rkv::launch_channel_stats(rotated, rows, C, stat == RKV_STAT_MEAN_ABS, stats, cs);
    std::vector<double> key(static_cast<size_t>(C));
    if (e == cudaSuccess) e = cudaMemcpyAsync(key.data(), stats, key.size() * sizeof(double), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return cuda_fail(e, "calibrate_reorder_device");
    sort_channels(key, perm_out, inverse_out);
    return RKV_OK;
}

size_t rkv_cache_wire_bytes(const rkv_layer_desc* desc, int64_t tokens, int64_t num_sinks, int32_t format) {
    if (validate(desc) != RKV_OK || tokens < 0 || num_sinks < 0 || num_sinks > tokens) return 0;
    const size_t C = static_cast<size_t>(desc->num_kv_heads) * desc->head_dim, G = C / 128;
    const size_t block = (format == RKV_WIRE_FP16_SCALE ? 2 : 1) + 1 + 32;
    const size_t sink_row = format == RKV_WIRE_FP16_SCALE ? 2 : 4;  // raw fp16 rows vs fused-frame fp32 rows
    return 25 + static_cast<size_t>(tokens) + static_cast<size_t>(num_sinks) * 2 * C * sink_row +
           static_cast<size_t>(tokens - num_sinks) * 2 * G * block;
}

rkv_status rkv_cache_export(const rkv_layer_desc* desc, const rkv_cache* cache, int64_t seq, int64_t tokens,
                            const int32_t* perm, int32_t format, uint8_t* out, size_t out_bytes, size_t* written,
                            void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (!perm || !out) return fail(RKV_ERR_INVALID_ARGUMENT, "cache serialize: null argument");
    if (format != RKV_WIRE_REFERENCE && format != RKV_WIRE_FP16_SCALE)
        return fail(RKV_ERR_INVALID_ARGUMENT, "cache serialize: unknown wire format");
    if (seq < 0 || seq >= desc->batch) return fail(RKV_ERR_OUT_OF_RANGE, "cache serialize: sequence index");
    if (tokens < 0 || tokens > desc->max_tokens) return fail(RKV_ERR_OUT_OF_RANGE, "cache serialize: token count");
    const int64_t C = static_cast<int64_t>(desc->num_kv_heads) * desc->head_dim, W = C / 16, MG = C / 128;
    const int64_t N = static_cast<int64_t>(desc->heads_per_group) * desc->head_dim, T = desc->max_tokens;
    const int64_t MW = (T + 31) / 32, S = desc->max_sinks;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    std::vector<uint32_t> kc(static_cast<size_t>(tokens * W)), vc(kc.size()), km(static_cast<size_t>(tokens * MG)),
        vm(km.size()), mask(static_cast<size_t>(MW));
    std::vector<uint16_t> sk(static_cast<size_t>(S * C)), sv(sk.size());
    std::vector<int32_t> spos(static_cast<size_t>(S));
    int32_t scount = 0;
    const int64_t r0 = seq * T;
    cudaError_t e = cudaSuccess;
    auto d2h = [&](void* dst, const void* src, size_t n) {
        if (e == cudaSuccess && n) e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, cs);
    };
    d2h(kc.data(), cache->k_codes + r0 * W, kc.size() * 4);
    d2h(vc.data(), cache->v_codes + r0 * W, vc.size() * 4);
    d2h(km.data(), cache->k_meta + r0 * MG, km.size() * 4);
    d2h(vm.data(), cache->v_meta + r0 * MG, vm.size() * 4);
    d2h(mask.data(), cache->sink_mask + seq * MW, mask.size() * 4);
    d2h(&scount, cache->sink_count + seq, 4);
    if (S > 0 && cache->sink_k && cache->sink_v && cache->sink_pos) {
        d2h(sk.data(), cache->sink_k + seq * S * C, sk.size() * 2);
        d2h(sv.data(), cache->sink_v + seq * S * C, sv.size() * 2);
        d2h(spos.data(), cache->sink_pos + seq * S, spos.size() * 4);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return cuda_fail(e, "cache serialize");
    scount = std::min<int32_t>(scount, static_cast<int32_t>(S));

    std::vector<uint8_t> o;
    o.reserve(rkv_cache_wire_bytes(desc, tokens, 0, format));
    o.push_back(static_cast<uint8_t>(desc->bits | (format == RKV_WIRE_FP16_SCALE ? 0x80 : 0)));
    put_u64(o, static_cast<uint64_t>(desc->group_size));
    put_u64(o, static_cast<uint64_t>(C));
    put_u64(o, static_cast<uint64_t>(tokens));
    std::vector<float> row(static_cast<size_t>(C)), tmp(static_cast<size_t>(C));
    for (int64_t t = 0; t < tokens; ++t) {
        const bool sink = (mask[static_cast<size_t>(t >> 5)] >> (t & 31)) & 1u;
        o.push_back(sink ? 1 : 0);
        if (sink) {
            int s = -1;
            for (int i = 0; i < scount; ++i)
                if (spos[static_cast<size_t>(i)] == t) s = i;
            if (s < 0) return fail(RKV_ERR_RUNTIME, "cache serialize: sink row missing from the sidecar");
            if (format == RKV_WIRE_FP16_SCALE) {  // lossless: the raw fp16 rows as stored
                for (int64_t j = 0; j < C; ++j) {
                    o.push_back(static_cast<uint8_t>(sk[static_cast<size_t>(s * C + j)] & 0xffu));
                    o.push_back(static_cast<uint8_t>(sk[static_cast<size_t>(s * C + j)] >> 8));
                }
                for (int64_t j = 0; j < C; ++j) {
                    o.push_back(static_cast<uint8_t>(sv[static_cast<size_t>(s * C + j)] & 0xffu));
                    o.push_back(static_cast<uint8_t>(sv[static_cast<size_t>(s * C + j)] >> 8));
                }
                continue;
            }
            // K' = apply_reorder(rotate_rows(k, G)) (slot j <- channel perm[j]); V' = rotate_rows(v, 1)
            for (int64_t j = 0; j < C; ++j) tmp[static_cast<size_t>(j)] = half_bits_to_float(sk[static_cast<size_t>(s * C + j)]);
            fwht_row(tmp.data(), C, N);
            for (int64_t j = 0; j < C; ++j) row[static_cast<size_t>(j)] = tmp[static_cast<size_t>(perm[j])];
            for (float f : row) put_f32(o, f);
            for (int64_t j = 0; j < C; ++j) row[static_cast<size_t>(j)] = half_bits_to_float(sv[static_cast<size_t>(s * C + j)]);
            fwht_row(row.data(), C, desc->head_dim);
            for (float f : row) put_f32(o, f);
            continue;
        }
        for (int kv = 0; kv < 2; ++kv) {
            const uint32_t* codes = (kv ? vc : kc).data() + t * W;
            const uint32_t* meta = (kv ? vm : km).data() + t * MG;
            for (int64_t g = 0; g < MG; ++g) {
                const uint16_t sbits = static_cast<uint16_t>(meta[g] & 0xffffu);
                const float zero = half_bits_to_float(static_cast<uint16_t>(meta[g] >> 16));
                if (format == RKV_WIRE_REFERENCE) {
                    uint8_t code;
                    if (!e4m3_code_of(half_bits_to_float(sbits), &code))
                        return fail(RKV_ERR_INVALID_ARGUMENT,
                                    "cache serialize: scale is not an e4m3 value (use RKV_WIRE_FP16_SCALE or "
                                    "scale_format = RKV_SCALE_E4M3_CEIL)");
                    o.push_back(code);
                } else {
                    o.push_back(static_cast<uint8_t>(sbits & 0xffu));
                    o.push_back(static_cast<uint8_t>(sbits >> 8));
                }
                o.push_back(static_cast<uint8_t>(zero));
                for (int w = 0; w < 8; ++w)
                    for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(codes[g * 8 + w] >> (8 * i)));
            }
        }
    }
    if (written) *written = o.size();
    if (out_bytes < o.size()) return fail(RKV_ERR_INVALID_ARGUMENT, "cache serialize: output buffer too small");
    std::memcpy(out, o.data(), o.size());
    return RKV_OK;
}

rkv_status rkv_cache_import(const rkv_layer_desc* desc, const uint8_t* bytes, size_t num_bytes, const int32_t* perm,
                            int64_t seq, const rkv_cache* cache, int64_t* tokens_out, void* stream) {
    rkv_status st = validate(desc);
    if (st != RKV_OK) return st;
    if ((st = check_cache(cache)) != RKV_OK) return st;
    if (!perm) return fail(RKV_ERR_INVALID_ARGUMENT, "cache deserialize: null argument");
    if (seq < 0 || seq >= desc->batch) return fail(RKV_ERR_OUT_OF_RANGE, "cache deserialize: sequence index");
    if (!bytes || num_bytes == 0) return fail(RKV_ERR_RUNTIME, "cache deserialize: empty input");
    size_t off = 0;
    auto need = [&](size_t n) { return off + n <= num_bytes; };
    auto u64 = [&]() {
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(bytes[off + i]) << (8 * i);
        off += 8;
        return v;
    };
    if (!need(25)) return fail(RKV_ERR_RUNTIME, "cache deserialize: truncated");
    const uint8_t hdr = bytes[off++];
    const bool fp16 = (hdr & 0x80) != 0;
    const int bits = hdr & 0x7f;
    const uint64_t group = u64(), channels = u64(), tokens = u64();
    const int64_t C = static_cast<int64_t>(desc->num_kv_heads) * desc->head_dim, W = C / 16, MG = C / 128;
    const int64_t N = static_cast<int64_t>(desc->heads_per_group) * desc->head_dim, T = desc->max_tokens;
    const int64_t MW = (T + 31) / 32, S = desc->max_sinks;
    if (bits != desc->bits || group != static_cast<uint64_t>(desc->group_size) || channels != static_cast<uint64_t>(C))
        return fail(RKV_ERR_INVALID_ARGUMENT, "cache deserialize: bits / group / channels differ from the layer");
    if (tokens > static_cast<uint64_t>(T)) return fail(RKV_ERR_OUT_OF_RANGE, "cache deserialize: more tokens than max_tokens");
    const int64_t n = static_cast<int64_t>(tokens);
    std::vector<uint32_t> kc(static_cast<size_t>(n * W), 0u), vc(kc.size(), 0u), km(static_cast<size_t>(n * MG), 0u),
        vm(km.size(), 0u), mask(static_cast<size_t>(MW), 0u);
    std::vector<uint16_t> sk(static_cast<size_t>(S * C), 0), sv(sk.size(), 0);
    std::vector<int32_t> spos(static_cast<size_t>(S), 0);
    int32_t scount = 0;
    std::vector<float> row(static_cast<size_t>(C)), tmp(static_cast<size_t>(C));
    auto f32 = [&]() {
        uint32_t b = 0;
        for (int i = 0; i < 4; ++i) b |= static_cast<uint32_t>(bytes[off + i]) << (8 * i);
        off += 4;
        float f;
        std::memcpy(&f, &b, 4);
        return f;
    };
    const size_t block = (fp16 ? 2 : 1) + 1 + 32;
    for (int64_t t = 0; t < n; ++t) {
        if (!need(1)) return fail(RKV_ERR_RUNTIME, "cache deserialize: truncated");
        const bool sink = bytes[off++] != 0;
        if (sink) {
            if (!need(static_cast<size_t>(2 * C * (fp16 ? 2 : 4)))) return fail(RKV_ERR_RUNTIME, "cache deserialize: truncated");
            if (scount >= S) return fail(RKV_ERR_OUT_OF_RANGE, "cache deserialize: more sinks than max_sinks");
            spos[static_cast<size_t>(scount)] = static_cast<int32_t>(t);
            mask[static_cast<size_t>(t >> 5)] |= 1u << (t & 31);
            if (fp16) {  // raw fp16 rows (RKV_WIRE_FP16_SCALE)
                for (int64_t j = 0; j < 2 * C; ++j) {
                    const uint16_t h = static_cast<uint16_t>(bytes[off] | (bytes[off + 1] << 8));
                    off += 2;
                    (j < C ? sk : sv)[static_cast<size_t>(scount * C + (j % C))] = h;
                }
                ++scount;
                continue;
            }
            // back to the raw frame: k = rotate_G(unreorder(K')), v = rotate_1(V') (the FWHT is an involution)
            for (int64_t j = 0; j < C; ++j) row[static_cast<size_t>(j)] = f32();
            for (int64_t j = 0; j < C; ++j) tmp[static_cast<size_t>(perm[j])] = row[static_cast<size_t>(j)];
            fwht_row(tmp.data(), C, N);
            for (int64_t j = 0; j < C; ++j) sk[static_cast<size_t>(scount * C + j)] = float_to_half_bits(tmp[static_cast<size_t>(j)]);
            for (int64_t j = 0; j < C; ++j) row[static_cast<size_t>(j)] = f32();
            fwht_row(row.data(), C, desc->head_dim);
            for (int64_t j = 0; j < C; ++j) sv[static_cast<size_t>(scount * C + j)] = float_to_half_bits(row[static_cast<size_t>(j)]);
            ++scount;
            continue;
        }
        if (!need(static_cast<size_t>(2 * MG) * block)) return fail(RKV_ERR_RUNTIME, "cache deserialize: truncated");
        for (int kv = 0; kv < 2; ++kv) {
            uint32_t* codes = (kv ? vc : kc).data() + t * W;
            uint32_t* meta = (kv ? vm : km).data() + t * MG;
            for (int64_t g = 0; g < MG; ++g) {
                uint16_t sbits;
                if (fp16) {
                    sbits = static_cast<uint16_t>(bytes[off] | (bytes[off + 1] << 8));
                    off += 2;
                } else {
                    sbits = float_to_half_bits(e4m3_value(bytes[off++]));  // exact: e4m3 values are fp16 values
                }
                const uint16_t zbits = float_to_half_bits(static_cast<float>(bytes[off++]));
                meta[g] = static_cast<uint32_t>(sbits) | (static_cast<uint32_t>(zbits) << 16);
                for (int w = 0; w < 8; ++w) {
                    uint32_t v = 0;
                    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(bytes[off + i]) << (8 * i);
                    off += 4;
                    codes[g * 8 + w] = v;
                }
            }
        }
    }
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const int64_t r0 = seq * T;
    cudaError_t e = cudaSuccess;
    auto h2d = [&](void* dst, const void* src, size_t nb) {
        if (e == cudaSuccess && nb) e = cudaMemcpyAsync(dst, src, nb, cudaMemcpyHostToDevice, cs);
    };
    h2d(cache->k_codes + r0 * W, kc.data(), kc.size() * 4);
    h2d(cache->v_codes + r0 * W, vc.data(), vc.size() * 4);
    h2d(cache->k_meta + r0 * MG, km.data(), km.size() * 4);
    h2d(cache->v_meta + r0 * MG, vm.data(), vm.size() * 4);
    h2d(cache->sink_mask + seq * MW, mask.data(), mask.size() * 4);
    h2d(cache->sink_count + seq, &scount, 4);
    if (S > 0 && cache->sink_k && cache->sink_v && cache->sink_pos) {
        h2d(cache->sink_k + seq * S * C, sk.data(), sk.size() * 2);
        h2d(cache->sink_v + seq * S * C, sv.data(), sv.size() * 2);
        h2d(cache->sink_pos + seq * S, spos.data(), spos.size() * 4);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);  // host staging buffers die on return
    if (e != cudaSuccess) return cuda_fail(e, "cache deserialize");
    if (tokens_out) *tokens_out = n;
    return RKV_OK;
}

rkv_status rkv_detect_sinks(const float* hidden, int64_t b, int64_t s, int64_t h, double rel_threshold,
                            double abs_floor, uint8_t* flags, int64_t* num_sinks) {
    if (!hidden || !flags) return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: null argument");
    if (b < 1 || h < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: expected [b,s,hidden]");
    if (!(rel_threshold > 1.0))
        return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: rel_threshold must be > 1");
    if (s < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: empty sequence");
    const int64_t n = b * s * h;
    std::vector<float> mags(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) mags[static_cast<size_t>(i)] = std::fabs(hidden[i]);
    // the element a full ascending sort would put at index n/2
    std::nth_element(mags.begin(), mags.begin() + n / 2, mags.end());
    const double threshold = rel_threshold * static_cast<double>(mags[static_cast<size_t>(n / 2)]);
    int64_t count = 0;
    for (int64_t t = 0; t < s; ++t) {
        bool hit = t == 0;
        for (int64_t bi = 0; bi < b && !hit; ++bi) {
            const float* row = hidden + (bi * s + t) * h;
            for (int64_t c = 0; c < h; ++c) {
                const double v = std::fabs(row[c]);
                if (v > threshold && v > abs_floor) {
                    hit = true;
                    break;
                }
            }
        }
        flags[t] = hit ? 1 : 0;
        count += hit ? 1 : 0;
    }
    if (num_sinks) *num_sinks = count;
    return RKV_OK;
}

size_t rkv_detect_sinks_workspace_bytes(void) { return rkv::detect_sinks_workspace_bytes(); }

rkv_status rkv_detect_sinks_device(const float* hidden, int64_t b, int64_t s, int64_t h, double rel_threshold,
                                   double abs_floor, uint8_t* flags, float* median_out, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    if (!hidden || !flags || !workspace)
        return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: null argument");
    if (b < 1 || h < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: expected [b,s,hidden]");
    if (!(rel_threshold > 1.0))
        return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: rel_threshold must be > 1");
    if (s < 1) return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: empty sequence");
    if (workspace_bytes < rkv::detect_sinks_workspace_bytes())
        return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: workspace too small");
    if (reinterpret_cast<uintptr_t>(hidden) & 15u)
        return fail(RKV_ERR_INVALID_ARGUMENT, "detect_massive_activations: hidden must be 16-byte aligned");
    cudaError_t e = rkv::launch_detect_sinks(hidden, b, s, h, rel_threshold, abs_floor, flags, median_out, workspace,
                                             static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "detect_massive_activations");
    return RKV_OK;
}

}  // extern "C"
