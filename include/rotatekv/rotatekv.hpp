// rotatekv.hpp -- C++ host API over the C ABI (rotatekv.h), mirroring the
// reference's hot-path API (namespace rotatekv, /root/reference/proj/include/
// rotatekv/{reorder,kv_cache,pipeline}.hpp) so a reference caller switches by
// changing the namespace and handing device pointers.  Header-only; link
// against paper_2501_16383_b200/_lib/librotatekv_b200.so and cudart.
//
//   reference                                   rotatekv_b200
//   ------------------------------------------  -----------------------------------------
//   ReorderPlan calibrate_reorder(layers)        ReorderPlan calibrate_reorder(layers, C, stat)
//   LayerKVCache(cfg, C); append(k, v, sink)     DeviceLayerCache(desc, perm); append(...)
//   LayerKVCache::size()/is_sink()               DeviceLayerCache::size(b)/sink_count(b)
//   decode_step(...) attention half              DeviceLayerCache::decode_attention(q, out)
//   prefill(...) attention half                  DeviceLayerCache::prefill_attention(q, n, q_start, out)
//
// Exceptions are the reference's: std::invalid_argument, std::out_of_range,
// std::runtime_error (CUDA failures included).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rotatekv/rotatekv.h"

namespace rotatekv_b200 {

inline void check(rkv_status s) {
    switch (s) {
        case RKV_OK: return;
        case RKV_ERR_INVALID_ARGUMENT: throw std::invalid_argument(rkv_last_error());
        case RKV_ERR_OUT_OF_RANGE: throw std::out_of_range(rkv_last_error());
        default: throw std::runtime_error(rkv_last_error());
    }
}

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// proj/include/rotatekv/reorder.hpp:14-28
struct ReorderPlan {
    std::vector<std::vector<int32_t>> perm;     // perm[l][j] = source channel of slot j
    std::vector<std::vector<int32_t>> inverse;  // inverse[l][perm[l][j]] == j
    int64_t layers() const { return static_cast<int64_t>(perm.size()); }
    int64_t channels() const { return perm.empty() ? 0 : static_cast<int64_t>(perm[0].size()); }
};

// calibrate_reorder (proj/src/reorder.cpp:91-110): one [rows x channels]
// row-major fp32 tensor of ROTATED keys per layer.
inline ReorderPlan calibrate_reorder(const std::vector<std::vector<float>>& rotated_keys_per_layer,
                                     int64_t channels, rkv_calib_stat stat = RKV_STAT_SUM) {
    if (rotated_keys_per_layer.empty()) throw std::invalid_argument("calibrate_reorder: empty calibration set");
    ReorderPlan plan;
    for (const auto& layer : rotated_keys_per_layer) {
        if (channels < 1 || layer.size() % static_cast<size_t>(channels) != 0)
            throw std::invalid_argument("calibrate_reorder: rows must be [tokens, channels]");
        std::vector<int32_t> p(static_cast<size_t>(channels)), inv(static_cast<size_t>(channels));
        check(rkv_calibrate_reorder(layer.data(), static_cast<int64_t>(layer.size()) / channels, channels, stat,
                                    p.data(), inv.data()));
        plan.perm.push_back(std::move(p));
        plan.inverse.push_back(std::move(inv));
    }
    return plan;
}

// apply_reorder (proj/src/reorder.cpp:112-128) on host rows.
// rotate_rows + calibrate_reorder on device keys (proj/src/pipeline.cpp:101-109):
// k_rows [rows][C] fp16 device -> perm / inverse of one layer (bit-identical to the host path).
inline void calibrate_reorder_device(const rkv_layer_desc& desc, const uint16_t* k_rows, int64_t rows, int32_t stat,
                                     std::vector<int32_t>& perm, std::vector<int32_t>& inverse,
                                     cudaStream_t stream = nullptr) {
    const size_t c = static_cast<size_t>(desc.num_kv_heads) * desc.head_dim;
    const size_t ws_bytes = rkv_calibrate_workspace_bytes(&desc, rows);
    void* ws = nullptr;
    if (ws_bytes) check_cuda(cudaMalloc(&ws, ws_bytes), "cudaMalloc calibration workspace");
    perm.resize(c);
    inverse.resize(c);
    const rkv_status st =
        rkv_calibrate_reorder_device(&desc, k_rows, rows, stat, ws, ws_bytes, perm.data(), inverse.data(), stream);
    cudaFree(ws);
    check(st);
}

inline std::vector<float> apply_reorder(const std::vector<float>& x, const ReorderPlan& plan, int64_t layer,
                                        bool inverse) {
    if (layer < 0 || layer >= plan.layers()) throw std::invalid_argument("apply_reorder: layer out of range");
    const auto& p = inverse ? plan.inverse[static_cast<size_t>(layer)] : plan.perm[static_cast<size_t>(layer)];
    const size_t c = p.size();
    if (c == 0 || x.size() % c != 0) throw std::invalid_argument("apply_reorder: trailing dimension mismatch");
    std::vector<float> out(x.size());
    for (size_t r = 0; r < x.size() / c; ++r)
        for (size_t j = 0; j < c; ++j) out[r * c + j] = x[r * c + static_cast<size_t>(p[j])];
    return out;
}

// detect_massive_activations (proj/src/sink.cpp:14-45) on device memory:
// hidden [b][s][h] fp32 -> flags [s] u8 (device), optional device median.
// Allocates its small workspace per call; use rkv_detect_sinks_device with a
// persistent workspace inside CUDA graphs.
inline void detect_massive_activations_device(const float* hidden, int64_t b, int64_t s, int64_t h, uint8_t* flags,
                                              double rel_threshold = 50.0, double abs_floor = 0.0,
                                              float* median_out = nullptr, cudaStream_t stream = nullptr) {
    const size_t nws = rkv_detect_sinks_workspace_bytes();
    void* ws = nullptr;
    check_cuda(cudaMalloc(&ws, nws), "cudaMalloc sink workspace");
    const rkv_status st =
        rkv_detect_sinks_device(hidden, b, s, h, rel_threshold, abs_floor, flags, median_out, ws, nws, stream);
    cudaStreamSynchronize(stream);
    cudaFree(ws);
    check(st);
}

// One layer's 2-bit rotated KV cache on the device (LayerKVCache,
// proj/include/rotatekv/kv_cache.hpp:13-50, for a batch of sequences).
class DeviceLayerCache {
public:
    DeviceLayerCache(const rkv_layer_desc& desc, const std::vector<int32_t>& perm, cudaStream_t stream = nullptr)
        : desc_(desc), stream_(stream), len_(static_cast<size_t>(desc.batch), 0),
          sinks_(static_cast<size_t>(desc.batch), 0), perm_host_(perm) {
        check(rkv_layer_validate(&desc_));
        const size_t c = static_cast<size_t>(desc.num_kv_heads) * desc.head_dim;
        if (perm.size() != c) throw std::invalid_argument("reorder plan: wrong channel count in layer line");
        bytes_ = rkv_cache_bytes(&desc_);
        check_cuda(cudaMalloc(&base_, bytes_), "cudaMalloc cache");
        check(rkv_cache_carve(&desc_, base_, bytes_, &cache_));
        check_cuda(cudaMalloc(&perm_, c * sizeof(int32_t)), "cudaMalloc perm");
        check_cuda(cudaMemcpyAsync(perm_, perm.data(), c * sizeof(int32_t), cudaMemcpyHostToDevice, stream_), "perm");
        rope_bytes_ = rkv_rope_table_bytes(&desc_, desc.max_tokens);
        check_cuda(cudaMalloc(&rope_, rope_bytes_), "cudaMalloc rope");
        check(rkv_rope_table_init(&desc_, static_cast<float*>(rope_), desc.max_tokens, stream_));
        plan_bytes_ = rkv_layer_plan_bytes(&desc_);
        check_cuda(cudaMalloc(&plan_, plan_bytes_), "cudaMalloc plan");
        check(rkv_layer_plan_init(&desc_, perm.data(), plan_, plan_bytes_, stream_));
        ws_bytes_ = rkv_decode_workspace_bytes(&desc_, desc.max_tokens);
        check_cuda(cudaMalloc(&ws_, ws_bytes_), "cudaMalloc workspace");
        // a small ring of device length vectors: a call whose lengths changed
        // stages them through pinned host memory into the next slot
        // (stream-ordered; the slot's event guards the pinned copy's reuse)
        check_cuda(cudaMalloc(&dev_pos_, kPosRing * static_cast<size_t>(desc.batch) * sizeof(int64_t)),
                   "cudaMalloc pos");
        check_cuda(cudaMallocHost(&host_pos_, kPosRing * static_cast<size_t>(desc.batch) * sizeof(int64_t)),
                   "cudaMallocHost pos");
        for (auto& e : pos_ev_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "pos event");
        sink_set_.resize(static_cast<size_t>(desc.batch));
        check(rkv_cache_reset(&desc_, &cache_, stream_));
    }
    DeviceLayerCache(const DeviceLayerCache&) = delete;
    DeviceLayerCache& operator=(const DeviceLayerCache&) = delete;
    ~DeviceLayerCache() {
        cudaFree(base_);
        cudaFree(perm_);
        cudaFree(rope_);
        cudaFree(ws_);
        cudaFree(plan_);
        cudaFree(dev_pos_);
        cudaFreeHost(host_pos_);
        for (auto e : pos_ev_) cudaEventDestroy(e);
        cudaFree(dev_qs_);
        cudaFree(pf_ws_);
        cudaFree(flags_);
        cudaFree(tok_);
    }

    int64_t size(int b) const { return len_.at(static_cast<size_t>(b)); }
    int64_t sink_count(int b) const { return sinks_.at(static_cast<size_t>(b)); }
    const rkv_cache& view() const { return cache_; }
    const rkv_layer_desc& desc() const { return desc_; }

    // LayerKVCache::append for num_new tokens of every sequence.
    // k_new/v_new: device [B][num_new][C] fp16; sink_flags_host: [B][num_new] or empty.
    // Stream-ordered: returns without synchronizing (k_new/v_new must stay valid
    // until the stream reaches the append).  No allocation after the first
    // call of a given flag size.
    void append(const uint16_t* k_new, const uint16_t* v_new, int64_t num_new,
                const std::vector<uint8_t>& sink_flags_host = {}) {
        append_with(num_new, sink_flags_host, [&](const uint8_t* dflags, const int64_t* pos) {
            return rkv_quantize_kv(&desc_, k_new, v_new, perm_, dflags, pos, num_new, &cache_, stream_);
        });
    }

    // LayerKVCache::append in the reference's fused frame (fuse_weights,
    // proj/src/pipeline.cpp:88-99): k_rows = P H_G k, v_rows = H_128 v, device
    // [B][num_new][C] in `dtype` (RKV_ROWS_F32 = what the reference appends).
    // Quantization only (rkv_quantize_kv_fused); otherwise as append().
    void append_fused(const void* k_rows, const void* v_rows, rkv_rows_dtype dtype, int64_t num_new,
                      const std::vector<uint8_t>& sink_flags_host = {}) {
        append_with(num_new, sink_flags_host, [&](const uint8_t* dflags, const int64_t* pos) {
            return rkv_quantize_kv_fused(&desc_, k_rows, v_rows, dtype, perm_, dflags, pos, num_new, &cache_, stream_);
        });
    }

  private:
    // capacity checks, flag staging and the host mirror around one append call
    template <typename Call>
    void append_with(int64_t num_new, const std::vector<uint8_t>& sink_flags_host, Call&& call) {
        const int B = desc_.batch;
        for (int b = 0; b < B; ++b)
            if (len_[static_cast<size_t>(b)] + num_new > desc_.max_tokens)
                throw std::out_of_range("cache: token index out of range");
        uint8_t* dflags = nullptr;
        if (!sink_flags_host.empty()) {
            if (sink_flags_host.size() != static_cast<size_t>(B) * static_cast<size_t>(num_new))
                throw std::invalid_argument("sink flags must be [batch, new tokens]");
            for (int b = 0; b < B; ++b) {
                int64_t add = 0;
                for (int64_t i = 0; i < num_new; ++i) add += sink_flags_host[static_cast<size_t>(b * num_new + i)] != 0;
                if (sinks_[static_cast<size_t>(b)] + add > desc_.max_sinks)
                    throw std::out_of_range("cache: sink sidecar capacity exceeded");
            }
            dflags = static_cast<uint8_t*>(grow(flags_, flags_bytes_, sink_flags_host.size()));
            // pageable source: the call returns once the bytes are staged, so the
            // host vector may change afterwards; the device copy is stream-ordered
            check_cuda(cudaMemcpyAsync(dflags, sink_flags_host.data(), sink_flags_host.size(), cudaMemcpyHostToDevice,
                                       stream_), "flags");
        }
        int64_t* pos = stage_lengths();
        check(call(dflags, pos));
        for (int b = 0; b < B; ++b) {
            len_[static_cast<size_t>(b)] += num_new;
            if (!sink_flags_host.empty())
                for (int64_t i = 0; i < num_new; ++i)
                    if (sink_flags_host[static_cast<size_t>(b * num_new + i)]) {
                        ++sinks_[static_cast<size_t>(b)];
                        sink_set_[static_cast<size_t>(b)].push_back(len_[static_cast<size_t>(b)] - num_new + i);
                    }
        }
    }

  public:
    // LayerKVCache::promote_to_sink / route_sinks (proj/src/kv_cache.cpp:43-55,
    // proj/src/sink.cpp:47-63): tokens[b] = token indices of sequence b;
    // k_rows/v_rows: device [B][n][C] fp16 raw rows of those tokens, n = the
    // longest list (row i of sequence b belongs to tokens[b][i]).  Tokens that
    // are already sinks are skipped; indices past the cache length throw
    // std::out_of_range like the reference.  Stream-ordered.
    void route_sinks(const std::vector<std::vector<int64_t>>& tokens, const uint16_t* k_rows, const uint16_t* v_rows) {
        const int B = desc_.batch;
        if (tokens.size() != static_cast<size_t>(B)) throw std::invalid_argument("route_sinks: one token list per sequence");
        size_t n = 1;
        for (const auto& t : tokens) n = std::max(n, t.size());
        std::vector<int64_t> flat(static_cast<size_t>(B) * n, -1);
        std::vector<std::vector<int64_t>> fresh(static_cast<size_t>(B));
        for (int b = 0; b < B; ++b) {
            auto& known = sink_set_[static_cast<size_t>(b)];
            for (size_t i = 0; i < tokens[static_cast<size_t>(b)].size(); ++i) {
                const int64_t t = tokens[static_cast<size_t>(b)][i];
                if (t < 0 || t >= len_[static_cast<size_t>(b)]) throw std::out_of_range("route_sinks: token index out of range");
                flat[static_cast<size_t>(b) * n + i] = t;
                if (std::find(known.begin(), known.end(), t) == known.end() &&
                    std::find(fresh[static_cast<size_t>(b)].begin(), fresh[static_cast<size_t>(b)].end(), t) ==
                        fresh[static_cast<size_t>(b)].end())
                    fresh[static_cast<size_t>(b)].push_back(t);
            }
            if (sinks_[static_cast<size_t>(b)] + static_cast<int64_t>(fresh[static_cast<size_t>(b)].size()) >
                desc_.max_sinks)
                throw std::out_of_range("cache: sink sidecar capacity exceeded");
        }
        int64_t* dtok = static_cast<int64_t*>(grow(tok_, tok_bytes_, flat.size() * sizeof(int64_t)));
        check_cuda(cudaMemcpyAsync(dtok, flat.data(), flat.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream_),
                   "tokens");
        check(rkv_promote_sinks(&desc_, &cache_, dtok, static_cast<int64_t>(n), k_rows, v_rows, nullptr, stream_));
        for (int b = 0; b < B; ++b) {
            sinks_[static_cast<size_t>(b)] += static_cast<int64_t>(fresh[static_cast<size_t>(b)].size());
            for (int64_t t : fresh[static_cast<size_t>(b)]) sink_set_[static_cast<size_t>(b)].push_back(t);
        }
    }

    // The attention half of decode_step (proj/src/pipeline.cpp:211-261): q
    // [B][Hq][d] fp16 device (pre-RoPE, position = size-1), out [B][Hq][d] fp32.
    // Stream-ordered: synchronize the stream (or copy out on it) before reading out.
    void decode_attention(const uint16_t* q, float* out) {
        int64_t mx = 0;
        for (int64_t l : len_) {
            if (l < 1) throw std::invalid_argument("decode_step: position must equal current cache length");
            mx = l > mx ? l : mx;
        }
        int64_t* lens = stage_lengths();
        check(rkv_decode_attention(&desc_, q, lens, mx, &cache_, plan_, static_cast<const float*>(rope_), out, ws_,
                                   ws_bytes_, stream_));
    }

    void synchronize() const { check_cuda(cudaStreamSynchronize(stream_), "synchronize"); }

    // LayerKVCache::key_row / value_row / keys / values (proj/src/kv_cache.cpp:57-85):
    // tokens [t0, t0 + n) of sequence b into device [n][C] fp32 rows, the stored
    // fused frame (RKV_FRAME_STORED, the reference's rows) or the model's frame
    // (RKV_FRAME_RAW).  Throws std::out_of_range past the cache length.
    void rows(int b, int64_t t0, int64_t n, int32_t frame, float* k_out, float* v_out) const {
        if (b < 0 || b >= desc_.batch || t0 < 0 || n < 0 || t0 + n > len_[static_cast<size_t>(b)])
            throw std::out_of_range("cache: token index out of range");
        check(rkv_cache_read(&desc_, &cache_, perm_, b, t0, n, frame, k_out, v_out, stream_));
    }

    // The attention half of prefill (proj/src/pipeline.cpp:156-191: reconstruct_cache,
    // causal reference_attention): q [B][num_q][Hq][d] fp16 device, row i of
    // sequence b at position q_start[b] + i attending to cache tokens
    // 0 .. q_start[b] + i; out [B][num_q][Hq][d] fp32 device.
    void prefill_attention(const uint16_t* q, int64_t num_q, const std::vector<int64_t>& q_start, float* out) {
        if (q_start.size() != len_.size()) throw std::invalid_argument("prefill: q_start must hold one entry per sequence");
        if (num_q < 0) throw std::invalid_argument("prefill: negative query count");
        int64_t mx = 1;
        for (size_t b = 0; b < len_.size(); ++b) {
            if (q_start[b] < 0 || q_start[b] + num_q > len_[b])
                throw std::out_of_range("prefill: query rows past the cache length");
            mx = std::max(mx, len_[b]);
        }
        if (num_q == 0) return;
        const size_t need = rkv_prefill_workspace_bytes(&desc_, num_q, mx);
        if (need > pf_ws_bytes_) {
            cudaFree(pf_ws_);
            pf_ws_ = nullptr;
            check_cuda(cudaMalloc(&pf_ws_, need), "cudaMalloc prefill workspace");
            pf_ws_bytes_ = need;
        }
        if (!dev_qs_) check_cuda(cudaMalloc(&dev_qs_, len_.size() * sizeof(int64_t)), "cudaMalloc q_start");
        check_cuda(cudaMemcpyAsync(dev_qs_, q_start.data(), len_.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                                   stream_), "q_start");
        int64_t* lens = stage_lengths();
        check(rkv_prefill_attention(&desc_, q, num_q, dev_qs_, lens, mx, &cache_, plan_,
                                    static_cast<const float*>(rope_), out, pf_ws_, pf_ws_bytes_, stream_));
    }

    // LayerKVCache::serialize (proj/src/kv_cache.cpp:119-139) of sequence b;
    // format RKV_WIRE_REFERENCE (the reference's bytes, e4m3 scales) or
    // RKV_WIRE_FP16_SCALE (lossless for fp16 scales).
    std::vector<uint8_t> serialize(int b, int32_t format) const {
        const int64_t n = size(b);
        std::vector<uint8_t> out(rkv_cache_wire_bytes(&desc_, n, std::min<int64_t>(n, desc_.max_sinks), format));
        size_t written = 0;
        check(rkv_cache_export(&desc_, &cache_, b, n, perm_host_.data(), format, out.data(), out.size(), &written,
                               stream_));
        out.resize(written);
        return out;
    }
    // LayerKVCache::deserialize (proj/src/kv_cache.cpp:141-173) into sequence b.
    void deserialize(const std::vector<uint8_t>& bytes, int b) {
        int64_t n = 0;
        check(rkv_cache_import(&desc_, bytes.data(), bytes.size(), perm_host_.data(), b, &cache_, &n, stream_));
        len_.at(static_cast<size_t>(b)) = n;
        int32_t count = 0;
        check_cuda(cudaMemcpy(&count, cache_.sink_count + b, sizeof(int32_t), cudaMemcpyDeviceToHost), "sink count");
        sinks_[static_cast<size_t>(b)] = count;
        std::vector<int32_t> pos(static_cast<size_t>(count));
        if (count > 0)
            check_cuda(cudaMemcpy(pos.data(), cache_.sink_pos + static_cast<int64_t>(b) * desc_.max_sinks,
                                  pos.size() * sizeof(int32_t), cudaMemcpyDeviceToHost),
                       "sink positions");
        sink_set_[static_cast<size_t>(b)].assign(pos.begin(), pos.end());
    }

private:
    static constexpr size_t kPosRing = 8;
    // the device copy of the host lengths: re-staged only when they changed
    // since the last upload (a decode step after an append uploads once; repeated
    // decodes upload nothing)
    int64_t* stage_lengths() {
        if (last_pos_ && last_len_ == len_) return last_pos_;
        const size_t k = pos_next_++ % kPosRing;
        check_cuda(cudaEventSynchronize(pos_ev_[k]), "lengths slot");  // its previous copy has been read
        int64_t* h = host_pos_ + k * len_.size();
        std::copy(len_.begin(), len_.end(), h);
        int64_t* slot = dev_pos_ + k * len_.size();
        check_cuda(cudaMemcpyAsync(slot, h, len_.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream_), "lengths");
        check_cuda(cudaEventRecord(pos_ev_[k], stream_), "lengths event");
        last_len_ = len_;
        last_pos_ = slot;
        return slot;
    }
    // grow-only device scratch (the old buffer is freed only when it grows)
    void* grow(void*& buf, size_t& have, size_t need) {
        if (need > have) {
            if (buf) {
                check_cuda(cudaStreamSynchronize(stream_), "scratch");
                cudaFree(buf);
                buf = nullptr;
            }
            check_cuda(cudaMalloc(&buf, need), "cudaMalloc scratch");
            have = need;
        }
        return buf;
    }
    rkv_layer_desc desc_;
    cudaStream_t stream_;
    std::vector<int64_t> len_, sinks_;
    void* base_ = nullptr;
    size_t bytes_ = 0;
    rkv_cache cache_{};
    int32_t* perm_ = nullptr;
    void* rope_ = nullptr;
    size_t rope_bytes_ = 0;
    void* ws_ = nullptr;
    size_t ws_bytes_ = 0;
    void* plan_ = nullptr;
    size_t plan_bytes_ = 0;
    int64_t* dev_pos_ = nullptr;
    int64_t* host_pos_ = nullptr;  // pinned staging ring
    cudaEvent_t pos_ev_[kPosRing] = {};
    std::vector<int64_t> last_len_;
    int64_t* last_pos_ = nullptr;
    int64_t* dev_qs_ = nullptr;
    void* pf_ws_ = nullptr;
    size_t pf_ws_bytes_ = 0;
    void* flags_ = nullptr;
    size_t flags_bytes_ = 0;
    void* tok_ = nullptr;
    size_t tok_bytes_ = 0;
    size_t pos_next_ = 0;
    std::vector<std::vector<int64_t>> sink_set_;
    std::vector<int32_t> perm_host_;
};

}  // namespace rotatekv_b200
