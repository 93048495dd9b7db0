// rkv_runtime.cu -- host-side runtime state shared by the launchers.
//
//  * options(): the experiment switches (kernel selection, split counts, the
//    2-SM prefill).  They used to be getenv() calls on every launch; now they
//    are process-global atomics set through rkv_set_debug_option and read
//    when a plan is built.  Every layer plan records the kernel kind it was
//    built for and the decode kernels check it, so a plan built under other
//    switches yields NaN outputs instead of silently wrong attention.
//  * ensure_smem(): cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per
//    (kernel, device, size high-water mark) instead of on every launch.
//  * cached_plan(): decode plans memoised per (descriptor, max_seq_len,
//    device, option epoch) -- the planner runs occupancy queries.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "rkv_internal.h"

namespace rkv {

Options& options() {
    static Options o;
    return o;
}

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    return dev;
}

int num_sms() {
    static std::atomic<int> cache[64];
    const int dev = current_device();
    const int slot = dev & 63;
    int n = cache[slot].load(std::memory_order_relaxed);
    if (n == 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        cache[slot].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t ensure_smem(const void* kern, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = set[{kern, dev}];
    if (have >= bytes && have != 0) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e == cudaSuccess) have = bytes;
    return e;
}

int choose_splits(int slots, int batch, int64_t max_split) {
    max_split = std::max<int64_t>(1, max_split);
    const int S0 = static_cast<int>(std::min<int64_t>(max_split, std::max(1, slots / batch)));
    int S = S0;
    double best = 0.0;
    for (int cand = S0; cand <= std::min<int64_t>(max_split, 4 * S0 + 4); ++cand) {
        const int64_t n = static_cast<int64_t>(cand) * batch;
        const double eff = static_cast<double>(n) / (static_cast<double>((n + slots - 1) / slots) * slots);
        if (eff > best + 0.02) {
            best = eff;
            S = cand;
        }
        if (best >= 0.95) break;
    }
    return S;
}

const DecodePlan& cached_plan(const rkv_layer_desc& d, int64_t max_seq_len) {
    static std::mutex mu;
    using Key = std::tuple<std::string, int64_t, int, int>;
    static std::map<Key, DecodePlan> plans;
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    Key key{std::string(reinterpret_cast<const char*>(&d), sizeof(d)), max_seq_len, current_device(),
            options().epoch.load()};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = plans.find(key);
        if (it != plans.end()) return it->second;
    }
    DecodePlan pl = plan_decode(d, max_seq_len);  // outside the lock: occupancy queries
    std::lock_guard<std::mutex> lk(mu);
    if (plans.size() > 4096) plans.clear();  // bounded (a serving process sees few shapes)
    return plans.emplace(key, pl).first->second;
}

}  // namespace rkv

extern "C" rkv_status rkv_set_debug_option(const char* name, int64_t value) {
    rkv::Options& o = rkv::options();
    if (!name) return RKV_ERR_INVALID_ARGUMENT;
    const std::string n(name);
    std::atomic<int>* slot = nullptr;
    if (n == "decode_kernel_simt") slot = &o.force_simt;
    else if (n == "gqa_warps_per_group") slot = &o.gqa_pw;
    else if (n == "gqa_tmem") slot = &o.gqa_tmem;
    else if (n == "decode_splits") slot = &o.dec_splits;
    else if (n == "prefill_pair") slot = &o.prefill_pair;
    else if (n == "simt_pairs") slot = &o.simt_p;
    else if (n == "simt_stages") slot = &o.simt_stages;
    else if (n == "quant_stages") slot = &o.quant_stages;
    else if (n == "quant_vsplit") slot = &o.quant_vsplit;
    else if (n == "quant_vcfg") slot = &o.quant_vcfg;
    else if (n == "decode_pdl") slot = &o.decode_pdl;
    else if (n == "generic_tile") slot = &o.generic_tile;
    else if (n == "gqa_head_sets") slot = &o.gqa_sets;
    if (!slot) return RKV_ERR_INVALID_ARGUMENT;
    slot->store(static_cast<int>(value));
    o.epoch.fetch_add(1);
    return RKV_OK;
}

extern "C" rkv_status rkv_decode_plan_info(const rkv_layer_desc* desc, int64_t max_seq_len, int64_t out[10]) {
    if (!desc || !out) return RKV_ERR_INVALID_ARGUMENT;
    if (rkv_layer_validate(desc) != RKV_OK) return RKV_ERR_INVALID_ARGUMENT;
    const rkv::DecodePlan& pl = rkv::cached_plan(*desc, max_seq_len);
    const int64_t v[10] = {pl.kind, pl.N, pl.NT, pl.S, pl.NP, pl.chunk, pl.TT, pl.per_sm,
                           static_cast<int64_t>(pl.smem), pl.stages};
    for (int i = 0; i < 10; ++i) out[i] = v[i];
    return RKV_OK;
}
