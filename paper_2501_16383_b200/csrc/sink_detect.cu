// sink_detect.cu -- massive-activation sink detection on the device
// (detect_massive_activations, proj/src/sink.cpp:14-45), so the sink flags
// fed to rkv_quantize_kv never leave the GPU.
//
//   median    = element n/2 of the ascending sort of |x| over the whole
//               [b][s][hidden] tensor (sink.cpp:25-28)
//   threshold = rel_threshold * median                      (sink.cpp:30)
//   token t is a sink  <=>  t == 0  or  some |x[bi][t][c]| > threshold and
//                                        > abs_floor        (sink.cpp:32-42)
//
// The median is found exactly by a 3-pass radix select on the bits of |x|
// (non-negative floats order like their bit patterns): each pass histograms
// one digit of the elements whose higher digits match the prefix found so
// far (HBM-bound streaming pass, shared-memory histogram, 2048 bins), and a
// one-block kernel picks the digit holding the rank.  The float comparison
// against the double threshold is exact in fp32: for float v,
// v > thr  <=>  v > RD_f32(thr).
#include <cstdint>

#include "rkv_internal.h"

namespace rkv {

namespace {

constexpr int kBins = 2048;

struct SelectState {
    uint32_t prefix;   // digits fixed so far (bits above the current pass)
    uint32_t pad;
    uint64_t rank;     // rank still to find among elements matching prefix
    uint32_t hist[kBins];
};

// pass p: digit = bits [lo, lo + width) of |x|; elements must match
// prefix on bits [lo + width, 31)
__global__ void __launch_bounds__(512) radix_hist_kernel(const float* __restrict__ x, int64_t n,
                                                         SelectState* st, int lo, int width) {
    __shared__ uint32_t h[kBins];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int hi = lo + width;
    const uint32_t prefix = st->prefix;
    const uint32_t mask = (1u << width) - 1u;
    const int64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    auto add = [&](float v) {
        const uint32_t u = __float_as_uint(v) & 0x7fffffffu;
        if (hi >= 31 || (u >> hi) == prefix) atomicAdd(&h[(u >> lo) & mask], 1u);
    };
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 v = __ldg(x4 + i);
        add(v.x);
        add(v.y);
        add(v.z);
        add(v.w);
    }
    for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        add(__ldg(x + i));
    __syncthreads();
    for (int i = threadIdx.x; i <= static_cast<int>(mask); i += blockDim.x)
        if (h[i]) atomicAdd(&st->hist[i], h[i]);
}

// one block: find the digit whose cumulative count passes the rank, append
// it to the prefix, clear the histogram for the next pass
__global__ void __launch_bounds__(1024) radix_select_kernel(SelectState* st, int width) {
    __shared__ uint32_t cnt[kBins];
    __shared__ uint64_t base[1024 + 1];
    const int nb = 1 << width;
    const uint64_t r = st->rank;  // read by every thread before the single writer below
    const uint32_t prefix = st->prefix;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) cnt[i] = st->hist[i];
    __syncthreads();
    // per-thread chunk sums, then an exclusive scan over threads (blockDim = 1024)
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per;
    uint64_t s = 0;
    for (int i = b0; i < b0 + per && i < nb; ++i) s += cnt[i];
    base[threadIdx.x + 1] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        base[0] = 0;
        for (int i = 1; i <= static_cast<int>(blockDim.x); ++i) base[i] += base[i - 1];
    }
    __syncthreads();
    if (base[threadIdx.x] <= r && r < base[threadIdx.x + 1]) {  // the rank falls in this thread's chunk
        uint64_t acc = base[threadIdx.x];
        for (int i = b0; i < b0 + per && i < nb; ++i) {
            if (r < acc + cnt[i]) {
                st->prefix = (prefix << width) | static_cast<uint32_t>(i);
                st->rank = r - acc;
                break;
            }
            acc += cnt[i];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) st->hist[i] = 0;
}

// selection state and flags initialised on the stream (graph-capturable)
__global__ void sink_init_kernel(SelectState* st, uint64_t rank, uint8_t* flags, int64_t s) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < s) flags[t] = t == 0 ? 1 : 0;
    if (t < kBins) st->hist[t] = 0;
    if (t == 0) {
        st->prefix = 0;
        st->rank = rank;
    }
}

// grid-stride over [b][s][hidden] rows; a row with any |x| above the
// threshold flags its token
__global__ void __launch_bounds__(256) sink_flags_kernel(const float* __restrict__ x, int64_t b, int64_t s,
                                                         int64_t hidden, const SelectState* st, double rel,
                                                         double abs_floor, uint8_t* flags, float* median_out) {
    const float median = __uint_as_float(st->prefix);
    const double thr = rel * static_cast<double>(median);
    const float t_f = fmaxf(__double2float_rd(thr), __double2float_rd(abs_floor));
    if (median_out && blockIdx.x == 0 && threadIdx.x == 0) *median_out = median;
    const int64_t rows = b * s;
    const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * warps + threadIdx.x / 32; row < rows;
         row += static_cast<int64_t>(gridDim.x) * warps) {
        const float* r = x + row * hidden;
        bool hit = false;
        for (int64_t c = lane; c < hidden; c += 32) hit |= fabsf(__ldg(r + c)) > t_f;
        if (__any_sync(0xffffffffu, hit) && lane == 0) flags[row % s] = 1;
    }
}

}  // namespace

size_t detect_sinks_workspace_bytes() { return sizeof(SelectState); }

cudaError_t launch_detect_sinks(const float* x, int64_t b, int64_t s, int64_t hidden, double rel, double abs_floor,
                                uint8_t* flags, float* median_out, void* ws, cudaStream_t stream) {
    SelectState* st = static_cast<SelectState*>(ws);
    const int64_t n = b * s * hidden;
    const int64_t m = s > kBins ? s : kBins;
    sink_init_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, stream>>>(st, static_cast<uint64_t>(n / 2),
                                                                                 flags, s);
    const int grid = num_sms() * 4;
    // digits of the 31-bit magnitude: bits [21,31), [10,21), [0,10)
    const int lo[3] = {21, 10, 0}, width[3] = {10, 11, 10};
    for (int p = 0; p < 3; ++p) {
        radix_hist_kernel<<<grid, 512, 0, stream>>>(x, n, st, lo[p], width[p]);
        radix_select_kernel<<<1, 1024, 0, stream>>>(st, width[p]);
    }
    sink_flags_kernel<<<grid, 256, 0, stream>>>(x, b, s, hidden, st, rel, abs_floor, flags, median_out);
    return cudaGetLastError();
}

}  // namespace rkv
