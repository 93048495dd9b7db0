// generic.cu -- quantize-append and decode attention for every layer shape the
// reference accepts that the specialised kernels do not tile: any rotation
// size n = G*128 <= 8192 with G | H (RotationPlan::make,
// proj/src/hadamard.cpp:18-33) and any q/KV head ratio, e.g. G = 4 with 4 q
// heads per KV head (GQA at the paper's default rotation), G = 8 .. 64, or
// G = 1 at C = 8192.
//
// Both kernels keep a whole fp32 row in shared memory and run the FWHT stage
// by stage over it (half = 1, 2, ..., n/2 -- the reference's order,
// proj/src/hadamard.cpp:51-60, one CTA barrier per stage), so:
//   * quantize_generic_kernel: codes, scales and zeros are bit-identical to
//     the specialised kernel and to the oracle (same fp32 stage order, same
//     x 1/sqrt(n) rounding, same exact thresholds: group_params);
//   * decode_generic_kernel: the dequantised row s*(c - z) stays fp32 (no
//     fp16 operand rounding at all), is un-reordered (slot j -> perm[j]),
//     inverse-rotated, RoPE'd per head and dotted with every q head of its KV
//     head; online softmax and P.V in fp32.  It writes the same split
//     partials as the other decode kernels, so the shared combine adds the
//     exact sink rows and V's H_128.
// They trade speed for generality (a CTA walks one token at a time); the
// BASELINE configurations all run on the specialised kernels.
#include <cmath>

#include "rkv_common.cuh"
#include "rkv_internal.h"
#include "rkv_layout.h"

namespace rkv {

namespace {

constexpr int kGenThreads = 256;

// In-place FWHT of every n-channel unit of row[0, C), reference stage order.
__device__ __forceinline__ void fwht_row(float* row, int C, int n) {
    for (int half = 1; half < n; half <<= 1) {
        for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {
            // butterfly i: the i-th pair (lo, lo + half) in unit order
            const int blk = i / half, off = i % half;
            const int lo = blk * 2 * half + off;
            const float a = row[lo], b = row[lo + half];
            row[lo] = __fadd_rn(a, b);
            row[lo + half] = __fsub_rn(a, b);
        }
        __syncthreads();
    }
}

template <int FMT>
__global__ void __launch_bounds__(kGenThreads) quantize_generic_kernel(QuantParams p, int nk, int64_t items) {
    extern __shared__ __align__(16) float grow[];  // [C]
    __shared__ int s_slot;
    const int C = p.C, W = C / 16, MG = C / kQuantGroup;
    const int num_new = static_cast<int>(p.num_new);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const bool isv = it & 1;
        const int64_t bi = it >> 1;  // b * num_new + i
        const int b = static_cast<int>(bi / num_new), i = static_cast<int>(bi % num_new);
        const int64_t pos = p.start_pos[b] + i;
        const uint16_t* src = (isv ? p.v_new : p.k_new) + bi * C;
        if (threadIdx.x == 0) {  // sidecar slot (the specialised kernel's rule)
            int slot = -1;
            if (p.sink_flags && pos >= 0 && pos < p.max_tokens && p.sink_flags[bi]) {
                int before = 0;
                for (int q = 0; q < i; ++q) before += p.sink_flags[static_cast<int64_t>(b) * num_new + q] ? 1 : 0;
                slot = p.cache.sink_count[b] + before;
                if (slot >= p.max_sinks) slot = -1;
            }
            s_slot = slot;
        }
        for (int c = threadIdx.x; c < C; c += blockDim.x) grow[c] = h2f(src[c]);
        __syncthreads();
        const int n = isv ? kHeadDim : nk;
        fwht_row(grow, C, n);
        const float norm = isv ? p.v_norm : p.k_norm;
        for (int c = threadIdx.x; c < C; c += blockDim.x) grow[c] = __fmul_rn(grow[c], norm);
        __syncthreads();
        const int slot = s_slot;
        if (pos >= 0 && pos < p.max_tokens) {
            uint32_t* codes = (isv ? p.cache.v_codes : p.cache.k_codes) + (static_cast<int64_t>(b) * p.max_tokens + pos) * W;
            uint32_t* meta = (isv ? p.cache.v_meta : p.cache.k_meta) + (static_cast<int64_t>(b) * p.max_tokens + pos) * MG;
            // a warp covers 32 packed words = 4 quantization groups; lane = one word
            for (int w0 = warp * 32; w0 < W; w0 += blockDim.x) {
                const int w = w0 + lane;  // W is a multiple of 8, so groups never straddle warps
                const bool live = w < W;
                float x[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int j = (live ? w : 0) * 16 + e;
                    x[e] = grow[isv ? j : p.perm[j]];  // K: slot j <- channel perm[j] (proj/src/reorder.cpp:112-128)
                }
                float mn = x[0], mx = x[0];
#pragma unroll
                for (int e = 1; e < 16; ++e) {
                    mn = fminf(mn, x[e]);
                    mx = fmaxf(mx, x[e]);
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                const GroupQuant gq = group_params<FMT>(mn, mx);
                uint32_t word = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const uint32_t c = (x[e] >= gq.t1) + (x[e] >= gq.t2) + (x[e] >= gq.t3);
                    word |= c << (2 * e);
                }
                if (live) {
                    codes[w] = slot >= 0 ? 0u : word;
                    if ((w & 7) == 0) meta[w >> 3] = slot >= 0 ? 0u : gq.meta;
                }
            }
        }
        if (slot >= 0) {  // raw fp16 row into the sidecar
            uint16_t* side = (isv ? p.cache.sink_v : p.cache.sink_k) + (static_cast<int64_t>(b) * p.max_sinks + slot) * C;
            for (int c = threadIdx.x; c < C; c += blockDim.x) side[c] = src[c];
            if (threadIdx.x == 0 && !isv) p.cache.sink_pos[b * p.max_sinks + slot] = static_cast<int32_t>(pos);
        }
        if (threadIdx.x == 0 && !isv && pos >= 0 && pos < p.max_tokens) {
            uint32_t* mw = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32) + (pos >> 5);
            const uint32_t bit = 1u << (pos & 31);
            if (slot >= 0) atomicOr(mw, bit);
            else atomicAnd(mw, ~bit);
        }
        __syncthreads();
    }
}

// One split of one sequence per CTA, one token at a time.
__global__ void __launch_bounds__(kGenThreads) decode_generic_kernel(DecodeParams p, int n, int rep) {
    extern __shared__ __align__(16) float dsm[];
    pdl_trigger();
    const int C = p.C, W = C / 16, MG = C / kQuantGroup, Hq = p.Hq;
    float* krow = dsm;                     // [C]
    float* qr = krow + C;                  // [Hq][128] RoPE'd query x qscale x k_norm
    float* acc = qr + Hq * kHeadDim;       // [Hq][128] P.V (rotated V frame)
    float* ml = acc + Hq * kHeadDim;       // [Hq][2] running (max, sum), log2 domain
    const uint32_t* slot_ch = p.plan + kPlanHeader + W;  // generic plan: channel of slot 16 w + e at [(e/4) W + w][e%4]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    const int64_t tb = p.tok_begin ? p.tok_begin[b] : 0, te = p.tok_end ? (p.tok_end[b] < T ? p.tok_end[b] : T) : T;
    const int64_t t_begin = tb + static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = t_begin + p.chunk < te ? t_begin + p.chunk : te;
    const bool bad_plan = !plan_matches(p.plan, kDecodeGeneric, n, C);
    if (t_begin >= t_end || bad_plan) {
        const float fill = bad_plan ? __int_as_float(0x7fc00000) : 0.0f;
        for (int h = threadIdx.x; h < Hq; h += blockDim.x) {
            const int64_t row = (static_cast<int64_t>(b) * p.NP + split) * Hq + h;
            p.ws_ml[row * 2] = bad_plan ? fill : -INFINITY;
            p.ws_ml[row * 2 + 1] = fill;
            for (int k = 0; k < kHeadDim; ++k) p.ws_o[row * kHeadDim + k] = fill;
        }
        return;
    }
    // query: RoPE at T-1 (proj/src/pipeline.cpp:144-152), x log2(e)/sqrt(d) x 1/sqrt(n)
    const float qs = p.qscale * p.k_norm;
    for (int i = threadIdx.x; i < Hq * 64; i += blockDim.x) {
        const int h = i / 64, f = i % 64;
        const float a = h2f(p.q[(static_cast<int64_t>(b) * Hq + h) * kHeadDim + f]);
        const float bb = h2f(p.q[(static_cast<int64_t>(b) * Hq + h) * kHeadDim + f + 64]);
        const float2 cs = rope_at(p.rope, T - 1, f);
        qr[h * kHeadDim + f] = (a * cs.x - bb * cs.y) * qs;
        qr[h * kHeadDim + f + 64] = (a * cs.y + bb * cs.x) * qs;
    }
    for (int i = threadIdx.x; i < Hq * kHeadDim; i += blockDim.x) acc[i] = 0.f;
    for (int h = threadIdx.x; h < Hq; h += blockDim.x) {
        ml[2 * h] = -INFINITY;
        ml[2 * h + 1] = 0.f;
    }
    __syncthreads();
    const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;
    for (int64_t t = t_begin; t < t_end; ++t) {
        if ((smask[t >> 5] >> (t & 31)) & 1u) continue;  // sinks: exact fp16 rows, added by the combine
        // dequantise (fp32, exact s*(c - z)) and un-reorder: slot j -> channel perm[j]
        const uint32_t* kc = p.cache.k_codes + (row0 + t) * W;
        const uint32_t* km = p.cache.k_meta + (row0 + t) * MG;
        for (int w = threadIdx.x; w < W; w += blockDim.x) {
            const uint32_t word = kc[w], m = km[w >> 3];
            const float s = h2f(static_cast<uint16_t>(m & 0xffffu)), z = h2f(static_cast<uint16_t>(m >> 16));
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float c = static_cast<float>((word >> (2 * e)) & 3u);
                krow[slot_ch[(static_cast<size_t>(e / 4) * W + w) * 4 + e % 4]] = s * (c - z);
            }
        }
        __syncthreads();
        fwht_row(krow, C, n);  // inverse rotation (H is its own inverse up to 1/n; 1/sqrt(n) is in q)
        // logits: warp per q head; RoPE the key pair (f, f + 64) at position t
        for (int h0 = warp; h0 < Hq; h0 += 8 * nwarps) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int h = h0 + r * nwarps;
                if (h >= Hq) continue;
                const int kv = h / rep;
                float part = 0.f;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int f = lane + 32 * k;
                    const float ka = krow[kv * kHeadDim + f], kb = krow[kv * kHeadDim + f + 64];
                    const float2 cs = rope_at(p.rope, t, f);
                    part += qr[h * kHeadDim + f] * (ka * cs.x - kb * cs.y) +
                            qr[h * kHeadDim + f + 64] * (ka * cs.y + kb * cs.x);
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                // online softmax (log2 domain); every lane holds the same values
                const float m_old = ml[2 * h], m_new = fmaxf(m_old, part);
                const float alpha = exp2f(m_old - m_new), pr = exp2f(part - m_new);
                __syncwarp();
                if (lane == 0) {
                    ml[2 * h] = m_new;
                    ml[2 * h + 1] = ml[2 * h + 1] * alpha + pr;
                }
                // V of the KV head, rotated frame: lane owns channels 4 lane .. 4 lane + 3
                const uint32_t vword = p.cache.v_codes[(row0 + t) * W + kv * 8 + (lane >> 2)];
                const uint32_t vm = p.cache.v_meta[(row0 + t) * MG + kv];
                const float vs = h2f(static_cast<uint16_t>(vm & 0xffffu)), vz = h2f(static_cast<uint16_t>(vm >> 16));
                float4* a4 = reinterpret_cast<float4*>(acc + h * kHeadDim) + lane;
                float4 av = *a4;
                const int e0 = 4 * (lane & 3);
                const float v0 = vs * (static_cast<float>((vword >> (2 * e0)) & 3u) - vz);
                const float v1 = vs * (static_cast<float>((vword >> (2 * e0 + 2)) & 3u) - vz);
                const float v2 = vs * (static_cast<float>((vword >> (2 * e0 + 4)) & 3u) - vz);
                const float v3 = vs * (static_cast<float>((vword >> (2 * e0 + 6)) & 3u) - vz);
                av = make_float4(av.x * alpha + pr * v0, av.y * alpha + pr * v1, av.z * alpha + pr * v2,
                                 av.w * alpha + pr * v3);
                *a4 = av;
            }
        }
        __syncthreads();  // krow and the per-head state are rewritten by the next token
    }
    for (int h = warp; h < Hq; h += nwarps) {
        const int64_t row = (static_cast<int64_t>(b) * p.NP + split) * Hq + h;
        if (lane == 0) {
            p.ws_ml[row * 2] = ml[2 * h];
            p.ws_ml[row * 2 + 1] = ml[2 * h + 1];
        }
        reinterpret_cast<float4*>(p.ws_o + row * kHeadDim)[lane] = reinterpret_cast<const float4*>(acc + h * kHeadDim)[lane];
    }
}

// rotate_rows (proj/src/hadamard.cpp:75-84) for rotation sizes beyond the
// register-layout kernel: one CTA per row, the row in shared memory.
__global__ void __launch_bounds__(kGenThreads) rotate_keys_generic_kernel(const uint16_t* __restrict__ k, int64_t rows,
                                                                       int C, int n, float norm, float* out) {
    extern __shared__ __align__(16) float rrow[];
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        for (int c = threadIdx.x; c < C; c += blockDim.x) rrow[c] = h2f(k[r * C + c]);
        __syncthreads();
        fwht_row(rrow, C, n);
        for (int c = threadIdx.x; c < C; c += blockDim.x) out[r * C + c] = __fmul_rn(rrow[c], norm);
        __syncthreads();
    }
}

// LayerKVCache::key_row / value_row / keys / values (proj/src/kv_cache.cpp:
// 57-85): tokens [t0, t0 + n) of sequence b, K and V, as fp32 rows.
//   frame 0 (RKV_FRAME_STORED): what the reference returns -- the stored
//     fused-frame row s*(c - z) (K reordered + rotated, V rotated), and for a
//     sink the fused frame of its raw fp16 row (rotate [+ reorder] in fp32,
//     the reference's sidecar content);
//   frame 1 (RKV_FRAME_RAW): back in the model's frame -- dequantised, the
//     reorder and the rotation undone (K: inverse reorder, then FWHT over G
//     heads; V: FWHT per head), sinks exact.
// One CTA per row; the row is staged in shared memory.
__global__ void __launch_bounds__(kGenThreads) cache_read_kernel(rkv_cache cache, const int32_t* __restrict__ perm,
                                                              int64_t max_tokens, int max_sinks, int C, int nk,
                                                              float k_norm, float v_norm, int b, int64_t t0, int64_t n,
                                                              int frame, float* __restrict__ k_out,
                                                              float* __restrict__ v_out) {
    extern __shared__ __align__(16) float crow[];  // [C]
    float* a = crow;
    const int W = C / 16, MG = C / kQuantGroup;
    const uint32_t* smask = cache.sink_mask + static_cast<int64_t>(b) * ((max_tokens + 31) / 32);
    for (int64_t r = blockIdx.x; r < 2 * n; r += gridDim.x) {
        const bool isv = r >= n;
        const int64_t t = t0 + (isv ? r - n : r);
        const int nn = isv ? kHeadDim : nk;
        const float norm = isv ? v_norm : k_norm;
        float* dst = (isv ? v_out : k_out) + (isv ? r - n : r) * C;
        const bool sink = (smask[t >> 5] >> (t & 31)) & 1u;
        if (sink) {
            int slot = 0;
            while (slot < max_sinks && cache.sink_pos[b * max_sinks + slot] != t) ++slot;
            const uint16_t* src = (isv ? cache.sink_v : cache.sink_k) + (static_cast<int64_t>(b) * max_sinks + slot) * C;
            if (frame == 1) {
                for (int c = threadIdx.x; c < C; c += blockDim.x) dst[c] = h2f(src[c]);
                continue;
            }
            for (int c = threadIdx.x; c < C; c += blockDim.x) a[c] = h2f(src[c]);
            __syncthreads();
            fwht_row(a, C, nn);
            for (int c = threadIdx.x; c < C; c += blockDim.x) {
                const float x = __fmul_rn(a[isv ? c : perm[c]], norm);  // K: slot c <- channel perm[c]
                dst[c] = x;
            }
            __syncthreads();
            continue;
        }
        const uint32_t* codes = (isv ? cache.v_codes : cache.k_codes) + (static_cast<int64_t>(b) * max_tokens + t) * W;
        const uint32_t* meta = (isv ? cache.v_meta : cache.k_meta) + (static_cast<int64_t>(b) * max_tokens + t) * MG;
        for (int j = threadIdx.x; j < C; j += blockDim.x) {  // dequantize_group (proj/src/quant.cpp:99-107)
            const uint32_t m = meta[j >> 7];
            const float sc = h2f(static_cast<uint16_t>(m & 0xffffu)), z = h2f(static_cast<uint16_t>(m >> 16));
            const float x = sc * (static_cast<float>((codes[j >> 4] >> (2 * (j & 15))) & 3u) - z);
            if (frame == 0) dst[j] = x;
            else a[isv ? j : perm[j]] = x;  // inverse reorder: channel perm[j] <- slot j
        }
        if (frame == 0) continue;
        __syncthreads();
        fwht_row(a, C, nn);
        for (int c = threadIdx.x; c < C; c += blockDim.x) dst[c] = __fmul_rn(a[c], norm);
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_cache_read(const rkv_layer_desc& d, const rkv_cache& cache, const int32_t* perm, int b, int64_t t0,
                              int64_t n, int frame, float* k_out, float* v_out, cudaStream_t s) {
    const int C = d.num_kv_heads * d.head_dim, nk = d.heads_per_group * d.head_dim;
    const size_t smem = static_cast<size_t>(C) * sizeof(float);
    cudaError_t e = ensure_smem_k(cache_read_kernel, smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(2 * n, static_cast<int64_t>(num_sms()) * 8);
    cache_read_kernel<<<static_cast<unsigned>(grid), kGenThreads, smem, s>>>(
        cache, perm, d.max_tokens, d.max_sinks, C, nk, 1.0f / sqrtf(static_cast<float>(nk)),
        1.0f / sqrtf(static_cast<float>(d.head_dim)), b, t0, n, frame, k_out, v_out);
    return cudaGetLastError();
}

cudaError_t launch_rotate_keys_generic(const rkv_layer_desc& d, const uint16_t* k, int64_t rows, float* out,
                                       cudaStream_t s) {
    const int C = d.num_kv_heads * d.head_dim, n = d.heads_per_group * d.head_dim;
    const float norm = 1.0f / sqrtf(static_cast<float>(n));
    const size_t smem = static_cast<size_t>(C) * sizeof(float);
    cudaError_t e = ensure_smem_k(rotate_keys_generic_kernel, smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(rows, static_cast<int64_t>(num_sms()) * 8);
    rotate_keys_generic_kernel<<<static_cast<unsigned>(grid), kGenThreads, smem, s>>>(k, rows, C, n, norm, out);
    return cudaGetLastError();
}

bool generic_quantize_needed(const rkv_layer_desc& d) {
    const int n = d.heads_per_group * d.head_dim;
    return n != 128 && n != 256 && n != 512;
}

cudaError_t launch_quantize_generic(const rkv_layer_desc& d, const QuantParams& p, cudaStream_t s) {
    const int n = d.heads_per_group * d.head_dim;
    const size_t smem = static_cast<size_t>(p.C) * sizeof(float);
    const int64_t items = 2 * static_cast<int64_t>(d.batch) * p.num_new;
    const int64_t grid = std::min<int64_t>(items, static_cast<int64_t>(num_sms()) * 8);
    cudaError_t e;
    if (p.scale_format == RKV_SCALE_E4M3_CEIL) {
        if ((e = ensure_smem_k(quantize_generic_kernel<RKV_SCALE_E4M3_CEIL>, smem)) != cudaSuccess) return e;
        quantize_generic_kernel<RKV_SCALE_E4M3_CEIL><<<static_cast<unsigned>(grid), kGenThreads, smem, s>>>(p, n, items);
    } else {
        if ((e = ensure_smem_k(quantize_generic_kernel<RKV_SCALE_FP16_CEIL>, smem)) != cudaSuccess) return e;
        quantize_generic_kernel<RKV_SCALE_FP16_CEIL><<<static_cast<unsigned>(grid), kGenThreads, smem, s>>>(p, n, items);
    }
    return cudaGetLastError();
}

size_t generic_decode_smem(const rkv_layer_desc& d) {
    const size_t C = static_cast<size_t>(d.num_kv_heads) * d.head_dim, Hq = static_cast<size_t>(d.num_q_heads);
    return (C + 2 * Hq * kHeadDim + 2 * Hq) * sizeof(float);
}

DecodePlan plan_decode_generic(const rkv_layer_desc& d, int64_t max_seq_len) {
    DecodePlan pl{};
    pl.kind = kDecodeGeneric;
    pl.N = d.heads_per_group * d.head_dim;
    pl.REP = d.num_q_heads / d.num_kv_heads;
    pl.P = pl.PP = 1;
    pl.TT = 1;
    pl.NT = kGenThreads;
    pl.stages = 1;
    pl.per_sm = 1;
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    pl.smem = generic_decode_smem(d);
    const int S0 = std::max(1, 2 * num_sms() / std::max(1, d.batch));
    const int S = static_cast<int>(std::min<int64_t>(S0, std::max<int64_t>(1, (max_seq_len + 15) / 16)));
    pl.chunk = static_cast<int>((max_seq_len + S - 1) / S);
    pl.S = static_cast<int>((max_seq_len + pl.chunk - 1) / pl.chunk);
    pl.NP = pl.S;
    pl.ok = pl.smem <= 227 * 1024;
    return pl;
}

cudaError_t launch_decode_generic(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p,
                                  cudaStream_t s) {
    cudaError_t e = ensure_smem_k(decode_generic_kernel, plan.smem);
    if (e != cudaSuccess) return e;
    decode_generic_kernel<<<dim3(plan.S, d.batch), kGenThreads, plan.smem, s>>>(p, plan.N, plan.REP);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_decode_combine(p, d.batch, s);
}

}  // namespace rkv
