// quantize_kv.cu -- fused quantize-append for sm_100a.
//
// Grid (X, B, 2): z selects K or V; a CTA loops over token pairs of one
// sequence (every register holds a float2 = the same channel of the pair's
// two tokens, so each FWHT butterfly is one FADD2):
//   1. K rows: grouped-head FWHT over G KV heads (n = G*128) in registers
//      (layout A -> smem transpose -> layout B, rkv_common.cuh), x 1/sqrt(n).
//      V rows: per-head FWHT (n = 128).  Results land in shared memory.
//   2. Each thread owns one packed word (16 slots).  K slots gather their
//      channel through the calibrated permutation (slot j <- channel perm[j],
//      proj/src/reorder.cpp:112-128); 8 consecutive lanes form one 128-slot
//      quant group: min/max by shuffles, the group leader derives the stored
//      scale / zero in double exactly as proj/src/quant.cpp:53-97 does and
//      turns the reference's round-half-away division into three float
//      thresholds, so code = (x>=T1)+(x>=T2)+(x>=T3) is bit-identical.
//   3. Sink tokens (proj/src/kv_cache.cpp:8-22 `sink`) keep their raw fp16
//      rows in the sidecar; their packed words/meta are zero.
// Reference chain restated: rotate_rows -> apply_reorder -> quantize_token ->
// LayerKVCache::append (proj/src/pipeline.cpp:171-176, :317-324).
#include <cstdio>

#include "rkv_common.cuh"
#include "rkv_internal.h"

namespace rkv {

namespace {

// Shared-memory swizzle of an N-point unit region (see rkv_common.cuh):
// XOR the float4-chunk index with the owning lane (conflict-free layout-A
// float4 traffic) and the unit index with the lane-group slot inside a warp
// (conflict-free layout-B scalar traffic).
template <int N, int L>
__device__ __forceinline__ int swz(int c) {
    constexpr int R = N / L;
    constexpr int LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    return c ^ (((c >> LR) & (R / 4 - 1)) << 2) ^ (((c >> LN) & (32 / L - 1)) << LL);
}

// FWHT of unit u (N contiguous channels) of two fp16 rows into smem rows
// dst0/dst1 (natural order, swizzled).  Lanes of the unit: lam = 0..L-1.
template <int N, int L>
__device__ __forceinline__ void fwht_unit(const uint16_t* __restrict__ src0, const uint16_t* __restrict__ src1,
                                          float* dst0, float* dst1, int u, int lam, bool active, float norm) {
    constexpr int R = N / L;
    constexpr int LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    float2 x[R];
    if (active) {
        const uint4* a = reinterpret_cast<const uint4*>(src0 + u * N + lam * R);
        const uint4* b = reinterpret_cast<const uint4*>(src1 + u * N + lam * R);
#pragma unroll
        for (int q = 0; q < R / 8; ++q) {
            uint4 va = __ldg(a + q), vb = __ldg(b + q);
            const uint16_t* ha = reinterpret_cast<const uint16_t*>(&va);
            const uint16_t* hb = reinterpret_cast<const uint16_t*>(&vb);
#pragma unroll
            for (int e = 0; e < 8; ++e) x[8 * q + e] = make_float2(h2f(ha[e]), h2f(hb[e]));
        }
        bfly_range<R, 0, LR>(x);  // index bits 0 .. LR-1
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
            int p = swz<N, L>(u * N + lam * R + 4 * q);
            *reinterpret_cast<float4*>(dst0 + p) = make_float4(x[4 * q].x, x[4 * q + 1].x, x[4 * q + 2].x, x[4 * q + 3].x);
            *reinterpret_cast<float4*>(dst1 + p) = make_float4(x[4 * q].y, x[4 * q + 1].y, x[4 * q + 2].y, x[4 * q + 3].y);
        }
    }
    __syncwarp();
    if (active) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
            int p = swz<N, L>(u * N + lam + L * j);
            x[j] = make_float2(dst0[p], dst1[p]);
        }
        bfly_range<R, LR - LL, LN - LL>(x);  // index bits LR .. LN-1
        const float2 nn = make_float2(norm, norm);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            int p = swz<N, L>(u * N + lam + L * j);
            float2 y = mul2(x[j], nn);
            dst0[p] = y.x;
            dst1[p] = y.y;
        }
    }
    __syncwarp();
}

struct GroupQuant {
    float t1, t2, t3;
    uint32_t meta;
};

// proj/src/quant.cpp:74-94 for bits = 2, evaluated once per group.
__device__ __forceinline__ GroupQuant group_params(float mn, float mx, int scale_format) {
    double range = __dsub_rn(static_cast<double>(mx), static_cast<double>(mn));
    float raw = __double2float_rn(__ddiv_rn(range, 3.0));
    if (raw < 1e-8f) raw = 1e-8f;
    uint16_t sbits;
    float sf;
    if (scale_format == RKV_SCALE_E4M3_CEIL) {
        sf = e4m3_ceil_value(raw);
        sbits = __half_as_ushort(__float2half_rn(sf));  // exact: e4m3 values are fp16 values
    } else {
        sbits = fp16_ceil(raw);
        sf = __half2float(__ushort_as_half(sbits));
    }
    const double s = static_cast<double>(sf);
    double zero = round(__ddiv_rn(-static_cast<double>(mn), s));
    zero = fmin(fmax(zero, 0.0), 3.0);
    GroupQuant g;
    float t[3];
#pragma unroll
    for (int k = 1; k <= 3; ++k) {
        // code >= k  <=>  round_half_away(x/s) >= k - zero  (m = k - zero)
        //            <=>  x >= (m - 0.5) s  for m >= 1,  x > (m - 0.5) s  for m <= 0
        double m = static_cast<double>(k) - zero;
        double tt = __dmul_rn(m - 0.5, s);  // exact: (m-0.5) has 3 bits, s has 11
        float f = __double2float_ru(tt);
        if (m <= 0.0 && static_cast<double>(f) == tt) f = nextafterf(f, INFINITY);
        t[k - 1] = f;
    }
    g.t1 = t[0];
    g.t2 = t[1];
    g.t3 = t[2];
    g.meta = static_cast<uint32_t>(sbits) |
             (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(static_cast<float>(zero)))) << 16);
    return g;
}

// Grid (X, B, 2): z = 0 quantizes K rows, z = 1 V rows; each CTA loops over
// token pairs blockIdx.x, blockIdx.x + X, ... of sequence b, so the slot ->
// channel address table is built once per CTA.
template <int N>
__global__ void __launch_bounds__(256) quantize_kv_kernel(QuantParams p) {
    constexpr int LK = N >= 256 ? 16 : 8;
    extern __shared__ float4 smem4[];
    const int C = p.C, W = C / 16, MG = C / kQuantGroup;
    float* row = reinterpret_cast<float*>(smem4);                // [2][C]
    uint16_t* addr = reinterpret_cast<uint16_t*>(row + 2 * C);   // [C]
    __shared__ int s_slot[2];

    const int b = blockIdx.y;
    const bool isv = blockIdx.z == 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t npairs = (p.num_new + 1) / 2;

    for (int j = tid; j < C; j += blockDim.x)
        addr[j] = static_cast<uint16_t>(isv ? swz<128, 8>(j) : swz<N, LK>(__ldg(p.perm + j)));

    for (int64_t pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
        const int64_t i0 = pi * 2;
        const bool has1 = i0 + 1 < p.num_new;
        // sink bookkeeping: slot = sink_count + #sinks among earlier new tokens of b
        if (tid < 2) {
            int slot = -1;
            const int64_t i = i0 + tid;
            if (p.sink_flags && i < p.num_new && p.sink_flags[b * p.num_new + i]) {
                int before = 0;
                for (int64_t k = 0; k < i; ++k) before += p.sink_flags[b * p.num_new + k] ? 1 : 0;
                slot = p.cache.sink_count[b] + before;
            }
            s_slot[tid] = slot;
        }
        const uint16_t* src0 = (isv ? p.v_new : p.k_new) + (static_cast<int64_t>(b) * p.num_new + i0) * C;
        const uint16_t* src1 = has1 ? src0 + C : src0;
        __syncthreads();  // addr / s_slot ready; previous pair's reads of row done

        if (!isv) {  // K: C/N grouped-head units, LK lanes each
            constexpr int UPW = 32 / LK;
            const int NG = C / N;
            for (int ub = warp * UPW; ub < NG; ub += nwarps * UPW) {
                const int u = ub + lane / LK;
                fwht_unit<N, LK>(src0, src1, row, row + C, u, lane % LK, u < NG, p.k_norm);
            }
        } else {  // V: per-head units (n = 128), 8 lanes each (proj/src/pipeline.cpp:120)
            const int NU = C / 128;
            for (int ub = warp * 4; ub < NU; ub += nwarps * 4) {
                const int u = ub + lane / 8;
                fwht_unit<128, 8>(src0, src1, row, row + C, u, lane % 8, u < NU, p.v_norm);
            }
        }
        __syncthreads();

        // quantize: item = (token, word); 8 lanes = one 128-slot group
        const int items = 2 * W;  // multiple of 32 (C % 256 == 0)
        for (int base = warp * 32; base < items; base += nwarps * 32) {
            const int it = base + lane;
            const int tok = it / W;
            const int w = it - tok * W;
            const float* rw = row + tok * C;
            const uint16_t* ad = addr + 16 * w;
            float x[16];
            {
                const uint4 a0 = lds128(ad), a1 = lds128(ad + 8);
                const uint16_t* h0 = reinterpret_cast<const uint16_t*>(&a0);
                const uint16_t* h1 = reinterpret_cast<const uint16_t*>(&a1);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    x[e] = rw[h0[e]];
                    x[8 + e] = rw[h1[e]];
                }
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
            GroupQuant gq{};
            if ((lane & 7) == 0) gq = group_params(mn, mx, p.scale_format);
            const int leader = lane & ~7;
            gq.t1 = __shfl_sync(0xffffffffu, gq.t1, leader);
            gq.t2 = __shfl_sync(0xffffffffu, gq.t2, leader);
            gq.t3 = __shfl_sync(0xffffffffu, gq.t3, leader);
            uint32_t word = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const uint32_t c = (x[e] >= gq.t1) + (x[e] >= gq.t2) + (x[e] >= gq.t3);
                word |= c << (2 * e);
            }
            if (tok == 0 || has1) {
                const int64_t pos = p.start_pos[b] + i0 + tok;
                const bool sink = s_slot[tok] >= 0;
                const int64_t rowi = static_cast<int64_t>(b) * p.max_tokens + pos;
                uint32_t* codes = isv ? p.cache.v_codes : p.cache.k_codes;
                uint32_t* meta = isv ? p.cache.v_meta : p.cache.k_meta;
                codes[rowi * W + w] = sink ? 0u : word;
                if ((lane & 7) == 0) meta[rowi * MG + w / 8] = sink ? 0u : gq.meta;
            }
        }

        // sink rows: raw fp16 rows into the sidecar (exact, proj/tests/test_kv_cache.cpp:22-45)
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {
            const int slot = s_slot[tok];
            if (slot < 0 || slot >= p.max_sinks) continue;
            const uint4* srcr = reinterpret_cast<const uint4*>(tok ? src1 : src0);
            uint16_t* side = isv ? p.cache.sink_v : p.cache.sink_k;
            uint4* dst = reinterpret_cast<uint4*>(side + (static_cast<int64_t>(b) * p.max_sinks + slot) * C);
            for (int j = tid; j < C / 8; j += blockDim.x) dst[j] = __ldg(srcr + j);
            if (tid == 0 && !isv)
                p.cache.sink_pos[b * p.max_sinks + slot] = static_cast<int32_t>(p.start_pos[b] + i0 + tok);
        }
        __syncthreads();  // s_slot and row are rewritten by the next pair
    }
}

// Sink counts and per-token sink bits for the appended tokens.
__global__ void quantize_finalize_kernel(QuantParams p) {
    const int b = blockIdx.x;
    __shared__ int s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int local = 0;
    for (int64_t i = threadIdx.x; i < p.num_new; i += blockDim.x) {
        const bool sink = p.sink_flags && p.sink_flags[b * p.num_new + i];
        const int64_t pos = p.start_pos[b] + i;
        if (pos < 0 || pos >= p.max_tokens) continue;
        const int64_t words = (p.max_tokens + 31) / 32;
        uint32_t* mw = p.cache.sink_mask + b * words + (pos >> 5);
        const uint32_t bit = 1u << (pos & 31);
        if (sink) {
            atomicOr(mw, bit);
            ++local;
        } else {
            atomicAnd(mw, ~bit);
        }
    }
    if (local) atomicAdd(&s_count, local);
    __syncthreads();
    if (threadIdx.x == 0 && s_count) p.cache.sink_count[b] += s_count;
}

template <int N>
cudaError_t launch_quantize_n(const QuantParams& p, int B, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(p.C) * (2 * sizeof(float) + sizeof(uint16_t));
    cudaError_t e = cudaFuncSetAttribute(quantize_kv_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, quantize_kv_kernel<N>, 256, smem) != cudaSuccess) {
        cudaGetLastError();
        per_sm = 1;
    }
    const int64_t npairs = (p.num_new + 1) / 2;
    // enough CTAs for ~4 waves; each loops over token pairs (amortises the address table)
    int64_t x = (static_cast<int64_t>(num_sms()) * (per_sm > 0 ? per_sm : 1) * 4 + 2 * B - 1) / (2 * B);
    if (x > npairs) x = npairs;
    if (x < 1) x = 1;
    dim3 grid(static_cast<unsigned>(x), static_cast<unsigned>(B), 2);
    quantize_kv_kernel<N><<<grid, 256, smem, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    quantize_finalize_kernel<<<B, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const rkv_layer_desc& d, const QuantParams& p, cudaStream_t s) {
    const int n = d.heads_per_group * d.head_dim;
    switch (n) {
        case 128: return launch_quantize_n<128>(p, d.batch, s);
        case 256: return launch_quantize_n<256>(p, d.batch, s);
        case 512: return launch_quantize_n<512>(p, d.batch, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkv
