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
//   * decode_generic_kernel: the dequantised rows s*(c - z) stay fp32 (no
//     fp16 operand rounding at all), are un-reordered (slot j -> perm[j]),
//     inverse-rotated, RoPE'd per head and dotted with every q head of their
//     KV head; online softmax and P.V in fp32, a tile of up to 32 tokens per
//     CTA step (see the kernel).  It writes the same split partials as the
//     other decode kernels, so the shared combine adds the exact sink rows and
//     V's H_128.
// The quantize kernel trades speed for generality (a CTA walks one row at a
// time); the BASELINE configurations all run on the specialised kernels.
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

// ---- tiled decode -----------------------------------------------------------
// One split of one sequence per CTA, TT tokens (<= 32) per tile.  Every phase
// is spread over the whole CTA and ends in one barrier, so a tile costs
// log2(n)/5 + 3 barriers instead of log2(n) + 2 per token:
//   A  dequantise the tile's K rows (exact fp32 s*(c - z), proj/src/quant.cpp:
//      99-107) and un-reorder them (slot j -> channel perm[j]) into a padded
//      fp32 tile kt[TT][RS] (4 floats of padding per 32 channels);
//   B  inverse FWHT over each n-channel unit (H is its own inverse; 1/sqrt(n)
//      is folded into q), radix-32 passes: a thread holds one 2^nb-element
//      column of a pass in registers;
//   L  logits: thread pair per (KV head, token), frequency halves; RoPE on the
//      key (proj/src/pipeline.cpp:144-152), dot with each q head of the KV
//      head, pair sum by shuffle;
//   S  online softmax (log2 domain) per q head over the tile;
//   V  P.V in the rotated V frame from the packed codes: per (word, head
//      chunk, channel part) sum_t p s c - sum_t p s z in registers, merged
//      into the per-head accumulator once per tile (deterministic: each
//      accumulator element has one owner).
// Writes the same split partials (m, l, o') as the other decode kernels; the
// shared combine adds the exact sink rows and V's H_128.
constexpr int kTileMax = 32;

__host__ __device__ inline int tile_row_stride(int C) { return C + C / 8 + 4; }  // floats; = 4 mod 8
__device__ __forceinline__ int padc(int c) { return c + ((c >> 5) << 2); }
constexpr int kAccStride = 136;  // per-head accumulator row (128 + 8), channel padded by 1 per 16

struct TileSmem {
    size_t kt, q, acc, lg, ml, al, kst, vst, total;
};
__host__ __device__ inline TileSmem tile_smem(int C, int Hq, int TT, bool reg_acc) {
    TileSmem s{};
    const size_t W = C / 16, MG = C / kQuantGroup;
    s.kt = 0;
    s.kst = s.kt + static_cast<size_t>(TT) * tile_row_stride(C) * 4;  // [TT][W] K words + [TT][W] their meta
    s.vst = s.kst + static_cast<size_t>(TT) * W * 8;                   // [TT][W] V words + [TT][MG] meta
    s.q = (s.vst + static_cast<size_t>(TT) * (W + MG) * 4 + 15) & ~size_t(15);
    s.acc = s.q + static_cast<size_t>(Hq) * kHeadDim * 4;
    s.lg = s.acc + (reg_acc ? 0 : static_cast<size_t>(Hq) * kAccStride * 4);
    s.ml = s.lg + static_cast<size_t>(TT) * Hq * 4;
    s.al = s.ml + static_cast<size_t>(Hq) * 8;
    s.total = (s.al + static_cast<size_t>(Hq) * 4 + 15) & ~size_t(15);
    return s;
}

// floor(x / d) for 0 <= x < 2^17 from rcp = 1/d (d <= 2^13): the quotient's
// fractional part is >= 0.5/d from an integer, far above the fp32 error
__device__ __forceinline__ int fdiv(int x, float rcp) { return static_cast<int>((static_cast<float>(x) + 0.5f) * rcp); }
// the two codes in bits [0, 4) of w as exact floats
__device__ __forceinline__ float2 code2_f32(uint32_t w) {
    return add2(make_float2(__uint_as_float(0x4B000000u | (w & 3u)), __uint_as_float(0x4B000000u | ((w >> 2) & 3u))),
                make_float2(-8388608.0f, -8388608.0f));
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One radix-2^NB pass of the FWHT over bits [b0, b0 + NB) of every row
// (b0 == 0: NB == 5, one padded 36-float block per column, float4 accesses;
// b0 >= 5: column stride 2^b0 channels = 9 * 2^(b0-3) padded floats).  With
// ROPE (the pass over bits 5 and 6 .. that runs last) the column then holds,
// for its two frequencies f = c0 and c0 + 32, the (d, d + 64) pairs of every
// head of the unit, and RoPE_t is applied before the store
// (proj/src/pipeline.cpp:144-152).
template <int NB, bool CONTIG, bool ROPE>
__device__ __forceinline__ void fwht_pass(float* kt, int RS, int TT, int C, int b0, const float4* rope, int64_t t0) {
    constexpr int M = 1 << NB, M2 = M / 2;
    const int cols = C >> NB, stride = CONTIG ? 1 : 9 << (b0 - 3);
    const float rcols = 1.0f / static_cast<float>(cols);
    for (int task = threadIdx.x; task < TT * cols; task += blockDim.x) {
        const int t = fdiv(task, rcols), col = task - t * cols;
        const int base = ((col >> b0) << (b0 + NB)) | (col & ((1 << b0) - 1));
        float* row = kt + t * RS + padc(base);
        float2 cs0, cs1;
        if (ROPE) {  // issued ahead of the butterflies
            cs0 = rope_at(rope, t0 + t, base & 31);
            cs1 = rope_at(rope, t0 + t, (base & 31) + 32);
        }
        float2 x[M2];  // x[i] = elements (2i, 2i + 1)
        if (CONTIG) {
            const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
            for (int j = 0; j < M / 4; ++j) {
                const float4 v = r4[j];
                x[2 * j] = make_float2(v.x, v.y);
                x[2 * j + 1] = make_float2(v.z, v.w);
            }
        } else {
#pragma unroll
            for (int i = 0; i < M2; ++i) x[i] = make_float2(row[(2 * i) * stride], row[(2 * i + 1) * stride]);
        }
#pragma unroll
        for (int i = 0; i < M2; ++i) x[i] = make_float2(x[i].x + x[i].y, x[i].x - x[i].y);  // stage h = 1
#pragma unroll
        for (int H = 1; H < M2; H <<= 1)  // stages h = 2H: float2 butterflies
#pragma unroll
            for (int i = 0; i < M2; ++i)
                if (!(i & H)) {
                    const float2 a = x[i], b = x[i + H];
                    x[i] = add2(a, b);
                    x[i + H] = sub2(a, b);
                }
        if (ROPE) {  // element bit 0: frequency f = c0 + 32 (j & 1); bit 1: d vs d + 64; j >> 2: head
            const float2 c2 = make_float2(cs0.x, cs1.x), s2 = make_float2(cs0.y, cs1.y);
            const float2 ns2 = make_float2(-cs0.y, -cs1.y);
#pragma unroll
            for (int hh = 0; hh < M / 4; ++hh) {
                const float2 a = x[2 * hh], bq = x[2 * hh + 1];
                x[2 * hh] = fma2(a, c2, mul2(bq, ns2));
                x[2 * hh + 1] = fma2(a, s2, mul2(bq, c2));
            }
        }
        if (CONTIG) {
            float4* r4 = reinterpret_cast<float4*>(row);
#pragma unroll
            for (int j = 0; j < M / 4; ++j) r4[j] = make_float4(x[2 * j].x, x[2 * j].y, x[2 * j + 1].x, x[2 * j + 1].y);
        } else {
#pragma unroll
            for (int i = 0; i < M2; ++i) {
                row[(2 * i) * stride] = x[i].x;
                row[(2 * i + 1) * stride] = x[i].y;
            }
        }
    }
}

// Inverse rotation of every n-channel unit of the tile, then RoPE: bits
// [0, 5), then bits [10, ln) (n > 1024), then bits [5, min(ln, 10)) with RoPE
// fused (the butterflies of different bits commute).
__device__ __forceinline__ void fwht_rope_tile(float* kt, int RS, int TT, int C, int ln, const float4* rope,
                                               int64_t t0) {
    fwht_pass<5, true, false>(kt, RS, TT, C, 0, rope, t0);
    __syncthreads();
    if (ln > 10) {
        switch (ln - 10) {
            case 1: fwht_pass<1, false, false>(kt, RS, TT, C, 10, rope, t0); break;
            case 2: fwht_pass<2, false, false>(kt, RS, TT, C, 10, rope, t0); break;
            default: fwht_pass<3, false, false>(kt, RS, TT, C, 10, rope, t0); break;
        }
        __syncthreads();
    }
    switch (ln < 10 ? ln - 5 : 5) {
        case 2: fwht_pass<2, false, true>(kt, RS, TT, C, 5, rope, t0); break;
        case 3: fwht_pass<3, false, true>(kt, RS, TT, C, 5, rope, t0); break;
        case 4: fwht_pass<4, false, true>(kt, RS, TT, C, 5, rope, t0); break;
        default: fwht_pass<5, false, true>(kt, RS, TT, C, 5, rope, t0); break;
    }
    __syncthreads();
}

// Live (in range, not a sink) tokens of the tile [t0, t0 + TT) as a bit mask.
__device__ __forceinline__ uint32_t tile_live(const uint32_t* smask, int64_t t0, int64_t t_end, int TT) {
    const int64_t n = t_end - t0 < TT ? t_end - t0 : TT;
    if (n <= 0) return 0u;
    const int sh = static_cast<int>(t0 & 31);
    uint32_t sinks = smask[t0 >> 5] >> sh;
    if (sh != 0 && sh + n > 32) sinks |= smask[(t0 >> 5) + 1] << (32 - sh);
    const uint32_t range = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
    return range & ~sinks;
}

// REG: every V unit has its own thread (units <= blockDim.x), whose
// accumulators stay in registers for the whole split (no shared accumulator);
// ntq > 1 token phases split a tile's tokens over that many units per
// channel group, merged in a fixed order at the end.
template <int CPT, bool REG>
__global__ void __launch_bounds__(kGenThreads, 2) decode_generic_kernel(DecodeParams p, int ln, int rep, int TT,
                                                                      int ntq) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int C = p.C, W = C / 16, MG = C / kQuantGroup, Hq = p.Hq, Hkv = p.Hkv, RS = tile_row_stride(C);
    const TileSmem lay = tile_smem(C, Hq, TT, REG);
    float* kt = reinterpret_cast<float*>(dsm + lay.kt);    // [TT][RS] keys, natural channel order (padded)
    float* qr = reinterpret_cast<float*>(dsm + lay.q);     // [Hq][128] RoPE'd q x qscale x k_norm
    float* accs = reinterpret_cast<float*>(dsm + lay.acc); // [Hq][kAccStride] P.V, rotated V frame (!REG)
    float* lg = reinterpret_cast<float*>(dsm + lay.lg);    // [TT][Hq] logits, then p
    float* ml = reinterpret_cast<float*>(dsm + lay.ml);    // [Hq][2] running (max, sum), log2 domain
    float* al = reinterpret_cast<float*>(dsm + lay.al);    // [Hq] this tile's rescale of the running state
    uint32_t* kst = reinterpret_cast<uint32_t*>(dsm + lay.kst);  // cp.async stage: K words, per-word meta
    uint32_t* vst = reinterpret_cast<uint32_t*>(dsm + lay.vst);  // cp.async stage: V words, meta
    const uint4* slot_ch = reinterpret_cast<const uint4*>(p.plan + kPlanHeader + W);  // [(e/4) W + w] -> 4 padded channels
    const int tid = threadIdx.x, NT = blockDim.x;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    const int64_t tb = p.tok_begin ? p.tok_begin[b] : 0, te = p.tok_end ? (p.tok_end[b] < T ? p.tok_end[b] : T) : T;
    const int64_t t_begin = tb + static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = t_begin + p.chunk < te ? t_begin + p.chunk : te;
    const bool bad_plan = !plan_matches(p.plan, kDecodeGeneric, 1 << ln, C);
    const int64_t prow = (static_cast<int64_t>(b) * p.NP + split) * Hq;
    if (t_begin >= t_end || bad_plan) {
        const float fill = bad_plan ? __int_as_float(0x7fc00000) : 0.0f;
        for (int h = tid; h < Hq; h += NT) {
            p.ws_ml[(prow + h) * 2] = bad_plan ? fill : -INFINITY;
            p.ws_ml[(prow + h) * 2 + 1] = fill;
            for (int k = 0; k < kHeadDim; ++k) p.ws_o[(prow + h) * kHeadDim + k] = fill;
        }
        pdl_trigger();
        return;
    }
    // query: RoPE at T-1 (proj/src/pipeline.cpp:144-152), x log2(e)/sqrt(d) x 1/sqrt(n)
    const float qs = p.qscale * p.k_norm;
    for (int i = tid; i < Hq * 64; i += NT) {
        const int h = i / 64, f = i % 64;
        const float a = h2f(p.q[(static_cast<int64_t>(b) * Hq + h) * kHeadDim + f]);
        const float bb = h2f(p.q[(static_cast<int64_t>(b) * Hq + h) * kHeadDim + f + 64]);
        const float2 cs = rope_at(p.rope, T - 1, f);
        qr[h * kHeadDim + f] = (a * cs.x - bb * cs.y) * qs;
        qr[h * kHeadDim + f + 64] = (a * cs.y + bb * cs.x) * qs;
    }
    if (!REG)
        for (int i = tid; i < Hq * kAccStride; i += NT) accs[i] = 0.f;
    for (int h = tid; h < Hq; h += NT) {
        ml[2 * h] = -INFINITY;
        ml[2 * h + 1] = 0.f;
    }
    const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;
    const float rW = 1.0f / static_cast<float>(W);
    const int ltt = __ffs(TT) - 1;  // TT is a power of two
    constexpr int NPART = 16 / CPT;
    const int nhc = (rep + 3) / 4, vunits = W * NPART * nhc, units = vunits * ntq;
    const float rV = 1.0f / static_cast<float>(vunits);
    float2 racc[4][CPT / 2];  // REG: this thread's unit, running over the split
    float rbz[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        rbz[r] = 0.f;
#pragma unroll
        for (int e = 0; e < CPT / 2; ++e) racc[r][e] = make_float2(0.f, 0.f);
    }
    // K of a tile: every thread stages exactly the (token, word) tasks it
    // dequantises in A (its own cp.async groups, no barrier), with a private
    // copy of the word's meta
    auto stage_k = [&](int64_t t0) {
        const int64_t n = t_end - t0 < TT ? t_end - t0 : TT;
        for (int i = tid; i < n * W; i += NT) {
            const int t = fdiv(i, rW), w = i - t * W;
            const int64_t r = row0 + t0 + t;
            cp_async4(kst + i, p.cache.k_codes + r * W + w);
            cp_async4(kst + TT * W + i, p.cache.k_meta + r * MG + (w >> 3));
        }
        cp_async_commit();
    };
    auto stage_v = [&](int64_t t0) {  // read in V after a barrier
        const int64_t n = t_end - t0 < TT ? t_end - t0 : TT;
        for (int i = tid; i < n * W; i += NT) cp_async4(vst + i, p.cache.v_codes + (row0 + t0) * W + i);
        for (int i = tid; i < n * MG; i += NT) cp_async4(vst + TT * W + i, p.cache.v_meta + (row0 + t0) * MG + i);
        cp_async_commit();
    };
    stage_k(t_begin);
    for (int64_t t0 = t_begin; t0 < t_end; t0 += TT) {
        const uint32_t live = tile_live(smask, t0, t_end, TT);
        // A: dequantise + un-reorder the tile's keys
        cp_async_wait<0>();
        for (int i = tid; i < TT * W; i += NT) {
            const int t = fdiv(i, rW), w = i - t * W;
            if (!((live >> t) & 1u)) continue;
            const uint32_t word = kst[i], m = kst[TT * W + i];
            const float s = h2f(static_cast<uint16_t>(m & 0xffffu)), z = h2f(static_cast<uint16_t>(m >> 16));
            float* row = kt + t * RS;
            const float2 s2 = make_float2(s, s), nz2 = make_float2(-z, -z);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
                const uint4 ch = __ldg(slot_ch + e4 * W + w);
                const float2 v0 = mul2(s2, add2(code2_f32(word >> (8 * e4)), nz2));  // exact s*(c - z)
                const float2 v1 = mul2(s2, add2(code2_f32(word >> (8 * e4 + 4)), nz2));
                row[ch.x] = v0.x;
                row[ch.y] = v0.y;
                row[ch.z] = v1.x;
                row[ch.w] = v1.y;
            }
        }
        __syncthreads();
        stage_v(t0);  // the previous tile's V phase is done (barrier above)
        if (t0 + TT < t_end) stage_k(t0 + TT);
        else cp_async_commit();  // keep the group count uniform
        // B: inverse rotation of every n-channel unit, RoPE on each head
        fwht_rope_tile(kt, RS, TT, C, ln, p.rope, t0);
        // L: logits, four threads per (KV head, token), frequency quarter fq
        for (int i0 = 0; i0 < Hkv * TT * 4; i0 += NT) {
            const int i = i0 + tid, fq = i & 3, pr = i >> 2, t = pr & (TT - 1), kv = pr >> ltt;
            const bool in = i < Hkv * TT * 4, act = in && ((live >> t) & 1u);
            float4 ka[4], kb[4];
            if (act) {
                const float* row = kt + t * RS + kv * (kHeadDim + kHeadDim / 8);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    ka[j] = *reinterpret_cast<const float4*>(row + padc(16 * fq + 4 * j));
                    kb[j] = *reinterpret_cast<const float4*>(row + padc(64 + 16 * fq + 4 * j));
                }
            }
            auto dot = [&](int h) {
                const float4* qa = reinterpret_cast<const float4*>(qr + h * kHeadDim + 16 * fq);
                const float4* qb = reinterpret_cast<const float4*>(qr + h * kHeadDim + 64 + 16 * fq);
                float2 s2[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {  // four independent float2 chains
                    const float4 x = qa[j], y = qb[j];
                    float2 s = mul2(make_float2(x.x, x.y), make_float2(ka[j].x, ka[j].y));
                    s = fma2(make_float2(x.z, x.w), make_float2(ka[j].z, ka[j].w), s);
                    s = fma2(make_float2(y.x, y.y), make_float2(kb[j].x, kb[j].y), s);
                    s2[j] = fma2(make_float2(y.z, y.w), make_float2(kb[j].z, kb[j].w), s);
                }
                const float2 u = add2(add2(s2[0], s2[1]), add2(s2[2], s2[3]));
                return u.x + u.y;
            };
            if ((rep & 3) == 0) {  // four heads at a time, reduce-scatter over the quarter lanes
                for (int r0 = 0; r0 < rep; r0 += 4) {
                    float v[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[r] = act ? dot(kv * rep + r0 + r) : 0.f;
                    const bool hi = fq & 2, lo = fq & 1;
                    float k0 = hi ? v[2] : v[0], k1 = hi ? v[3] : v[1];
                    k0 += __shfl_xor_sync(0xffffffffu, hi ? v[0] : v[2], 2);
                    k1 += __shfl_xor_sync(0xffffffffu, hi ? v[1] : v[3], 2);
                    float kk = lo ? k1 : k0;
                    kk += __shfl_xor_sync(0xffffffffu, lo ? k0 : k1, 1);
                    if (in) lg[t * Hq + kv * rep + r0 + fq] = act ? kk : -INFINITY;  // lane fq: head r0 + fq
                }
            } else {
                for (int r = 0; r < rep; ++r) {
                    float part = act ? dot(kv * rep + r) : 0.f;
                    part += __shfl_xor_sync(0xffffffffu, part, 1);
                    part += __shfl_xor_sync(0xffffffffu, part, 2);
                    if (fq == 0 && in) lg[t * Hq + kv * rep + r] = act ? part : -INFINITY;
                }
            }
        }
        __syncthreads();
        // S: online softmax per q head over the tile
        for (int h = tid; h < Hq; h += NT) {
            const float mo = ml[2 * h];
            float mt = -INFINITY;
            for (int t = 0; t < TT; ++t) mt = fmaxf(mt, lg[t * Hq + h]);
            const float mn = fmaxf(mo, mt);
            float alpha = 1.f, sum = 0.f;
            if (mn != -INFINITY) {
                alpha = exp2f(mo - mn);
                for (int t = 0; t < TT; ++t) {
                    const float pv = exp2f(lg[t * Hq + h] - mn);
                    lg[t * Hq + h] = pv;
                    sum += pv;
                }
            }
            ml[2 * h] = mn;
            ml[2 * h + 1] = ml[2 * h + 1] * alpha + sum;
            al[h] = alpha;
        }
        cp_async_wait<1>();  // this tile's V stage (the next tile's K may still be in flight)
        __syncthreads();
        // V: per (word, channel part, head chunk, token phase), sum over the
        // phase's tokens of the tile in registers
        for (int u = tid; u < units; u += NT) {
            const int tq = fdiv(u, rV), vu = u - tq * vunits;
            const int rest = fdiv(vu, rW), w = vu - rest * W, part = rest % NPART, hc = rest / NPART;
            const int kv = w >> 3, h0 = kv * rep + 4 * hc, nh = rep - 4 * hc < 4 ? rep - 4 * hc : 4;
            float2 tacc[4][CPT / 2];
            float tbz[4];
            float2 (&acc)[4][CPT / 2] = REG ? racc : tacc;
            float (&bz)[4] = REG ? rbz : tbz;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (REG) {  // rescale the running sums to this tile's maximum
                    const float a = r < nh ? al[h0 + r] : 0.f;
                    bz[r] *= a;
#pragma unroll
                    for (int e = 0; e < CPT / 2; ++e) acc[r][e] = mul2(acc[r][e], make_float2(a, a));
                } else {
                    bz[r] = 0.f;
#pragma unroll
                    for (int e = 0; e < CPT / 2; ++e) acc[r][e] = make_float2(0.f, 0.f);
                }
            }
            for (int t = tq; t < TT; t += ntq) {
                if (!((live >> t) & 1u)) continue;
                const uint32_t word = vst[t * W + w] >> (2 * CPT * part), m = vst[TT * W + t * MG + kv];
                const float s = h2f(static_cast<uint16_t>(m & 0xffffu)), z = h2f(static_cast<uint16_t>(m >> 16));
                float ps[4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    ps[rr] = rr < nh ? lg[t * Hq + h0 + rr] * s : 0.f;
                    bz[rr] = fmaf(ps[rr], z, bz[rr]);
                }
#pragma unroll
                for (int e = 0; e < CPT / 2; ++e) {
                    const float2 c = code2_f32(word >> (4 * e));
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) acc[rr][e] = fma2(make_float2(ps[rr], ps[rr]), c, acc[rr][e]);
                }
            }
            if (!REG) {
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    if (rr >= nh) break;
                    const float a = al[h0 + rr];
                    float* dst = accs + (h0 + rr) * kAccStride;
#pragma unroll
                    for (int e = 0; e < CPT; ++e) {
                        const int ch = (w & 7) * 16 + part * CPT + e;
                        const int ci = ch + (ch >> 4);
                        dst[ci] = fmaf(dst[ci], a, (e & 1 ? acc[rr][e / 2].y : acc[rr][e / 2].x) - bz[rr]);
                    }
                }
            }
        }
        // the next tile's A and L phases touch kt / lg only after their own
        // barriers; V reads lg and al, rewritten two barriers later
    }
    __syncthreads();
    pdl_trigger();
    for (int h = tid; h < Hq; h += NT) {
        p.ws_ml[(prow + h) * 2] = ml[2 * h];
        p.ws_ml[(prow + h) * 2 + 1] = ml[2 * h + 1];
    }
    if (REG) {
        // token phases: partial sums through the (now free) key tile, merged in phase order
        float* scr = ntq > 1 ? kt : nullptr;
        if (tid < units) {
            const int tq = fdiv(tid, rV), vu = tid - tq * vunits;
            const int rest = fdiv(vu, rW), w = vu - rest * W, part = rest % NPART, hc = rest / NPART;
            const int h0 = (w >> 3) * rep + 4 * hc, nh = rep - 4 * hc < 4 ? rep - 4 * hc : 4;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                if (rr >= nh) break;
                const int o = (h0 + rr) * kHeadDim + (w & 7) * 16 + part * CPT;
                float* dst = scr ? scr + tq * Hq * kHeadDim + o : p.ws_o + prow * kHeadDim + o;
#pragma unroll
                for (int e = 0; e < CPT / 2; ++e) {
                    dst[2 * e] = racc[rr][e].x - rbz[rr];
                    dst[2 * e + 1] = racc[rr][e].y - rbz[rr];
                }
            }
        }
        if (scr) {
            __syncthreads();
            for (int i = tid; i < Hq * kHeadDim; i += NT) {
                float s = scr[i];
                for (int q = 1; q < ntq; ++q) s += scr[q * Hq * kHeadDim + i];
                p.ws_o[prow * kHeadDim + i] = s;
            }
        }
    } else {
        for (int i = tid; i < Hq * kHeadDim; i += NT) {
            const int h = i / kHeadDim, d = i % kHeadDim;
            p.ws_o[(prow + h) * kHeadDim + d] = accs[h * kAccStride + d + (d >> 4)];
        }
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

namespace {
// V phase: units of (packed word, channel part of CPT codes, chunk of <= 4 q
// heads[, token phase]).  Few units (<= 128 at CPT 8): each has a thread of
// its own and keeps its sums in registers (REG), with token phases filling the
// CTA; otherwise units loop over the threads and merge into shared memory,
// CPT 16 halved down to 4 while threads would idle.
struct GenV {
    int cpt;
    bool reg;
};
GenV generic_v(const rkv_layer_desc& d) {
    const int W = d.num_kv_heads * d.head_dim / 16, rep = d.num_q_heads / d.num_kv_heads;
    const int base = W * ((rep + 3) / 4);
    if (2 * base <= kGenThreads) return {8, true};
    int cpt = 16;
    while (cpt > 4 && base * (16 / cpt) < kGenThreads) cpt /= 2;
    return {cpt, false};
}
int generic_ntq(const rkv_layer_desc& d, int TT) {  // token phases (REG): fill the CTA, partials fit the key tile
    const GenV v = generic_v(d);
    if (!v.reg) return 1;
    const int C = d.num_kv_heads * d.head_dim, base = C / 16 * ((d.num_q_heads / d.num_kv_heads + 3) / 4) * 2;
    int ntq = 1;
    while (ntq < 8 && ntq * 2 <= TT && 2 * ntq * base <= kGenThreads &&
           static_cast<size_t>(2 * ntq) * d.num_q_heads * kHeadDim <= static_cast<size_t>(TT) * tile_row_stride(C))
        ntq *= 2;
    return ntq;
}
}  // namespace

size_t generic_decode_smem(const rkv_layer_desc& d, int TT) {
    return tile_smem(d.num_kv_heads * d.head_dim, d.num_q_heads, TT, generic_v(d).reg).total;
}

DecodePlan plan_decode_generic(const rkv_layer_desc& d, int64_t max_seq_len) {
    DecodePlan pl{};
    pl.kind = kDecodeGeneric;
    pl.N = d.heads_per_group * d.head_dim;
    pl.REP = d.num_q_heads / d.num_kv_heads;
    pl.P = pl.PP = 1;
    pl.NT = kGenThreads;
    pl.stages = generic_v(d).cpt * (generic_v(d).reg ? -1 : 1);  // the V-phase specialisation (launch_decode_generic)
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    // tile: the largest of 16/8/4 tokens that leaves room for two CTAs per SM,
    // else the largest of 32..1 that fits one
    pl.TT = 0;
    if (const int o = options().generic_tile.load())  // experiment switch
        if (o >= 1 && o <= kTileMax && !(o & (o - 1)) && generic_decode_smem(d, o) <= 227u * 1024u) pl.TT = o;
    for (int tt = 16; tt >= 4 && !pl.TT; tt /= 2)
        if (generic_decode_smem(d, tt) + 1024 <= 227u * 1024u / 2) pl.TT = tt;
    for (int tt = kTileMax; tt >= 1 && !pl.TT; tt /= 2)
        if (generic_decode_smem(d, tt) <= 227u * 1024u) pl.TT = tt;
    if (!pl.TT) pl.TT = 1;
    pl.smem = generic_decode_smem(d, pl.TT);
    pl.PP = generic_ntq(d, pl.TT);
    pl.per_sm = pl.smem + 1024 <= 227u * 1024u / 2 ? 2 : 1;
    const int slots = num_sms() * pl.per_sm;
    const int64_t max_split = std::max<int64_t>(1, (max_seq_len + 4 * pl.TT - 1) / (4 * pl.TT));  // >= 4 tiles each
    int S = choose_splits(slots, d.batch, max_split);
    if (const int o = options().dec_splits.load())  // experiment switch: splits per sequence
        if (o > 0) S = static_cast<int>(std::min<int64_t>(max_split, o));
    int64_t chunk = (max_seq_len + S - 1) / S;
    chunk = (chunk + pl.TT - 1) / pl.TT * pl.TT;
    pl.chunk = static_cast<int>(chunk);
    pl.S = static_cast<int>((max_seq_len + pl.chunk - 1) / pl.chunk);
    pl.NP = pl.S;
    pl.ok = pl.smem <= 227 * 1024;
    return pl;
}

cudaError_t launch_decode_generic(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p,
                                  cudaStream_t s) {
    int ln = 0;
    while ((1 << ln) < plan.N) ++ln;
    const dim3 grid(plan.S, d.batch);
    cudaError_t e;
    auto go = [&](auto kern) {
        cudaError_t err = ensure_smem_k(kern, plan.smem);
        if (err != cudaSuccess) return err;
        kern<<<grid, kGenThreads, plan.smem, s>>>(p, ln, plan.REP, plan.TT, plan.PP);
        return cudaSuccess;
    };
    switch (plan.stages) {
        case 16: e = go(decode_generic_kernel<16, false>); break;
        case 8: e = go(decode_generic_kernel<8, false>); break;
        case 4: e = go(decode_generic_kernel<4, false>); break;
        default: e = go(decode_generic_kernel<8, true>); break;
    }
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_decode_combine(p, d.batch, s);
}

}  // namespace rkv
