// quantize_kv.cu -- fused quantize-append for sm_100a.
//
// One work item = (K or V, sequence b, token pair).  A persistent CTA walks
// items blockIdx.x, blockIdx.x + gridDim.x, ...; the pair's two fp16 rows
// (contiguous in [B][num_new][C]) arrive by one TMA bulk copy into a
// double-buffered stage, so the next item's rows stream in while this one is
// computed.  Every register holds a float2 = one channel of both tokens, so
// each FWHT butterfly, normalisation and threshold subtraction is one
// packed FP32x2 instruction.
//
//   1. FWHT (thread g owns channels [32g, 32g+32) = its "region"):
//      layout A: registers = channel bits 0..4 (5 stages), result to the
//      token-pair row in shared memory (float4 = 2 channels x 2 tokens,
//      16-byte chunks XOR-swizzled by region);  layout B': lane lam of a
//      unit holds chunk pairs lam + L*j, registers = channel bit 0 and the
//      high bits (stages 5 .. log2(n)-1), x 1/sqrt(n), back to the row.
//      K units: n = G*128 channels (grouped-head rotation), V: n = 128.
//      The fp16 rows are read in a per-lane XOR-relabelled chunk order so the
//      LDS.128 stream is bank-conflict free; the relabelling turns into a
//      +-1 per 8-channel block after the A stages (H P_s = D_s H), applied
//      exactly before the row is stored.
//   2. Quantize (thread g owns slots [32g, 32g+32) = two packed words per
//      token; 4 lanes = one 128-slot group).  K slots gather their channel
//      through the calibrated permutation (slot j <- channel perm[j],
//      proj/src/reorder.cpp:112-128) via a per-CTA byte-offset table; V slots
//      are the natural channels.  Group min/max by shuffles; one lane per
//      (group, token) derives scale / zero as proj/src/quant.cpp:53-97 does and
//      turns round-half-away(x/s) + zero into three exact fp32 thresholds, so
//      code = #{k : x >= T_k} -- taken from the sign bits of x - T_k (one
//      FADD2 covers both tokens) and packed with funnel shifts.
//   3. Sink tokens (proj/src/kv_cache.cpp:8-22 `sink`) keep their raw fp16
//      rows in the sidecar; their packed words/meta are zero.
// Reference chain restated: rotate_rows -> apply_reorder -> quantize_token ->
// LayerKVCache::append (proj/src/pipeline.cpp:171-176, :317-324).
#include <cstdio>

#include "rkv_common.cuh"
#include "rkv_internal.h"

namespace rkv {

namespace {

// float2 index (one channel of both tokens) of channel c in the token-pair
// row: 32-channel regions padded to 33 slots, so layout-A stores (one region
// per lane), layout-B reads (consecutive channels of one region per unit) and
// the V quantize reads are bank-conflict free per half-warp with plain
// [reg + immediate] addressing.
__device__ __forceinline__ int pos2(int c) { return (c >> 5) * 33 + (c & 31); }

// STS.64 straight from an FP32x2 result pair (a plain float2 store makes the
// compiler copy the pair first).
__device__ __forceinline__ void sts64(uint32_t addr, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

// Layout-A half of the FWHT for region g: channels [32g, 32g+32) of both
// tokens from the fp16 stage rows, stages on channel bits 0..4, stored to the
// token-pair row.
__device__ __forceinline__ void fwht_region_a_regs(const uint16_t* st0, const uint16_t* st1, int g, float2 (&x)[32]) {
    const int s = (g >> 1) & 3;  // chunk relabel: conflict-free 64-byte-strided LDS.128
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 va = lds128(st0 + 32 * g + 8 * (q ^ s));
        const uint4 vb = lds128(st1 + 32 * g + 8 * (q ^ s));
        const uint16_t* ha = reinterpret_cast<const uint16_t*>(&va);
        const uint16_t* hb = reinterpret_cast<const uint16_t*>(&vb);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[8 * q + e] = make_float2(h2f(ha[e]), h2f(hb[e]));
    }
    bfly_range<32, 0, 5>(x);
    // block q now holds true block q times (-1)^popcount(q & s)
    const float f1 = (s & 1) ? -1.0f : 1.0f, f2 = (s & 2) ? -1.0f : 1.0f;
    const float2 sg1 = make_float2(f1, f1), sg2 = make_float2(f2, f2), sg3 = make_float2(f1 * f2, f1 * f2);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        x[8 + e] = mul2(x[8 + e], sg1);
        x[16 + e] = mul2(x[16 + e], sg2);
        x[24 + e] = mul2(x[24 + e], sg3);
    }
}
__device__ __forceinline__ void fwht_region_a(const uint16_t* st0, const uint16_t* st1, float2* row, int g) {
    float2 x[32];
    fwht_region_a_regs(st0, st1, g, x);
    const uint32_t dst = smem_u32(row + 33 * g);
#pragma unroll
    for (int c = 0; c < 32; ++c) sts64(dst + 8 * c, x[c]);
}

// Layout-B half: lane lam of an n-channel unit u (L = n/32 lanes) holds the
// channels u*n + lam + L*j, j = 0..31; stages on channel bits 5..log2(n)-1,
// then x norm (proj/src/hadamard.cpp:62-63), back in place.
template <int N>
__device__ __forceinline__ void fwht_unit_b(float2* row, int u, int lam, float norm) {
    constexpr int L = N / 32, LL = ilog2(L), LN = ilog2(N);
    float2 x[32];
    float2* base = row + 33 * (u * L) + lam;  // channel u*N + lam + L*j -> base + pos2(L*j)
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = base[pos2(L * j)];
    bfly_range<32, 5 - LL, LN - LL>(x);
    const float2 nn = make_float2(norm, norm);
    const uint32_t b32 = smem_u32(base);
#pragma unroll
    for (int j = 0; j < 32; ++j) sts64(b32 + 8 * pos2(L * j), mul2(x[j], nn));
}

// Slots [32g, 32g+32) of both tokens -> two packed words per token + group meta.
struct QuantOut {
    uint32_t w[2][2];  // [token][word]
    uint32_t meta;     // this lane's (group, token) meta: lane&3 == 0 -> token 0, == 1 -> token 1
};

// sign bits of x - T_k for 8 consecutive slots of one token -> 16 code bits
// (inverted: bit set = below threshold).  bit1 = sign(d2),
// bit0 = sign(d1) ^ sign(d2) ^ sign(d3)  (T1 <= T2 <= T3).
template <int TOK>
__device__ __forceinline__ uint32_t code_bits8(const float2* x, float2 n1, float2 n2, float2 n3) {
    uint32_t a = 0;
#pragma unroll
    for (int e = 7; e >= 0; --e) {
        const float2 d1 = add2(x[e], n1), d2 = add2(x[e], n2), d3 = add2(x[e], n3);
        const float s1 = TOK ? d1.y : d1.x, s2 = TOK ? d2.y : d2.x, s3 = TOK ? d3.y : d3.x;
        a = __funnelshift_l(__float_as_uint(s2), a, 1);
        a = __funnelshift_l(__float_as_uint(s1) ^ __float_as_uint(s2) ^ __float_as_uint(s3), a, 1);
    }
    return a;
}

template <int FMT>
__device__ __forceinline__ QuantOut quantize_run(const float2 (&x)[32], int lane) {
    float mn0 = x[0].x, mx0 = x[0].x, mn1 = x[0].y, mx1 = x[0].y;
#pragma unroll
    for (int e = 1; e < 31; e += 2) {
        mn0 = fminf(mn0, fminf(x[e].x, x[e + 1].x));
        mx0 = fmaxf(mx0, fmaxf(x[e].x, x[e + 1].x));
        mn1 = fminf(mn1, fminf(x[e].y, x[e + 1].y));
        mx1 = fmaxf(mx1, fmaxf(x[e].y, x[e + 1].y));
    }
    mn0 = fminf(mn0, x[31].x);
    mx0 = fmaxf(mx0, x[31].x);
    mn1 = fminf(mn1, x[31].y);
    mx1 = fmaxf(mx1, x[31].y);
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, o));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const bool odd = lane & 1;
    const GroupQuant gq = group_params<FMT>(odd ? mn1 : mn0, odd ? mx1 : mx0);
    const int l0 = lane & ~3;
    const float2 n1 = make_float2(-__shfl_sync(0xffffffffu, gq.t1, l0), -__shfl_sync(0xffffffffu, gq.t1, l0 + 1));
    const float2 n2 = make_float2(-__shfl_sync(0xffffffffu, gq.t2, l0), -__shfl_sync(0xffffffffu, gq.t2, l0 + 1));
    const float2 n3 = make_float2(-__shfl_sync(0xffffffffu, gq.t3, l0), -__shfl_sync(0xffffffffu, gq.t3, l0 + 1));
    QuantOut o;
    o.meta = gq.meta;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        o.w[0][h] = ~__byte_perm(code_bits8<0>(x + 16 * h, n1, n2, n3), code_bits8<0>(x + 16 * h + 8, n1, n2, n3),
                                 0x5410);
        o.w[1][h] = ~__byte_perm(code_bits8<1>(x + 16 * h, n1, n2, n3), code_bits8<1>(x + 16 * h + 8, n1, n2, n3),
                                 0x5410);
    }
    return o;
}

struct Item {
    bool isv, has1;
    int b;
    int i0;
};

// item = (K or V, sequence, token pair); with k_only (V quantized by
// quantize_v_kernel) the items are K only
// x / d for 32-bit x, d without the integer-division sequence: the fp64
// quotient is within one of the truth, fixed up exactly.
__device__ __forceinline__ uint32_t udiv32(uint32_t x, uint32_t d) {
    uint32_t q = static_cast<uint32_t>(__dmul_rz(static_cast<double>(x), __drcp_rn(static_cast<double>(d))));
    if (static_cast<uint64_t>(q) * d > x) --q;
    else if (static_cast<uint64_t>(q + 1) * d <= x) ++q;
    return q;
}

__device__ __forceinline__ Item decode_item(uint32_t it, uint32_t npairs, int num_new, int k_only) {
    Item r;
    r.isv = k_only ? false : (it & 1u);
    const uint32_t rest = k_only ? it : it >> 1;
    const uint32_t b = udiv32(rest, npairs);
    r.b = static_cast<int>(b);
    r.i0 = static_cast<int>(rest - b * npairs) * 2;
    r.has1 = r.i0 + 1 < num_new;
    return r;
}

__device__ __forceinline__ void issue_item(const QuantParams& p, uint32_t it, uint32_t npairs, uint16_t* dst,
                                           uint64_t* bar) {
    const Item r = decode_item(it, npairs, static_cast<int>(p.num_new), p.k_only);
    const uint16_t* src = (r.isv ? p.v_new : p.k_new) + (static_cast<int64_t>(r.b) * p.num_new + r.i0) * p.C;
    const uint32_t bytes = static_cast<uint32_t>((r.has1 ? 2 : 1) * p.C * 2);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(dst, src, bytes, bar);
}

// Per-item metadata, computed one item ahead by threads 0..2 (global loads
// off the critical path) and published by the item-end barrier.
struct ItemMeta {
    int slot[2];  // sidecar slot of the pair's tokens, -1 = not a sink
    int64_t pos0; // cache position of the pair's first token
};

__device__ __forceinline__ void item_meta(const QuantParams& p, uint32_t it, uint32_t npairs, int num_new,
                                          ItemMeta* m, int tid) {
    const Item r = decode_item(it, npairs, num_new, p.k_only);
    const int64_t pos0 = p.start_pos[r.b] + r.i0;
    if (tid < 2) {
        int slot = -1;
        const int i = r.i0 + tid;
        const int64_t pos = pos0 + tid;
        if (p.sink_flags && i < num_new && pos >= 0 && pos < p.max_tokens &&
            p.sink_flags[static_cast<int64_t>(r.b) * num_new + i]) {
            int before = 0;
            for (int q = 0; q < i; ++q) before += p.sink_flags[static_cast<int64_t>(r.b) * num_new + q] ? 1 : 0;
            slot = p.cache.sink_count[r.b] + before;
            // a full sidecar keeps the token quantized (mask bit clear, not counted)
            if (slot >= p.max_sinks) slot = -1;
        }
        m->slot[tid] = slot;
    } else {
        m->pos0 = pos0;
    }
}

// Shared memory: row [C/32][33] float2 (8.25 C B) | gather table [8][C/32] of
// 4 x u16 float2 indices (2C B) | stage [2 buffers][2 tokens][C] fp16 (8C B).
// Item k's rows land in stage k & 1; item k+1's copy is issued at item k-1's
// end, so it has a whole item to arrive.
template <int N, int FMT, int NS>
__global__ void __launch_bounds__(256, 2) quantize_kv_kernel(QuantParams p, uint32_t items, uint32_t npairs) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar[2];
    __shared__ ItemMeta s_meta[2];
    const int C = p.C, G32 = C / 32, W = C / 16, MG = C / kQuantGroup;
    const int num_new = static_cast<int>(p.num_new);
    float2* row = reinterpret_cast<float2*>(smem);
    uint16_t* tbl = reinterpret_cast<uint16_t*>(smem + G32 * 33 * 8);
    uint16_t* stage = reinterpret_cast<uint16_t*>(smem + G32 * 33 * 8 + 2 * C);  // [2][2][C]

    const int tid = threadIdx.x, lane = tid & 31;
    const bool act = tid < G32;
    const int g = act ? tid : tid - 16;  // C/32 is a multiple of 16: idle half-warps mirror the previous one
    const uint32_t step = gridDim.x;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
        if (blockIdx.x < items) issue_item(p, blockIdx.x, npairs, stage, &bar[0]);
        if (NS == 2 && blockIdx.x + step < items) issue_item(p, blockIdx.x + step, npairs, stage + 2 * C, &bar[1]);
    }
    if (tid < 3 && blockIdx.x < items) item_meta(p, blockIdx.x, npairs, num_new, &s_meta[0], tid);
    // K gather table, only if this CTA sees a K item (even item index):
    // slot j = 32t + 4q + e  ->  tbl[(q * G32 + t) * 4 + e] = float2 index of channel perm[j]
    if (act && (p.k_only || (gridDim.x & 1u) || !(blockIdx.x & 1u))) {
        const int4* pv = reinterpret_cast<const int4*>(p.perm) + 8 * g;
        int4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(pv + q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t lo = static_cast<uint32_t>(pos2(v[q].x)) | (static_cast<uint32_t>(pos2(v[q].y)) << 16);
            const uint32_t hi = static_cast<uint32_t>(pos2(v[q].z)) | (static_cast<uint32_t>(pos2(v[q].w)) << 16);
            *reinterpret_cast<uint2*>(tbl + (q * G32 + g) * 4) = make_uint2(lo, hi);
        }
    }
    __syncthreads();

    uint32_t k = 0;
    for (uint32_t it = blockIdx.x; it < items; it += step, ++k) {
        const Item r = decode_item(it, npairs, num_new, p.k_only);
        const int sb = k & 1;  // metadata slot; TMA stage sb (NS = 2) or 0 (NS = 1)
        const uint16_t* st = stage + (NS == 2 ? sb : 0) * 2 * C;
        mbar_wait(&bar[NS == 2 ? sb : 0], NS == 2 ? (k >> 1) & 1u : k & 1u);

        fwht_region_a(st, r.has1 ? st + C : st, row, g);
        __syncwarp();
        if (!r.isv) {
            fwht_unit_b<N>(row, g / (N / 32), g % (N / 32), p.k_norm);
        } else {
            fwht_unit_b<128>(row, g / 4, g % 4, p.v_norm);
        }
        __syncthreads();  // stage sb consumed, row complete
        if (NS == 2 && tid == 0 && it + 2 * step < items)
            issue_item(p, it + 2 * step, npairs, stage + sb * 2 * C, &bar[sb]);
        if (NS == 1 && tid == 0 && it + step < items) issue_item(p, it + step, npairs, stage, &bar[0]);
        if (tid < 3 && it + step < items) item_meta(p, it + step, npairs, num_new, &s_meta[sb ^ 1], tid);
        const ItemMeta& meta = s_meta[sb];  // read from shared memory where used (registers are tight)

        float2 x[32];
        if (!r.isv) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint2 a = *reinterpret_cast<const uint2*>(tbl + (q * G32 + g) * 4);
                x[4 * q + 0] = row[a.x & 0xffffu];
                x[4 * q + 1] = row[a.x >> 16];
                x[4 * q + 2] = row[a.y & 0xffffu];
                x[4 * q + 3] = row[a.y >> 16];
            }
        } else {
            const float2* src = row + 33 * g;
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = src[c];
        }
        const QuantOut qo = quantize_run<FMT>(x, lane);
        if (act) {
            uint32_t* codes = r.isv ? p.cache.v_codes : p.cache.k_codes;
            uint32_t* mt = r.isv ? p.cache.v_meta : p.cache.k_meta;
            const int64_t row0 = static_cast<int64_t>(r.b) * p.max_tokens + meta.pos0;
#pragma unroll
            for (int tok = 0; tok < 2; ++tok) {
                if (tok == 1 && !r.has1) break;
                if (meta.pos0 + tok < 0 || meta.pos0 + tok >= p.max_tokens) break;  // past the cache: never written
                const bool sink = meta.slot[tok] >= 0;
                const int64_t rowi = row0 + tok;
                *reinterpret_cast<uint2*>(codes + rowi * W + 2 * g) =
                    sink ? make_uint2(0u, 0u) : make_uint2(qo.w[tok][0], qo.w[tok][1]);
                if ((lane & 3) == tok) mt[rowi * MG + g / 4] = sink ? 0u : qo.meta;
            }
        }

        // sink rows: raw fp16 rows into the sidecar (exact, proj/tests/test_kv_cache.cpp:22-45)
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {
            const int slot = meta.slot[tok];
            if (slot < 0) continue;  // slot < max_sinks by construction
            const uint4* srcr = reinterpret_cast<const uint4*>(
                (r.isv ? p.v_new : p.k_new) + (static_cast<int64_t>(r.b) * p.num_new + r.i0 + tok) * C);
            uint16_t* side = r.isv ? p.cache.sink_v : p.cache.sink_k;
            uint4* dst = reinterpret_cast<uint4*>(side + (static_cast<int64_t>(r.b) * p.max_sinks + slot) * C);
            for (int j = tid; j < C / 8; j += blockDim.x) dst[j] = __ldg(srcr + j);
            if (tid == 0 && !r.isv) p.cache.sink_pos[r.b * p.max_sinks + slot] = static_cast<int32_t>(meta.pos0 + tok);
        }
        // per-token sink bits (the K item owns them)
        if (tid < 2 && !r.isv && (tid == 0 || r.has1)) {
            const int64_t pos = meta.pos0 + tid;
            if (pos >= 0 && pos < p.max_tokens) {
                uint32_t* mw = p.cache.sink_mask + static_cast<int64_t>(r.b) * ((p.max_tokens + 31) / 32) + (pos >> 5);
                const uint32_t bit = 1u << (pos & 31);
                if (meta.slot[tid] >= 0) atomicOr(mw, bit);
                else atomicAnd(mw, ~bit);
            }
        }
        __syncthreads();  // row rewritten next; s_meta[sb ^ 1] visible
    }
    // launched as the V kernel's programmatic dependent (k_only): this grid's
    // completion must imply the V grid's, for the sink-count kernel after it
    pdl_wait();
}

// V quantize, warp-independent.  V's rotation is per head (128 channels) and
// V has no reorder, so a warp can own a 1024-channel segment of a token pair
// outright: its own TMA stage (double-buffered, its own mbarriers), layout A
// on its 32 regions, then (SH, the default) the head's last two stages as
// shuffle butterflies between the 4 lanes of a head and quantize on the
// registers, or (row buffer) layout B on its 8 heads through shared memory,
// quantize on its own slots -- only __syncwarp, never a CTA barrier.  Sub-item = (sequence, token pair,
// segment); the K items (global reorder: a CTA-wide gather) stay on
// quantize_kv_kernel.  Same arithmetic as there (fwht_region_a,
// fwht_unit_b<128>, quantize_run): bit-identical codes.
constexpr int kVSeg = 1024;                 // channels per warp segment (32 regions)
constexpr int kVRowF2 = (kVSeg / 32) * 33;  // float2 per segment row (padded regions)
// warps per CTA (1 CTA per SM) and TMA stages per warp: VS = 2 gives each
// copy a whole sub-item of lead time; VS = 1 trades it for occupancy
// SH: the head FWHT's last two stages (channel bits 5, 6 = lane bits 0, 1)
// as shuffle butterflies between lanes, then quantize_run on the registers:
// no row buffer, only the TMA stages in shared memory
template <int VW, int VS, bool SH = false>
struct VCfg {
    static constexpr int warp_bytes = VS * 2 * kVSeg * 2 + (SH ? 0 : kVRowF2 * 8);
};
template <int FMT, int VW, int VS, bool SH = false>
__global__ void __launch_bounds__(32 * VW, 1) quantize_v_kernel(QuantParams p, uint32_t subitems, uint32_t npairs,
                                                               uint32_t nseg) {
    constexpr int kVWarps = VW;
    constexpr int kVWarpBytes = VCfg<VW, VS, SH>::warp_bytes;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar[kVWarps][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = p.C, W = C / 16, MG = C / kQuantGroup;
    const int num_new = static_cast<int>(p.num_new);
    uint8_t* base = smem + warp * kVWarpBytes;
    uint16_t* stage = reinterpret_cast<uint16_t*>(base);                  // [VS][2][kVSeg]
    float2* row = reinterpret_cast<float2*>(base + VS * 2 * kVSeg * 2);   // [32][33]
    const uint32_t gw = blockIdx.x * kVWarps + warp, step = gridDim.x * kVWarps;

    // sub-item si = (b npairs + ip) nseg + seg.  A warp's sub-items advance by
    // `step`: the cursors carry (b, ip, seg) forward with two compares instead
    // of two divisions per sub-item
    struct Cursor {
        uint32_t b, ip, seg;
    };
    auto locate = [&](uint32_t si) {
        const uint32_t pr = udiv32(si, nseg), bb = udiv32(pr, npairs);
        return Cursor{bb, pr - bb * npairs, si - pr * nseg};
    };
    const Cursor dstep = locate(step);
    auto advance = [&](Cursor& c) {
        c.seg += dstep.seg;
        const uint32_t c1 = c.seg >= nseg ? 1u : 0u;
        c.seg -= c1 * nseg;
        c.ip += dstep.ip + c1;
        const uint32_t c2 = c.ip >= npairs ? 1u : 0u;
        c.ip -= c2 * npairs;
        c.b += dstep.b + c2;
    };
    auto issue = [&](const Cursor& c, int sb) {
        const int b = static_cast<int>(c.b), i0 = static_cast<int>(c.ip) * 2, seg = static_cast<int>(c.seg);
        const bool has1 = i0 + 1 < num_new;
        const uint16_t* src = p.v_new + (static_cast<int64_t>(b) * num_new + i0) * C + seg * kVSeg;
        uint16_t* dst = stage + sb * 2 * kVSeg;
        mbar_arrive_expect_tx(&bar[warp][sb], (has1 ? 2u : 1u) * kVSeg * 2);
        bulk_g2s(dst, src, kVSeg * 2, &bar[warp][sb]);
        if (has1) bulk_g2s(dst + kVSeg, src + C, kVSeg * 2, &bar[warp][sb]);
    };
    pdl_trigger();  // the K kernel (independent outputs) may start in this kernel's tail
    if (lane == 0) {
        mbar_init(&bar[warp][0], 1);
        mbar_init(&bar[warp][1], 1);
        mbar_fence_init();
        if (gw < subitems) issue(locate(gw), 0);
        if (VS == 2 && gw + step < subitems) issue(locate(gw + step), 1);
    }
    __syncwarp();
    Cursor cur = locate(gw), nxt = locate(gw + VS * step);  // this sub-item, the one whose copy we issue next
    uint32_t k = 0;
    for (uint32_t si = gw; si < subitems; si += step, ++k, advance(cur), advance(nxt)) {
        const int b = static_cast<int>(cur.b), i0 = static_cast<int>(cur.ip) * 2, seg = static_cast<int>(cur.seg);
        const bool has1 = i0 + 1 < num_new;
        const int sb = VS == 2 ? (k & 1) : 0;
        // the pair's position and sink flags: loads issued here, used after the
        // FWHT (the sidecar slot rule of quantize_kv_kernel, same inputs)
        const int64_t pos0 = p.start_pos[b] + i0;
        const uint8_t flag = lane < 2 && p.sink_flags && i0 + lane < num_new
                                 ? p.sink_flags[static_cast<int64_t>(b) * num_new + i0 + lane]
                                 : uint8_t{0};
        mbar_wait(&bar[warp][sb], VS == 2 ? (k >> 1) & 1u : k & 1u);
        const uint16_t* st = stage + sb * 2 * kVSeg;
        float2 x[32];
        if constexpr (SH) {
            fwht_region_a_regs(st, has1 ? st + kVSeg : st, lane, x);
            __syncwarp();
            // the stage is consumed: refill it with the sub-item after next
            if (lane == 0 && si + VS * step < subitems) issue(nxt, sb);
            // stages on channel bits 5, 6 (lane bits 0, 1): lower lane a + b, upper lane a - b
#pragma unroll
            for (int m = 1; m <= 2; m <<= 1) {
                const float sg = (lane & m) ? -1.0f : 1.0f;
                const float2 s2 = make_float2(sg, sg);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float2 q = make_float2(__shfl_xor_sync(0xffffffffu, x[j].x, m),
                                                 __shfl_xor_sync(0xffffffffu, x[j].y, m));
                    x[j] = fma2(x[j], s2, q);
                }
            }
            const float2 nn = make_float2(p.v_norm, p.v_norm);
#pragma unroll
            for (int j = 0; j < 32; ++j) x[j] = mul2(x[j], nn);
        } else {
            fwht_region_a(st, has1 ? st + kVSeg : st, row, lane);
            __syncwarp();
            // the stage is consumed: refill it with the sub-item after next
            if (lane == 0 && si + VS * step < subitems) issue(nxt, sb);
            fwht_unit_b<128>(row, lane / 4, lane % 4, p.v_norm);
            __syncwarp();
            const float2* srcr = row + 33 * lane;
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = srcr[c];
        }
        const QuantOut qo = quantize_run<FMT>(x, lane);
        int slot = -1;
        if (flag && pos0 + lane >= 0 && pos0 + lane < p.max_tokens) {  // lanes 0, 1: tokens i0, i0 + 1
            const int i = i0 + lane;
            int before = 0;
            for (int q = 0; q < i; ++q) before += p.sink_flags[static_cast<int64_t>(b) * num_new + q] ? 1 : 0;
            slot = p.cache.sink_count[b] + before;
            if (slot >= p.max_sinks) slot = -1;
        }
        const int slot0 = __shfl_sync(0xffffffffu, slot, 0), slot1 = __shfl_sync(0xffffffffu, slot, 1);
        const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens + pos0;
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {
            if (tok == 1 && !has1) break;
            if (pos0 + tok < 0 || pos0 + tok >= p.max_tokens) break;  // past the cache: never written
            const bool sink = (tok ? slot1 : slot0) >= 0;
            const int64_t rowi = row0 + tok;
            *reinterpret_cast<uint2*>(p.cache.v_codes + rowi * W + seg * (kVSeg / 16) + 2 * lane) =
                sink ? make_uint2(0u, 0u) : make_uint2(qo.w[tok][0], qo.w[tok][1]);
            if ((lane & 3) == tok) p.cache.v_meta[rowi * MG + seg * (kVSeg / 128) + lane / 4] = sink ? 0u : qo.meta;
        }
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {  // sink rows: this segment of the raw fp16 row into the sidecar
            const int sl = tok ? slot1 : slot0;
            if (sl < 0) continue;
            const uint4* srcv = reinterpret_cast<const uint4*>(p.v_new + (static_cast<int64_t>(b) * num_new + i0 + tok) * C +
                                                               seg * kVSeg);
            uint4* dst = reinterpret_cast<uint4*>(p.cache.sink_v + (static_cast<int64_t>(b) * p.max_sinks + sl) * C +
                                                  seg * kVSeg);
            for (int j = lane; j < kVSeg / 8; j += 32) dst[j] = __ldg(srcv + j);
        }
        if (!SH) __syncwarp();  // the row is rewritten by the next sub-item
    }
}

// Fused-frame append (the reference's own deployment frame).
// With fuse_weights (proj/src/pipeline.cpp:88-99) the projections emit
// K' = P H_G k and V' = H_128 v directly and LayerKVCache::append
// (proj/src/kv_cache.cpp:8-22, called at proj/src/pipeline.cpp:171-176 and
// :207-209) only quantizes them.  No rotation and no reorder, so a warp owns
// a 1024-slot segment of a token pair of K' or V' outright.  Each lane's 32
// slots of both tokens are copied by the warp with coalesced 16-byte
// cp.async into padded per-lane runs (conflict-free LDS.128 afterwards),
// double-buffered so the next sub-item streams in while this one is
// quantized; then quantize_run (the exact thresholds of the other kernels:
// codes bit-identical to rkv_quantize_kv's when K'/V' are the fp32 rows it
// forms) and the packed words and metadata out.  Sub-item = ((sequence,
// token pair, segment), K or V).  Sink tokens get zero words/meta and the K
// sub-item of segment 0 owns their mask bits; their sidecar rows come from
// fused_sink_rows_kernel (below).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// one lane's 32-slot run of both tokens (fp32 rows; padded runs in shared memory) -> float2 per slot
__device__ __forceinline__ void read_run(const float* r0, const float* r1, float2 (&x)[32]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint4 a = lds128(r0 + 4 * q), b = lds128(r1 + 4 * q);
        x[4 * q] = make_float2(__uint_as_float(a.x), __uint_as_float(b.x));
        x[4 * q + 1] = make_float2(__uint_as_float(a.y), __uint_as_float(b.y));
        x[4 * q + 2] = make_float2(__uint_as_float(a.z), __uint_as_float(b.z));
        x[4 * q + 3] = make_float2(__uint_as_float(a.w), __uint_as_float(b.w));
    }
}

// fp16 rows: quantize_run straight from the padded shared-memory run in two
// passes (min/max, then the codes), 8 slots of both tokens live at a time
// instead of 32 -- the same arithmetic, a third of the registers
template <int FMT>
__device__ __forceinline__ QuantOut quantize_run_h(const uint16_t* r0, const uint16_t* r1, int lane) {
    auto chunk = [&](int q, float2 (&x)[8]) {
        const uint4 a = lds128(r0 + 8 * q), b = lds128(r1 + 8 * q);
        const uint16_t* ha = reinterpret_cast<const uint16_t*>(&a);
        const uint16_t* hb = reinterpret_cast<const uint16_t*>(&b);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = make_float2(h2f(ha[e]), h2f(hb[e]));
    };
    float2 x[8];
    chunk(0, x);
    float mn0 = x[0].x, mx0 = x[0].x, mn1 = x[0].y, mx1 = x[0].y;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q) chunk(q, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            mn0 = fminf(mn0, x[e].x);
            mx0 = fmaxf(mx0, x[e].x);
            mn1 = fminf(mn1, x[e].y);
            mx1 = fmaxf(mx1, x[e].y);
        }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, o));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const bool odd = lane & 1;
    const GroupQuant gq = group_params<FMT>(odd ? mn1 : mn0, odd ? mx1 : mx0);
    const int l0 = lane & ~3;
    const float2 n1 = make_float2(-__shfl_sync(0xffffffffu, gq.t1, l0), -__shfl_sync(0xffffffffu, gq.t1, l0 + 1));
    const float2 n2 = make_float2(-__shfl_sync(0xffffffffu, gq.t2, l0), -__shfl_sync(0xffffffffu, gq.t2, l0 + 1));
    const float2 n3 = make_float2(-__shfl_sync(0xffffffffu, gq.t3, l0), -__shfl_sync(0xffffffffu, gq.t3, l0 + 1));
    QuantOut o;
    o.meta = gq.meta;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float2 xb[8];
        chunk(2 * h, x);
        chunk(2 * h + 1, xb);
        o.w[0][h] = ~__byte_perm(code_bits8<0>(x, n1, n2, n3), code_bits8<0>(xb, n1, n2, n3), 0x5410);
        o.w[1][h] = ~__byte_perm(code_bits8<1>(x, n1, n2, n3), code_bits8<1>(xb, n1, n2, n3), 0x5410);
    }
    return o;
}

constexpr int kFusedSeg = 1024;  // slots per warp sub-item
template <typename IN>
struct FusedStage {
    static constexpr int run = 32 * static_cast<int>(sizeof(IN));  // bytes of one lane's 32 slots
    static constexpr int stride = run + 16;                         // padded: conflict-free LDS.128
    static constexpr int chunks = run / 16;
    static constexpr int buf = 2 * 32 * stride;                     // both tokens
    static constexpr int warp_bytes = 2 * buf;                      // double-buffered
};
constexpr int kFusedWarps = 4;
#ifndef RKV_FUSED_F16_CTAS
#define RKV_FUSED_F16_CTAS 5  // resident CTAs per SM for fp16 rows (fp32 rows: 3, the shared memory)
#endif

template <int FMT, typename IN>
__global__ void __launch_bounds__(32 * kFusedWarps, sizeof(IN) == 4 ? 3 : RKV_FUSED_F16_CTAS) quantize_fused_kernel(QuantParams p, const IN* __restrict__ kf,
                                                                            const IN* __restrict__ vf,
                                                                            uint32_t subitems, uint32_t npairs,
                                                                            uint32_t nseg) {
    using S = FusedStage<IN>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * kFusedWarps + warp, step = gridDim.x * kFusedWarps;
    const int C = p.C, W = C / 16, MG = C / kQuantGroup;
    const int num_new = static_cast<int>(p.num_new);
    const uint32_t wbase = smem_u32(smem) + static_cast<uint32_t>(warp * S::warp_bytes);
    // sub-item si = ((b npairs + ip) nseg + seg) 2 + isv; a warp's sub-items
    // advance by `step`: cursors carry (b, ip, seg, isv) forward with compares
    // instead of divisions (as quantize_v_kernel)
    struct Sub {
        uint32_t b, ip, seg, isv;
    };
    auto locate = [&](uint32_t si) {
        const uint32_t rest = si >> 1, pr = udiv32(rest, nseg), bb = udiv32(pr, npairs);
        return Sub{bb, pr - bb * npairs, rest - pr * nseg, si & 1u};
    };
    const Sub dstep = locate(step);
    auto advance = [&](Sub& c) {
        c.isv += dstep.isv;
        const uint32_t c0 = c.isv >> 1;
        c.isv &= 1u;
        c.seg += dstep.seg + c0;
        const uint32_t c1 = c.seg >= nseg ? 1u : 0u;
        c.seg -= c1 * nseg;
        c.ip += dstep.ip + c1;
        const uint32_t c2 = c.ip >= npairs ? 1u : 0u;
        c.ip -= c2 * npairs;
        c.b += dstep.b + c2;
    };
    // chunk c of the segment (16 bytes, coalesced over the warp) -> run c / chunks, part c % chunks
    auto issue = [&](const Sub& u, int buf) {
        const int seg = static_cast<int>(u.seg), i0 = static_cast<int>(u.ip) * 2;
        const int live = min(kFusedSeg, C - seg * kFusedSeg) * static_cast<int>(sizeof(IN)) / 16;
        const uint8_t* src = reinterpret_cast<const uint8_t*>((u.isv ? vf : kf) +
                                                              (static_cast<int64_t>(u.b) * num_new + i0) * C +
                                                              seg * kFusedSeg);
        const uint32_t dst = wbase + static_cast<uint32_t>(buf * S::buf);
        const bool has1 = i0 + 1 < num_new;
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {
            const uint8_t* st = tok && has1 ? src + static_cast<int64_t>(C) * sizeof(IN) : src;
#pragma unroll
            for (int j = 0; j < S::chunks; ++j) {
                const int c = j * 32 + lane;
                if (c < live)
                    cp_async16(dst + static_cast<uint32_t>(tok * 32 * S::stride + (c / S::chunks) * S::stride +
                                                           (c % S::chunks) * 16),
                               st + c * 16);
            }
        }
        cp_async_commit();
    };
    Sub cur = locate(gw), nxt = locate(gw + step);  // this sub-item, the one whose copies we issue next
    if (gw < subitems) issue(cur, 0);
    int buf = 0;
    for (uint32_t si = gw; si < subitems; si += step, buf ^= 1, advance(cur), advance(nxt)) {
        if (si + step < subitems) issue(nxt, buf ^ 1);
        else cp_async_commit();  // an empty group keeps wait_group 1 meaning "this sub-item's copies"
        const Sub& c = cur;
        const int b = static_cast<int>(c.b), seg = static_cast<int>(c.seg), i0 = static_cast<int>(c.ip) * 2;
        const bool isv = c.isv != 0u, has1 = i0 + 1 < num_new;
        const int s0 = seg * kFusedSeg + 32 * lane;
        const bool act = s0 < C;  // C % 128 == 0: a 4-lane group is live or idle as a whole
        const int64_t pos0 = p.start_pos[b] + i0;
        const uint8_t flag = lane < 2 && p.sink_flags && i0 + lane < num_new
                                 ? p.sink_flags[static_cast<int64_t>(b) * num_new + i0 + lane]
                                 : uint8_t{0};
        cp_async_wait1();
        __syncwarp();  // every lane's copies of this buffer have landed
        // (the buffer is refilled by the next iteration's issue: __syncwarp once it is read)
        const QuantOut qo = [&]() -> QuantOut {
            const uint8_t* rb = smem + warp * S::warp_bytes + buf * S::buf + lane * S::stride;
            if constexpr (sizeof(IN) == 2) {
                const QuantOut r = quantize_run_h<FMT>(reinterpret_cast<const uint16_t*>(rb),
                                                       reinterpret_cast<const uint16_t*>(rb + 32 * S::stride), lane);
                __syncwarp();
                return r;
            } else {
                float2 x[32];
                read_run(reinterpret_cast<const IN*>(rb), reinterpret_cast<const IN*>(rb + 32 * S::stride), x);
                __syncwarp();
                return quantize_run<FMT>(x, lane);
            }
        }();
        int slot = -1;  // the sidecar slot rule of the other quantize kernels
        if (flag && pos0 + lane >= 0 && pos0 + lane < p.max_tokens) {
            const int i = i0 + lane;
            int before = 0;
            for (int q = 0; q < i; ++q) before += p.sink_flags[static_cast<int64_t>(b) * num_new + q] ? 1 : 0;
            slot = p.cache.sink_count[b] + before;
            if (slot >= p.max_sinks) slot = -1;
        }
        const int slot0 = __shfl_sync(0xffffffffu, slot, 0), slot1 = __shfl_sync(0xffffffffu, slot, 1);
        uint32_t* codes = isv ? p.cache.v_codes : p.cache.k_codes;
        uint32_t* mt = isv ? p.cache.v_meta : p.cache.k_meta;
        const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens + pos0;
#pragma unroll
        for (int tok = 0; tok < 2; ++tok) {
            if (tok == 1 && !has1) break;
            if (pos0 + tok < 0 || pos0 + tok >= p.max_tokens) break;  // past the cache: never written
            const bool sink = (tok ? slot1 : slot0) >= 0;
            const int64_t rowi = row0 + tok;
            if (act) {
                *reinterpret_cast<uint2*>(codes + rowi * W + s0 / 16) =
                    sink ? make_uint2(0u, 0u) : make_uint2(qo.w[tok][0], qo.w[tok][1]);
                if ((lane & 3) == tok) mt[rowi * MG + s0 / kQuantGroup] = sink ? 0u : qo.meta;
            }
        }
        // per-token sink bits: the K sub-item of segment 0
        if (!isv && seg == 0 && lane < 2 && (lane == 0 || has1)) {
            const int64_t pos = pos0 + lane;
            if (pos >= 0 && pos < p.max_tokens) {
                uint32_t* mw = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32) + (pos >> 5);
                const uint32_t bit = 1u << (pos & 31);
                if (slot >= 0) atomicOr(mw, bit);
                else atomicAnd(mw, ~bit);
            }
        }
    }
}

template <int FMT, typename IN>
cudaError_t launch_quantize_fused_t(const QuantParams& p, int B, const IN* kf, const IN* vf, cudaStream_t s) {
    const int64_t npairs = (p.num_new + 1) / 2, nseg = (p.C + kFusedSeg - 1) / kFusedSeg;
    const int64_t sub = 2 * static_cast<int64_t>(B) * npairs * nseg;
    if (sub >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
    const size_t smem = static_cast<size_t>(kFusedWarps) * FusedStage<IN>::warp_bytes;
    cudaError_t e = ensure_smem_k(quantize_fused_kernel<FMT, IN>, smem);
    if (e != cudaSuccess) return e;
    static int per_sm = 0;
    if (per_sm == 0) {
        int n = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, quantize_fused_kernel<FMT, IN>, 32 * kFusedWarps, smem);
        if (e != cudaSuccess) return e;
        per_sm = n > 0 ? n : 1;
    }
    const int64_t grid =
        std::min<int64_t>(static_cast<int64_t>(num_sms()) * per_sm, (sub + kFusedWarps - 1) / kFusedWarps);
    quantize_fused_kernel<FMT, IN><<<static_cast<unsigned>(grid), 32 * kFusedWarps, smem, s>>>(
        p, kf, vf, static_cast<uint32_t>(sub), static_cast<uint32_t>(npairs), static_cast<uint32_t>(nseg));
    return cudaGetLastError();
}

// Sidecar rows of sink tokens appended in the fused frame
// (rkv_quantize_kv_fused).  The reference's sidecar keeps the fused-frame fp32
// row (proj/src/kv_cache.cpp:8-22); this cache's sidecar keeps the model-frame
// fp16 row (decode applies RoPE to it directly), so K' goes back through the
// inverse reorder (channel perm[j] <- slot j) and H_G, V' through H_128 (each
// an involution after its 1/sqrt(n)), rounded once to fp16.  One CTA per
// sequence walks its flagged tokens in order (ballot ranks) and applies the
// quantize kernels' slot rule.
constexpr int kSinkThreads = 256;
// radix-2 FWHT of every n-channel unit of a shared-memory row (any n; the
// sidecar rows need no particular stage order: they are rounded to fp16)
__device__ __forceinline__ void fwht_row_smem(float* row, int C, int n) {
    for (int half = 1; half < n; half <<= 1) {
        for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {
            const int lo = (i / half) * 2 * half + i % half;
            const float a = row[lo], b = row[lo + half];
            row[lo] = a + b;
            row[lo + half] = a - b;
        }
        __syncthreads();
    }
}
__device__ __forceinline__ float load_row_elem(const float* r, int64_t i) { return r[i]; }
__device__ __forceinline__ float load_row_elem(const uint16_t* r, int64_t i) { return h2f(r[i]); }

template <typename IN>
__global__ void __launch_bounds__(kSinkThreads) fused_sink_rows_kernel(QuantParams p, const IN* __restrict__ kf,
                                                                    const IN* __restrict__ vf, int nk) {
    extern __shared__ __align__(16) float srow[];  // [C]
    __shared__ int s_list[kSinkThreads];
    __shared__ int s_wcnt[kSinkThreads / 32];
    const int b = blockIdx.x, C = p.C, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int num_new = static_cast<int>(p.num_new);
    const int count = p.cache.sink_count[b];
    int before = 0;  // flagged tokens of earlier chunks
    for (int c0 = 0; c0 < num_new; c0 += kSinkThreads) {
        const int i = c0 + tid;
        const bool f = i < num_new && p.sink_flags[static_cast<int64_t>(b) * num_new + i];
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();
        int rank = __popc(bal & ((1u << lane) - 1u)), total = 0;
        for (int w = 0; w < kSinkThreads / 32; ++w) {
            rank += w < warp ? s_wcnt[w] : 0;
            total += s_wcnt[w];
        }
        if (f) s_list[rank] = i;
        __syncthreads();
        for (int e = 0; e < total; ++e) {
            const int ti = s_list[e];
            const int64_t pos = p.start_pos[b] + ti;
            const int slot = count + before + e;
            if (pos < 0 || pos >= p.max_tokens || slot >= p.max_sinks) continue;  // uniform over the CTA
            const int64_t src = (static_cast<int64_t>(b) * num_new + ti) * C;
            const int64_t dst = (static_cast<int64_t>(b) * p.max_sinks + slot) * C;
            for (int j = tid; j < C; j += blockDim.x) srow[p.perm[j]] = load_row_elem(kf, src + j);
            __syncthreads();
            fwht_row_smem(srow, C, nk);
            for (int c = tid; c < C; c += blockDim.x)
                p.cache.sink_k[dst + c] = __half_as_ushort(__float2half_rn(__fmul_rn(srow[c], p.k_norm)));
            __syncthreads();
            for (int c = tid; c < C; c += blockDim.x) srow[c] = load_row_elem(vf, src + c);
            __syncthreads();
            fwht_row_smem(srow, C, kHeadDim);
            for (int c = tid; c < C; c += blockDim.x)
                p.cache.sink_v[dst + c] = __half_as_ushort(__float2half_rn(__fmul_rn(srow[c], p.v_norm)));
            if (tid == 0) p.cache.sink_pos[b * p.max_sinks + slot] = static_cast<int32_t>(pos);
            __syncthreads();
        }
        before += total;
        __syncthreads();  // s_wcnt / s_list reused
    }
}

// Sink counts for the appended tokens (only launched with sink flags; it runs
// after every item has read the old count).
__global__ void quantize_sink_count_kernel(QuantParams p) {
    const int b = blockIdx.x;
    __shared__ int s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int local = 0;
    for (int64_t i = threadIdx.x; i < p.num_new; i += blockDim.x) {
        const int64_t pos = p.start_pos[b] + i;
        if (pos >= 0 && pos < p.max_tokens && p.sink_flags[b * p.num_new + i]) ++local;
    }
    if (local) atomicAdd(&s_count, local);
    __syncthreads();
    // the main kernel gave sidecar slots to the first (max_sinks - count) of them only
    if (threadIdx.x == 0 && s_count) {
        const int c = p.cache.sink_count[b];
        p.cache.sink_count[b] = c + min(s_count, max(0, p.max_sinks - c));
    }
}

// promote_to_sink / route_sinks (proj/src/kv_cache.cpp:43-55,
// proj/src/sink.cpp:47-63): one CTA per sequence.  Thread 0 walks the
// sequence's token list in order (deterministic slots): tokens out of
// [0, max_tokens), already sinks (the reference returns early: idempotent,
// also for duplicates in the list) or past a full sidecar are skipped; the
// others get the next sidecar slot, their mask bit and sink_pos.  Then the
// CTA copies the raw fp16 rows into the sidecar and zeroes the token's packed
// words and metadata (the reference clears its blocks).
constexpr int kPromoteMax = 256;  // tokens per sequence and call
__global__ void promote_sinks_kernel(QuantParams p, const int64_t* __restrict__ tokens, int n,
                                     int32_t* __restrict__ promoted) {
    __shared__ int s_slot[kPromoteMax];
    __shared__ int64_t s_tok[kPromoteMax];
    const int b = blockIdx.x, C = p.C, W = C / 16, MG = C / kQuantGroup;
    const int64_t mwords = (p.max_tokens + 31) / 32;
    uint32_t* mask = p.cache.sink_mask + static_cast<int64_t>(b) * mwords;
    if (threadIdx.x == 0) {
        int cnt = p.cache.sink_count[b], np = 0;  // np: promoted by this call
        for (int i = 0; i < n; ++i) {
            const int64_t t = tokens[static_cast<int64_t>(b) * n + i];
            s_slot[i] = -1;
            if (t < 0 || t >= p.max_tokens) continue;
            const uint32_t bit = 1u << (t & 31);
            if (mask[t >> 5] & bit) continue;  // already a sink
            if (cnt >= p.max_sinks) continue;  // sidecar full: stays quantized
            mask[t >> 5] |= bit;
            p.cache.sink_pos[b * p.max_sinks + cnt] = static_cast<int32_t>(t);
            s_slot[i] = cnt++;
            s_tok[i] = t;
            ++np;
        }
        p.cache.sink_count[b] = cnt;
        if (promoted) promoted[b] = np;
    }
    __syncthreads();
    for (int i = 0; i < n; ++i) {
        const int slot = s_slot[i];
        if (slot < 0) continue;
        const int64_t t = s_tok[i];
        const int64_t src = (static_cast<int64_t>(b) * n + i) * C;
        const int64_t dst = (static_cast<int64_t>(b) * p.max_sinks + slot) * C;
        for (int j = threadIdx.x; j < C; j += blockDim.x) {
            p.cache.sink_k[dst + j] = p.k_new[src + j];
            p.cache.sink_v[dst + j] = p.v_new[src + j];
        }
        const int64_t row = static_cast<int64_t>(b) * p.max_tokens + t;
        for (int j = threadIdx.x; j < W; j += blockDim.x) {
            p.cache.k_codes[row * W + j] = 0u;
            p.cache.v_codes[row * W + j] = 0u;
        }
        for (int j = threadIdx.x; j < MG; j += blockDim.x) {
            p.cache.k_meta[row * MG + j] = 0u;
            p.cache.v_meta[row * MG + j] = 0u;
        }
    }
}

template <int N, int FMT, int NS>
cudaError_t launch_quantize_ns(const QuantParams& p, int B, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(p.C / 32) * 33 * 8 + static_cast<size_t>(p.C) * (2 + 4 * NS);
    static int per_sm_cache[9] = {0};  // keyed by C / 1024 (C <= 8192)
    int& per_sm = per_sm_cache[p.C / 1024];
    const int threads = (p.C / 32 + 31) / 32 * 32;
    {
        const cudaError_t e = ensure_smem_k(quantize_kv_kernel<N, FMT, NS>, smem);
        if (e != cudaSuccess) return e;
    }
    if (per_sm == 0) {
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, quantize_kv_kernel<N, FMT, NS>, threads, smem);
        if (e != cudaSuccess) return e;
        if (n < 1) return cudaErrorInvalidConfiguration;
        per_sm = n;
    }
    const int64_t npairs = (p.num_new + 1) / 2;
    QuantParams pk = p;
    // V on the warp-independent kernel when the row splits into 1024-channel segments
    // (only when there are at least as many V segments as the V kernel has warps:
    // a decode step's one-token append stays one launch)
    const bool vsplit = p.C % kVSeg == 0 && options().quant_vsplit.load() != 0 &&
                        static_cast<int64_t>(B) * npairs * (p.C / kVSeg) >= static_cast<int64_t>(num_sms()) * 12;
    if (vsplit) {
        const int64_t nseg = p.C / kVSeg, sub = static_cast<int64_t>(B) * npairs * nseg;
        if (sub >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
        auto launch_v = [&](auto kern, int vw, size_t wb) -> cudaError_t {
            const size_t vsmem = static_cast<size_t>(vw) * wb;
            cudaError_t e = ensure_smem_k(kern, vsmem);
            if (e != cudaSuccess) return e;
            const int64_t vgrid = std::min<int64_t>(num_sms(), (sub + vw - 1) / vw);
            kern<<<static_cast<unsigned>(vgrid), 32 * vw, vsmem, s>>>(p, static_cast<uint32_t>(sub),
                                                                       static_cast<uint32_t>(npairs),
                                                                       static_cast<uint32_t>(nseg));
            return cudaGetLastError();
        };
        // shapes (warps x TMA stages per warp): 0 = 16 x 2 with the shuffle
        // stages (no row buffer), 1 = 16 x 1, 2 = 14 x 1, 3 = 12 x 2 with the row
        // buffer, 4 = 20 x 2 with the shuffle stages
        const int vcfg = options().quant_vcfg.load();
        cudaError_t e = vcfg == 1   ? launch_v(quantize_v_kernel<FMT, 16, 1>, 16, VCfg<16, 1>::warp_bytes)
                        : vcfg == 2 ? launch_v(quantize_v_kernel<FMT, 14, 1>, 14, VCfg<14, 1>::warp_bytes)
                        : vcfg == 3 ? launch_v(quantize_v_kernel<FMT, 12, 2>, 12, VCfg<12, 2>::warp_bytes)
                        : vcfg == 4 ? launch_v(quantize_v_kernel<FMT, 20, 2, true>, 20, VCfg<20, 2, true>::warp_bytes)
                                    : launch_v(quantize_v_kernel<FMT, 16, 2, true>, 16, VCfg<16, 2, true>::warp_bytes);
        if (e != cudaSuccess) return e;
        pk.k_only = 1;
    }
    const int64_t items = (vsplit ? 1 : 2) * static_cast<int64_t>(B) * npairs;
    if (items >= (int64_t{1} << 30)) return cudaErrorInvalidValue;
    int64_t grid = static_cast<int64_t>(num_sms()) * per_sm;
    if (grid > items) grid = items;
    cudaError_t e;
    if (vsplit) {  // programmatic dependent of the V kernel: starts in its tail (no data dependency)
        e = launch_pdl(quantize_kv_kernel<N, FMT, NS>, dim3(static_cast<unsigned>(grid)), dim3(threads), smem, s, pk,
                       static_cast<uint32_t>(items), static_cast<uint32_t>(npairs));
    } else {
        quantize_kv_kernel<N, FMT, NS><<<static_cast<unsigned>(grid), threads, smem, s>>>(
            pk, static_cast<uint32_t>(items), static_cast<uint32_t>(npairs));
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    if (!p.sink_flags) return cudaSuccess;
    quantize_sink_count_kernel<<<B, 256, 0, s>>>(p);
    return cudaGetLastError();
}

template <int N, int FMT>
cudaError_t launch_quantize_n(const QuantParams& p, int B, cudaStream_t s) {
    return options().quant_stages.load() == 2 ? launch_quantize_ns<N, FMT, 2>(p, B, s)
                                              : launch_quantize_ns<N, FMT, 1>(p, B, s);
}

template <int N>
cudaError_t launch_quantize_fmt(const QuantParams& p, int B, cudaStream_t s) {
    return p.scale_format == RKV_SCALE_E4M3_CEIL ? launch_quantize_n<N, RKV_SCALE_E4M3_CEIL>(p, B, s)
                                                 : launch_quantize_n<N, RKV_SCALE_FP16_CEIL>(p, B, s);
}

}  // namespace

cudaError_t launch_promote_sinks(const rkv_layer_desc& d, const QuantParams& p, const int64_t* tokens, int n,
                                 int32_t* promoted, cudaStream_t s) {
    if (n < 1 || n > kPromoteMax) return cudaErrorInvalidValue;
    promote_sinks_kernel<<<d.batch, 256, 0, s>>>(p, tokens, n, promoted);
    return cudaGetLastError();
}
int promote_sinks_max() { return kPromoteMax; }

cudaError_t launch_fused_sink_rows(const rkv_layer_desc& d, const QuantParams& p, const void* k_rows,
                                   const void* v_rows, int dtype, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(p.C) * sizeof(float);
    const int nk = d.heads_per_group * d.head_dim;
    if (dtype == RKV_ROWS_F16) {
        auto kern = fused_sink_rows_kernel<uint16_t>;
        cudaError_t e = ensure_smem_k(kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<d.batch, kSinkThreads, smem, s>>>(p, static_cast<const uint16_t*>(k_rows),
                                                static_cast<const uint16_t*>(v_rows), nk);
    } else {
        auto kern = fused_sink_rows_kernel<float>;
        cudaError_t e = ensure_smem_k(kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<d.batch, kSinkThreads, smem, s>>>(p, static_cast<const float*>(k_rows),
                                                static_cast<const float*>(v_rows), nk);
    }
    return cudaGetLastError();
}

cudaError_t launch_quantize_fused(const rkv_layer_desc& d, const QuantParams& p, const void* k_rows,
                                  const void* v_rows, int dtype, cudaStream_t s) {
    cudaError_t e;
    const bool e4 = p.scale_format == RKV_SCALE_E4M3_CEIL;
    if (dtype == RKV_ROWS_F16) {
        const auto* kf = static_cast<const uint16_t*>(k_rows);
        const auto* vf = static_cast<const uint16_t*>(v_rows);
        e = e4 ? launch_quantize_fused_t<RKV_SCALE_E4M3_CEIL>(p, d.batch, kf, vf, s)
               : launch_quantize_fused_t<RKV_SCALE_FP16_CEIL>(p, d.batch, kf, vf, s);
    } else {
        const auto* kf = static_cast<const float*>(k_rows);
        const auto* vf = static_cast<const float*>(v_rows);
        e = e4 ? launch_quantize_fused_t<RKV_SCALE_E4M3_CEIL>(p, d.batch, kf, vf, s)
               : launch_quantize_fused_t<RKV_SCALE_FP16_CEIL>(p, d.batch, kf, vf, s);
    }
    if (e != cudaSuccess || !p.sink_flags) return e;
    if ((e = launch_fused_sink_rows(d, p, k_rows, v_rows, dtype, s)) != cudaSuccess) return e;
    quantize_sink_count_kernel<<<d.batch, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_quantize(const rkv_layer_desc& d, const QuantParams& p, cudaStream_t s) {
    const int n = d.heads_per_group * d.head_dim;
    if (generic_quantize_needed(d) || p.C % 512 != 0) {  // any other power-of-two rotation size (generic.cu)
        cudaError_t e = launch_quantize_generic(d, p, s);
        if (e != cudaSuccess || !p.sink_flags) return e;
        quantize_sink_count_kernel<<<d.batch, 256, 0, s>>>(p);
        return cudaGetLastError();
    }
    switch (n) {
        case 128: return launch_quantize_fmt<128>(p, d.batch, s);
        case 256: return launch_quantize_fmt<256>(p, d.batch, s);
        case 512: return launch_quantize_fmt<512>(p, d.batch, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkv
