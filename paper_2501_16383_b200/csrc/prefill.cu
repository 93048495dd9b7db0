// prefill.cu -- causal attention of a block of queries over the 2-bit rotated
// cache (the attention half of prefill,
// proj/src/pipeline.cpp:156-191: reconstruct_cache, then causal
// reference_attention, proj/src/attention.cpp:20-49).
//
// Four launches, mirroring the reference's decomposition (reconstruct the
// cache, then attend):
//   1. reconstruct_keys_kernel (== reconstruct_cache for K): per token the
//      un-reorder scatter, the tensor-core inverse FWHT of decode_mma.cu (two
//      chained H_16 mma.sync with the fp16 hi/lo split) and RoPE at the
//      token's position, stored as fp16 hi + lo straight into 64-key operand
//      tiles (K-major SWIZZLE_128B).  Every key is reconstructed once.
//   2. reconstruct_values_kernel: the dequantized rotated values, fp16,
//      transposed into the same tiles.
//   3. prepare_queries_kernel: RoPE'd, scaled, hi/lo-split query rows laid out
//      for tensor memory.
//   4. prefill_attn_kernel: flash attention on tcgen05 (section 4 below):
//      S and O accumulate in tensor memory, Q and P are A operands from tensor
//      memory, K/V tiles stream through shared memory by cp.async.bulk; sink
//      rows and V's inverse rotation H_128 are applied in its epilogue.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "rkv_common.cuh"
#include "rkv_internal.h"
#include "rkv_layout.h"
#include "rkv_mma.cuh"
#include "rkv_umma.cuh"

namespace rkv {

namespace {

using namespace mma;

constexpr int kRopeRowF4 = 128;  // float4 per position-pair row of the RoPE table (decode_attention.cu)

__device__ __forceinline__ float2 rope_cs(const float4* t, int64_t pos, int f) {
    const float4 r = __ldg(t + (pos >> 1) * kRopeRowF4 + f);
    return (pos & 1) ? make_float2(r.y, r.w) : make_float2(r.x, r.z);
}

// operand tile of (sequence b, KV head, 64-key tile): K hi slabs [0, 16K),
// K lo slabs [16K, 32K), V^T [32K, 48K)
__device__ __forceinline__ unsigned char* kv_tile(const PrefillParams& p, int b, int kvh, int64_t j) {
    return p.kv_tiles + ((static_cast<int64_t>(b) * p.Hkv + kvh) * p.kv_tiles_per_seq + j) * kPrefillTileBytes;
}

// channels d, d + 1 (d even) of key `pos`, split into fp16 hi + lo, at their
// K-major SWIZZLE_128B position (slab d / 64, row pos % 64)
__device__ __forceinline__ void store_key_pair(const PrefillParams& p, int b, int64_t pos, int kvh, int d, float x0,
                                               float x1) {
    unsigned char* t = kv_tile(p, b, kvh, pos >> 6);
    const uint32_t off = static_cast<uint32_t>(d >> 6) * 8192u + umma::sw128(static_cast<uint32_t>(pos & 63), (d & 63) >> 3) +
                         static_cast<uint32_t>(d & 7) * 2u;
    const uint32_t h = pack_h2(x0, x1);
    *reinterpret_cast<uint32_t*>(t + off) = h;
    *reinterpret_cast<uint32_t*>(t + 16384 + off) = pack_h2(sub_lo(x0, h), sub_hi(x1, h));
}

// ------------------------------------------------------------------ 1. keys
// CTA = (4-token tile, sequence), one warp per FWHT group.
// G = 4: 512-channel tiles (the MHA decode layout; AG = heads per rotation
// group, 4, 2 or 1, picks the second FWHT factor); G = 2: GQA 256-channel groups
// (AG = 1: per-head rotation, H_8 x I_2 over the head bit in the second factor).
// PAIR (GQA at G = 4 on the 256-channel plan, G = 2 here): the group's two
// half-group warps hold u, v = H_256 of their halves (RoPE'd); the keys are
// u + v (KV heads 0, 1) and u - v (heads 2, 3) -- swapped through shared
// memory after all four tokens, one 64-thread named barrier per warp pair.
template <int G, int AG = G, bool PAIR = false>
__global__ void __launch_bounds__(512) reconstruct_keys_kernel(PrefillParams p) {
    constexpr int N = 128 * G, NJ = N / 128, TT = 4;
    static_assert(!PAIR || G == 2, "half-group pairs run on the 256-channel plan");
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_trigger();  // the value and query kernels do not read the keys: let them start in this one's tail
    const int C = p.C, W = C / 16, MG = C / 128, NG = C / N;
    const int b = blockIdx.y, tid = threadIdx.x, NT = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * TT;
    const int64_t T = p.seq_len[b];
    if (t0 >= T) return;
    const int nv = static_cast<int>(lmin64(TT, T - t0));
    const uint32_t pair_bytes = static_cast<uint32_t>(C) * 4u;
    unsigned char* knat = smem;                                             // 2 token-pair rows
    uint32_t* kcs = reinterpret_cast<uint32_t*>(smem + 2 * pair_bytes);    // [TT][W]
    uint32_t* kms = kcs + TT * W;                                           // [TT][MG]
    float4* rps = reinterpret_cast<float4*>(kms + TT * MG);                // [TT][32] RoPE frequency-pair rows
    float4* xk = rps + TT * 32;  // PAIR: [NG warps][TT][2 f1][32 lanes] RoPE'd (ka0, ka1, kb0, kb1)
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens + t0;
    for (int i = tid; i < TT * W; i += NT) kcs[i] = i / W < nv ? p.cache.k_codes[row0 * W + i] : 0u;
    for (int i = tid; i < TT * MG; i += NT) kms[i] = i / MG < nv ? p.cache.k_meta[row0 * MG + i] : 0u;
    for (int i = tid; i < TT * 32; i += NT)  // staged with the codes: no dependent load in the MMA half
        if (i / 32 < nv) rps[i] = __ldg(p.rope + ((t0 + i / 32) >> 1) * kRopeRowF4 + 64 + ((t0 + i / 32) & 1) * 32 + (i & 31));
    __syncthreads();
    // scatter (same plan and arithmetic as the decode kernel): thread = word position(s)
    const uint32_t* plan = p.plan + kPlanHeader;
    auto bexp = [](int sh) -> uint32_t { const uint32_t be = static_cast<uint32_t>(25 - 2 * sh) << 10; return be | (be << 16); };
    for (int item = tid; item < 2 * W; item += NT) {
        const int wp = item % W, pq = item / W, tt0 = 2 * pq;
        const int wsrc = static_cast<int>(__ldg(plan + wp));
        const uint32_t w0 = kcs[tt0 * W + wsrc], w1 = kcs[(tt0 + 1) * W + wsrc];
        const uint32_t m0 = kms[tt0 * MG + (wsrc >> 3)], m1 = kms[(tt0 + 1) * MG + (wsrc >> 3)];
        const uint32_t ss = prmt(m0, m1, 0x5410u), zz = prmt(m0, m1, 0x7632u);
        uint32_t bz[5];
#pragma unroll
        for (int e = 0; e < 5; ++e) bz[e] = h2add(bexp(e), zz);
        const uint32_t xl = prmt(w0, w1, 0x5410u), xh = prmt(w0, w1, 0x7632u);
        const uint32_t xls = xl >> 10, xhs = xh >> 10;
        const uint32_t dst = smem_u32(knat) + static_cast<uint32_t>(pq) * pair_bytes;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int ee = e & 7;
            const uint32_t src = ee < 5 ? (e < 8 ? xl : xh) : (e < 8 ? xls : xhs);
            const int sh = ee < 5 ? ee : ee - 5;
            const uint32_t h = and_or(src, 0x00030003u << (2 * sh), bexp(sh));
            const uint32_t x = h2mul(h2sub(h, bz[sh]), ss);
            const uint32_t ad = __ldg(plan + W + (e / 4) * W * 4 + wp * 4 + e % 4);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(dst + ad), "r"(x) : "memory");
        }
    }
    __syncthreads();
    if (warp >= NG) return;
    const int gam = warp, g = lane >> 2, tl = lane & 3;
    uint32_t AH[4], AF2buf[4];
    hadamard16_frag(AH, lane, static_cast<uint32_t>(p.max_tokens >> 40));
    if constexpr (AG != G) {
        if constexpr (G == 2)  // 256-channel GQA tile at G = 1: H_8 x I_2 over the head bit
            hadamard_mask_frag(AF2buf, lane, 11, static_cast<uint32_t>(p.max_tokens >> 40));
        else
            hadamard_f2_frag<AG>(AF2buf, lane, static_cast<uint32_t>(p.max_tokens >> 40));
    }
    uint32_t(&AF2)[4] = *(AG == G ? &AH : &AF2buf);  // second FWHT factor of the tile
    const float kn = p.k_norm;
    const int swz = mma_swz(N, lane);
    const unsigned char* lbase = knat + gam * N * 4 + lane * NJ * 16;
    for (int pq = 0; pq < 2; ++pq) {
        uint32_t bf[2][NJ][2];
#pragma unroll
        for (int jc = 0; jc < NJ; ++jc) {
            const uint4 u = lds128(lbase + static_cast<size_t>(pq) * pair_bytes + ((jc ^ swz) << 4));
            bf[0][jc][0] = prmt(u.x, u.y, 0x5410u);
            bf[0][jc][1] = prmt(u.z, u.w, 0x5410u);
            bf[1][jc][0] = prmt(u.x, u.y, 0x7632u);
            bf[1][jc][1] = prmt(u.z, u.w, 0x7632u);
        }
#pragma unroll
        for (int tk = 0; tk < 2; ++tk) {
            const int tt = 2 * pq + tk;
            if (tt >= nv) break;
            const int64_t pos = t0 + tt;
            float yf[NJ][4];
            const float zero[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int jc = 0; jc < NJ; ++jc) mma16816(yf[jc], AH, bf[tk][jc][0], bf[tk][jc][1], zero);
            // frequency-pair row of the token (rope section 2): (u,u',w,w') for G = 4, (c,c',s,s') else
            const float4* rrow = rps + tt * 32;
#pragma unroll
            for (int f1 = 0; f1 < 2; ++f1) {
                const int f = 2 * tl + 8 * f1 + 16 * (g & 3);
                const float4 r4 = rrow[rope_pair_slot(f >> 1)];
                if constexpr (G == 4) {
                    float z[2][4];
#pragma unroll
                    for (int o = 0; o < 2; ++o) {
                        const float* ya = yf[2 * o];
                        const float* yb = yf[2 * o + 1];
                        const uint32_t h0 = pack_h2(ya[2 * f1], ya[2 * f1 + 1]);
                        const uint32_t h1 = pack_h2(yb[2 * f1], yb[2 * f1 + 1]);
                        const uint32_t l0 = pack_h2(sub_lo(ya[2 * f1], h0), sub_hi(ya[2 * f1 + 1], h0));
                        const uint32_t l1 = pack_h2(sub_lo(yb[2 * f1], h1), sub_hi(yb[2 * f1 + 1], h1));
                        float t4[4];
                        mma16816(t4, AF2, h0, h1, zero);
                        mma16816(z[o], AF2, l0, l1, t4);
                    }
#pragma unroll
                    for (int rh = 0; rh < 2; ++rh) {
                        const int kvh = gam * G + (g >> 2) + 2 * rh;
                        float ka[2], kb[2];
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const float a = z[0][2 * rh + i], bb = z[1][2 * rh + i];
                            const float u = i ? r4.y : r4.x, w = i ? r4.w : r4.z;
                            ka[i] = (a * u + bb * w) * kn;  // RoPE(H_2 (a', b')) channel f
                            kb[i] = (a * w - bb * u) * kn;  // channel f + 64
                        }
                        store_key_pair(p, b, pos, kvh, f, ka[0], ka[1]);
                        store_key_pair(p, b, pos, kvh, f + 64, kb[0], kb[1]);
                    }
                } else {
                    const uint32_t h0 = pack_h2(yf[0][2 * f1], yf[0][2 * f1 + 1]);
                    const uint32_t h1 = pack_h2(yf[1][2 * f1], yf[1][2 * f1 + 1]);
                    const uint32_t l0 = pack_h2(sub_lo(yf[0][2 * f1], h0), sub_hi(yf[0][2 * f1 + 1], h0));
                    const uint32_t l1 = pack_h2(sub_lo(yf[1][2 * f1], h1), sub_hi(yf[1][2 * f1 + 1], h1));
                    float t4[4], z[4];
                    mma16816(t4, AF2, h0, h1, zero);
                    mma16816(z, AF2, l0, l1, t4);
                    const int kvh = gam * G + (g >> 2);
                    float ka[2], kb[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const float a = z[i], bb = z[2 + i];  // channels f+i and f+64+i
                        const float c = i ? r4.y : r4.x, s = i ? r4.w : r4.z;
                        ka[i] = (a * c - bb * s) * kn;
                        kb[i] = (a * s + bb * c) * kn;
                    }
                    if constexpr (PAIR) {
                        xk[((warp * TT + tt) * 2 + f1) * 32 + lane] = make_float4(ka[0], ka[1], kb[0], kb[1]);
                    } else {
                        store_key_pair(p, b, pos, kvh, f, ka[0], ka[1]);
                        store_key_pair(p, b, pos, kvh, f + 64, kb[0], kb[1]);
                    }
                }
            }
        }
    }
    if constexpr (PAIR) {  // lower half: u + v -> KV heads 0, 1; upper half: u - v -> heads 2, 3
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
        const bool upper = gam & 1;
        const int kvh = gam * G + (g >> 2);
        for (int tt = 0; tt < nv; ++tt) {
#pragma unroll
            for (int f1 = 0; f1 < 2; ++f1) {
                const float4 own = xk[((warp * TT + tt) * 2 + f1) * 32 + lane];
                const float4 oth = xk[(((warp ^ 1) * TT + tt) * 2 + f1) * 32 + lane];
                const float4 k4 = upper ? make_float4(oth.x - own.x, oth.y - own.y, oth.z - own.z, oth.w - own.w)
                                        : make_float4(own.x + oth.x, own.y + oth.y, own.z + oth.z, own.w + oth.w);
                const int f = 2 * tl + 8 * f1 + 16 * (g & 3);
                store_key_pair(p, b, t0 + tt, kvh, f, k4.x, k4.y);
                store_key_pair(p, b, t0 + tt, kvh, f + 64, k4.z, k4.w);
            }
        }
    }
}

// ---------------------------------------------------------------- 2. values
// V^T tile of (sequence, KV head, 64 keys): the dequantized rotated values
// s (c - z), rounded once to fp16 (the decode kernels' operand rounding),
// [128 channels][64 keys] K-major SWIZZLE_128B; keys >= seq_len are zero.
// Thread t: code word w = t >> 4 (channels 16w..16w+15), keys 8kc..8kc+7
// (kc = (t >> 1) & 7), codes 8 (t & 1) .. + 7 of the word.
__global__ void __launch_bounds__(128) reconstruct_values_kernel(PrefillParams p) {
    pdl_trigger();
    const int64_t j = blockIdx.x;
    const int kvh = blockIdx.y, b = blockIdx.z, t = threadIdx.x;
    const int W = p.C / 16, MG = p.C / 128;
    const int w = t >> 4, kc = (t >> 1) & 7, e0 = 8 * (t & 1);
    const int64_t T = p.seq_len[b], row0 = static_cast<int64_t>(b) * p.max_tokens;
    uint32_t cw[8];
    float sc[8], zr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t key = j * kPrefillKT + 8 * kc + i;
        const bool ok = key < T;
        cw[i] = ok ? __ldg(p.cache.v_codes + (row0 + key) * W + kvh * 8 + w) : 0u;
        const uint32_t m = ok ? __ldg(p.cache.v_meta + (row0 + key) * MG + kvh) : 0u;
        sc[i] = h2f(static_cast<uint16_t>(m & 0xffffu));
        zr[i] = h2f(static_cast<uint16_t>(m >> 16));
    }
    unsigned char* vt = kv_tile(p, b, kvh, j) + 32768;
#pragma unroll
    for (int e = e0; e < e0 + 8; ++e) {
        uint32_t h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float c0 = static_cast<float>((cw[2 * i] >> (2 * e)) & 3u), c1 = static_cast<float>((cw[2 * i + 1] >> (2 * e)) & 3u);
            h[i] = pack_h2(sc[2 * i] * (c0 - zr[2 * i]), sc[2 * i + 1] * (c1 - zr[2 * i + 1]));
        }
        *reinterpret_cast<uint4*>(vt + umma::sw128(static_cast<uint32_t>(16 * w + e), static_cast<uint32_t>(kc))) =
            make_uint4(h[0], h[1], h[2], h[3]);
    }
    pdl_wait();  // this grid completes only after the key kernel (the attention kernel waits on the chain)
}

// --------------------------------------------------------------- 3. queries
// Query rows, staged once for every (head, 128-row block) CTA: RoPE at the
// row's position, x log2(e)/sqrt(d), split into fp16 hi + lo and written as
// the 512-byte TMEM-ready row the attention kernel bulk-copies (u32 u =
// dims (2u, 2u + 1) of hi for u < 64, of lo for u >= 64; 16-byte chunk c
// stored at c ^ (row & 31) so the per-row shared-memory reads do not
// conflict).  Warp = (sequence, query row, 4 heads); lane = frequencies
// 2 lane, 2 lane + 1; padding rows (>= num_q) are zero.
__global__ void __launch_bounds__(128) prepare_queries_kernel(PrefillParams p) {
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x;
    const int b = blockIdx.z, h0 = (blockIdx.y * 4 + warp) * 4;
    if (h0 >= p.Hq) return;
    const bool live = i < p.num_q;
    const int f = 2 * lane;
    float cs[2] = {0.f, 0.f}, sn[2] = {0.f, 0.f};
    if (live) {
        const int64_t pos = p.q_start[b] + i;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float2 r = rope_cs(p.rope, pos, f + k);
            cs[k] = r.x;
            sn[k] = r.y;
        }
    }
    const uint32_t sw = static_cast<uint32_t>(i & 31);
    auto put = [&](uint32_t* row, uint32_t u, uint32_t v) { row[((((u >> 2) ^ sw) & 31u) << 2) | (u & 3u)] = v; };
    // the 4 heads' query words, requested together before any store
    uint32_t qw[4][2] = {};
    if (live)
#pragma unroll
        for (int hh = 0; hh < 4; ++hh)
            if (h0 + hh < p.Hq) {
                const uint32_t* qr = reinterpret_cast<const uint32_t*>(
                    p.q + ((static_cast<int64_t>(b) * p.num_q + i) * p.Hq + h0 + hh) * 128);
                qw[hh][0] = __ldg(qr + lane);
                qw[hh][1] = __ldg(qr + 32 + lane);
            }
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
        const int h = h0 + hh;
        if (h >= p.Hq) break;
        float qa[2] = {0.f, 0.f}, qv[2] = {0.f, 0.f};
        if (live) {
            const uint32_t wa = qw[hh][0], wb = qw[hh][1];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const float a = h2f(static_cast<uint16_t>(k ? wa >> 16 : wa & 0xffffu));
                const float bb = h2f(static_cast<uint16_t>(k ? wb >> 16 : wb & 0xffffu));
                qa[k] = (a * cs[k] - bb * sn[k]) * p.qscale;
                qv[k] = (a * sn[k] + bb * cs[k]) * p.qscale;
            }
        }
        uint32_t* row = reinterpret_cast<uint32_t*>(p.q_rows + ((static_cast<int64_t>(b) * p.Hq + h) * p.num_q_pad + i) * 512);
        const uint32_t ha = pack_h2(qa[0], qa[1]), hb = pack_h2(qv[0], qv[1]);
        put(row, lane, ha);
        put(row, 32 + lane, hb);
        put(row, 64 + lane, pack_h2(sub_lo(qa[0], ha), sub_hi(qa[1], ha)));
        put(row, 96 + lane, pack_h2(sub_lo(qv[0], hb), sub_hi(qv[1], hb)));
    }
    pdl_wait();  // completes only after the value kernel (and through it the key kernel)
}

// ------------------------------------------------------------- 4. attention
// Flash attention on the 5th-generation tensor cores.  CTA = (sequence, q
// head, 128 query rows); 12 warps: warp 0 bulk-copies the staged query block
// and streams the key tiles (cp.async.bulk, 3 deep), warp 3 streams the
// value tiles (2 deep), warp 1 (one elected lane) issues tcgen05.mma, warp 2
// stages the sink rows, and two softmax groups of 4 warps (one query row
// per thread, TMEM lane = row) take the 64-key tiles in turn: group X owns
// the tiles j = X mod 2, its score buffer S_X and its own output
// accumulator O_X and running (m, l), merged in the epilogue.  Per tile j:
//   S_X = Qhi Khi^T + Qhi Klo^T + Qlo Khi^T   (M = 128, N = 64, 3 x 8 K-steps;
//     ~2^-22 relative, Q hi / lo read from tensor memory),
//   softmax: causal / length / sink mask, running max with lazy rescale (O_X
//     rescaled in place only when the row max grows by more than 2^14),
//     P = 2^(S - m) as fp16 pairs written over the first 32 columns of S_X,
//   O_X += P V_j   (M = 128, N = 128, 4 K-steps, P read from tensor memory).
// The MMA lane issues PV(j) and then QK(j + 2) into the same S_X: tcgen05
// operations of one thread execute in order, so the scores of j + 2 never
// overwrite P_j before PV(j) read it, and S(j) being complete implies PV(j - 2)
// is, so O_X can be rescaled without waiting.  While group X runs its
// softmax the tensor core works on the other group's tile.  Shared memory
// only carries the K / V tiles.  Every hand-off is an mbarrier (TMA
// transaction bytes, tcgen05.commit, or thread arrivals).
// Epilogue (the reference's exact sink rows, as decode_combine_kernel): the
// row's sink logits q . RoPE(k_s) join the merged (m, l);
// out = (H_128 O / sqrt(128) * 2^(m - M) + sum_s 2^(e_s - M) v_s) / L, where
// group X produces output dims [64 X, 64 X + 64) through H_128 = H_2 (x) H_64.
#ifdef RKV_PF_TRACE
// development trace (build with RKV_NVCC_EXTRA=-DRKV_PF_TRACE): SM clock at
// per-tile hand-off events of CTA (0, 0, 0), read back by rkv_debug_prefill_trace
__device__ long long g_pf_trace[8][256];
__device__ unsigned long long g_pf_cta[4096][4];  // %globaltimer: start, q staged, last P, end
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PF_CTA(k)                                                                                       \
    do {                                                                                                \
        const int cid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;                  \
        if (cid < 4096) g_pf_cta[cid][k] = gtimer();                                                    \
    } while (0)
#define PF_TRACE(ev, j)                                                                                     \
    do {                                                                                                  \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 256) g_pf_trace[ev][j] = clock64(); \
        if (blockIdx.x == 1 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 256 && (ev) <= 1)                  \
            g_pf_trace[6 + (ev)][j] = clock64();                                                            \
    } while (0)
#else
#define PF_TRACE(ev, j) \
    do {                \
    } while (0)
#define PF_CTA(k) \
    do {          \
    } while (0)
#endif
#define PF_CTA_START()         \
    do {                       \
        if (threadIdx.x == 0) PF_CTA(0); \
    } while (0)
constexpr int kQR = 128, kAttnThreads = 384, kKSlots = 3, kVSlots = 2, kMaxSinkRows = kPrefillMaxSinks;
constexpr uint32_t kQRow = 512, kKSlab = 8192, kKTile = 32768, kVTile = 16384;
// shared-memory carve-up; PAIR (2-SM mode): each CTA of the cluster holds half of every K tile
// (keys 32 r .. 32 r + 31: 4 half-slabs of 4 KB) and half of every V^T tile (channels 64 r ..)
template <bool PAIR>
struct AttnSmem {
    static constexpr uint32_t kt = PAIR ? kKTile / 2 : kKTile, vt = PAIR ? kVTile / 2 : kVTile;
    static constexpr uint32_t k = kQR * kQRow, v = k + kKSlots * kt, sink = v + kVSlots * vt,
                              ml = sink + kMaxSinkRows * 128 * 6 + 64, bar = ml + 2 * 128 * 8;
    static constexpr size_t total = bar + 256 + 1024;  // + barriers, + alignment slack
};
// tensor-memory columns: S_0 [0, 64), S_1 [64, 128), O_0 [128, 256), O_1 [256, 384), Q hi [384, 448), Q lo [448, 512)
constexpr uint32_t kColO = 128, kColQhi = 384, kColQlo = 448;
constexpr float kLazy = 14.0f;  // rescale O only when the max grows by > 2^14 (P <= 2^14 in fp16)

template <bool PAIR>
__global__ void __launch_bounds__(kAttnThreads, 1) prefill_attn_kernel(PrefillParams p) {
    using L = AttnSmem<PAIR>;
    constexpr uint32_t kOffK = L::k, kOffV = L::v, kOffSink = L::sink, kOffML = L::ml, kOffBar = L::bar;
    constexpr uint32_t kKT2 = L::kt, kVT2 = L::vt;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-byte aligned
    const uint32_t sbase = smem_u32(smem);
    float* sink_k = reinterpret_cast<float*>(smem + kOffSink);                          // [16][128] RoPE'd
    uint16_t* sink_v = reinterpret_cast<uint16_t*>(smem + kOffSink + kMaxSinkRows * 512);  // [16][128] fp16
    int* sink_p = reinterpret_cast<int*>(smem + kOffSink + kMaxSinkRows * 768);             // [16] positions
    float2* ml_s = reinterpret_cast<float2*>(smem + kOffML);                               // [2][128] (m, l)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint64_t *kfull = bar, *kempty = bar + kKSlots, *vfull = bar + 2 * kKSlots, *vempty = vfull + 2, *s_full = vfull + 4,
             *p_full = vfull + 6, *o_done = vfull + 8, *q_full = vfull + 9, *q_tmem = vfull + 10, *sink_ready = vfull + 11,
             *kpeer = vfull + 12, *vpeer = kpeer + kKSlots,  // PAIR: the upper CTA's K / V halves landed,
             *ppeer = vpeer + 2, *qpeer = ppeer + 2;          // its P rows and its Q rows are in TMEM
    uint32_t* tslot = reinterpret_cast<uint32_t*>(qpeer + 1);

    pdl_wait();  // the key, value and query kernels before it (a chain of programmatic dependents)
    const int h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int REP = p.Hq / p.Hkv, kvh = h / REP;
    const int64_t nq = p.num_q;
    // heaviest query blocks first; PAIR: a cluster of two CTAs takes 256 rows, CTA rank r rows 128 r ..
    const uint32_t rank = PAIR ? umma::cluster_rank() : 0u;
    const int64_t blk0 = PAIR ? static_cast<int64_t>((gridDim.x >> 1) - 1 - (blockIdx.x >> 1)) * 2 * kQR
                              : static_cast<int64_t>(gridDim.x - 1 - blockIdx.x) * kQR;
    const int64_t i0 = blk0 + kQR * rank;
    const int nrows = static_cast<int>(lmin64(kQR, nq - i0));  // may be <= 0 for the upper CTA of the last pair
    const int64_t q0 = p.q_start[b] + i0, T = p.seq_len[b];
    const int64_t kend = lmin64(T, p.q_start[b] + blk0 + lmin64(PAIR ? 2 * kQR : kQR, nq - blk0));
    const int nt = kend > 0 ? static_cast<int>((kend + kPrefillKT - 1) / kPrefillKT) : 0;
    const int nsink = min(min(p.cache.sink_count[b], p.max_sinks), kMaxSinkRows);

    PF_CTA_START();
    if (tid == 0) {
        for (int i = 0; i < kKSlots; ++i) {
            mbar_init(kfull + i, 1);
            mbar_init(kempty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(vfull + i, 1);
            mbar_init(vempty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, 128);
            mbar_init(vpeer + i, 1);
            mbar_init(ppeer + i, 1);
        }
        for (int i = 0; i < kKSlots; ++i) mbar_init(kpeer + i, 1);
        mbar_init(qpeer, 1);
        mbar_init(o_done, 1);
        mbar_init(q_full, 1);
        mbar_init(q_tmem, 256);
        mbar_init(sink_ready, 32);
        mbar_fence_init();
    }
    if (warp == 1) {
        if constexpr (PAIR) umma::alloc2<512>(tslot);
        else umma::alloc<512>(tslot);
    }
    umma::fence_before();
    if constexpr (PAIR) umma::cluster_sync();  // the leader's barriers exist before any remote arrival
    else __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tslot;
    // hand-offs to the MMA issuer: every thread arrives in its own CTA (cheap, CTA scope); in PAIR
    // mode one thread of the upper CTA relays each completed phase to the leader's *peer barrier
    // with a single cluster-scope arrive, and the leader waits for both
    auto wait_both = [&](uint64_t* local, uint64_t* peer, uint32_t parity) {
        mbar_wait(local, parity);
        if constexpr (PAIR) umma::mbar_wait_cluster(peer, parity);
    };

    if (warp == 0) {
        // ---- query block, then the key tiles (kKSlots deep)
        if (umma::elect_one()) {
            mbar_arrive_expect_tx(q_full, kQR * kQRow);
            const unsigned char* qsrc = p.q_rows + ((static_cast<int64_t>(b) * p.Hq + h) * p.num_q_pad + i0) * kQRow;
            for (int c = 0; c < 4; ++c) bulk_g2s(smem + c * 16384, qsrc + c * 16384, 16384, q_full);
            for (int j = 0; j < nt; ++j) {
                const int sl = j % kKSlots;
                if (j >= kKSlots) mbar_wait_sleep(kempty + sl, ((j / kKSlots) - 1) & 1);
                const unsigned char* src = kv_tile(p, b, kvh, j);
                unsigned char* dst = smem + kOffK + sl * kKT2;
                mbar_arrive_expect_tx(kfull + sl, kKT2);
                if constexpr (PAIR) {  // rows 32 r .. of the 4 slabs (hi s0, hi s1, lo s0, lo s1)
#pragma unroll
                    for (int q = 0; q < 4; ++q) bulk_g2s(dst + q * 4096, src + q * 8192 + rank * 4096, 4096, kfull + sl);
                } else {
                    bulk_g2s(dst, src, kKTile / 2, kfull + sl);
                    bulk_g2s(dst + kKTile / 2, src + kKTile / 2, kKTile / 2, kfull + sl);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1 && rank == 0) {
        // ---- MMA issuer (PAIR: the leader issues 2-SM MMAs, M = 256, B halves in both CTAs)
        if (umma::elect_one()) {
            constexpr int M = PAIR ? 256 : 128;
            constexpr uint32_t idS = umma::idesc_f16(M, 64), idO = umma::idesc_f16(M, 128);
            constexpr uint32_t kHiSlab = PAIR ? 4096 : kKSlab, kLoOff = PAIR ? 8192 : 2 * kKSlab;
            auto mma = [&](uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
                if constexpr (PAIR) umma::mma2_f16_ts(d, a, bdesc, idesc, acc);
                else umma::mma_f16_ts(d, a, bdesc, idesc, acc);
            };
            auto commit_all = [&](uint64_t* bar) {
                if constexpr (PAIR) umma::commit2(bar);
                else umma::commit(bar);
            };
            wait_both(q_tmem, qpeer, 0);
            PF_CTA(1);
            auto qk = [&](int j) {
                const int sl = j % kKSlots, sb = j & 1;
                wait_both(kfull + sl, kpeer + sl, (j / kKSlots) & 1);
                umma::fence_after();
                PF_TRACE(4, j);
                const uint32_t d = tmem + 64u * sb, kb = sbase + kOffK + sl * kKT2;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint32_t ko = (ks >> 2) * kHiSlab + (ks & 3) * 32;
                    const uint64_t bh = umma::sdesc(kb + ko), bl = umma::sdesc(kb + kLoOff + ko);
                    mma(d, tmem + kColQhi + 8 * ks, bh, idS, ks > 0);
                    mma(d, tmem + kColQhi + 8 * ks, bl, idS, 1);
                    mma(d, tmem + kColQlo + 8 * ks, bh, idS, 1);
                }
                commit_all(s_full + sb);
                commit_all(kempty + sl);
            };
            auto pv = [&](int j) {
                const int sb = j & 1;
                wait_both(vfull + sb, vpeer + sb, (j >> 1) & 1);
                mbar_wait(p_full + sb, (j >> 1) & 1);
                if constexpr (PAIR) umma::mbar_wait_cluster(ppeer + sb, (j >> 1) & 1);
                umma::fence_after();
                PF_TRACE(2, j);
                const uint32_t vb = sbase + kOffV + sb * kVT2;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma(tmem + kColO + 128u * sb, tmem + 64u * sb + 8 * kk, umma::sdesc(vb + kk * 32), idO, (j >= 2 || kk > 0));
                commit_all(vempty + sb);
                PF_TRACE(3, j);
            };
            if (nt > 0) qk(0);
            if (nt > 1) qk(1);
            for (int j = 0; j < nt; ++j) {
                pv(j);
                if (j + 2 < nt) qk(j + 2);
            }
            commit_all(o_done);
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- PAIR, upper CTA: relay "Q rows in TMEM", then per tile "V half landed" and
        // "P rows written" to the leader
        if (umma::elect_one()) {
            // suspending waits: a spinning relay would take issue slots from the softmax warps
            mbar_wait_sleep(q_tmem, 0);
            umma::mbar_arrive_cluster(umma::peer_addr(qpeer, 0));
            for (int j = 0; j < nt; ++j) {
                mbar_wait_sleep(vfull + (j & 1), (j >> 1) & 1);
                umma::mbar_arrive_cluster(umma::peer_addr(vpeer + (j & 1), 0));
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---- sink rows of this KV head: keys RoPE'd at their own position (fp32), values raw
        for (int s = 0; s < nsink; ++s) {
            const int pos = p.cache.sink_pos[b * p.max_sinks + s];
            const int64_t srow = (static_cast<int64_t>(b) * p.max_sinks + s) * p.C + kvh * 128;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int f = lane + 32 * k;
                const float ka = h2f(p.cache.sink_k[srow + f]), kb = h2f(p.cache.sink_k[srow + f + 64]);
                const float2 r = rope_cs(p.rope, pos, f);
                sink_k[s * 128 + f] = ka * r.x - kb * r.y;
                sink_k[s * 128 + f + 64] = ka * r.y + kb * r.x;
            }
            reinterpret_cast<uint2*>(sink_v + s * 128)[lane] = *reinterpret_cast<const uint2*>(p.cache.sink_v + srow + 4 * lane);
            if (lane == 0) sink_p[s] = pos;
        }
        mbar_arrive(sink_ready);
        if (PAIR && rank == 1) {
            if (lane == 0) {  // tell the leader when this CTA's K halves have landed
                for (int j = 0; j < nt; ++j) {
                    mbar_wait_sleep(kfull + j % kKSlots, (j / kKSlots) & 1);
                    umma::mbar_arrive_cluster(umma::peer_addr(kpeer + j % kKSlots, 0));
                }
            } else if (lane == 1) {  // ... and when this CTA's P rows of tile j are in TMEM
                for (int j = 0; j < nt; ++j) {  // on the critical path: a polling wait
                    mbar_wait(p_full + (j & 1), (j >> 1) & 1);
                    umma::mbar_arrive_cluster(umma::peer_addr(ppeer + (j & 1), 0));
                }
            }
        }
        __syncwarp();
    } else if (warp == 3) {
        // ---- value tiles
        if (umma::elect_one()) {
            for (int j = 0; j < nt; ++j) {
                const int sl = j & 1;
                if (j >= kVSlots) mbar_wait_sleep(vempty + sl, ((j >> 1) - 1) & 1);
                PF_TRACE(5, j);
                mbar_arrive_expect_tx(vfull + sl, kVT2);
                bulk_g2s(smem + kOffV + sl * kVT2, kv_tile(p, b, kvh, j) + kKTile + rank * kVT2, kVT2, vfull + sl);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---- softmax group X = (warp - 4) / 4: tiles j = X mod 2, one query row per thread
        const int X = (warp - 4) >> 2;
        const int row = 32 * (warp & 3) + lane;
        const int64_t qpos = q0 + row;
        const uint32_t lrow = static_cast<uint32_t>(32 * (warp & 3)) << 16;
        const uint32_t colS = 64u * X, colO = kColO + 128u * X;
        const unsigned char* qrow = smem + row * kQRow;
        auto qchunk = [&](int c) { return *reinterpret_cast<const uint4*>(qrow + (((c ^ row) & 31) << 4)); };
        // this row of Q hi (group 0) / lo (group 1) -> tensor memory
        mbar_wait(q_full, 0);
        {
            uint32_t v[64];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint4 u = qchunk(16 * X + c);
                v[4 * c] = u.x;
                v[4 * c + 1] = u.y;
                v[4 * c + 2] = u.z;
                v[4 * c + 3] = u.w;
            }
            const uint32_t col = tmem + lrow + (X ? kColQlo : kColQhi);
#pragma unroll
            for (int c = 0; c < 4; ++c) umma::st16(col + 16 * c, reinterpret_cast<const uint32_t(&)[16]>(v[16 * c]));
        }
        umma::wait_st();
        umma::fence_before();
        mbar_arrive(q_tmem);

        const int64_t mask_words = (p.max_tokens + 31) / 32;
        const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * mask_words;
        float m = -INFINITY, l = 0.f;
        for (int j = X; j < nt; j += 2) {
            mbar_wait(s_full + X, (j >> 1) & 1);
            umma::fence_after();
            if (lane == 0 && warp == 4) PF_TRACE(0, j);
            uint32_t v[4][16];
#pragma unroll
            for (int c = 0; c < 4; ++c) umma::ld16(tmem + lrow + colS + 16u * c, v[c]);
#pragma unroll
            for (int c = 0; c < 4; ++c) umma::wait_ld(v[c]);
            float s[64];
#pragma unroll
            for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(v[c >> 4][c & 15]);
            const int64_t k0 = static_cast<int64_t>(j) * kPrefillKT;
            // the second word exists only when the row has one past k0/32 (max_tokens > k0 + 32)
            const uint32_t sm0 = __ldg(smask + (k0 >> 5));
            const uint32_t sm1 = (k0 >> 5) + 1 < mask_words ? __ldg(smask + (k0 >> 5) + 1) : 0u;
            if (k0 + kPrefillKT - 1 > q0 || k0 + kPrefillKT > T || (sm0 | sm1)) {
                const int64_t lim = lmin64(qpos + 1, T) - k0;  // keys k0 + c, c < lim, are in range
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    const bool sink = ((c < 32 ? sm0 : sm1) >> (c & 31)) & 1u;
                    s[c] = (c < lim && !sink) ? s[c] : -INFINITY;
                }
            }
            float mx8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                mx8[i] = fmaxf(fmaxf(s[i], s[i + 8]), s[i + 16]);
                mx8[i] = fmaxf(fmaxf(mx8[i], s[i + 24]), s[i + 32]);
                mx8[i] = fmaxf(fmaxf(mx8[i], s[i + 40]), s[i + 48]);
                mx8[i] = fmaxf(mx8[i], s[i + 56]);
            }
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
            float alpha = 1.0f;
            bool resc = false;
            if (mx != -INFINITY) {
                if (m == -INFINITY) {
                    m = mx;
                } else if (mx > m + kLazy) {
                    alpha = ex2(m - mx);
                    m = mx;
                    resc = true;
                }
            }
            if (__any_sync(0xffffffffu, resc)) {  // PV(j - 2) is complete (it precedes QK(j)): rescale O_X in place
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    uint32_t o[16];
                    umma::ld16(tmem + lrow + colO + 16u * c, o);
                    umma::wait_ld(o);
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    umma::st16(tmem + lrow + colO + 16u * c, o);
                }
                l *= alpha;
            }
            const float mu = m == -INFINITY ? 0.f : m;
            const float2 mu2 = make_float2(mu, mu);
            float2 ls[4];
            uint32_t hv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float2 d = sub2(make_float2(s[2 * i], s[2 * i + 1]), mu2);
                const float2 pp = make_float2(ex2(d.x), ex2(d.y));
                ls[i & 3] = i < 4 ? pp : add2(ls[i & 3], pp);
                hv[i] = pack_h2(pp.x, pp.y);
            }
            const float2 lt = add2(add2(ls[0], ls[1]), add2(ls[2], ls[3]));
            l += lt.x + lt.y;
            umma::st16(tmem + lrow + colS, reinterpret_cast<const uint32_t(&)[16]>(hv[0]));
            umma::st16(tmem + lrow + colS + 16, reinterpret_cast<const uint32_t(&)[16]>(hv[16]));
            umma::wait_st();
            umma::fence_before();
            mbar_arrive(p_full + X);
            if (lane == 0 && warp == 4) PF_TRACE(1, j);
        }
        if (tid == 128) PF_CTA(2);

        // ---- epilogue: merge the two groups' (m, l), the sink logits (q = hi + lo of the staged row)
        ml_s[X * 128 + row] = make_float2(m, l);
        asm volatile("bar.sync 2, 256;" ::: "memory");
        const float2 other = ml_s[(1 - X) * 128 + row];
        const float mA = X ? other.x : m, lA = X ? other.y : l, mB = X ? m : other.x, lB = X ? l : other.y;
        mbar_wait(sink_ready, 0);
        float es[kMaxSinkRows];
        float M = fmaxf(mA, mB);
#pragma unroll 1
        for (int s = 0; s < nsink; ++s) {
            const int pos = sink_p[s];
            float e = -INFINITY;
            if (pos <= qpos && pos < T) {
                const float* kr = sink_k + s * 128;
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const uint4 hi = qchunk(c), lo = qchunk(16 + c);
                    const uint32_t hw[4] = {hi.x, hi.y, hi.z, hi.w}, lw[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float2 qh = __half22float2(*reinterpret_cast<const __half2*>(&hw[k]));
                        const float2 ql = __half22float2(*reinterpret_cast<const __half2*>(&lw[k]));
                        const float2 kk = *reinterpret_cast<const float2*>(kr + 8 * c + 2 * k);
                        acc = fma2(add2(qh, ql), kk, acc);
                    }
                }
                e = acc.x + acc.y;
            }
            es[s & (kMaxSinkRows - 1)] = e;
            M = fmaxf(M, e);
        }
        const float aA = mA == -INFINITY ? 0.f : ex2(mA - M), aB = mB == -INFINITY ? 0.f : ex2(mB - M);
        float L = lA * aA + lB * aB;
        for (int s = 0; s < nsink; ++s) {
            const float w = es[s] == -INFINITY ? 0.f : ex2(es[s] - M);
            es[s] = w;
            L += w;
        }
        const float inv = L > 0.f ? 1.0f / L : 0.f;
        // u = O[0:64] +/- O[64:128] (group 0: +, group 1: -), O = aA O_0 + aB O_1; a group
        // without tiles never wrote its accumulator and is skipped
        float u[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) u[i] = 0.f;
        if (nt > 0) {
            mbar_wait(o_done, 0);
            umma::fence_after();
            const float sg = X ? -1.f : 1.f;
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const float ag = g ? aB : aA;
                if (g == 1 && nt < 2) break;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t lo[16], hi[16];
                    umma::ld16(tmem + lrow + kColO + 128u * g + 16u * c, lo);
                    umma::ld16(tmem + lrow + kColO + 128u * g + 64u + 16u * c, hi);
                    umma::wait_ld(lo);
                    umma::wait_ld(hi);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        u[16 * c + i] += ag * (__uint_as_float(lo[i]) + sg * __uint_as_float(hi[i]));
                }
            }
        }
        // H_64 butterflies in registers (with the H_2 stage above: V's inverse rotation H_128)
#pragma unroll
        for (int len = 1; len < 64; len <<= 1)
#pragma unroll
            for (int i = 0; i < 64; ++i)
                if (!(i & len)) {
                    const float a = u[i], c = u[i + len];
                    u[i] = a + c;
                    u[i + len] = a - c;
                }
        const float sc = inv * (1.0f / sqrtf(128.0f));
#pragma unroll
        for (int i = 0; i < 64; ++i) u[i] *= sc;
#pragma unroll 1
        for (int s = 0; s < nsink; ++s) {
            const float w = es[s] * inv;
            if (w != 0.f) {
                const __half2* vr = reinterpret_cast<const __half2*>(sink_v + s * 128 + 64 * X);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float2 vv = __half22float2(vr[i]);
                    u[2 * i] += w * vv.x;
                    u[2 * i + 1] += w * vv.y;
                }
            }
        }
        if (row < nrows) {
            float4* dst = reinterpret_cast<float4*>(p.out + ((static_cast<int64_t>(b) * nq + i0 + row) * p.Hq + h) * 128 + 64 * X);
#pragma unroll
            for (int c = 0; c < 16; ++c) dst[c] = make_float4(u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
        }
    }
    umma::fence_before();
    if constexpr (PAIR) umma::cluster_sync();  // the peer's shared memory / TMEM stay live until both are done
    else __syncthreads();
    if (warp == 1) {
        umma::fence_after();
        if constexpr (PAIR) umma::dealloc2<512>(tmem);
        else umma::dealloc<512>(tmem);
    }
    if (tid == 0) PF_CTA(3);
}

}  // namespace

#ifdef RKV_PF_TRACE
extern "C" int rkv_debug_prefill_trace(long long* out) {
    return cudaMemcpyFromSymbol(out, g_pf_trace, sizeof(g_pf_trace)) == cudaSuccess ? 0 : 1;
}
extern "C" int rkv_debug_prefill_cta(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_pf_cta, sizeof(g_pf_cta)) == cudaSuccess ? 0 : 1;
}
#endif

namespace {
// 2-SM mode (opt-in, RKV_PREFILL_PAIR=1): correct, but the per-tile cluster-scope hand-offs
// (P rows of the upper CTA -> leader) cost ~2,000 cycles, more than the halved shared-memory
// traffic saves
bool prefill_pair() { return options().prefill_pair.load() == 1; }
}  // namespace

cudaError_t launch_prefill(const rkv_layer_desc& d, const PrefillParams& p, int64_t max_seq_len, cudaStream_t s) {
    const int C = p.C, W = C / 16, MG = C / 128;
    const int N = mma_layout_n(d), NG = C / N;
    const bool pair = N == 256 && d.heads_per_group == 4;
    const size_t ksmem = 2 * static_cast<size_t>(C) * 4 + 4 * static_cast<size_t>(W + MG) * 4 + 4 * 32 * 16 +
                         (pair ? static_cast<size_t>(NG) * 4 * 2 * 32 * 16 : 0);
    const int nthreads = std::min(512, std::max(NG * 32, ((2 * W + 31) / 32) * 32));
    const dim3 kgrid(static_cast<unsigned>((max_seq_len + 3) / 4), static_cast<unsigned>(d.batch));
    cudaError_t e;
    if (N == 512) {
        auto kern = d.heads_per_group == 1   ? reconstruct_keys_kernel<4, 1>
                    : d.heads_per_group == 2 ? reconstruct_keys_kernel<4, 2>
                                             : reconstruct_keys_kernel<4, 4>;
        if ((e = ensure_smem_k(kern, ksmem)) != cudaSuccess) return e;
        kern<<<kgrid, nthreads, ksmem, s>>>(p);
    } else if (N == 256 && pair) {  // GQA at G = 4: half-group pairs
        if ((e = ensure_smem_k(reconstruct_keys_kernel<2, 2, true>, ksmem)) != cudaSuccess) return e;
        reconstruct_keys_kernel<2, 2, true><<<kgrid, nthreads, ksmem, s>>>(p);
    } else if (N == 256) {  // GQA at G = 2, or G = 1 (per-head rotation, AG = 1)
        auto kern = d.heads_per_group == 1 ? reconstruct_keys_kernel<2, 1> : reconstruct_keys_kernel<2>;
        if ((e = ensure_smem_k(kern, ksmem)) != cudaSuccess) return e;
        kern<<<kgrid, nthreads, ksmem, s>>>(p);
    } else {
        return cudaErrorInvalidValue;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const dim3 vgrid(static_cast<unsigned>((max_seq_len + kPrefillKT - 1) / kPrefillKT), static_cast<unsigned>(p.Hkv),
                     static_cast<unsigned>(d.batch));
    // values and queries are programmatic dependents: they start in the key
    // kernel's tail; each completes only after its predecessor (pdl_wait at
    // its end), so the attention kernel's wait covers all three
    if ((e = launch_pdl(reconstruct_values_kernel, vgrid, dim3(128), 0, s, p)) != cudaSuccess) return e;
    if ((e = launch_pdl(prepare_queries_kernel,
                        dim3(static_cast<unsigned>(p.num_q_pad), static_cast<unsigned>((p.Hq + 15) / 16),
                             static_cast<unsigned>(d.batch)),
                        dim3(128), 0, s, p)) != cudaSuccess)
        return e;
    const dim3 agrid(static_cast<unsigned>(p.num_q_pad / kQR), static_cast<unsigned>(p.Hq), static_cast<unsigned>(d.batch));
    if (prefill_pair()) {  // 2-SM clusters (num_q_pad is a multiple of 256)
        constexpr size_t sm = AttnSmem<true>::total;
        if ((e = ensure_smem_k(prefill_attn_kernel<true>, sm)) != cudaSuccess) return e;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = agrid;
        cfg.blockDim = dim3(kAttnThreads);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, prefill_attn_kernel<true>, p);
    }
    constexpr size_t sm = AttnSmem<false>::total;
    if ((e = ensure_smem_k(prefill_attn_kernel<false>, sm)) != cudaSuccess) return e;
    return launch_pdl(prefill_attn_kernel<false>, agrid, dim3(kAttnThreads), sm, s, p);
}

}  // namespace rkv
