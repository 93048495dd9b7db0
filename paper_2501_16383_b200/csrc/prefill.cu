// prefill.cu -- causal attention of a block of queries over the 2-bit rotated
// cache (the attention half of prefill,
// proj/src/pipeline.cpp:156-191: reconstruct_cache, then causal
// reference_attention, proj/src/attention.cpp:20-49).
//
// Three launches, mirroring the reference's decomposition:
//   1. reconstruct_keys_kernel (== reconstruct_cache for K): per token the
//      un-reorder scatter, the tensor-core inverse FWHT of decode_mma.cu (two
//      chained H_16 mma.sync with the fp16 hi/lo split) and RoPE at the
//      token's position, written once as fp16 hi + fp16 lo rows [B][T][C]
//      (natural channel order, FWHT normalisation applied).  Every key is
//      reconstructed once and reused by every query.
//   2. prefill_attn_kernel: flash attention per (sequence, q head, 64-query
//      block), 4 warps x 16 query rows.  S = Q K^T on mma.sync m16n8k16 with
//      both operands split into fp16 hi + lo (three MMAs: hi.hi + hi.lo +
//      lo.hi, ~2^-22 relative); causal + sink + length mask; online softmax
//      in the exp2 domain; P.V on mma.sync with the 2-bit V codes as exact fp16
//      subnormals (B operand) and fp16(p * s) as the A operand (the chained S
//      accumulator fragment), the zero point folded per row.  Sink tokens are
//      skipped here and one (m, l, o') partial per query row is written.
//   3. prefill_combine_kernel: adds the fp16 sink rows (exact, natural frame,
//      RoPE at their own position) and applies H_128 (V's inverse rotation),
//      like decode_combine_kernel, with the row's own query position.
#include <algorithm>
#include <cmath>

#include "rkv_common.cuh"
#include "rkv_internal.h"
#include "rkv_layout.h"
#include "rkv_mma.cuh"

namespace rkv {

namespace {

using namespace mma;

constexpr int kRopeRowF4 = 128;  // float4 per position-pair row of the RoPE table (decode_attention.cu)

__device__ __forceinline__ float2 rope_cs(const float4* t, int64_t pos, int f) {
    const float4 r = __ldg(t + (pos >> 1) * kRopeRowF4 + f);
    return (pos & 1) ? make_float2(r.y, r.w) : make_float2(r.x, r.z);
}

// ------------------------------------------------------------------ 1. keys
// CTA = (4-token tile, sequence), one warp per FWHT group.
template <int G>
__global__ void __launch_bounds__(512) reconstruct_keys_kernel(PrefillParams p) {
    constexpr int N = 128 * G, NJ = N / 128, TT = 4;
    extern __shared__ __align__(16) unsigned char smem[];
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
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens + t0;
    for (int i = tid; i < TT * W; i += NT) kcs[i] = i / W < nv ? p.cache.k_codes[row0 * W + i] : 0u;
    for (int i = tid; i < TT * MG; i += NT) kms[i] = i / MG < nv ? p.cache.k_meta[row0 * MG + i] : 0u;
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
    uint32_t AH[4];
    hadamard16_frag(AH, lane, static_cast<uint32_t>(p.max_tokens >> 40));
    const float kn = p.k_norm;
    const int swz = mma_swz(N, lane);
    const unsigned char* lbase = knat + gam * N * 4 + lane * NJ * 16;
    uint16_t* khi = p.kr_hi + row0 * C;
    uint16_t* klo = p.kr_lo + row0 * C;
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
            const float4* rrow = p.rope + (pos >> 1) * kRopeRowF4 + 64 + (pos & 1) * 32;
#pragma unroll
            for (int f1 = 0; f1 < 2; ++f1) {
                const int f = 2 * tl + 8 * f1 + 16 * (g & 3);
                const float4 r4 = __ldg(rrow + (f >> 1));
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
                        mma16816(t4, AH, h0, h1, zero);
                        mma16816(z[o], AH, l0, l1, t4);
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
                        const int64_t o0 = tt * static_cast<int64_t>(C) + kvh * 128 + f;
                        const uint32_t ha = pack_h2(ka[0], ka[1]), hb = pack_h2(kb[0], kb[1]);
                        *reinterpret_cast<uint32_t*>(khi + o0) = ha;
                        *reinterpret_cast<uint32_t*>(khi + o0 + 64) = hb;
                        *reinterpret_cast<uint32_t*>(klo + o0) = pack_h2(sub_lo(ka[0], ha), sub_hi(ka[1], ha));
                        *reinterpret_cast<uint32_t*>(klo + o0 + 64) = pack_h2(sub_lo(kb[0], hb), sub_hi(kb[1], hb));
                    }
                } else {
                    const uint32_t h0 = pack_h2(yf[0][2 * f1], yf[0][2 * f1 + 1]);
                    const uint32_t h1 = pack_h2(yf[1][2 * f1], yf[1][2 * f1 + 1]);
                    const uint32_t l0 = pack_h2(sub_lo(yf[0][2 * f1], h0), sub_hi(yf[0][2 * f1 + 1], h0));
                    const uint32_t l1 = pack_h2(sub_lo(yf[1][2 * f1], h1), sub_hi(yf[1][2 * f1 + 1], h1));
                    float t4[4], z[4];
                    mma16816(t4, AH, h0, h1, zero);
                    mma16816(z, AH, l0, l1, t4);
                    const int kvh = gam * G + (g >> 2);
                    float ka[2], kb[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const float a = z[i], bb = z[2 + i];  // channels f+i and f+64+i
                        const float c = i ? r4.y : r4.x, s = i ? r4.w : r4.z;
                        ka[i] = (a * c - bb * s) * kn;
                        kb[i] = (a * s + bb * c) * kn;
                    }
                    const int64_t o0 = tt * static_cast<int64_t>(C) + kvh * 128 + f;
                    const uint32_t ha = pack_h2(ka[0], ka[1]), hb = pack_h2(kb[0], kb[1]);
                    *reinterpret_cast<uint32_t*>(khi + o0) = ha;
                    *reinterpret_cast<uint32_t*>(khi + o0 + 64) = hb;
                    *reinterpret_cast<uint32_t*>(klo + o0) = pack_h2(sub_lo(ka[0], ha), sub_hi(ka[1], ha));
                    *reinterpret_cast<uint32_t*>(klo + o0 + 64) = pack_h2(sub_lo(kb[0], hb), sub_hi(kb[1], hb));
                }
            }
        }
    }
}

// -------------------------------------------------------------- 2. attention
constexpr int kQB = 64, kKT = 32, kRowH = 136;  // queries per CTA, keys per tile, padded smem row (halves)
// one K/V tile buffer: K hi + lo rows, V words of the KV head, V meta words, sink-mask word
constexpr int kTileBytes = 2 * kKT * kRowH * 2 + kKT * 8 * 4 + kKT * 4 + 16;

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(128) prefill_attn_kernel(PrefillParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint16_t* qhi = reinterpret_cast<uint16_t*>(smem);  // [64][136]
    uint16_t* qlo = qhi + kQB * kRowH;
    unsigned char* tiles = reinterpret_cast<unsigned char*>(qlo + kQB * kRowH);  // 2 x kTileBytes

    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tl = lane & 3;
    const int C = p.C, W = C / 16, MG = C / 128, Hq = p.Hq, REP = p.Hq / p.Hkv;
    const int kvh = h / REP;
    const int64_t nq = p.num_q, i0 = static_cast<int64_t>(qb) * kQB;
    const int nrows = static_cast<int>(lmin64(kQB, nq - i0));
    const int64_t qpos0 = p.q_start[b] + i0;
    const int64_t T = p.seq_len[b];
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;
    const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
    const int64_t kend = lmin64(T, qpos0 + nrows);  // keys [0, kend)

    // K/V tile k0 -> buffer bi, cp.async (rows past the end are zero-filled)
    auto issue = [&](int bi, int64_t k0) {
        unsigned char* tb = tiles + bi * kTileBytes;
        const uint32_t khs = smem_u32(tb), kls = khs + kKT * kRowH * 2;
        const uint32_t vws = kls + kKT * kRowH * 2, vms = vws + kKT * 8 * 4, mks = vms + kKT * 4;
        const int nk = static_cast<int>(lmin64(kKT, kend - k0));
        {
            // thread -> chunk column (tid & 15) of key rows (tid >> 4) + 8 i
            const int ch = (tid & 15) * 8, kr0 = tid >> 4;
            const uint16_t* sh = p.kr_hi + (row0 + k0) * C + kvh * 128 + ch;
            const uint16_t* sl = p.kr_lo + (row0 + k0) * C + kvh * 128 + ch;
            const uint32_t dofs = (kr0 * kRowH + ch) * 2;
#pragma unroll
            for (int i = 0; i < kKT / 8; ++i) {
                const int kk = kr0 + 8 * i;
                const int64_t so = static_cast<int64_t>(kk < nk ? kk : 0) * C;
                const uint32_t nb = kk < nk ? 16u : 0u;
                cp_async16(khs + dofs + i * 8 * kRowH * 2, sh + so, nb);
                cp_async16(kls + dofs + i * 8 * kRowH * 2, sl + so, nb);
            }
        }
        if (tid < kKT * 2) {  // V words: 8 per key = two 16-byte chunks
            const int kk = tid >> 1;
            const int64_t src = (row0 + k0 + (kk < nk ? kk : 0)) * W + kvh * 8 + (tid & 1) * 4;
            cp_async16(vws + tid * 16, p.cache.v_codes + src, kk < nk ? 16u : 0u);
        } else if (tid < kKT * 3) {  // V meta word of the KV head
            const int kk = tid - kKT * 2;
            cp_async4(vms + kk * 4, p.cache.v_meta + (row0 + k0 + (kk < nk ? kk : 0)) * MG + kvh, kk < nk ? 4u : 0u);
        } else if (tid == kKT * 3) {
            cp_async4(mks, smask + (k0 >> 5), 4u);  // k0 % 32 == 0
        }
        cp_async_commit();
    };
    if (kend > 0) issue(0, 0);

    // q: RoPE at each row's position, x log2(e)/sqrt(d), split into fp16 hi + lo
    for (int idx = tid; idx < kQB * 64; idx += blockDim.x) {
        const int r = idx >> 6, f = idx & 63;
        float qa = 0.f, qb2 = 0.f;
        if (r < nrows) {
            const uint16_t* qr = p.q + ((static_cast<int64_t>(b) * nq + i0 + r) * Hq + h) * 128;
            const float a = h2f(qr[f]), bb = h2f(qr[f + 64]);
            const float2 cs = rope_cs(p.rope, qpos0 + r, f);
            qa = (a * cs.x - bb * cs.y) * p.qscale;
            qb2 = (a * cs.y + bb * cs.x) * p.qscale;
        }
        const __half ha = __float2half_rn(qa), hb = __float2half_rn(qb2);
        qhi[r * kRowH + f] = __half_as_ushort(ha);
        qhi[r * kRowH + f + 64] = __half_as_ushort(hb);
        qlo[r * kRowH + f] = __half_as_ushort(__float2half_rn(qa - __half2float(ha)));
        qlo[r * kRowH + f + 64] = __half_as_ushort(__float2half_rn(qb2 - __half2float(hb)));
    }

    const int wr = warp * 16;  // this warp's first row
    const int64_t qp_a = qpos0 + wr + g, qp_b = qp_a + 8;
    const int64_t warp_last = qpos0 + std::min(wr + 15, nrows - 1);
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f}, zc_r[2] = {0.f, 0.f};
    float o[16][4];
#pragma unroll
    for (int e = 0; e < 16; ++e)
#pragma unroll
        for (int c = 0; c < 4; ++c) o[e][c] = 0.f;
    // ldmatrix lane addresses: A (Q rows wr.., matrices (r0-7,c0-7),(r8-15,c0-7),(r0-7,c8-15),(r8-15,c8-15));
    // B (K rows = keys: (k0-7,c0-7),(k0-7,c8-15),(k8-15,c0-7),(k8-15,c8-15) -> two n-tiles)
    const int mi = lane >> 3, mr = lane & 7;
    const uint32_t qa_hi = smem_u32(qhi + (wr + mr + 8 * (mi & 1)) * kRowH + 8 * (mi >> 1));
    const uint32_t qa_lo = qa_hi + kQB * kRowH * 2;
    const uint32_t kb_off = ((mr + 8 * (mi >> 1)) * kRowH + 8 * (mi & 1)) * 2;

    int bi = 0;
    for (int64_t k0 = 0; k0 < kend; k0 += kKT, bi ^= 1) {
        if (k0 + kKT < kend) {
            issue(bi ^ 1, k0 + kKT);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();  // tile k0 (and the q tile) visible
        const unsigned char* tb = tiles + bi * kTileBytes;
        const uint32_t khs = smem_u32(tb), kls = khs + kKT * kRowH * 2;
        const uint32_t* vws = reinterpret_cast<const uint32_t*>(tb + 2 * kKT * kRowH * 2);
        const uint32_t* vms = vws + kKT * 8;
        const uint32_t mbits = vms[kKT];
        const int nk = static_cast<int>(lmin64(kKT, kend - k0));
        if (!(k0 > warp_last || wr >= nrows)) {
            // S = Q K^T (16 rows x 32 keys), fp16 hi/lo split on both operands
            float s[4][4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c) s[nt][c] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                uint32_t ah[4], al[4];
                ldsm_x4(ah, qa_hi + ks * 32);
                ldsm_x4(al, qa_lo + ks * 32);
#pragma unroll
                for (int np = 0; np < 2; ++np) {  // n-tile pairs (2np, 2np+1)
                    uint32_t bh[4], bl[4];
                    const uint32_t off = kb_off + (np * 16 * kRowH + ks * 16) * 2;
                    ldsm_x4(bh, khs + off);
                    ldsm_x4(bl, kls + off);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        float (&acc)[4] = s[2 * np + j];
                        mma16816(acc, ah, bh[2 * j], bh[2 * j + 1], acc);
                        mma16816(acc, ah, bl[2 * j], bl[2 * j + 1], acc);
                        mma16816(acc, al, bh[2 * j], bh[2 * j + 1], acc);
                    }
                }
            }
            // mask (causal, length, sinks) -- only tiles that need it: the warp's
            // first row sees the whole tile, no sink in it, tile full
            float mx[2] = {-INFINITY, -INFINITY};
            const bool full = nk == kKT && mbits == 0u && k0 + kKT - 1 <= qpos0 + wr;
            if (!full) {
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int kk = nt * 8 + 2 * tl + (c & 1);
                        const int64_t kp = k0 + kk;
                        const int64_t qp = (c >> 1) ? qp_b : qp_a;
                        const bool ok = kk < nk && kp <= qp && !((mbits >> kk) & 1u);
                        s[nt][c] = ok ? s[nt][c] : -INFINITY;
                    }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c) mx[c >> 1] = fmaxf(mx[c >> 1], s[nt][c]);
            float alpha[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
                const float mn = fmaxf(m_r[r], mx[r]);
                alpha[r] = mn == -INFINITY ? 1.0f : ex2(m_r[r] - mn);
                m_r[r] = mn;
                l_r[r] *= alpha[r];
                zc_r[r] *= alpha[r];
            }
            if (alpha[0] != 1.0f || alpha[1] != 1.0f) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    o[e][0] *= alpha[0];
                    o[e][1] *= alpha[0];
                    o[e][2] *= alpha[1];
                    o[e][3] *= alpha[1];
                }
            }
            // P (x the key's V scale, fp16) as the A operand of P.V; zero point folded per row
            uint32_t pa[2][4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                float w[4], zr[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int kk = nt * 8 + 2 * tl + (c & 1);
                    const float pr = s[nt][c] == -INFINITY ? 0.f : ex2(s[nt][c] - m_r[c >> 1]);
                    l_r[c >> 1] += pr;
                    const uint32_t vm = pr > 0.f ? vms[kk] : 0u;
                    w[c] = pr * h2f(static_cast<uint16_t>(vm & 0xffffu));
                    zr[c] = h2f(static_cast<uint16_t>(vm >> 16));
                }
                const uint32_t p01 = pack_h2(w[0], w[1]), p23 = pack_h2(w[2], w[3]);
                const uint32_t z01 = pack_h2(zr[0], zr[1]), z23 = pack_h2(zr[2], zr[3]);
                zc_r[0] = fhfma<0, 0>(p01, z01, zc_r[0]);
                zc_r[0] = fhfma<1, 1>(p01, z01, zc_r[0]);
                zc_r[1] = fhfma<0, 0>(p23, z23, zc_r[1]);
                zc_r[1] = fhfma<1, 1>(p23, z23, zc_r[1]);
                pa[nt >> 1][(nt & 1) * 2 + 0] = p01;  // rows g: keys 2tl..(+8)
                pa[nt >> 1][(nt & 1) * 2 + 1] = p23;  // rows g+8
            }
#pragma unroll
            for (int kb = 0; kb < 2; ++kb) {
                const uint32_t a[4] = {pa[kb][0], pa[kb][1], pa[kb][2], pa[kb][3]};
                const int ka = 16 * kb + 2 * tl;
                const uint32_t w0 = vws[ka * 8 + g], w1 = vws[(ka + 1) * 8 + g];
                const uint32_t w8 = vws[(ka + 8) * 8 + g], w9 = vws[(ka + 9) * 8 + g];
                const uint32_t xl0 = prmt(w0, w1, 0x5410u), xh0 = prmt(w0, w1, 0x7632u);
                const uint32_t xl8 = prmt(w8, w9, 0x5410u), xh8 = prmt(w8, w9, 0x7632u);
                const uint32_t xl0s = xl0 >> 10, xh0s = xh0 >> 10, xl8s = xl8 >> 10, xh8s = xh8 >> 10;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int ee = e & 7;
                    const int sh = ee < 5 ? ee : ee - 5;
                    const uint32_t m = 0x00030003u << (2 * sh);
                    const uint32_t b0 = (e < 8 ? (ee < 5 ? xl0 : xl0s) : (ee < 5 ? xh0 : xh0s)) & m;
                    const uint32_t b1 = (e < 8 ? (ee < 5 ? xl8 : xl8s) : (ee < 5 ? xh8 : xh8s)) & m;
                    mma16816(o[e], a, b0, b1, o[e]);
                }
            }
        }
        __syncthreads();  // buffer bi free for the tile after next
    }
    // per-row partials: l, zc summed over the quad; o' = o * 2^(24-2e') - zc
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
        zc_r[r] += __shfl_xor_sync(0xffffffffu, zc_r[r], 1);
        zc_r[r] += __shfl_xor_sync(0xffffffffu, zc_r[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int row = wr + g + 8 * r;
        if (row >= nrows) continue;
        const int64_t orow = (static_cast<int64_t>(b) * nq + i0 + row) * Hq + h;
        if (tl == 0) {
            p.ws_ml[orow * 2] = m_r[r];
            p.ws_ml[orow * 2 + 1] = l_r[r];
        }
        float* dst = p.ws_o + orow * 128;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int ee = e & 7, sh = ee < 5 ? ee : ee - 5;
            const float sc = __int_as_float((127 + 24 - 2 * sh) << 23);
#pragma unroll
            for (int c = 0; c < 2; ++c) dst[(2 * tl + c) * 16 + e] = o[e][2 * r + c] * sc - zc_r[r];
        }
    }
}

// ---------------------------------------------------------------- 3. combine
__global__ void __launch_bounds__(128) prefill_combine_kernel(PrefillParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t nq = p.num_q;
    const int64_t wid = static_cast<int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (wid >= static_cast<int64_t>(p.B) * nq * p.Hq) return;
    const int h = static_cast<int>(wid % p.Hq);
    const int64_t bi = wid / p.Hq;
    const int b = static_cast<int>(bi / nq);
    const int64_t i = bi % nq;
    const int C = p.C, kvh = h / (p.Hq / p.Hkv);
    const int64_t qp = p.q_start[b] + i, T = p.seq_len[b];
    float M = p.ws_ml[wid * 2], L = p.ws_ml[wid * 2 + 1];
    float4 rot = M == -INFINITY ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(p.ws_o + wid * 128)[lane];
    if (M == -INFINITY) L = 0.f;
    float4 raw = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nsink = min(min(p.cache.sink_count[b], p.max_sinks), 16);
    if (nsink > 0) {
        float qd[4];
        const uint16_t* qh = p.q + (bi * p.Hq + h) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int d = 4 * lane + j, f = d & 63;
            const float a = h2f(qh[f]), bb = h2f(qh[f + 64]);
            const float2 r = rope_cs(p.rope, qp, f);
            qd[j] = (d < 64 ? (a * r.x - bb * r.y) : (a * r.y + bb * r.x)) * p.qscale;
        }
        for (int s = 0; s < nsink; ++s) {
            const int pos = p.cache.sink_pos[b * p.max_sinks + s];
            if (pos > qp || pos >= T) continue;
            const int64_t srow = (static_cast<int64_t>(b) * p.max_sinks + s) * C + kvh * 128;
            float prod = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int d = 4 * lane + j, f = d & 63;
                const float ka = h2f(p.cache.sink_k[srow + f]), kb = h2f(p.cache.sink_k[srow + f + 64]);
                const float2 rk = rope_cs(p.rope, pos, f);
                prod += qd[j] * (d < 64 ? (ka * rk.x - kb * rk.y) : (ka * rk.y + kb * rk.x));
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
            const float mn = fmaxf(M, prod);
            const float a = exp2f(M - mn), e = exp2f(prod - mn);
            L = L * a + e;
            rot = make_float4(rot.x * a, rot.y * a, rot.z * a, rot.w * a);
            const uint2 vv = *reinterpret_cast<const uint2*>(p.cache.sink_v + srow + 4 * lane);
            raw = make_float4(raw.x * a + e * h2f(static_cast<uint16_t>(vv.x & 0xffffu)),
                              raw.y * a + e * h2f(static_cast<uint16_t>(vv.x >> 16)),
                              raw.z * a + e * h2f(static_cast<uint16_t>(vv.y & 0xffffu)),
                              raw.w * a + e * h2f(static_cast<uint16_t>(vv.y >> 16)));
            M = mn;
        }
    }
    float x[4] = {rot.x, rot.y, rot.z, rot.w};
    {
        const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
        x[0] = a0 + a2;
        x[1] = a1 + a3;
        x[2] = a0 - a2;
        x[3] = a1 - a3;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const bool upper = lane & o;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float y = __shfl_xor_sync(0xffffffffu, x[j], o);
            x[j] = upper ? y - x[j] : x[j] + y;
        }
    }
    const float inv = L > 0.f ? 1.0f / L : 0.f, nrm = 1.0f / sqrtf(128.0f);
    reinterpret_cast<float4*>(p.out + wid * 128)[lane] =
        make_float4((x[0] * nrm + raw.x) * inv, (x[1] * nrm + raw.y) * inv, (x[2] * nrm + raw.z) * inv,
                    (x[3] * nrm + raw.w) * inv);
}

}  // namespace

size_t prefill_attn_smem() { return static_cast<size_t>(2 * kQB * kRowH) * 2 + 2 * static_cast<size_t>(kTileBytes); }

cudaError_t launch_prefill(const rkv_layer_desc& d, const PrefillParams& p, int64_t max_seq_len, cudaStream_t s) {
    const int C = p.C, W = C / 16, MG = C / 128;
    const int N = d.heads_per_group * d.head_dim, NG = C / N;
    const size_t ksmem = 2 * static_cast<size_t>(C) * 4 + 4 * static_cast<size_t>(W + MG) * 4;
    const int nthreads = std::min(512, std::max(NG * 32, ((2 * W + 31) / 32) * 32));
    const dim3 kgrid(static_cast<unsigned>((max_seq_len + 3) / 4), static_cast<unsigned>(d.batch));
    cudaError_t e;
    if (N == 512) {
        if ((e = cudaFuncSetAttribute(reconstruct_keys_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ksmem))) != cudaSuccess)
            return e;
        reconstruct_keys_kernel<4><<<kgrid, nthreads, ksmem, s>>>(p);
    } else if (N == 256) {
        if ((e = cudaFuncSetAttribute(reconstruct_keys_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ksmem))) != cudaSuccess)
            return e;
        reconstruct_keys_kernel<2><<<kgrid, nthreads, ksmem, s>>>(p);
    } else {
        return cudaErrorInvalidValue;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t asmem = prefill_attn_smem();
    if ((e = cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(asmem))) != cudaSuccess)
        return e;
    const dim3 agrid(static_cast<unsigned>((p.num_q + kQB - 1) / kQB), static_cast<unsigned>(p.Hq),
                     static_cast<unsigned>(d.batch));
    prefill_attn_kernel<<<agrid, 128, asmem, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int64_t warps = static_cast<int64_t>(d.batch) * p.num_q * p.Hq;
    prefill_combine_kernel<<<static_cast<unsigned>((warps + 3) / 4), 128, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace rkv
