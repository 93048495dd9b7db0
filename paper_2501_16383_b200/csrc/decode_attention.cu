// decode_attention.cu -- split-K decode attention over the 2-bit rotated cache.
//
// Restates the attention half of decode_step (proj/src/pipeline.cpp:133-152,
// 211-261) for B sequences at once:
//   keys   = RoPE_t( H_G^-1 . P^-1 . dequant(k') )    (reconstruct_cache)
//   query  = RoPE_{T-1}(q)                             (prepare_queries)
//   logits = q.k / sqrt(d), softmax, o' = sum p v'     (v' in the rotated frame)
//   out    = H_128 o'                                  (V's inverse rotation, W_o_f)
//
// B200 mapping.  Grid = splits x B (one CTA per SM, shared-memory bound);
// inside a CTA a "lane group" of L = 16 lanes (8 for G = 1) owns one FWHT
// group g (G KV heads = GH*REP q heads) and one token pair per tile.
//   * TMA bulk copies (cp.async.bulk -> UBLKCP) stream each tile of TT tokens
//     (packed K/V words, scale|zero words, the tile's RoPE rows) into an
//     NS-stage shared-memory ring guarded by mbarriers.
//   * K1 (all threads): each thread takes a whole packed word (one quant
//     group, one scale) for a token pair, dequantizes the 16 codes exactly
//     (s*(c-z), proj/src/quant.cpp:99-107) as FADD2/FMUL2 over the pair and
//     scatters them (STS.64) to their natural channel (slot j -> perm[j]) in
//     a pair-interleaved, XOR-swizzled fp32 tile.  __syncthreads.
//   * K2 (per lane group, no CTA barrier): inverse grouped FWHT (== forward,
//     proj/src/hadamard.cpp:75) on float2 = (token, token+1) registers:
//     layout A (LDS.128) -> butterfly stages on the low index bits -> STS.128
//     -> layout B (LDS.64) -> stages on the high bits; every butterfly is one
//     FADD2/FFMA2.  RoPE, q.k with 1/sqrt(n) folded into q; reduce-scatter
//     of the logits over the lane group.
//   * online softmax (exp2 domain) and V accumulation for the group's heads,
//     each lane owning VW packed V words: acc += 4ps*(1 + c/4) (codes turned
//     into floats by a mantissa OR, zero point folded once per token), never
//     materialising dequantized V.  __syncthreads closes the tile.
//   * every lane group writes its own (m, l, o') partial; the combine kernel
//     merges partials in a fixed order, adds the fp16 sink rows (computed
//     inline, natural frame) and applies H_128.  Deterministic.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "rkv_common.cuh"
#include "rkv_internal.h"
#include "rkv_layout.h"

namespace rkv {

namespace {

constexpr int kMaxStages = 4;

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float2 lds64(const unsigned char* p) { return *reinterpret_cast<const float2*>(p); }
// RoPE table rows are per position pair, 128 float4 (2 KB): [0, 64) section 1
// (cos p0, cos p1, sin p0, sin p1) per frequency; [64, 128) section 2 (one
// 32-float4 frequency-pair row per position, tensor-core decode).
__device__ __forceinline__ void sts64(uint32_t addr, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

struct SmemLayout {
    size_t stage_bytes, kc, km, vc, vm, rope;  // offsets inside one stage
    size_t stages, mbar, knat, q, addr, mask, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout smem_layout(int C, int Hq, int TT, int chunk, int N, int plan_smem_words,
                                                 int kStages) {
    SmemLayout s{};
    const int W = C / 16, MG = C / 128;
    s.kc = 0;
    s.km = align16(s.kc + size_t(TT) * W * 4);
    s.vc = align16(s.km + size_t(TT) * MG * 4);
    s.vm = align16(s.vc + size_t(TT) * W * 4);
    s.rope = align16(s.vm + size_t(TT) * MG * 4);
    s.stage_bytes = align16(s.rope + size_t(TT) * 64 * 8);
    s.stages = 0;
    s.mbar = s.stages + kStages * s.stage_bytes;
    s.knat = align16(s.mbar + kStages * 8);
    s.q = align16(s.knat + size_t(TT / 2) * knat_pair_f2(N, C) * 8);  // TT/2 token pairs
    s.addr = align16(s.q + size_t(Hq) * 128 * 4 * 3 / 2);              // padded q rows (<= 1.5x)
    s.mask = align16(s.addr + size_t(plan_smem_words) * 4);            // omega + scatter schedule
    s.total = align16(s.mask + size_t(chunk / 32 + 2) * 4);  // the split's sink-mask words
    return s;
}

template <int N>
constexpr int max_threads() { return N == 512 ? 320 : 256; }

template <int N, int REP>
__global__ void __launch_bounds__(max_threads<N>(), 1) decode_split_kernel(DecodeParams p) {
    constexpr int L = N >= 256 ? 16 : 8;  // lanes per FWHT group
    constexpr int R = N / L;              // float2 registers per lane (one token pair)
    constexpr int LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    constexpr int GH = N / 128;           // KV heads per FWHT group
    constexpr int JJ = 128 / L;           // layout-B registers per head
    constexpr int HALF = JJ / 2;          // RoPE partner distance (d vs d+64)
    constexpr int NV = GH * REP;          // q heads served by one group
    constexpr int V0 = 2 * NV;            // logits per token pair
    constexpr int WPG = GH * 8;           // packed V words per token per group
    constexpr int VW = WPG / L;           // V words per lane
    constexpr int VH = VW * REP;          // q heads per lane in the V phase
    constexpr int QS = JJ + 4;            // padded q_l row (conflict-free LDS.128)
    static_assert(R >= L && R >= 16, "layouts A/B must cover all index bits");
    static_assert(V0 <= L && WPG % L == 0 && VH <= 4, "unsupported (G, Hq/Hkv) combination");

    extern __shared__ __align__(128) unsigned char smem[];
    const int C = p.C, W = C / 16, MG = C / 128, Hq = p.Hq;
    const int NG = C / N, PP = p.P, TT = 2 * PP;
    const int kStages = p.stages;
    const SmemLayout lay = smem_layout(C, Hq, TT, p.chunk, N, 17 * W, kStages);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    unsigned char* knat = smem + lay.knat;
    float* q_l = reinterpret_cast<float*>(smem + lay.q);
    uint32_t* omega_s = reinterpret_cast<uint32_t*>(smem + lay.addr);   // [W]
    const uint4* saddr4 = reinterpret_cast<const uint4*>(omega_s + W);  // [4][W] x 4 scatter offsets
    uint32_t* mask_s = reinterpret_cast<uint32_t*>(smem + lay.mask);

    const int tid = threadIdx.x, NT = blockDim.x;
    const int lg = tid / L, lam = tid % L, lbase = (tid & 31) & ~(L - 1);
    const int g = lg % NG, pp = lg / NG;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    const int64_t tb = p.tok_begin ? p.tok_begin[b] : 0, te = p.tok_end ? lmin(p.tok_end[b], T) : T;
    const int64_t t_begin = tb + static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = lmin(te, t_begin + p.chunk);

    const bool bad_plan = !plan_matches(p.plan, kDecodeSimt, N, C);
    if (t_begin >= t_end || bad_plan) {  // empty split: neutral partials for every lane group (NaN: foreign plan)
        const float fill = bad_plan ? __int_as_float(0x7fc00000) : 0.0f;
        for (int i = tid; i < PP * Hq; i += NT) {
            const int64_t row = (static_cast<int64_t>(b) * p.NP + static_cast<int64_t>(split) * PP + i / Hq) * Hq + i % Hq;
            p.ws_ml[row * 2] = bad_plan ? fill : -INFINITY;
            p.ws_ml[row * 2 + 1] = fill;
            float4* o = reinterpret_cast<float4*>(p.ws_o + row * 128);
            for (int k = 0; k < 32; ++k) o[k] = make_float4(fill, fill, fill, fill);
        }
        return;
    }
    const int ntiles = static_cast<int>((t_end - t_begin + TT - 1) / TT);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;

    auto issue_tile = [&](int it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const uint32_t n = static_cast<uint32_t>(lmin(TT, t_end - t0));
        unsigned char* st = smem + lay.stages + (it % kStages) * lay.stage_bytes;
        uint64_t* bar = mbar + (it % kStages);
        const uint32_t bw = n * W * 4, bm = n * MG * 4, npr = (n + 1) >> 1;
        mbar_arrive_expect_tx(bar, 2 * bw + 2 * bm + npr * 1024);
        bulk_g2s(st + lay.kc, p.cache.k_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.km, p.cache.k_meta + (row0 + t0) * MG, bm, bar);
        bulk_g2s(st + lay.vc, p.cache.v_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.vm, p.cache.v_meta + (row0 + t0) * MG, bm, bar);
        for (uint32_t r = 0; r < npr; ++r)  // section 1 of each position-pair row
            bulk_g2s(st + lay.rope + r * 1024, p.rope + ((t0 >> 1) + r) * kRopeRow, 1024, bar);
    };

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(mbar + s, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < kStages - 1 && it < ntiles; ++it) issue_tile(it);

    // the layer's scatter plan (rkv_plan.cu): word assignment + scatter offsets
    {
        const uint4* src = reinterpret_cast<const uint4*>(p.plan + kPlanHeader);
        uint4* dst = reinterpret_cast<uint4*>(omega_s);
        const int n4 = 17 * W / 4;
        for (int i = tid; i < n4; i += NT) dst[i] = __ldg(src + i);
    }

    // q: RoPE at position T-1 (prepare_queries), x log2(e)/sqrt(d) x 1/sqrt(n)
    // (the FWHT normalisation), lane-major: q_l[(h*L + lam)*QS + jj] = q[h][lam + L*jj]
    {
        const float4* cs = p.rope + ((T - 1) >> 1) * kRopeRow;
        const bool odd = (T - 1) & 1;
        const uint16_t* qb = p.q + static_cast<int64_t>(b) * Hq * 128;
        const float qs = p.qscale * p.k_norm;
        for (int i = tid; i < Hq * 64; i += NT) {
            const int h = i >> 6, f = i & 63;
            const float a = h2f(qb[h * 128 + f]), bb = h2f(qb[h * 128 + f + 64]);
            const float4 r4 = __ldg(cs + f);
            const float2 r = odd ? make_float2(r4.y, r4.w) : make_float2(r4.x, r4.z);
            q_l[(h * L + f % L) * QS + f / L] = (a * r.x - bb * r.y) * qs;
            q_l[(h * L + (f + 64) % L) * QS + (f + 64) / L] = (a * r.y + bb * r.x) * qs;
        }
    }

    // the split's sink-mask words (bit t%32 of word t/32 = sink), so no thread
    // touches global memory for token validity inside the tile loop
    const int64_t mw0 = t_begin >> 5;
    {
        const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
        const int nw = static_cast<int>(((t_end - 1) >> 5) - mw0 + 1);
        for (int i = tid; i < nw; i += NT) mask_s[i] = smask[mw0 + i];
    }

    // per-lane constants (padded rows: see rkv_layout.h)
    constexpr int RS = R + 1;                                 // row stride in float2
    const int pair_bytes = knat_pair_f2(N, C) * 8;
    unsigned char* kpair = knat + pp * pair_bytes;           // this lane group's token pair
    unsigned char* kunit = kpair + g * L * RS * 8;           // its FWHT group
    unsigned char* arow = kunit + lam * RS * 8;              // its layout-A row

    float m_run[VH], l_run[VH], zc[VH];
    float2 acc[VH][8];
#pragma unroll
    for (int v = 0; v < VH; ++v) {
        m_run[v] = -INFINITY;
        l_run[v] = 0.f;
        zc[v] = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[v][e] = make_float2(0.f, 0.f);
    }
    __syncthreads();  // plan and q_l complete

    // K1 item mapping (loop invariant; plan_decode guarantees NT % W == 0 or
    // W % NT == 0): thread -> word position k1w (+NT...), token pairs k1p0,
    // k1p0+k1ps, ...; a half-warp = 16 consecutive word positions
    const int k1w = NT >= W ? tid % W : tid;
    const int k1p0 = __shfl_sync(0xffffffffu, NT >= W ? tid / W : 0, 0);  // warp-uniform (W % 32 == 0)
    const int k1ps = NT >= W ? NT / W : 1;

    for (int it = 0; it < ntiles; ++it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const int nv = static_cast<int>(lmin(TT, t_end - t0));
        const unsigned char* st = smem + lay.stages + (it % kStages) * lay.stage_bytes;
        const uint32_t* kc = reinterpret_cast<const uint32_t*>(st + lay.kc);
        const uint32_t* km = reinterpret_cast<const uint32_t*>(st + lay.km);
        const uint32_t* vc = reinterpret_cast<const uint32_t*>(st + lay.vc);
        const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + lay.vm);
        const float4* rope4 = reinterpret_cast<const float4*>(st + lay.rope);
        mbar_wait(mbar + (it % kStages), (it / kStages) & 1);

        // ---- K1: dequantize a word for a token pair + scatter (STS.64); pq is
        // warp-uniform, so the pair offset rides in a uniform register
        for (int wp = k1w; wp < W; wp += NT) {
            const int w = omega_s[wp];
            uint32_t ad[16];  // scatter offsets of the word's 16 codes, reused for every pair
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const uint4 a4 = saddr4[q4 * W + wp];
                ad[4 * q4] = a4.x;
                ad[4 * q4 + 1] = a4.y;
                ad[4 * q4 + 2] = a4.z;
                ad[4 * q4 + 3] = a4.w;
            }
            for (int pq = k1p0; pq < PP; pq += k1ps) {
                const int tt0 = 2 * pq;
                if (tt0 >= nv) break;
                const bool has1 = tt0 + 1 < nv;
                const uint32_t w0 = kc[tt0 * W + w], w1 = has1 ? kc[(tt0 + 1) * W + w] : 0u;
                const uint32_t m0 = km[tt0 * MG + (w >> 3)], m1 = has1 ? km[(tt0 + 1) * MG + (w >> 3)] : 0u;
                // x = 1 + c/4 (code OR'd into the mantissa): s*(c - z) = x*(4s) - (4 + z)*s,
                // every term exact, so one FFMA2 per token pair
                const float s0 = h2f(static_cast<uint16_t>(m0 & 0xffffu)), s1 = h2f(static_cast<uint16_t>(m1 & 0xffffu));
                const float2 s4 = make_float2(4.0f * s0, 4.0f * s1);
                const float2 nzb = make_float2(-(4.0f + h2f(static_cast<uint16_t>(m0 >> 16))) * s0,
                                               -(4.0f + h2f(static_cast<uint16_t>(m1 >> 16))) * s1);
                const uint32_t dst = smem_u32(knat) + pq * pair_bytes;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int sh = 21 - 2 * e;
                    const uint32_t a0 = sh >= 0 ? (w0 << sh) : (w0 >> -sh);
                    const uint32_t a1 = sh >= 0 ? (w1 << sh) : (w1 >> -sh);
                    const float2 xx = make_float2(__uint_as_float(and_or(a0, 0x600000u, 0x3F800000u)),
                                                  __uint_as_float(and_or(a1, 0x600000u, 0x3F800000u)));
                    sts64(dst + ad[e], fma2(xx, s4, nzb));
                }
            }
        }
        __syncthreads();
        if (tid == 0 && it + kStages - 1 < ntiles) issue_tile(it + kStages - 1);

        // ---- K2: inverse grouped FWHT of the lane group's token pair
        const int tt0 = 2 * pp;
        float2 x[R];
#pragma unroll
        for (int j = 0; j < R; ++j) x[j] = lds64(arow + 8 * j);
        bfly_range<R, 0, LR>(x);
        {
            const uint32_t a = smem_u32(arow);
#pragma unroll
            for (int j = 0; j < R; ++j) sts64(a + 8 * j, x[j]);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < R; ++j) {
            // channel lam + L*j of the group: row (L*j)/R, column lam + (L*j)%R
            x[j] = lds64(kunit + (((L * j) >> LR) * RS + ((L * j) & (R - 1)) + lam) * 8);
        }
        bfly_range<R, LR - LL, LN - LL>(x);

        // RoPE at each token's position, dot with the group's q heads
        float2 part[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) part[v] = make_float2(0.f, 0.f);
#pragma unroll
        for (int jj = 0; jj < HALF; ++jj) {
            const int f = lam + L * jj;  // frequency of (d, d+64)
            // pair-interleaved table row: (cos t0, cos t1, sin t0, sin t1)
            const float4 cq = rope4[pp * 64 + f];
            const float2 cs = make_float2(cq.x, cq.y), sn = make_float2(cq.z, cq.w);
#pragma unroll
            for (int hh = 0; hh < GH; ++hh) {
                const float2 a = x[hh * JJ + jj], bb = x[hh * JJ + jj + HALF];
                const float2 ar = fma2(a, cs, mul2(make_float2(-bb.x, -bb.y), sn));  // a c - b s
                const float2 br = fma2(a, sn, mul2(bb, cs));                         // a s + b c
#pragma unroll
                for (int r = 0; r < REP; ++r) {
                    const float* qh = q_l + (((g * GH + hh) * REP + r) * L + lam) * QS;
                    const float qa = qh[jj], qb = qh[jj + HALF];
                    part[hh * REP + r] = fma2(make_float2(qa, qa), ar, part[hh * REP + r]);
                    part[hh * REP + r] = fma2(make_float2(qb, qb), br, part[hh * REP + r]);
                }
            }
        }
        // reduce-scatter the V0 = 2*NV partials over the L lanes; afterwards lane
        // lam holds value (lam >> SH) = 2*local_head + token
        float val[V0];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            val[2 * v] = part[v].x;
            val[2 * v + 1] = part[v].y;
        }
        {
            int nvals = V0;
#pragma unroll
            for (int stp = L / 2; stp >= 1; stp >>= 1) {
                const bool upper = (lam & stp) != 0;
                if (nvals > 1) {
                    const int hv = nvals / 2;
#pragma unroll
                    for (int i = 0; i < V0 / 2; ++i) {
                        if (i < hv) {
                            const float send = upper ? val[i] : val[i + hv];
                            const float keep = upper ? val[i + hv] : val[i];
                            val[i] = keep + __shfl_xor_sync(0xffffffffu, send, stp);
                        }
                    }
                    nvals = hv;
                } else {
                    val[0] += __shfl_xor_sync(0xffffffffu, val[0], stp);
                }
            }
        }
        constexpr int SH = LL - ilog2(V0);

        // ---- online softmax for the lane's V heads (replicated per lane)
        bool ok0, ok1;
        {
            const int64_t ta = t0 + tt0, tb = ta + 1;
            ok0 = tt0 < nv && !((mask_s[(ta >> 5) - mw0] >> (ta & 31)) & 1u);
            ok1 = tt0 + 1 < nv && !((mask_s[(tb >> 5) - mw0] >> (tb & 31)) & 1u);
        }
        float pr0[VH], pr1[VH];
#pragma unroll
        for (int v = 0; v < VH; ++v) {
            const int i = v / REP, r = v % REP;
            const int kvl = (lam + L * i) >> 3;
            const int hv = kvl * REP + r;
            const float l0 = __shfl_sync(0xffffffffu, val[0], lbase + ((2 * hv) << SH));
            const float l1 = __shfl_sync(0xffffffffu, val[0], lbase + ((2 * hv + 1) << SH));
            const float mx = fmaxf(ok0 ? l0 : -INFINITY, ok1 ? l1 : -INFINITY);
            const float m_new = fmaxf(m_run[v], mx);
            const float alpha = (m_new == -INFINITY) ? 1.0f : exp2f(m_run[v] - m_new);
            pr0[v] = ok0 ? exp2f(l0 - m_new) : 0.0f;
            pr1[v] = ok1 ? exp2f(l1 - m_new) : 0.0f;
            l_run[v] = l_run[v] * alpha + pr0[v] + pr1[v];
            m_run[v] = m_new;
            zc[v] *= alpha;
            const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[v][e] = mul2(acc[v][e], a2);
        }

        // ---- V: acc += 4 p s (1 + c/4); zero point and the +1 folded into zc
#pragma unroll
        for (int i = 0; i < VW; ++i) {
            const int gw = g * WPG + lam + L * i;
            const uint32_t w0 = vc[tt0 * W + gw], w1 = vc[(tt0 + 1) * W + gw];
            const uint32_t m0 = vm[tt0 * MG + (gw >> 3)], m1 = vm[(tt0 + 1) * MG + (gw >> 3)];
            float2 xa[8], xb[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int s0 = 21 - 2 * e, s1 = 21 - 2 * (e + 8);
                const uint32_t ca = s0 >= 0 ? (w0 << s0) : (w0 >> -s0);
                const uint32_t cb = s1 >= 0 ? (w0 << s1) : (w0 >> -s1);
                const uint32_t cc = s0 >= 0 ? (w1 << s0) : (w1 >> -s0);
                const uint32_t cd = s1 >= 0 ? (w1 << s1) : (w1 >> -s1);
                xa[e] = make_float2(__uint_as_float(and_or(ca, 0x600000u, 0x3F800000u)),
                                    __uint_as_float(and_or(cb, 0x600000u, 0x3F800000u)));
                xb[e] = make_float2(__uint_as_float(and_or(cc, 0x600000u, 0x3F800000u)),
                                    __uint_as_float(and_or(cd, 0x600000u, 0x3F800000u)));
            }
            const float s0 = h2f(static_cast<uint16_t>(m0 & 0xffffu)), z0 = h2f(static_cast<uint16_t>(m0 >> 16));
            const float s1 = h2f(static_cast<uint16_t>(m1 & 0xffffu)), z1 = h2f(static_cast<uint16_t>(m1 >> 16));
#pragma unroll
            for (int r = 0; r < REP; ++r) {
                const int v = i * REP + r;
                const float ps0 = pr0[v] > 0.0f ? pr0[v] * s0 : 0.0f;
                const float ps1 = pr1[v] > 0.0f ? pr1[v] * s1 : 0.0f;
                // garbage metadata of masked tokens never reaches the sums
                zc[v] += (ps0 != 0.0f ? ps0 * (z0 + 4.0f) : 0.0f) + (ps1 != 0.0f ? ps1 * (z1 + 4.0f) : 0.0f);
                const float2 f0 = make_float2(4.0f * ps0, 4.0f * ps0), f1 = make_float2(4.0f * ps1, 4.0f * ps1);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    acc[v][e] = fma2(f0, xa[e], acc[v][e]);
                    acc[v][e] = fma2(f1, xb[e], acc[v][e]);
                }
            }
        }
        __syncthreads();  // knat and this stage are free for the next tile
    }

    // ---- this lane group's partial (m, l, o')
    const int64_t prow = static_cast<int64_t>(b) * p.NP + static_cast<int64_t>(split) * PP + pp;
#pragma unroll
    for (int v = 0; v < VH; ++v) {
        const int i = v / REP, r = v % REP;
        const int wl = lam + L * i;
        const int h = (g * GH + (wl >> 3)) * REP + r;
        const int64_t row = prow * Hq + h;
        if ((wl & 7) == 0) {
            p.ws_ml[row * 2] = m_run[v];
            p.ws_ml[row * 2 + 1] = l_run[v];
        }
        float4* o = reinterpret_cast<float4*>(p.ws_o + row * 128 + (wl & 7) * 16);
        const float z = zc[v];
        o[0] = make_float4(acc[v][0].x - z, acc[v][1].x - z, acc[v][2].x - z, acc[v][3].x - z);
        o[1] = make_float4(acc[v][4].x - z, acc[v][5].x - z, acc[v][6].x - z, acc[v][7].x - z);
        o[2] = make_float4(acc[v][0].y - z, acc[v][1].y - z, acc[v][2].y - z, acc[v][3].y - z);
        o[3] = make_float4(acc[v][4].y - z, acc[v][5].y - z, acc[v][6].y - z, acc[v][7].y - z);
    }
}

// Merge the NP partials of (b, h) (rotated V frame) in a fixed order (online,
// deterministic), add the sink tokens' raw fp16 rows (natural frame, RoPE at
// their own position, kept exact like the reference's sidecar), then
// out = (H_128 o'_rot / sqrt(128) + o_sink) / l.  One warp per (b, h); lane
// owns channels 4*lane .. 4*lane+3, so H_128 is 2 register stages + 5 shuffle
// stages and the sink dot products are warp reductions.
__global__ void __launch_bounds__(256) decode_combine_kernel(DecodeParams p, int nw) {
    // the queries, lengths, RoPE table and sink rows predate the split kernel
    // (it waited for them): requested while it drains; the partials after
    // pdl_wait below
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // nw == 1: four (b, h) per CTA, a warp merges all partials; nw > 1 (few
    // heads, many partials): a CTA per (b, h), warp w merges the w-th range of
    // partials and warp 0 folds the nw results in order
    const int64_t wid = nw == 1 ? static_cast<int64_t>(blockIdx.x) * 4 + warp : blockIdx.x;
    if (wid >= static_cast<int64_t>(p.B) * p.Hq) return;
    const int span = (p.NP + nw - 1) / nw;
    const int s_begin = nw == 1 ? 0 : warp * span, s_end = nw == 1 ? p.NP : min(p.NP, s_begin + span);
    const int b = static_cast<int>(wid / p.Hq), h = static_cast<int>(wid % p.Hq), C = p.C;
    const int64_t base = static_cast<int64_t>(b) * p.NP * p.Hq;
    const int64_t T = p.seq_len[b];
    const int kvh = h / (p.Hq / p.Hkv);
    // merge the packed partials: lanes fetch (m, l) of 32 partials at a time,
    // the warp max fixes the weights, then the o' rows are summed with loads
    // that do not depend on each other (unrolled), in a fixed order
    // Latency-bound (a few warps per SM): everything that does not depend on
    // the partials' weights is requested up front -- the o' rows of the first
    // 32 partials, the query values and RoPE row for the sink logits.
    const int nsink = p.partial_ml ? 0 : min(p.cache.sink_count[b], p.max_sinks);
    float qraw[8];
    float2 rq[4];
    if (warp == 0 || nw == 1) {
        const uint16_t* qh = p.q + (static_cast<int64_t>(b) * p.Hq + h) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int f = (4 * lane + j) & 63;
            qraw[2 * j] = h2f(qh[f]);
            qraw[2 * j + 1] = h2f(qh[f + 64]);
            rq[j] = rope_at(p.rope, T - 1, f);
        }
    }
    // the first sinks' raw rows and positions, requested before the merge
    // (their RoPE rows once the positions are in): one round trip for all of
    // them instead of one per sink after it
    constexpr int kSP = 4;
    const int npre = min(nsink, kSP);
    int spos[kSP];
    uint2 ska[kSP], skb[kSP], sva[kSP];
    if (warp == 0 || nw == 1) {
        const int f0 = (4 * lane) & 63;
#pragma unroll
        for (int s = 0; s < kSP; ++s) {
            if (s >= npre) break;
            const int64_t srow = (static_cast<int64_t>(b) * p.max_sinks + s) * C + kvh * 128;
            spos[s] = p.cache.sink_pos[b * p.max_sinks + s];
            ska[s] = *reinterpret_cast<const uint2*>(p.cache.sink_k + srow + f0);
            skb[s] = *reinterpret_cast<const uint2*>(p.cache.sink_k + srow + f0 + 64);
            sva[s] = *reinterpret_cast<const uint2*>(p.cache.sink_v + srow + 4 * lane);
        }
    }
    pdl_wait();  // the split kernel's partials
    float4 ov[32];
    {
        const int n0 = min(32, s_end - s_begin);
        const float4* src = reinterpret_cast<const float4*>(p.ws_o + (base + static_cast<int64_t>(s_begin) * p.Hq + h) * 128) + lane;
        const int64_t stride = static_cast<int64_t>(p.Hq) * 32;  // float4 per partial row step
#pragma unroll
        for (int k = 0; k < 32; ++k) ov[k] = k < n0 ? src[k * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float M = -INFINITY, L = 0.f;
    float4 rot = make_float4(0.f, 0.f, 0.f, 0.f);
    bool poisoned = false;  // a partial's m is NaN: the decode kernel rejected the layer plan
    for (int s0 = s_begin; s0 < s_end; s0 += 32) {
        const int s = s0 + lane;
        const int64_t r = base + static_cast<int64_t>(s) * p.Hq + h;
        const float ms = s < s_end ? p.ws_ml[r * 2] : -INFINITY;
        const float ls = s < s_end ? p.ws_ml[r * 2 + 1] : 0.f;
        poisoned |= __any_sync(0xffffffffu, ms != ms);
        float mx = ms;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (mx == -INFINITY) continue;
        const float mn = fmaxf(M, mx);
        const float a = exp2f(M - mn);
        const float w = ms == -INFINITY ? 0.f : exp2f(ms - mn);
        float lw = w * ls;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o);
        L = L * a + lw;
        rot = make_float4(rot.x * a, rot.y * a, rot.z * a, rot.w * a);
        M = mn;
        const int n = min(32, s_end - s0);
        if (s0 > s_begin) {  // partials beyond the first 32 (long sequences with many splits)
            const float4* src = reinterpret_cast<const float4*>(p.ws_o + (base + static_cast<int64_t>(s0) * p.Hq + h) * 128) + lane;
            const int64_t stride = static_cast<int64_t>(p.Hq) * 32;
#pragma unroll
            for (int k = 0; k < 32; ++k) ov[k] = k < n ? src[k * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const float wk = __shfl_sync(0xffffffffu, w, k);  // 0 past n (ms = -inf)
            rot = make_float4(rot.x + wk * ov[k].x, rot.y + wk * ov[k].y, rot.z + wk * ov[k].z, rot.w + wk * ov[k].w);
        }
    }
    if (poisoned) {  // keep the NaN visible through the fold and the normalisation
        M = 0.f;
        L = __int_as_float(0x7fc00000);
    }
    if (nw > 1) {  // fold the warps' (M, L, rot) in warp order
        __shared__ float4 s_rot[8][32];
        __shared__ float s_ml[8][2];
        s_rot[warp][lane] = rot;
        if (lane == 0) {
            s_ml[warp][0] = M;
            s_ml[warp][1] = L;
        }
        __syncthreads();
        if (warp != 0) return;
        for (int w = 1; w < nw; ++w) {
            const float mw = s_ml[w][0];
            if (mw == -INFINITY) continue;
            const float mn = fmaxf(M, mw), a = exp2f(M - mn), c = exp2f(mw - mn);
            const float4 r = s_rot[w][lane];
            L = L * a + s_ml[w][1] * c;
            rot = make_float4(rot.x * a + r.x * c, rot.y * a + r.y * c, rot.z * a + r.z * c, rot.w * a + r.w * c);
            M = mn;
        }
    }
    if (p.partial_ml) {  // sequence-parallel partial: merged (m, l) and the unnormalised rotated o'
        if (lane == 0) {
            p.partial_ml[wid * 2] = M;
            p.partial_ml[wid * 2 + 1] = L;
        }
        reinterpret_cast<float4*>(p.out + wid * 128)[lane] = rot;
        return;
    }
    // sinks: logits from q and the raw fp16 key rows, both RoPE'd (log2 domain)
    float4 raw = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nsink > 0) {
        float qd[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int d = 4 * lane + j;
            const float a = qraw[2 * j], bb = qraw[2 * j + 1];
            const float2 r = rq[j];
            qd[j] = (d < 64 ? (a * r.x - bb * r.y) : (a * r.y + bb * r.x)) * p.qscale;
        }
        // one sink: logit from its RoPE'd raw key (k2a: dims f..f+3, k2b: f+64..,
        // f = (4 lane) & 63), online-softmax fold, raw V row
        auto fold_sink = [&](int pos, uint2 k2a, uint2 k2b, const float2 (&rk)[4], uint2 vv) {
            const uint16_t kah[4] = {static_cast<uint16_t>(k2a.x & 0xffffu), static_cast<uint16_t>(k2a.x >> 16),
                                     static_cast<uint16_t>(k2a.y & 0xffffu), static_cast<uint16_t>(k2a.y >> 16)};
            const uint16_t kbh[4] = {static_cast<uint16_t>(k2b.x & 0xffffu), static_cast<uint16_t>(k2b.x >> 16),
                                     static_cast<uint16_t>(k2b.y & 0xffffu), static_cast<uint16_t>(k2b.y >> 16)};
            float prod = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int d = 4 * lane + j;
                const float ka = h2f(kah[j]), kb = h2f(kbh[j]);
                prod += qd[j] * (d < 64 ? (ka * rk[j].x - kb * rk[j].y) : (ka * rk[j].y + kb * rk[j].x));
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
            const float mn = fmaxf(M, prod);
            const float a = exp2f(M - mn), e = exp2f(prod - mn);
            L = L * a + e;
            rot = make_float4(rot.x * a, rot.y * a, rot.z * a, rot.w * a);
            raw = make_float4(raw.x * a + e * h2f(static_cast<uint16_t>(vv.x & 0xffffu)),
                              raw.y * a + e * h2f(static_cast<uint16_t>(vv.x >> 16)),
                              raw.z * a + e * h2f(static_cast<uint16_t>(vv.y & 0xffffu)),
                              raw.w * a + e * h2f(static_cast<uint16_t>(vv.y >> 16)));
            M = mn;
        };
        float2 srk[kSP][4];  // the prefetched sinks' RoPE rows, all requested at once
#pragma unroll
        for (int s = 0; s < kSP; ++s) {
            if (s >= npre) break;
#pragma unroll
            for (int j = 0; j < 4; ++j) srk[s][j] = rope_at(p.rope, spos[s] < T ? spos[s] : 0, (4 * lane + j) & 63);
        }
#pragma unroll
        for (int s = 0; s < kSP; ++s) {
            if (s >= npre) break;
            if (spos[s] < T) fold_sink(spos[s], ska[s], skb[s], srk[s], sva[s]);
        }
        for (int s = kSP; s < nsink; ++s) {  // beyond the prefetched ones
            const int pos = p.cache.sink_pos[b * p.max_sinks + s];
            if (pos >= T) continue;
            const int64_t srow = (static_cast<int64_t>(b) * p.max_sinks + s) * C + kvh * 128;
            const int f0 = (4 * lane) & 63;
            float2 rk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) rk[j] = rope_at(p.rope, pos, f0 + j);
            fold_sink(pos, *reinterpret_cast<const uint2*>(p.cache.sink_k + srow + f0),
                      *reinterpret_cast<const uint2*>(p.cache.sink_k + srow + f0 + 64), rk,
                      *reinterpret_cast<const uint2*>(p.cache.sink_v + srow + 4 * lane));
        }
    }
    // H_128 on the rotated-frame accumulator (value_rotation inverse): index
    // bits 0-1 in registers, bits 2-6 across lanes (xor 1..16)
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
    pdl_trigger();  // the next kernel may launch while the combine drains
    const float inv = (L > 0.f || L != L) ? 1.0f / L : 0.f, nrm = 1.0f / sqrtf(128.0f);  // NaN L: foreign plan
    reinterpret_cast<float4*>(p.out + (static_cast<int64_t>(b) * p.Hq + h) * 128)[lane] =
        make_float4((x[0] * nrm + raw.x) * inv, (x[1] * nrm + raw.y) * inv, (x[2] * nrm + raw.z) * inv,
                    (x[3] * nrm + raw.w) * inv);
}

// table[pos/2][f] = (cos(p0 th_f), cos(p1 th_f), sin(p0 th_f), sin(p1 th_f)),
// p0 = pos & ~1, p1 = p0 + 1: a token pair's rotation is one LDS.128
// (section 1 of the kRopeRow-float4 position-pair row).
__global__ void rope_table_kernel(float4* table, int64_t npairs, double base) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= npairs * 64) return;
    const int64_t pr = i / 64;
    const int f = static_cast<int>(i % 64);
    const double theta = pow(base, -2.0 * static_cast<double>(f) / 128.0);  // proj/src/rope.cpp:17-24
    const double a0 = 1.0 * static_cast<double>(2 * pr) * theta;            // dir * pos * theta
    const double a1 = 1.0 * static_cast<double>(2 * pr + 1) * theta;
    table[pr * kRopeRow + f] = make_float4(static_cast<float>(cos(a0)), static_cast<float>(cos(a1)),
                                           static_cast<float>(sin(a0)), static_cast<float>(sin(a1)));
}

// Second section (tensor-core decode): token-major, one float4 per frequency
// pair (f, f+1) = 2j, 2j+1:  G = 4: (u_f, u_f+1, w_f, w_f+1), u = cos - sin,
// w = cos + sin (the bit-6 butterfly folded into RoPE, decode_mma.cu);
// otherwise (cos_f, cos_f+1, sin_f, sin_f+1).  Evaluated in double.
__global__ void rope_table2_kernel(float4* table, int64_t npos, double base, int fold) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= npos * 32) return;
    const int64_t pos = i / 32;
    const int j = static_cast<int>(i % 32);
    double c[2], sn[2];
    for (int k = 0; k < 2; ++k) {
        const double theta = pow(base, -2.0 * static_cast<double>(2 * j + k) / 128.0);
        c[k] = cos(static_cast<double>(pos) * theta);
        sn[k] = sin(static_cast<double>(pos) * theta);
    }
    table[(pos >> 1) * kRopeRow + 64 + (pos & 1) * 32 + rope_pair_slot(j)] = fold ? make_float4(static_cast<float>(c[0] - sn[0]), static_cast<float>(c[1] - sn[1]),
                                  static_cast<float>(c[0] + sn[0]), static_cast<float>(c[1] + sn[1]))
                    : make_float4(static_cast<float>(c[0]), static_cast<float>(c[1]), static_cast<float>(sn[0]),
                                  static_cast<float>(sn[1]));
}

constexpr int kRotRows = 8;  // rows per rotate_keys CTA

template <int N, int L>
// CTA = kRotRows rows x L lanes (one FWHT unit u = blockIdx.y of each row); rows
// on grid.x (2^31 - 1 blocks), so calibration sets of any practical size
// launch in one go.  The L lanes of a row sit in one warp: __syncwarp orders
// the shared-memory transpose.
__global__ void rotate_keys_kernel(const uint16_t* __restrict__ k, int64_t rows, int C, float norm, float* out) {
    constexpr int R = N / L, LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    const int rr = threadIdx.x / L, lam = threadIdx.x % L;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / L) + rr;
    const int u = blockIdx.y;
    __shared__ float buf[kRotRows][N];
    const bool ok = r < rows;
    const uint16_t* src = k + (ok ? r : 0) * C + u * N;
    float2 x[R];
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = make_float2(ok ? h2f(src[lam * R + j]) : 0.f, 0.f);
    bfly_range<R, 0, LR>(x);
#pragma unroll
    for (int j = 0; j < R; ++j) buf[rr][lam * R + j] = x[j].x;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = make_float2(buf[rr][lam + L * j], 0.f);
    bfly_range<R, LR - LL, LN - LL>(x);
    if (!ok) return;
#pragma unroll
    for (int j = 0; j < R; ++j) out[r * C + u * N + lam + L * j] = __fmul_rn(x[j].x, norm);
}

// Per-channel calibration statistic (proj/src/reorder.cpp:98-105): thread c
// accumulates sum_r x[r][c] (or |x|) in double over r = 0, 1, ... in order --
// the reference's summation order, so the result is bit-identical.  Reads are
// coalesced across threads (consecutive channels).
__global__ void channel_stats_kernel(const float* __restrict__ x, int64_t rows, int64_t C, int mean_abs,
                                     double* __restrict__ out) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double acc = 0.0;
    for (int64_t r = 0; r < rows; ++r) {
        const double v = x[r * C + c];
        acc += mean_abs ? fabs(v) : v;
    }
    out[c] = mean_abs ? acc / static_cast<double>(rows) : acc;
}

template <int N, int REP>
cudaError_t launch_decode_nr(const DecodePlan& plan, const DecodeParams& p, int B, cudaStream_t s) {
    auto kern = decode_split_kernel<N, REP>;
    cudaError_t e = ensure_smem_k(kern, plan.smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(plan.S, B), plan.NT, plan.smem, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_decode_combine(p, B, s);
}

}  // namespace

cudaError_t launch_decode_combine(const DecodeParams& p, int B, cudaStream_t s) {
    const int64_t heads = static_cast<int64_t>(B) * p.Hq;
    // few heads and many partials (small batch, long splits): one CTA per head,
    // up to 8 warps each merging a range of partials
    const int nw = heads < 2 * num_sms() ? static_cast<int>(std::min<int64_t>(8, (p.NP + 31) / 32)) : 1;
    if (nw > 1) return launch_pdl(decode_combine_kernel, dim3(static_cast<unsigned>(heads)), dim3(32 * nw), 0, s, p, nw);
    return launch_pdl(decode_combine_kernel, dim3(static_cast<unsigned>((heads + 3) / 4)), dim3(128), 0, s, p, 1);
}

template <int N, int REP>
int occupancy_nr(const DecodePlan& pl) {
    int n = 0;
    if (ensure_smem_k(decode_split_kernel<N, REP>, pl.smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_split_kernel<N, REP>, pl.NT, pl.smem) != cudaSuccess) {
        cudaGetLastError();
        const int by_smem = static_cast<int>((227u * 1024u) / (pl.smem + 1024));
        return std::max(1, by_smem);
    }
    return std::max(1, n);
}

int occupancy(const DecodePlan& pl) {
    switch (pl.N * 16 + pl.REP) {
        case 512 * 16 + 1: return occupancy_nr<512, 1>(pl);
        case 512 * 16 + 2: return occupancy_nr<512, 2>(pl);
        case 256 * 16 + 1: return occupancy_nr<256, 1>(pl);
        case 256 * 16 + 2: return occupancy_nr<256, 2>(pl);
        case 256 * 16 + 4: return occupancy_nr<256, 4>(pl);
        case 128 * 16 + 1: return occupancy_nr<128, 1>(pl);
        case 128 * 16 + 2: return occupancy_nr<128, 2>(pl);
        case 128 * 16 + 4: return occupancy_nr<128, 4>(pl);
        default: return 1;
    }
}

bool decode_supported(int N, int REP) {
    switch (N) {
        case 512: return REP == 1 || REP == 2;
        case 256: return REP == 1 || REP == 2 || REP == 4;
        case 128: return REP == 1 || REP == 2 || REP == 4;
        default: return false;
    }
}

// The CUDA-core split kernel's shape limits (plan_decode below, without the
// occupancy query): rotation size 128/256/512, its head ratios, C % 512 == 0
// and a thread count that tiles the packed words.
bool simt_shape_ok(const rkv_layer_desc& d) {
    const int C = d.num_kv_heads * d.head_dim, N = d.heads_per_group * d.head_dim;
    if (d.head_dim != 128 || C % 512 != 0 || (N != 128 && N != 256 && N != 512)) return false;
    if (d.num_q_heads % d.num_kv_heads != 0 || !decode_supported(N, d.num_q_heads / d.num_kv_heads)) return false;
    const int L = N >= 256 ? 16 : 8, NG = C / N, max_nt = N == 512 ? 320 : 256, W = C / 16;
    const int P = std::max(1, std::min(4, max_nt / (NG * L)));
    const int NT = NG * P * L;
    if (NT > max_nt || !(NT % W == 0 || W % NT == 0)) return false;
    return smem_layout(C, d.num_q_heads, 2 * P, 16 + 2 * P, N, 17 * W, 3).total <= 227 * 1024;
}

DecodePlan plan_decode(const rkv_layer_desc& d, int64_t max_seq_len) {
    const int kind = decode_kind(d);
    if (kind == kDecodeMma) return plan_decode_mma(d, max_seq_len);
    if (kind == kDecodeGeneric) return plan_decode_generic(d, max_seq_len);
    DecodePlan pl{};
    pl.kind = kDecodeSimt;
    const int C = d.num_kv_heads * d.head_dim;
    pl.N = d.heads_per_group * d.head_dim;
    pl.REP = d.num_q_heads / d.num_kv_heads;
    const int L = pl.N >= 256 ? 16 : 8;
    const int NG = C / pl.N;
    const int max_nt = pl.N == 512 ? 320 : 256;
    int P = max_nt / (NG * L);
    if (P > 4) P = 4;
    if (P < 1) P = 1;
    pl.stages = 3;
    if (const int o = options().simt_p.load()) P = std::max(1, std::min(P, o));  // experiment switches
    if (const int o = options().simt_stages.load()) pl.stages = std::max(2, std::min(kMaxStages, o));
    pl.P = P;
    pl.TT = 2 * P;
    pl.NT = NG * P * L;
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    // CTAs resident per SM (shared memory and registers decide)
    pl.smem = smem_layout(C, d.num_q_heads, pl.TT, static_cast<int>(max_seq_len) + pl.TT, pl.N, 17 * (C / 16),
                          pl.stages).total;  // upper bound (chunk <= max_seq_len)
    pl.per_sm = occupancy(pl);
    const int ctas = num_sms() * pl.per_sm;
    int S = ctas / d.batch;
    if (S < 1) S = 1;
    const int64_t max_split = (max_seq_len + 4 * pl.TT - 1) / (4 * pl.TT);  // >= 4 tiles per split
    if (S > max_split) S = static_cast<int>(max_split > 0 ? max_split : 1);
    int64_t chunk = (max_seq_len + S - 1) / S;
    chunk = (chunk + pl.TT - 1) / pl.TT * pl.TT;
    pl.chunk = static_cast<int>(chunk);
    pl.S = static_cast<int>((max_seq_len + chunk - 1) / chunk);
    pl.NP = pl.S * P;
    pl.smem = smem_layout(C, d.num_q_heads, pl.TT, pl.chunk, pl.N, 17 * (C / 16), pl.stages).total;
    pl.PP = P;
    const int W = C / 16;
    pl.ok = pl.NT <= max_nt && pl.smem <= 227 * 1024 && (pl.NT % W == 0 || W % pl.NT == 0);
    return pl;
}

cudaError_t launch_decode(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p, cudaStream_t s) {
    if (plan.kind == kDecodeMma) return launch_decode_mma(d, plan, p, s);
    if (plan.kind == kDecodeGeneric) return launch_decode_generic(d, plan, p, s);
    const int B = d.batch;
    switch (plan.N * 16 + plan.REP) {
        case 512 * 16 + 1: return launch_decode_nr<512, 1>(plan, p, B, s);
        case 512 * 16 + 2: return launch_decode_nr<512, 2>(plan, p, B, s);
        case 256 * 16 + 1: return launch_decode_nr<256, 1>(plan, p, B, s);
        case 256 * 16 + 2: return launch_decode_nr<256, 2>(plan, p, B, s);
        case 256 * 16 + 4: return launch_decode_nr<256, 4>(plan, p, B, s);
        case 128 * 16 + 1: return launch_decode_nr<128, 1>(plan, p, B, s);
        case 128 * 16 + 2: return launch_decode_nr<128, 2>(plan, p, B, s);
        case 128 * 16 + 4: return launch_decode_nr<128, 4>(plan, p, B, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_channel_stats(const float* rows_f32, int64_t rows, int64_t C, bool mean_abs, double* stats,
                                 cudaStream_t s) {
    channel_stats_kernel<<<static_cast<unsigned>((C + 127) / 128), 128, 0, s>>>(rows_f32, rows, C, mean_abs ? 1 : 0,
                                                                                stats);
    return cudaGetLastError();
}

cudaError_t launch_rope_table(const rkv_layer_desc& d, float4* table, int64_t max_pos, cudaStream_t s) {
    const int64_t npairs = (max_pos + 1) / 2;
    const int64_t n = npairs * 64;
    rope_table_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(table, npairs, d.rope_base);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t npos = 2 * npairs;
    rope_table2_kernel<<<static_cast<unsigned>((npos * 32 + 255) / 256), 256, 0, s>>>(
        table, npos, d.rope_base, decode_kind(d) == kDecodeMma && mma_layout_n(d) == 512 ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_rotate_keys(const rkv_layer_desc& d, const uint16_t* k, int64_t rows, float* out, cudaStream_t s) {
    const int C = d.num_kv_heads * d.head_dim, N = d.heads_per_group * d.head_dim;
    const float norm = 1.0f / sqrtf(static_cast<float>(N));
    if (rows <= 0) return cudaSuccess;
    if ((N != 128 && N != 256 && N != 512) || C % 512 != 0) return launch_rotate_keys_generic(d, k, rows, out, s);
    const int L = N == 128 ? 8 : 16;
    const int64_t blocks = (rows + kRotRows - 1) / kRotRows;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(C / N));
    const unsigned threads = static_cast<unsigned>(kRotRows * L);
    switch (N) {
        case 128: rotate_keys_kernel<128, 8><<<grid, threads, 0, s>>>(k, rows, C, norm, out); break;
        case 256: rotate_keys_kernel<256, 16><<<grid, threads, 0, s>>>(k, rows, C, norm, out); break;
        case 512: rotate_keys_kernel<512, 16><<<grid, threads, 0, s>>>(k, rows, C, norm, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace rkv
