// decode_mma.cu -- split-K decode attention over the 2-bit rotated cache with
// the inverse FWHT on the tensor cores (mma.sync m16n8k16, fp16 in, fp32 acc).
//
// Same contract as decode_attention.cu (the attention half of decode_step,
// proj/src/pipeline.cpp:133-152,211-261): keys = RoPE_t(H_G . P^-1 . deq(k')),
// logits = q.k/sqrt(d), online softmax, o' = sum p v' (rotated V frame); the
// combine kernel (decode_attention.cu) merges the split partials, adds the
// fp16 sink rows and applies H_128 (V's inverse rotation).
//
// Why tensor cores here.  The CUDA-core kernel spends ~4.5 FADD2 per cached
// K element on the 9-stage FWHT and FADD2/FFMA2 run at half rate on sm_100
// (measured: 60 instr/clk/SM), so the FWHT alone costs more FMA-pipe time
// than streaming the 2-bit cache from HBM.  The Sylvester Hadamard matrix
// factors over index bits: H_512 = H_2(bit 6) (x) H_16(F2 bits) (x)
// H_16(F1 bits).  Per token and FWHT group the two H_16 factors are two
// chained mma.sync: the fp32 accumulator fragment of the first MMA is, element
// for element, the B fragment of the second (D[m][n] -> B[k=n][n'=m]), so the
// rotation never leaves registers.  The remaining H_2 acts on bit 6 -- the
// RoPE partner bit -- and folds into the RoPE coefficients for free:
//   q.(R_t (a'+b', a'-b')) = a'(q_a u + q_b w) + b'(q_a w - q_b u),
//   u = cos - sin, w = cos + sin.
// Precision: the MMA inputs are fp16.  The dequantised K (s*(c-z)) is rounded
// to fp16 once, and the half-way result of the first MMA is split into an
// fp16 hi part and an fp16 residual (two MMAs), so the rotation is accurate to
// ~2^-22 (tools/hmma_precision.py: 2e-5 normalised max error vs 7.6e-4 with a
// single fp16 rounding; the north star allows 2e-3).
//
// G = 1 and 2 (one q head per KV head) run on the same 512-channel tiles: the
// second factor becomes H_4 (x) I_4 / H_8 (x) I_2 over the same bits, leaving
// the head bits to the q.k stage (hadamard_f2_frag, template parameter AG).
//
// Pipeline per CTA (one split of one sequence; one warp per 512-channel tile):
//   * TMA bulk copies stream each 4-token tile (packed K/V words, scale|zero
//     words, the tile's RoPE rows) into a 3-stage ring (mbarrier complete_tx).
//   * scatter (all threads, thread = word position): dequantise the word's 16
//     codes for both tokens of a pair as half2 ops (code -> 2^(10-2e)+c by one
//     LOP3 on the interleaved pair, HSUB2 of the zero point, HMUL2 of the
//     scale) and store them (STS.32) to their natural channel (slot j ->
//     perm[j]) in B-fragment order; a barrier separates scatter and compute,
//     a second one protects the single token-pair buffer and the stage.
//   * compute (warp = tile, per token pair): 4 LDS.128 + PRMT give the B
//     fragments of both tokens, 4 + 8 mma.sync per token, RoPE+q.k on the fp32
//     fragments (FFMA2), a reduce-scatter over shuffles, online softmax, and
//     the V accumulation on CUDA cores: one LOP3 turns two codes into fp16
//     subnormals c*2^(2e-24) and a mixed FHFMA (fp16 x fp16 + fp32) adds p*s*c;
//     the zero point is folded once per token.
// The GQA kernel (G = 2 or 4, 4 q heads per KV head and set; ratios that are
// multiples of 4 run as head sets, two per key tile at 8:1) shares the K side,
// runs P.V on m16n8k8 and parks its accumulators in tensor memory between
// phases.  SP
// instantiations restrict a split to a token range (sequence-parallel
// partials, rkv_decode_attention_partial).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "rkv_common.cuh"
#include "rkv_mma.cuh"
#include "rkv_umma.cuh"
#include "rkv_internal.h"
#include "rkv_layout.h"

namespace rkv {

namespace {

using namespace mma;

constexpr int kMmaMaxThreads = 512;  // one warp per FWHT group: C <= 8192 at G = 4

struct MmaSmem {
    size_t stage_bytes, kc, km, vc, vm, rope;  // offsets inside one stage
    size_t stages, mbar, knat, plan, mask, xch, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline MmaSmem mma_smem(int C, int TT, int chunk, int stages) {
    MmaSmem s{};
    const int W = C / 16, MG = C / 128, PP = TT / 2;
    s.kc = 0;
    s.km = al16(s.kc + size_t(TT) * W * 4);
    s.vc = al16(s.km + size_t(TT) * MG * 4);
    s.vm = al16(s.vc + size_t(TT) * W * 4);
    s.rope = al16(s.vm + size_t(TT) * MG * 4);
    s.stage_bytes = al16(s.rope + size_t(PP) * 64 * 16);
    s.stages = 0;
    s.mbar = s.stages + stages * s.stage_bytes;
    s.knat = al16(s.mbar + stages * 8);
    s.plan = al16(s.knat + size_t(PP) * C * 4);         // token-pair rows of one tile
    s.mask = al16(s.plan + size_t(17) * (C / 16) * 4);  // scatter plan: omega + 16 offsets per word
    s.total = al16(s.mask + size_t(chunk / 32 + 2) * 4);
    return s;
}

// Tile geometry (compile time): TT = 4 tokens = 2 token pairs per tile, one
// warp per FWHT group, 3-deep TMA ring; ~102 KB of shared memory and <= 96
// registers so that two CTAs (20 warps) share an SM and cover each other's
// barrier and MMA-latency stalls.
constexpr int kPP = 2, kTT = 2 * kPP, kNS = 3, kCtasPerSm = 2;

// G = 4 (N = 512), one q head per KV head.  NGC = number of FWHT groups
// (C / 512) when known at compile time (8: LLaMA-2-7B, 10: 13B), so every
// shared-memory offset folds into an immediate; 0 = taken from the launch
// (<= 10 groups: 320 threads, two CTAs per SM); -1 = taken from the launch,
// 11 .. 16 groups (up to 512 threads, one CTA per SM).
// AG = heads per rotation group of the layer (4, 2 or 1): the kernel always
// works on 512-channel (pseudo-)groups; only the second FWHT factor differs
// (hadamard_f2_frag) -- the head bits 7, 8 pass through it when AG < 4.
#ifdef RKV_DEC_TRACE
// per-CTA timeline (tools/decode_trace.py): [start, loop start, end, SM id]
__device__ unsigned long long g_dec_trace[4096][4];
__device__ __forceinline__ unsigned long long dec_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DEC_TRACE(k)                                                                   \
    do {                                                                               \
        const int cid = blockIdx.y * gridDim.x + blockIdx.x;                           \
        if (threadIdx.x == 0 && cid < 4096) {                                          \
            unsigned sm;                                                               \
            asm volatile("mov.u32 %0, %smid;" : "=r"(sm));                            \
            g_dec_trace[cid][k] = dec_gtimer();                                        \
            g_dec_trace[cid][3] = sm;                                                  \
        }                                                                              \
    } while (0)
#else
#define DEC_TRACE(k) \
    do {             \
    } while (0)
#endif
template <int G, int REP, int NGC, int AG, bool SP = false>
__global__ void __launch_bounds__(NGC < 0 ? kMmaMaxThreads : 320, NGC < 0 ? 1 : kCtasPerSm) decode_mma_kernel(DecodeParams p) {
    static_assert(G == 4 && REP == 1 && (AG == 4 || AG == 2 || AG == 1), "decode_mma_kernel: MHA, 512-channel tiles");
    constexpr int N = 128 * G;
    constexpr int NJ = N / 128;  // MMA-1 instances per token (F2 bit 3, outer bit 6)

    extern __shared__ __align__(128) unsigned char smem[];
    const int NG = NGC > 0 ? NGC : p.C / N;
    const int C = NG * N, W = C / 16, MG = C / 128, Hq = NGC > 0 ? NGC * G * REP : p.Hq;
    const MmaSmem lay = mma_smem(C, kTT, p.chunk, kNS);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    uint32_t* mask_s = reinterpret_cast<uint32_t*>(smem + lay.mask);

    const int tid = threadIdx.x, NT = blockDim.x;
    // the layer plan is static: stage it while the previous kernel drains
    {
        const uint4* src = reinterpret_cast<const uint4*>(p.plan + kPlanHeader);
        uint4* dst = reinterpret_cast<uint4*>(smem + lay.plan);
        for (int i = tid; i < 17 * W / 4; i += NT) dst[i] = __ldg(src + i);
    }
    pdl_wait();  // lengths, queries and the cache may come from the previous kernel
    const int warp = tid >> 5, lane = tid & 31;
    const int gam = warp % NG;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    // SP (sequence-parallel partial): only cache tokens [tok_begin, tok_end)
    const int64_t tb = SP ? p.tok_begin[b] : 0, te = SP ? lmin64(p.tok_end[b], T) : T;
    const int64_t t_begin = tb + static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = lmin64(te, t_begin + p.chunk);

    const bool bad_plan = !plan_matches(p.plan, kDecodeMma, N, C);
    if (t_begin >= t_end || bad_plan) {  // empty split: neutral partials (NaN: foreign plan)
        const float fill = bad_plan ? __int_as_float(0x7fc00000) : 0.0f;
        for (int i = tid; i < Hq; i += NT) {
            const int64_t row = (static_cast<int64_t>(b) * p.NP + split) * Hq + i;
            p.ws_ml[row * 2] = bad_plan ? fill : -INFINITY;
            p.ws_ml[row * 2 + 1] = fill;
            float4* o = reinterpret_cast<float4*>(p.ws_o + row * 128);
            for (int k = 0; k < 32; ++k) o[k] = make_float4(fill, fill, fill, fill);
        }
        return;
    }
    DEC_TRACE(0);
    const int ntiles = static_cast<int>((t_end - t_begin + kTT - 1) / kTT);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;

    auto issue_tile = [&](int it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * kTT;
        const uint32_t n = static_cast<uint32_t>(lmin64(kTT, t_end - t0));
        unsigned char* st = smem + lay.stages + (it % kNS) * lay.stage_bytes;
        uint64_t* bar = mbar + (it % kNS);
        const uint32_t bw = n * W * 4, bm = n * MG * 4, npr = (n + 1) >> 1;
        mbar_arrive_expect_tx(bar, 2 * bw + 2 * bm + npr * 1024);
        bulk_g2s(st + lay.kc, p.cache.k_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.km, p.cache.k_meta + (row0 + t0) * MG, bm, bar);
        bulk_g2s(st + lay.vc, p.cache.v_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.vm, p.cache.v_meta + (row0 + t0) * MG, bm, bar);
        for (uint32_t r = 0; r < npr; ++r)  // section 2 (frequency-pair rows) of each position-pair row
            bulk_g2s(st + lay.rope + r * 1024, p.rope + ((t0 >> 1) + r) * 128 + 64, 1024, bar);
    };

    if (tid == 0) {
        for (int s = 0; s < kNS; ++s) mbar_init(mbar + s, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < kNS && it < ntiles; ++it) issue_tile(it);

    const int64_t mw0 = t_begin >> 5;
    {
        const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
        const int nw = static_cast<int>(((t_end - 1) >> 5) - mw0 + 1);
        for (int i = tid; i < nw; i += NT) mask_s[i] = smask[mw0 + i];
    }

    // ---- scatter role: word position wp = tid (NT == W for G = 4); the plan
    // (omega + the 16 store offsets of each word position) lives in shared
    // memory (staged before pdl_wait above)
    const uint32_t* plan_s = reinterpret_cast<const uint32_t*>(smem + lay.plan);
    const uint32_t pair_bytes = static_cast<uint32_t>(C) * 4u;

    // B_e = 2^(10 - 2e') as fp16 exponent bits, e' = 0..4: code e' of a 16-bit lane ORed into the mantissa
    auto bexp = [](int sh) -> uint32_t { const uint32_t be = static_cast<uint32_t>(25 - 2 * sh) << 10; return be | (be << 16); };

    // Branch-free tile bodies: tokens past the end of the split (last tile only)
    // are processed on whatever the stage holds and masked out of the softmax
    // (their probability is 0 and their V weight is exactly 0).
    auto scatter_tile = [&](int slot) {
        const unsigned char* st = smem + lay.stages + slot * lay.stage_bytes;
        const uint32_t* kc = reinterpret_cast<const uint32_t*>(st + lay.kc);
        const uint32_t* km = reinterpret_cast<const uint32_t*>(st + lay.km);
        const uint32_t buf = static_cast<uint32_t>(lay.knat) + smem_u32(smem);
        const int wsrc = static_cast<int>(plan_s[tid]);
        uint32_t ad[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 a4 = reinterpret_cast<const uint4*>(plan_s + W)[q4 * W + tid];
            ad[4 * q4] = a4.x;
            ad[4 * q4 + 1] = a4.y;
            ad[4 * q4 + 2] = a4.z;
            ad[4 * q4 + 3] = a4.w;
        }
#pragma unroll
        for (int pq = 0; pq < kPP; ++pq) {
            const int tt0 = 2 * pq;
            const uint32_t w0 = kc[tt0 * W + wsrc], w1 = kc[(tt0 + 1) * W + wsrc];
            const uint32_t m0 = km[tt0 * MG + (wsrc >> 3)], m1 = km[(tt0 + 1) * MG + (wsrc >> 3)];
            const uint32_t ss = prmt(m0, m1, 0x5410u);  // (s0, s1)
            const uint32_t zz = prmt(m0, m1, 0x7632u);  // (z0, z1)
            uint32_t bz[5];
#pragma unroll
            for (int e = 0; e < 5; ++e) bz[e] = h2add(bexp(e), zz);  // B_e + z, exact
            const uint32_t xl = prmt(w0, w1, 0x5410u), xh = prmt(w0, w1, 0x7632u);  // codes 0-7 | 8-15 of (t0, t1)
            const uint32_t xls = xl >> 10, xhs = xh >> 10;
            const uint32_t dst = buf + static_cast<uint32_t>(pq) * pair_bytes;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int ee = e & 7;
                const uint32_t src = ee < 5 ? (e < 8 ? xl : xh) : (e < 8 ? xls : xhs);
                const int sh = ee < 5 ? ee : ee - 5;
                const uint32_t h = and_or(src, 0x00030003u << (2 * sh), bexp(sh));  // (B + c0, B + c1)
                const uint32_t x = h2mul(h2sub(h, bz[sh]), ss);                      // s * (c - z), fp16
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(dst + ad[e]), "r"(x) : "memory");
            }
        }
    };

    // ---- compute role constants
    const int g = lane >> 2, tl = lane & 3;
    uint32_t AH[4], AF2[4];
    hadamard16_frag(AH, lane, static_cast<uint32_t>(p.max_tokens >> 40));  // max_tokens <= 2^30
    if constexpr (AG != 4) hadamard_f2_frag<AG>(AF2, lane, static_cast<uint32_t>(p.max_tokens >> 40));
    // second FWHT factor: H_16 itself (AH) for AG = 4
    auto mma_f2 = [&](float (&d)[4], uint32_t b0, uint32_t b1, const float (&c)[4]) {
        if constexpr (AG == 4) {
            mma16816(d, AH, b0, b1, c);
        } else {
            mma16816(d, AF2, b0, b1, c);
        }
    };
    // q: RoPE at T-1, x log2(e)/sqrt(d) x 1/sqrt(N).  Frequency pair (f, f+1),
    // f = 2tl + 8 f1 + 16 (g&3); head hq = 4 gam + (g>>2) + 2 rh.
    float2 P2[2][2], Q2[2][2];
    {
        const float4* cs = p.rope + ((T - 1) >> 1) * 128;
        const bool odd = (T - 1) & 1;
        const uint16_t* qb = p.q + static_cast<int64_t>(b) * Hq * 128;
        const float qs = p.qscale * p.k_norm;
#pragma unroll
        for (int f1 = 0; f1 < 2; ++f1) {
#pragma unroll
            for (int rh = 0; rh < 2; ++rh) {
                const int hq = gam * G + (g >> 2) + 2 * rh;
                float pv[2], qv[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int f = 2 * tl + i + 8 * f1 + 16 * (g & 3);
                    const float4 r4 = __ldg(cs + f);
                    const float cT = odd ? r4.y : r4.x, sT = odd ? r4.w : r4.z;
                    const float a = h2f(qb[hq * 128 + f]), bb = h2f(qb[hq * 128 + f + 64]);
                    pv[i] = (a * cT - bb * sT) * qs;
                    qv[i] = (a * sT + bb * cT) * qs;
                }
                P2[f1][rh] = make_float2(pv[0], pv[1]);
                Q2[f1][rh] = make_float2(qv[0], qv[1]);
            }
        }
    }
    const int bit1 = (lane >> 1) & 1, bit2 = (lane >> 2) & 1, bit3 = (lane >> 3) & 1;
    const int hv = (lane >> 4) + 2 * bit3;                 // V head (= head of the reduced logits)
    const int gw = gam * (N / 16) + hv * 8 + (lane & 7);  // V word of the group
    const int gm = gam * G + hv;                           // V meta word (= kv head = q head)
    float m_run = -INFINITY, l_run = 0.f, zc = 0.f;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;

    const uint32_t lane_off = static_cast<uint32_t>(gam * N * 4 + lane * NJ * 16);
    const int swz = (lane >> 1) & 3;
    const int fpi = tl + 4 * (g & 3);  // RoPE slot of frequency pair f / 2, f = 2 tl + 16 (g & 3) (+ 8 f1: slot + 16)

    // K phase of a tile: logits lg[tk] of head hv (log2 domain)
    auto k_tile = [&](int slot, float (&lg)[kTT]) {
        const unsigned char* st = smem + lay.stages + slot * lay.stage_bytes;
        const float4* rope4 = reinterpret_cast<const float4*>(st + lay.rope);  // [token][32] frequency pairs
        const unsigned char* bufp = smem + lay.knat;
        float pv[kTT][2];  // partial logits [token][rh]
#pragma unroll
        for (int pq = 0; pq < kPP; ++pq) {
            uint32_t bf[2][NJ][2];
            const unsigned char* lb = bufp + static_cast<size_t>(pq) * pair_bytes + lane_off;
#pragma unroll
            for (int jc = 0; jc < NJ; ++jc) {
                const uint4 u = lds128(lb + ((jc ^ swz) << 4));
                bf[0][jc][0] = prmt(u.x, u.y, 0x5410u);
                bf[0][jc][1] = prmt(u.z, u.w, 0x5410u);
                bf[1][jc][0] = prmt(u.x, u.y, 0x7632u);
                bf[1][jc][1] = prmt(u.z, u.w, 0x7632u);
            }
#pragma unroll
            for (int tk = 0; tk < 2; ++tk) {
                // Y = H_16(F1) X in fp32; B fragments of the second MMA: hi = fp16(Y)
                // and the residual lo = fp16(Y - hi) (one FHADD per element).
                // (The tensor core can produce the split itself -- fp16
                // accumulator, C = -hi, exact: tools/mb_f16acc.cu -- but the
                // extra MMA per instance and the register-pair MOVs it needs
                // made the kernel slower: 247 vs 242 us at config 2.)
                float yf[NJ][4];
                const float zero[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int jc = 0; jc < NJ; ++jc) mma16816(yf[jc], AH, bf[tk][jc][0], bf[tk][jc][1], zero);
                float2 part[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int f1 = 0; f1 < 2; ++f1) {
                    float z[2][4];  // [outer]: Z = H_16(F2) Y, fragments of channels with bit 6 = outer
#pragma unroll
                    for (int o = 0; o < 2; ++o) {
                        const float* ya = yf[2 * o];      // F2 bit 3 = 0
                        const float* yb = yf[2 * o + 1];  // F2 bit 3 = 1
                        const uint32_t h0 = pack_h2(ya[2 * f1], ya[2 * f1 + 1]);
                        const uint32_t h1 = pack_h2(yb[2 * f1], yb[2 * f1 + 1]);
                        const uint32_t l0 = pack_h2(sub_lo(ya[2 * f1], h0), sub_hi(ya[2 * f1 + 1], h0));
                        const uint32_t l1 = pack_h2(sub_lo(yb[2 * f1], h1), sub_hi(yb[2 * f1 + 1], h1));
                        float t4[4];
                        mma_f2(t4, h0, h1, zero);
                        mma_f2(z[o], l0, l1, t4);
                    }
                    // RoPE (bit-6 butterfly folded into u, w) and q.k over the frequency pair
                    const float4 r4 = rope4[(2 * pq + tk) * 32 + fpi + 16 * f1];  // (u f, u f+1, w f, w f+1)
                    const float2 u = make_float2(r4.x, r4.y), w = make_float2(r4.z, r4.w);
#pragma unroll
                    for (int rh = 0; rh < 2; ++rh) {
                        const float2 al = fma2(Q2[f1][rh], w, mul2(P2[f1][rh], u));   // q_a u + q_b w
                        const float2 be = fma2(make_float2(-Q2[f1][rh].x, -Q2[f1][rh].y), u, mul2(P2[f1][rh], w));  // q_a w - q_b u
                        part[rh] = fma2(make_float2(z[0][2 * rh], z[0][2 * rh + 1]), al, part[rh]);
                        part[rh] = fma2(make_float2(z[1][2 * rh], z[1][2 * rh + 1]), be, part[rh]);
                    }
                }
                pv[2 * pq + tk][0] = part[0].x + part[0].y;
                pv[2 * pq + tk][1] = part[1].x + part[1].y;
            }
        }
        // reduce-scatter the 8 partials over the 16 lanes of the half-warp:
        // lane keeps (rh = bit3, token = 2*bit2 + bit1)
        float r4v[4], r2v[2];
#pragma unroll
        for (int tk = 0; tk < 4; ++tk) {
            const float keep = bit3 ? pv[tk][1] : pv[tk][0], send = bit3 ? pv[tk][0] : pv[tk][1];
            r4v[tk] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {  // token pair bit2
            const float keep = bit2 ? r4v[2 + j] : r4v[j], send = bit2 ? r4v[j] : r4v[2 + j];
            r2v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        float v;
        {
            const float keep = bit1 ? r2v[1] : r2v[0], send = bit1 ? r2v[0] : r2v[1];
            v = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        // the 4 logits of head hv: token tk sits in the lanes with bits (2,1) = tk
#pragma unroll
        for (int tk = 0; tk < kTT; ++tk) lg[tk] = __shfl_sync(0xffffffffu, v, (lane & 0x19) | (tk << 1));
    };

    // online softmax for head hv over a tile's tokens (valid: in range and not a
    // sink); rescales the running state, returns the tile's probabilities
    auto softmax_tile = [&](int it, const float (&lg)[kTT], float (&pr)[kTT]) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * kTT;
        const int nv = static_cast<int>(lmin64(kTT, t_end - t0));
        // valid tokens: in range and not a sink (t0 % 4 == 0: one mask word)
        const uint32_t ok = ~(mask_s[(t0 >> 5) - mw0] >> (t0 & 31)) & ((1u << nv) - 1u);
        float mx = m_run;
#pragma unroll
        for (int tk = 0; tk < kTT; ++tk) mx = fmaxf(mx, ((ok >> tk) & 1u) ? lg[tk] : -INFINITY);
        if (mx > m_run) {  // rescale only when the running max moves (rare after the first tiles)
            const float alpha = ex2(m_run - mx);
            l_run *= alpha;
            zc *= alpha;
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] *= alpha;
            m_run = mx;
        }
#pragma unroll
        for (int tk = 0; tk < kTT; ++tk) {
            pr[tk] = ((ok >> tk) & 1u) ? ex2(lg[tk] - m_run) : 0.0f;
            l_run += pr[tk];
        }
    };

    // V phase of a tile: acc[e] += fp16(p s) * c_e * 2^(2e'-24) (codes as fp16
    // subnormals), the zero point folded into zc with the same rounded weights
    auto v_tile = [&](int slot, const float (&pr)[kTT]) {
        const unsigned char* st = smem + lay.stages + slot * lay.stage_bytes;
        const uint32_t* vc = reinterpret_cast<const uint32_t*>(st + lay.vc);
        const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + lay.vm);
#pragma unroll
        for (int pq = 0; pq < kPP; ++pq) {
            const int tt0 = 2 * pq;
            const uint32_t vw0 = vc[tt0 * W + gw], vw1 = vc[(tt0 + 1) * W + gw];
            // weight-0 tokens may carry garbage metadata (NaN z would poison zc)
            const uint32_t vm0 = pr[tt0] > 0.f ? vm[tt0 * MG + gm] : 0u;
            const uint32_t vm1 = pr[tt0 + 1] > 0.f ? vm[(tt0 + 1) * MG + gm] : 0u;
            const float ps0 = pr[tt0] * h2f(static_cast<uint16_t>(vm0 & 0xffffu));
            const float ps1 = pr[tt0 + 1] * h2f(static_cast<uint16_t>(vm1 & 0xffffu));
            const uint32_t wt = pack_h2(ps0, ps1);
            const uint32_t zz = prmt(vm0, vm1, 0x7632u);  // (z0, z1)
            zc = fhfma<0, 0>(wt, zz, zc);
            zc = fhfma<1, 1>(wt, zz, zc);
            const uint32_t v0s = vw0 >> 10, v1s = vw1 >> 10;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int sh = e < 5 ? e : e - 5;
                const uint32_t m = 0x00030003u << (2 * sh);
                const uint32_t c0 = (e < 5 ? vw0 : v0s) & m, c1 = (e < 5 ? vw1 : v1s) & m;
                acc[e] = fhfma<0, 0>(c0, wt, acc[e]);
                acc[e + 8] = fhfma<1, 0>(c0, wt, acc[e + 8]);
                acc[e] = fhfma<0, 1>(c1, wt, acc[e]);
                acc[e + 8] = fhfma<1, 1>(c1, wt, acc[e + 8]);
            }
        }
    };

    // Per tile: scatter into the (single) token-pair buffer, barrier, logits +
    // softmax + V, barrier, re-arm the stage with tile it + kNS.  The second
    // resident CTA fills the barrier bubbles.
    __syncthreads();  // mask words and plan
    DEC_TRACE(1);
    int slot = 0;
    uint32_t phase = 0;
    for (int it = 0; it < ntiles; ++it) {
        mbar_wait(mbar + slot, phase);
        scatter_tile(slot);
        __syncthreads();
        float lg[kTT], pr[kTT];
        k_tile(slot, lg);
        softmax_tile(it, lg, pr);
        v_tile(slot, pr);
        __syncthreads();
        if (tid == 0 && it + kNS < ntiles) issue_tile(it + kNS);
        if (++slot == kNS) {
            slot = 0;
            phase ^= 1u;
        }
    }

    pdl_trigger();  // the combine may launch while the last CTAs drain
    // ---- this warp's partial (m, l, o') for head gm
    const int64_t row = (static_cast<int64_t>(b) * p.NP + split) * Hq + gm;
    if ((lane & 7) == 0) {
        p.ws_ml[row * 2] = m_run;
        p.ws_ml[row * 2 + 1] = l_run;
    }
    float o[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const int sh = (e & 7) < 5 ? (e & 7) : (e & 7) - 5;
        o[e] = acc[e] * __int_as_float((127 + 24 - 2 * sh) << 23) - zc;
    }
    float4* dst = reinterpret_cast<float4*>(p.ws_o + row * 128 + (lane & 7) * 16);
    dst[0] = make_float4(o[0], o[1], o[2], o[3]);
    dst[1] = make_float4(o[4], o[5], o[6], o[7]);
    dst[2] = make_float4(o[8], o[9], o[10], o[11]);
    dst[3] = make_float4(o[12], o[13], o[14], o[15]);
    DEC_TRACE(2);
}

// ---------------------------------------------------------------------------
// GQA variant: G = 2 (N = 256, two KV heads per FWHT group), REP q heads per
// KV head (BASELINE config 3: LLaMA-3-8B, 32 q / 8 KV heads).  G = 4 (the
// paper's default rotation) runs the same kernel on 256-channel half groups:
// H_512 = H_2(channel bit 8) (x) H_256, so with u, v the H_256 outputs of the
// two halves the keys are u + v (KV heads 0, 1 of the group) and u - v (heads
// 2, 3).  RoPE and q.k are linear, so each warp dots its half's RoPE'd u (or v)
// with the q heads of both KV heads that use it -- its "own" two (whose
// softmax and V it runs, as for G = 2) and the partner half's two -- and the
// two warps of a group swap the partner partial logits through shared memory
// (one 64-thread named barrier per tile); the minus sign of u - v is folded
// into the upper half's own queries.  The K side is
// the same H_16 (x) H_16 chain (no outer bit: channel bit 6, the RoPE
// partner, is F2 bit 3, i.e. the row half of the second MMA's output).  With
// REP = 4 the P.V product is a real matrix product and runs on the tensor
// cores too: per 8 tokens and code position e, one m16n8k8 with A = the
// codes of 16 channels (8 words x {e, e+8}) as fp16 subnormals (one LOP3 per
// register) and B = the 4 heads' weights p*s split into fp16 hi and lo
// columns.  A warp owns one group and 8 consecutive tokens of a tile (PW warps
// per group split the tile), keeps 64 fp32 P.V accumulators and its own
// softmax state, and emits one partial per (warp, head).
constexpr int kGqaNS = 3;

// 64-thread named barrier of warp pair `pair` (ids 1..8 as immediates, so the
// kernel reserves only the barriers it can use)
__device__ __forceinline__ void pair_bar_sync(int pair) {
    switch (pair) {
        case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
        case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
        case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
        case 3: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
        case 4: asm volatile("bar.sync 5, 64;" ::: "memory"); break;
        case 5: asm volatile("bar.sync 6, 64;" ::: "memory"); break;
        case 6: asm volatile("bar.sync 7, 64;" ::: "memory"); break;
        default: asm volatile("bar.sync 8, 64;" ::: "memory"); break;
    }
}

__host__ __device__ inline MmaSmem gqa_smem(int C, int TT, int chunk) {
    MmaSmem s{};
    const int W = C / 16, MG = C / 128, PP = TT / 2;
    s.kc = 0;
    s.km = al16(s.kc + size_t(TT) * W * 4);
    const size_t slack = MG % 4 ? 16 : 0;  // meta rows copied from a 16-byte aligned start (C % 512 != 0)
    s.vc = al16(s.km + size_t(TT) * MG * 4 + slack);
    s.vm = al16(s.vc + size_t(TT) * W * 4);
    s.rope = al16(s.vm + size_t(TT) * MG * 4 + slack);
    s.stage_bytes = al16(s.rope + size_t(PP) * 64 * 16);
    s.stages = 0;
    s.mbar = s.stages + kGqaNS * s.stage_bytes;
    s.knat = al16(s.mbar + kGqaNS * 8);
    s.plan = al16(s.knat + size_t(PP) * C * 4);
    s.mask = al16(s.plan + size_t(17) * W * 4);
    s.xch = al16(s.mask + size_t(chunk / 32 + 2) * 4);  // G = 4: partial-logit exchange, float2 per thread
    s.total = al16(s.xch + size_t(C / 256) * (TT / 8) * 32 * 8);
    return s;
}

// TM: the 64 P.V accumulators and the 32 RoPE'd query registers of every lane
// are parked in tensor memory between the phases that use them (tcgen05.st /
// tcgen05.ld, a few instructions per tile), so the register peak is the larger
// phase instead of their sum and two CTAs fit on an SM.
// NS = 2 (8 or more q heads per KV head, G = 2): two sets of 4 q heads share
// each reconstructed key tile -- logits, softmax state and P.V per set, the
// set's accumulators parked in their own 64 columns.
// WIDE: 5 .. 8 (half-)groups per CTA (over 8 KV heads at G = 2), PW = 1 with
// TM; the launch bounds keep the register budget of the 4-group kernels.
template <int PW, bool TM, int NS, bool WIDE>
constexpr int gqa_max_threads() { return WIDE ? 32 * 8 : 32 * 4 * PW; }
template <int PW, bool TM, int NS, bool WIDE>
constexpr int gqa_min_blocks() { return WIDE ? (NS == 2 ? 1 : 2) : TM ? (NS == 2 ? 2 : PW == 1 ? 4 : 2) : 1; }
// tensor-memory columns a CTA of `warps` warps allocates (a power of two >= 32)
__host__ __device__ constexpr uint32_t gqa_tmem_cols(uint32_t warp_cols, int warps) {
    const uint32_t need = warp_cols * static_cast<uint32_t>((warps + 3) / 4);
    return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
}
template <int REP, int PW, bool TM, bool SP = false, int GR = 2, int NS = 1, bool WIDE = false>
__global__ void __launch_bounds__(gqa_max_threads<PW, TM, NS, WIDE>(), gqa_min_blocks<PW, TM, NS, WIDE>())
    decode_gqa_kernel(DecodeParams p) {
    static_assert(REP == 4, "decode_gqa_kernel: 4 q heads per KV head and set");
    static_assert(GR == 2 || (GR == 4 && PW <= 2 && TM), "decode_gqa_kernel: G = 2, or G = 4 at PW <= 2 with TMEM parking");
    static_assert(NS == 1 || (NS == 2 && GR == 2 && PW == 1 && TM), "decode_gqa_kernel: two head sets at G = 2, PW = 1, TMEM");
    static_assert(!WIDE || (PW == 1 && TM), "decode_gqa_kernel: more than 4 groups at PW = 1 with TMEM");
    constexpr int G = 2, N = 256, NJ = 2, TT = 8 * PW, PPT = TT / 2;  // G, N: KV heads / channels per warp group
    constexpr bool X = GR == 4;  // partner-half exchange
    constexpr bool Y = NS == 2;  // second head set
    constexpr uint32_t kQCols = X || Y ? 64 : 32, kWarpCols = kQCols + 64 * NS;
    extern __shared__ __align__(128) unsigned char smem[];
    const int C = p.C, W = C / 16, MG = C / 128, Hq = p.Hq, NG = C / N;
    const MmaSmem lay = gqa_smem(C, TT, p.chunk);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    uint32_t* mask_s = reinterpret_cast<uint32_t*>(smem + lay.mask);
    {  // the layer plan is static: stage it while the previous kernel drains
        const uint4* src = reinterpret_cast<const uint4*>(p.plan + kPlanHeader);
        uint4* dst = reinterpret_cast<uint4*>(smem + lay.plan);
        for (int i = threadIdx.x; i < 17 * W / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    pdl_wait();  // lengths, queries and the cache may come from the previous kernel

    const int tid = threadIdx.x, NT = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int gam = warp % NG, pw = warp / NG;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    // SP (sequence-parallel partial): only cache tokens [tok_begin, tok_end)
    const int64_t tb = SP ? p.tok_begin[b] : 0, te = SP ? lmin64(p.tok_end[b], T) : T;
    const int64_t t_begin = tb + static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = lmin64(te, t_begin + p.chunk);

    const bool bad_plan = !plan_matches(p.plan, kDecodeMma, N, C);
    if (t_begin >= t_end || bad_plan) {  // empty split: neutral partials (NaN: foreign plan)
        const float fill = bad_plan ? __int_as_float(0x7fc00000) : 0.0f;
        for (int i = tid; i < PW * Hq; i += NT) {
            const int64_t row = (static_cast<int64_t>(b) * p.NP + static_cast<int64_t>(split) * PW + i / Hq) * Hq + i % Hq;
            p.ws_ml[row * 2] = bad_plan ? fill : -INFINITY;
            p.ws_ml[row * 2 + 1] = fill;
            float4* o = reinterpret_cast<float4*>(p.ws_o + row * 128);
            for (int k = 0; k < 32; ++k) o[k] = make_float4(fill, fill, fill, fill);
        }
        return;
    }
    const int ntiles = static_cast<int>((t_end - t_begin + TT - 1) / TT);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;

    // byte offset of token t0's meta row from the 16-byte boundary below it (the
    // cache arrays are 256-byte aligned, so K and V share it)
    auto meta_off = [&](int64_t t0) { return MG % 4 ? static_cast<uint32_t>(((row0 + t0) * MG * 4) & 15) : 0u; };
    auto issue_tile = [&](int it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const uint32_t n = static_cast<uint32_t>(lmin64(TT, t_end - t0));
        unsigned char* st = smem + lay.stages + (it % kGqaNS) * lay.stage_bytes;
        uint64_t* bar = mbar + (it % kGqaNS);
        const uint32_t bw = n * W * 4, bm = n * MG * 4, npr = (n + 1) >> 1;
        // meta rows are C/32 bytes: 16-byte aligned only when C % 512 == 0, so the
        // copy starts at the aligned address below and the readers skip meta_off
        const uint32_t mo = meta_off(t0), bma = (bm + mo + 15u) & ~15u;
        mbar_arrive_expect_tx(bar, 2 * bw + 2 * bma + npr * 1024);
        bulk_g2s(st + lay.kc, p.cache.k_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.km, reinterpret_cast<const unsigned char*>(p.cache.k_meta + (row0 + t0) * MG) - mo, bma, bar);
        bulk_g2s(st + lay.vc, p.cache.v_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.vm, reinterpret_cast<const unsigned char*>(p.cache.v_meta + (row0 + t0) * MG) - mo, bma, bar);
        for (uint32_t r = 0; r < npr; ++r)
            bulk_g2s(st + lay.rope + r * 1024, p.rope + ((t0 >> 1) + r) * 128 + 64, 1024, bar);
    };

    if (tid == 0) {
        for (int s = 0; s < kGqaNS; ++s) mbar_init(mbar + s, 1);
        mbar_fence_init();
    }
    __shared__ uint32_t s_tmem;
    // 4 groups: 128 columns (PW = 1, one set) or 256; WIDE: by the warp count
    const uint32_t tcols = WIDE ? gqa_tmem_cols(kWarpCols, NT / 32) : PW == 1 && !Y ? 128u : 256u;
    if constexpr (TM) {
        if (warp == 0) {
            if (tcols <= 128) umma::alloc<128>(&s_tmem);
            else if (tcols <= 256) umma::alloc<256>(&s_tmem);
            else umma::alloc<512>(&s_tmem);
        }
        umma::fence_before();
    }
    __syncthreads();
    uint32_t tq = 0;  // this warp's columns: q (32) then accumulators (64), lanes of quarter warp & 3
    if constexpr (TM) {
        umma::fence_after();
        tq = s_tmem + ((32u * (warp & 3)) << 16) + kWarpCols * (warp >> 2);
    }
    if (tid == 0)
        for (int it = 0; it < kGqaNS && it < ntiles; ++it) issue_tile(it);

    const int64_t mw0 = t_begin >> 5;
    {
        const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);
        const int nw = static_cast<int>(((t_end - 1) >> 5) - mw0 + 1);
        for (int i = tid; i < nw; i += NT) mask_s[i] = smask[mw0 + i];
    }
    const uint32_t* plan_s = reinterpret_cast<const uint32_t*>(smem + lay.plan);
    const uint32_t pair_bytes = static_cast<uint32_t>(C) * 4u;
    auto bexp = [](int sh) -> uint32_t { const uint32_t be = static_cast<uint32_t>(25 - 2 * sh) << 10; return be | (be << 16); };

    // scatter: thread -> word position wp, token pairs pq0 and pq0 + NT/W (two per thread)
    const int wp = tid % W, pq0 = tid / W, pqs = NT / W;
    auto scatter_tile = [&](int it, int slot) {
        const unsigned char* st = smem + lay.stages + slot * lay.stage_bytes;
        const uint32_t* kc = reinterpret_cast<const uint32_t*>(st + lay.kc);
        const uint32_t* km = reinterpret_cast<const uint32_t*>(st + lay.km + meta_off(t_begin + static_cast<int64_t>(it) * TT));
        const uint32_t buf = static_cast<uint32_t>(lay.knat) + smem_u32(smem);
        const int wsrc = static_cast<int>(plan_s[wp]);
        uint32_t ad[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 a4 = reinterpret_cast<const uint4*>(plan_s + W)[q4 * W + wp];
            ad[4 * q4] = a4.x;
            ad[4 * q4 + 1] = a4.y;
            ad[4 * q4 + 2] = a4.z;
            ad[4 * q4 + 3] = a4.w;
        }
        for (int pq = pq0; pq < PPT; pq += pqs) {
            const int tt0 = 2 * pq;
            const uint32_t w0 = kc[tt0 * W + wsrc], w1 = kc[(tt0 + 1) * W + wsrc];
            const uint32_t m0 = km[tt0 * MG + (wsrc >> 3)], m1 = km[(tt0 + 1) * MG + (wsrc >> 3)];
            const uint32_t ss = prmt(m0, m1, 0x5410u), zz = prmt(m0, m1, 0x7632u);
            uint32_t bz[5];
#pragma unroll
            for (int e = 0; e < 5; ++e) bz[e] = h2add(bexp(e), zz);
            const uint32_t xl = prmt(w0, w1, 0x5410u), xh = prmt(w0, w1, 0x7632u);
            const uint32_t xls = xl >> 10, xhs = xh >> 10;
            const uint32_t dst = buf + static_cast<uint32_t>(pq) * pair_bytes;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int ee = e & 7;
                const uint32_t src = ee < 5 ? (e < 8 ? xl : xh) : (e < 8 ? xls : xhs);
                const int sh = ee < 5 ? ee : ee - 5;
                const uint32_t h = and_or(src, 0x00030003u << (2 * sh), bexp(sh));
                const uint32_t x = h2mul(h2sub(h, bz[sh]), ss);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(dst + ad[e]), "r"(x) : "memory");
            }
        }
    };

    // ---- compute role: lane (g, tl); KV head kvh = lane >> 4 of the group
    const int g = lane >> 2, tl = lane & 3, kvh = lane >> 4;
    const int bit0 = lane & 1, bit1 = (lane >> 1) & 1;
    uint32_t AH[4];
    hadamard16_frag(AH, lane, static_cast<uint32_t>(p.max_tokens >> 40));  // max_tokens <= 2^30
    // second FWHT factor: H_16 (G = 2) or H_8 x I_2 over the head bit (G = 1);
    // the G = 4 half-group pairs use H_16
    uint32_t AF2buf[4];
    if constexpr (!X) hadamard_mask_frag(AF2buf, lane, p.f2_mask, static_cast<uint32_t>(p.max_tokens >> 40));
    uint32_t(&AF2)[4] = *(X ? &AH : &AF2buf);
    // RoPE(T-1) q of the frequency pairs (f, f+1), (f+64, f+65).  Slot sl holds
    // head r = sl ^ (g & 3): the first two reduce-scatter steps then keep / send
    // fixed slots on every lane (no selects) and leave head g & 3 in slot 0.
    // X: QA/QB[.][REP + r] hold the partner half's KV head (same slot kvh), and
    // the upper half's own heads are negated (keys u - v).  Y: QA/QB[.][REP + r]
    // hold the second head set
    constexpr int NQ = X || Y ? 2 * REP : REP;
    float2 QA[2][NQ], QB[2][NQ];
    {
        const float4* cs = p.rope + ((T - 1) >> 1) * 128;
        const bool odd = (T - 1) & 1;
        const uint16_t* qb = p.q + static_cast<int64_t>(b) * Hq * 128;
        const float qs = p.qscale * p.k_norm;
#pragma unroll
        for (int f1 = 0; f1 < 2; ++f1) {
#pragma unroll
            for (int sl = 0; sl < NQ; ++sl) {
                const int r = (sl % REP) ^ (g & 3);
                const bool other = sl >= REP;
                // head hr of its KV head; a set's heads past the ratio (e.g. 5:1 as
                // 4 + 1) get q = 0 and their partials are never written
                const int hr = p.q_rep_off + (!X && other ? REP : 0) + r;
                const bool live = hr < p.q_rep;
                const int hq = ((X && other ? gam ^ 1 : gam) * G + kvh) * p.q_rep + (live ? hr : 0);
                const float sg = !live ? 0.0f : X && !other && (gam & 1) ? -qs : qs;
                float a2[2], b2[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int f = 2 * tl + i + 8 * f1 + 16 * (g & 3);
                    const float4 r4 = __ldg(cs + f);
                    const float cT = odd ? r4.y : r4.x, sT = odd ? r4.w : r4.z;
                    const float a = h2f(qb[hq * 128 + f]), bb = h2f(qb[hq * 128 + f + 64]);
                    a2[i] = (a * cT - bb * sT) * sg;
                    b2[i] = (a * sT + bb * cT) * sg;
                }
                QA[f1][sl] = make_float2(a2[0], a2[1]);
                QB[f1][sl] = make_float2(b2[0], b2[1]);
            }
        }
    }
    const uint32_t lane_off = static_cast<uint32_t>(gam * N * 4 + lane * NJ * 16);
    const int swz = (lane >> 2) & 1;
    const int fpi = tl + 4 * (g & 3);  // rope_pair_slot(tl + 8 (g & 3)); f1 adds 16
    // softmax state of head (kvh, r = g & 3) over this lane's tokens (replicated over tl lanes)
    float m_run[NS], l_part[NS], zc_part[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        m_run[s] = -INFINITY;
        l_part[s] = 0.f;
        zc_part[s] = 0.f;
    }
    float acc[2][8][4];  // P.V accumulators [kvh][code position][fragment]
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 8; ++e)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[h][e][c] = 0.f;
    // tensor-memory parking (TM): q at columns [0, kQCols), then 64 accumulator columns per set
    auto park_q = [&]() {
        if constexpr (TM) {
#pragma unroll
            for (int hs = 0; hs < NQ / REP; ++hs) {
                uint32_t v[2][16];
#pragma unroll
                for (int f1 = 0; f1 < 2; ++f1)
#pragma unroll
                    for (int r = 0; r < REP; ++r) {
                        v[f1][4 * r] = __float_as_uint(QA[f1][hs * REP + r].x);
                        v[f1][4 * r + 1] = __float_as_uint(QA[f1][hs * REP + r].y);
                        v[f1][4 * r + 2] = __float_as_uint(QB[f1][hs * REP + r].x);
                        v[f1][4 * r + 3] = __float_as_uint(QB[f1][hs * REP + r].y);
                    }
                umma::st16(tq + 32 * hs, v[0]);
                umma::st16(tq + 32 * hs + 16, v[1]);
            }
            umma::wait_st();
        }
    };
    auto fetch_q = [&]() {
        if constexpr (TM) {
            uint32_t v[NQ / REP][2][16];
#pragma unroll
            for (int hs = 0; hs < NQ / REP; ++hs) {
                umma::ld16(tq + 32 * hs, v[hs][0]);
                umma::ld16(tq + 32 * hs + 16, v[hs][1]);
            }
#pragma unroll
            for (int hs = 0; hs < NQ / REP; ++hs) {
                umma::wait_ld(v[hs][0]);
                umma::wait_ld(v[hs][1]);
#pragma unroll
                for (int f1 = 0; f1 < 2; ++f1)
#pragma unroll
                    for (int r = 0; r < REP; ++r) {
                        QA[f1][hs * REP + r] =
                            make_float2(__uint_as_float(v[hs][f1][4 * r]), __uint_as_float(v[hs][f1][4 * r + 1]));
                        QB[f1][hs * REP + r] =
                            make_float2(__uint_as_float(v[hs][f1][4 * r + 2]), __uint_as_float(v[hs][f1][4 * r + 3]));
                    }
            }
        }
    };
    auto park_acc = [&](int set) {
        if constexpr (TM) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                uint32_t v[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(acc[q4 >> 1][4 * (q4 & 1) + (i >> 2)][i & 3]);
                umma::st16(tq + kQCols + 64 * set + 16 * q4, v);
            }
            umma::wait_st();
        }
    };
    auto fetch_acc = [&](int set) {
        if constexpr (TM) {
            uint32_t v[4][16];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) umma::ld16(tq + kQCols + 64 * set + 16 * q4, v[q4]);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                umma::wait_ld(v[q4]);
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[q4 >> 1][4 * (q4 & 1) + (i >> 2)][i & 3] = __uint_as_float(v[q4][i]);
            }
        }
    };
    park_q();
#pragma unroll
    for (int s = 0; s < NS; ++s) park_acc(s);

    auto compute_tile = [&](int it, int slot) {
        fetch_q();
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const int nv = static_cast<int>(lmin64(TT, t_end - t0));
        const unsigned char* st = smem + lay.stages + slot * lay.stage_bytes;
        const uint32_t* vc = reinterpret_cast<const uint32_t*>(st + lay.vc);
        const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + lay.vm + meta_off(t0));
        const float4* rope4 = reinterpret_cast<const float4*>(st + lay.rope);
        const unsigned char* bufp = smem + lay.knat;
        float bq[8], bo[8];  // per token: the partial logits (own / X: partner heads) after two reduce-scatter steps
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
            const int tp = 4 * pw + pq;  // token pair in the tile
            uint32_t bf[2][NJ][2];
            const unsigned char* lb = bufp + static_cast<size_t>(tp) * pair_bytes + lane_off;
#pragma unroll
            for (int jc = 0; jc < NJ; ++jc) {
                const uint4 u = lds128(lb + ((jc ^ swz) << 4));
                bf[0][jc][0] = prmt(u.x, u.y, 0x5410u);
                bf[0][jc][1] = prmt(u.z, u.w, 0x5410u);
                bf[1][jc][0] = prmt(u.x, u.y, 0x7632u);
                bf[1][jc][1] = prmt(u.z, u.w, 0x7632u);
            }
#pragma unroll
            for (int tk = 0; tk < 2; ++tk) {
                float yf[NJ][4];
                const float zero[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int jc = 0; jc < NJ; ++jc) mma16816(yf[jc], AH, bf[tk][jc][0], bf[tk][jc][1], zero);
                float2 part[NQ];
#pragma unroll
                for (int r = 0; r < NQ; ++r) part[r] = make_float2(0.f, 0.f);
#pragma unroll
                for (int f1 = 0; f1 < 2; ++f1) {
                    const uint32_t h0 = pack_h2(yf[0][2 * f1], yf[0][2 * f1 + 1]);
                    const uint32_t h1 = pack_h2(yf[1][2 * f1], yf[1][2 * f1 + 1]);
                    const uint32_t l0 = pack_h2(sub_lo(yf[0][2 * f1], h0), sub_hi(yf[0][2 * f1 + 1], h0));
                    const uint32_t l1 = pack_h2(sub_lo(yf[1][2 * f1], h1), sub_hi(yf[1][2 * f1 + 1], h1));
                    float t4[4], z[4];
                    mma16816(t4, AF2, h0, h1, zero);
                    mma16816(z, AF2, l0, l1, t4);
                    // z: (c0, c1) channels f, f+1 (bit 6 = 0), (c2, c3) channels f+64, f+65
                    const float4 r4 = rope4[(2 * tp + tk) * 32 + fpi + 16 * f1];  // (cos f, cos f+1, sin f, sin f+1)
                    const float2 cs2 = make_float2(r4.x, r4.y), sn2 = make_float2(r4.z, r4.w);
                    const float2 a2 = make_float2(z[0], z[1]), b2 = make_float2(z[2], z[3]);
                    const float2 kra = fma2(cs2, a2, mul2(make_float2(-sn2.x, -sn2.y), b2));
                    const float2 krb = fma2(sn2, a2, mul2(cs2, b2));
#pragma unroll
                    for (int r = 0; r < NQ; ++r) {
                        part[r] = fma2(QA[f1][r], kra, part[r]);
                        part[r] = fma2(QB[f1][r], krb, part[r]);
                    }
                }
                // reduce-scatter steps 1-2 over lanes ^8 and ^4 (partners differ in g & 3,
                // so slot s+2 / 1 of one lane is slot s / 0 of the other; see QA)
                float pv[NQ];
#pragma unroll
                for (int r = 0; r < NQ; ++r) pv[r] = part[r].x + part[r].y;
                const float a0 = pv[0] + __shfl_xor_sync(0xffffffffu, pv[2], 8);
                const float a1 = pv[1] + __shfl_xor_sync(0xffffffffu, pv[3], 8);
                bq[2 * pq + tk] = a0 + __shfl_xor_sync(0xffffffffu, a1, 4);
                if constexpr (X || Y) {
                    const float o0 = pv[REP] + __shfl_xor_sync(0xffffffffu, pv[REP + 2], 8);
                    const float o1 = pv[REP + 1] + __shfl_xor_sync(0xffffffffu, pv[REP + 3], 8);
                    bo[2 * pq + tk] = o0 + __shfl_xor_sync(0xffffffffu, o1, 4);
                }
            }
        }
        // reduce-scatter steps 3-4 over the 16 lanes of the KV head: lane keeps tokens
        // (2tl, 2tl+1) of head r = g & 3
        float d[2];
        auto scatter34 = [&](const float (&in)[8], float (&out)[2]) {
            float cq[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float keep = bit1 ? in[j + 4] : in[j], send = bit1 ? in[j] : in[j + 4];
                cq[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float keep = bit0 ? cq[u + 2] : cq[u], send = bit0 ? cq[u] : cq[u + 2];
                out[u] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
        };
        scatter34(bq, d);
        float dx[2];  // X: the partner half's partial logits; Y: the second head set's logits
        if constexpr (X || Y) scatter34(bo, dx);
        if constexpr (X) {  // swap the partner half's partial logits (same lane = same head slot and tokens)
            float2* xch = reinterpret_cast<float2*>(smem + lay.xch);
            xch[warp * 32 + lane] = make_float2(dx[0], dx[1]);
            pair_bar_sync(warp >> 1);  // the group's two warps
            const float2 rx = xch[(warp ^ 1) * 32 + lane];
            d[0] += rx.x;
            d[1] += rx.y;
        }
        // online softmax (log2 domain) for head (kvh, g & 3) over the warp's 8 tokens
        const int64_t tw = t0 + 8 * pw;  // multiple of 8
        const int nvw = nv - 8 * pw;
        const uint32_t okm = ~(mask_s[(tw >> 5) - mw0] >> (tw & 31)) & (nvw >= 8 ? 0xffu : nvw > 0 ? (1u << nvw) - 1u : 0u);
        const bool ok0 = (okm >> (2 * tl)) & 1u, ok1 = (okm >> (2 * tl + 1)) & 1u;
        auto softmax_pv = [&](int set, const float (&dd)[2]) {
            float mx = fmaxf(ok0 ? dd[0] : -INFINITY, ok1 ? dd[1] : -INFINITY);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m_run[set], mx);
            fetch_acc(set);
            if (__any_sync(0xffffffffu, m_new > m_run[set])) {
                const float alpha = m_new > m_run[set] ? ex2(m_run[set] - m_new) : 1.0f;
                l_part[set] *= alpha;
                zc_part[set] *= alpha;
                // accumulator columns 2tl, 2tl+1 = heads ((2tl)&3, (2tl+1)&3) of both KV heads
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int r = (2 * tl + c) & 3;
                        const float al = __shfl_sync(0xffffffffu, alpha, ((h * 4 + r) << 2));
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            acc[h][e][c] *= al;
                            acc[h][e][c + 2] *= al;
                        }
                    }
            }
            m_run[set] = m_new;
            const float p0 = ok0 ? ex2(dd[0] - m_run[set]) : 0.f, p1 = ok1 ? ex2(dd[1] - m_run[set]) : 0.f;
            l_part[set] += p0 + p1;
            // weights p * s (V scale of the KV head), zero point folded into zc
            const int tt = 8 * pw + 2 * tl;  // token of dd[0] within the tile
            const uint32_t vm0 = p0 > 0.f ? vm[tt * MG + gam * G + kvh] : 0u;
            const uint32_t vm1 = p1 > 0.f ? vm[(tt + 1) * MG + gam * G + kvh] : 0u;
            const float ps0 = p0 * h2f(static_cast<uint16_t>(vm0 & 0xffffu)), ps1 = p1 * h2f(static_cast<uint16_t>(vm1 & 0xffffu));
            zc_part[set] += ps0 * h2f(static_cast<uint16_t>(vm0 >> 16)) + ps1 * h2f(static_cast<uint16_t>(vm1 >> 16));
            const uint32_t whi = pack_h2(ps0, ps1);
            const uint32_t wlo = pack_h2(sub_lo(ps0, whi), sub_hi(ps1, whi));
            const uint32_t recv = __shfl_xor_sync(0xffffffffu, kvh ? whi : wlo, 16);
            const uint32_t bv[2] = {kvh ? recv : whi, kvh ? wlo : recv};  // B columns (r = g&3, hi | lo) per KV head
            // P.V: per KV head and code position, m16n8k8 over the warp's 8 tokens
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int word = gam * (N / 16) + h * 8 + g;
                const int ta = 8 * pw + 2 * tl;
                const uint32_t w0 = vc[ta * W + word], w1 = vc[(ta + 1) * W + word];
                const uint32_t xl = prmt(w0, w1, 0x5410u), xh = prmt(w0, w1, 0x7632u);
                const uint32_t xls = xl >> 10, xhs = xh >> 10;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int sh = e < 5 ? e : e - 5;
                    const uint32_t m = 0x00030003u << (2 * sh);
                    mma1688(acc[h][e], (e < 5 ? xl : xls) & m, (e < 5 ? xh : xhs) & m, bv[h]);
                }
            }
            park_acc(set);
        };
        softmax_pv(0, d);
        if constexpr (Y) softmax_pv(1, dx);
    };

    __syncthreads();  // mask words and plan
    int slot = 0;
    uint32_t phase = 0;
    for (int it = 0; it < ntiles; ++it) {
        mbar_wait(mbar + slot, phase);
        scatter_tile(it, slot);
        __syncthreads();
        compute_tile(it, slot);
        __syncthreads();
        if (tid == 0 && it + kGqaNS < ntiles) issue_tile(it + kGqaNS);
        if (++slot == kGqaNS) {
            slot = 0;
            phase ^= 1u;
        }
    }

    pdl_trigger();  // the combine may launch while the last CTAs drain
    // ---- partials: lane (g, tl) holds columns 2tl, 2tl+1 (heads r = (2tl)&3 + c, hi for tl < 2,
    // lo for tl >= 2) of channels g*16 + e and g*16 + e + 8, for both KV heads
    const int64_t rbase = (static_cast<int64_t>(b) * p.NP + static_cast<int64_t>(split) * PW + pw) * Hq;
#pragma unroll
    for (int set = 0; set < NS; ++set) {
        float lsum = l_part[set], zsum = zc_part[set];
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
        zsum += __shfl_xor_sync(0xffffffffu, zsum, 1);
        zsum += __shfl_xor_sync(0xffffffffu, zsum, 2);
        fetch_acc(set);
        if (tl == 0 && p.q_rep_off + REP * set + (g & 3) < p.q_rep) {
            const int hq = (gam * G + kvh) * p.q_rep + p.q_rep_off + REP * set + (g & 3);
            p.ws_ml[(rbase + hq) * 2] = m_run[set];
            p.ws_ml[(rbase + hq) * 2 + 1] = lsum;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int r = (2 * tl + c) & 3;
                const float z = __shfl_sync(0xffffffffu, zsum, ((h * 4 + r) << 2));
                const int hr = p.q_rep_off + REP * set + r;
                const int hq = (gam * G + h) * p.q_rep + hr;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int sh = e < 5 ? e : e - 5;
                    const float sc = __int_as_float((127 + 24 - 2 * sh) << 23);
                    const float o0 = acc[h][e][c] + __shfl_xor_sync(0xffffffffu, acc[h][e][c], 2);          // hi + lo
                    const float o1 = acc[h][e][c + 2] + __shfl_xor_sync(0xffffffffu, acc[h][e][c + 2], 2);
                    if (tl < 2 && hr < p.q_rep) {
                        float* orow = p.ws_o + (rbase + hq) * 128 + g * 16;
                        orow[e] = o0 * sc - z;
                        orow[e + 8] = o1 * sc - z;
                    }
                }
            }
    }
    if constexpr (TM) {
        umma::fence_before();
        __syncthreads();
        if (warp == 0) {
            umma::fence_after();
            if (tcols <= 128) umma::dealloc<128>(s_tmem);
            else if (tcols <= 256) umma::dealloc<256>(s_tmem);
            else umma::dealloc<512>(s_tmem);
        }
    }
}

}  // namespace

// MHA (one q head per KV head) with G = 4, 2 or 1 heads per rotation group
// runs on 512-channel tiles (C a multiple of 512); GQA with G = 2 or 4 and 4 q
// heads per KV head has its own kernel (256-channel (half) groups, at most 4
// per CTA).
bool decode_mma_supported(int G, int REP, int C) {
    if (REP == 1 && (G == 4 || G == 2 || G == 1)) return C % 512 == 0 && C / 512 * 32 <= kMmaMaxThreads;
    if (REP >= 2 && REP <= 64 && (G == 1 || G == 2 || G == 4)) return C % (128 * std::max(G, 2)) == 0 && C / 256 <= 8;
    return false;
}

int mma_layout_n(const rkv_layer_desc& d) {
    const int rep = d.num_q_heads / d.num_kv_heads;
    return (d.heads_per_group == 1 || d.heads_per_group == 2 || d.heads_per_group == 4) && rep > 1 ? 256 : 512;
}

namespace {
using MhaKernel = void (*)(DecodeParams);
// compile-time tile counts for the LLaMA-2-7B / 13B widths (8 and 10 tiles of 512 channels)
template <int AG>
MhaKernel mha_kernel_g(int NG, bool sp) {
    if (NG > 10) return sp ? decode_mma_kernel<4, 1, -1, AG, true> : decode_mma_kernel<4, 1, -1, AG>;
    if (sp) return decode_mma_kernel<4, 1, 0, AG, true>;  // partials: generic tile count
    return NG == 10 ? decode_mma_kernel<4, 1, 10, AG> : NG == 8 ? decode_mma_kernel<4, 1, 8, AG> : decode_mma_kernel<4, 1, 0, AG>;
}
MhaKernel mha_kernel(int NG, int G, bool sp = false) {
    return G == 1 ? mha_kernel_g<1>(NG, sp) : G == 2 ? mha_kernel_g<2>(NG, sp) : mha_kernel_g<4>(NG, sp);
}
int gqa_pw() { return std::max(1, std::min(4, options().gqa_pw.load())); }
bool gqa_tmem() { return options().gqa_tmem.load() != 0; }
template <int PW>
void* gqa_kernel_ptr() {
    return gqa_tmem() ? reinterpret_cast<void*>(decode_gqa_kernel<4, PW, true>)
                      : reinterpret_cast<void*>(decode_gqa_kernel<4, PW, false>);
}
// 4-head sets per launch: two (one key tile, up to 8 q heads) when the ratio
// exceeds 4 at G = 2 and PW = 1 with tensor-memory parking
int gqa_sets(const rkv_layer_desc& d, int pw) {
    const int rep = d.num_q_heads / d.num_kv_heads;
    return d.heads_per_group <= 2 && rep > 4 && pw == 1 && gqa_tmem() && options().gqa_sets.load() != 1 ? 2 : 1;
}
void* gqa_kernel(int pw, bool sp = false, bool g4 = false, int sets = 1, bool wide = false) {
    if (wide) {  // 5 .. 8 (half-)groups: PW = 1 with tensor-memory parking
        if (sets == 2)
            return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true, 2, 2, true>)
                      : reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, false, 2, 2, true>);
        if (g4)
            return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true, 4, 1, true>)
                      : reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, false, 4, 1, true>);
        return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true, 2, 1, true>)
                  : reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, false, 2, 1, true>);
    }
    if (sets == 2)
        return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true, 2, 2>)
                  : reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, false, 2, 2>);
    if (g4) {  // G = 4: half-group pairs, PW 1 or 2, accumulators and queries parked in tensor memory
        if (pw == 1)
            return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true, 4>)
                      : reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, false, 4>);
        return sp ? reinterpret_cast<void*>(decode_gqa_kernel<4, 2, true, true, 4>)
                  : reinterpret_cast<void*>(decode_gqa_kernel<4, 2, true, false, 4>);
    }
    if (sp)  // partials: PW 1 or 2 with tensor-memory parking
        return pw == 1 ? reinterpret_cast<void*>(decode_gqa_kernel<4, 1, true, true>)
                       : reinterpret_cast<void*>(decode_gqa_kernel<4, 2, true, true>);
    switch (pw) {
        case 4: return gqa_kernel_ptr<4>();
        case 3: return gqa_kernel_ptr<3>();
        case 1: return gqa_kernel_ptr<1>();
        default: return gqa_kernel_ptr<2>();
    }
}
}  // namespace

// Kernel family for a layer shape (host only, no CUDA calls): the tensor-core
// kernels where they tile, else the CUDA-core split kernel, else the generic
// kernel (any rotation size / head ratio, generic.cu).
int decode_kind(const rkv_layer_desc& d) {
    const int REP = d.num_q_heads / d.num_kv_heads;
    if (d.head_dim == 128 && d.num_q_heads % d.num_kv_heads == 0 && !options().force_simt.load() &&
        decode_mma_supported(d.heads_per_group, REP, d.num_kv_heads * d.head_dim))
        return kDecodeMma;
    return simt_shape_ok(d) ? kDecodeSimt : kDecodeGeneric;
}

DecodePlan plan_decode_mma(const rkv_layer_desc& d, int64_t max_seq_len) {
    DecodePlan pl{};
    const int C = d.num_kv_heads * d.head_dim;
    pl.kind = kDecodeMma;
    pl.N = mma_layout_n(d);
    pl.REP = d.num_q_heads / d.num_kv_heads;
    const int NG = C / pl.N;
    const bool gqa = pl.N == 256, g4 = gqa && d.heads_per_group == 4;
    // more than 4 (half-)groups (over 8 KV heads): one warp per group with tensor-memory parking
    const bool wide = gqa && NG > 4;
    const int PW = wide ? 1 : g4 ? std::min(2, gqa_pw()) : gqa ? gqa_pw() : 1, PP = gqa ? 4 * PW : kPP;
    pl.stages = gqa ? kGqaNS : kNS;
    pl.P = PW;
    pl.PP = PP;
    pl.TT = 2 * PP;
    pl.NT = NG * 32 * PW;
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    auto smem_of = [&](int chunk) {
        return gqa ? gqa_smem(C, pl.TT, chunk).total : mma_smem(C, pl.TT, chunk, pl.stages).total;
    };
    pl.smem = smem_of(static_cast<int>(max_seq_len) + pl.TT);
    pl.per_sm = std::max(1, std::min(kCtasPerSm, static_cast<int>((227u * 1024u) / (pl.smem + 1024))));
    {
        int n = 0;
        const int sets = gqa ? gqa_sets(d, PW) : 1;
        const void* kern = gqa ? gqa_kernel(PW, false, g4, sets, wide) : reinterpret_cast<const void*>(mha_kernel(NG, d.heads_per_group));
        if (ensure_smem(kern, pl.smem) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, pl.NT, pl.smem) == cudaSuccess && n > 0)
            pl.per_sm = n;
        else
            cudaGetLastError();
        // the occupancy query reports one CTA per SM for the tensor-memory GQA
        // kernels (it does not see their real limits): plan with tensor memory,
        // registers (128, or 192 with two head sets) and shared memory
        if (gqa && (gqa_tmem() || wide)) {
            const uint32_t wcols = (g4 || sets == 2 ? 64u : 32u) + 64u * static_cast<uint32_t>(sets);
            const int tm = static_cast<int>(512u / gqa_tmem_cols(wcols, pl.NT / 32));
            const int rg = 65536 / (pl.NT * (sets == 2 ? 192 : 128));
            const int sm = static_cast<int>((227u * 1024u) / (pl.smem + 1024));
            pl.per_sm = std::max(1, std::min(tm, std::min(rg, sm)));
        }
    }
    // splits per sequence: fill every resident CTA slot, and prefer a split count
    // whose CTA total is close to a whole number of waves (within 4x the minimum)
    const int slots = num_sms() * pl.per_sm;
    const int64_t max_split = std::max<int64_t>(1, (max_seq_len + 4 * pl.TT - 1) / (4 * pl.TT));
    int S = choose_splits(slots, d.batch, max_split);
    if (const int o = options().dec_splits.load())  // experiment switch: splits per sequence
        if (o > 0) S = static_cast<int>(std::min<int64_t>(max_split, o));
    int64_t chunk = (max_seq_len + S - 1) / S;
    chunk = (chunk + pl.TT - 1) / pl.TT * pl.TT;
    pl.chunk = static_cast<int>(chunk);
    pl.S = static_cast<int>((max_seq_len + chunk - 1) / chunk);
    pl.NP = pl.S * PW;
    pl.smem = smem_of(pl.chunk);
    pl.ok = pl.smem <= 227 * 1024 && (gqa ? pl.NT <= 512 : pl.NT <= kMmaMaxThreads && pl.NT % (C / 16) == 0);
    return pl;
}

cudaError_t launch_decode_mma(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p, cudaStream_t s) {
    const bool sp = p.tok_begin != nullptr;
    if (plan.N == 256) {
        if (sp && plan.P > 2) return cudaErrorNotSupported;  // partials are instantiated for PW = 1, 2
        const int sets = gqa_sets(d, plan.P);
        const bool wide = d.num_kv_heads * d.head_dim / 256 > 4;
        const void* kern = gqa_kernel(plan.P, sp, d.heads_per_group == 4, sets, wide);
        cudaError_t e = ensure_smem(kern, plan.smem);
        if (e != cudaSuccess) return e;
        DecodeParams pp = p;
        void* args[] = {&pp};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(plan.S, d.batch);
        cfg.blockDim = dim3(plan.NT);
        cfg.dynamicSmemBytes = plan.smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        pp.f2_mask = d.heads_per_group == 1 ? 11 : 15;
        // 4 (sets = 2: 8) q heads per KV head per launch: larger ratios run as
        // passes over disjoint head sets (each pass re-reads the cache), one combine
        const int rep = d.num_q_heads / d.num_kv_heads;
        for (int off = 0; off < rep; off += 4 * sets) {
            pp.q_rep = rep;
            pp.q_rep_off = off;
            if ((e = cudaLaunchKernelExC(&cfg, kern, args)) != cudaSuccess) return e;
        }
        return launch_decode_combine(p, d.batch, s);
    }
    auto kern = mha_kernel(p.C / 512, d.heads_per_group, sp);
    cudaError_t e = ensure_smem_k(kern, plan.smem);
    if (e != cudaSuccess) return e;
    if (options().decode_pdl.load()) {
        if ((e = launch_pdl(kern, dim3(plan.S, d.batch), dim3(plan.NT), plan.smem, s, p)) != cudaSuccess) return e;
    } else {
        kern<<<dim3(plan.S, d.batch), plan.NT, plan.smem, s>>>(p);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return launch_decode_combine(p, d.batch, s);
}

}  // namespace rkv

#ifdef RKV_DEC_TRACE
extern "C" int rkv_debug_decode_trace(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, rkv::g_dec_trace, sizeof(rkv::g_dec_trace)) == cudaSuccess ? 0 : 1;
}
#endif
