// decode_attention.cu -- split-K decode attention over the 2-bit rotated cache.
//
// Restates the attention half of decode_step (proj/src/pipeline.cpp:133-152,
// 211-261) for B sequences at once:
//   keys   = RoPE_t( H_G^-1 . P^-1 . dequant(k') )    (reconstruct_cache)
//   query  = RoPE_{T-1}(q)                             (prepare_queries)
//   logits = q.k / sqrt(d), softmax, o' = sum p v'     (v' in the rotated frame)
//   out    = H_128 o'                                  (V's inverse rotation, W_o_f)
// B200 mapping (one CTA per (split, sequence), grid = splits x B sized to the
// 148 SMs):
//   * TMA bulk copies (cp.async.bulk, UBLKCP) stream each tile of TT tokens --
//     packed K/V words, K/V scale|zero words and the tile's RoPE rows -- into
//     an NS-stage shared-memory ring guarded by mbarriers;
//   * K1: every thread dequantizes whole packed words (one quant group per
//     word, so one scale) and scatters the 16 values to their natural channel
//     (slot j -> channel perm[j]) in a swizzled fp32 tile;
//   * K2: a 16-lane group owns one FWHT group (G KV heads) of a token PAIR:
//     float2 registers hold the same channel of both tokens, so the inverse
//     FWHT (== the forward one, proj/src/hadamard.cpp:75), RoPE and the q.k
//     dot are FADD2/FFMA2; lane partials reduce by shuffles;
//   * online softmax in exp2 domain per head;
//   * V: each thread owns one packed V word x one q head and accumulates
//     sum p*s*code (zero point folded once per token), never materialising
//     dequantized V;
//   * sinks (raw fp16 sidecar rows) are one extra partial (decode_sinks_kernel)
//     and a combine kernel merges the partials in a fixed order and applies
//     H_128 to the rotated-frame accumulator.  Deterministic.
#include <cfloat>
#include <cmath>

#include "rkv_common.cuh"
#include "rkv_internal.h"

namespace rkv {

namespace {

constexpr int kStages = 3;

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
constexpr int kMaxThreads = 320;  // plan_decode keeps NT <= 320 (204 registers per thread)

// knat swizzle (same construction as quantize_kv.cu): float4 chunks of a
// lane's layout-A row XOR the lane, unit parity moves a lane group's scalar
// layout-B traffic to the other 16 banks.
template <int N, int L>
__device__ __forceinline__ int kswz(int c) {
    constexpr int R = N / L;
    constexpr int LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    return c ^ (((c >> LR) & (R / 4 - 1)) << 2) ^ (((c >> LN) & (32 / L - 1)) << LL);
}

struct SmemLayout {
    size_t stage_bytes, kc, km, vc, vm, rope;  // offsets inside a stage
    size_t stages, mbar, knat, q, addr, logit, prob, alpha, mask, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout smem_layout(int C, int Hq, int TT) {
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
    s.q = align16(s.knat + size_t(TT) * C * 4);
    s.addr = align16(s.q + size_t(Hq) * 128 * 4);
    s.logit = align16(s.addr + size_t(C) * 2);
    s.prob = align16(s.logit + size_t(TT) * Hq * 4);
    s.alpha = align16(s.prob + size_t(TT) * Hq * 4);
    s.mask = align16(s.alpha + size_t(Hq) * 4);
    s.total = align16(s.mask + 16);
    return s;
}

template <int N, int REP>
__global__ void __launch_bounds__(kMaxThreads, 1) decode_split_kernel(DecodeParams p) {
    constexpr int L = N >= 256 ? 16 : 8;  // lanes per FWHT group
    constexpr int R = N / L;              // float2 registers per lane
    constexpr int LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    constexpr int GH = N / 128;           // KV heads per FWHT group
    constexpr int JJ = 128 / L;           // registers per head in layout B
    constexpr int HALF = JJ / 2;          // RoPE partner distance (bit 6 of d)
    constexpr int NV = GH * REP;          // q heads served by one group
    static_assert(R >= L, "layout A/B must cover all index bits");

    extern __shared__ __align__(128) unsigned char smem[];
    const int C = p.C, W = C / 16, MG = C / 128, Hq = p.Hq;
    const int NG = C / N, P = p.P, TT = 2 * P;
    const SmemLayout lay = smem_layout(C, Hq, TT);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    float* knat = reinterpret_cast<float*>(smem + lay.knat);
    uint16_t* saddr = reinterpret_cast<uint16_t*>(smem + lay.addr);
    float* logit_s = reinterpret_cast<float*>(smem + lay.logit);
    float* prob_s = reinterpret_cast<float*>(smem + lay.prob);
    float* alpha_s = reinterpret_cast<float*>(smem + lay.alpha);
    uint32_t* mask_s = reinterpret_cast<uint32_t*>(smem + lay.mask);

    const int tid = threadIdx.x, lane = tid & 31, NT = blockDim.x;
    const int b = blockIdx.y, split = blockIdx.x;
    const int64_t T = p.seq_len[b];
    const int64_t t_begin = static_cast<int64_t>(split) * p.chunk;
    const int64_t t_end = min(T, t_begin + p.chunk);
    const int64_t ws_row = (static_cast<int64_t>(b) * (p.S + 1) + split) * Hq;

    if (t_begin >= t_end) {  // empty split: neutral partial
        for (int h = tid; h < Hq; h += NT) {
            p.ws_ml[(ws_row + h) * 2] = -INFINITY;
            p.ws_ml[(ws_row + h) * 2 + 1] = 0.0f;
        }
        for (int i = tid; i < Hq * 128; i += NT) p.ws_o[ws_row * 128 + i] = 0.0f;
        return;
    }
    const int ntiles = static_cast<int>((t_end - t_begin + TT - 1) / TT);
    const int64_t row0 = static_cast<int64_t>(b) * p.max_tokens;

    auto issue_tile = [&](int it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const uint32_t n = static_cast<uint32_t>(lmin(TT, t_end - t0));
        unsigned char* st = smem + lay.stages + (it % kStages) * lay.stage_bytes;
        uint64_t* bar = mbar + (it % kStages);
        const uint32_t bw = n * W * 4, bm = n * MG * 4, br = n * 64 * 8;
        mbar_arrive_expect_tx(bar, 2 * bw + 2 * bm + br);
        bulk_g2s(st + lay.kc, p.cache.k_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.km, p.cache.k_meta + (row0 + t0) * MG, bm, bar);
        bulk_g2s(st + lay.vc, p.cache.v_codes + (row0 + t0) * W, bw, bar);
        bulk_g2s(st + lay.vm, p.cache.v_meta + (row0 + t0) * MG, bm, bar);
        bulk_g2s(st + lay.rope, p.rope + t0 * 64, br, bar);
    };

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(mbar + s, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < kStages - 1 && it < ntiles; ++it) issue_tile(it);

    // slot -> swizzled natural channel address inside a knat row
    for (int j = tid; j < C; j += NT) saddr[j] = static_cast<uint16_t>(kswz<N, L>(__ldg(p.perm + j)));

    // q: RoPE at position T-1 (prepare_queries), pre-scaled by log2(e)/sqrt(d),
    // stored lane-major: q_l[(h*L + lam)*JJ + jj] = q[h][lam + L*jj]
    float* q_l = reinterpret_cast<float*>(smem + lay.q);
    {
        const float2* cs = p.rope + (T - 1) * 64;
        const uint16_t* qb = p.q + static_cast<int64_t>(b) * Hq * 128;
        auto qaddr = [&](int h, int d) { return (h * L + (d % L)) * JJ + d / L; };
        for (int i = tid; i < Hq * 64; i += NT) {
            const int h = i >> 6, f = i & 63;
            const float a = h2f(qb[h * 128 + f]), bb = h2f(qb[h * 128 + f + 64]);
            const float2 r = __ldg(cs + f);
            q_l[qaddr(h, f)] = (a * r.x - bb * r.y) * p.qscale;
            q_l[qaddr(h, f + 64)] = (a * r.y + bb * r.x) * p.qscale;
        }
    }

    // lane group = (FWHT group g, token pair pp)
    const int lg = tid / L, lam = tid % L;
    const int g = lg % NG, pp = lg / NG;

    // V ownership: one packed word x one q head of its KV head
    const int vw = tid % W, vr = tid / W;
    const bool v_owner = tid < W * REP;
    const int vh = (vw / 8) * REP + vr;
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.f, 0.f);
    float zsum = 0.f;
    float m_run = -INFINITY, l_run = 0.f;  // head tid (tid < Hq)
    __syncthreads();  // q_l and saddr complete

    const uint32_t* smask = p.cache.sink_mask + static_cast<int64_t>(b) * ((p.max_tokens + 31) / 32);

    for (int it = 0; it < ntiles; ++it) {
        const int64_t t0 = t_begin + static_cast<int64_t>(it) * TT;
        const int nv = static_cast<int>(lmin(TT, t_end - t0));
        const unsigned char* st = smem + lay.stages + (it % kStages) * lay.stage_bytes;
        const uint32_t* kc = reinterpret_cast<const uint32_t*>(st + lay.kc);
        const uint32_t* km = reinterpret_cast<const uint32_t*>(st + lay.km);
        const uint32_t* vc = reinterpret_cast<const uint32_t*>(st + lay.vc);
        const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + lay.vm);
        const float2* rope = reinterpret_cast<const float2*>(st + lay.rope);
        mbar_wait(mbar + (it % kStages), (it / kStages) & 1);

        // ---- K1: dequantize + un-reorder scatter
        if (tid == 0) {
            uint32_t m = 0;
            for (int tt = 0; tt < nv; ++tt) {
                const int64_t t = t0 + tt;
                if (!((smask[t >> 5] >> (t & 31)) & 1u)) m |= 1u << tt;
            }
            *mask_s = m;
        }
        for (int item = tid; item < nv * W; item += NT) {
            const int tt = item / W, w = item % W;
            const uint32_t wd = kc[tt * W + w];
            const uint32_t mt = km[tt * MG + (w >> 3)];
            const float s = h2f(static_cast<uint16_t>(mt & 0xffffu));
            const float zb = 8388608.0f + h2f(static_cast<uint16_t>(mt >> 16));
            const uint4 a0 = lds128(saddr + 16 * w), a1 = lds128(saddr + 16 * w + 8);
            const uint16_t* ad0 = reinterpret_cast<const uint16_t*>(&a0);
            const uint16_t* ad1 = reinterpret_cast<const uint16_t*>(&a1);
            float* dst = knat + tt * C;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                // (2^23 + c) - (2^23 + z) = c - z exactly, times s exactly (proj/src/quant.cpp:99-107)
                const float cz = __uint_as_float(0x4B000000u | ((wd >> (2 * e)) & 3u)) - zb;
                dst[e < 8 ? ad0[e] : ad1[e - 8]] = s * cz;
            }
        }
        __syncthreads();
        if (tid == 0 && it + kStages - 1 < ntiles) issue_tile(it + kStages - 1);

        // ---- K2: inverse grouped FWHT + RoPE + q.k for a token pair
        for (int pq = pp; pq < P; pq += NT / (NG * L)) {
            const int tt0 = 2 * pq;
            float* r0 = knat + tt0 * C;
            float* r1 = r0 + C;
            float2 x[R];
#pragma unroll
            for (int q4 = 0; q4 < R / 4; ++q4) {
                const int a = kswz<N, L>(g * N + lam * R + 4 * q4);
                const float4 u = *reinterpret_cast<const float4*>(r0 + a);
                const float4 v = *reinterpret_cast<const float4*>(r1 + a);
                x[4 * q4] = make_float2(u.x, v.x);
                x[4 * q4 + 1] = make_float2(u.y, v.y);
                x[4 * q4 + 2] = make_float2(u.z, v.z);
                x[4 * q4 + 3] = make_float2(u.w, v.w);
            }
            bfly_range<R, 0, LR>(x);
#pragma unroll
            for (int q4 = 0; q4 < R / 4; ++q4) {
                const int a = kswz<N, L>(g * N + lam * R + 4 * q4);
                *reinterpret_cast<float4*>(r0 + a) = make_float4(x[4 * q4].x, x[4 * q4 + 1].x, x[4 * q4 + 2].x, x[4 * q4 + 3].x);
                *reinterpret_cast<float4*>(r1 + a) = make_float4(x[4 * q4].y, x[4 * q4 + 1].y, x[4 * q4 + 2].y, x[4 * q4 + 3].y);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int a = kswz<N, L>(g * N + lam + L * j);
                x[j] = make_float2(r0[a], r1[a]);
            }
            bfly_range<R, LR - LL, LN - LL>(x);
            // RoPE at each token's position, then the dot with every q head of the group
            float2 part[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) part[v] = make_float2(0.f, 0.f);
            const float2 nn = make_float2(p.k_norm, p.k_norm);
#pragma unroll
            for (int jj = 0; jj < HALF; ++jj) {
                const int f = lam + L * jj;  // frequency index of (d, d+64)
                const float2 c0 = rope[tt0 * 64 + f], c1 = rope[(tt0 + 1) * 64 + f];
                const float2 cs = make_float2(c0.x, c1.x), sn = make_float2(c0.y, c1.y);
#pragma unroll
                for (int hh = 0; hh < GH; ++hh) {
                    const float2 a = mul2(x[hh * JJ + jj], nn);
                    const float2 bb = mul2(x[hh * JJ + jj + HALF], nn);
                    const float2 ar = fma2(a, cs, mul2(make_float2(-bb.x, -bb.y), sn));  // a c - b s
                    const float2 br = fma2(a, sn, mul2(bb, cs));                         // a s + b c
#pragma unroll
                    for (int r = 0; r < REP; ++r) {
                        const float* qh = q_l + (((g * GH + hh) * REP + r) * L + lam) * JJ;
                        const float qa = qh[jj], qb = qh[jj + HALF];
                        part[hh * REP + r] = fma2(make_float2(qa, qa), ar, part[hh * REP + r]);
                        part[hh * REP + r] = fma2(make_float2(qb, qb), br, part[hh * REP + r]);
                    }
                }
            }
            // reduce the NV x 2 partials over the L lanes of the group
            float val[2 * NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                val[2 * v] = part[v].x;
                val[2 * v + 1] = part[v].y;
            }
            constexpr int V0 = 2 * NV;
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
            // after the halvings lane lam holds value index lam >> (LL - log2(V0)) (V0 <= L)
            // or values lam*(V0/L) + k (V0 > L)
            if constexpr (V0 <= L) {
                constexpr int sh = LL - ilog2(V0);
                if ((lam & ((1 << sh) - 1)) == 0) {
                    const int vidx = lam >> sh;
                    const int v = vidx >> 1, tok = vidx & 1;
                    const int h = (g * GH + v / REP) * REP + (v % REP);
                    logit_s[(tt0 + tok) * Hq + h] = val[0];
                }
            } else {
#pragma unroll
                for (int k = 0; k < V0 / L; ++k) {
                    const int vidx = lam * (V0 / L) + k;
                    const int v = vidx >> 1, tok = vidx & 1;
                    const int h = (g * GH + v / REP) * REP + (v % REP);
                    logit_s[(tt0 + tok) * Hq + h] = val[k];
                }
            }
            __syncwarp();
        }
        __syncthreads();

        // ---- online softmax (exp2 domain), one thread per q head
        const uint32_t tmask = *mask_s;
        for (int h = tid; h < Hq; h += NT) {
            float mx = -INFINITY;
            for (int tt = 0; tt < TT; ++tt)
                if ((tmask >> tt) & 1u) mx = fmaxf(mx, logit_s[tt * Hq + h]);
            const float m_new = fmaxf(m_run, mx);
            const float alpha = (m_new == -INFINITY) ? 1.0f : exp2f(m_run - m_new);
            float lsum = 0.f;
            for (int tt = 0; tt < TT; ++tt) {
                const float pr = ((tmask >> tt) & 1u) ? exp2f(logit_s[tt * Hq + h] - m_new) : 0.0f;
                prob_s[tt * Hq + h] = pr;
                lsum += pr;
            }
            l_run = l_run * alpha + lsum;
            m_run = m_new;
            alpha_s[h] = alpha;
        }
        __syncthreads();

        // ---- V: acc += p * s * code, zero folded per token; rotated frame kept
        if (v_owner) {
            const float al = alpha_s[vh];
            const float2 a2 = make_float2(al, al);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = mul2(acc[i], a2);
            zsum *= al;
            for (int tt = 0; tt < nv; tt += 2) {
                const float p0 = prob_s[tt * Hq + vh];
                const float p1 = (tt + 1 < nv) ? prob_s[(tt + 1) * Hq + vh] : 0.0f;
                if (p0 == 0.0f && p1 == 0.0f) continue;
                const uint32_t w0 = vc[tt * W + vw];
                const uint32_t w1 = (tt + 1 < nv) ? vc[(tt + 1) * W + vw] : 0u;
                const uint32_t m0 = vm[tt * MG + (vw >> 3)];
                const uint32_t m1 = (tt + 1 < nv) ? vm[(tt + 1) * MG + (vw >> 3)] : 0u;
                const float ps0 = p0 > 0.0f ? p0 * h2f(static_cast<uint16_t>(m0 & 0xffffu)) : 0.0f;
                const float ps1 = p1 > 0.0f ? p1 * h2f(static_cast<uint16_t>(m1 & 0xffffu)) : 0.0f;
                if (p0 > 0.0f) zsum += ps0 * h2f(static_cast<uint16_t>(m0 >> 16));
                if (p1 > 0.0f) zsum += ps1 * h2f(static_cast<uint16_t>(m1 >> 16));
                const float2 ps = make_float2(ps0, ps1);
                const float2 off = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 c = add2(make_float2(__uint_as_float(0x4B000000u | ((w0 >> (2 * i)) & 3u)),
                                                      __uint_as_float(0x4B000000u | ((w1 >> (2 * i)) & 3u))),
                                          off);
                    acc[i] = fma2(ps, c, acc[i]);
                }
            }
        }
        // next iteration's first barrier orders these reads before prob_s is rewritten
    }

    // ---- partial (m, l, o') of this split
    for (int h = tid; h < Hq; h += NT) {
        p.ws_ml[(ws_row + h) * 2] = m_run;
        p.ws_ml[(ws_row + h) * 2 + 1] = l_run;
    }
    if (v_owner) {
        float4* o = reinterpret_cast<float4*>(p.ws_o + (ws_row + vh) * 128 + (vw & 7) * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            o[i] = make_float4(acc[4 * i].x + acc[4 * i].y - zsum, acc[4 * i + 1].x + acc[4 * i + 1].y - zsum,
                               acc[4 * i + 2].x + acc[4 * i + 2].y - zsum, acc[4 * i + 3].x + acc[4 * i + 3].y - zsum);
    }
}

// Sink partial (split index S): raw fp16 K/V rows of the sidecar, natural
// frame, RoPE at each sink's own position.  One CTA per sequence, thread = d.
__global__ void __launch_bounds__(128) decode_sinks_kernel(DecodeParams p, int max_sinks) {
    const int b = blockIdx.x, d = threadIdx.x, Hq = p.Hq, C = p.C;
    const int rep = p.Hq / p.Hkv;
    const int64_t T = p.seq_len[b];
    const int64_t ws_row = (static_cast<int64_t>(b) * (p.S + 1) + p.S) * Hq;
    __shared__ float red[4];
    const int nsink = min(p.cache.sink_count[b], max_sinks);
    const float2* cq = p.rope + (T - 1) * 64;
    const int f = d & 63;
    for (int h = 0; h < Hq; ++h) {
        const uint16_t* qh = p.q + (static_cast<int64_t>(b) * Hq + h) * 128;
        const float a = h2f(qh[f]), bb = h2f(qh[f + 64]);
        const float2 r = __ldg(cq + f);
        const float qd = (d < 64 ? (a * r.x - bb * r.y) : (a * r.y + bb * r.x)) * p.qscale;
        const int kvh = h / rep;
        float m = -INFINITY, l = 0.f, o = 0.f;
        for (int s = 0; s < nsink; ++s) {
            const int pos = p.cache.sink_pos[b * max_sinks + s];
            if (pos >= T) continue;
            const uint16_t* kr = p.cache.sink_k + (static_cast<int64_t>(b) * max_sinks + s) * C + kvh * 128;
            const uint16_t* vr = p.cache.sink_v + (static_cast<int64_t>(b) * max_sinks + s) * C + kvh * 128;
            const float ka = h2f(kr[f]), kb = h2f(kr[f + 64]);
            const float2 rk = __ldg(p.rope + static_cast<int64_t>(pos) * 64 + f);
            const float kd = d < 64 ? (ka * rk.x - kb * rk.y) : (ka * rk.y + kb * rk.x);
            float prod = qd * kd;
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o2);
            __syncthreads();
            if ((d & 31) == 0) red[d >> 5] = prod;
            __syncthreads();
            const float lg = red[0] + red[1] + red[2] + red[3];
            const float m_new = fmaxf(m, lg);
            const float al = exp2f(m - m_new), pr = exp2f(lg - m_new);
            l = l * al + pr;
            o = o * al + pr * h2f(vr[d]);
            m = m_new;
        }
        if (d == 0) {
            p.ws_ml[(ws_row + h) * 2] = m;
            p.ws_ml[(ws_row + h) * 2 + 1] = l;
        }
        p.ws_o[(ws_row + h) * 128 + d] = o;
    }
}

// Merge S packed partials (rotated V frame) and the sink partial (natural
// frame) in a fixed order; out = (H_128 o'_rot + o_sink) / l.
__global__ void __launch_bounds__(128) decode_combine_kernel(DecodeParams p) {
    const int h = blockIdx.x, b = blockIdx.y, d = threadIdx.x, Hq = p.Hq;
    const int64_t base = static_cast<int64_t>(b) * (p.S + 1) * Hq;
    __shared__ float buf[128];
    float M = -INFINITY;
    for (int s = 0; s <= p.S; ++s) M = fmaxf(M, p.ws_ml[((base + static_cast<int64_t>(s) * Hq) + h) * 2]);
    float L = 0.f, rot = 0.f, raw = 0.f;
    for (int s = 0; s <= p.S; ++s) {
        const int64_t r = base + static_cast<int64_t>(s) * Hq + h;
        const float ms = p.ws_ml[r * 2];
        if (ms == -INFINITY) continue;
        const float e = exp2f(ms - M);
        L += e * p.ws_ml[r * 2 + 1];
        const float ov = p.ws_o[r * 128 + d];
        if (s < p.S) rot += e * ov; else raw += e * ov;
    }
    // H_128 on the rotated-frame accumulator (value_rotation inverse)
    buf[d] = rot;
    __syncthreads();
#pragma unroll
    for (int half = 1; half < 128; half <<= 1) {
        const float a = buf[d & ~half], bb = buf[d | half];
        const float y = (d & half) ? a - bb : a + bb;
        __syncthreads();
        buf[d] = y;
        __syncthreads();
    }
    const float hv = buf[d] * (1.0f / sqrtf(128.0f));
    p.out[(static_cast<int64_t>(b) * Hq + h) * 128 + d] = (hv + raw) / L;
}

__global__ void rope_table_kernel(float2* table, int64_t max_pos, double base) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= max_pos * 64) return;
    const int64_t pos = i / 64;
    const int f = static_cast<int>(i % 64);
    const double theta = pow(base, -2.0 * static_cast<double>(f) / 128.0);  // proj/src/rope.cpp:17-24
    const double ang = 1.0 * static_cast<double>(pos) * theta;              // dir * pos * theta
    table[i] = make_float2(static_cast<float>(cos(ang)), static_cast<float>(sin(ang)));
}

template <int N, int L>
__global__ void rotate_keys_kernel(const uint16_t* __restrict__ k, int64_t rows, int C, float norm, float* out) {
    constexpr int R = N / L, LR = ilog2(R), LN = ilog2(N), LL = ilog2(L);
    const int64_t r = blockIdx.y;
    const int u = blockIdx.x, lam = threadIdx.x;
    const uint16_t* src = k + r * C + u * N;
    __shared__ float buf[N];
    float2 x[R];
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = make_float2(h2f(src[lam * R + j]), 0.f);
    bfly_range<R, 0, LR>(x);
#pragma unroll
    for (int j = 0; j < R; ++j) buf[lam * R + j] = x[j].x;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = make_float2(buf[lam + L * j], 0.f);
    bfly_range<R, LR - LL, LN - LL>(x);
#pragma unroll
    for (int j = 0; j < R; ++j) out[r * C + u * N + lam + L * j] = __fmul_rn(x[j].x, norm);
}

template <int N, int REP>
cudaError_t launch_decode_nr(const DecodePlan& plan, const DecodeParams& p, int B, int max_sinks,
                             cudaStream_t s) {
    auto kern = decode_split_kernel<N, REP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(plan.smem));
    if (e != cudaSuccess) return e;
    kern<<<dim3(plan.S, B), plan.NT, plan.smem, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    decode_sinks_kernel<<<B, 128, 0, s>>>(p, max_sinks);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    decode_combine_kernel<<<dim3(p.Hq, B), 128, 0, s>>>(p);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_decode_n(const DecodePlan& plan, const DecodeParams& p, int B, int max_sinks, cudaStream_t s) {
    switch (plan.REP) {
        case 1: return launch_decode_nr<N, 1>(plan, p, B, max_sinks, s);
        case 2: return launch_decode_nr<N, 2>(plan, p, B, max_sinks, s);
        case 4: return launch_decode_nr<N, 4>(plan, p, B, max_sinks, s);
        case 8: return launch_decode_nr<N, 8>(plan, p, B, max_sinks, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            n = 148;
    }
    return n;
}

DecodePlan plan_decode(const rkv_layer_desc& d, int64_t max_seq_len) {
    DecodePlan pl{};
    const int C = d.num_kv_heads * d.head_dim;
    pl.N = d.heads_per_group * d.head_dim;
    pl.REP = d.num_q_heads / d.num_kv_heads;
    const int L = pl.N >= 256 ? 16 : 8;
    const int NG = C / pl.N;
    // enough lane groups for >= 256 threads and >= one V owner per (word, q head)
    int P = 1;
    while (NG * P * L < 256 || NG * P * L < d.num_q_heads * 8) ++P;
    pl.P = P;
    pl.TT = 2 * P;
    pl.NT = NG * P * L;
    pl.smem = smem_layout(C, d.num_q_heads, pl.TT).total;
    if (max_seq_len <= 0 || max_seq_len > d.max_tokens) max_seq_len = d.max_tokens;
    const int ctas = num_sms();  // one CTA per SM (shared memory bound)
    int S = ctas / d.batch;
    if (S < 1) S = 1;
    // keep >= 4 tiles per split
    const int64_t max_split = (max_seq_len + 4 * pl.TT - 1) / (4 * pl.TT);
    if (S > max_split) S = static_cast<int>(max_split > 0 ? max_split : 1);
    int64_t chunk = (max_seq_len + S - 1) / S;
    chunk = (chunk + pl.TT - 1) / pl.TT * pl.TT;
    pl.chunk = static_cast<int>(chunk);
    pl.S = static_cast<int>((max_seq_len + chunk - 1) / chunk);
    return pl;
}

cudaError_t launch_decode(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p, cudaStream_t s) {
    switch (plan.N) {
        case 128: return launch_decode_n<128>(plan, p, d.batch, d.max_sinks, s);
        case 256: return launch_decode_n<256>(plan, p, d.batch, d.max_sinks, s);
        case 512: return launch_decode_n<512>(plan, p, d.batch, d.max_sinks, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_rope_table(const rkv_layer_desc& d, float2* table, int64_t max_pos, cudaStream_t s) {
    const int64_t n = max_pos * 64;
    rope_table_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(table, max_pos, d.rope_base);
    return cudaGetLastError();
}

cudaError_t launch_rotate_keys(const rkv_layer_desc& d, const uint16_t* k, int64_t rows, float* out, cudaStream_t s) {
    const int C = d.num_kv_heads * d.head_dim, N = d.heads_per_group * d.head_dim;
    const float norm = 1.0f / sqrtf(static_cast<float>(N));
    dim3 grid(C / N, static_cast<unsigned>(rows));
    switch (N) {
        case 128: rotate_keys_kernel<128, 8><<<grid, 8, 0, s>>>(k, rows, C, norm, out); break;
        case 256: rotate_keys_kernel<256, 16><<<grid, 16, 0, s>>>(k, rows, C, norm, out); break;
        case 512: rotate_keys_kernel<512, 16><<<grid, 16, 0, s>>>(k, rows, C, norm, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace rkv
