// rkv_plan.cu -- host construction of the per-layer decode plan: which packed
// word each decode thread scatters, chosen to minimise shared-memory bank
// conflicts of the un-reorder scatter.
//
// The scatter (K1 in decode_attention.cu) sends slot j of a packed row to
// natural channel perm[j] (proj/src/reorder.cpp:112-128, inverted).  Lanes
// store code e of their word in round e (e = 0..15; the code order stays
// static so no per-round index arithmetic is needed).  A half-warp's 16
// 8-byte stores cost as many shared-memory wavefronts as the largest number
// of lanes hitting one bank slot.  With the calibrated (random) permutation
// that is ~3.1 per round when words are taken in order.  The permutation is
// fixed per layer, so the words are re-assigned to word positions (16
// consecutive positions = one half-warp) once, by simulated annealing on the
// summed per-round maximum multiplicity (~2.2 per round), and the kernel
// reads its word index and the 16 store addresses from the plan.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "rkv_internal.h"
#include "rkv_layout.h"

namespace rkv {

namespace {

struct SplitMix {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// sum over rounds e of the largest bank-slot multiplicity among the GS words
// of one store group (16 lanes x 8-byte slots, or 32 lanes x 4-byte banks)
int group_cost(const int* cls, const int* words, int GS) {
    int cost = 0;
    for (int e = 0; e < 16; ++e) {
        int cnt[32] = {0};
        int mx = 0;
        for (int i = 0; i < GS; ++i) mx = std::max(mx, ++cnt[cls[words[i] * 16 + e]]);
        cost += mx;
    }
    return cost;
}

}  // namespace

bool build_decode_plan(const rkv_layer_desc& d, const int32_t* perm, std::vector<uint32_t>& out, int& cost_out) {
    const int kind = decode_kind(d);
    const int C = d.num_kv_heads * d.head_dim, N = kind == kDecodeMma ? mma_layout_n(d) : d.heads_per_group * d.head_dim;
    const int W = C / 16;
    if (kind == kDecodeGeneric) {  // generic kernel: identity word order, offsets = padded channel perm[j]
        out.assign(static_cast<size_t>(plan_words(W)), 0u);
        out[PH_MAGIC] = kPlanMagic;
        out[PH_VERSION] = 3;
        out[PH_N] = static_cast<uint32_t>(N);
        out[PH_L] = 0;
        out[PH_C] = static_cast<uint32_t>(C);
        out[PH_W] = static_cast<uint32_t>(W);
        out[PH_KIND] = static_cast<uint32_t>(kind);
        uint32_t* om = out.data() + kPlanHeader;
        uint32_t* addr = om + W;
        for (int w = 0; w < W; ++w) {
            om[w] = static_cast<uint32_t>(w);
            for (int e = 0; e < 16; ++e)
                addr[(static_cast<size_t>(e / 4) * W + w) * 4 + e % 4] = static_cast<uint32_t>(
                    perm[w * 16 + e] + ((perm[w * 16 + e] >> 5) << 2));  // padded (generic.cu padc)
        }
        cost_out = 0;
        return true;
    }
    const int GS = kind == kDecodeMma ? 32 : 16;  // lanes whose stores share a wavefront
    const int G = (W + GS - 1) / GS;              // store groups; the last one may be partial (e.g. C = 1280)
    auto gsize = [&](int k) { return std::min(GS, W - k * GS); };
    auto pos = [&](int c) { return kind == kDecodeMma ? mma_pos(N, c) : knat_pos(N, c) * 8; };
    std::vector<int> cls(static_cast<size_t>(C));
    for (int j = 0; j < C; ++j)
        cls[static_cast<size_t>(j)] = kind == kDecodeMma ? (pos(perm[j]) >> 2) & 31 : (pos(perm[j]) >> 3) & 15;

    std::vector<int> omega(static_cast<size_t>(W));
    for (int w = 0; w < W; ++w) omega[static_cast<size_t>(w)] = w;
    std::vector<int> cost(static_cast<size_t>(G));
    for (int k = 0; k < G; ++k)
        cost[static_cast<size_t>(k)] = group_cost(cls.data(), &omega[static_cast<size_t>(k) * GS], gsize(k));
    if (G > 1) {
        SplitMix rng{0x5EEDULL ^ static_cast<uint64_t>(C) * 0x9E3779B97F4A7C15ULL};
        const long iters = 120000L * std::min(G, 8);
        for (long it = 0; it < iters; ++it) {
            const double T = 1.5 * (1.0 - static_cast<double>(it) / static_cast<double>(iters)) + 1e-3;
            const int p1 = static_cast<int>(rng.next() % static_cast<uint64_t>(W));
            const int p2 = static_cast<int>(rng.next() % static_cast<uint64_t>(W));
            const int g1 = p1 / GS, g2 = p2 / GS;
            if (g1 == g2) continue;
            std::swap(omega[static_cast<size_t>(p1)], omega[static_cast<size_t>(p2)]);
            const int c1 = group_cost(cls.data(), &omega[static_cast<size_t>(g1) * GS], gsize(g1));
            const int c2 = group_cost(cls.data(), &omega[static_cast<size_t>(g2) * GS], gsize(g2));
            const int dl = c1 + c2 - cost[static_cast<size_t>(g1)] - cost[static_cast<size_t>(g2)];
            if (dl <= 0 || rng.uniform() < std::exp(-dl / T)) {
                cost[static_cast<size_t>(g1)] = c1;
                cost[static_cast<size_t>(g2)] = c2;
            } else {
                std::swap(omega[static_cast<size_t>(p1)], omega[static_cast<size_t>(p2)]);
            }
        }
    }
    int total = 0;
    for (int c : cost) total += c;
    cost_out = total;

    out.assign(static_cast<size_t>(plan_words(W)), 0u);
    out[PH_MAGIC] = kPlanMagic;
    out[PH_VERSION] = 3;
    out[PH_N] = static_cast<uint32_t>(N);
    out[PH_L] = static_cast<uint32_t>(fwht_lanes(N));
    out[PH_C] = static_cast<uint32_t>(C);
    out[PH_W] = static_cast<uint32_t>(W);
    out[PH_COST] = static_cast<uint32_t>(total);
    out[PH_KIND] = static_cast<uint32_t>(kind);
    uint32_t* om = out.data() + kPlanHeader;
    uint32_t* addr = om + W;
    for (int wp = 0; wp < W; ++wp) {
        const int w = omega[static_cast<size_t>(wp)];
        om[wp] = static_cast<uint32_t>(w);
        for (int e = 0; e < 16; ++e)
            addr[(static_cast<size_t>(e / 4) * W + wp) * 4 + e % 4] = static_cast<uint32_t>(pos(perm[w * 16 + e]));
    }
    return true;
}

}  // namespace rkv
