// rkv_layout.h -- shared (host + device) layout of the decode kernel's
// shared-memory K tile and of the per-layer decode plan.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define RKV_HD __host__ __device__
#else
#define RKV_HD
#endif

namespace rkv {

// Lanes per FWHT group and float2 registers per lane for an N-point group.
RKV_HD constexpr int fwht_lanes(int N) { return N >= 256 ? 16 : 8; }
RKV_HD constexpr int fwht_regs(int N) { return N / fwht_lanes(N); }

// The K tile holds, per token pair, one float2 (token, token+1) per channel.
// FWHT group g occupies a unit of L rows; row la (the layout-A owner lane)
// holds R channels plus one float2 of padding, so the 16 lanes of a
// half-warp hit 16 different 8-byte bank slots for every layout-A access
// (row stride 8*(R+1) bytes) and for every layout-B access (16 consecutive
// channels of one row).  No address swizzle, no per-access ALU.
RKV_HD inline int knat_unit(int N) { return fwht_lanes(N) * (fwht_regs(N) + 1); }
RKV_HD inline int knat_pos(int N, int c) {
    const int L = fwht_lanes(N), R = N / L;
    const int g = c / N, i = c % N;
    return g * L * (R + 1) + (i / R) * (R + 1) + (i % R);
}
RKV_HD inline int knat_pair_f2(int N, int C) { return (C / N) * knat_unit(N); }  // float2 per pair row

// ---------------------------------------------------------------------------
// Tensor-core decode (decode_mma.cu) K tile: per token pair one u32 =
// half2(token, token+1) per channel, laid out in mma.sync B-fragment order.
// A group's N = 128*G channel index i is split into bit fields:
//   F1 = bits 0-3                   contraction of the first  H_16 MMA
//   F2 = bits {4,5,7,8} (G = 4)     contraction of the second H_16 MMA
//        bits {4,5,7,6} (G = 2)
//   outer = bit 6 (G = 4 only)      the last H_2, fused into RoPE
// B fragment of m16n8k16 (k = F1, n = F2 bits 0-2): lane = 4*n + (k>>1 & 3)
// holds k = 2t,2t+1 (kreg 0) and 2t+8,2t+9 (kreg 1); instance jc = F2 bit 3
// (+ 2*outer).  Each lane's EPL = N/32 elements (4 per 16-byte chunk, one
// chunk per instance) are contiguous; chunks are XOR-swizzled by lane so the
// per-lane LDS.128 fragment loads are bank-conflict free.
// Slot of frequency pair j (f = 2j, 2j+1) in section 2 of a RoPE table row:
// the tensor-core kernels read pairs j = tl + 4 f1 + 8 q (lane bits tl, q) as
// one LDS.128 per lane; with slot = tl + 4 q + 16 f1 a warp's 16 distinct
// entries are 256 contiguous bytes (2 wavefronts, no bank conflict).
RKV_HD constexpr int rope_pair_slot(int j) { return (j & 3) | (((j >> 3) & 3) << 2) | (((j >> 2) & 1) << 4); }

RKV_HD inline int mma_nj(int N) { return N / 128; }  // MMA-1 instances = 16-byte chunks per lane
RKV_HD inline int mma_swz(int N, int lane) { return N == 512 ? (lane >> 1) & 3 : (lane >> 2) & 1; }
RKV_HD inline int mma_pos(int N, int c) {  // byte offset of channel c in a token-pair row
    const int g = c / N, i = c % N;
    const int k = i & 15;
    const int n = ((i >> 4) & 1) | (((i >> 5) & 1) << 1) | (((i >> 7) & 1) << 2);
    const int jc = N == 512 ? (((i >> 8) & 1) | (((i >> 6) & 1) << 1)) : ((i >> 6) & 1);
    const int lane = 4 * n + ((k >> 1) & 3);
    const int nj = mma_nj(N);
    const int chunk = jc ^ mma_swz(N, lane);
    return g * N * 4 + lane * nj * 16 + chunk * 16 + ((k >> 3) * 2 + (k & 1)) * 4;
}

// Decode plan (rkv_layer_plan_init, rkv_plan.cu): the un-reorder scatter's
// word assignment.
//   words[0 .. kPlanHeader)   header (magic, version, N, L, C, W, cost)
//   then W u32                omega[wp]: packed word handled at word position wp
//   then 16*W u32             byte offset (within a token-pair row of the K
//                             tile) of code e of word omega[wp], laid out
//                             [e/4][wp][e%4] so a warp's uint4 loads are
//                             conflict-free
// A half-warp = 16 consecutive word positions; in round e every lane stores
// code e of its word.  omega is chosen per layer to spread each round's 16
// stores over distinct 8-byte bank slots.
// For the tensor-core kernel (PH_KIND = 1) the offsets are mma_pos() bytes,
// a warp = 32 consecutive word positions stores half2 words (STS.32) and
// omega spreads each round's 32 stores over distinct 4-byte banks.
constexpr uint32_t kPlanMagic = 0x504B5652u;  // "RVKP"
constexpr int kPlanHeader = 16;
enum { PH_MAGIC = 0, PH_VERSION, PH_N, PH_L, PH_C, PH_W, PH_COST, PH_KIND };
enum { kDecodeSimt = 0, kDecodeMma = 1, kDecodeGeneric = 2 };

RKV_HD inline int plan_words(int W) { return kPlanHeader + W + 16 * W; }

// Header check in the decode kernels' prologue: a plan built for another layer
// shape or kernel kind makes the decode emit NaN (loud) instead of attention
// computed with the wrong scatter offsets or RoPE layout.
RKV_HD inline bool plan_matches(const uint32_t* plan, int kind, int N, int C) {
    return plan[PH_MAGIC] == kPlanMagic && plan[PH_KIND] == static_cast<uint32_t>(kind) &&
           plan[PH_N] == static_cast<uint32_t>(N) && plan[PH_C] == static_cast<uint32_t>(C);
}

}  // namespace rkv
