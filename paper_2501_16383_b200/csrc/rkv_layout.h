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
constexpr uint32_t kPlanMagic = 0x504B5652u;  // "RVKP"
constexpr int kPlanHeader = 16;
enum { PH_MAGIC = 0, PH_VERSION, PH_N, PH_L, PH_C, PH_W, PH_COST };

RKV_HD inline int plan_words(int W) { return kPlanHeader + W + 16 * W; }

}  // namespace rkv
