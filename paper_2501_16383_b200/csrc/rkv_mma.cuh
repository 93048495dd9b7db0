// rkv_mma.cuh -- register-level helpers of the tensor-core kernels
// (decode_mma.cu, prefill.cu): packed half2 arithmetic, mixed fp16/fp32
// FMAs, PRMT, and mma.sync wrappers with the H_16 A fragment.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace rkv {
namespace mma {

__device__ __forceinline__ int64_t lmin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t h2sub(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t h2mul(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t h2add(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// half2(lo, hi) from two floats, round to nearest (F2FP.F16.F32.PACK_AB)
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// d - float(half) in one FHADD (mixed f16 + f32 add, sm_100)
__device__ __forceinline__ float sub_lo(float d, uint32_t h) {
    float r;
    asm("{.reg .b16 l, u, n; mov.b32 {l, u}, %1; neg.f16 n, l; add.rn.f32.f16 %0, n, %2;}" : "=f"(r) : "r"(h), "f"(d));
    return r;
}
__device__ __forceinline__ float sub_hi(float d, uint32_t h) {
    float r;
    asm("{.reg .b16 l, u, n; mov.b32 {l, u}, %1; neg.f16 n, u; add.rn.f32.f16 %0, n, %2;}" : "=f"(r) : "r"(h), "f"(d));
    return r;
}
// c + a.half(SA) * b.half(SB) in fp32 (FHFMA)
template <int SA, int SB>
__device__ __forceinline__ float fhfma(uint32_t a, uint32_t b, float c) {
    float r;
    if constexpr (SA == 0 && SB == 0)
        asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, al, bl, %3;}"
            : "=f"(r) : "r"(a), "r"(b), "f"(c));
    else if constexpr (SA == 1 && SB == 0)
        asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, ah, bl, %3;}"
            : "=f"(r) : "r"(a), "r"(b), "f"(c));
    else if constexpr (SA == 0 && SB == 1)
        asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, al, bh, %3;}"
            : "=f"(r) : "r"(a), "r"(b), "f"(c));
    else
        asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, ah, bh, %3;}"
            : "=f"(r) : "r"(a), "r"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float ex2(float x) {  // 2^x, MUFU.EX2 (2^-inf = 0)
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// D = A(16x16, fp16) * B(16x8, fp16) + C, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                         const float (&c)[4]) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]),
          "f"(c[3]));
}

// D = RN16(A(16x16) * B(16x8) + C), fp16 accumulator.  The tensor core adds
// the exact products and C and rounds once (tools/mb_f16acc.cu: 8.4 M
// dequantised-K-like H_16 products, every result == RN16 of the exact sum),
// so with C = 0 it yields hi = RN16(Y) and with A = -H, C = hi the residual
// -(Y - hi) rounded once: the fp16 hi/lo split of Y without F2FP/FHADD.
__device__ __forceinline__ void mma16816h(uint32_t (&d)[2], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                          uint32_t c0, uint32_t c1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%9};"
        : "=r"(d[0]), "=r"(d[1])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c0), "r"(c1));
}
// the same fragment negated (sign bit of every fp16 entry; 0 -> -0 is harmless)
__device__ __forceinline__ void negate_frag(uint32_t (&dst)[4], const uint32_t (&src)[4]) {
#pragma unroll
    for (int r = 0; r < 4; ++r) dst[r] = src[r] ^ 0x80008000u;
}

__device__ __forceinline__ void mma1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b));
}

// H_16 as an m16n8k16 A fragment (row-major, +-1 in fp16): a[0] = (g, 2t..),
// a[1] = (g+8, 2t..), a[2] = (g, 2t+8..), a[3] = (g+8, 2t+8..)
__device__ __forceinline__ void hadamard16_frag(uint32_t (&a)[4], int lane) {
    const int g = lane >> 2, t = lane & 3;
    auto h = [](int m, int k) -> uint32_t { return (__popc(m & k) & 1) ? 0xBC00u : 0x3C00u; };
    const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r] = h(rows[r], cols[r]) | (h(rows[r], cols[r] + 1) << 16);
}
// a[2] == a[0] and a[3] == a[1] on every lane (H_16 rows never see column bit
// 3 for g < 8).  XOR-ing an opaque zero keeps the four registers distinct;
// otherwise the compiler shares them and rebuilds the aligned register quad
// the mma.sync A operand needs (4 MOVs) in front of every MMA.
__device__ __forceinline__ void hadamard16_frag(uint32_t (&a)[4], int lane, uint32_t opaque_zero) {
    hadamard16_frag(a, lane);
    a[2] ^= opaque_zero;
    a[3] ^= opaque_zero;
}

// A fragment of a masked H_16: (-1)^popcount(m & k & mask) where m and k agree
// outside `mask`, 0 elsewhere -- H over the mask bits, the identity over the
// others.  The GQA tiles' second factor contracts over channel bits (4, 5, 7,
// 6) = k bits (0, 1, 2, 3): mask 15 for G = 2 (H_256), 11 for G = 1 (H_128 per
// head, the identity over the head bit 7).
__device__ __forceinline__ void hadamard_mask_frag(uint32_t (&a)[4], int lane, int mask, uint32_t opaque_zero) {
    const int g = lane >> 2, t = lane & 3;
    auto h = [mask](int m, int k) -> uint32_t {
        if ((m ^ k) & ~mask & 15) return 0u;
        return (__popc(m & k & mask) & 1) ? 0xBC00u : 0x3C00u;
    };
    const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r] = h(rows[r], cols[r]) | (h(rows[r], cols[r] + 1) << 16);
    a[2] ^= opaque_zero;
    a[3] ^= opaque_zero;
}

// A fragment of the second FWHT factor of a 512-channel (pseudo-)group, over
// channel bits (4, 5, 7, 8) = k bits (0, 1, 2, 3):  AG = 4 (G = 4 heads per
// rotation group): H_16;  AG = 2: H_8 on bits 4, 5, 7 and the identity on
// bit 8 (two 256-channel groups);  AG = 1: H_4 on bits 4, 5 and the identity
// on the head bits 7, 8 (four per-head rotations).  Entries +-1 or 0.
template <int AG>
__device__ __forceinline__ void hadamard_f2_frag(uint32_t (&a)[4], int lane, uint32_t opaque_zero) {
    constexpr int kMask = AG == 4 ? 15 : AG == 2 ? 7 : 3;
    const int g = lane >> 2, t = lane & 3;
    auto h = [](int m, int k) -> uint32_t {
        if ((m & ~kMask) != (k & ~kMask)) return 0u;
        return (__popc(m & k & kMask) & 1) ? 0xBC00u : 0x3C00u;
    };
    const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r] = h(rows[r], cols[r]) | (h(rows[r], cols[r] + 1) << 16);
    a[2] ^= opaque_zero;
    a[3] ^= opaque_zero;
}

}  // namespace mma
}  // namespace rkv
