// rkv_common.cuh -- shared device helpers for the sm_100a RotateKV kernels.
//
// FWHT layouts.  An N-point Walsh-Hadamard vector (N = G*128) is owned by a
// group of L lanes, R = N/L values per lane:
//   layout A: lane l holds indices l*R + j      (register bits = low index bits)
//   layout B: lane l holds indices l + L*j      (register bits = high index bits)
// Stages on index bits 0..log2(R)-1 run in registers in layout A, one
// transpose through shared memory, then stages on the remaining high bits run
// in registers in layout B.  Stage order is bit 0 first, exactly the
// reference's half = 1, 2, ..., N/2 order (proj/src/hadamard.cpp:51-60), so
// results are bit-identical to fwht_inplace.  Every register holds a float2:
// the SAME index of two tokens, so every butterfly is one FADD2.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rotatekv/rotatekv.h"

namespace rkv {

constexpr int kHeadDim = 128;
constexpr int kQuantGroup = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kRopeRow = 128;  // float4 per position pair in the RoPE table (decode_attention.cu)

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// ------------------------------------------------------------ FWHT stages
// Butterflies between registers j and j+H (H a power of two), packed.
template <int R, int H>
__device__ __forceinline__ void bfly(float2 (&x)[R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if ((j & H) == 0) {
            float2 a = x[j], b = x[j + H];
            x[j] = add2(a, b);
            x[j + H] = sub2(a, b);
        }
    }
}

// Stages on register bits [lo, hi) in increasing order.
template <int R, int LO, int HI>
__device__ __forceinline__ void bfly_range(float2 (&x)[R]) {
    if constexpr (LO < HI) {
        bfly<R, (1 << LO)>(x);
        bfly_range<R, LO + 1, HI>(x);
    }
}

// ------------------------------------------------------ TMA bulk + mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release (default .release.cta)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RKV_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RKV_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// mbar_wait for a role thread that may wait long (TMA producer, MMA issuer):
// the try_wait suspends in hardware for up to `hint` ns between polls instead
// of spinning, leaving issue slots to the warps sharing its SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RKV_WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra RKV_WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// 1-D TMA bulk copy global -> shared (SASS: UBLKCP), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// (a & mask) | orv in ONE LOP3 (the compiler otherwise emits two).
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t mask, uint32_t orv) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(orv));
    return r;
}

__device__ __forceinline__ uint4 lds128(const void* p) {
    return *reinterpret_cast<const uint4*>(p);
}

// ----------------------------------------------------- scale / code helpers
// Smallest fp16 >= x (x > 0), saturating at 65504 (mirrors
// e4m3_encode_ceil's saturation, proj/src/fp8.cpp:68-75).
__device__ __forceinline__ uint16_t fp16_ceil(float x) {
    if (!(x < 65504.0f)) return 0x7bffu;
    __half h = __float2half_rn(x);
    uint16_t b = __half_as_ushort(h);
    if (__half2float(h) < x) b = static_cast<uint16_t>(b + 1u);
    return b;
}

// Smallest OCP e4m3fn value >= x (x >= 0), == e4m3_decode(e4m3_encode_ceil(x))
// (proj/src/fp8.cpp:68-75): RNE-then-bump equals "first table entry >= x".
__device__ __forceinline__ float e4m3_ceil_value(float x) {
    if (x >= 448.0f) return 448.0f;
    // walk the monotone positive table: codes 0..0x7e
    int lo = 0, hi = 0x7e;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        int e = (mid >> 3) & 0xf, m = mid & 7;
        float v = e == 0 ? ldexpf(static_cast<float>(m), -9) : ldexpf(1.0f + m * 0.125f, e - 7);
        if (v >= x) hi = mid; else lo = mid + 1;
    }
    int e = (lo >> 3) & 0xf, m = lo & 7;
    return e == 0 ? ldexpf(static_cast<float>(m), -9) : ldexpf(1.0f + m * 0.125f, e - 7);
}

struct GroupQuant {
    float t1, t2, t3;
    uint32_t meta;
};

// proj/src/quant.cpp:74-94 for bits = 2 (scale rounded up to fp16
// or e4m3 as in the reference).
//   zero = clamp(rhaz(-mn / s), 0, 3): RN64(-mn/s) >= k + 0.5 exactly when
//   -mn >= (k + 0.5) s (mn is fp32, s has <= 11 significant bits, so the
//   quotient's rounding can never reach k + 0.5 from below), and (k + 0.5) s
//   is exact in fp32.
//   code >= k  <=>  rhaz(x/s) >= m := k - zero  <=>  x >= (m - 0.5) s (m >= 1),
//   x > (m - 0.5) s (m <= 0); (m - 0.5) s is exact in fp32 and the strict
//   case becomes >= on the next float up.
template <int FMT>
__device__ __forceinline__ GroupQuant group_params(float mn, float mx) {
    const double range = __dsub_rn(static_cast<double>(mx), static_cast<double>(mn));
    float raw = __double2float_rn(__ddiv_rn(range, 3.0));
    if (raw < 1e-8f) raw = 1e-8f;
    uint16_t sbits;
    float sf;
    if constexpr (FMT == RKV_SCALE_E4M3_CEIL) {
        sf = e4m3_ceil_value(raw);
        sbits = __half_as_ushort(__float2half_rn(sf));  // exact: e4m3 values are fp16 values
    } else {
        sbits = fp16_ceil(raw);
        sf = __half2float(__ushort_as_half(sbits));
    }
    const float nm = -mn;
    const int z = (nm >= 0.5f * sf) + (nm >= 1.5f * sf) + (nm >= 2.5f * sf);
    float t[3];
#pragma unroll
    for (int k = 1; k <= 3; ++k) {
        const int m = k - z;
        float tt = __fmul_rn(static_cast<float>(m) - 0.5f, sf);
        if (m <= 0) tt = __uint_as_float(__float_as_uint(tt) - 1u);  // tt < 0: next float toward +inf
        t[k - 1] = tt;
    }
    GroupQuant g;
    g.t1 = t[0];
    g.t2 = t[1];
    g.t3 = t[2];
    g.meta = static_cast<uint32_t>(sbits) | (static_cast<uint32_t>(__half_as_ushort(__int2half_rn(z))) << 16);
    return g;
}

// Programmatic dependent launch (griddepcontrol, sm_90+).  A kernel launched
// with cudaLaunchAttributeProgrammaticStreamSerialization may start while the
// previous kernel in the stream drains; pdl_wait() blocks until that kernel
// has completed and its memory is visible (a no-op without the attribute).
// pdl_trigger() lets the NEXT kernel's CTAs launch once every CTA of this one
// has triggered or exited.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// (cos, sin) of position pos, frequency f from section 1 of the RoPE table
__device__ __forceinline__ float2 rope_at(const float4* t, int64_t pos, int f) {
    const float4 r = __ldg(t + (pos >> 1) * kRopeRow + f);
    return (pos & 1) ? make_float2(r.y, r.w) : make_float2(r.x, r.z);
}

}  // namespace rkv
