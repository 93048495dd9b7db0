/*
 * rkv_oracle.c -- CPU restatement of the RotateKV KV-cache hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see rkv_oracle.h).  Plain C11, single thread,
 * compiled with -ffp-contract=off so that every float/double operation rounds
 * exactly where the reference's does.  Function headers cite the reference
 * file:line they restate; "PAPER" / "SURVEY D<n>" cite the documented
 * north-star deviations (fp16 scales, GQA, raw fp16 sinks).
 */
#include "rkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ fp16 */

float rkvo_half_to_float(uint16_t h) {
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
    float f;
    if (e == 0) {
        f = ldexpf((float)m, -24);
        memcpy(&x, &f, 4);
        x |= sign;
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e - 15u + 127u) << 23) | (m << 13);
    }
    memcpy(&f, &x, 4);
    return f;
}

/* IEEE round-to-nearest-even float -> binary16 (the semantics of
 * __float2half_rn on the device). */
uint16_t rkvo_float_to_half_rn(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t a = x & 0x7fffffffu;
    if (a >= 0x7f800000u) return (uint16_t)(sign | (a > 0x7f800000u ? 0x7e00u : 0x7c00u));
    if (a < 0x38800000u) { /* below 2^-14: subnormal half or zero */
        if (a < 0x33000000u) return (uint16_t)sign; /* < 2^-25 (2^-25 ties to 0) */
        uint32_t e = a >> 23, m = (a & 0x7fffffu) | 0x800000u;
        int shift = 126 - (int)e;
        uint32_t q = m >> shift, rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1);
        if (rem > half || (rem == half && (q & 1u))) q++;
        return (uint16_t)(sign | q);
    }
    uint32_t e = (a >> 23) - 127u + 15u, m = a & 0x7fffffu;
    uint32_t q = (e << 10) | (m >> 13), rem = m & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) q++;
    if (q >= 0x7c00u) q = 0x7c00u;
    return (uint16_t)(sign | q);
}

/* the north star stores fp16 scales.  Following the reference's
 * no-undershoot rule (proj/src/quant.cpp:79-82 storing e4m3_encode_ceil,
 * proj/src/fp8.cpp:68-75) the stored scale is the smallest fp16 >= x,
 * saturating at the largest finite value like fp8.cpp:71. */
uint16_t rkvo_fp16_ceil(float x) {
    if (!(x < 65504.0f)) return 0x7bffu;
    uint16_t h = rkvo_float_to_half_rn(x);
    if (rkvo_half_to_float(h) < x) h = (uint16_t)(h + 1u);
    return h;
}

/* ------------------------------------------------------------------ e4m3 */

/* proj/src/fp8.cpp:14-27 (positive table of OCP e4m3fn). */
static float e4m3_table(int code) {
    int exp = (code >> 3) & 0xf, man = code & 0x7;
    if (code == 0x7f) return NAN;
    if (exp == 0) return ldexpf((float)man, -9);
    return ldexpf(1.0f + (float)man / 8.0f, exp - 7);
}

/* proj/src/fp8.cpp:56-59 */
float rkvo_e4m3_decode(uint8_t code) {
    float mag = e4m3_table(code & 0x7f);
    return (code & 0x80) ? -mag : mag;
}

/* proj/src/fp8.cpp:34-53: binary search for the largest code <= a, then RNE. */
static uint8_t e4m3_encode_magnitude_rne(float a) {
    const int kmax = 0x7e;
    if (a >= e4m3_table(kmax)) return (uint8_t)kmax;
    int lo = 0, hi = kmax;
    while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if (e4m3_table(mid) <= a) lo = mid; else hi = mid - 1;
    }
    if (lo == kmax) return (uint8_t)kmax;
    float below = e4m3_table(lo), above = e4m3_table(lo + 1);
    float dlo = a - below, dhi = above - a;
    if (dlo < dhi) return (uint8_t)lo;
    if (dhi < dlo) return (uint8_t)(lo + 1);
    return (lo % 2 == 0) ? (uint8_t)lo : (uint8_t)(lo + 1);
}

/* proj/src/fp8.cpp:61-66 */
uint8_t rkvo_e4m3_encode(float x) {
    if (isnan(x)) return 0x7f;
    uint8_t sign = signbit(x) ? 0x80 : 0x00;
    return (uint8_t)(sign | e4m3_encode_magnitude_rne(fabsf(x)));
}

/* proj/src/fp8.cpp:68-75 */
uint8_t rkvo_e4m3_encode_ceil(float x) {
    float a = fabsf(x);
    if (a >= e4m3_table(0x7e)) return 0x7e;
    int code = e4m3_encode_magnitude_rne(a);
    if (e4m3_table(code) < a) ++code;
    return (uint8_t)code;
}

/* --------------------------------------------------------------- hadamard */

static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

/* proj/src/hadamard.cpp:18-33 (RotationPlan::make validation);
 * kMaxHadamardLog2 = 13 (proj/include/rotatekv/hadamard.hpp:21). */
static int rotation_plan_ok(int64_t head_dim, int64_t heads_per_group, int64_t num_heads) {
    if (head_dim < 1 || heads_per_group < 1 || num_heads < 1) return 0;
    if (num_heads % heads_per_group != 0) return 0;
    int64_t n = heads_per_group * head_dim;
    if (!is_pow2(n)) return 0;
    if (n > ((int64_t)1 << 13)) return 0;
    return 1;
}

/* proj/src/hadamard.cpp:47-64: radix-2 stages half = 1, 2, ..., n/2, fp32
 * a+b / a-b, then one multiply by 1.0f/sqrtf(n).  Stage order matters for
 * bit-exactness. */
int rkvo_fwht_inplace(float* v, int64_t n) {
    if (!is_pow2(n)) return -1;
    for (int64_t half = 1; half < n; half <<= 1) {
        for (int64_t base = 0; base < n; base += 2 * half) {
            for (int64_t i = base; i < base + half; ++i) {
                float a = v[i], b = v[i + half];
                v[i] = a + b;
                v[i + half] = a - b;
            }
        }
    }
    float scale = 1.0f / sqrtf((float)n);
    for (int64_t i = 0; i < n; ++i) v[i] *= scale;
    return 0;
}

/* proj/src/hadamard.cpp:66-84: FWHT over each contiguous block of G heads. */
int rkvo_rotate_rows(float* x, int64_t rows, int64_t head_dim, int64_t heads_per_group,
                     int64_t num_heads) {
    if (!rotation_plan_ok(head_dim, heads_per_group, num_heads)) return -1;
    int64_t c = head_dim * num_heads, n = head_dim * heads_per_group;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t g = 0; g < num_heads / heads_per_group; ++g)
            rkvo_fwht_inplace(x + r * c + g * n, n);
    return 0;
}

/* ---------------------------------------------------------------- reorder */

/* proj/src/reorder.cpp:25-29 */
int rkvo_invert_perm(const int32_t* perm, int64_t channels, int32_t* inverse) {
    for (int64_t i = 0; i < channels; ++i) inverse[i] = -1;
    for (int64_t i = 0; i < channels; ++i) {
        int32_t p = perm[i];
        if (p < 0 || p >= channels || inverse[p] != -1) return -1;
        inverse[p] = (int32_t)i;
    }
    return 0;
}

/* proj/src/reorder.cpp:112-128: dst[j] = src[p[j]], p = perm or its inverse. */
int rkvo_apply_reorder(const float* x, int64_t rows, int64_t channels, const int32_t* perm,
                       int inverse, float* out) {
    int32_t* inv = NULL;
    const int32_t* p = perm;
    if (inverse) {
        inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)channels);
        if (!inv || rkvo_invert_perm(perm, channels, inv) != 0) { free(inv); return -1; }
        p = inv;
    }
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t j = 0; j < channels; ++j) out[r * channels + j] = x[r * channels + p[j]];
    free(inv);
    return 0;
}

/* stable ascending argsort by key (std::stable_sort semantics). */
static void stable_argsort(const double* key, int32_t* idx, int32_t* tmp, int64_t lo, int64_t hi) {
    if (hi - lo < 2) return;
    int64_t mid = (lo + hi) / 2;
    stable_argsort(key, idx, tmp, lo, mid);
    stable_argsort(key, idx, tmp, mid, hi);
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        if (key[idx[j]] < key[idx[i]]) tmp[k++] = idx[j++];
        else tmp[k++] = idx[i++];
    }
    while (i < mid) tmp[k++] = idx[i++];
    while (j < hi) tmp[k++] = idx[j++];
    for (int64_t t = lo; t < hi; ++t) idx[t] = tmp[t];
}

/* proj/src/reorder.cpp:91-110: per-channel double sums over the rows in
 * sequence, stable ascending argsort.  SURVEY D3: stat=MEAN_ABS uses the
 * north star's mean |K| statistic instead of the signed sum. */
int rkvo_calibrate_reorder(const float* rows, int64_t n_rows, int64_t channels, int stat,
                           int32_t* perm_out, int32_t* inverse_out) {
    if (n_rows < 1 || channels < 1) return -1;
    double* sums = (double*)calloc((size_t)channels, sizeof(double));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)channels);
    if (!sums || !tmp) { free(sums); free(tmp); return -1; }
    for (int64_t i = 0; i < n_rows; ++i)
        for (int64_t j = 0; j < channels; ++j) {
            double v = (double)rows[i * channels + j];
            sums[j] += (stat == RKVO_STAT_MEAN_ABS) ? fabs(v) : v;
        }
    if (stat == RKVO_STAT_MEAN_ABS)
        for (int64_t j = 0; j < channels; ++j) sums[j] /= (double)n_rows;
    for (int64_t j = 0; j < channels; ++j) perm_out[j] = (int32_t)j;
    stable_argsort(sums, perm_out, tmp, 0, channels);
    free(sums);
    free(tmp);
    if (inverse_out) return rkvo_invert_perm(perm_out, channels, inverse_out);
    return 0;
}

/* ------------------------------------------------------------------- rope */

/* proj/src/rope.cpp:17-36,67-84: half-split pairs (i, i+d/2), theta_i =
 * base^(-2i/d) in double, rotation in double, stored as float. */
int rkvo_apply_rope_rows(float* x, int64_t rows, int64_t num_heads, int64_t head_dim,
                         double base, const int64_t* positions, int inverse) {
    if (head_dim < 2 || head_dim % 2 != 0 || !(base > 1.0)) return -1;
    int64_t half = head_dim / 2, c = num_heads * head_dim;
    double* thetas = (double*)malloc(sizeof(double) * (size_t)half);
    if (!thetas) return -1;
    for (int64_t i = 0; i < half; ++i)
        thetas[i] = pow(base, -2.0 * (double)i / (double)head_dim);
    double dir = inverse ? -1.0 : 1.0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t h = 0; h < num_heads; ++h) {
            float* head = x + r * c + h * head_dim;
            for (int64_t i = 0; i < half; ++i) {
                double angle = dir * (double)positions[r] * thetas[i];
                double cs = cos(angle), sn = sin(angle);
                double a = head[i], b = head[i + half];
                head[i] = (float)(a * cs - b * sn);
                head[i + half] = (float)(a * sn + b * cs);
            }
        }
    free(thetas);
    return 0;
}

/* ------------------------------------------------------------------ quant */

/* proj/src/quant.cpp:25-35: LSB-first n-bit packing. */
void rkvo_pack_codes(const uint8_t* codes, int64_t n, int bits, uint8_t* out) {
    int64_t nbytes = (n * bits + 7) / 8;
    memset(out, 0, (size_t)nbytes);
    int64_t bitpos = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int b = 0; b < bits; ++b, ++bitpos)
            if (codes[i] & (1u << b)) out[bitpos >> 3] |= (uint8_t)(1u << (bitpos & 7));
}

/* proj/src/quant.cpp:37-51 */
void rkvo_unpack_codes(const uint8_t* packed, int64_t n, int bits, uint8_t* out) {
    int64_t bitpos = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint8_t c = 0;
        for (int b = 0; b < bits; ++b, ++bitpos)
            if (packed[bitpos >> 3] & (1u << (bitpos & 7))) c |= (uint8_t)(1u << b);
        out[i] = c;
    }
}

/* proj/src/quant.cpp:53-97 (clip ratios 0, the path's configuration):
 * min/max, raw scale (max-min)/qmax in double -> float, 1e-8 floor, stored
 * scale rounded UP (e4m3 as in the reference, or fp16 per SURVEY D1), zero =
 * clamp(round-half-away(-min/s)), code = clamp(round-half-away(x/s) + zero). */
int rkvo_quantize_group(const float* x, int64_t n, int bits, int scale_format, float* scale_out,
                        uint8_t* zero_out, uint8_t* codes_out, uint16_t* scale_code_out) {
    if (bits < 1 || bits > 8 || n < 1) return -1;
    float cmin = x[0], cmax = x[0];
    for (int64_t i = 1; i < n; ++i) {
        if (x[i] < cmin) cmin = x[i];
        if (x[i] > cmax) cmax = x[i];
    }
    const double qmax = (double)((1 << bits) - 1);
    float raw = (float)(((double)cmax - (double)cmin) / qmax);
    if (raw < 1e-8f) raw = 1e-8f;
    float sf;
    uint16_t code;
    if (scale_format == RKVO_SCALE_E4M3_CEIL) {
        code = rkvo_e4m3_encode_ceil(raw);
        sf = rkvo_e4m3_decode((uint8_t)code);
    } else {
        code = rkvo_fp16_ceil(raw);
        sf = rkvo_half_to_float(code);
    }
    const double s = (double)sf;
    double zero = round(-(double)cmin / s);
    if (zero < 0.0) zero = 0.0;
    if (zero > qmax) zero = qmax;
    for (int64_t i = 0; i < n; ++i) {
        double q = round((double)x[i] / s) + zero;
        if (q < 0.0) q = 0.0;
        if (q > qmax) q = qmax;
        codes_out[i] = (uint8_t)q;
    }
    if (scale_out) *scale_out = sf;
    if (zero_out) *zero_out = (uint8_t)zero;
    if (scale_code_out) *scale_code_out = code;
    return 0;
}

/* proj/src/quant.cpp:99-107 */
void rkvo_dequantize_group(const uint8_t* codes, int64_t n, float scale, uint8_t zero,
                           float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = scale * ((float)codes[i] - (float)zero);
}

/* quantize_token (proj/src/quant.cpp:109-119) of one row into the packed
 * word/meta layout; group 128, 2 bits. */
static void quantize_row_words(const float* row, int64_t c, int scale_format, uint32_t* codes,
                               uint32_t* meta) {
    uint8_t q[128];
    for (int64_t g = 0; g < c / 128; ++g) {
        float sf;
        uint8_t z;
        rkvo_quantize_group(row + g * 128, 128, 2, scale_format, &sf, &z, q, NULL);
        for (int w = 0; w < 8; ++w) {
            uint32_t word = 0;
            for (int i = 0; i < 16; ++i) word |= (uint32_t)q[w * 16 + i] << (2 * i);
            codes[g * 8 + w] = word;
        }
        /* both storage formats decode to a value exactly representable in fp16 */
        uint16_t sh = rkvo_float_to_half_rn(sf);
        uint16_t zh = rkvo_float_to_half_rn((float)z);
        meta[g] = (uint32_t)sh | ((uint32_t)zh << 16);
    }
}

static void dequant_row_words(const uint32_t* codes, const uint32_t* meta, int64_t c, float* out) {
    for (int64_t g = 0; g < c / 128; ++g) {
        float s = rkvo_half_to_float((uint16_t)(meta[g] & 0xffffu));
        float z = rkvo_half_to_float((uint16_t)(meta[g] >> 16));
        for (int64_t i = 0; i < 128; ++i) {
            uint32_t word = codes[(g * 128 + i) / 16];
            uint32_t code = (word >> (2 * ((g * 128 + i) % 16))) & 3u;
            out[g * 128 + i] = s * ((float)code - z);
        }
    }
}

/* The on-the-fly K/V transform chain, restated as compare_pipelines composes
 * it (proj/src/pipeline.cpp:317-324): K' = apply_reorder(rotate_rows(K, G)),
 * quantize_token(K'); V' = rotate_rows(V, g=1) (proj/src/pipeline.cpp:120),
 * quantize_token(V'). */
int rkvo_quantize_kv_rows(const uint16_t* k_raw, const uint16_t* v_raw, int64_t rows,
                          int64_t num_kv_heads, int64_t head_dim, int64_t heads_per_group,
                          const int32_t* perm, int scale_format, uint32_t* k_codes,
                          uint32_t* k_meta, uint32_t* v_codes, uint32_t* v_meta) {
    int64_t c = num_kv_heads * head_dim;
    if (c % 128 != 0 || !rotation_plan_ok(head_dim, heads_per_group, num_kv_heads)) return -1;
    float* a = (float*)malloc(sizeof(float) * (size_t)c);
    float* b = (float*)malloc(sizeof(float) * (size_t)c);
    if (!a || !b) { free(a); free(b); return -1; }
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t j = 0; j < c; ++j) a[j] = rkvo_half_to_float(k_raw[r * c + j]);
        rkvo_rotate_rows(a, 1, head_dim, heads_per_group, num_kv_heads);
        rkvo_apply_reorder(a, 1, c, perm, 0, b);
        quantize_row_words(b, c, scale_format, k_codes + r * (c / 16), k_meta + r * (c / 128));
        for (int64_t j = 0; j < c; ++j) a[j] = rkvo_half_to_float(v_raw[r * c + j]);
        rkvo_rotate_rows(a, 1, head_dim, 1, num_kv_heads);
        quantize_row_words(a, c, scale_format, v_codes + r * (c / 16), v_meta + r * (c / 128));
    }
    free(a);
    free(b);
    return 0;
}

/* proj/src/attention.cpp:9-18: float exp, double sum. */
static void softmax_inplace(float* row, int64_t n) {
    float m = row[0];
    for (int64_t i = 0; i < n; ++i) if (row[i] > m) m = row[i];
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        row[i] = expf(row[i] - m);
        sum += row[i];
    }
    for (int64_t i = 0; i < n; ++i) row[i] = (float)(row[i] / sum);
}

/* Decode attention for one sequence.
 *   reconstruct_cache (proj/src/pipeline.cpp:133-142): dequantize, inverse
 *     reorder, inverse grouped FWHT, RoPE at positions 0..T-1.  Sink tokens
 *     come from raw fp16 rows, which equals the reference's
 *     fused-frame sidecar row after its inverse transforms.
 *   prepare_queries (proj/src/pipeline.cpp:144-152): RoPE of the raw q at the
 *     query position (T-1: decode_step appends before attending,
 *     proj/src/pipeline.cpp:197-211).
 *   attention loop (proj/src/pipeline.cpp:243-261) with GQA kv head =
 *     h / (Hq/Hkv), V in its rotated frame; V's inverse rotation
 *     (absorbed into W_o_f, proj/src/pipeline.cpp:97) is applied to the
 *     per-head output. */
int rkvo_decode_attention(const uint32_t* k_codes, const uint32_t* k_meta,
                          const uint32_t* v_codes, const uint32_t* v_meta,
                          const uint8_t* is_sink, const uint16_t* sink_k,
                          const uint16_t* sink_v, int64_t T, const uint16_t* q,
                          int64_t num_q_heads, int64_t num_kv_heads, int64_t head_dim,
                          int64_t heads_per_group, const int32_t* perm, double rope_base,
                          float* out) {
    int64_t c = num_kv_heads * head_dim, d = head_dim;
    if (T < 1 || num_q_heads % num_kv_heads != 0 || c % 128 != 0) return -1;
    if (!rotation_plan_ok(head_dim, heads_per_group, num_kv_heads)) return -1;
    int64_t rep = num_q_heads / num_kv_heads;
    float* k = (float*)malloc(sizeof(float) * (size_t)(T * c));
    float* v = (float*)malloc(sizeof(float) * (size_t)(T * c));
    float* tmp = (float*)malloc(sizeof(float) * (size_t)c);
    float* qr = (float*)malloc(sizeof(float) * (size_t)(num_q_heads * d));
    float* logits = (float*)malloc(sizeof(float) * (size_t)T);
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
    if (!k || !v || !tmp || !qr || !logits || !pos) {
        free(k); free(v); free(tmp); free(qr); free(logits); free(pos);
        return -1;
    }
    for (int64_t t = 0; t < T; ++t) {
        float* kr = k + t * c;
        float* vr = v + t * c;
        if (is_sink && is_sink[t]) {
            for (int64_t j = 0; j < c; ++j) {
                kr[j] = rkvo_half_to_float(sink_k[t * c + j]);
                vr[j] = rkvo_half_to_float(sink_v[t * c + j]);
            }
            rkvo_rotate_rows(vr, 1, d, 1, num_kv_heads);
        } else {
            dequant_row_words(k_codes + t * (c / 16), k_meta + t * (c / 128), c, tmp);
            rkvo_apply_reorder(tmp, 1, c, perm, 1, kr);
            rkvo_rotate_rows(kr, 1, d, heads_per_group, num_kv_heads);
            dequant_row_words(v_codes + t * (c / 16), v_meta + t * (c / 128), c, vr);
        }
        pos[t] = t;
    }
    rkvo_apply_rope_rows(k, T, num_kv_heads, d, rope_base, pos, 0);
    for (int64_t j = 0; j < num_q_heads * d; ++j) qr[j] = rkvo_half_to_float(q[j]);
    int64_t qpos = T - 1;
    rkvo_apply_rope_rows(qr, 1, num_q_heads, d, rope_base, &qpos, 0);
    double inv_sqrt_d = 1.0 / sqrt((double)d);
    for (int64_t h = 0; h < num_q_heads; ++h) {
        int64_t kvh = h / rep;
        for (int64_t t = 0; t < T; ++t) {
            double dot = 0.0;
            for (int64_t i = 0; i < d; ++i)
                dot += (double)qr[h * d + i] * (double)k[t * c + kvh * d + i];
            logits[t] = (float)(dot * inv_sqrt_d);
        }
        softmax_inplace(logits, T);
        float* o = out + h * d;
        for (int64_t i = 0; i < d; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < T; ++t) acc += (double)logits[t] * (double)v[t * c + kvh * d + i];
            o[i] = (float)acc;
        }
        rkvo_fwht_inplace(o, d);
    }
    free(k); free(v); free(tmp); free(qr); free(logits); free(pos);
    return 0;
}

/* ------------------------------------------------------------------ sinks */

static int cmp_float(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/* proj/src/sink.cpp:14-45: median of |x| over the whole tensor by full sort;
 * a token is a sink iff some |x| exceeds rel*median and abs_floor; token 0
 * always is. */
int64_t rkvo_detect_sinks(const float* hidden, int64_t b, int64_t s, int64_t h,
                          double rel_threshold, double abs_floor, uint8_t* flags) {
    if (b < 1 || s < 1 || h < 1 || !(rel_threshold > 1.0)) return -1;
    int64_t n = b * s * h;
    float* mags = (float*)malloc(sizeof(float) * (size_t)n);
    if (!mags) return -1;
    for (int64_t i = 0; i < n; ++i) mags[i] = fabsf(hidden[i]);
    qsort(mags, (size_t)n, sizeof(float), cmp_float);
    double median = mags[n / 2];
    free(mags);
    double threshold = rel_threshold * median;
    int64_t count = 0;
    for (int64_t t = 0; t < s; ++t) {
        int hit = 0;
        for (int64_t bi = 0; bi < b && !hit; ++bi)
            for (int64_t ch = 0; ch < h; ++ch) {
                double v = fabsf(hidden[(bi * s + t) * h + ch]);
                if (v > threshold && v > abs_floor) { hit = 1; break; }
            }
        flags[t] = (uint8_t)(t == 0 || hit);
        count += flags[t];
    }
    return count;
}
