/*
 * rkv_oracle.h -- CPU restatement of the RotateKV KV-cache hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA path in paper_2501_16383_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  The product path never
 * links it and never falls back to it.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Pinning: tests/test_oracle_kat.py checks this
 * restatement against the reference's own known-answer tests, and
 * tests/test_oracle_vs_ref.py / tests/test_golden.py check it against the
 * unmodified reference library compiled by oracle/Makefile (oracle/_ref).
 *
 * Cache layout (identical to the GPU layout, one sequence):
 *   codes[t][C/16]   u32, 16 two-bit codes per word, code i of the row at
 *                    bits 2*(i%16) of word i/16 (== LSB-first byte packing of
 *                    proj/src/quant.cpp:25-35 read as little-endian u32)
 *   meta [t][C/128]  u32 = fp16 scale in bits 0..15, fp16 zero in bits 16..31
 */
#ifndef RKV_ORACLE_H
#define RKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RKVO_SCALE_FP16_CEIL = 0, RKVO_SCALE_E4M3_CEIL = 1 };
enum { RKVO_STAT_SUM = 0, RKVO_STAT_MEAN_ABS = 1 };

/* fp16 / e4m3 codecs */
float rkvo_half_to_float(uint16_t h);
uint16_t rkvo_float_to_half_rn(float f);
uint16_t rkvo_fp16_ceil(float x);
float rkvo_e4m3_decode(uint8_t code);
uint8_t rkvo_e4m3_encode(float x);
uint8_t rkvo_e4m3_encode_ceil(float x);

/* transforms */
int rkvo_fwht_inplace(float* v, int64_t n);
int rkvo_rotate_rows(float* x, int64_t rows, int64_t head_dim, int64_t heads_per_group,
                     int64_t num_heads);
int rkvo_apply_reorder(const float* x, int64_t rows, int64_t channels, const int32_t* perm,
                       int inverse, float* out);
int rkvo_invert_perm(const int32_t* perm, int64_t channels, int32_t* inverse);
int rkvo_calibrate_reorder(const float* rows, int64_t n_rows, int64_t channels, int stat,
                           int32_t* perm_out, int32_t* inverse_out);
int rkvo_apply_rope_rows(float* x, int64_t rows, int64_t num_heads, int64_t head_dim,
                         double base, const int64_t* positions, int inverse);

/* quantization */
void rkvo_pack_codes(const uint8_t* codes, int64_t n, int bits, uint8_t* out);
void rkvo_unpack_codes(const uint8_t* packed, int64_t n, int bits, uint8_t* out);
/* Returns 0 on success.  scale_out = decoded stored scale, zero_out = zero point,
 * codes_out = unpacked codes, scale_code_out = storage bits (fp16 or e4m3). */
int rkvo_quantize_group(const float* x, int64_t n, int bits, int scale_format, float* scale_out,
                        uint8_t* zero_out, uint8_t* codes_out, uint16_t* scale_code_out);
void rkvo_dequantize_group(const uint8_t* codes, int64_t n, float scale, uint8_t zero,
                           float* out);

/* The composed north-star chain for rows of one layer.
 * k_raw/v_raw: [rows][C] fp16 bits, pre-RoPE.  perm: [C] slot j <- channel perm[j].
 * Writes codes [rows][C/16] and meta [rows][C/128] for K and V (2-bit, group 128). */
int rkvo_quantize_kv_rows(const uint16_t* k_raw, const uint16_t* v_raw, int64_t rows,
                          int64_t num_kv_heads, int64_t head_dim, int64_t heads_per_group,
                          const int32_t* perm, int scale_format, uint32_t* k_codes,
                          uint32_t* k_meta, uint32_t* v_codes, uint32_t* v_meta);

/* Decode attention for one sequence over T cached tokens (restates
 * proj/src/pipeline.cpp:133-152,243-261 with GQA).
 *   is_sink[T]: 1 -> the token's K/V come from sink_k/sink_v (raw fp16 rows,
 *                  [T][C] indexed by token) instead of the packed cache.
 *   q: [Hq][d] fp16 pre-RoPE; query position = T-1.
 *   out: [Hq][d] fp32, V rotation undone. */
int rkvo_decode_attention(const uint32_t* k_codes, const uint32_t* k_meta,
                          const uint32_t* v_codes, const uint32_t* v_meta,
                          const uint8_t* is_sink, const uint16_t* sink_k,
                          const uint16_t* sink_v, int64_t T, const uint16_t* q,
                          int64_t num_q_heads, int64_t num_kv_heads, int64_t head_dim,
                          int64_t heads_per_group, const int32_t* perm, double rope_base,
                          float* out);

/* Massive-activation sink detection (proj/src/sink.cpp:14-45).  hidden: [b][s][h]
 * fp32.  Writes flags[s] (1 = sink).  Returns number of sink tokens or <0. */
int64_t rkvo_detect_sinks(const float* hidden, int64_t b, int64_t s, int64_t h,
                          double rel_threshold, double abs_floor, uint8_t* flags);

#ifdef __cplusplus
}
#endif

#endif
