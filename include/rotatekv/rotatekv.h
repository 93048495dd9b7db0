/*
 * rotatekv.h -- C ABI of the B200-native RotateKV KV-cache hot path.
 *
 * A drop-in for the reference's C++ hot-path API (namespace rotatekv in
 * /root/reference/proj/include/rotatekv/).  Each entry point names the
 * reference interface it replaces.  Conventions:
 *   - plain pointers and sizes only; fp16 tensors are passed as uint16_t bits;
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - device pointers unless stated otherwise; the ABI never allocates in
 *     hot calls and is stream-ordered and re-entrant;
 *   - errors: the reference throws std::invalid_argument / std::out_of_range /
 *     std::runtime_error; here the same conditions return
 *     RKV_ERR_INVALID_ARGUMENT / RKV_ERR_OUT_OF_RANGE / RKV_ERR_RUNTIME, and
 *     rkv_last_error() holds the thread-local message.
 *
 * Layout of one layer's cache (all device memory, caller-owned, see
 * rkv_cache_bytes / rkv_cache_carve), C = num_kv_heads * head_dim, W = C/16:
 *   k_codes, v_codes  [B][max_tokens][W]        u32: 16 two-bit codes, code i of
 *                     the (reordered, rotated) row at bits 2*(i%16) of word
 *                     i/16 -- byte-identical to the reference's LSB-first
 *                     pack_codes (proj/src/quant.cpp:25-35)
 *   k_meta, v_meta    [B][max_tokens][C/128]    u32: fp16 scale | fp16 zero<<16
 *   sink_k, sink_v    [B][max_sinks][C]         fp16 raw (pre-rotation) rows
 *   sink_pos          [B][max_sinks]            i32 token position of each sink
 *   sink_count        [B]                       i32
 *   sink_mask         [B][ceil(max_tokens/32)]  u32 bit t%32 of word t/32 = sink
 * Every array starts 16-byte aligned and its allocation is a multiple of 16
 * bytes (rkv_cache_carve: 256): the decode kernels copy meta rows in 16-byte
 * aligned blocks, up to 12 bytes past a row when C is not a multiple of 512.
 */
#ifndef ROTATEKV_B200_H
#define ROTATEKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RKV_OK = 0,
    RKV_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    RKV_ERR_OUT_OF_RANGE = 2,     /* reference: std::out_of_range */
    RKV_ERR_RUNTIME = 3,          /* reference: std::runtime_error */
    RKV_ERR_CUDA = 4              /* CUDA launch / runtime failure */
} rkv_status;

typedef enum {
    RKV_SCALE_FP16_CEIL = 0, /* north star: fp16 scale, rounded up */
    RKV_SCALE_E4M3_CEIL = 1  /* reference storage (proj/src/quant.cpp:82): e4m3 ceil */
} rkv_scale_format;

typedef enum {
    RKV_STAT_SUM = 0,     /* reference: signed channel sum (proj/src/reorder.cpp:98-100) */
    RKV_STAT_MEAN_ABS = 1 /* north star: mean |K| */
} rkv_calib_stat;

/* One attention layer (replaces PipelineConfig + QuantConfig + RotationPlan,
 * proj/include/rotatekv/pipeline.hpp:50-64, quant.hpp:11-18, hadamard.hpp:8-16). */
typedef struct {
    int32_t batch;           /* sequences held by this cache (this rank's shard) */
    int32_t num_q_heads;     /* Hq */
    int32_t num_kv_heads;    /* Hkv; Hq % Hkv == 0 (GQA extension) */
    int32_t head_dim;        /* d: 128 */
    int32_t heads_per_group; /* G: K FWHT spans G KV heads (n = G*d, power of 2) */
    int32_t group_size;      /* quantization group: 128 */
    int32_t bits;            /* 2 */
    int32_t scale_format;    /* rkv_scale_format */
    int64_t max_tokens;      /* cache capacity per sequence */
    int32_t max_sinks;       /* sidecar capacity per sequence */
    int32_t reserved;        /* must be 0 */
    double rope_base;        /* RoPE theta (RopeConfig::base, rope.hpp:12) */
} rkv_layer_desc;

typedef struct {
    uint32_t* k_codes;
    uint32_t* v_codes;
    uint32_t* k_meta;
    uint32_t* v_meta;
    uint16_t* sink_k;
    uint16_t* sink_v;
    int32_t* sink_pos;
    int32_t* sink_count;
    uint32_t* sink_mask;
} rkv_cache;

/* Thread-local message of the last failing call on this thread. */
const char* rkv_last_error(void);
const char* rkv_version(void);

/* RotationPlan::make + QuantConfig::validate checks
 * (proj/src/hadamard.cpp:18-33, proj/src/quant.cpp:15-23) plus the
 * sm_100a kernels' shape limits.  Host only. */
rkv_status rkv_layer_validate(const rkv_layer_desc* desc);

/* Bytes of one layer's cache; carve a caller-allocated, 256-byte aligned
 * device buffer into the arrays above.  Host only. */
size_t rkv_cache_bytes(const rkv_layer_desc* desc);
rkv_status rkv_cache_carve(const rkv_layer_desc* desc, void* base, size_t bytes, rkv_cache* out);

/* Empty every sequence of the cache (LayerKVCache construction,
 * proj/include/rotatekv/kv_cache.hpp:17): sink counts and masks to zero. */
rkv_status rkv_cache_reset(const rkv_layer_desc* desc, const rkv_cache* cache, void* stream);

/* RoPE table [ceil(max_pos/2)][head_dim/2] float4: for the position pair
 * (2k, 2k+1) and frequency i, (cos 2k*th_i, cos (2k+1)*th_i, sin 2k*th_i,
 * sin (2k+1)*th_i) with th_i = base^(-2i/d) evaluated in double like
 * proj/src/rope.cpp:17-24.  Read by rkv_decode_attention; build once per
 * (rope_base, max_pos). */
size_t rkv_rope_table_bytes(const rkv_layer_desc* desc, int64_t max_pos);
rkv_status rkv_rope_table_init(const rkv_layer_desc* desc, float* table, int64_t max_pos, void* stream);

/* Fused quantize-append (replaces rotate_rows -> apply_reorder ->
 * quantize_token -> LayerKVCache::append, proj/src/hadamard.cpp:75-84,
 * proj/src/reorder.cpp:112-128, proj/src/quant.cpp:109-119,
 * proj/src/kv_cache.cpp:8-22, as composed at proj/src/pipeline.cpp:171-176).
 *   k_new, v_new : [B][num_new][C] fp16, pre-RoPE, unrotated
 *   perm         : [C] int32, slot j <- channel perm[j] (ReorderPlan::perm[layer])
 *   sink_flags   : [B][num_new] u8 (1 = keep the token in the fp16 sidecar), or NULL
 *   start_pos    : [B] int64, cache index of each sequence's first new token
 * k_new, v_new and perm must be 16-byte aligned (TMA / vector loads).
 * Tokens are written at start_pos[b] .. start_pos[b]+num_new-1.  The device
 * cannot throw: callers (the C++ layer) validate capacities first. */
rkv_status rkv_quantize_kv(const rkv_layer_desc* desc, const uint16_t* k_new, const uint16_t* v_new,
                           const int32_t* perm, const uint8_t* sink_flags, const int64_t* start_pos,
                           int64_t num_new, const rkv_cache* cache, void* stream);

/* Fused-frame append (the reference's own deployment frame).
 * With fuse_weights (proj/src/pipeline.cpp:88-99) the projections already
 * emit K' = P H_G k (rotated + reordered, pre-RoPE) and V' = H_128 v, and
 * LayerKVCache::append (proj/src/kv_cache.cpp:8-22; called at
 * proj/src/pipeline.cpp:171-176, 207-209) only quantizes them -- this call.
 *   k_rows, v_rows : [B][num_new][C] fused-frame rows, 16-byte aligned, in
 *                    `dtype`: RKV_ROWS_F32 (what append receives) or RKV_ROWS_F16
 *   perm           : [C] int32 (only the sink rows use it, see below)
 * Other arguments, errors and the device-side rules as rkv_quantize_kv.  The
 * packed words and metadata equal rkv_quantize_kv's for raw rows whose fp32
 * rotated + reordered image is k_rows / v_rows (the same quantizer).  Sink
 * tokens: the sidecar keeps model-frame fp16 rows, so K' / V' go back
 * through the inverse reorder and FWHT and are rounded to fp16. */
typedef enum { RKV_ROWS_F32 = 0, RKV_ROWS_F16 = 1 } rkv_rows_dtype;
rkv_status rkv_quantize_kv_fused(const rkv_layer_desc* desc, const void* k_rows, const void* v_rows, int32_t dtype,
                                 const int32_t* perm, const uint8_t* sink_flags, const int64_t* start_pos,
                                 int64_t num_new, const rkv_cache* cache, void* stream);

/* promote_to_sink / route_sinks (proj/src/kv_cache.cpp:43-55,
 * proj/src/sink.cpp:47-63): move already-appended tokens into the fp16
 * sidecar.
 *   tokens   : [B][num_tokens] int64, device: token index per sequence (-1 = no entry)
 *   k_rows, v_rows : [B][num_tokens][C] fp16, device: the raw (pre-rotation,
 *              pre-RoPE) K/V rows of those tokens -- what append's sink path stores
 *   promoted : [B] int32 device (tokens newly promoted per sequence) or NULL
 * Per sequence, tokens are taken in list order: indices outside
 * [0, max_tokens) and tokens that are already sinks are skipped (the
 * reference returns early for sinks: idempotent, duplicates included), and a
 * full sidecar (max_sinks) leaves the rest quantized.  A promoted token gets
 * the next sidecar slot, its sink-mask bit and sink_pos, and its packed
 * words and metadata are zeroed.  The caller checks token < cache length
 * (the reference's std::out_of_range; the device cannot throw).
 * num_tokens <= 256.  Stream-ordered, graph-capturable. */
rkv_status rkv_promote_sinks(const rkv_layer_desc* desc, const rkv_cache* cache, const int64_t* tokens,
                             int64_t num_tokens, const uint16_t* k_rows, const uint16_t* v_rows, int32_t* promoted,
                             void* stream);

/* LayerKVCache::key_row / value_row / keys / values (proj/src/kv_cache.cpp:
 * 57-85), for tokens [t0, t0 + num_tokens) of sequence seq:
 *   k_out, v_out : [num_tokens][C] fp32, device
 *   frame        : RKV_FRAME_STORED -- what the reference returns: the stored
 *                  fused-frame row s*(c - z) (K reordered + rotated, V rotated;
 *                  sinks: the fused frame of the exact fp16 row, i.e. the
 *                  reference's fp32 sidecar content);
 *                  RKV_FRAME_RAW -- the same rows back in the model's frame
 *                  (reorder and rotation undone; sinks exact)
 *   perm         : [C] int32, device (the layer's reorder)
 * Out-of-range tokens: RKV_ERR_OUT_OF_RANGE (the reference's
 * std::out_of_range).  Debug / cross-check path, stream-ordered. */
typedef enum { RKV_FRAME_STORED = 0, RKV_FRAME_RAW = 1 } rkv_row_frame;
rkv_status rkv_cache_read(const rkv_layer_desc* desc, const rkv_cache* cache, const int32_t* perm, int64_t seq,
                          int64_t t0, int64_t num_tokens, int32_t frame, float* k_out, float* v_out, void* stream);

/* Experiment switches (process-global; defaults are the production
 * choices): "decode_kernel_simt" (1 = decode tensor-core shapes on the
 * CUDA-core kernel), "gqa_warps_per_group" (1..4, default 1), "gqa_tmem" (0/1),
 * "gqa_head_sets" (1 or 2, default 2: 8 q heads per KV head share a key tile),
 * "decode_splits" (> 0 forces the split count), "prefill_pair" (1 = 2-SM
 * prefill attention), "simt_pairs", "simt_stages".  The kernel selection is
 * recorded in layer plans and RoPE tables: build them after setting a switch
 * (a decode with a plan of another kernel kind returns NaN). */
rkv_status rkv_set_debug_option(const char* name, int64_t value);

/* Diagnostic: the decode plan rkv_decode_attention uses for (desc,
 * max_seq_len) on the current device -- out[0..9] = kernel kind (0 CUDA-core,
 * 1 tensor-core, 2 generic), channels per FWHT tile, threads per CTA, splits
 * per sequence, partial rows per sequence, tokens per split, tokens per
 * tile, resident CTAs per SM, shared-memory bytes per CTA, TMA stages. */
rkv_status rkv_decode_plan_info(const rkv_layer_desc* desc, int64_t max_seq_len, int64_t out[10]);

/* Per-layer decode plan (once per layer, after calibration): from the HOST
 * permutation perm [C] (slot j <- channel perm[j]) choose which packed word
 * each decode thread un-reorders so the shared-memory scatter's bank
 * conflicts are minimal, and upload word indices + scatter offsets to
 * `plan_dev` (>= rkv_layer_plan_bytes).  rkv_layer_plan_build writes the same
 * words to host memory and reports the schedule cost (sum over half-warps and
 * rounds of the worst bank-slot multiplicity; 16 per half-warp is ideal). */
size_t rkv_layer_plan_bytes(const rkv_layer_desc* desc);
rkv_status rkv_layer_plan_build(const rkv_layer_desc* desc, const int32_t* perm, uint32_t* plan_host,
                                size_t bytes, int32_t* cost_out);
rkv_status rkv_layer_plan_init(const rkv_layer_desc* desc, const int32_t* perm, void* plan_dev, size_t bytes,
                               void* stream);

/* Split-K decode attention over the 2-bit cache (replaces the attention half
 * of decode_step: reconstruct_cache + prepare_queries + the per-head loop,
 * proj/src/pipeline.cpp:133-152,211-261).
 *   q        : [B][Hq][d] fp16, pre-RoPE; query position = seq_len[b]-1
 *              (decode_step appends the token before attending, pipeline.cpp:197-211)
 *   seq_len  : [B] int64 device, tokens 0..seq_len[b]-1 are attended (>= 1)
 *   max_seq_len : host upper bound of seq_len (0 = desc->max_tokens)
 *   layer_plan : from rkv_layer_plan_init for the layer's permutation
 *              (un-reordering scatters slot j back to channel perm[j])
 *   rope_table : from rkv_rope_table_init with max_pos >= max_seq_len
 *   out      : [B][Hq][d] fp32, V's rotation undone (what W_o_f absorbs, pipeline.cpp:97)
 *   workspace: >= rkv_decode_workspace_bytes(desc, max_seq_len) bytes of device memory */
size_t rkv_decode_workspace_bytes(const rkv_layer_desc* desc, int64_t max_seq_len);
rkv_status rkv_decode_attention(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len,
                                int64_t max_seq_len, const rkv_cache* cache, const void* layer_plan,
                                const float* rope_table, float* out, void* workspace, size_t ws_bytes,
                                void* stream);

/* Sequence-parallel decode (batch < GPUs, split-K across ranks
 * plus one small all-gather).  A rank attends to the quantized cache tokens
 * [tok_begin[b], tok_end[b]) of every sequence (device [B] int64; tok_begin a
 * multiple of 64, tok_end a multiple of 64 or >= seq_len; sink tokens are
 * skipped) with q at position seq_len[b] - 1, and emits one unnormalised
 * partial per (b, h):
 *   part_ml : [B][Hq][2] fp32 (running max in log2 units, sum of weights)
 *   part_o  : [B][Hq][d] fp32 (rotated V frame)
 *   max_span: host bound of tok_end - tok_begin (sizes the split plan)
 *   workspace: rkv_decode_workspace_bytes(desc, max_span) bytes
 * rkv_decode_merge then folds num_parts gathered partials, laid out
 * [B][num_parts][Hq][2] and [B][num_parts][Hq][d], with the exact sink rows
 * and V's inverse rotation into out [B][Hq][d] -- the same combine the
 * single-GPU decode runs over its splits.  Stream-ordered. */
rkv_status rkv_decode_attention_partial(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len,
                                        const int64_t* tok_begin, const int64_t* tok_end, int64_t max_span,
                                        const rkv_cache* cache, const void* layer_plan, const float* rope_table,
                                        float* part_ml, float* part_o, void* workspace, size_t workspace_bytes,
                                        void* stream);
rkv_status rkv_decode_merge(const rkv_layer_desc* desc, const uint16_t* q, const int64_t* seq_len, int32_t num_parts,
                            const float* parts_ml, const float* parts_o, const rkv_cache* cache,
                            const float* rope_table, float* out, void* stream);

/* Causal attention of a block of queries over the cache (the
 * attention half of prefill, proj/src/pipeline.cpp:156-191 -- reconstruct_cache
 * then causal reference_attention, proj/src/attention.cpp:20-49):
 *   q          : [B][num_q][Hq][d] fp16 pre-RoPE; row i of sequence b sits at
 *                position q_start[b] + i and attends to cache tokens
 *                0 .. q_start[b] + i (and < seq_len[b])
 *   q_start, seq_len : [B] int64, device
 *   max_seq_len: host upper bound of seq_len (sizes the key reconstruction)
 *   out        : [B][num_q][Hq][d] fp32, V's rotation undone (like decode)
 *   workspace  : rkv_prefill_workspace_bytes(desc, num_q, max_seq_len) bytes
 * Keys (tensor-core FWHT + RoPE, fp16 hi/lo) and values (dequantized fp16)
 * are reconstructed once into 64-key operand tiles, the queries are staged,
 * then a flash-attention kernel runs Q.K^T and P.V on tcgen05 (accumulators
 * in tensor memory); sinks are merged exactly in its epilogue (max_sinks
 * <= 16, else RKV_ERR_INVALID_ARGUMENT).  Layer shapes:
 * those with a tensor-core decode kernel (G = 1, 2 or 4 with Hq == Hkv; G = 2
 * or 4 with Hq == 4 Hkv, Hkv <= 8).  Stream-ordered. */
size_t rkv_prefill_workspace_bytes(const rkv_layer_desc* desc, int64_t num_q, int64_t max_seq_len);
rkv_status rkv_prefill_attention(const rkv_layer_desc* desc, const uint16_t* q, int64_t num_q, const int64_t* q_start,
                                 const int64_t* seq_len, int64_t max_seq_len, const rkv_cache* cache,
                                 const void* layer_plan, const float* rope_table, float* out, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* Grouped-head FWHT of raw fp16 K rows into fp32 (rotate_rows,
 * proj/src/hadamard.cpp:75-84) -- the device half of calibration. */
rkv_status rkv_rotate_keys(const rkv_layer_desc* desc, const uint16_t* k, int64_t rows, float* out,
                           void* stream);

/* calibrate_reorder (proj/src/reorder.cpp:91-110) on HOST memory:
 * rotated_keys [rows][channels] fp32 -> perm/inverse [channels] int32. */
rkv_status rkv_calibrate_reorder(const float* rotated_keys, int64_t rows, int64_t channels, int32_t stat,
                                 int32_t* perm_out, int32_t* inverse_out);

/* calibrate_reorder from raw fp16 pre-RoPE keys on DEVICE memory (SURVEY
 * 8(f) 2; proj/src/pipeline.cpp:101-109 rotate_rows -> proj/src/reorder.cpp:
 * 91-110 calibrate_reorder):
 *   k_rows     : [rows][C] fp16, device (pre-RoPE K of the calibration set)
 *   stat       : RKV_STAT_SUM (reference) or RKV_STAT_MEAN_ABS (north star)
 *   workspace  : rkv_calibrate_workspace_bytes(desc, rows) bytes of device memory
 *   perm_out   : [C] int32, HOST (slot j <- channel perm[j]); inverse_out: [C] or NULL
 * The rows are rotated on the device (bit-identical to rotate_rows) and each
 * channel's statistic is accumulated in double over the rows IN ORDER, the
 * reference's summation order, so the statistics and the stable argsort (host)
 * are bit-identical to rkv_calibrate_reorder on the rotated rows.  Synchronizes
 * the stream (the permutation is returned on the host). */
size_t rkv_calibrate_workspace_bytes(const rkv_layer_desc* desc, int64_t rows);
rkv_status rkv_calibrate_reorder_device(const rkv_layer_desc* desc, const uint16_t* k_rows, int64_t rows,
                                        int32_t stat, void* workspace, size_t workspace_bytes, int32_t* perm_out,
                                        int32_t* inverse_out, void* stream);

/* Cache wire format: LayerKVCache::serialize /
 * deserialize (proj/src/kv_cache.cpp:119-173, blocks proj/src/quant.cpp:
 * 139-158): u8 bits, u64 group, u64 channels, u64 tokens (little endian), then
 * per token a sink byte and either two fp32 rows (K then V, the fused frame:
 * K' = reorder(rotate_G(k)), V' = rotate_1(v), what the reference's sidecar
 * holds) or the K blocks then the V blocks, each [e4m3 scale][u8 zero][codes
 * LSB-first].  RKV_WIRE_REFERENCE is that format byte for byte (needs
 * scale_format == RKV_SCALE_E4M3_CEIL, or fp16 scales that are e4m3 values);
 * RKV_WIRE_FP16_SCALE is the same layout with a 2-byte fp16 scale per block,
 * the sink rows as the raw fp16 rows the sidecar holds (2 x C x 2 bytes) and
 * bits | 0x80 in the header: lossless for every cache.  Importing the
 * reference format turns the fused-frame fp32 sink rows back into the raw
 * frame (inverse reorder + FWHT) and rounds them to fp16.
 * Both calls move ONE sequence (index seq) between device cache and host
 * bytes and synchronize the stream.  perm: [C] int32 host (the layer's
 * reorder, for the sink rows' frame).  Import replaces the sequence. */
typedef enum { RKV_WIRE_REFERENCE = 0, RKV_WIRE_FP16_SCALE = 1 } rkv_wire_format;
size_t rkv_cache_wire_bytes(const rkv_layer_desc* desc, int64_t tokens, int64_t num_sinks, int32_t format);
rkv_status rkv_cache_export(const rkv_layer_desc* desc, const rkv_cache* cache, int64_t seq, int64_t tokens,
                            const int32_t* perm, int32_t format, uint8_t* out, size_t out_bytes, size_t* written,
                            void* stream);
rkv_status rkv_cache_import(const rkv_layer_desc* desc, const uint8_t* bytes, size_t num_bytes, const int32_t* perm,
                            int64_t seq, const rkv_cache* cache, int64_t* tokens_out, void* stream);

/* Massive-activation sink detection (proj/src/sink.cpp:14-45) on HOST memory:
 * hidden [b][s][h] fp32 -> flags[s] (token 0 always flagged).  Returns the
 * count through *num_sinks. */
rkv_status rkv_detect_sinks(const float* hidden, int64_t b, int64_t s, int64_t h, double rel_threshold,
                            double abs_floor, uint8_t* flags, int64_t* num_sinks);

/* The same detection on DEVICE memory (no host round trip):
 *   hidden     : [b][s][h] fp32, device
 *   flags      : [s] u8, device (1 = sink; token 0 always), ready for
 *                rkv_quantize_kv's sink_flags once broadcast over the batch
 *   median_out : device float (the median of |hidden|), or NULL
 *   workspace  : rkv_detect_sinks_workspace_bytes() bytes of device memory
 * Exact: the median is a radix select on the magnitude bits, the threshold
 * compare is done in fp32 against RD(rel * median) (== the reference's
 * double compare for float inputs).  Stream-ordered, graph-capturable. */
size_t rkv_detect_sinks_workspace_bytes(void);
rkv_status rkv_detect_sinks_device(const float* hidden, int64_t b, int64_t s, int64_t h, double rel_threshold,
                                   double abs_floor, uint8_t* flags, float* median_out, void* workspace,
                                   size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ROTATEKV_B200_H */
