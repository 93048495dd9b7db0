// rkv_internal.h -- launch-side declarations shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <utility>
#include <cstdint>
#include <vector>

#include "rotatekv/rotatekv.h"

namespace rkv {

// Experiment switches (rkv_set_debug_option, rkv_runtime.cu).  Defaults are the
// production choices; the epoch bumps on every change so cached plans rebuild.
struct Options {
    std::atomic<int> force_simt{0};    // decode on the CUDA-core kernel for tensor-core shapes
    std::atomic<int> gqa_pw{1};        // GQA kernel: warps per FWHT group (1..4)
    std::atomic<int> gqa_tmem{1};      // GQA kernel: park accumulators in tensor memory
    std::atomic<int> dec_splits{0};    // > 0: force the split count per sequence
    std::atomic<int> prefill_pair{0};  // 2-SM (cta_group::2) prefill attention
    std::atomic<int> simt_p{0};        // CUDA-core kernel: token pairs per tile (0 = planner)
    std::atomic<int> simt_stages{0};   // CUDA-core kernel: TMA ring depth (0 = planner)
    std::atomic<int> quant_stages{1};  // quantize kernel: TMA stage buffers (1 or 2)
    std::atomic<int> quant_vsplit{1};  // quantize: V on the warp-independent kernel
    std::atomic<int> quant_vcfg{0};    // V kernel shape: 0 = 16 warps x 2 stages, shuffle stages; 1 = 16 x 1,
                                       // 2 = 14 x 1, 3 = 12 x 2 (row buffer); 4 = 20 x 2, shuffle stages
    std::atomic<int> decode_pdl{1};    // launch the MHA decode kernel with programmatic stream serialization
    std::atomic<int> generic_tile{0};  // generic decode: tokens per tile (0 = planner)
    std::atomic<int> gqa_sets{2};      // GQA kernel: 4-head sets sharing one key tile (1 or 2)
    std::atomic<int> epoch{0};
};
Options& options();
int current_device();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, high-water mark)
cudaError_t ensure_smem(const void* kern, size_t bytes);
// split count per sequence: fill every resident CTA slot, preferring a count
// whose CTA total is close to a whole number of waves
int choose_splits(int slots, int batch, int64_t max_split);
template <typename K>
inline cudaError_t ensure_smem_k(K* kern, size_t bytes) {
    return ensure_smem(reinterpret_cast<const void*>(kern), bytes);
}

constexpr float kLog2eHost = 1.4426950408889634f;

// Launch with programmatic stream serialization (the kernel's prologue may
// overlap the previous kernel's tail; it must pdl_wait() before reading that
// kernel's outputs).  Exact parameter types, like cudaLaunchKernelEx.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct QuantParams {
    const uint16_t* k_new;
    const uint16_t* v_new;
    const int32_t* perm;
    const uint8_t* sink_flags;
    const int64_t* start_pos;
    int64_t num_new;
    int64_t max_tokens;
    int C;
    int max_sinks;
    int scale_format;
    float k_norm;  // 1.0f / sqrtf(float(G*d))   (proj/src/hadamard.cpp:62)
    float v_norm;  // 1.0f / sqrtf(float(d))
    rkv_cache cache;
    int k_only;    // quantize_kv_kernel: K items only (V runs on quantize_v_kernel)
};

struct DecodeParams {
    const uint16_t* q;
    const int64_t* seq_len;    // [B] cache length; q sits at position seq_len - 1
    const int64_t* tok_begin;  // [B] or null: attend to cache tokens [tok_begin, tok_end) only
    const int64_t* tok_end;    //     (sequence-parallel partials; multiples of 64 apart from seq_len)
    float* partial_ml;         // non-null: the combine emits the merged partial (m, l) here and the
                               // unnormalised rotated o' in out, without sinks or H_128
    const uint32_t* plan;  // rkv_layer_plan_init (rkv_layout.h)
    const float4* rope;  // [max_pos/2][128]: section 1 (cos p0, cos p1, sin p0, sin p1) x 64, section 2
                         // two [32] frequency-pair rows (decode_attention.cu, kRopeRow)
    rkv_cache cache;
    float* ws_ml;  // [B][NP][Hq][2]   partial (m, l) per lane-group partition
    float* ws_o;   // [B][NP][Hq][128] partial o' (rotated V frame)
    float* out;    // [B][Hq][128]
    int64_t max_tokens;
    int B, Hq, Hkv, C;
    int S;      // splits (CTAs per sequence)
    int NP;     // partial rows per sequence = S * P
    int chunk;  // tokens per split, multiple of the tile
    int P;      // partial partitions per split (simt: token pairs per tile; mma: warps per FWHT group)
    int P_pairs;  // mma kernel: token pairs per tile
    int stages; // TMA ring depth
    int max_sinks;
    // GQA kernel passes (q heads per KV head a multiple of 4): this launch
    // covers q heads kv * q_rep + q_rep_off + 0..3 of every KV head kv
    int q_rep, q_rep_off;
    int f2_mask;   // GQA kernel: second FWHT factor's H mask (15: G = 2, 11: G = 1), hadamard_mask_frag
    float k_norm;  // 1/sqrt(G*d), folded into q
    float qscale;  // log2(e) / sqrt(d)
};

// prefill operand tiles (prefill.cu): 64 keys per tile, K hi + K lo + V^T
constexpr int kPrefillKT = 64;
constexpr int kPrefillMaxSinks = 16;  // sink rows staged per attention CTA
constexpr size_t kPrefillTileBytes = 3 * 16384;
inline int64_t prefill_q_pad(int64_t num_q) { return (num_q + 255) / 256 * 256; }  // 256 query rows per CTA pair
struct PrefillParams {
    const uint16_t* q;        // [B][num_q][Hq][128] fp16 pre-RoPE
    const int64_t* q_start;   // [B] position of query row 0
    const int64_t* seq_len;   // [B] cache length (keys [0, seq_len))
    const uint32_t* plan;     // layer plan (tensor-core layout)
    const float4* rope;       // rope table (decode_attention.cu layout)
    rkv_cache cache;
    // reconstructed operand tiles, [B][Hkv][kv_tiles] x 48 KB: per 64 keys the
    // keys' fp16 hi and lo planes (2 x 2 K-major SWIZZLE_128B slabs of 64 dims)
    // and the dequantized values transposed ([128 channels][64 keys], one slab)
    unsigned char* kv_tiles;
    int64_t kv_tiles_per_seq;
    // staged query rows, [B][Hq][num_q_pad] x 512 B: RoPE'd, x log2(e)/sqrt(d),
    // fp16 hi (64 words) + lo (64 words), 16-byte chunk c at c ^ (row & 31)
    unsigned char* q_rows;
    int64_t num_q_pad;
    float* out;               // [B][num_q][Hq][128]
    int64_t max_tokens, num_q;
    int B, Hq, Hkv, C, max_sinks;
    float k_norm, qscale;
};

// quantize_kv.cu
cudaError_t launch_quantize(const rkv_layer_desc& d, const QuantParams& p, cudaStream_t s);
// fused-frame append (rkv_quantize_kv_fused): K'/V' rows in `dtype` (rkv_rows_dtype)
cudaError_t launch_quantize_fused(const rkv_layer_desc& d, const QuantParams& p, const void* k_rows,
                                  const void* v_rows, int dtype, cudaStream_t s);
cudaError_t launch_fused_sink_rows(const rkv_layer_desc& d, const QuantParams& p, const void* k_rows,
                                   const void* v_rows, int dtype, cudaStream_t s);
cudaError_t launch_promote_sinks(const rkv_layer_desc& d, const QuantParams& p, const int64_t* tokens, int n,
                                 int32_t* promoted, cudaStream_t s);
int promote_sinks_max();
// decode_attention.cu
struct DecodePlan {
    int kind, N, REP, P, PP, TT, NT, S, NP, chunk, stages, per_sm;
    bool ok;
    size_t smem;
};
bool decode_supported(int N, int REP);
DecodePlan plan_decode(const rkv_layer_desc& d, int64_t max_seq_len);
const DecodePlan& cached_plan(const rkv_layer_desc& d, int64_t max_seq_len);  // memoised plan_decode
cudaError_t launch_decode(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p,
                          cudaStream_t s);
cudaError_t launch_decode_combine(const DecodeParams& p, int B, cudaStream_t s);
// decode_mma.cu (tensor-core FWHT kernel)
int decode_kind(const rkv_layer_desc& d);  // kDecodeSimt / kDecodeMma (rkv_layout.h)
bool decode_mma_supported(int G, int REP, int C);
int mma_layout_n(const rkv_layer_desc& d);  // channels per tensor-core FWHT tile: 512 (MHA) or 256 (GQA)
DecodePlan plan_decode_mma(const rkv_layer_desc& d, int64_t max_seq_len);
cudaError_t launch_decode_mma(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p,
                              cudaStream_t s);
cudaError_t launch_rope_table(const rkv_layer_desc& d, float4* table, int64_t max_pos, cudaStream_t s);
cudaError_t launch_rotate_keys(const rkv_layer_desc& d, const uint16_t* k, int64_t rows, float* out,
                               cudaStream_t s);
int num_sms();
cudaError_t launch_channel_stats(const float* rows_f32, int64_t rows, int64_t C, bool mean_abs, double* stats,
                                 cudaStream_t s);
// generic.cu (any power-of-two rotation size and head ratio)
bool generic_quantize_needed(const rkv_layer_desc& d);
cudaError_t launch_quantize_generic(const rkv_layer_desc& d, const QuantParams& p, cudaStream_t s);
size_t generic_decode_smem(const rkv_layer_desc& d, int tile_tokens = 1);
DecodePlan plan_decode_generic(const rkv_layer_desc& d, int64_t max_seq_len);
cudaError_t launch_decode_generic(const rkv_layer_desc& d, const DecodePlan& plan, const DecodeParams& p,
                                  cudaStream_t s);
bool simt_shape_ok(const rkv_layer_desc& d);
cudaError_t launch_rotate_keys_generic(const rkv_layer_desc& d, const uint16_t* k, int64_t rows, float* out,
                                       cudaStream_t s);
cudaError_t launch_cache_read(const rkv_layer_desc& d, const rkv_cache& cache, const int32_t* perm, int b, int64_t t0,
                              int64_t n, int frame, float* k_out, float* v_out, cudaStream_t s);
// prefill.cu
cudaError_t launch_prefill(const rkv_layer_desc& d, const PrefillParams& p, int64_t max_seq_len, cudaStream_t s);
// sink_detect.cu
size_t detect_sinks_workspace_bytes();
cudaError_t launch_detect_sinks(const float* x, int64_t b, int64_t s, int64_t hidden, double rel, double abs_floor,
                                uint8_t* flags, float* median_out, void* ws, cudaStream_t stream);
// rkv_plan.cu
bool build_decode_plan(const rkv_layer_desc& d, const int32_t* perm, std::vector<uint32_t>& out, int& cost);

}  // namespace rkv
