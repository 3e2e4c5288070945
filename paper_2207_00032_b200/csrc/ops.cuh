// Non-GEMM device operators of the decode step and the weight-initialisation kernels.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace dsinf {
namespace ops {

// Logical (un-sharded) position of a local weight element under Megatron TP sharding.
//   global row = (n / sec_local) * sec_global + row_off + n % sec_local
//   global col = col_off + k;  flat = row * K_global + col
constexpr int kI8Group = 128;  // INT8 K-group size (128 consecutive k share an fp16 scale)

struct ShardMap {
  int64_t N_local, K_local;
  int64_t N_global, K_global;
  int64_t sec_local, sec_global, row_off, col_off;
  int64_t valid_rows;  // global rows >= valid_rows are zero padding (vocab)
  uint64_t base;       // synth_base(seed, layer, tensor)
  float amp;
};

// Synthetic weight tensor written in the reference packed layout, fp16, pack_M = 2.
void init_packed_f16(const ShardMap& m, uint32_t* packed, cudaStream_t s);
// Same tensor quantised per global output row to int8 (pack_M = 4) + fp32 row scales.
// biased: bytes stored as s + 128 (XOR 0x80), the W8A16 decode GEMMs' layout (no XOR when widening)
void init_packed_i8(const ShardMap& m, uint32_t* packed, float* scales, cudaStream_t s, bool biased = false);
// Same tensor quantised per (global row, 128-k group): fp16 scales [K_local/128][N_local].
void init_packed_i8_groups(const ShardMap& m, uint32_t* packed, __half* gscales, cudaStream_t s, bool biased = false);
// Row-major [N_local][K_local] copy of the same tensor for the tensor-core path: fp16, or int8
// quantised with the given (packed-layout) row scales.
void init_rowmajor_map_f16(const ShardMap& m, __half* out, cudaStream_t s);
// Packed decode weights -> the row-major [N][K] operand of the tensor-core prefill: both layouts
// are 32-bit words (pack_M consecutive k of one output row), so this is the word transpose
// [rows][N] -> [N][rows] (rows = K / pack_M, K % pack_M == 0), smem-tiled, coalesced both ways.
// xor_mask 0x80808080 un-biases W8A16-biased int8 words.
void packed_to_rowmajor(const uint32_t* packed, int64_t rows, int64_t N, uint32_t* out, cudaStream_t s,
                        uint32_t xor_mask = 0);
void init_rowmajor_map_i8(const ShardMap& m, const float* scales, int8_t* out, cudaStream_t s);
// 1-D tensor (bias / LN) of length n_local: value = offset + unit(flat = row(n)) * amp.
void init_vector_f16(const ShardMap& m, float offset, __half* out, cudaStream_t s);
// Row-major fp16 [rows][cols] (replicated embedding table).
void init_rowmajor_f16(uint64_t base, float amp, int64_t rows, int64_t cols, __half* out, cudaStream_t s);

// pack_weights on device (gemm.hpp:113-130): row-major [N][K] -> [ceil(K/M)][N][M] fp16.
void pack_f16(const void* w, bool src_f32, int64_t N, int64_t K, int pack_M, __half* out, cudaStream_t s);
// Per-row int8 quantisation of a row-major fp16 matrix into the packed M=4 layout.
void quantize_weights_i8(const __half* w, int64_t N, int64_t K, int8_t* packed, float* scales, cudaStream_t s);
// K-group scales (kI8Group = 128 consecutive k per row share an fp16 scale; gscales [ceil(K/128)][N]),
// packed like quantize_weights_i8; the W8A16 GEMM dequantises w = fp16(q * s) per group.
void quantize_weights_i8_groups(const __half* w, int64_t N, int64_t K, int8_t* packed, __half* gscales,
                                cudaStream_t s);
// Per-token int8 quantisation of activations [B][K] (same formula as the GEMM prologue).
void quantize_act_i8(const __half* x, int64_t B, int64_t K, int8_t* q, float* scales, cudaStream_t s);

// Decode attention (paper region 2): split over ctx chunks inside a cluster of `chunks` CTAs.
struct AttnParams {
  const __half* q;        // [B][H*d]
  const __half* kc;       // [B][H][max_seq][d]
  const __half* vc;
  const int* pos;         // attend to positions 0..*pos
  __half* out;            // [B][H*d]
  int B, H, d, max_seq;
  float scale;
  unsigned* amax_out;         // row max |out| stripes for the int8 attn-out prologue, or null
  unsigned long long* trace;  // launch timeline slot or null
  // > 0: K/V rows of the earlier positions of a CTA's chunk (at most kv_rows_cap) are copied into
  // shared memory BEFORE the dependency wait (they were written by earlier steps); only q and the
  // new position's K/V row are read after it.  Set by ops::attention.
  int kv_rows_cap;
  int tma_ring;  // bulk-copy variant: K/V ring slots (set by ops::attention)
  int early_kv;  // bulk-copy variant: stages of earlier positions requested before the dependency wait
  int late_trigger;  // bulk-copy variant: release dependents after the dependency wait, not at kernel start
};
int attention_chunks(int B, int H);
// Sets kernel attributes (dynamic smem, non-portable clusters); call before graph capture.
void configure();
bool carveout_max();            // DSINF_CARVEOUT=0 leaves the driver's default L1/shared split
void configure_step_kernels();  // called by configure()
void attention(const AttnParams& p, int chunks, cudaStream_t s, bool pdl);

// Row preparation for the x-streaming GEMM plan (large batch): one CTA per batch row writes the
// GEMM-ready x of the next SBI-GeMM.
enum PrepMode : int {
  PREP_LN_F16 = 0,    // out fp16 = LayerNorm(res) with the producer's row sums
  PREP_LN_I8 = 1,     // out int8 = quantise(fp16 LayerNorm(res)), scale = row max / 127
  PREP_QUANT_I8 = 2,  // out int8 = quantise(x fp16), scale from the producer's row max (amax), or
                      // from the row itself when amax is null
};
struct PrepParams {
  int mode;
  const float* res;            // LN: residual [B][K] fp32
  const float* res_delta;      // LN, optional: residual = res + (res_delta + delta_bias) ...
  const __half* delta_bias;
  int delta_slots;             // fused all-reduce: res_delta = rank-order sum of this many partials
  long long delta_stride;      //   `delta_stride` floats apart, readable once red_flag reaches
  const unsigned long long* red_flag;  //   (*step_ctr + 1) * red_per_step
  const long long* step_ctr;
  unsigned long long red_per_step;
  float* res_out;              // ... stored here (this kernel is the row's only writer)
  const long long* ln_stats;   // LN: fixed-point row sums (gemm::kLnSlotWords layout), or null:
                               // computed here with the same fixed-point scheme
  const __half* ln_g;
  const __half* ln_b;
  float eps;
  double inv_k;  // 1 / K (set by row_prep)
  const __half* x;             // QUANT: fp16 [B][x_ld]
  int x_ld;
  const unsigned* amax;        // QUANT: row max stripes (gemm::kAmaxSlotWords layout)
  void* out;                   // [B][K] fp16 or int8 (row stride K)
  float* out_scale;            // int8: [B]
  int B, K;
  unsigned long long* trace;
  int split;  // CTAs (cluster) per row: 0 = the measured in-model rule, else 1, 2, 4 or 8
};
void row_prep(const PrepParams& p, cudaStream_t s, bool pdl);

// Step-boundary kernels.
struct EmbedParams {
  const __half* wte;      // [V][h]
  const int32_t* prompt;  // [B][prompt_ld]
  int prompt_len, prompt_ld;
  const int32_t* next_tok;  // [B]
  const int* pos;
  int32_t* hist;          // [B][max_ctx]
  int max_ctx;
  float* res;             // [B][h]
  int B, h, V;
  long long* ln_stats_out;  // fixed-point row sums of res for the first LayerNorm, or null
  unsigned long long* trace;
};
void embed(const EmbedParams& p, cudaStream_t s, bool pdl);

struct ArgmaxParams {
  const float* logits;  // [B][ld]
  int ld, valid, B;
  int64_t idx_offset;   // global vocab index of local column 0
  float* out_val;       // [B]
  int32_t* out_idx;     // [B]
  unsigned long long* trace;
};
void argmax(const ArgmaxParams& p, cudaStream_t s, bool pdl);

struct SelectParams {
  long long* step_ctr;   // optional: decode-step counter (+1 per step; fused all-reduce flags)
  const float* vals;     // [shards][B] (row stride B)
  const int32_t* idxs;   // [shards][B]
  const unsigned long long* keys;  // or: packed (logit, index) keys [shards][B] (gemm::argmax_key)
  int shards, B;
  int32_t* next_tok;
  int* pos;
  int32_t* hist;
  int max_ctx;
  // DSINF_TP_IPC: this rank's keys ([rank][B] of `keys`) are first stored into every peer's key
  // array over CUDA-IPC / NVLink and each peer's arrival counter bumped (system scope); the kernel
  // then waits until its own counter shows the other t - 1 ranks' keys of this step.
  int ipc_t = 0, ipc_rank = 0;
  unsigned long long* ipc_keys[8] = {};  // every rank's key array [t][B] (index ipc_rank: ours)
  unsigned long long* ipc_flag[8] = {};  // every rank's arrival counter
};
void select_token(const SelectParams& p, cudaStream_t s, bool pdl);

// ---- prompt prefill (large-batch regime): M = B * P rows, row m = token (m % P) of sequence m / P
struct PrefillEmbedParams {
  const __half* wte;       // [V][h]
  const int32_t* prompt;   // [B][prompt_ld]
  int prompt_ld, P;
  int32_t* hist;           // [B][max_ctx]
  int max_ctx;
  float* res;              // [M][h]
  int B, h, V;
};
void prefill_embed(const PrefillEmbedParams& p, cudaStream_t s);

// Causal attention of every prompt token over the prompt's KV cache (positions 0..t).
struct PrefillAttnParams {
  const __half* q;   // [M][H*d] (RoPE applied)
  const __half* kc;  // [B][H][max_seq][d] (this layer)
  const __half* vc;
  __half* out;       // [M][H*d]
  int B, P, H, d, max_seq;
  float scale;
};
void configure_prefill();
void prefill_attention(const PrefillAttnParams& p, cudaStream_t s);

// Hands the last prompt token's residual row of every sequence to the decode state: res [B][h],
// the final LayerNorm's fixed-point row sums (stripe 0 of `ln_stats`), *pos = P - 1.
struct PrefillGatherParams {
  const float* res_rows;  // [M][h]
  int P;
  float* res;             // [B][h]
  long long* ln_stats;    // kLnSlotWords slot (zeroed by the caller)
  int* pos;
  int B, h;
};
void prefill_gather(const PrefillGatherParams& p, cudaStream_t s);
// TP > 1: res[i] += part[i] + bias[i % h] (the all-reduced row-parallel output, bias added once).
void prefill_residual_add(float* res, const float* part, const __half* bias, int64_t count, int h, cudaStream_t s);

// Sum of `n` shard buffers (in shard order), written back to every shard buffer.
struct LocalReduceParams {
  float* buf[8];
  int shards;
  int64_t count;
};
void local_allreduce(const LocalReduceParams& p, cudaStream_t s, bool pdl);

}  // namespace ops
}  // namespace dsinf
