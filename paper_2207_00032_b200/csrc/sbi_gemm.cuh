// SBI-GeMM for sm_100a: the skinny decode GEMM (infersim gemm.hpp:147-202)
// with Deep-Fusion prologues (LayerNorm / residual add / activation quantisation) and
// epilogues (bias, GeLU, RoPE + KV-cache append, INT8 dequant).
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace dsinf {
namespace gemm {

constexpr int kConsumerWarps = 4;
constexpr int kThreads = 32 * (kConsumerWarps + 1);
constexpr int kWarpCols = 32;                              // columns per consumer warp (one TMA box)
constexpr int kColTile = kWarpCols * kConsumerWarps;       // 128 output columns per CTA
constexpr int kRowsPerStage = 32;                          // packed rows per pipeline stage
constexpr int kBoxBytes = kWarpCols * 4 * kRowsPerStage;   // 4 KB: one 128B-swizzled TMA box
constexpr int kStageBytes = kBoxBytes * kConsumerWarps;    // 16 KB
constexpr int kMaxStages = 16;                             // ring slots (persistent step kernel: up to 13)
constexpr int kMaxB = 16;                                  // batch rows per launch
constexpr int kMaxSplit = 16;                              // K splits per column tile (cluster size)
constexpr int kPartLd = kColTile + 4;                      // split-K partial row stride (floats)
constexpr int kHeaderBytes = 1024;                         // barriers + per-row scalars
// x-streaming mode (large batch): each stage also carries the B x 32-word x tile by TMA
constexpr int kXBoxBytes = kMaxB * 128;                    // 2 KB (B rows x 128 B, 128B swizzle)
constexpr int kStageBytesXS = kStageBytes + kXBoxBytes;    // 18 KB, multiple of 1024
// W8A16 x-streaming: int8 weight stages cover 128 k, i.e. two 32-word boxes of fp16 x pairs
constexpr int kStageBytesXS16 = kStageBytes + 2 * kXBoxBytes;  // 20 KB
// LayerNorm-streaming (Plan::ln_stream, TP = 1): each stage carries the fp32 RESIDUAL boxes of its k
// range (32 floats x B rows per box: 2 for a 64-k fp16 stage, 4 for a 128-k int8 stage) and the
// consumers normalise them into the fp16 x boxes of the same stage with the producer's row sums:
// no row_prep launch between the residual-producing GEMM and the LayerNorm GEMM.
// Box slots: 1 KB (one 128B-swizzle atom) for B <= 8, else kXBoxBytes; stage = 16 KB + 3 slots
// (fp16: 2 residual + 1 x) or 6 slots (W8A16: 4 + 2).
inline int ln_box_bytes(int B) { return B <= 8 ? 1024 : kXBoxBytes; }

// Row statistics handed from a producing epilogue to the next kernel's prologue (TP = 1 path):
//   LayerNorm: per row, sum(y) and sum(y*y) in fixed point (int64; y * 2^32 and y^2 * 2^28,
//   rounded per element), so the integer atomics make them independent of CTA order;
//   int8 activations: per row, max |x| as fp32 bits (u32 atomicMax; order-independent).
// Each is striped over kStatStripes 128-byte-aligned copies to spread same-address atomics.
constexpr int kStatStripes = 8;
constexpr int kLnSlotWords = kStatStripes * kMaxB * 2;  // int64 words per LayerNorm slot
constexpr int kAmaxSlotWords = kStatStripes * 32;       // u32 words per amax slot
constexpr float kSumScale = 4294967296.0f;               // 2^32
constexpr float kSqScale = 268435456.0f;                 // 2^28

// Order-preserving key of (logit, vocab index): larger logit wins, then the LOWER index.
__host__ __device__ __forceinline__ unsigned long long argmax_key(float v, long long idx) {
  unsigned u;
  memcpy(&u, &v, 4);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | static_cast<unsigned>(~static_cast<unsigned>(idx));
}
__host__ __device__ __forceinline__ int argmax_key_index(unsigned long long k) {
  return static_cast<int>(~static_cast<unsigned>(k & 0xffffffffu));
}

enum Prologue : int {
  PRO_F16 = 0,    // x fp16 [B][x_ld] from global
  PRO_I8 = 1,     // x int8 [B][x_ld] + scales from global (already quantised)
  PRO_LN = 2,     // LayerNorm of (res_in [+ res_delta + delta_bias]) -> fp16 (or int8)
  PRO_QUANT = 3,  // x fp16 from global, per-token int8 quantisation on the fly
};

enum Epilogue : int {
  EPI_F32 = 0,       // out fp32 = y (+ bias)
  EPI_F16 = 1,       // out fp16 = y (+ bias)
  EPI_GELU_F16 = 2,  // out fp16 = gelu(y + bias)
  EPI_QKV = 3,       // q/k/v = y + bias, RoPE on q,k, q -> q_out, k/v -> KV cache at pos
  EPI_RESID = 4,     // out fp32 += y + bias (residual stream; one writer per column)
};

struct Params {
  // packed weights viewed by TMA as a 2-D tensor of 32-bit words [rows][N]; a word holds pack_M
  // consecutive k of one output column (gemm.hpp:108-111)
  alignas(64) CUtensorMap tmap;
  // x-streaming mode: x as a 2-D tensor of 32-bit words [B][ceil(K/M)] (GEMM-ready fp16 pairs
  // or int8 quads); each stage loads one box of 32 words x B rows next to the weight boxes
  alignas(64) CUtensorMap xmap;
  const float* w_scale;  // int8: per-output-row scale [N]
  const __half* w_gscale;  // W8A16 only, optional: K-group scales [ceil(K/128)][N] (then w_scale unused)
  int N, rows, K, B;
  int rows_per_split;    // multiple of kRowsPerStage; split s covers [s*rps, (s+1)*rps)
  int stages;
  int x_row_words;       // smem stride of one x row (== 8 mod 32)
  int box_bytes;         // LayerNorm-streaming: smem slot of one activation box (set by launch)
  // prologue
  int pro;
  int a16;               // int8 weights with fp16 x (W8A16, weight-only): fp32 accumulate, y = acc * w_scale
  const void* x;
  int x_ld;
  const float* x_scale;
  const float* res_in;
  const float* res_delta;
  const __half* delta_bias;
  // fused tensor-parallel all-reduce (consumer side): res_delta holds `delta_slots` partials
  // `delta_stride` floats apart (one per rank, summed in rank order); red_flag must reach
  // (*step_ctr + 1) * red_per_step before they are read (0 slots = plain res_delta)
  int delta_slots;
  long long delta_stride;
  const unsigned long long* red_flag;
  const long long* step_ctr;
  unsigned long long red_per_step;
  float* res_out;
  const __half* ln_g;
  const __half* ln_b;
  float ln_eps;
  double ln_inv_k;               // 1 / K (set by launch)
  const long long* ln_stats_in;  // PRO_LN: row sums from the producer (else a full-row pass)
  const unsigned* amax_in;       // PRO_QUANT: row max |x| from the producer (else a full-row pass)
  // epilogue
  int epi;
  const __half* bias;
  void* out;
  int out_ld;
  __half* q_out;      // [B][heads*head_dim]
  __half* k_cache;    // [B][heads][max_seq][head_dim] (this layer)
  __half* v_cache;
  const float2* rope;  // [max_seq][head_dim/2] (cos, sin)
  const int* pos;
  int heads, head_dim, max_seq;
  // EPI_QKV attention tail (Deep-Fusion region 2 inside the QKV launch, LayerNorm-streaming plan):
  // after its epilogue a cluster bumps head_ctr[h] for every head its column tile touches (q, k or v
  // section); the cluster completing a head runs that head's decode attention over positions
  // 0..*pos, its nsplit CTAs splitting the context and merging through DSMEM, and writes attn_out
  // [B][heads*head_dim] fp16 (+ attn_amax row max |out| stripes when non-null).  The standalone
  // attention launch is skipped.  head_ctr: [heads] per layer, zero at rest (the completer resets).
  int attn_tail;
  unsigned* head_ctr;
  __half* attn_out;
  unsigned* attn_amax;
  float attn_scale;
  long long* ln_stats_out;  // EPI_RESID: accumulate the new residual's row sums (slot, zeroed per step)
  unsigned* amax_out;       // EPI_F16 / EPI_GELU_F16: accumulate row max |out|
  // fused all-reduce (producer side, EPI_F32): the partial [B][N] goes to push_dst[q] (rank q's slot
  // for this rank) for q < push_n, then each CTA adds 1 to every push_flag[q] (system scope)
  int push_n;
  int push_gpu_scope;  // 1: every destination is on this GPU (TP_LOCAL / TP_SLICE): gpu-scope fence
  float* push_dst[8];
  unsigned long long* push_flag[8];
  // system-scope pushes (cross-process / cross-GPU): each CTA bumps this gpu-local counter after a
  // gpu-scope fence and only the grid's LAST CTA issues the system-scope fence and signals the t
  // destinations (one signal per rank instead of one per CTA); null = every CTA signals
  unsigned long long* push_done;
  const long long* push_step;
  unsigned long long push_ctas;
  // EPI_F32 without bias (LM head): greedy argmax fused into the epilogue -- per row the max of
  // pack(value, global column) over columns < am_valid, atomicMax'd into am_out[b] (zeroed per
  // step); ties resolve to the lowest column (moe.hpp:69-74).
  unsigned long long* am_out;
  int am_valid;
  long long am_offset;
  // Flag-granular dependency (x-streaming W8A16 / fp16 plans, TP = 1, DSINF_DOWN_FLAGS): instead of
  // griddepcontrol.wait before its first x box, the producer waits until the x-producing GEMM's
  // column-tile counters covering this CTA's k range reach (*dep_step + 1) * dep_per_step; the
  // epilogue still waits for the whole previous grid.  out_flags: the producer side (+1 per CTA per
  // column tile after its epilogue stores).
  const unsigned* dep_flags;
  unsigned dep_per_step;
  const long long* dep_step;
  unsigned* out_flags;
  unsigned long long* trace;  // launch timeline slot (ptx::trace_begin / trace_end) or null
  unsigned long long* cta_log;  // diagnostics: per-CTA [smid, start, release, prologue end, loop end, end] or null
};

struct Plan {
  int x_stream;  // 1: x streamed per stage by TMA (PRO_F16 / PRO_I8 only), no smem x slice
  int ln_stream;  // 1 (with x_stream): the residual is streamed and LayerNorm'd per stage (PRO_LN)
  int k_groups;   // 1: smem for the CTA's K-group scales ([stage][128] fp16 after the x / gamma-beta region)
  int a16;       // W8A16 plan (int8 weights, fp16 x): 1 signed weight bytes, 2 biased (s + 128)
  int col_tiles;
  int ksplit;
  int rows_per_split;
  int stages;
  int nb8;
  size_t smem_bytes;
};

// TMA descriptor of a packed weight matrix (N words per row, `rows` rows), 128B swizzle,
// box = 32 words x kRowsPerStage rows.  Out-of-bounds rows / columns read as zero.
void make_weight_map(CUtensorMap* map, const void* w_packed, int N, int rows);
// Sets kernel attributes for every instantiation; call before graph capture.
void configure();
// a16_biased: the W8A16 weights are stored biased (s + 128 per byte; the decode model's own weights)
// k_groups: W8A16 with K-group scales (the CTA's group scales are staged in shared memory)
// stage_cap > 0: that many ring stages (at most; per-GEMM request from the model)
Plan make_plan(int N, int K, int B, bool int8_weights, int forced_split, bool x_stream = false, bool a16 = false,
               bool ln_stream = false, bool a16_biased = false, bool k_groups = false, int stage_cap = 0);
// TMA descriptor of x for the x-streaming mode: `words` 32-bit words per row, `B` rows, row
// stride ld_words (ld_words * 4 must be a multiple of 16 and x 16-byte aligned).
void make_x_map(CUtensorMap* map, const void* x, int words, int B, int ld_words);
// Whether x (fp16 [B][x_ld] or int8) can be streamed: alignment of base and row stride.
bool x_streamable(const void* x, int x_ld, int K, bool int8_x);
// Batch sizes that use the x-streaming plan (DSINF_XS=0 never, =1 always; default B >= kXsMinBatch).
// Measured with the cluster-split row_prep: x-streaming wins at every batch (GPT-J B=1 fp16 2.75 ->
// 2.71 ms, int8 2.04 -> 1.98; GPT-2 int8 1.74 -> 1.60; B=2 fp16 2.98 -> 2.75)
constexpr int kXsMinBatch = 1;
// `tp`: the layer's LayerNorm input is an all-reduced sum (TP > 1), so its row statistics cannot
// come from the producing GEMM's epilogue: one row_prep launch + x-streaming beats every CTA
// re-deriving them (GPT3-175B t=8 rank slice at B = 1: 12.8 -> 9.7 ms fp16, 10.3 -> 7.4 ms int8)
bool prefer_x_stream(int B, bool tp = false);
void launch(const Params& p, const Plan& plan, bool int8_weights, cudaStream_t stream, bool pdl);

}  // namespace gemm
}  // namespace dsinf
