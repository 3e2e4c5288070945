// Large-batch dense GEMM on the 5th-generation tensor cores (tcgen05 + TMEM), the paper's
// large-batch regime (infersim fusion.hpp:145-154 isolates the GEMMs when the
// batch is large; test_fusion.cpp:123-137).  Used for prompt prefill, where M = batch x prompt
// tokens reaches thousands of rows and the contraction is tensor-bound, not HBM-bound.
//
//   out[M][N] = epilogue( x[M][K] . W[N][K]^T )
//
// Both operands are K-major (x row-major, W the reference's row-major N x K input of
// pack_weights, gemm.hpp:113), fp16 (kind::f16, fp32 accumulate) or int8 (kind::i8, exact int32
// accumulate with per-row x scales and per-row W scales -- the W8A8 recipe of the decode path).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace dsinf {
namespace tc {

constexpr int kBM = 128;             // rows per tile (TMEM lanes)
constexpr int kBN = 256;             // columns per tile (TMEM fp32/int32 columns)
constexpr int kBK = 128;             // K bytes per pipeline stage (64 fp16 / 128 int8): one 128B swizzle atom
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK;   // 16 KB
constexpr int kBBytes = kBN * kBK;   // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;        // warp 0 TMA, warp 1 MMA issue + TMEM owner, warps 2..5 epilogue
constexpr int kEpiThreads = 128;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
// split-K mode (small M): 128 x kSBN tiles.  kSBN = 256: 4 stages of 48 KB, one CTA per SM (2/3 of
// every stage is weights); kSBN = 128: 3 stages of 32 KB, two CTAs per SM.
template <int kSBN>
struct SplitCfg {
  static constexpr int kStagesS = kSBN == 256 ? 4 : 3;
  static constexpr int kStageBytesS = kABytes + kSBN * kBK;
  static constexpr int kPartLd = kSBN + 4;  // fp32 / int32 partial row stride (floats)
  static constexpr int kSmem = kStagesS * kStageBytesS + 1024 + 256;
  static_assert(kBM * kPartLd * 4 <= kStagesS * kStageBytesS, "partial tile must fit the drained ring");
};

enum Epi : int {
  EPI_F32 = 0,       // out fp32 = y (+ bias)
  EPI_F16 = 1,       // out fp16 = y (+ bias)
  EPI_GELU_F16 = 2,  // out fp16 = gelu(y + bias)
  EPI_RESID = 3,     // out fp32 += y + bias (residual stream)
  EPI_QKV = 4,       // bias, RoPE on q/k, q -> q_out, k/v -> KV cache at the row's position
};

struct Params {
  alignas(64) CUtensorMap amap;  // x [M][K]: box 128 B x 128 rows, 128B swizzle
  alignas(64) CUtensorMap bmap;  // W [N][K]: box 128 B x 256 rows, 128B swizzle
  int M, N, K;
  int k_blocks;                  // ceil(K * elem / 128)
  int pair;                      // cluster-pair mode (set by make_maps: >= 2 row tiles)
  int bf16;                      // 16-bit operands are bfloat16 (kind::f16 with BF16 A/B formats)
  int split;                     // > 1: split-K mode for one row tile (M <= 128): `sbn`-column tiles, a cluster
                                 // of `split` CTAs per tile reduces its partials through DSMEM
  int sbn;                       // split-K column tile: 128 (default) or 256
  int w_early;                   // split-K under PDL: the first ring stages of W are issued before
                                 // griddepcontrol.wait (W must not be written by the previous kernels)
  const float* x_scale;          // int8: [M]
  const float* w_scale;          // int8: [N]
  const __half* bias;            // optional [N]
  int epi;
  void* out;
  int out_ld;
  // EPI_QKV: row m is token (m % seq_len) of sequence (m / seq_len), at position pos0 + m % seq_len
  __half* q_out;                 // [M][heads * head_dim]
  __half* k_cache;               // [B][heads][max_seq][head_dim]
  __half* v_cache;
  const float2* rope;            // [max_seq][head_dim / 2]
  int seq_len, pos0, heads, head_dim, max_seq;
};

// Builds the two TMA maps (x and W viewed as byte matrices) and checks alignment.
void make_maps(Params& p, const void* x, int x_ld_bytes, const void* w, int w_ld_bytes, int elem_bytes);
void configure();
// pdl: programmatic dependent launch (split-K mode only; the other modes ignore it)
void launch(const Params& p, bool int8, cudaStream_t s, bool pdl = false);

}  // namespace tc
}  // namespace dsinf
