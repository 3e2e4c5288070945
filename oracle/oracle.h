/*
 * CPU oracle for the decoder-layer decode hot path.  TEST INFRASTRUCTURE ONLY: it is linked
 * or executed only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the
 * checker.  The product path (libdsinf.so) never calls it.
 *
 * What it restates, and from where:
 *   - or_derive_schedule      infersim::derive_schedule   (gemm.hpp:65-96)
 *   - or_packed_index/or_pack infersim::packed_index / pack_weights (gemm.hpp:108-130)
 *   - or_exec_sameorder       infersim::exec_reference    (gemm.hpp:147-202): fp64, identical
 *                             per-output addition order (warp slices, then warps, then
 *                             input tiles), so it is bit-identical when built with
 *                             -ffp-contract=off (checked against oracle/_ref in tests).
 *   - the layer numerics the reference does not define: LayerNorm,
 *     GPT-J rotary embedding, KV-cache attention, tanh GeLU, INT8 W8A8 quantisation,
 *     LM head and greedy argmax, arranged as the paper's layer and the
 *     canonical layer graph (fusion.hpp:242-288).
 * Parity status: GEMM order and packed layout pinned against the compiled reference and
 * golden vectors; layer numerics beyond the GEMM are "parity unpinned" (no reference
 * implementation exists for them).
 */
#ifndef DSINF_ORACLE_H_
#define DSINF_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_schedule {
  int32_t two_d;           /* TilingMode::twoD */
  int64_t output_tiles;
  int64_t input_tiles;
  int32_t warps_per_block;
  int32_t kernel_count;
  int32_t pack_M;
} or_schedule;

int32_t or_cache_line_pack(int32_t dtype_bytes);
int or_derive_schedule(int64_t N, int64_t K, int64_t B, int32_t dtype_bytes, int32_t sm_count, or_schedule* out);
int64_t or_packed_index(int64_t n, int64_t k, int64_t N, int32_t M);
/* W row-major [N][K] -> packed [ceil(K/M)*M * N] (zero K pad). */
void or_pack(const double* W, int64_t N, int64_t K, int32_t M, double* out);
/* exec_reference order over a packed matrix. */
int or_exec_sameorder(const double* packed, int64_t N, int64_t K, int32_t M, const or_schedule* s,
                      const double* x, int64_t B, double* out);
/* Same order over row-major fp32 weights (values exactly representable), multi-threaded. */
void or_gemm_f64(const float* W, int64_t N, int64_t K, const or_schedule* s, const double* x, int64_t B,
                 double* out);

/* fp16 helpers (round to nearest even) */
uint16_t or_f32_to_f16(float f);
float or_f16_to_f32(uint16_t h);
double or_round_f16(double v);

/* INT8: per-row symmetric scale = max|row| / 127 (fp32 division), q = clamp(rint(x/s)) */
void or_quant_rows(const float* x, int64_t rows, int64_t K, int8_t* q, float* scales);
void or_quant_groups(const float* x, int64_t rows, int64_t K, int64_t group, int8_t* q, uint16_t* scales_f16);
/* y[b][n] = fp32(fp32(acc) * xs[b]) * ws[n], acc = sum_k q_w[n][k] q_x[b][k] exact */
void or_gemm_i8(const int8_t* wq, const float* ws, const int8_t* xq, const float* xs, int64_t N, int64_t K,
                int64_t B, int32_t* acc, float* y);

/* Synthetic weights (same bits as the device generator). */
uint64_t or_synth_base(uint64_t seed, int32_t layer, int32_t tensor);
float or_synth_unit(uint64_t base, uint64_t flat);

/* Whole global synthetic tensors (tensor ids: include/dsinf.h DSINF_T_*): a [rows][cols] matrix
 * with rows >= valid_rows zero, or a bias / LayerNorm vector with its offset and amplitude. */
void or_synth_matrix(uint64_t seed, int32_t layer, int32_t tensor, int64_t rows, int64_t cols, int64_t valid_rows,
                     float* out);
void or_synth_vector(uint64_t seed, int32_t layer, int32_t tensor, int64_t n, float* out);

/* ------------------------------------------------------------------ decoder model */
typedef struct or_config {
  int64_t hidden, layers, heads, vocab, max_ctx;
  int32_t dtype_bytes; /* 2 fp16, 1 int8 */
  int32_t tp;          /* tensor-parallel degree mirrored (per-rank schedules / scales) */
  int32_t batch;
  int32_t sm_count;    /* device spec for derive_schedule (148 on B200) */
  uint64_t seed;
  float ln_eps, rope_base;
  int32_t int8_act;    /* int8 weights: 0 = W8A8 (per-token int8 x, int32 accumulate), 1 = W8A16 (fp16 x),
                          0x100 | mask = per GEMM (bit 0 QKV, 1 attn-out, 2 MLP-up, 3 MLP-down set = W8A16) */
  int32_t int8_group;  /* 0 = per-row weight scales; 128 = K-group fp16 scales (weight-only GEMMs) */
} or_config;

typedef struct or_model or_model;
or_model* or_model_create(const or_config* cfg);
void or_model_destroy(or_model* m);
/* One decode step at position `pos` for tokens[B]; writes logits [B][vocab] (fp32) and the
 * greedy tokens.  Appends to the oracle's KV cache. */
int or_model_step(or_model* m, const int32_t* tokens, int64_t pos, float* logits, int32_t* next_tokens);
/* Switch the int8 activation mode between steps (e.g. the W8A8 prompt prefill, then decode modes). */
void or_model_set_int8_act(or_model* m, int32_t int8_act);
/* Optional GEMM hook for the fp16 path (e.g. the reference's own exec_reference from oracle/_ref):
 * out[B][N] = x[B][K] . W^T over a row-major fp32 [N][K] shard. NULL restores the built-in
 * same-order restatement (bit-identical to exec_reference under -ffp-contract=off). */
typedef void (*or_gemm_hook_fn)(const float* W, int64_t N, int64_t K, const double* x, int64_t B, double* out,
                                void* ctx);
void or_model_set_gemm_hook(or_model* m, or_gemm_hook_fn fn, void* ctx);
/* Last step's final hidden (post-LN, fp16-rounded) [B][hidden], for debugging. */
void or_model_final_hidden(const or_model* m, float* out);

#ifdef __cplusplus
}
#endif
#endif
