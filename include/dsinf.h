/*
 * dsinf.h — C ABI of the B200-native DeepSpeed-Inference decoder-layer decode hot path.
 *
 * Every entry point replaces one symbol of the reference's header-only C++ library
 * (`infersim`, reference proj/include/infersim/{gemm,fusion,model,costmodel}.hpp).  The
 * reference has no FFI;
 * this ABI is what a maintainer would bind from any host language.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types.
 *   - Return value: DSINF_OK (0) or an error code; the thread-local text is available
 *     from dsinf_last_error().  ConfigError (bad input) -> 2, InfeasibleError (does not
 *     fit) -> 3, matching the reference CLI's exit-code convention.
 *   - `stream` arguments are cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Device-side entry points never allocate, never synchronise and are capturable in a
 *     CUDA graph; host-side entry points are pure and reentrant.
 */
#ifndef DSINF_H_
#define DSINF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status codes */
#define DSINF_OK 0
#define DSINF_ERR_CONFIG 2     /* infersim::ConfigError     (errors.hpp:24-27) */
#define DSINF_ERR_INFEASIBLE 3 /* infersim::InfeasibleError (errors.hpp:30-34) */
#define DSINF_ERR_CUDA 4
#define DSINF_ERR_NCCL 5
#define DSINF_ERR_INTERNAL 6

/* ---------------------------------------------------------------- element types */
#define DSINF_DT_F16 1 /* IEEE binary16 */
#define DSINF_DT_F32 2
#define DSINF_DT_I8 3  /* symmetric int8 with fp32 scales */
#define DSINF_DT_F64 4 /* host-side only (reference container type) */
#define DSINF_DT_BF16 5 /* bfloat16 (large-batch tensor-core GEMM) */

const char* dsinf_last_error(void);
const char* dsinf_version(void);

/* ================================================================ gemm.hpp (SBI-GeMM) */

/* infersim::GemmShape (gemm.hpp:28-40): out = W (N x K) * x^T for B token vectors. */
typedef struct dsinf_gemm_shape {
  int64_t out_dim; /* N */
  int64_t in_dim;  /* K */
  int64_t batch;   /* B */
  int32_t dtype_bytes;
} dsinf_gemm_shape;

/* infersim::TilingMode (gemm.hpp:42) */
#define DSINF_TILING_1D 0
#define DSINF_TILING_2D 1

/* infersim::GemmSchedule (gemm.hpp:47-54) */
typedef struct dsinf_gemm_schedule {
  int32_t mode; /* DSINF_TILING_1D / DSINF_TILING_2D */
  int64_t output_tiles;
  int64_t input_tiles;
  int32_t warps_per_block;
  int32_t kernel_count;
  int32_t pack_M;
} dsinf_gemm_schedule;

/* infersim::DeviceSpec (hardware.hpp:36-69).  The reference's peak_flops_by_dtype map
 * becomes three slots; a slot <= 0 means "no entry" (peak_flops() throws ConfigError). */
typedef struct dsinf_device_spec {
  int64_t mem_bytes;
  double mem_bw; /* bytes/s */
  int32_t sm_count;
  double kernel_launch_overhead; /* seconds */
  double peak_flops_fp32;        /* dtype_bytes 4 */
  double peak_flops_fp16;        /* dtype_bytes 2 */
  double peak_flops_int8;        /* dtype_bytes 1 */
} dsinf_device_spec;

/* B200 values (148 SMs; mem_bw from MEASURED_PEAKS when the caller has it). */
void dsinf_b200_device_spec(dsinf_device_spec* out);

/* infersim::kOutputTileWidth (gemm.hpp:45) */
int64_t dsinf_output_tile_width(void);
/* infersim::cache_line_pack (gemm.hpp:57-60) */
int32_t dsinf_cache_line_pack(int32_t dtype_bytes);
/* infersim::derive_schedule (gemm.hpp:65-96) */
int dsinf_derive_schedule(const dsinf_gemm_shape* shape, const dsinf_device_spec* device,
                          dsinf_gemm_schedule* out);
/* infersim::packed_index (gemm.hpp:108-111) */
int64_t dsinf_packed_index(int64_t n, int64_t k, int64_t out_dim, int32_t pack_M);
/* infersim::pack_weights (gemm.hpp:113-130), host fp64 container.
 * `packed` must hold out_dim * padded_in_dim doubles (query with packed==NULL). */
int dsinf_pack_weights_f64(const double* matrix, int64_t matrix_len, const dsinf_gemm_shape* shape,
                           int32_t pack_M, double* packed, int64_t packed_len,
                           int64_t* padded_in_dim);
/* infersim::unpack_weights (gemm.hpp:132-139) */
int dsinf_unpack_weights_f64(const double* packed, int64_t packed_len,
                             const dsinf_gemm_shape* shape, int32_t pack_M, double* matrix,
                             int64_t matrix_len);
/* infersim::exec_reference (gemm.hpp:147-202) executed on the GPU.
 * Host fp64 in/out like the reference; the device computes in `compute_dtype`
 * (DSINF_DT_F16: fp16 operands, fp32 accumulate; DSINF_DT_I8: W8A8 int32 accumulate).
 * `packed` is the reference layout produced by pack_weights with `packed_pack_M`
 * (PackedWeights::pack_M): the data is read with that M, as exec_reference reads it with
 * packed.pack_M; schedule->pack_M only groups the iteration (gemm.hpp:180-183), so any
 * packed_pack_M in {1, 2, 4} gives the same result under any schedule. */
int dsinf_exec_device(const double* packed, int64_t packed_len, int32_t packed_pack_M,
                      const dsinf_gemm_shape* shape, const dsinf_gemm_schedule* schedule,
                      const double* x, int64_t x_len, int64_t batch, int32_t compute_dtype,
                      double* out, int64_t out_len);

/* ---- device-resident SBI-GeMM (the decode hot path; pointers are device pointers) */

/* pack_weights on device: row-major W (N x K, element type src_dtype in {F16,F32})
 * -> packed [ceil(K/M)][N][M] in dst_dtype F16 (M = 2 or the given pack_M). */
int dsinf_pack_weights_device(const void* w_rowmajor, int32_t src_dtype, int64_t N, int64_t K,
                              int32_t pack_M, void* packed_f16, void* stream);
/* INT8 weight quantisation: per-output-row symmetric scale s_n = max|w_n.| / 127 (fp32
 * IEEE divide), q = clamp(rint(w / s_n), -127, 127); packed with pack_M = 4. */
int dsinf_quantize_weights_int8(const void* w_rowmajor_f16, int64_t N, int64_t K,
                                int8_t* packed_i8, float* row_scales, void* stream);
/* INT8 K-group weight quantisation ("per-group dequant"; SURVEY §8c K-group
 * recipe): every `group` (= 128) consecutive k of an output row share an fp16 scale
 * s = fp16(max|w| / 127) (fp32 divide, round to nearest; 1 for an all-zero group) and
 * q = clamp(rint(w / s), -127, 127) with an fp32 divide; packed with pack_M = 4 like the row mode,
 * group_scales_f16 [ceil(K/group)][N].  The W8A16 GEMM computes y = sum_g s_g * sum_{k in g} q x
 * (fp32 per-group partial sums folded with the group scale). */
int dsinf_quantize_weights_int8_groups(const void* w_rowmajor_f16, int64_t N, int64_t K, int32_t group,
                                       int8_t* packed_i8, void* group_scales_f16, void* stream);
/* Per-token activation quantisation (same formula, scale per row of x). */
int dsinf_quantize_activations_int8(const void* x_f16, int64_t B, int64_t K, int8_t* xq,
                                    float* scales, void* stream);

/* INT8 weight modes ("INT8 weight-quantized GEMMs"):
 *  W8A8  per-token int8 activations, exact int32 accumulation (bit-exact vs the oracle);
 *  W8A16 weight-only: fp16 activations, int8 weights widened in registers, fp32 accumulation,
 *        per-output-row dequant -- no activation quantisation on the decode critical path. */
#define DSINF_INT8_W8A8 0
#define DSINF_INT8_W8A16 1
#define DSINF_INT8_AUTO 2 /* runtime config only (measured): W8A16 at TP = 1 and for batch <= 8; W8A8
                             everywhere at TP > 1 and batch > 8 */

#define DSINF_EPI_NONE 0
#define DSINF_EPI_GELU 1 /* tanh GeLU after the bias */

typedef struct dsinf_gemm_args {
  const void* w_packed;   /* F16: [ceil(K/2)][N][2] halves; I8: [ceil(K/4)][N][4] int8 */
  int32_t w_dtype;        /* DSINF_DT_F16 or DSINF_DT_I8 */
  const float* w_scales;  /* I8 only: [N] per-row scales */
  int64_t N, K, B;
  const void* x;          /* [B][K] row-major; F16, or I8 (pre-quantised) */
  int32_t x_dtype;        /* F16 (int8 GEMMs quantise it per token on the fly) or I8 */
  const float* x_scales;  /* I8 x only: [B] */
  const void* bias;       /* optional F16 [N] */
  void* out;              /* [B][N] row-major */
  int32_t out_dtype;      /* F32 or F16 */
  int32_t epilogue;       /* DSINF_EPI_* */
  int32_t ksplit;         /* 0 = launch plan chooses; else cluster split count {1,2,4,8,16} */
  int32_t int8_act;       /* I8 weights: DSINF_INT8_W8A8 (int8 x, int32 accumulate) or DSINF_INT8_W8A16 */
  const void* w_group_scales; /* W8A16 only, optional: fp16 [ceil(K/128)][N] K-group scales
                                 (dsinf_quantize_weights_int8_groups); w_scales is then unused */
  int32_t group_size;     /* 0: per-output-row scales; 128: K-group scales */
} dsinf_gemm_args;

int dsinf_gemm(const dsinf_gemm_args* args, void* stream);

/* ---- large-batch regime (fusion.hpp:145-154: GEMMs isolated when the batch is large; the paper's
 * prompt / large-batch path): tcgen05 tensor-core GEMM with TMEM accumulators.
 * Weights are the row-major N x K matrix pack_weights takes as input (gemm.hpp:113), K-major like
 * x.  F16: fp16 operands, fp32 accumulate.  I8: W8A8, exact int32 accumulate, per-row W scales
 * and per-row x scales (the decode recipe; quantise both with dsinf_quantize_activations_int8). */
#define DSINF_EPI_RESID 2 /* out (F32) += x.W^T + bias: residual-stream update */
typedef struct dsinf_gemm_lb_args {
  const void* w;          /* [N][K] row-major, F16 or I8 */
  int32_t w_dtype;        /* DSINF_DT_F16, DSINF_DT_BF16 (F32 out, no bias) or DSINF_DT_I8 (x has the same type) */
  const float* w_scales;  /* I8: [N] */
  int64_t N, K, M;
  const void* x;          /* [M][K] row-major */
  const float* x_scales;  /* I8: [M] */
  const void* bias;       /* optional F16 [N] */
  void* out;              /* [M][N] row-major */
  int32_t out_dtype;      /* F32 or F16 (DSINF_EPI_GELU needs F16, DSINF_EPI_RESID F32) */
  int32_t epilogue;       /* DSINF_EPI_NONE / DSINF_EPI_GELU / DSINF_EPI_RESID */
} dsinf_gemm_lb_args;
int dsinf_gemm_large_batch(const dsinf_gemm_lb_args* args, void* stream);

/* The B200 launch plan the device GEMM uses for a shape (extension of derive_schedule):
 * column tile width, split-K cluster size and packed rows per split. */
typedef struct dsinf_launch_plan {
  int32_t col_tile;
  int32_t ksplit;
  int32_t rows_per_split;
  int32_t ctas;
  int32_t stages;
} dsinf_launch_plan;
int dsinf_gemm_launch_plan(int64_t N, int64_t K, int64_t B, int32_t w_dtype,
                           dsinf_launch_plan* out);

/* ---- decode attention over the KV cache (paper region 2, "transposition + attention") */
/* q: [B][H][d] F16; kcache/vcache: [B][H][max_seq][d] F16; positions 0..pos are attended.
 * out: [B][H*d] F16.  pos_dev: device int32 (current position). */
int dsinf_attention_decode(const void* q, const void* kcache, const void* vcache,
                           const int32_t* pos_dev, int64_t B, int64_t H, int64_t d,
                           int64_t max_seq, void* out, void* stream);

/* ================================================================ decoder model (Deep-Fusion) */

typedef struct dsinf_model_config { /* infersim::ModelConfig (model.hpp:42-64), dense */
  int64_t hidden_dim;
  int64_t num_layers;
  int64_t num_heads;
  int64_t vocab_size;
  int64_t max_seq;
  int32_t dtype_bytes; /* 2 = FP16 weights, 1 = INT8 (W8A8) weights */
} dsinf_model_config;

#define DSINF_TP_NONE 0
#define DSINF_TP_NCCL 1  /* one process per GPU, NCCL all-reduce over NVLink */
#define DSINF_TP_LOCAL 2 /* all shards on this device (single-GPU sharding check) */
#define DSINF_TP_IPC 4   /* one process per rank, every cross-rank exchange over CUDA-IPC peer memory
                            (fused all-reduce in the GEMM epilogues, argmax keys in select): no NCCL.
                            Ranks may share a device.  Handles are exchanged by the caller:
                            dsinf_model_ipc_handle -> all-gather -> dsinf_model_ipc_attach. */
#define DSINF_TP_SLICE 3 /* rank tp_rank's shard alone on this device, collectives skipped: per-rank
                            step timing of a TP model on one GPU (outputs are not the model's) */

typedef struct dsinf_runtime_config {
  int32_t batch;        /* sequences per step, 1..16 per launch */
  int32_t tp_size;      /* tensor-parallel degree t */
  int32_t tp_rank;      /* this process's rank (NCCL mode) */
  int32_t tp_mode;      /* DSINF_TP_* */
  int32_t use_cuda_graph;
  int32_t use_pdl;      /* programmatic dependent launch between kernels */
  int64_t max_ctx;      /* KV-cache capacity per sequence (<= max_seq) */
  uint64_t seed;        /* synthetic-weight seed */
  float ln_eps;
  float rope_base;
  int32_t device;       /* CUDA device ordinal */
  int32_t use_step_kernel; /* TP = 1: run each decode step as ONE persistent kernel */
  int32_t int8_act;     /* dtype_bytes 1: DSINF_INT8_W8A8 (default), DSINF_INT8_W8A16 or DSINF_INT8_AUTO
                           (decode GEMMs; the tensor-core prefill stays W8A8) */
  int32_t int8_group;   /* dtype_bytes 1: 0 = per-output-row scales; 128 = K-group scales (fp16 per
                           128 k of a row; decode GEMMs W8A16 with per-group dequant; no prefill) */
} dsinf_runtime_config;

typedef struct dsinf_model dsinf_model;

/* nccl_comm: ncclComm_t from dsinf_nccl_comm_create (NCCL mode) or NULL. */
int dsinf_model_create(const dsinf_model_config* cfg, const dsinf_runtime_config* rt,
                       void* nccl_comm, dsinf_model** out);
int dsinf_model_destroy(dsinf_model* m);
/* DSINF_TP_IPC: this rank's CUDA-IPC handles (an opaque blob of *len bytes, the same size on every
 * rank; out may be NULL to query the size).  The caller all-gathers the blobs in rank order (any
 * host channel: gloo, MPI, sockets) and passes the t * len bytes to dsinf_model_ipc_attach before
 * the first decode step.  Replaces the NCCL handle all-gather of DSINF_TP_NCCL's fused all-reduce
 * (costmodel.hpp:84-85: the per-layer all-reduce moved into the producing GEMM's epilogue). */
int dsinf_model_ipc_handle(dsinf_model* m, void* out, int64_t cap, int64_t* len);
int dsinf_model_ipc_attach(dsinf_model* m, const void* all, int64_t len);
/* Load B prompts of prompt_len tokens (host int32 [B][prompt_len]) and reset position 0. */
int dsinf_model_set_prompt(dsinf_model* m, const int32_t* prompt_host, int64_t prompt_len,
                           void* stream);
/* Same with a device buffer (no host copy). */
int dsinf_model_set_prompt_device(dsinf_model* m, const int32_t* prompt_dev, int64_t prompt_len,
                                  void* stream);
/* Enqueue one decode step: embed the token at the current position (prompt token while
 * pos < prompt_len, else the previous greedy token), run every layer, the LM head and the
 * greedy argmax, then advance the position.  Replays a CUDA graph when enabled. */
/* Prompt prefill in the large-batch regime (fusion.hpp:145-154): all B x P
 * prompt tokens through every layer at once on the tcgen05 tensor cores, leaving the model in the
 * state dsinf_decode_steps(m, P) would (KV cache rows 0..P-1, history, next token, position P).
 * Needs a prompt set at position 0.  Every TP mode is supported: TP_NONE, TP_LOCAL and TP_NCCL
 * give the model's outputs (column-/row-parallel GEMMs, the row-parallel partials all-reduced,
 * vocab-parallel LM head with the argmax keys gathered); TP_SLICE runs rank tp_rank's shard alone
 * and its outputs are for timing only; TP_IPC and int8_group = 128 are rejected (ConfigError).
 * First call generates row-major weight copies, or -- when they would not fit -- one layer's
 * operands refilled from the packed weights before each layer (one resident weight copy). */
int dsinf_model_prefill(dsinf_model* m, void* stream);
int dsinf_decode_step(dsinf_model* m, void* stream);
/* Enqueue `steps` decode steps back to back. */
int dsinf_decode_steps(dsinf_model* m, int64_t steps, void* stream);
/* One end-to-end step with host buffers: tokens_in [B] (used once pos >= prompt_len) is copied
 * host->device, the step runs, the greedy tokens come back in tokens_out [B]; synchronises. */
int dsinf_decode_step_host(dsinf_model* m, const int32_t* tokens_in, int32_t* tokens_out, void* stream);
/* Device pointers to the step outputs. logits: [B][vocab_local_padded] F32 (this rank's
 * vocab shard); next_tokens: [B] int32; history: [B][max_ctx] int32 (token at each pos). */
int dsinf_model_outputs(dsinf_model* m, float** logits, int64_t* logits_ld, int32_t** next_tokens,
                        int32_t** history, int32_t** pos);
/* Host copies of the same (synchronises `stream`). */
int dsinf_model_read_logits(dsinf_model* m, float* host, int64_t len, void* stream);
int dsinf_model_read_tokens(dsinf_model* m, int32_t* next_host, int32_t* history_host,
                            int64_t history_len, void* stream);
typedef struct dsinf_model_info {
  int64_t weight_bytes;        /* device bytes of all weights on this rank */
  int64_t bytes_per_token;     /* algorithmic HBM bytes per decode step at current pos */
  int64_t kernels_per_step;    /* kernel launches per step (ours, excluding NCCL) */
  int64_t vocab_local;         /* logits row length per rank (padded) */
  int64_t heads_local;
  int64_t kv_bytes;
  int32_t shards;              /* shards resident on this device */
  int32_t graph_ready;
  int32_t fused_allreduce;     /* 1: row-parallel GEMM epilogues push to the peers' slots (no all-reduce launch) */
  int32_t plan_flags;          /* DSINF_PLAN_* bits of the decode schedule in use */
} dsinf_model_info;
#define DSINF_PLAN_X_STREAM 1     /* LayerNorm'd x written once by row_prep and streamed by TMA */
#define DSINF_PLAN_FUSED_STATS 2  /* LayerNorm row statistics fused into the producing epilogues */
#define DSINF_PLAN_STEP_KERNEL 4  /* the persistent whole-step kernel */
#define DSINF_PLAN_STREAM_KERNEL 8 /* the statically scheduled persistent decode kernel */
int dsinf_model_get_info(const dsinf_model* m, dsinf_model_info* out);
/* Per-CTA phase timeline of the last persistent step (built with DSINF_STEP_TRACE=1):
 * [grid][phases][4] globaltimer ns (wait begins, wait satisfied, phase done, producer's last
 * weight load issued).  out == NULL queries the length; returns DSINF_ERR_CONFIG if not traced. */
int dsinf_model_step_trace(dsinf_model* m, uint64_t* out, int64_t len, int64_t* needed, int32_t* grid,
                           int32_t* phases);
/* Per-launch timeline of the last per-kernel decode step when launch tracing is on
 * (DSINF_LAUNCH_TRACE=1 at creation, or dsinf_model_set_launch_trace): for launch i in enqueue
 * order, out[3*i] / out[3*i+1] = globaltimer ns of its first CTA start / last CTA end and
 * out[3*i+2] = its kind (DSINF_LK_*).  out == NULL queries the launch count. */
#define DSINF_LK_EMBED 0
#define DSINF_LK_QKV 1
#define DSINF_LK_ATTN 2
#define DSINF_LK_O 3
#define DSINF_LK_UP 4
#define DSINF_LK_DOWN 5
#define DSINF_LK_LM 6
#define DSINF_LK_ARGMAX 7
#define DSINF_LK_PREP 8 /* row preparation (LayerNorm / quantisation) of the x-streaming plan */
int dsinf_model_launch_trace(dsinf_model* m, uint64_t* out, int64_t len, int64_t* launches);
/* Phase stamps of the same launches (SBI-GeMM only; other kernels leave ~0 / 0): out[8*i + 0] =
 * earliest dependency release, [8*i + 1] = latest prologue end, [8*i + 2] = latest main-loop end
 * (globaltimer ns), [8*i + 3] = longest per-CTA prologue (ns), [8*i + 4] = latest release,
 * [8*i + 5..7] = sub-phase probes (longest per-CTA time since release, ns).
 * Diagnostics, not on the reference path. */
int dsinf_model_launch_phases(dsinf_model* m, uint64_t* out, int64_t len);
/* Diagnostics (DSINF_CTA_LOG=<n> at creation): per-CTA [smid, start, release, prologue end, loop
 * end, end] globaltimer stamps of the n-th SBI-GeMM launch of the last step, 6 words per CTA. */
int dsinf_model_cta_log(dsinf_model* m, uint64_t* out, int64_t len);
/* Turn the per-launch timeline on (1) or off (0) after creation; re-captures the step graph. */
int dsinf_model_set_launch_trace(dsinf_model* m, int on);
/* Bytes per step for an arbitrary position (ctx = pos + 1). */
int64_t dsinf_model_bytes_per_step(const dsinf_model* m, int64_t pos);
/* Copy one synthetic weight tensor of layer `layer` in logical row-major fp32 form
 * (tensor ids: DSINF_T_*), for tests.  Returns the full (un-sharded) matrix. */
#define DSINF_T_QKV 1
#define DSINF_T_QKV_BIAS 2
#define DSINF_T_O 3
#define DSINF_T_O_BIAS 4
#define DSINF_T_UP 5
#define DSINF_T_UP_BIAS 6
#define DSINF_T_DOWN 7
#define DSINF_T_DOWN_BIAS 8
#define DSINF_T_LN1_G 9
#define DSINF_T_LN1_B 10
#define DSINF_T_LN2_G 11
#define DSINF_T_LN2_B 12
#define DSINF_T_WTE 13
#define DSINF_T_LNF_G 14
#define DSINF_T_LNF_B 15
/* Host-side generator (same bits the device generator writes). */
int dsinf_synthetic_tensor(uint64_t seed, int32_t layer, int32_t tensor, int64_t rows,
                           int64_t cols, float* out_fp32_of_fp16);
/* Rank `rank`'s tensor-parallel shard of one tensor, logical row-major [rows][cols] fp16
 * values as fp32 (the map the device generator uses; out == NULL queries rows/cols).
 * layer = -1 for the embedding / LM head (DSINF_T_WTE) and the final LayerNorm. */
int dsinf_shard_tensor(const dsinf_model_config* cfg, int32_t tp, int32_t rank, int32_t layer,
                       int32_t tensor, uint64_t seed, float* out, int64_t out_len, int64_t* rows,
                       int64_t* cols);

/* ---- NCCL (loaded with dlopen on first use; NCCL mode only) */
int dsinf_nccl_get_unique_id(uint8_t id_out[128]);
int dsinf_nccl_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                           void** comm_out);
int dsinf_nccl_comm_destroy(void* comm);
/* Probe of the NCCL-mode all-reduce buffers: *symmetric = 1 when libnccl exports ncclMemAlloc /
 * ncclCommWindowRegister (NCCL >= 2.27), in which case a `count`-float buffer is allocated with
 * ncclMemAlloc and registered as an NCCL_WIN_COLL_SYMMETRIC window (as the model's per-layer
 * all-reduce buffers are in DSINF_TP_NCCL; DSINF_NCCL_WINDOWS=0 disables that); a sum all-reduce of
 * ones runs on it and *first_out receives element 0 (= the number of ranks).  Collective. */
int dsinf_nccl_window_check(void* comm, int64_t count, int32_t* symmetric, float* first_out);

/* ================================================================ model.hpp accounting */

/* infersim::param_count (model.hpp:93-101), dense models */
int dsinf_param_count(const dsinf_model_config* cfg, int64_t* out);
/* infersim::param_bytes (model.hpp:103-105) */
int dsinf_param_bytes(const dsinf_model_config* cfg, int64_t* out);
#define DSINF_PHASE_PROMPT 0
#define DSINF_PHASE_GENERATION 1
/* infersim::layer_flops (model.hpp:121-132) */
int dsinf_layer_flops(const dsinf_model_config* cfg, int64_t batch, int64_t prompt_len,
                      int64_t gen_tokens, int32_t phase, double* out);
/* infersim::kv_cache_bytes (model.hpp:135-140) */
int dsinf_kv_cache_bytes(const dsinf_model_config* cfg, int64_t batch, int64_t prompt_len,
                         int64_t gen_tokens, int64_t* out);

/* ================================================================ costmodel.hpp */

typedef struct dsinf_kernel_cost { /* infersim::KernelCost (costmodel.hpp:31-38) */
  double compute_time, memory_time, launch_overhead, total;
  int32_t memory_bound;
} dsinf_kernel_cost;
/* infersim::kernel_time (costmodel.hpp:42-56) */
int dsinf_kernel_time(double flops, double bytes_moved, const dsinf_device_spec* device,
                      int32_t dtype_bytes, int64_t fused_launches, int32_t cuda_graph,
                      dsinf_kernel_cost* out);

typedef struct dsinf_link_spec { double bandwidth, latency; } dsinf_link_spec;
typedef struct dsinf_topology { /* the fields of infersim::Topology collective_time reads */
  int32_t num_nodes, gpus_per_node;
  dsinf_link_spec intra, inter;
  dsinf_device_spec device;
} dsinf_topology;
#define DSINF_COLL_ALLREDUCE 0
#define DSINF_COLL_ALLGATHER 1
#define DSINF_COLL_ALLTOALL 2
#define DSINF_COLL_BROADCAST 3
#define DSINF_COLL_P2P 4
/* infersim::collective_time (costmodel.hpp:70-104) */
int dsinf_collective_time(int32_t kind, double bytes_per_rank, const int32_t* group,
                          int32_t group_size, const dsinf_topology* topo, double* out);
/* infersim::min_latency_bound (costmodel.hpp:113-125) */
int dsinf_min_latency_bound(const dsinf_model_config* cfg, int32_t tp, int32_t pp,
                            const dsinf_topology* topo, double* out);

/* ================================================================ fusion.hpp (Deep-Fusion) */

#define DSINF_OP_ELEMENTWISE 0 /* infersim::OpKind (fusion.hpp:29) */
#define DSINF_OP_REDUCTION 1
#define DSINF_OP_TRANSPOSE 2
#define DSINF_OP_GEMM 3
#define DSINF_OP_QUANTIZE 4
#define DSINF_REGIME_SMALL_BATCH 0 /* infersim::BatchRegime (fusion.hpp:135) */
#define DSINF_REGIME_LARGE_BATCH 1

/* Flattened infersim::OpGraph (fusion.hpp:39-116).  Edge e's tile_dep map is stored as
 * CSR: consumer tiles dep_consumer[dep_off[e] .. dep_off[e+1]) each with producer set
 * dep_prod[prod_off[i] .. prod_off[i+1]). */
typedef struct dsinf_op_graph {
  int32_t num_nodes;
  const int32_t* node_kind;       /* [num_nodes] DSINF_OP_* */
  const int32_t* node_tile_count; /* [num_nodes] */
  const int64_t* node_out_elems;  /* [num_nodes] */
  int32_t num_edges;
  const int32_t* edge_from;       /* [num_edges] */
  const int32_t* edge_to;         /* [num_edges] */
  const int32_t* dep_off;         /* [num_edges + 1] into dep_consumer */
  const int32_t* dep_consumer;    /* consumer tile ids */
  const int32_t* prod_off;        /* [len(dep_consumer) + 1] into dep_prod */
  const int32_t* dep_prod;        /* producer tile ids */
  int32_t dtype_bytes;
} dsinf_op_graph;

/* infersim::fusable (fusion.hpp:126-133) */
int dsinf_fusable(const dsinf_op_graph* g, int32_t edge, int32_t* out);
/* infersim::partition_layer (fusion.hpp:140-173): region_of[node] = region index. */
int dsinf_partition_layer(const dsinf_op_graph* g, int32_t regime, int32_t* region_of,
                          int32_t* num_regions);
/* infersim::fusion_savings (fusion.hpp:183-215) */
int dsinf_fusion_savings(const dsinf_op_graph* g, const int32_t* region_of, int32_t num_regions,
                         int64_t* launches_saved, int64_t* bytes_saved);
/* infersim::canonical_layer_graph (fusion.hpp:242-357) partitioned in one call:
 * region_of[8] over the canonical nodes input_layernorm, qkv_gemm, attn_transpose,
 * attention, post_attn_layernorm, intermediate_gemm, bias_add, residual_add. */
int dsinf_canonical_layer_partition(int64_t hidden, int64_t batch, int32_t dtype_bytes,
                                    int32_t regime, int32_t region_of[8], int32_t* num_regions,
                                    int64_t* launches_saved, int64_t* bytes_saved);

/* infersim::canonical_layer_graph (fusion.hpp:242-357) as a flattened graph.  Call once with
 * node_kind == NULL to get num_nodes / num_edges / num_deps / num_prods, then with buffers of
 * those sizes (dep_off: num_edges + 1, prod_off: num_deps + 1). */
typedef struct dsinf_graph_buffers {
  int32_t num_nodes, num_edges, num_deps, num_prods, dtype_bytes;
  int32_t* node_kind;
  int32_t* node_tile_count;
  int64_t* node_out_elems;
  int32_t* edge_from;
  int32_t* edge_to;
  int32_t* dep_off;
  int32_t* dep_consumer;
  int32_t* prod_off;
  int32_t* dep_prod;
} dsinf_graph_buffers;
int dsinf_canonical_layer_graph(int64_t hidden, int64_t batch, int32_t dtype_bytes,
                                dsinf_graph_buffers* out);

#ifdef __cplusplus
} /* extern "C" */
#endif
#endif /* DSINF_H_ */
