// Persistent decode-step kernel: one launch runs a whole decode step (embedding, every layer's
// Deep-Fusion regions, LM head and greedy argmax) for tensor-parallel degree 1, fp16 or INT8
// weight-only (W8A16) weights, on a static per-CTA schedule (step_kernel.cu).
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "ops.cuh"
#include "sbi_gemm.cuh"

namespace dsinf {
namespace step {

// Host description of one step; pointers are device pointers owned by the model.
struct StepDesc {
  int B = 1, L = 0, H = 1, d = 64, max_ctx = 0, V = 0, Vl = 0;
  bool int8 = false;  // int8 layer weights (then every layer GEMM must be W8A16: Params::a16)
  // per layer, in order: qkv (PRO_LN, EPI_QKV), attn-out (PRO_F16, EPI_RESID), up (PRO_LN,
  // EPI_GELU_F16), down (PRO_F16, EPI_RESID); then the LM head (PRO_LN, EPI_F32).  The LayerNorm
  // GEMMs read their row sums from ln_stats_in; the residual GEMMs (and the embedding) write the
  // next LayerNorm's into ln_stats_out (slots zeroed per step by the caller, as am_key).
  std::vector<gemm::Params> gemms;
  std::vector<ops::AttnParams> attn;  // per layer
  ops::EmbedParams embed{};
  float* logits = nullptr;
  int32_t* next_tok = nullptr;
  int32_t* hist = nullptr;
  int* pos = nullptr;
  unsigned long long* am_key = nullptr;  // [B] greedy-argmax keys, zeroed before every launch
};

class StepProgram {
 public:
  // Builds the phase table, per-CTA work segments and workspaces.  Throws ConfigError when the
  // shape is not supported by the persistent path (the caller falls back to per-kernel launches).
  void build(const StepDesc& desc);
  void launch(cudaStream_t s) const;
  // Replace the embedding descriptor (new prompt / prompt length) without rebuilding.
  void set_embed(const ops::EmbedParams& e);
  void release();
  ~StepProgram() { release(); }
  int grid() const { return grid_; }
  int stages() const { return stages_; }
  bool ready() const { return built_; }

 private:
  bool built_ = false;
  int grid_ = 0;
  int stages_ = 0;
  size_t smem_ = 0;
  int variant_ = 0;
  int n_phases_ = 0;
  size_t trace_len_ = 0;
  unsigned long long* trace_ptr_ = nullptr;

 public:
  // Phase timeline of the last step ([grid][phases][4] globaltimer ns) when DSINF_STEP_TRACE=1.
  size_t trace(unsigned long long* host, size_t len) const;
  int phases() const { return n_phases_; }

 private:
  void* prog_dev_ = nullptr;  // device copy of the kernel's program header
  std::vector<void*> allocs_;
  struct ProgHost;
  std::vector<uint8_t> prog_host_;
};

}  // namespace step
}  // namespace dsinf
