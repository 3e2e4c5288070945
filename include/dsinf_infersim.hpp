// C++ drop-in for the reference's decode-path operator API (header-only, over the C ABI).
//
// A caller of the reference library includes <infersim/gemm.hpp> / <infersim/model.hpp> and calls
// infersim::derive_schedule, infersim::pack_weights, infersim::exec_reference, ...  Including
// this header instead and aliasing the namespace (`namespace infersim = dsinf::infersim;`) keeps
// every name, argument meaning and exception type while the work runs in libdsinf.so on the B200:
//
//   reference (file:line)                       here
//   GemmShape / validate   gemm.hpp:28-40       GemmShape (validate throws ConfigError)
//   TilingMode             gemm.hpp:42          TilingMode
//   GemmSchedule           gemm.hpp:47-54       GemmSchedule
//   kOutputTileWidth       gemm.hpp:45          kOutputTileWidth()
//   cache_line_pack        gemm.hpp:57-60       cache_line_pack
//   derive_schedule        gemm.hpp:65-96       derive_schedule
//   PackedWeights          gemm.hpp:101-106     PackedWeights
//   packed_index           gemm.hpp:108-111     packed_index
//   pack_weights           gemm.hpp:113-130     pack_weights
//   unpack_weights         gemm.hpp:132-139     unpack_weights
//   exec_reference         gemm.hpp:147-202     exec (same signature; runs SBI-GeMM on the GPU)
//   DeviceSpec             hardware.hpp:36-69   DeviceSpec (peak map -> three dtype slots)
//   ModelConfig            model.hpp:42-64      ModelConfig (dense)
//   param_count/bytes      model.hpp:93-105     param_count / param_bytes
//   layer_flops            model.hpp:121-132    layer_flops
//   kv_cache_bytes         model.hpp:135-140    kv_cache_bytes
//   KernelCost/kernel_time costmodel.hpp:31-56  KernelCost / kernel_time
//   min_latency_bound      costmodel.hpp:113-125 min_latency_bound (flat topology arguments)
//   ConfigError/InfeasibleError errors.hpp:24-34  same names, rethrown from the ABI return codes
// plus the decode loop the reference only describes: DecoderSession (dsinf_model_*).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dsinf.h"

namespace dsinf {
namespace infersim {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InfeasibleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == DSINF_OK) return;
  const std::string msg = dsinf_last_error();
  if (rc == DSINF_ERR_CONFIG) throw ConfigError(msg);
  if (rc == DSINF_ERR_INFEASIBLE) throw InfeasibleError(msg);
  throw DeviceError(msg);
}

// ---------------------------------------------------------------- gemm.hpp
struct GemmShape {
  std::int64_t out_dim = 0;
  std::int64_t in_dim = 0;
  std::int64_t batch = 1;
  int dtype_bytes = 2;
  dsinf_gemm_shape c() const { return {out_dim, in_dim, batch, dtype_bytes}; }
  void validate() const {
    dsinf_device_spec d{};
    dsinf_b200_device_spec(&d);
    dsinf_gemm_schedule s{};
    const dsinf_gemm_shape cs = c();
    check(dsinf_derive_schedule(&cs, &d, &s));
  }
};

enum class TilingMode { oneD = DSINF_TILING_1D, twoD = DSINF_TILING_2D };

struct GemmSchedule {
  TilingMode mode = TilingMode::oneD;
  std::int64_t output_tiles = 1;
  std::int64_t input_tiles = 1;
  int warps_per_block = 1;
  int kernel_count = 1;
  int pack_M = 1;
  dsinf_gemm_schedule c() const {
    return {static_cast<int32_t>(mode), output_tiles, input_tiles, warps_per_block, kernel_count, pack_M};
  }
};

struct DeviceSpec {
  std::int64_t mem_bytes = 0;
  double mem_bw = 0.0;
  std::map<int, double> peak_flops_by_dtype;  // dtype_bytes -> FLOP/s (4, 2, 1 are carried)
  int sm_count = 0;
  double kernel_launch_overhead = 5e-6;
  dsinf_device_spec c() const {
    auto get = [&](int dt) {
      auto it = peak_flops_by_dtype.find(dt);
      return it == peak_flops_by_dtype.end() ? 0.0 : it->second;
    };
    return {mem_bytes, mem_bw, sm_count, kernel_launch_overhead, get(4), get(2), get(1)};
  }
  static DeviceSpec b200() {
    dsinf_device_spec d{};
    dsinf_b200_device_spec(&d);
    DeviceSpec s;
    s.mem_bytes = d.mem_bytes;
    s.mem_bw = d.mem_bw;
    s.sm_count = d.sm_count;
    s.kernel_launch_overhead = d.kernel_launch_overhead;
    s.peak_flops_by_dtype = {{4, d.peak_flops_fp32}, {2, d.peak_flops_fp16}, {1, d.peak_flops_int8}};
    return s;
  }
};

inline std::int64_t kOutputTileWidth() { return dsinf_output_tile_width(); }
inline int cache_line_pack(int dtype_bytes) { return dsinf_cache_line_pack(dtype_bytes); }

inline GemmSchedule derive_schedule(const GemmShape& shape, const DeviceSpec& device) {
  const dsinf_gemm_shape cs = shape.c();
  const dsinf_device_spec cd = device.c();
  dsinf_gemm_schedule s{};
  check(dsinf_derive_schedule(&cs, &cd, &s));
  GemmSchedule r;
  r.mode = static_cast<TilingMode>(s.mode);
  r.output_tiles = s.output_tiles;
  r.input_tiles = s.input_tiles;
  r.warps_per_block = s.warps_per_block;
  r.kernel_count = s.kernel_count;
  r.pack_M = s.pack_M;
  return r;
}

inline std::int64_t packed_index(std::int64_t n, std::int64_t k, std::int64_t out_dim, int pack_M) {
  return dsinf_packed_index(n, k, out_dim, pack_M);
}

struct PackedWeights {
  std::vector<double> data;
  GemmShape shape;
  int pack_M = 1;
  std::int64_t padded_in_dim = 0;
};

inline PackedWeights pack_weights(const std::vector<double>& matrix, const GemmShape& shape, int pack_M) {
  const dsinf_gemm_shape cs = shape.c();
  PackedWeights p;
  p.shape = shape;
  p.pack_M = pack_M;
  check(dsinf_pack_weights_f64(matrix.data(), static_cast<std::int64_t>(matrix.size()), &cs, pack_M, nullptr, 0,
                               &p.padded_in_dim));
  p.data.assign(static_cast<size_t>(shape.out_dim * p.padded_in_dim), 0.0);
  check(dsinf_pack_weights_f64(matrix.data(), static_cast<std::int64_t>(matrix.size()), &cs, pack_M, p.data.data(),
                               static_cast<std::int64_t>(p.data.size()), &p.padded_in_dim));
  return p;
}

inline std::vector<double> unpack_weights(const PackedWeights& packed) {
  const dsinf_gemm_shape cs = packed.shape.c();
  std::vector<double> m(static_cast<size_t>(packed.shape.out_dim * packed.shape.in_dim));
  check(dsinf_unpack_weights_f64(packed.data.data(), static_cast<std::int64_t>(packed.data.size()), &cs,
                                 packed.pack_M, m.data(), static_cast<std::int64_t>(m.size())));
  return m;
}

// exec_reference's signature, executed by SBI-GeMM on the current CUDA device.  compute_dtype
// DSINF_DT_F16 (fp16 operands, fp32 accumulation) or DSINF_DT_I8 (W8A8, int32 accumulation).
inline std::vector<double> exec(const PackedWeights& packed, const std::vector<double>& x, std::int64_t batch,
                                const GemmSchedule& schedule, int compute_dtype = DSINF_DT_F16) {
  const dsinf_gemm_shape cs = packed.shape.c();
  const dsinf_gemm_schedule sc = schedule.c();
  std::vector<double> out(static_cast<size_t>(batch * packed.shape.out_dim));
  check(dsinf_exec_device(packed.data.data(), static_cast<std::int64_t>(packed.data.size()), &cs, &sc, x.data(),
                          static_cast<std::int64_t>(x.size()), batch, compute_dtype, out.data(),
                          static_cast<std::int64_t>(out.size())));
  return out;
}

// ---------------------------------------------------------------- model.hpp (dense)
struct ModelConfig {
  std::string name;
  std::int64_t hidden_dim = 0;
  std::int64_t num_layers = 0;
  std::int64_t num_heads = 1;
  std::int64_t vocab_size = 50257;
  std::int64_t max_seq = 2048;
  int dtype_bytes = 2;
  dsinf_model_config c() const { return {hidden_dim, num_layers, num_heads, vocab_size, max_seq, dtype_bytes}; }
};

enum class Phase { prompt = DSINF_PHASE_PROMPT, generation = DSINF_PHASE_GENERATION };

struct SeqWorkload {
  std::int64_t batch = 1;
  std::int64_t prompt_len = 0;
  std::int64_t gen_tokens = 0;
};

inline std::int64_t param_count(const ModelConfig& cfg) {
  const dsinf_model_config c = cfg.c();
  std::int64_t v = 0;
  check(dsinf_param_count(&c, &v));
  return v;
}
inline std::int64_t param_bytes(const ModelConfig& cfg) {
  const dsinf_model_config c = cfg.c();
  std::int64_t v = 0;
  check(dsinf_param_bytes(&c, &v));
  return v;
}
inline double layer_flops(const ModelConfig& cfg, const SeqWorkload& w, Phase phase) {
  const dsinf_model_config c = cfg.c();
  double v = 0;
  check(dsinf_layer_flops(&c, w.batch, w.prompt_len, w.gen_tokens, static_cast<int32_t>(phase), &v));
  return v;
}
inline std::int64_t kv_cache_bytes(const ModelConfig& cfg, const SeqWorkload& w) {
  const dsinf_model_config c = cfg.c();
  std::int64_t v = 0;
  check(dsinf_kv_cache_bytes(&c, w.batch, w.prompt_len, w.gen_tokens, &v));
  return v;
}

// ---------------------------------------------------------------- costmodel.hpp
struct KernelCost {
  double compute_time = 0, memory_time = 0, launch_overhead = 0, total = 0;
  bool memory_bound = false;
};
inline KernelCost kernel_time(double flops, double bytes_moved, const DeviceSpec& device, int dtype_bytes,
                              std::int64_t fused_launches = 1, bool cuda_graph = false) {
  const dsinf_device_spec d = device.c();
  dsinf_kernel_cost k{};
  check(dsinf_kernel_time(flops, bytes_moved, &d, dtype_bytes, fused_launches, cuda_graph ? 1 : 0, &k));
  return {k.compute_time, k.memory_time, k.launch_overhead, k.total, k.memory_bound != 0};
}
inline double min_latency_bound(const ModelConfig& cfg, int tp, int pp, const dsinf_topology& topo) {
  const dsinf_model_config c = cfg.c();
  double v = 0;
  check(dsinf_min_latency_bound(&c, tp, pp, &topo, &v));
  return v;
}

// ---------------------------------------------------------------- the decode loop (new)
// Owns the device weights, KV cache and step graph of one model replica / TP rank.
class DecoderSession {
 public:
  DecoderSession(const ModelConfig& cfg, const dsinf_runtime_config& rt, void* nccl_comm = nullptr) {
    const dsinf_model_config c = cfg.c();
    check(dsinf_model_create(&c, &rt, nccl_comm, &m_));
  }
  ~DecoderSession() {
    if (m_) dsinf_model_destroy(m_);
  }
  DecoderSession(const DecoderSession&) = delete;
  DecoderSession& operator=(const DecoderSession&) = delete;
  DecoderSession(DecoderSession&& o) noexcept : m_(std::exchange(o.m_, nullptr)) {}

  // prompts: host int32 [B][prompt_len]
  void set_prompt(const std::vector<std::int32_t>& prompts, std::int64_t prompt_len, void* stream = nullptr) {
    check(dsinf_model_set_prompt(m_, prompts.data(), prompt_len, stream));
  }
  void step(std::int64_t n = 1, void* stream = nullptr) { check(dsinf_decode_steps(m_, n, stream)); }
  // the whole prompt at once on the tensor cores (same resulting state as step(prompt_len))
  void prefill(void* stream = nullptr) { check(dsinf_model_prefill(m_, stream)); }
  // one step with host buffers: tokens_in -> the model -> tokens_out (synchronous)
  void step_host(const std::int32_t* tokens_in, std::int32_t* tokens_out, void* stream = nullptr) {
    check(dsinf_decode_step_host(m_, tokens_in, tokens_out, stream));
  }
  dsinf_model_info info() const {
    dsinf_model_info i{};
    check(dsinf_model_get_info(m_, &i));
    return i;
  }
  dsinf_model* handle() const { return m_; }

 private:
  dsinf_model* m_ = nullptr;
};

}  // namespace infersim
}  // namespace dsinf
