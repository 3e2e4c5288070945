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
//   exec_reference         gemm.hpp:147-202     exec_reference / exec (same signature; SBI-GeMM on the GPU)
//   DeviceSpec             hardware.hpp:36-69   DeviceSpec (peak map -> three dtype slots)
//   ModelConfig            model.hpp:42-64      ModelConfig (dense)
//   param_count/bytes      model.hpp:93-105     param_count / param_bytes
//   layer_flops            model.hpp:121-132    layer_flops
//   kv_cache_bytes         model.hpp:135-140    kv_cache_bytes
//   KernelCost/kernel_time costmodel.hpp:31-56  KernelCost / kernel_time
//   min_latency_bound      costmodel.hpp:113-125 min_latency_bound (flat topology arguments)
//   CollectiveKind/collective_time costmodel.hpp:40,70-104  same (LinkSpec / Topology: the fields it reads)
//   OpKind/OpNode/GraphEdge/OpGraph fusion.hpp:29-116  same (dims carried as names only)
//   fusable / BatchRegime / partition_layer fusion.hpp:126-173  same
//   FusionRegion / FusionSavings / fusion_savings fusion.hpp:118-215  same
//   canonical_layer_graph  fusion.hpp:242-357   same (built by the library)
//   ConfigError/InfeasibleError errors.hpp:24-34  same names, rethrown from the ABI return codes
// plus the decode loop the reference only describes: DecoderSession (dsinf_model_*).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <set>
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
  check(dsinf_exec_device(packed.data.data(), static_cast<std::int64_t>(packed.data.size()), packed.pack_M, &cs, &sc, x.data(),
                          static_cast<std::int64_t>(x.size()), batch, compute_dtype, out.data(),
                          static_cast<std::int64_t>(out.size())));
  return out;
}

// The reference's name for the same call (gemm.hpp:147): a caller can keep writing exec_reference.
inline std::vector<double> exec_reference(const PackedWeights& packed, const std::vector<double>& x,
                                          std::int64_t batch, const GemmSchedule& schedule) {
  return exec(packed, x, batch, schedule);
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

enum class CollectiveKind {  // costmodel.hpp:40
  allreduce = DSINF_COLL_ALLREDUCE,
  allgather = DSINF_COLL_ALLGATHER,
  alltoall = DSINF_COLL_ALLTOALL,
  broadcast = DSINF_COLL_BROADCAST,
  p2p = DSINF_COLL_P2P
};
struct LinkSpec {  // hardware.hpp:30-34
  double bandwidth = 0.0;
  double latency = 0.0;
};
struct Topology {  // the fields of hardware.hpp:80-123 collective_time and min_latency_bound read
  int num_nodes = 1;
  int gpus_per_node = 1;
  DeviceSpec device;
  LinkSpec intra, inter;
  int device_count() const { return num_nodes * gpus_per_node; }
  dsinf_topology c() const {
    return {num_nodes, gpus_per_node, {intra.bandwidth, intra.latency}, {inter.bandwidth, inter.latency}, device.c()};
  }
};
inline double collective_time(CollectiveKind kind, double bytes_per_rank, const std::vector<int>& group,
                              const Topology& topo) {
  const std::vector<std::int32_t> g(group.begin(), group.end());
  const dsinf_topology t = topo.c();
  double v = 0;
  check(dsinf_collective_time(static_cast<std::int32_t>(kind), bytes_per_rank, g.data(),
                              static_cast<std::int32_t>(g.size()), &t, &v));
  return v;
}
inline double min_latency_bound(const ModelConfig& cfg, int tp, int pp, const Topology& topo) {
  return min_latency_bound(cfg, tp, pp, topo.c());
}

// ---------------------------------------------------------------- fusion.hpp (Deep-Fusion)
enum class OpKind {  // fusion.hpp:29
  elementwise = DSINF_OP_ELEMENTWISE,
  reduction = DSINF_OP_REDUCTION,
  transpose = DSINF_OP_TRANSPOSE,
  gemm = DSINF_OP_GEMM,
  quantize = DSINF_OP_QUANTIZE
};
enum class BatchRegime { small_batch = DSINF_REGIME_SMALL_BATCH, large_batch = DSINF_REGIME_LARGE_BATCH };

struct OpNode {  // fusion.hpp:39-65; legality depends on the tile structure only
  std::string name;
  OpKind kind = OpKind::elementwise;
  std::int64_t out_elems = 0;
  int tile_count = 1;
};
struct GraphEdge {  // fusion.hpp:68-72
  int from = -1;
  int to = -1;
  std::map<int, std::set<int>> tile_dep;  // consumer tile -> producer tiles
};
struct OpGraph {  // fusion.hpp:74-116
  std::vector<OpNode> nodes;
  std::vector<GraphEdge> edges;
  int dtype_bytes = 2;
  std::int64_t edge_bytes(const GraphEdge& e) const { return nodes[e.from].out_elems * dtype_bytes; }
};
struct FusionRegion {  // fusion.hpp:118-121
  std::vector<int> node_ids;
  int launch_count = 1;
};
struct FusionSavings {  // fusion.hpp:175-178
  std::int64_t launches_saved = 0;
  std::int64_t bytes_saved = 0;
};

namespace detail {
// Keeps the flattened (CSR) image of an OpGraph alive for one C-ABI call.
struct FlatGraph {
  std::vector<std::int32_t> kind, tiles, from, to, dep_off{0}, cons, prod_off{0}, prod;
  std::vector<std::int64_t> elems;
  dsinf_op_graph c{};
  explicit FlatGraph(const OpGraph& g) {
    for (const auto& n : g.nodes) {
      kind.push_back(static_cast<std::int32_t>(n.kind));
      tiles.push_back(n.tile_count);
      elems.push_back(n.out_elems);
    }
    for (const auto& e : g.edges) {
      from.push_back(e.from);
      to.push_back(e.to);
      for (const auto& [ct, ps] : e.tile_dep) {
        cons.push_back(ct);
        for (int p : ps) prod.push_back(p);
        prod_off.push_back(static_cast<std::int32_t>(prod.size()));
      }
      dep_off.push_back(static_cast<std::int32_t>(cons.size()));
    }
    c = {static_cast<std::int32_t>(g.nodes.size()), kind.data(), tiles.data(), elems.data(),
         static_cast<std::int32_t>(g.edges.size()), from.data(), to.data(), dep_off.data(), cons.data(),
         prod_off.data(), prod.data(), g.dtype_bytes};
  }
};
}  // namespace detail

inline bool fusable(const OpGraph& graph, const GraphEdge& edge) {  // fusion.hpp:126-133
  OpGraph one{graph.nodes, {edge}, graph.dtype_bytes};
  detail::FlatGraph fg(one);
  std::int32_t out = 0;
  check(dsinf_fusable(&fg.c, 0, &out));
  return out != 0;
}
inline std::vector<FusionRegion> partition_layer(const OpGraph& graph, BatchRegime regime) {  // fusion.hpp:140-173
  detail::FlatGraph fg(graph);
  std::vector<std::int32_t> region_of(std::max<size_t>(1, graph.nodes.size()));
  std::int32_t nreg = 0;
  check(dsinf_partition_layer(&fg.c, static_cast<std::int32_t>(regime), region_of.data(), &nreg));
  std::vector<FusionRegion> regions(static_cast<size_t>(nreg));
  for (size_t i = 0; i < graph.nodes.size(); ++i) regions[region_of[i]].node_ids.push_back(static_cast<int>(i));
  return regions;
}
inline FusionSavings fusion_savings(const std::vector<FusionRegion>& regions, const OpGraph& graph) {  // :183-215
  std::vector<std::int32_t> region_of(graph.nodes.size(), -1);
  size_t covered = 0;
  for (size_t r = 0; r < regions.size(); ++r)
    for (int id : regions[r].node_ids) {
      if (id < 0 || id >= static_cast<int>(graph.nodes.size()) || region_of[id] != -1)
        throw ConfigError("regions must partition the graph");
      region_of[id] = static_cast<std::int32_t>(r);
      ++covered;
    }
  if (covered != graph.nodes.size()) throw ConfigError("regions must cover every node");
  detail::FlatGraph fg(graph);
  FusionSavings s;
  check(dsinf_fusion_savings(&fg.c, region_of.data(), static_cast<std::int32_t>(regions.size()), &s.launches_saved,
                             &s.bytes_saved));
  return s;
}
inline OpGraph canonical_layer_graph(std::int64_t hidden, std::int64_t batch, int dtype_bytes = 2) {  // :242-357
  static const char* const kNames[] = {"input_layernorm", "qkv_gemm", "attn_transpose", "attention",
                                       "post_attn_layernorm", "intermediate_gemm", "bias_add", "residual_add"};
  dsinf_graph_buffers gb{};
  check(dsinf_canonical_layer_graph(hidden, batch, dtype_bytes, &gb));
  std::vector<std::int32_t> kind(gb.num_nodes), tiles(gb.num_nodes), from(gb.num_edges), to(gb.num_edges),
      dep_off(gb.num_edges + 1), cons(std::max(1, gb.num_deps)), prod_off(gb.num_deps + 1),
      prod(std::max(1, gb.num_prods));
  std::vector<std::int64_t> elems(gb.num_nodes);
  gb.node_kind = kind.data();
  gb.node_tile_count = tiles.data();
  gb.node_out_elems = elems.data();
  gb.edge_from = from.data();
  gb.edge_to = to.data();
  gb.dep_off = dep_off.data();
  gb.dep_consumer = cons.data();
  gb.prod_off = prod_off.data();
  gb.dep_prod = prod.data();
  check(dsinf_canonical_layer_graph(hidden, batch, dtype_bytes, &gb));
  OpGraph g;
  g.dtype_bytes = gb.dtype_bytes;
  for (int i = 0; i < gb.num_nodes; ++i)
    g.nodes.push_back({i < 8 ? kNames[i] : "node", static_cast<OpKind>(kind[i]), elems[i], tiles[i]});
  for (int e = 0; e < gb.num_edges; ++e) {
    GraphEdge ge;
    ge.from = from[e];
    ge.to = to[e];
    for (int c = dep_off[e]; c < dep_off[e + 1]; ++c)
      ge.tile_dep[cons[c]] = std::set<int>(prod.begin() + prod_off[c], prod.begin() + prod_off[c + 1]);
    g.edges.push_back(std::move(ge));
  }
  return g;
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
