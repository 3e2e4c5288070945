// Host-side operator API of the decode hot path: the SBI-GeMM schedule and the packed weight
// layout (gemm.hpp), the layer accounting (model.hpp), the roofline / collective cost model
// (costmodel.hpp) and the Deep-Fusion partition (fusion.hpp).  Every function is a fresh
// implementation of the reference contract cited beside it; tests/test_host_parity.py checks
// each one against the reference headers compiled into oracle/_ref.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "common.h"

namespace dsinf {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// ------------------------------------------------------------------ gemm.hpp

// GemmShape::validate (gemm.hpp:34-40)
static void validate_shape(const dsinf_gemm_shape& s) {
  if (s.out_dim < 1 || s.in_dim < 1 || s.batch < 1)
    throw ConfigError("gemm shape dims must be positive");
  if (s.dtype_bytes != 1 && s.dtype_bytes != 2 && s.dtype_bytes != 4)
    throw ConfigError("dtype_bytes must be one of {1, 2, 4}");
}

// cache_line_pack (gemm.hpp:57-60): elements per lane that fill a 128-byte line across a warp.
static int32_t line_pack(int32_t dtype_bytes) {
  if (dtype_bytes <= 0) return 4;
  const int32_t m = 128 / (32 * dtype_bytes);
  return std::min(4, std::max(1, m));
}

static constexpr int64_t kTileWidth = 32;  // gemm.hpp:45

// derive_schedule (gemm.hpp:65-96).  The batch never enters the decision; the device spec is
// not validated, both as in the reference.
static dsinf_gemm_schedule schedule_for(const dsinf_gemm_shape& shape, const dsinf_device_spec& dev) {
  validate_shape(shape);
  dsinf_gemm_schedule s{};
  s.pack_M = line_pack(shape.dtype_bytes);
  s.output_tiles = (shape.out_dim + kTileWidth - 1) / kTileWidth;
  const int64_t groups = (shape.in_dim + s.pack_M - 1) / s.pack_M;
  s.warps_per_block = static_cast<int32_t>(std::min<int64_t>(8, std::max<int64_t>(1, groups / kTileWidth)));
  s.mode = DSINF_TILING_1D;
  s.input_tiles = 1;
  s.kernel_count = 1;
  if (s.output_tiles >= dev.sm_count) return s;
  int64_t split = 1;
  while (s.output_tiles * split < dev.sm_count && split * 2 <= groups) split <<= 1;
  if (split > 1) {
    s.mode = DSINF_TILING_2D;
    s.input_tiles = split;
    s.kernel_count = 2;
  }
  return s;
}

static int64_t pidx(int64_t n, int64_t k, int64_t N, int32_t M) {
  return (k / M) * (N * M) + n * M + (k % M);  // [K/M][N][M], gemm.hpp:108-111
}

static void check_pack_m(int32_t m) {
  if (m != 1 && m != 2 && m != 4) throw ConfigError("pack_M must be one of {1, 2, 4}");
}

// ------------------------------------------------------------------ model.hpp

static void validate_model(const dsinf_model_config& c) {  // ModelConfig::validate (:52-63)
  if (c.hidden_dim < 1) throw ConfigError("hidden_dim must be positive");
  if (c.num_layers < 0) throw ConfigError("num_layers must be non-negative");
  if (c.num_heads < 1) throw ConfigError("num_heads must be positive");
  if (c.vocab_size < 0) throw ConfigError("vocab_size must be non-negative");
  if (c.max_seq < 1) throw ConfigError("max_seq must be positive");
  if (c.dtype_bytes != 1 && c.dtype_bytes != 2 && c.dtype_bytes != 4)
    throw ConfigError("dtype_bytes must be one of {1, 2, 4}");
  if (c.hidden_dim % c.num_heads != 0)
    throw ConfigError("hidden_dim must be divisible by num_heads");
}

static int64_t params_of(const dsinf_model_config& c) {  // param_count (:93-101), dense
  validate_model(c);
  const int64_t h = c.hidden_dim;
  return 12 * h * h * c.num_layers + c.vocab_size * h;
}

// ------------------------------------------------------------------ costmodel.hpp

static double peak_of(const dsinf_device_spec& d, int dtype_bytes) {  // DeviceSpec::peak_flops
  double v = 0.0;
  if (dtype_bytes == 4) v = d.peak_flops_fp32;
  if (dtype_bytes == 2) v = d.peak_flops_fp16;
  if (dtype_bytes == 1) v = d.peak_flops_int8;
  if (!(v > 0.0))
    throw ConfigError("no peak FLOPs entry for dtype_bytes=" + std::to_string(dtype_bytes));
  return v;
}

// ------------------------------------------------------------------ fusion.hpp

struct Graph {
  std::vector<int32_t> kind, tiles;
  std::vector<int64_t> out_elems;
  struct Edge {
    int32_t from, to;
    std::map<int, std::set<int>> dep;
  };
  std::vector<Edge> edges;
  int32_t dtype_bytes = 2;
};

static Graph graph_from_c(const dsinf_op_graph& g) {
  Graph out;
  if (g.num_nodes < 0 || g.num_edges < 0) throw ConfigError("negative graph sizes");
  out.dtype_bytes = g.dtype_bytes;
  for (int i = 0; i < g.num_nodes; ++i) {
    out.kind.push_back(g.node_kind[i]);
    out.tiles.push_back(g.node_tile_count[i]);
    out.out_elems.push_back(g.node_out_elems[i]);
  }
  for (int e = 0; e < g.num_edges; ++e) {
    Graph::Edge ed{g.edge_from[e], g.edge_to[e], {}};
    for (int32_t i = g.dep_off[e]; i < g.dep_off[e + 1]; ++i) {
      auto& set = ed.dep[g.dep_consumer[i]];
      for (int32_t j = g.prod_off[i]; j < g.prod_off[i + 1]; ++j) set.insert(g.dep_prod[j]);
    }
    out.edges.push_back(std::move(ed));
  }
  return out;
}

// OpNode::validate / OpGraph::validate (fusion.hpp:51-115); the dim-name checks of OpNode do
// not apply to the flattened graph (it carries no dim names).
static void validate_graph(const Graph& g) {
  const int n = static_cast<int>(g.kind.size());
  for (int i = 0; i < n; ++i) {
    if (g.tiles[i] < 1) throw ConfigError("node " + std::to_string(i) + ": tile_count must be >= 1");
    if (g.out_elems[i] < 0) throw ConfigError("node " + std::to_string(i) + ": negative out_elems");
  }
  for (const auto& e : g.edges) {
    if (e.from < 0 || e.to < 0 || e.from >= n || e.to >= n) throw ConfigError("edge references unknown node");
    if (e.from >= e.to) throw ConfigError("nodes must be listed in topological order");
    for (const auto& [c, prods] : e.dep) {
      if (c < 0 || c >= g.tiles[e.to]) throw ConfigError("tile_dep consumer tile out of range");
      for (int p : prods)
        if (p < 0 || p >= g.tiles[e.from]) throw ConfigError("tile_dep producer tile out of range");
    }
  }
}

// fusable (fusion.hpp:126-133): every consumer tile has exactly one producer tile.
static bool edge_fusable(const Graph& g, const Graph::Edge& e) {
  for (int t = 0; t < g.tiles[e.to]; ++t) {
    auto it = e.dep.find(t);
    if (it == e.dep.end() || it->second.size() != 1) return false;
  }
  return true;
}

// partition_layer (fusion.hpp:140-173): greedy maximal fusable runs in topological order;
// in the large-batch regime a GEMM neither joins nor extends a region.
static std::vector<std::vector<int>> partition(const Graph& g, int regime) {
  validate_graph(g);
  std::vector<std::vector<int>> regions;
  const int n = static_cast<int>(g.kind.size());
  const bool large = regime == DSINF_REGIME_LARGE_BATCH;
  for (int v = 0; v < n; ++v) {
    bool joined = false;
    const bool isolate = large && g.kind[v] == DSINF_OP_GEMM;
    if (!regions.empty() && !isolate) {
      auto& cur = regions.back();
      bool cur_gemm = false;
      if (large)
        for (int id : cur) cur_gemm |= g.kind[id] == DSINF_OP_GEMM;
      bool touches = false, ok = true;
      for (const auto& e : g.edges) {
        if (e.to != v) continue;
        if (std::find(cur.begin(), cur.end(), e.from) == cur.end()) continue;
        touches = true;
        ok = ok && edge_fusable(g, e);
      }
      if (touches && ok && !cur_gemm) {
        cur.push_back(v);
        joined = true;
      }
    }
    if (!joined) regions.push_back({v});
  }
  return regions;
}

// fusion_savings (fusion.hpp:183-215)
static void savings(const Graph& g, const std::vector<int32_t>& region_of, int64_t* launches,
                    int64_t* bytes) {
  const int n = static_cast<int>(g.kind.size());
  std::set<int32_t> distinct(region_of.begin(), region_of.end());
  *launches = n - static_cast<int64_t>(distinct.size());
  int64_t b = 0;
  for (const auto& e : g.edges)
    if (region_of[e.from] == region_of[e.to]) b += g.out_elems[e.from] * g.dtype_bytes;
  for (int v = 0; v < n; ++v) {
    bool has_out = false, internal = true;
    for (const auto& e : g.edges)
      if (e.from == v) {
        has_out = true;
        internal = internal && region_of[e.to] == region_of[v];
      }
    if (has_out && internal) b += g.out_elems[v] * g.dtype_bytes;
  }
  *bytes = b;
}

// canonical_layer_graph (fusion.hpp:242-357): the decode layer as 8 micro-ops on abstract
// 2x2x2 tile grids (token x out-block x in-block for GEMMs, token x head for attention).
static Graph canonical_graph(int64_t hidden, int64_t batch, int32_t dtype_bytes) {
  if (hidden < 1 || batch < 1) throw ConfigError("canonical layer requires positive hidden and batch");
  constexpr int T = 2, HT = 2, OB = 2, IB = 2;
  auto gemm_tile = [](int tt, int ob, int ib) { return (tt * OB + ob) * IB + ib; };
  auto head_tile = [](int tt, int ht) { return tt * HT + ht; };
  auto col_tile = [](int tt, int ob) { return tt * OB + ob; };
  Graph g;
  g.dtype_bytes = dtype_bytes;
  auto node = [&](int kind, int64_t elems, int tiles) {
    g.kind.push_back(kind);
    g.out_elems.push_back(elems);
    g.tiles.push_back(tiles);
    return static_cast<int>(g.kind.size()) - 1;
  };
  const int ln1 = node(DSINF_OP_REDUCTION, batch * hidden, T);
  const int qkv = node(DSINF_OP_GEMM, batch * 3 * hidden, T * OB * IB);
  const int tr = node(DSINF_OP_TRANSPOSE, batch * 3 * hidden, T * HT);
  const int att = node(DSINF_OP_REDUCTION, batch * hidden, T * HT);
  const int ln2 = node(DSINF_OP_REDUCTION, batch * hidden, T);
  const int ff = node(DSINF_OP_GEMM, batch * 4 * hidden, T * OB * IB);
  const int bias = node(DSINF_OP_ELEMENTWISE, batch * 4 * hidden, T * OB);
  const int res = node(DSINF_OP_ELEMENTWISE, batch * 4 * hidden, T * OB);
  auto edge = [&](int a, int b) -> Graph::Edge& {
    g.edges.push_back({a, b, {}});
    return g.edges.back();
  };
  {  // broadcast LN output feeds every GEMM tile of the same token tile
    auto& e = edge(ln1, qkv);
    for (int tt = 0; tt < T; ++tt)
      for (int ob = 0; ob < OB; ++ob)
        for (int ib = 0; ib < IB; ++ib) e.dep[gemm_tile(tt, ob, ib)] = {tt};
  }
  {  // head tile waits on all input-block partials of its column block
    auto& e = edge(qkv, tr);
    for (int tt = 0; tt < T; ++tt)
      for (int ht = 0; ht < HT; ++ht)
        for (int ib = 0; ib < IB; ++ib) e.dep[head_tile(tt, ht)].insert(gemm_tile(tt, ht, ib));
  }
  {
    auto& e = edge(tr, att);
    for (int t = 0; t < T * HT; ++t) e.dep[t] = {t};
  }
  {  // a token's LN needs every head
    auto& e = edge(att, ln2);
    for (int tt = 0; tt < T; ++tt)
      for (int ht = 0; ht < HT; ++ht) e.dep[tt].insert(head_tile(tt, ht));
  }
  {
    auto& e = edge(ln2, ff);
    for (int tt = 0; tt < T; ++tt)
      for (int ob = 0; ob < OB; ++ob)
        for (int ib = 0; ib < IB; ++ib) e.dep[gemm_tile(tt, ob, ib)] = {tt};
  }
  {
    auto& e = edge(ff, bias);
    for (int tt = 0; tt < T; ++tt)
      for (int ob = 0; ob < OB; ++ob)
        for (int ib = 0; ib < IB; ++ib) e.dep[col_tile(tt, ob)].insert(gemm_tile(tt, ob, ib));
  }
  {
    auto& e = edge(bias, res);
    for (int t = 0; t < T * OB; ++t) e.dep[t] = {t};
  }
  validate_graph(g);
  return g;
}

}  // namespace dsinf

using namespace dsinf;

extern "C" {

const char* dsinf_last_error(void) { return g_last_error.c_str(); }
const char* dsinf_version(void) { return "dsinf-b200 0.1 (sm_100a)"; }

void dsinf_b200_device_spec(dsinf_device_spec* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->mem_bytes = 183359LL * 1024 * 1024;  // nvidia-smi total on B200
  out->mem_bw = 8.0e12;                     // nominal; benches use MEASURED_PEAKS.json
  out->sm_count = 148;
  out->kernel_launch_overhead = 5e-6;       // reference default (hardware.hpp:41)
  out->peak_flops_fp32 = 80e12;
  out->peak_flops_fp16 = 2.25e15;
  out->peak_flops_int8 = 4.5e15;
}

int64_t dsinf_output_tile_width(void) { return kTileWidth; }
int32_t dsinf_cache_line_pack(int32_t dtype_bytes) { return line_pack(dtype_bytes); }

int dsinf_derive_schedule(const dsinf_gemm_shape* shape, const dsinf_device_spec* device,
                          dsinf_gemm_schedule* out) {
  return guarded([&] {
    require(shape && device && out, "null argument");
    *out = schedule_for(*shape, *device);
  });
}

int64_t dsinf_packed_index(int64_t n, int64_t k, int64_t out_dim, int32_t pack_M) {
  return pidx(n, k, out_dim, pack_M);
}

int dsinf_pack_weights_f64(const double* matrix, int64_t matrix_len, const dsinf_gemm_shape* shape,
                           int32_t pack_M, double* packed, int64_t packed_len,
                           int64_t* padded_in_dim) {
  return guarded([&] {
    require(shape != nullptr, "null shape");
    validate_shape(*shape);  // pack_weights validates first (gemm.hpp:115)
    check_pack_m(pack_M);
    if (matrix_len != shape->out_dim * shape->in_dim)
      throw ConfigError("weight matrix size does not match shape");
    const int64_t kp = (shape->in_dim + pack_M - 1) / pack_M * pack_M;
    if (padded_in_dim) *padded_in_dim = kp;
    if (!packed) return;  // size query
    if (packed_len != shape->out_dim * kp) throw ConfigError("packed buffer size mismatch");
    require(matrix != nullptr, "null matrix");
    std::fill(packed, packed + packed_len, 0.0);  // the K pad stays zero
    const int64_t N = shape->out_dim, K = shape->in_dim;
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < K; ++k) packed[pidx(n, k, N, pack_M)] = matrix[n * K + k];
  });
}

int dsinf_unpack_weights_f64(const double* packed, int64_t packed_len,
                             const dsinf_gemm_shape* shape, int32_t pack_M, double* matrix,
                             int64_t matrix_len) {
  return guarded([&] {
    require(shape && packed && matrix, "null argument");
    check_pack_m(pack_M);
    const int64_t N = shape->out_dim, K = shape->in_dim;
    const int64_t kp = (K + pack_M - 1) / pack_M * pack_M;
    if (packed_len != N * kp || matrix_len != N * K) throw ConfigError("buffer size mismatch");
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < K; ++k) matrix[n * K + k] = packed[pidx(n, k, N, pack_M)];
  });
}

int dsinf_param_count(const dsinf_model_config* cfg, int64_t* out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    *out = params_of(*cfg);
  });
}

int dsinf_param_bytes(const dsinf_model_config* cfg, int64_t* out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    *out = params_of(*cfg) * cfg->dtype_bytes;
  });
}

int dsinf_layer_flops(const dsinf_model_config* cfg, int64_t batch, int64_t prompt_len,
                      int64_t gen_tokens, int32_t phase, double* out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    validate_model(*cfg);
    const double h = static_cast<double>(cfg->hidden_dim);
    const double b = static_cast<double>(batch);
    if (phase == DSINF_PHASE_PROMPT) {
      const double s = static_cast<double>(prompt_len);
      *out = 24.0 * h * h * b * s + 4.0 * b * s * s * h;
    } else {
      const double ctx = static_cast<double>(prompt_len + gen_tokens);
      *out = 24.0 * h * h * b + 4.0 * b * ctx * h;
    }
  });
}

int dsinf_kv_cache_bytes(const dsinf_model_config* cfg, int64_t batch, int64_t prompt_len,
                         int64_t gen_tokens, int64_t* out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    validate_model(*cfg);
    *out = 2 * cfg->num_layers * batch * (prompt_len + gen_tokens) * cfg->hidden_dim *
           cfg->dtype_bytes;
  });
}

int dsinf_kernel_time(double flops, double bytes_moved, const dsinf_device_spec* device,
                      int32_t dtype_bytes, int64_t fused_launches, int32_t cuda_graph,
                      dsinf_kernel_cost* out) {
  return guarded([&] {
    require(device && out, "null argument");
    if (flops < 0.0 || bytes_moved < 0.0 || fused_launches < 1)
      throw ConfigError("kernel_time: negative work or zero launches");
    dsinf_kernel_cost c{};
    c.compute_time = flops > 0.0 ? flops / peak_of(*device, dtype_bytes) : 0.0;
    c.memory_time = bytes_moved / device->mem_bw;
    c.launch_overhead = cuda_graph ? 0.0 : fused_launches * device->kernel_launch_overhead;
    c.total = std::max(c.compute_time, c.memory_time) + c.launch_overhead;
    c.memory_bound = c.memory_time >= c.compute_time;
    *out = c;
  });
}

int dsinf_collective_time(int32_t kind, double bytes_per_rank, const int32_t* group,
                          int32_t group_size, const dsinf_topology* topo, double* out) {
  return guarded([&] {
    require(topo && out, "null argument");
    if (group_size <= 0 || !group) throw ConfigError("collective over empty group");
    if (bytes_per_rank < 0.0) throw ConfigError("negative payload");
    const int devices = topo->num_nodes * topo->gpus_per_node;
    for (int i = 0; i < group_size; ++i)
      if (group[i] < 0 || group[i] >= devices)
        throw ConfigError("unknown device id " + std::to_string(group[i]));
    if (group_size == 1) {
      *out = 0.0;
      return;
    }
    // group_link (costmodel.hpp:60-66): inter-node link if the group spans nodes.
    const int node0 = group[0] / topo->gpus_per_node;
    bool spans = false;
    for (int i = 0; i < group_size; ++i) spans |= group[i] / topo->gpus_per_node != node0;
    const dsinf_link_spec& link = spans ? topo->inter : topo->intra;
    const double n = group_size, bw = link.bandwidth, lat = link.latency;
    switch (kind) {
      case DSINF_COLL_ALLREDUCE: *out = 2.0 * (n - 1.0) / n * bytes_per_rank / bw + (n - 1.0) * lat; break;
      case DSINF_COLL_ALLGATHER: *out = (n - 1.0) / n * bytes_per_rank / bw + (n - 1.0) * lat; break;
      case DSINF_COLL_ALLTOALL: *out = (n - 1.0) * (bytes_per_rank / n) / bw + (n - 1.0) * lat; break;
      case DSINF_COLL_BROADCAST: *out = bytes_per_rank / bw + (n - 1.0) * lat; break;
      case DSINF_COLL_P2P: *out = bytes_per_rank / bw + lat; break;
      default: throw ConfigError("unknown collective kind");
    }
  });
}

int dsinf_min_latency_bound(const dsinf_model_config* cfg, int32_t tp, int32_t pp,
                            const dsinf_topology* topo, double* out) {
  return guarded([&] {
    require(cfg && topo && out, "null argument");
    if (tp < 1 || pp < 1) throw ConfigError("parallel degrees must be >= 1");
    const double per_dev = static_cast<double>(params_of(*cfg) * cfg->dtype_bytes) / (tp * pp);
    if (per_dev > static_cast<double>(topo->device.mem_bytes))
      throw InfeasibleError("plan does not fit: " + std::to_string(per_dev) + " bytes per device");
    *out = per_dev / topo->device.mem_bw;
  });
}

int dsinf_fusable(const dsinf_op_graph* g, int32_t edge, int32_t* out) {
  return guarded([&] {
    require(g && out, "null argument");
    Graph gr = graph_from_c(*g);
    if (edge < 0 || edge >= static_cast<int>(gr.edges.size())) throw ConfigError("edge out of range");
    const auto& e = gr.edges[edge];
    if (e.to < 0 || e.to >= static_cast<int>(gr.kind.size())) throw ConfigError("edge references unknown node");
    *out = edge_fusable(gr, e) ? 1 : 0;
  });
}

int dsinf_partition_layer(const dsinf_op_graph* g, int32_t regime, int32_t* region_of,
                          int32_t* num_regions) {
  return guarded([&] {
    require(g && region_of && num_regions, "null argument");
    const auto regions = partition(graph_from_c(*g), regime);
    for (size_t r = 0; r < regions.size(); ++r)
      for (int id : regions[r]) region_of[id] = static_cast<int32_t>(r);
    *num_regions = static_cast<int32_t>(regions.size());
  });
}

int dsinf_fusion_savings(const dsinf_op_graph* g, const int32_t* region_of, int32_t num_regions,
                         int64_t* launches_saved, int64_t* bytes_saved) {
  return guarded([&] {
    require(g && region_of && launches_saved && bytes_saved, "null argument");
    Graph gr = graph_from_c(*g);
    std::vector<int32_t> ro(region_of, region_of + gr.kind.size());
    for (int32_t r : ro)
      if (r < 0 || r >= num_regions) throw ConfigError("regions must partition the graph");
    std::set<int32_t> used(ro.begin(), ro.end());
    if (static_cast<int32_t>(used.size()) != num_regions) throw ConfigError("regions must cover every node");
    savings(gr, ro, launches_saved, bytes_saved);
  });
}

int dsinf_canonical_layer_partition(int64_t hidden, int64_t batch, int32_t dtype_bytes,
                                    int32_t regime, int32_t region_of[8], int32_t* num_regions,
                                    int64_t* launches_saved, int64_t* bytes_saved) {
  return guarded([&] {
    require(region_of && num_regions, "null argument");
    Graph g = canonical_graph(hidden, batch, dtype_bytes);
    const auto regions = partition(g, regime);
    std::vector<int32_t> ro(g.kind.size());
    for (size_t r = 0; r < regions.size(); ++r)
      for (int id : regions[r]) ro[id] = static_cast<int32_t>(r);
    for (int i = 0; i < 8; ++i) region_of[i] = ro[i];
    *num_regions = static_cast<int32_t>(regions.size());
    int64_t l = 0, b = 0;
    savings(g, ro, &l, &b);
    if (launches_saved) *launches_saved = l;
    if (bytes_saved) *bytes_saved = b;
  });
}

// canonical_layer_graph (fusion.hpp:242-357) exported as the flattened CSR graph of dsinf.h.
int dsinf_canonical_layer_graph(int64_t hidden, int64_t batch, int32_t dtype_bytes, dsinf_graph_buffers* out) {
  return guarded([&] {
    require(out, "null argument");
    Graph g = canonical_graph(hidden, batch, dtype_bytes);
    int32_t nd = 0, np = 0;
    for (const auto& e : g.edges) {
      nd += static_cast<int32_t>(e.dep.size());
      for (const auto& [c, prods] : e.dep) np += static_cast<int32_t>(prods.size());
    }
    const bool query = !out->node_kind;
    out->num_nodes = static_cast<int32_t>(g.kind.size());
    out->num_edges = static_cast<int32_t>(g.edges.size());
    out->num_deps = nd;
    out->num_prods = np;
    out->dtype_bytes = g.dtype_bytes;
    if (query) return;
    require(out->node_tile_count && out->node_out_elems && out->edge_from && out->edge_to && out->dep_off &&
                out->dep_consumer && out->prod_off && out->dep_prod,
            "null graph buffer");
    for (size_t i = 0; i < g.kind.size(); ++i) {
      out->node_kind[i] = g.kind[i];
      out->node_tile_count[i] = g.tiles[i];
      out->node_out_elems[i] = g.out_elems[i];
    }
    int32_t di = 0, pi = 0;
    for (size_t e = 0; e < g.edges.size(); ++e) {
      out->edge_from[e] = g.edges[e].from;
      out->edge_to[e] = g.edges[e].to;
      out->dep_off[e] = di;
      for (const auto& [c, prods] : g.edges[e].dep) {
        out->dep_consumer[di] = c;
        out->prod_off[di] = pi;
        for (int p : prods) out->dep_prod[pi++] = p;
        ++di;
      }
    }
    out->dep_off[g.edges.size()] = di;
    out->prod_off[di] = pi;
  });
}

}  // extern "C"
