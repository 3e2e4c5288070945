// C entry points over the UNMODIFIED reference headers (infersim, compiled from the read-only
// reference tree via -I; nothing is copied).  TEST / BASELINE INFRASTRUCTURE ONLY: used by
// tests/ to pin the oracle and the host API, by tests/golden/make_golden.py to emit golden
// vectors, and by `bench.py --impl reference` to time exec_reference on the host cores.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "infersim/costmodel.hpp"
#include "infersim/fusion.hpp"
#include "infersim/gemm.hpp"
#include "infersim/hardware.hpp"
#include "infersim/model.hpp"

using namespace infersim;

namespace {

DeviceSpec device(int sm_count, double mem_bw = 8e12, int64_t mem_bytes = 192'000'000'000) {
  DeviceSpec d;
  d.mem_bytes = mem_bytes;
  d.mem_bw = mem_bw;
  d.sm_count = sm_count;
  d.kernel_launch_overhead = 5e-6;
  d.peak_flops_by_dtype[4] = 80e12;
  d.peak_flops_by_dtype[2] = 2.25e15;
  d.peak_flops_by_dtype[1] = 4.5e15;
  return d;
}

void put_schedule(const GemmSchedule& s, int64_t* out6) {
  out6[0] = s.mode == TilingMode::twoD ? 1 : 0;
  out6[1] = s.output_tiles;
  out6[2] = s.input_tiles;
  out6[3] = s.warps_per_block;
  out6[4] = s.kernel_count;
  out6[5] = s.pack_M;
}

GemmSchedule get_schedule(const int64_t* in6) {
  GemmSchedule s;
  s.mode = in6[0] ? TilingMode::twoD : TilingMode::oneD;
  s.output_tiles = in6[1];
  s.input_tiles = in6[2];
  s.warps_per_block = static_cast<int>(in6[3]);
  s.kernel_count = static_cast<int>(in6[4]);
  s.pack_M = static_cast<int>(in6[5]);
  return s;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError&) {
    return 2;
  } catch (const InfeasibleError&) {
    return 3;
  } catch (...) {
    return 6;
  }
}

ModelConfig model(int64_t h, int64_t L, int64_t heads, int64_t vocab, int64_t max_seq, int dtype) {
  ModelConfig c;
  c.hidden_dim = h;
  c.num_layers = L;
  c.num_heads = heads;
  c.vocab_size = vocab;
  c.max_seq = max_seq;
  c.dtype_bytes = dtype;
  return c;
}

}  // namespace

extern "C" {

int ref_cache_line_pack(int dtype) { return cache_line_pack(dtype); }

int ref_derive_schedule(int64_t N, int64_t K, int64_t B, int dtype, int sm_count, int64_t* out6) {
  return guard([&] {
    GemmShape s{N, K, B, dtype};
    put_schedule(derive_schedule(s, device(sm_count)), out6);
  });
}

int64_t ref_packed_index(int64_t n, int64_t k, int64_t N, int M) { return packed_index(n, k, N, M); }

int ref_pack_weights(const double* W, int64_t N, int64_t K, int dtype, int M, double* out, int64_t out_len) {
  return guard([&] {
    GemmShape s{N, K, 1, dtype};
    std::vector<double> m(W, W + (N > 0 && K > 0 ? N * K : 0));
    PackedWeights p = pack_weights(m, s, M);
    if (static_cast<int64_t>(p.data.size()) != out_len) throw ConfigError("size");
    std::memcpy(out, p.data.data(), p.data.size() * sizeof(double));
  });
}

int ref_unpack_weights(const double* packed, int64_t N, int64_t K, int dtype, int M, double* out) {
  return guard([&] {
    PackedWeights p;
    p.shape = GemmShape{N, K, 1, dtype};
    p.pack_M = M;
    p.padded_in_dim = (K + M - 1) / M * M;
    p.data.assign(packed, packed + N * p.padded_in_dim);
    std::vector<double> m = unpack_weights(p);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

int ref_exec_reference(const double* W, int64_t N, int64_t K, int dtype, const int64_t* sched6, const double* x,
                       int64_t B, double* out) {
  return guard([&] {
    GemmShape s{N, K, B, dtype};
    const GemmSchedule sch = get_schedule(sched6);
    std::vector<double> m(W, W + N * K);
    PackedWeights p = pack_weights(m, s, sch.pack_M);
    std::vector<double> xv(x, x + B * K);
    std::vector<double> o = exec_reference(p, xv, B, sch);
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

// Times exec_reference on `rows` output rows of an N x K GEMM (schedule of the full shape),
// the rows split across `threads` host threads (each thread runs the unmodified function on
// its own packed row block; per-output arithmetic is identical to a single call).
double ref_time_exec(int64_t N, int64_t K, int64_t B, int dtype, int sm_count, int64_t rows, int threads,
                     uint64_t seed, double* checksum) {
  GemmShape full{N, K, B, dtype};
  const GemmSchedule sch = derive_schedule(full, device(sm_count));
  if (threads < 1) threads = 1;
  if (rows < threads) rows = threads;
  // harness (not timed): synthetic x and per-thread weight blocks, generated and packed in
  // parallel with a cheap counter-based generator so the setup stays small next to the timed
  // exec_reference calls
  auto unit = [](uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  };
  std::vector<double> x(B * K);
  for (int64_t i = 0; i < B * K; ++i) x[i] = unit(seed ^ (0x1000000000ull + i));
  const int64_t per = (rows + threads - 1) / threads;
  int nblk = 0;
  for (int t = 0; t < threads; ++t)
    if (t * per < rows) nblk = t + 1;
  std::vector<PackedWeights> blocks(nblk);
  {
    std::vector<std::thread> gen;
    for (int t = 0; t < nblk; ++t)
      gen.emplace_back([&, t] {
        const int64_t r0 = t * per, r1 = std::min(rows, r0 + per);
        std::vector<double> w((r1 - r0) * K);
        for (int64_t i = 0; i < static_cast<int64_t>(w.size()); ++i) w[i] = unit(seed + static_cast<uint64_t>(r0 * K + i));
        blocks[t] = pack_weights(w, GemmShape{r1 - r0, K, B, dtype}, sch.pack_M);
      });
    for (auto& th : gen) th.join();
  }
  std::vector<double> sums(blocks.size(), 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (size_t i = 0; i < blocks.size(); ++i)
    pool.emplace_back([&, i] {
      const std::vector<double> o = exec_reference(blocks[i], x, B, sch);
      double s = 0.0;
      for (double v : o) s += v;
      sums[i] = s;
    });
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  if (checksum) {
    double s = 0.0;
    for (double v : sums) s += v;
    *checksum = s;
  }
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_param_count(int64_t h, int64_t L, int64_t heads, int64_t vocab, int64_t max_seq, int dtype, int64_t* out) {
  return guard([&] { *out = param_count(model(h, L, heads, vocab, max_seq, dtype)); });
}

int ref_layer_flops(int64_t h, int64_t L, int64_t heads, int64_t vocab, int64_t max_seq, int dtype, int64_t batch,
                    int64_t prompt, int64_t gen, int phase, double* out) {
  return guard([&] {
    SeqWorkload w{batch, prompt, gen};
    *out = layer_flops(model(h, L, heads, vocab, max_seq, dtype), w, phase == 0 ? Phase::prompt : Phase::generation);
  });
}

int ref_kv_cache_bytes(int64_t h, int64_t L, int64_t heads, int64_t vocab, int64_t max_seq, int dtype, int64_t batch,
                       int64_t prompt, int64_t gen, int64_t* out) {
  return guard([&] {
    SeqWorkload w{batch, prompt, gen};
    *out = kv_cache_bytes(model(h, L, heads, vocab, max_seq, dtype), w);
  });
}

int ref_kernel_time(double flops, double bytes, double mem_bw, int sm_count, int dtype, int64_t launches,
                    int cuda_graph, double* out4) {
  return guard([&] {
    const KernelCost c = kernel_time(flops, bytes, device(sm_count, mem_bw), dtype, launches, cuda_graph != 0);
    out4[0] = c.compute_time;
    out4[1] = c.memory_time;
    out4[2] = c.launch_overhead;
    out4[3] = c.total;
  });
}

int ref_collective_time(int kind, double bytes, const int* group, int n, int nodes, int gpus, double intra_bw,
                        double intra_lat, double inter_bw, double inter_lat, double* out) {
  return guard([&] {
    const Topology t = build_topology(nodes, gpus, device(148), LinkSpec{intra_bw, intra_lat, LinkKind::intra_node},
                                      LinkSpec{inter_bw, inter_lat, LinkKind::inter_node},
                                      LinkSpec{25e9, 5e-6, LinkKind::pcie});
    std::vector<int> g(group, group + n);
    *out = collective_time(static_cast<CollectiveKind>(kind), bytes, g, t);
  });
}

int ref_min_latency_bound(int64_t h, int64_t L, int64_t heads, int64_t vocab, int dtype, int tp, int pp,
                          double mem_bw, int64_t mem_bytes, double* out) {
  return guard([&] {
    const Topology t =
        build_topology(1, 8, device(148, mem_bw, mem_bytes), LinkSpec{900e9, 2e-6, LinkKind::intra_node},
                       LinkSpec{50e9, 5e-6, LinkKind::inter_node}, LinkSpec{25e9, 5e-6, LinkKind::pcie});
    *out = min_latency_bound(model(h, L, heads, vocab, 2048, dtype), ParallelismPlan{tp, pp}, t);
  });
}

int ref_canonical_partition(int64_t hidden, int64_t batch, int dtype, int regime, int32_t* region_of,
                            int32_t* nregions, int64_t* launches, int64_t* bytes) {
  return guard([&] {
    const OpGraph g = canonical_layer_graph(hidden, batch, dtype);
    const auto regions =
        partition_layer(g, regime == 0 ? BatchRegime::small_batch : BatchRegime::large_batch);
    for (size_t r = 0; r < regions.size(); ++r)
      for (int id : regions[r].node_ids) region_of[id] = static_cast<int32_t>(r);
    *nregions = static_cast<int32_t>(regions.size());
    const FusionSavings s = fusion_savings(regions, g);
    *launches = s.launches_saved;
    *bytes = s.bytes_saved;
  });
}

// Generic graph partition (flattened like dsinf_op_graph) for randomized parity tests.
int ref_partition_graph(int n_nodes, const int32_t* kind, const int32_t* tiles, const int64_t* out_elems, int n_edges,
                        const int32_t* efrom, const int32_t* eto, const int32_t* dep_off, const int32_t* dep_cons,
                        const int32_t* prod_off, const int32_t* dep_prod, int dtype, int regime, int32_t* region_of,
                        int32_t* nregions, int64_t* launches, int64_t* bytes) {
  return guard([&] {
    OpGraph g;
    g.dtype_bytes = dtype;
    for (int i = 0; i < n_nodes; ++i) {
      OpNode nd;
      nd.name = "n" + std::to_string(i);
      nd.kind = static_cast<OpKind>(kind[i]);
      nd.iter_dims = {{"token", 1}};
      nd.tileable_dims = {"token"};
      nd.out_elems = out_elems[i];
      nd.tile_count = tiles[i];
      g.nodes.push_back(nd);
    }
    for (int e = 0; e < n_edges; ++e) {
      GraphEdge ge{efrom[e], eto[e], {}};
      for (int i = dep_off[e]; i < dep_off[e + 1]; ++i) {
        auto& set = ge.tile_dep[dep_cons[i]];
        for (int j = prod_off[i]; j < prod_off[i + 1]; ++j) set.insert(dep_prod[j]);
      }
      g.edges.push_back(ge);
    }
    const auto regions =
        partition_layer(g, regime == 0 ? BatchRegime::small_batch : BatchRegime::large_batch);
    for (size_t r = 0; r < regions.size(); ++r)
      for (int id : regions[r].node_ids) region_of[id] = static_cast<int32_t>(r);
    *nregions = static_cast<int32_t>(regions.size());
    const FusionSavings s = fusion_savings(regions, g);
    *launches = s.launches_saved;
    *bytes = s.bytes_saved;
  });
}


// ---------------------------------------------------------------- whole decode steps
// One decode step of the reference's CPU path: every per-rank GEMM of every layer plus the LM head,
// each one full exec_reference over its output rows (rows split into `threads` packed blocks run
// concurrently; per-output arithmetic identical to one call).  The weights of each distinct shape
// are generated and packed once (not timed); a step runs shape g reps[g] times (L for the layer
// GEMMs, 1 for the LM head) -- the same work as L distinct layers, whose weights (0.1-1.7 GB of
// fp64 each) could not stay cached anyway.
struct RefStep {
  struct Shape {
    GemmSchedule sch;
    int64_t reps;
    std::vector<PackedWeights> blocks;
  };
  std::vector<Shape> shapes;
  std::vector<double> x;
  int64_t B;
  double checksum = 0.0;
};

void* ref_step_create(const int64_t* nk, const int64_t* reps, int G, int64_t B, int dtype, int sm_count, int threads,
                      uint64_t seed) {
  auto st = std::make_unique<RefStep>();
  st->B = B;
  if (threads < 1) threads = 1;
  int64_t kmax = 1;
  for (int g = 0; g < G; ++g) kmax = std::max<int64_t>(kmax, nk[2 * g + 1]);
  auto unit = [](uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  };
  st->x.resize(B * kmax);
  for (int64_t i = 0; i < B * kmax; ++i) st->x[i] = unit(seed ^ (0x1000000000ull + i));
  for (int g = 0; g < G; ++g) {
    const int64_t N = nk[2 * g], K = nk[2 * g + 1];
    RefStep::Shape sh;
    sh.sch = derive_schedule(GemmShape{N, K, B, dtype}, device(sm_count));
    sh.reps = reps[g];
    const int64_t per = (N + threads - 1) / threads;
    const int nblk = static_cast<int>((N + per - 1) / per);
    sh.blocks.resize(nblk);
#pragma omp parallel for schedule(static, 1) num_threads(threads)
    for (int t = 0; t < nblk; ++t) {
      const int64_t r0 = t * per, r1 = std::min(N, r0 + per);
      std::vector<double> w((r1 - r0) * K);
      for (int64_t i = 0; i < static_cast<int64_t>(w.size()); ++i)
        w[i] = unit(seed + (static_cast<uint64_t>(g) << 40) + static_cast<uint64_t>(r0 * K + i));
      sh.blocks[t] = pack_weights(w, GemmShape{r1 - r0, K, B, dtype}, sh.sch.pack_M);
    }
    st->shapes.push_back(std::move(sh));
  }
  return st.release();
}

// Runs one step; returns its wall time in seconds (exec_reference calls only).
double ref_step_run(void* h, int threads) {
  auto* st = static_cast<RefStep*>(h);
  double sum = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (auto& sh : st->shapes) {
    const int64_t K = sh.blocks.empty() ? 0 : sh.blocks[0].shape.in_dim;
    const std::vector<double> x(st->x.begin(), st->x.begin() + st->B * K);
    for (int64_t r = 0; r < sh.reps; ++r) {
#pragma omp parallel for schedule(static, 1) num_threads(threads) reduction(+ : sum)
      for (int t = 0; t < static_cast<int>(sh.blocks.size()); ++t) {
        const std::vector<double> o = exec_reference(sh.blocks[t], x, st->B, sh.sch);
        sum += o.empty() ? 0.0 : o[0];
      }
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  st->checksum += sum;
  return std::chrono::duration<double>(t1 - t0).count();
}

void ref_step_destroy(void* h) { delete static_cast<RefStep*>(h); }

// GEMM hook for the oracle decoder (or_model_set_gemm_hook): out[B][N] = exec_reference over W
// (row-major fp32 N x K, packed once per W pointer and cached), rows split across the OpenMP
// threads.  With it the oracle's decode runs every GEMM through the reference's own function.
namespace {
struct HookCache {
  std::mutex mu;
  std::map<const float*, std::pair<GemmSchedule, std::vector<PackedWeights>>> packed;
};
HookCache& hook_cache() {
  static HookCache c;
  return c;
}
}  // namespace

void ref_gemm_hook(const float* W, int64_t N, int64_t K, const double* x, int64_t B, double* out, void* ctx) {
  const int sm = ctx ? *static_cast<const int*>(ctx) : 148;
  HookCache& c = hook_cache();
  std::pair<GemmSchedule, std::vector<PackedWeights>>* entry = nullptr;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.packed.find(W);
    if (it == c.packed.end() || it->second.second.empty() || it->second.second[0].shape.in_dim != K) {
      const GemmSchedule sch = derive_schedule(GemmShape{N, K, B, 2}, device(sm));
      const int threads = std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
      const int64_t per = (N + threads - 1) / threads;
      const int nblk = static_cast<int>((N + per - 1) / per);
      std::vector<PackedWeights> blocks(nblk);
#pragma omp parallel for schedule(static, 1)
      for (int t = 0; t < nblk; ++t) {
        const int64_t r0 = t * per, r1 = std::min(N, r0 + per);
        std::vector<double> w((r1 - r0) * K);
        for (int64_t i = 0; i < static_cast<int64_t>(w.size()); ++i) w[i] = W[r0 * K + i];
        blocks[t] = pack_weights(w, GemmShape{r1 - r0, K, B, 2}, sch.pack_M);
      }
      c.packed[W] = {sch, std::move(blocks)};
    }
    entry = &c.packed[W];
  }
  // the schedule is derived for the call's batch (derive_schedule ignores B)
  const GemmSchedule sch = entry->first;
  const std::vector<double> xv(x, x + B * K);
  auto& blocks = entry->second;
  const int64_t per = blocks.empty() ? 0 : blocks[0].shape.out_dim;
#pragma omp parallel for schedule(static, 1)
  for (int t = 0; t < static_cast<int>(blocks.size()); ++t) {
    const std::vector<double> o = exec_reference(blocks[t], xv, B, sch);
    const int64_t r0 = t * per, n = blocks[t].shape.out_dim;
    for (int64_t b = 0; b < B; ++b)
      for (int64_t i = 0; i < n; ++i) out[b * N + r0 + i] = o[b * n + i];
  }
}

void ref_gemm_hook_clear() {
  std::lock_guard<std::mutex> lk(hook_cache().mu);
  hook_cache().packed.clear();
}

}  // extern "C"
