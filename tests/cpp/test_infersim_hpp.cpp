// Reference-style C++ caller of the drop-in header (include/dsinf_infersim.hpp): the same calls a
// user of the reference's infersim headers makes, checked against the reference's own examples
// and golden vectors (test_model.cpp:54-58).  Host-only: runs
// without a GPU.  Built and run by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "dsinf_infersim.hpp"

namespace infersim = dsinf::infersim;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  using infersim::GemmShape;
  // cache_line_pack (gemm.hpp:57-60): fp32 1, fp16 2, int8 4
  EXPECT(infersim::cache_line_pack(4) == 1 && infersim::cache_line_pack(2) == 2 && infersim::cache_line_pack(1) == 4);
  EXPECT(infersim::kOutputTileWidth() == 32);

  // derive_schedule: the A100 example of SPEC.md:301 (N=256 on 108 SMs -> 2D, 16 input tiles)
  infersim::DeviceSpec a100;
  a100.mem_bytes = 80LL << 30;
  a100.mem_bw = 2.0e12;
  a100.sm_count = 108;
  a100.peak_flops_by_dtype = {{4, 19.5e12}, {2, 312e12}, {1, 624e12}};
  const auto s = infersim::derive_schedule(GemmShape{256, 4096, 1, 2}, a100);
  EXPECT(s.mode == infersim::TilingMode::twoD && s.input_tiles == 16 && s.kernel_count == 2 && s.pack_M == 2);
  // B200: GPT-J QKV is 1D (ceil(12288/32) = 384 >= 148 tiles)
  const auto b200 = infersim::DeviceSpec::b200();
  EXPECT(b200.sm_count == 148);
  EXPECT(infersim::derive_schedule(GemmShape{12288, 4096, 1, 2}, b200).mode == infersim::TilingMode::oneD);

  // pack_weights golden vectors: element (n, k) = (n+1)*10 + k
  auto mat = [](int N, int K) {
    std::vector<double> m(N * K);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) m[n * K + k] = (n + 1) * 10 + k;
    return m;
  };
  {
    const auto p = infersim::pack_weights(mat(2, 4), GemmShape{2, 4, 1, 2}, 2);
    EXPECT((p.data == std::vector<double>{10, 11, 20, 21, 12, 13, 22, 23}));
  }
  {
    const auto p = infersim::pack_weights(mat(2, 8), GemmShape{2, 8, 1, 1}, 4);
    EXPECT((p.data == std::vector<double>{10, 11, 12, 13, 20, 21, 22, 23, 14, 15, 16, 17, 24, 25, 26, 27}));
  }
  {
    const auto p = infersim::pack_weights(mat(2, 3), GemmShape{2, 3, 1, 2}, 2);
    EXPECT((p.data == std::vector<double>{10, 11, 20, 21, 12, 0, 22, 0}));
    EXPECT(p.padded_in_dim == 4);
    EXPECT(infersim::unpack_weights(p) == mat(2, 3));
  }
  {
    const auto p = infersim::pack_weights(mat(2, 4), GemmShape{2, 4, 1, 4}, 1);
    EXPECT((p.data == std::vector<double>{10, 20, 11, 21, 12, 22, 13, 23}));
  }
  EXPECT(infersim::packed_index(1, 5, 2, 4) == 4 * 2 + 1 * 4 + 1);

  // errors: ConfigError for bad shapes / pack_M (gemm.hpp:36-38, :116-119)
  bool threw = false;
  try {
    infersim::derive_schedule(GemmShape{0, 16, 1, 2}, b200);
  } catch (const infersim::ConfigError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    infersim::pack_weights(mat(2, 4), GemmShape{2, 4, 1, 2}, 3);
  } catch (const infersim::ConfigError&) {
    threw = true;
  }
  EXPECT(threw);

  // model accounting (test_model.cpp:54-58): GPT-2 1.5B param_count
  infersim::ModelConfig gpt2{"gpt2", 1600, 48, 25, 50257, 1024, 2};
  EXPECT(infersim::param_count(gpt2) == 1554971200LL);
  EXPECT(infersim::param_bytes(gpt2) == 2 * 1554971200LL);
  // generation layer flops: 24 h^2 B + 4 B ctx h  (model.hpp:121-132)
  const double lf = infersim::layer_flops(gpt2, {1, 128, 8}, infersim::Phase::generation);
  EXPECT(lf > 24.0 * 1600 * 1600 && lf < 24.0 * 1600 * 1600 * 1.1);

  // kernel_time roofline (costmodel.hpp:42-56): memory bound, one launch overhead
  const auto kc = infersim::kernel_time(1e9, 1e9, a100, 2, 1, false);
  EXPECT(kc.memory_bound && std::fabs(kc.total - (1e9 / 2.0e12 + 5e-6)) < 1e-12);

  // Deep-Fusion: canonical layer graph -> small-batch partition (test_fusion.cpp:103-121) and the
  // savings golden (h=1600, B=1 -> 4 launches, 57,600 B)
  {
    const auto g = infersim::canonical_layer_graph(1600, 1);
    EXPECT(g.nodes.size() == 8 && g.edges.size() == 7);
    EXPECT(g.nodes[1].kind == infersim::OpKind::gemm && g.nodes[1].name == "qkv_gemm");
    const auto regions = infersim::partition_layer(g, infersim::BatchRegime::small_batch);
    EXPECT(regions.size() == 4);
    if (regions.size() == 4) {
      EXPECT((regions[0].node_ids == std::vector<int>{0, 1}));
      EXPECT((regions[1].node_ids == std::vector<int>{2, 3}));
      EXPECT((regions[2].node_ids == std::vector<int>{4, 5}));
      EXPECT((regions[3].node_ids == std::vector<int>{6, 7}));
    }
    const auto sv = infersim::fusion_savings(regions, g);
    EXPECT(sv.launches_saved == 4 && sv.bytes_saved == 57600);
    EXPECT(infersim::fusable(g, g.edges[0]) && !infersim::fusable(g, g.edges[1]));
    const auto large = infersim::partition_layer(g, infersim::BatchRegime::large_batch);
    for (const auto& r : large)
      for (int id : r.node_ids)
        if (g.nodes[id].kind == infersim::OpKind::gemm) EXPECT(r.node_ids.size() == 1);
    threw = false;
    try {
      infersim::fusion_savings({regions[0]}, g);
    } catch (const infersim::ConfigError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // collective_time: ring all-reduce 2(n-1)/n S/bw + (n-1) lat (test_costmodel.cpp:75-83)
  {
    infersim::Topology topo;
    topo.num_nodes = 1;
    topo.gpus_per_node = 8;
    topo.device = b200;
    topo.intra = {900e9, 2e-6};
    topo.inter = {50e9, 5e-6};
    const double t = infersim::collective_time(infersim::CollectiveKind::allreduce, 1e6, {0, 1, 2, 3}, topo);
    EXPECT(std::fabs(t - (2.0 * 3.0 / 4.0 * 1e6 / 900e9 + 3.0 * 2e-6)) < 1e-15);
    EXPECT(infersim::collective_time(infersim::CollectiveKind::allreduce, 1e6, {5}, topo) == 0.0);
  }

  if (gpu) {
    // exec_reference on the GPU: same results for every pack_M of the packed data under every schedule
    // (exec_reference reads packed.pack_M; the schedule's pack_M only groups its iteration)
    const int N = 96, K = 70, B = 3;
    std::vector<double> W(N * K), x(B * K), ref(B * N, 0.0);
    for (int i = 0; i < N * K; ++i) W[i] = (i * 7 % 17) - 8;
    for (int i = 0; i < B * K; ++i) x[i] = (i * 5 % 13) - 6;
    for (int b = 0; b < B; ++b)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) ref[b * N + n] += W[n * K + k] * x[b * K + k];
    for (int pm : {1, 2, 4})
      for (int sm : {1, 2, 4}) {
        const GemmShape shape{N, K, B, 2};
        auto sch = infersim::derive_schedule(shape, b200);
        sch.pack_M = sm;
        const auto packed = infersim::pack_weights(W, shape, pm);
        EXPECT(infersim::exec_reference(packed, x, B, sch) == ref);
      }
  }

  if (failures == 0) std::printf("ok\n");
  return failures == 0 ? 0 : 1;
}
