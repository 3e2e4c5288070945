// Reference-style C++ caller of the drop-in header (include/dsinf_infersim.hpp): the same calls a
// user of the reference's infersim headers makes, checked against the reference's own examples
// and golden vectors (test_model.cpp:54-58).  Host-only: runs
// without a GPU.  Built and run by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
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

int main() {
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

  if (failures == 0) std::printf("ok\n");
  return failures == 0 ? 0 : 1;
}
