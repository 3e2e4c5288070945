// C ABI for the device operators: SBI-GeMM, weight packing / INT8 quantisation, decode
// attention, and the exec_reference drop-in (gemm.hpp:147-202) executed on the GPU.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <cstring>
#include <vector>

#include "common.h"
#include "ops.cuh"
#include "sbi_gemm.cuh"
#include "tc_gemm.cuh"
#include "synth.h"

using namespace dsinf;

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Per-(device, stream) scratch for the once-per-launch activation quantisation: calls on one stream
// are ordered, so its buffer is reused without synchronisation (grown, after a stream sync, when a
// larger call arrives).  Under graph capture a stream-ordered allocation is used instead.
void* stream_scratch(cudaStream_t s, size_t bytes, bool* async_alloc) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DSINF_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) {
    void* p = nullptr;
    DSINF_CUDA_CHECK(cudaMallocAsync(&p, bytes, s));
    *async_alloc = true;
    return p;
  }
  *async_alloc = false;
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> cache;
  int dev = 0;
  DSINF_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto& e = cache[{dev, s}];
  if (e.second < bytes) {
    if (e.first != nullptr) {
      DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
      DSINF_CUDA_CHECK(cudaFree(e.first));
    }
    e.first = nullptr;
    DSINF_CUDA_CHECK(cudaMalloc(&e.first, bytes));
    e.second = bytes;
  }
  return e.first;
}

void run_gemm(const dsinf_gemm_args& a, cudaStream_t s) {
  require(a.w_packed && a.x && a.out, "null pointer argument");
  require(a.N >= 1 && a.K >= 1 && a.B >= 1, "gemm shape dims must be positive");
  require(a.N <= (1LL << 30) && a.K <= (1LL << 30), "gemm dims too large");
  require(a.w_dtype == DSINF_DT_F16 || a.w_dtype == DSINF_DT_I8, "w_dtype must be F16 or I8");
  require(a.out_dtype == DSINF_DT_F32 || a.out_dtype == DSINF_DT_F16, "out_dtype must be F32 or F16");
  require(a.epilogue == DSINF_EPI_NONE || a.epilogue == DSINF_EPI_GELU, "unknown epilogue");
  require(!(a.epilogue == DSINF_EPI_GELU && a.out_dtype == DSINF_DT_F32), "GeLU epilogue writes F16");
  const bool i8w = a.w_dtype == DSINF_DT_I8;
  require(a.group_size == 0 || a.group_size == ops::kI8Group, "group_size must be 0 (row scales) or 128");
  if (a.group_size != 0)
    require(i8w && a.int8_act == DSINF_INT8_W8A16 && a.w_group_scales != nullptr,
            "K-group scales: I8 weights, DSINF_INT8_W8A16 and w_group_scales");
  if (i8w) {
    require(a.w_scales != nullptr || a.group_size != 0, "I8 weights need w_scales");
    require(a.x_dtype == DSINF_DT_F16 || a.x_dtype == DSINF_DT_I8, "x_dtype must be F16 or I8");
    if (a.x_dtype == DSINF_DT_I8) require(a.x_scales != nullptr, "I8 x needs x_scales");
    require(a.int8_act == DSINF_INT8_W8A8 || a.int8_act == DSINF_INT8_W8A16, "unknown int8_act");
    require(a.int8_act != DSINF_INT8_W8A16 || a.x_dtype == DSINF_DT_F16, "W8A16 takes F16 x");
  } else {
    require(a.x_dtype == DSINF_DT_F16, "F16 weights take F16 x");
  }
  const int N = static_cast<int>(a.N), K = static_cast<int>(a.K);
  // W8A8 with fp16 x: the per-token quantisation runs ONCE per launch (row_prep, the same recipe as
  // the per-CTA PRO_QUANT prologue: scale = max|x| / 127, q = rint(x / scale)) into a stream-ordered
  // scratch buffer, and the GEMM streams the int8 rows by TMA; every CTA re-quantising the whole row
  // made the drop-in W8A8 GEMM 4-14x slower than the in-model plans at B = 16
  const bool quant_once = i8w && a.int8_act == DSINF_INT8_W8A8 && a.x_dtype == DSINF_DT_F16 && K % 8 == 0 &&
                          (reinterpret_cast<uintptr_t>(a.x) & 7) == 0;
  void* xq_scratch = nullptr;
  const int64_t bmax = std::min<int64_t>(gemm::kMaxB, a.B);
  bool scratch_async = false;
  if (quant_once) xq_scratch = stream_scratch(s, static_cast<size_t>(bmax) * (K + 4) + 256, &scratch_async);
  for (int64_t b0 = 0; b0 < a.B; b0 += gemm::kMaxB) {
    const int nb = static_cast<int>(std::min<int64_t>(gemm::kMaxB, a.B - b0));
    int xes = a.x_dtype == DSINF_DT_I8 ? 1 : 2;
    const void* xb = static_cast<const uint8_t*>(a.x) + b0 * a.K * xes;
    const float* xsc = a.x_scales ? a.x_scales + b0 : nullptr;
    if (quant_once) {
      int8_t* xq = static_cast<int8_t*>(xq_scratch);
      float* sc = reinterpret_cast<float*>(static_cast<uint8_t*>(xq_scratch) + ((static_cast<size_t>(bmax) * K + 255) / 256 * 256));
      ops::PrepParams pp{};
      pp.mode = ops::PREP_QUANT_I8;
      pp.x = static_cast<const __half*>(xb);
      pp.x_ld = K;
      pp.out = xq;
      pp.out_scale = sc;
      pp.B = nb;
      pp.K = K;
      // standalone: no GEMM to overlap, so spread long rows over the widest cluster (>= 512 k per CTA)
      pp.split = K >= 8 * 512 ? 8 : (K >= 4 * 512 ? 4 : (K >= 2 * 512 ? 2 : 1));
      ops::row_prep(pp, s, false);
      xb = xq;
      xsc = sc;
      xes = 1;
    }
    const bool a16 = i8w && a.int8_act == DSINF_INT8_W8A16;
    const bool x_i8 = a.x_dtype == DSINF_DT_I8 || quant_once;
    const bool ready_x = !i8w || a16 || x_i8;  // GEMM-ready x (no on-the-fly quantisation)
    const bool xs = ready_x && gemm::prefer_x_stream(nb) && gemm::x_streamable(xb, K, K, i8w && !a16);
    const gemm::Plan plan = gemm::make_plan(N, K, nb, i8w, a.ksplit, xs, a16, false, false, a.group_size != 0);
    gemm::Params p{};
    p.w_scale = a.w_scales;
    p.w_gscale = a.group_size != 0 ? static_cast<const __half*>(a.w_group_scales) : nullptr;
    p.N = N;
    p.K = K;
    p.rows = (K + (i8w ? 3 : 1)) / (i8w ? 4 : 2);
    gemm::make_weight_map(&p.tmap, a.w_packed, N, p.rows);
    p.B = nb;
    p.x = xb;
    p.x_ld = K;
    if (i8w && !a16)
      p.pro = x_i8 ? gemm::PRO_I8 : gemm::PRO_QUANT;
    else
      p.pro = gemm::PRO_F16;
    p.x_scale = xsc;
    p.bias = static_cast<const __half*>(a.bias);
    const int oes = a.out_dtype == DSINF_DT_F32 ? 4 : 2;
    p.out = static_cast<uint8_t*>(a.out) + b0 * a.N * oes;
    p.out_ld = N;
    p.epi = a.out_dtype == DSINF_DT_F32 ? gemm::EPI_F32
                                        : (a.epilogue == DSINF_EPI_GELU ? gemm::EPI_GELU_F16 : gemm::EPI_F16);
    gemm::launch(p, plan, i8w, s, false);
  }
  if (xq_scratch && scratch_async) DSINF_CUDA_CHECK(cudaFreeAsync(xq_scratch, s));
}

struct DeviceBuffer {
  void* p = nullptr;
  explicit DeviceBuffer(size_t bytes) { DSINF_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
  ~DeviceBuffer() { cudaFree(p); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

}  // namespace

extern "C" {

int dsinf_gemm(const dsinf_gemm_args* args, void* stream) {
  return guarded([&] {
    require(args != nullptr, "null args");
    gemm::configure();
    run_gemm(*args, as_stream(stream));
  });
}

int dsinf_gemm_large_batch(const dsinf_gemm_lb_args* a, void* stream) {
  return guarded([&] {
    require(a != nullptr, "null args");
    require(a->w && a->x && a->out, "null pointer argument");
    require(a->N >= 1 && a->K >= 1 && a->M >= 1, "gemm shape dims must be positive");
    require(a->N < (1 << 30) && a->K < (1 << 28) && a->M < (1 << 30), "gemm shape too large");
    require(a->w_dtype == DSINF_DT_F16 || a->w_dtype == DSINF_DT_BF16 || a->w_dtype == DSINF_DT_I8,
            "w_dtype must be F16, BF16 or I8");
    const bool i8 = a->w_dtype == DSINF_DT_I8;
    const bool bf = a->w_dtype == DSINF_DT_BF16;
    require(!bf || (a->out_dtype == DSINF_DT_F32 && a->bias == nullptr && a->epilogue != DSINF_EPI_GELU),
            "BF16 GEMM: F32 output, no bias, no GeLU");
    require(!i8 || (a->w_scales && a->x_scales), "I8 needs w_scales and x_scales");
    require(a->out_dtype == DSINF_DT_F32 || a->out_dtype == DSINF_DT_F16, "out_dtype must be F32 or F16");
    tc::Params p{};
    p.M = static_cast<int>(a->M);
    p.N = static_cast<int>(a->N);
    p.K = static_cast<int>(a->K);
    const int eb = i8 ? 1 : 2;
    tc::make_maps(p, a->x, p.K * eb, a->w, p.K * eb, eb);
    p.bf16 = bf ? 1 : 0;
    p.x_scale = a->x_scales;
    p.w_scale = a->w_scales;
    p.bias = static_cast<const __half*>(a->bias);
    p.out = a->out;
    p.out_ld = p.N;
    if (a->epilogue == DSINF_EPI_GELU) {
      require(a->out_dtype == DSINF_DT_F16, "GeLU epilogue writes F16");
      p.epi = tc::EPI_GELU_F16;
    } else if (a->epilogue == DSINF_EPI_RESID) {
      require(a->out_dtype == DSINF_DT_F32, "residual epilogue accumulates into F32");
      p.epi = tc::EPI_RESID;
    } else {
      require(a->epilogue == DSINF_EPI_NONE, "unknown epilogue");
      p.epi = a->out_dtype == DSINF_DT_F32 ? tc::EPI_F32 : tc::EPI_F16;
    }
    tc::configure();
    tc::launch(p, i8, as_stream(stream));
  });
}

int dsinf_gemm_launch_plan(int64_t N, int64_t K, int64_t B, int32_t w_dtype, dsinf_launch_plan* out) {
  return guarded([&] {
    require(out != nullptr, "null out");
    require(N >= 1 && K >= 1 && B >= 1, "gemm shape dims must be positive");
    const int nb = static_cast<int>(std::min<int64_t>(B, gemm::kMaxB));
    // the plan dsinf_gemm uses with fp16 x (int8 weights then quantise x on the fly: no streaming)
    const bool xs = w_dtype != DSINF_DT_I8 && gemm::prefer_x_stream(nb);
    const gemm::Plan p = gemm::make_plan(static_cast<int>(N), static_cast<int>(K), nb, w_dtype == DSINF_DT_I8, 0, xs);
    out->col_tile = gemm::kColTile;
    out->ksplit = p.ksplit;
    out->rows_per_split = p.rows_per_split;
    out->ctas = p.col_tiles * p.ksplit;
    out->stages = p.stages;
  });
}

int dsinf_pack_weights_device(const void* w_rowmajor, int32_t src_dtype, int64_t N, int64_t K, int32_t pack_M,
                              void* packed_f16, void* stream) {
  return guarded([&] {
    require(w_rowmajor && packed_f16, "null pointer argument");
    require(N >= 1 && K >= 1, "gemm shape dims must be positive");
    require(src_dtype == DSINF_DT_F16 || src_dtype == DSINF_DT_F32, "src_dtype must be F16 or F32");
    if (pack_M != 1 && pack_M != 2 && pack_M != 4) throw ConfigError("pack_M must be one of {1, 2, 4}");
    ops::pack_f16(w_rowmajor, src_dtype == DSINF_DT_F32, N, K, pack_M, static_cast<__half*>(packed_f16),
                  as_stream(stream));
  });
}

int dsinf_quantize_weights_int8(const void* w_rowmajor_f16, int64_t N, int64_t K, int8_t* packed_i8, float* row_scales,
                                void* stream) {
  return guarded([&] {
    require(w_rowmajor_f16 && packed_i8 && row_scales, "null pointer argument");
    require(N >= 1 && K >= 1, "gemm shape dims must be positive");
    ops::quantize_weights_i8(static_cast<const __half*>(w_rowmajor_f16), N, K, packed_i8, row_scales,
                             as_stream(stream));
  });
}

int dsinf_quantize_weights_int8_groups(const void* w_rowmajor_f16, int64_t N, int64_t K, int32_t group,
                                       int8_t* packed_i8, void* group_scales_f16, void* stream) {
  return guarded([&] {
    require(w_rowmajor_f16 && packed_i8 && group_scales_f16, "null pointer argument");
    require(N >= 1 && K >= 1, "gemm shape dims must be positive");
    require(group == ops::kI8Group, "group must be 128");
    ops::quantize_weights_i8_groups(static_cast<const __half*>(w_rowmajor_f16), N, K, packed_i8,
                                    static_cast<__half*>(group_scales_f16), as_stream(stream));
  });
}

int dsinf_quantize_activations_int8(const void* x_f16, int64_t B, int64_t K, int8_t* xq, float* scales, void* stream) {
  return guarded([&] {
    require(x_f16 && xq && scales, "null pointer argument");
    require(B >= 1 && K >= 1, "shape dims must be positive");
    ops::quantize_act_i8(static_cast<const __half*>(x_f16), B, K, xq, scales, as_stream(stream));
  });
}

int dsinf_attention_decode(const void* q, const void* kcache, const void* vcache, const int32_t* pos_dev, int64_t B,
                           int64_t H, int64_t d, int64_t max_seq, void* out, void* stream) {
  return guarded([&] {
    require(q && kcache && vcache && pos_dev && out, "null pointer argument");
    require(B >= 1 && H >= 1 && d >= 2 && max_seq >= 1, "bad attention shape");
    ops::configure();
    ops::AttnParams a{};
    a.q = static_cast<const __half*>(q);
    a.kc = static_cast<const __half*>(kcache);
    a.vc = static_cast<const __half*>(vcache);
    a.pos = pos_dev;
    a.out = static_cast<__half*>(out);
    a.B = static_cast<int>(B);
    a.H = static_cast<int>(H);
    a.d = static_cast<int>(d);
    a.max_seq = static_cast<int>(max_seq);
    a.scale = 1.0f / std::sqrt(static_cast<float>(d));
    ops::attention(a, ops::attention_chunks(a.B, a.H), as_stream(stream), false);
  });
}

int dsinf_exec_device(const double* packed, int64_t packed_len, int32_t packed_pack_M,
                      const dsinf_gemm_shape* shape, const dsinf_gemm_schedule* schedule, const double* x,
                      int64_t x_len, int64_t batch, int32_t compute_dtype, double* out, int64_t out_len) {
  return guarded([&] {
    require(packed && shape && schedule && x && out, "null pointer argument");
    const int64_t N = shape->out_dim, K = shape->in_dim;
    if (N < 1 || K < 1) throw ConfigError("gemm shape dims must be positive");
    if (batch < 1 || x_len != batch * K) throw ConfigError("input shape mismatch");  // gemm.hpp:153-154
    // the data layout is the packed buffer's own M (exec_reference reads packed.pack_M,
    // gemm.hpp:186); the schedule's pack_M only groups the reference's iteration
    const int M = packed_pack_M;
    if (M != 1 && M != 2 && M != 4) throw ConfigError("pack_M must be one of {1, 2, 4}");
    const int SM = schedule->pack_M;
    if (SM != 1 && SM != 2 && SM != 4) throw ConfigError("pack_M must be one of {1, 2, 4}");
    const int64_t kp = (K + M - 1) / M * M;
    if (packed_len != N * kp) throw ConfigError("packed buffer size mismatch");
    if (out_len != batch * N) throw ConfigError("output buffer size mismatch");
    require(compute_dtype == DSINF_DT_F16 || compute_dtype == DSINF_DT_I8, "compute_dtype must be F16 or I8");
    // unpack (host) -> fp16 row-major on device -> device pack / quantise -> SBI-GeMM.  The TMA view
    // of the packed weights needs N % 4 == 0 (16-byte row stride): out_dim is padded with zero rows
    // and the padding columns are dropped from the output (exec_reference takes any N).
    const int64_t Np = (N + 3) / 4 * 4;
    std::vector<uint16_t> w16(static_cast<size_t>(Np * K), 0);
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < K; ++k)
        w16[n * K + k] = f32_to_f16_bits(static_cast<float>(packed[(k / M) * (N * M) + n * M + (k % M)]));
    std::vector<uint16_t> x16(static_cast<size_t>(batch * K));
    for (int64_t i = 0; i < batch * K; ++i) x16[i] = f32_to_f16_bits(static_cast<float>(x[i]));
    cudaStream_t s = nullptr;
    DeviceBuffer dw(w16.size() * 2), dx(x16.size() * 2), dout(static_cast<size_t>(batch * Np) * 4);
    DSINF_CUDA_CHECK(cudaMemcpy(dw.p, w16.data(), w16.size() * 2, cudaMemcpyHostToDevice));
    DSINF_CUDA_CHECK(cudaMemcpy(dx.p, x16.data(), x16.size() * 2, cudaMemcpyHostToDevice));
    gemm::configure();
    dsinf_gemm_args a{};
    a.N = Np;
    a.K = K;
    a.B = batch;
    a.x = dx.p;
    a.x_dtype = DSINF_DT_F16;
    a.out = dout.p;
    a.out_dtype = DSINF_DT_F32;
    a.epilogue = DSINF_EPI_NONE;
    if (compute_dtype == DSINF_DT_F16) {
      DeviceBuffer dp(static_cast<size_t>((K + 1) / 2 * 2 * Np) * 2);
      ops::pack_f16(dw.p, false, Np, K, 2, static_cast<__half*>(dp.p), s);
      a.w_packed = dp.p;
      a.w_dtype = DSINF_DT_F16;
      run_gemm(a, s);
      DSINF_CUDA_CHECK(cudaDeviceSynchronize());
    } else {
      DeviceBuffer dp(static_cast<size_t>((K + 3) / 4 * 4 * Np)), ds(static_cast<size_t>(Np) * 4);
      ops::quantize_weights_i8(static_cast<const __half*>(dw.p), Np, K, static_cast<int8_t*>(dp.p),
                               static_cast<float*>(ds.p), s);
      a.w_packed = dp.p;
      a.w_dtype = DSINF_DT_I8;
      a.w_scales = static_cast<const float*>(ds.p);
      run_gemm(a, s);
      DSINF_CUDA_CHECK(cudaDeviceSynchronize());
    }
    std::vector<float> o(static_cast<size_t>(batch * Np));
    DSINF_CUDA_CHECK(cudaMemcpy(o.data(), dout.p, o.size() * 4, cudaMemcpyDeviceToHost));
    for (int64_t b = 0; b < batch; ++b)
      for (int64_t n = 0; n < N; ++n) out[b * N + n] = o[b * Np + n];
  });
}

}  // extern "C"
