// Device building blocks of SBI-GeMM (infersim gemm.hpp:147-202) shared by the
// standalone kernel (sbi_gemm.cu) and the persistent decode-step kernel (step_kernel.cu):
//   * Deep-Fusion prologues that fill a CTA's x slice in shared memory (LayerNorm with the
//     residual add folded in, per-token int8 quantisation, plain fp16 / int8 loads);
//   * the consumer loop over the TMA ring (warp MMAs on the reference packed layout);
//   * the epilogues (bias, GeLU, residual add, RoPE + KV-cache append, fp16/fp32 stores).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <type_traits>

#include "ptx.cuh"
#include "sbi_gemm.cuh"

namespace dsinf {
namespace gemm {
namespace dev {

struct Header {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  float xscale[kMaxB];
  float mean[kMaxB];
  float rstd[kMaxB];
  float red[8];
  int flag[4];
};

// Epilogue statistics of one CTA's columns (static smem of the standalone kernel).
struct EpiStats {
  unsigned long long esum[kMaxB][2];  // row sums (fixed point)
  unsigned emax[kMaxB];               // row max |out| (fp32 bits)
};
static_assert(sizeof(Header) <= kHeaderBytes, "header too large");

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int next_pow2(int b) {
  int p = 1;
  while (p < b) p <<= 1;
  return p;
}

// Consumer-thread -> (batch row, lane-in-row) map used by every per-row reduction: `tpr`
// consecutive consumer threads own one row.
struct RowMap {
  int tpr, b, j;
  bool active;
  __device__ __forceinline__ RowMap(int B, int ctid) {
    tpr = 128 / next_pow2(B);
    b = ctid / tpr;
    j = ctid % tpr;
    active = b < B;
  }
};

// Sum (or max) over the `tpr` threads of a row.  All threads of the row get the same bits
// (symmetric butterfly, then an in-order warp sum), so results are run-to-run deterministic.
template <bool kMax>
__device__ __forceinline__ float row_reduce(float v, int tpr, float* scratch, int cw, int lane) {
  const int width = tpr < 32 ? tpr : 32;
  for (int o = width >> 1; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, u) : v + u;
  }
  if (tpr > 32) {
    consumer_bar();
    if (lane == 0) scratch[cw] = v;
    consumer_bar();
    const int wpr = tpr >> 5;
    const int first = (cw / wpr) * wpr;
    float t = scratch[first];
    for (int i = 1; i < wpr; ++i) t = kMax ? fmaxf(t, scratch[first + i]) : t + scratch[first + i];
    v = t;
  }
  return v;
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Per-token int8: q = clamp(rint(x / s), -127, 127) with IEEE division (bit-exact vs oracle).
__device__ __forceinline__ uint32_t quant_byte(float x, float scale) {
  int q = __float2int_rn(__fdiv_rn(x, scale));
  q = max(-127, min(127, q));
  return static_cast<uint32_t>(q) & 0xffu;
}

__device__ __forceinline__ float act_scale(float maxabs) {
  return maxabs > 0.0f ? __fdiv_rn(maxabs, 127.0f) : 1.0f;
}

// Residual-stream element: r + (delta + delta_bias)  (delta optional; with `nd` > 1 slots the
// delta is the rank-order sum of the fused all-reduce's partials).
struct ResidualView {
  const float* r;
  const float* d;
  const __half* db;
  int K;
  int nd = 1;
  long long ds = 0;
  __device__ __forceinline__ float4 load4(int b, int k) const {
    float4 v = __ldcg(reinterpret_cast<const float4*>(r + static_cast<size_t>(b) * K + k));
    if (d) {
      float4 t = __ldcg(reinterpret_cast<const float4*>(d + static_cast<size_t>(b) * K + k));
      for (int q = 1; q < nd; ++q) {
        const float4 u = __ldcg(reinterpret_cast<const float4*>(d + q * ds + static_cast<size_t>(b) * K + k));
        t.x = __fadd_rn(t.x, u.x);
        t.y = __fadd_rn(t.y, u.y);
        t.z = __fadd_rn(t.z, u.z);
        t.w = __fadd_rn(t.w, u.w);
      }
      if (db) {
        const __half2 b01 = *reinterpret_cast<const __half2*>(db + k);
        const __half2 b23 = *reinterpret_cast<const __half2*>(db + k + 2);
        t.x = __fadd_rn(t.x, __low2float(b01));
        t.y = __fadd_rn(t.y, __high2float(b01));
        t.z = __fadd_rn(t.z, __low2float(b23));
        t.w = __fadd_rn(t.w, __high2float(b23));
      }
      v.x = __fadd_rn(v.x, t.x);
      v.y = __fadd_rn(v.y, t.y);
      v.z = __fadd_rn(v.z, t.z);
      v.w = __fadd_rn(v.w, t.w);
    }
    return v;
  }
};
__device__ __forceinline__ ResidualView residual_view(const Params& p) {
  ResidualView rv{p.res_in, p.res_delta, p.delta_bias, p.K};
  rv.nd = p.delta_slots > 0 ? p.delta_slots : 1;
  rv.ds = p.delta_stride;
  return rv;
}

__device__ __forceinline__ float ln_apply(float v, float mean, float rstd, const __half* g, const __half* bta,
                                          int k) {
  return (v - mean) * rstd * __half2float(g[k]) + __half2float(bta[k]);
}

// ------------------------------------------------------------------ per-row statistics
// LayerNorm statistics of the full row (single shifted pass) -> hd.mean / hd.rstd; with int8
// weights also the per-token scale of the fp16-rounded normalised row -> hd.xscale.
// `write_res` stores the residual (r + delta + bias) once (one CTA per launch / phase).
// Mean / rstd from the fixed-point row sums (int64, exact and order-independent).  Only
// multiplications in fp64 (inv_k = 1/K from the host) and one fp32 rsqrt: no fp64 divide / sqrt
// subroutines on the prologue's critical path.
__device__ __forceinline__ void ln_mean_rstd(long long s1, long long s2, double inv_k, float eps, float& mean,
                                             float& rstd) {
  const double m = static_cast<double>(s1) * (inv_k * (1.0 / static_cast<double>(kSumScale)));
  const double e2 = static_cast<double>(s2) * (inv_k * (1.0 / static_cast<double>(kSqScale)));
  const double var = fmax(fma(-m, m, e2), 0.0);
  mean = static_cast<float>(m);
  rstd = rsqrtf(static_cast<float>(var) + eps);
}
// Mean / rstd of row b from the producer's fixed-point sums (kStatStripes stripes).
__device__ __forceinline__ void ln_from_sums(const long long* st, int b, double inv_k, float eps, float& mean,
                                             float& rstd) {
  long long s1 = 0, s2 = 0;
#pragma unroll
  for (int s = 0; s < kStatStripes; ++s) {
    s1 += __ldcg(st + (s * kMaxB + b) * 2);
    s2 += __ldcg(st + (s * kMaxB + b) * 2 + 1);
  }
  ln_mean_rstd(s1, s2, inv_k, eps, mean, rstd);
}

// Row max |x| from the producer's stripes.
__device__ __forceinline__ float amax_from_stripes(const unsigned* a, int b) {
  unsigned m = 0;
#pragma unroll
  for (int s = 0; s < kStatStripes; ++s) m = max(m, __ldcg(a + s * 32 + b));
  return __uint_as_float(m);
}

template <bool kInt8>
__device__ void ln_row_stats(const Params& p, Header& hd, int ctid, int cw, int lane, bool write_res) {
  const RowMap rm(p.B, ctid);
  const int K = p.K;
  const ResidualView rv = residual_view(p);
  if (p.ln_stats_in != nullptr) {  // statistics from the producing epilogue: no full-row pass
    if (ctid < p.B) ln_from_sums(p.ln_stats_in, ctid, p.ln_inv_k, p.ln_eps, hd.mean[ctid], hd.rstd[ctid]);
    if (!kInt8) return;
    consumer_bar();
    const float mean = rm.active ? hd.mean[rm.b] : 0.f, rstd = rm.active ? hd.rstd[rm.b] : 0.f;
    float mx = 0.f;
    if (rm.active) {
#pragma unroll 8
      for (int c = rm.j; c < K / 4; c += rm.tpr) {
        const float4 v = rv.load4(rm.b, 4 * c);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          mx = fmaxf(mx, fabsf(__half2float(__float2half_rn(ln_apply(vv[i], mean, rstd, p.ln_g, p.ln_b, 4 * c + i)))));
      }
    }
    mx = row_reduce<true>(mx, rm.tpr, hd.red, cw, lane);
    if (rm.active && rm.j == 0) hd.xscale[rm.b] = act_scale(mx);
    return;
  }
  float c0 = 0.f, s1 = 0.f, s2 = 0.f;
  if (rm.active) {
    c0 = rv.load4(rm.b, 0).x;  // shift for a cancellation-free single pass
#pragma unroll 8
    for (int c = rm.j; c < K / 4; c += rm.tpr) {
      const float4 v = rv.load4(rm.b, 4 * c);
      if (write_res) *reinterpret_cast<float4*>(p.res_out + static_cast<size_t>(rm.b) * K + 4 * c) = v;
      const float d0 = v.x - c0, d1 = v.y - c0, d2 = v.z - c0, d3 = v.w - c0;
      s1 += (d0 + d1) + (d2 + d3);
      s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
  }
  s1 = row_reduce<false>(s1, rm.tpr, hd.red, cw, lane);
  s2 = row_reduce<false>(s2, rm.tpr, hd.red, cw, lane);
  const float inv_k = 1.0f / static_cast<float>(K);
  const float m1 = s1 * inv_k;
  const float var = fmaxf(s2 * inv_k - m1 * m1, 0.0f);
  const float mean = c0 + m1;
  const float rstd = 1.0f / sqrtf(var + p.ln_eps);
  if (kInt8) {
    float mx = 0.f;
    if (rm.active) {
#pragma unroll 8
      for (int c = rm.j; c < K / 4; c += rm.tpr) {
        const float4 v = rv.load4(rm.b, 4 * c);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float y = __half2float(__float2half_rn(ln_apply(vv[i], mean, rstd, p.ln_g, p.ln_b, 4 * c + i)));
          mx = fmaxf(mx, fabsf(y));
        }
      }
    }
    mx = row_reduce<true>(mx, rm.tpr, hd.red, cw, lane);
    if (rm.active && rm.j == 0) hd.xscale[rm.b] = act_scale(mx);
  }
  if (rm.active && rm.j == 0) {
    hd.mean[rm.b] = mean;
    hd.rstd[rm.b] = rstd;
  }
}

// Per-token scale of an fp16 activation row (PRO_QUANT) -> hd.xscale.
__device__ __forceinline__ void quant_row_scale(const Params& p, Header& hd, int ctid, int cw, int lane) {
  if (p.amax_in != nullptr) {  // row max from the producing epilogue
    if (ctid < p.B) hd.xscale[ctid] = act_scale(amax_from_stripes(p.amax_in, ctid));
    return;
  }
  const RowMap rm(p.B, ctid);
  const __half* x = static_cast<const __half*>(p.x);
  float mx = 0.f;
  if (rm.active)
  {
    const __half* row = x + static_cast<size_t>(rm.b) * p.x_ld;
    const bool vec = (p.x_ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 7) == 0;
    if (vec) {
#pragma unroll 8
      for (int c = rm.j; c < p.K / 4; c += rm.tpr) {
        const uint2 u = __ldcg(reinterpret_cast<const uint2*>(row + 4 * c));
        const __half2 h01 = *reinterpret_cast<const __half2*>(&u.x);
        const __half2 h23 = *reinterpret_cast<const __half2*>(&u.y);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(__low2float(h01)), fabsf(__high2float(h01))),
                             fmaxf(fabsf(__low2float(h23)), fabsf(__high2float(h23)))));
      }
      for (int k = (p.K / 4) * 4 + rm.j; k < p.K; k += rm.tpr) mx = fmaxf(mx, fabsf(__half2float(__ldcg(row + k))));
    } else {
      for (int k = rm.j; k < p.K; k += rm.tpr) mx = fmaxf(mx, fabsf(__half2float(__ldcg(row + k))));
    }
  }
  mx = row_reduce<true>(mx, rm.tpr, hd.red, cw, lane);
  if (rm.active && rm.j == 0) hd.xscale[rm.b] = act_scale(mx);
}

// ------------------------------------------------------------------ x slice
// Writes packed rows [row0, row0 + nrows) of x into sx[b * xrw + w] (w = row - row0), one 32-bit
// word per (row, b) holding M = 2 (fp16) or 4 (int8) consecutive k.  Requires the statistics
// of ln_row_stats / quant_row_scale in `hd` for PRO_LN / PRO_QUANT.
// Runs store(i, load(i)) for i = ctid, ctid + 128, ... < total with kChunk loads issued before
// the first store: the slice loads are L2 round trips, so independence (ILP) is what matters.
template <int kChunk = 8, class Load, class Store>
__device__ __forceinline__ void chunked(int ctid, int total, Load load, Store store) {
  using T = decltype(load(0));
  for (int base = ctid; base < total; base += 128 * kChunk) {
    T r[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (base + 128 * j < total) r[j] = load(base + 128 * j);
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (base + 128 * j < total) store(base + 128 * j, r[j]);
  }
}

// PRO_LN, fp16, statistics from the producer (p.ln_stats_in): the first residual / gamma / beta
// loads are issued BEFORE the statistics are read, so the two L2 round trips overlap.  Replaces
// ln_row_stats + consumer_bar + fill_x_slice for this case (all 128 consumer threads call it).
__device__ __forceinline__ void fill_x_ln_f16_pre(const Params& p, uint32_t* sx, Header& hd, int row0, int nrows, int ctid,
                                                  long long c_rel = 0) {
  constexpr int kPre = 8;
  const int K = p.K;
  const int xrw = p.x_row_words;
  const int total = p.B * nrows;
  float2 r[kPre];
  __half2 g[kPre], be[kPre];
  const __half2 zero2 = __floats2half2_rn(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kPre; ++j) {
    const int i = ctid + 128 * j;
    r[j] = make_float2(0.f, 0.f);
    g[j] = be[j] = zero2;
    if (i < total) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 2;
      if (k < K) {  // K % 8 == 0 on this path
        r[j] = __ldcg(reinterpret_cast<const float2*>(p.res_in + static_cast<size_t>(b) * K + k));
        g[j] = *reinterpret_cast<const __half2*>(p.ln_g + k);
        be[j] = *reinterpret_cast<const __half2*>(p.ln_b + k);
      }
    }
  }
  if (ctid < p.B) ln_from_sums(p.ln_stats_in, ctid, p.ln_inv_k, p.ln_eps, hd.mean[ctid], hd.rstd[ctid]);
  consumer_bar();
#pragma unroll
  for (int j = 0; j < kPre; ++j) {
    const int i = ctid + 128 * j;
    if (i < total) {
      const int b = i / nrows, w = i - b * nrows;
      const float mean = hd.mean[b], rstd = hd.rstd[b];
      sx[b * xrw + w] = pack_h2((r[j].x - mean) * rstd * __low2float(g[j]) + __low2float(be[j]),
                                (r[j].y - mean) * rstd * __high2float(g[j]) + __high2float(be[j]));
    }
  }
  if (total > 128 * kPre)
    chunked(ctid + 128 * kPre, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 2;
      return k < K ? __ldcg(reinterpret_cast<const float2*>(p.res_in + static_cast<size_t>(b) * K + k))
                   : make_float2(0.f, 0.f);
    }, [&](int i, float2 v) {
      const int b = i / nrows, w = i - b * nrows;
      const int k = (row0 + w) * 2;
      sx[b * xrw + w] = k < K ? pack_h2(ln_apply(v.x, hd.mean[b], hd.rstd[b], p.ln_g, p.ln_b, k),
                                        ln_apply(v.y, hd.mean[b], hd.rstd[b], p.ln_g, p.ln_b, k + 1))
                              : 0u;
    });
}

// PRO_LN with int8 weights and producer statistics, when the row fits in registers
// (K/4 <= tpr * kLnRegVec float4 per thread): the residual row, gamma, beta and the statistics
// are loaded in ONE L2 round trip; the fp16-rounded normalised row gives the per-token scale
// (row max), and the slice words are quantised straight from registers.
constexpr int kLnRegVec = 8;
__device__ __forceinline__ bool ln_i8_fits(int B, int K) { return K / 4 <= (128 / next_pow2(B)) * kLnRegVec; }

__device__ __forceinline__ void fill_x_ln_i8_regs(const Params& p, uint32_t* sx, Header& hd, int row0, int nrows,
                                                  int ctid, int cw, int lane) {
  const RowMap rm(p.B, ctid);
  const int K = p.K, K4 = K / 4;
  const int xrw = p.x_row_words;
  float4 v[kLnRegVec];
  uint2 g[kLnRegVec], be[kLnRegVec];
#pragma unroll
  for (int u = 0; u < kLnRegVec; ++u) {
    const int c = rm.j + u * rm.tpr;
    if (rm.active && c < K4) {
      v[u] = __ldcg(reinterpret_cast<const float4*>(p.res_in + static_cast<size_t>(rm.b) * K) + c);
      g[u] = *reinterpret_cast<const uint2*>(p.ln_g + 4 * c);
      be[u] = *reinterpret_cast<const uint2*>(p.ln_b + 4 * c);
    }
  }
  // one thread per row reads the producer's sums (every thread reading them would put ~all CTAs'
  // requests on the same few L2 lines)
  if (ctid < p.B) ln_from_sums(p.ln_stats_in, ctid, p.ln_inv_k, p.ln_eps, hd.mean[ctid], hd.rstd[ctid]);
  consumer_bar();
  const float mean = rm.active ? hd.mean[rm.b] : 0.f, rstd = rm.active ? hd.rstd[rm.b] : 0.f;
  uint2 hv[kLnRegVec];
  float mx = 0.f;
#pragma unroll
  for (int u = 0; u < kLnRegVec; ++u) {
    const int c = rm.j + u * rm.tpr;
    if (rm.active && c < K4) {
      const __half2 g01 = *reinterpret_cast<const __half2*>(&g[u].x), g23 = *reinterpret_cast<const __half2*>(&g[u].y);
      const __half2 b01 = *reinterpret_cast<const __half2*>(&be[u].x), b23 = *reinterpret_cast<const __half2*>(&be[u].y);
      const __half2 h01 = __floats2half2_rn((v[u].x - mean) * rstd * __low2float(g01) + __low2float(b01),
                                            (v[u].y - mean) * rstd * __high2float(g01) + __high2float(b01));
      const __half2 h23 = __floats2half2_rn((v[u].z - mean) * rstd * __low2float(g23) + __low2float(b23),
                                            (v[u].w - mean) * rstd * __high2float(g23) + __high2float(b23));
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(__low2float(h01)), fabsf(__high2float(h01))),
                           fmaxf(fabsf(__low2float(h23)), fabsf(__high2float(h23)))));
      hv[u].x = *reinterpret_cast<const uint32_t*>(&h01);
      hv[u].y = *reinterpret_cast<const uint32_t*>(&h23);
    }
  }
  mx = row_reduce<true>(mx, rm.tpr, hd.red, cw, lane);
  const float scale = act_scale(mx);
  if (rm.active && rm.j == 0) hd.xscale[rm.b] = scale;
#pragma unroll
  for (int u = 0; u < kLnRegVec; ++u) {
    const int c = rm.j + u * rm.tpr;
    if (rm.active && c < K4 && c >= row0 && c < row0 + nrows) {
      const __half2 h01 = *reinterpret_cast<const __half2*>(&hv[u].x), h23 = *reinterpret_cast<const __half2*>(&hv[u].y);
      sx[rm.b * xrw + (c - row0)] = quant_byte(__low2float(h01), scale) | (quant_byte(__high2float(h01), scale) << 8) |
                                    (quant_byte(__low2float(h23), scale) << 16) |
                                    (quant_byte(__high2float(h23), scale) << 24);
    }
  }
  for (int w = max(0, K4 - row0) + ctid; w < nrows; w += 128)  // zero words past K (last split)
    for (int b = 0; b < p.B; ++b) sx[b * xrw + w] = 0u;
}

// PRO_QUANT with the row max from the producer (p.amax_in): the first x-slice loads are issued
// before the scale is read, so the two L2 round trips overlap.
__device__ __forceinline__ void fill_x_quant_pre(const Params& p, uint32_t* sx, Header& hd, int row0, int nrows,
                                                 int ctid, long long c_rel = 0) {
  constexpr int kPre = 8;
  const int K = p.K;
  const int xrw = p.x_row_words;
  const int total = p.B * nrows;
  const __half* x = static_cast<const __half*>(p.x);
  uint2 r[kPre];
#pragma unroll
  for (int j = 0; j < kPre; ++j) {
    const int i = ctid + 128 * j;
    r[j] = make_uint2(0u, 0u);
    if (i < total) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 4;
      if (k < K) r[j] = __ldcg(reinterpret_cast<const uint2*>(x + static_cast<size_t>(b) * p.x_ld + k));
    }
  }
  if (ctid < p.B) hd.xscale[ctid] = act_scale(amax_from_stripes(p.amax_in, ctid));
  consumer_bar();
  auto qword = [](uint2 u, float scale) {
    const __half2 h01 = *reinterpret_cast<const __half2*>(&u.x), h23 = *reinterpret_cast<const __half2*>(&u.y);
    return quant_byte(__low2float(h01), scale) | (quant_byte(__high2float(h01), scale) << 8) |
           (quant_byte(__low2float(h23), scale) << 16) | (quant_byte(__high2float(h23), scale) << 24);
  };
#pragma unroll
  for (int j = 0; j < kPre; ++j) {
    const int i = ctid + 128 * j;
    if (i < total) {
      const int b = i / nrows, w = i - b * nrows;
      sx[b * xrw + w] = (row0 + w) * 4 < K ? qword(r[j], hd.xscale[b]) : 0u;
    }
  }
  if (total > 128 * kPre)
    chunked(ctid + 128 * kPre, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 4;
      return k < K ? __ldcg(reinterpret_cast<const uint2*>(x + static_cast<size_t>(b) * p.x_ld + k)) : make_uint2(0u, 0u);
    }, [&](int i, uint2 u) {
      const int b = i / nrows, w = i - b * nrows;
      sx[b * xrw + w] = (row0 + w) * 4 < K ? qword(u, hd.xscale[b]) : 0u;
    });
}

template <bool kInt8, int kChunk = 8>
__device__ void fill_x_slice(const Params& p, uint32_t* sx, const Header& hd, int row0, int nrows, int ctid) {
  const int K = p.K;
  const int xrw = p.x_row_words;
  const int total = p.B * nrows;
  auto put = [&](int i, uint32_t word) {
    const int b = i / nrows;
    sx[b * xrw + (i - b * nrows)] = word;
  };
  if (p.pro == PRO_LN) {
    const ResidualView rv = residual_view(p);
    // item i -> (b, packed row): fp16 takes 2 consecutive k (half of a float4), int8 all 4
    chunked<kChunk>(ctid, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * (kInt8 ? 4 : 2);
      return k < K ? rv.load4(b, k & ~3) : make_float4(0.f, 0.f, 0.f, 0.f);  // K % 8 == 0 on this path
    }, [&](int i, float4 v) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * (kInt8 ? 4 : 2);
      uint32_t word = 0;
      if (k < K) {
        const float mean = hd.mean[b], rstd = hd.rstd[b];
        if (!kInt8) {
          const float va = (k & 2) ? v.z : v.x, vb = (k & 2) ? v.w : v.y;
          word = pack_h2(ln_apply(va, mean, rstd, p.ln_g, p.ln_b, k), ln_apply(vb, mean, rstd, p.ln_g, p.ln_b, k + 1));
        } else {
          const float vv[4] = {v.x, v.y, v.z, v.w};
          const float scale = hd.xscale[b];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float y = __half2float(__float2half_rn(ln_apply(vv[e], mean, rstd, p.ln_g, p.ln_b, k + e)));
            word |= quant_byte(y, scale) << (8 * e);
          }
        }
      }
      put(i, word);
    });
  } else if (p.pro == PRO_F16) {
    const __half* x = static_cast<const __half*>(p.x);
    const bool vec = (p.x_ld % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0;
    chunked<kChunk>(ctid, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 2;
      const size_t base = static_cast<size_t>(b) * p.x_ld + k;
      uint32_t word = 0;
      if (k + 1 < K && vec) {
        word = __ldcg(reinterpret_cast<const unsigned int*>(x + base));
      } else if (k < K) {
        const __half lo = __ldcg(x + base);
        const __half hi = (k + 1 < K) ? __ldcg(x + base + 1) : __float2half(0.f);
        word = static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
      }
      return word;
    }, put);
  } else if (p.pro == PRO_I8) {
    const int8_t* x = static_cast<const int8_t*>(p.x);
    const bool vec = (p.x_ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0;
    chunked<kChunk>(ctid, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 4;
      const size_t base = static_cast<size_t>(b) * p.x_ld + k;
      uint32_t word = 0;
      if (k + 3 < K && vec) {
        word = __ldcg(reinterpret_cast<const unsigned int*>(x + base));
      } else {
        for (int e = 0; e < 4; ++e)
          if (k + e < K)
            word |= static_cast<uint32_t>(static_cast<uint8_t>(__ldcg(reinterpret_cast<const signed char*>(x) + base + e)))
                    << (8 * e);
      }
      return word;
    }, put);
  } else {  // PRO_QUANT: fp16 x, per-token scale in hd.xscale
    const __half* x = static_cast<const __half*>(p.x);
    const bool vec = (p.x_ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 7) == 0;
    chunked<kChunk>(ctid, total, [&](int i) {
      const int b = i / nrows;
      const int k = (row0 + i - b * nrows) * 4;
      const size_t base = static_cast<size_t>(b) * p.x_ld + k;
      uint2 u = make_uint2(0u, 0u);
      if (vec && k + 3 < K) {
        u = __ldcg(reinterpret_cast<const uint2*>(x + base));
      } else {
        unsigned short hs[4] = {0, 0, 0, 0};
        for (int e = 0; e < 4; ++e)
          if (k + e < K) hs[e] = __half_as_ushort(__ldcg(x + base + e));
        u = make_uint2(hs[0] | (static_cast<uint32_t>(hs[1]) << 16), hs[2] | (static_cast<uint32_t>(hs[3]) << 16));
      }
      return u;
    }, [&](int i, uint2 u) {
      const int b = i / nrows;
      const float scale = hd.xscale[b];
      const __half2 h01 = *reinterpret_cast<const __half2*>(&u.x);
      const __half2 h23 = *reinterpret_cast<const __half2*>(&u.y);
      put(i, quant_byte(__low2float(h01), scale) | (quant_byte(__high2float(h01), scale) << 8) |
                 (quant_byte(__low2float(h23), scale) << 16) | (quant_byte(__high2float(h23), scale) << 24));
    });
  }
}

__device__ __forceinline__ __half2 bits_h2(uint32_t u) { return *reinterpret_cast<const __half2*>(&u); }
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }

// int8 x4 (one packed weight word: 4 consecutive k) -> two fp16 pairs, exact:
// bytes (s + 128) under a 0x64 exponent byte are 1024 + s + 128 in fp16; subtract 1152.
// kBiased: the word already holds the biased bytes s + 128 (the decode model's W8A16 weights are
// stored that way, packed_weights_bias), which saves the XOR -- one of five widening instructions.
template <bool kBiased = false>
__device__ __forceinline__ void i8x4_to_h2x2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t u = kBiased ? w : (w ^ 0x80808080u);
  const uint32_t l = __byte_perm(u, 0x64646464u, 0x4140);
  const uint32_t h = __byte_perm(u, 0x64646464u, 0x4342);
  const __half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
  const __half2 lf = __hsub2(*reinterpret_cast<const __half2*>(&l), bias);
  const __half2 hf = __hsub2(*reinterpret_cast<const __half2*>(&h), bias);
  lo = *reinterpret_cast<const uint32_t*>(&lf);
  hi = *reinterpret_cast<const uint32_t*>(&hf);
}

// ------------------------------------------------------------------ consumer loop
// Accumulates `n_iters` ring stages into acc[j][bt][*] (warp `cw` owns 32 output columns).
// The ring position (s, phase) persists across calls.  Inside a k-step of 8 packed rows the MMA
// k-slot t reads smem row 2t (t+4 reads 2t+1), a k permutation applied to both operands that
// keeps every fragment read conflict-free under the 128-byte TMA swizzle.
// kA16 (with kInt8): W8A16 -- the int8 weight words are widened to fp16 pairs in registers and
// multiplied by fp16 x with mma.m16n8k16 (fp32 accumulate).  Per 16-k step thread t owns packed
// row 4*kk + t (4 consecutive k): weight word -> (a0, a2) / (a1, a3), x word pair 2*(4kk + t)
// -> (b0, b1), the same k assignment on both operands.
// kA16: 0 = not W8A16; 1 = W8A16 over signed int8 words; 2 = W8A16 over biased (s + 128) words.
template <bool kInt8, int kNB8, int kA16 = 0>
struct Consumer {
  using Acc = typename std::conditional<kInt8 && !kA16, int, float>::type;
  Acc acc[2][kNB8][4];
  // MMA row m of block j (A-fragment rows g and g + 8 of lane (g, t)) is output column
  // col(j, m) = 4 (m mod 8) + 2 j + (m >= 8) of the warp's 32: a lane's four A words of one packed
  // row are the 16 contiguous bytes of columns 4g .. 4g+3 -- ONE 128-bit shared load instead of
  // four 32-bit ones (the 128B swizzle moves whole 16-byte chunks; the 32 lanes of a load cover
  // 4 rows x 128 B, the minimum 4 wavefronts).  Word 2j + h of the chunk = block j, row g + 8h.
  uint32_t aoff4[2];  // [par] byte offset of the lane's chunk (kA16: par = parity of the 16-k step)
  int g, t;

  __device__ __forceinline__ void init(int lane) {
    g = lane >> 2;
    t = lane & 3;
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const int r = kA16 ? 4 * par + t : 2 * t + par;
      aoff4[par] = r * 128 + ((g ^ r) << 4);
    }
  }
  // output column (within the warp's 32) of accumulator element q of block j
  __device__ __forceinline__ int acc_col(int j, int q) const { return 4 * g + 2 * j + (q >= 2 ? 1 : 0); }
  // W8A16 main loop; xword(it, kk, bt) returns the (b0, b1) x words of batch tile bt.
  // `step` > 1: this warp group consumes every step-th ring slot (the persistent step kernel's
  // interleaved consumer groups; stages % step == 0).
  // K-group scales (gs != nullptr): one int8 stage is one 128-k group; gs points at the group of
  // the first stage for this warp's 32 columns ([group][gs_ld] fp16, gs_valid columns readable).
  // Each group's exact int8 x fp16 products accumulate in fp32 (accg), then acc += s_group * accg
  // per column at the stage end (the row scale is then 1).
  // `pre(s, it)` (optional) runs on every consumer thread right after stage s arrived, before its
  // MMAs (the LayerNorm-streaming plan normalises the stage's residual boxes there).
  struct NoPre {
    __device__ __forceinline__ void operator()(int, int) const {}
  };
  template <class XWord, class Pre = NoPre>
  __device__ __forceinline__ void run_a16(const uint8_t* ring, int stage_bytes, Header& hd, int stages, int& s,
                                          uint32_t& phase, int n_iters, int cw, int lane, XWord xword, int step = 1,
                                          const __half* gs = nullptr, int gs_ld = 0, int gs_valid = 0, Pre pre = Pre()) {
    // K-group scales are a compile-time variant (kA16 & 4): a kernel holding both loops runs the
    // row-scale one measurably slower in the step (GPT-J W8A16 B=1 attn-out 6.2 -> 11.1 us per layer)
    if constexpr ((kA16 & 4) != 0)
      run_a16_loop<true>(ring, stage_bytes, hd, stages, s, phase, n_iters, cw, lane, xword, step, gs, gs_ld, gs_valid,
                         pre);
    else
      run_a16_loop<false>(ring, stage_bytes, hd, stages, s, phase, n_iters, cw, lane, xword, step, nullptr, gs_ld,
                          gs_valid, pre);
  }
  template <bool kGroups, class XWord, class Pre>
  __device__ __forceinline__ void run_a16_loop(const uint8_t* ring, int stage_bytes, Header& hd, int stages, int& s,
                                               uint32_t& phase, int n_iters, int cw, int lane, XWord xword, int step,
                                               const __half* gs, int gs_ld, int gs_valid, Pre pre) {
    const uint8_t* wbox = ring + cw * kBoxBytes;
    __half2 gsc[2][2], gsn[2][2];
    auto load_gs = [&](int i, __half2 (&o)[2][2]) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 4 * g + 2 * j + h;
          o[j][h] = __half2half2(c < gs_valid ? gs[static_cast<size_t>(i) * gs_ld + c] : __ushort_as_half(0));
        }
    };
    float accg[kGroups ? 2 : 1][kGroups ? kNB8 : 1][4];  // this group's exact int8 x fp16 sums (fp32)
    if constexpr (kGroups) {
      if (n_iters > 0) load_gs(0, gsc);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
          for (int q = 0; q < 4; ++q) accg[j][bt][q] = 0.f;
    }
    for (int it = 0; it < n_iters; ++it) {
      if constexpr (kGroups) {
        if (it + 1 < n_iters) load_gs(it + 1, gsn);
      }
      ptx::mbar_wait(&hd.full[s], phase);
      pre(s, it);
      const uint8_t* sw = wbox + s * stage_bytes;
#pragma unroll
      for (int kk = 0; kk < kRowsPerStage / 4; ++kk) {
        uint2 bx[kNB8];
#pragma unroll
        for (int bt = 0; bt < kNB8; ++bt) bx[bt] = xword(s, it, kk, bt);
        const uint8_t* a = sw + (kk >> 1) * 8 * 128;
        const uint4 w4 = *reinterpret_cast<const uint4*>(a + aoff4[kk & 1]);
        const uint32_t wq[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t a0, a1, a2, a3;
          i8x4_to_h2x2<(kA16 & 3) == 2>(wq[2 * j], a0, a2);
          i8x4_to_h2x2<(kA16 & 3) == 2>(wq[2 * j + 1], a1, a3);
#pragma unroll
          for (int bt = 0; bt < kNB8; ++bt) {
            if constexpr (kGroups)
              ptx::mma_f16(accg[j][bt], a0, a1, a2, a3, bx[bt].x, bx[bt].y);
            else if constexpr (kA16)
              ptx::mma_f16(acc[j][bt], a0, a1, a2, a3, bx[bt].x, bx[bt].y);
          }
        }
      }
      if constexpr (kGroups) {  // the stage is one 128-k group: acc += s_group x (sum q x) per column
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[j][bt][q] = fmaf(accg[j][bt][q], __low2float(gsc[j][q >> 1]), acc[j][bt][q]);
              accg[j][bt][q] = 0.f;
            }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&hd.empty[s]);
      if ((s += step) >= stages) {
        s -= stages;
        phase ^= 1;
      }
      if constexpr (kGroups) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) gsc[j][h] = gsn[j][h];
      }
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][bt][e] = 0;
  }
  __device__ __forceinline__ void run(const uint8_t* ring, Header& hd, int stages, int& s, uint32_t& phase,
                                      int n_iters, const uint32_t* sx, int xrw, int B, int cw, int lane, int step = 1) {
    const uint32_t* xrow[kNB8];
    bool xvalid[kNB8];
#pragma unroll
    for (int bt = 0; bt < kNB8; ++bt) {
      xvalid[bt] = bt * 8 + g < B;
      xrow[bt] = sx + (bt * 8 + g) * xrw + 2 * t;
    }
    const uint8_t* wbox = ring + cw * kBoxBytes;
    for (int it = 0; it < n_iters; ++it) {
      ptx::mbar_wait(&hd.full[s], phase);
      const uint8_t* sw = wbox + s * kStageBytes;
      const int xr0 = it * kRowsPerStage * step;
#pragma unroll
      for (int ks = 0; ks < kRowsPerStage / 8; ++ks) {
        uint32_t b0[kNB8], b1[kNB8];
#pragma unroll
        for (int bt = 0; bt < kNB8; ++bt) {
          uint2 v = make_uint2(0u, 0u);
          if (xvalid[bt]) v = *reinterpret_cast<const uint2*>(xrow[bt] + xr0 + ks * 8);
          b0[bt] = v.x;
          b1[bt] = v.y;
        }
        const uint8_t* a = sw + ks * 8 * 128;
        const uint4 w0 = *reinterpret_cast<const uint4*>(a + aoff4[0]);  // packed row 2t
        const uint4 w1 = *reinterpret_cast<const uint4*>(a + aoff4[1]);  // packed row 2t + 1
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t a0 = j == 0 ? w0.x : w0.z;
          const uint32_t a1 = j == 0 ? w0.y : w0.w;
          const uint32_t a2 = j == 0 ? w1.x : w1.z;
          const uint32_t a3 = j == 0 ? w1.y : w1.w;
#pragma unroll
          for (int bt = 0; bt < kNB8; ++bt) {
            if constexpr (kInt8 && !kA16)
              ptx::mma_s8(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
            else
              ptx::mma_f16(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&hd.empty[s]);
      if ((s += step) >= stages) {
        s -= stages;
        phase ^= 1;
      }
    }
  }
  // x-streaming variant: stage s holds the 4 weight boxes then the x box (B rows x 128 B,
  // 128B-swizzled: 16-byte chunk c of row r sits at chunk c ^ (r & 7)).
  template <class Pre = NoPre>
  __device__ __forceinline__ void run_xs(const uint8_t* ring, Header& hd, int stages, int& s, uint32_t& phase,
                                         int n_iters, int B, int cw, int lane, int stage_bytes = kStageBytesXS,
                                         int x_off = kStageBytes, Pre pre = Pre()) {
    bool xvalid[kNB8];
    uint32_t xoff[kNB8][kRowsPerStage / 8];
#pragma unroll
    for (int bt = 0; bt < kNB8; ++bt) {
      const int r = bt * 8 + g;
      xvalid[bt] = r < B;
#pragma unroll
      for (int ks = 0; ks < kRowsPerStage / 8; ++ks)
        xoff[bt][ks] = x_off + r * 128 + (((2 * ks + (t >> 1)) ^ (r & 7)) << 4) + ((t & 1) << 3);
    }
    const uint8_t* wbox = ring + cw * kBoxBytes;
    for (int it = 0; it < n_iters; ++it) {
      ptx::mbar_wait(&hd.full[s], phase);
      pre(s, it);
      const uint8_t* stage = ring + s * stage_bytes;
      const uint8_t* sw = wbox + s * stage_bytes;
#pragma unroll
      for (int ks = 0; ks < kRowsPerStage / 8; ++ks) {
        uint32_t b0[kNB8], b1[kNB8];
#pragma unroll
        for (int bt = 0; bt < kNB8; ++bt) {
          uint2 v = make_uint2(0u, 0u);
          if (xvalid[bt]) v = *reinterpret_cast<const uint2*>(stage + xoff[bt][ks]);
          b0[bt] = v.x;
          b1[bt] = v.y;
        }
        const uint8_t* a = sw + ks * 8 * 128;
        const uint4 w0 = *reinterpret_cast<const uint4*>(a + aoff4[0]);  // packed row 2t
        const uint4 w1 = *reinterpret_cast<const uint4*>(a + aoff4[1]);  // packed row 2t + 1
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t a0 = j == 0 ? w0.x : w0.z;
          const uint32_t a1 = j == 0 ? w0.y : w0.w;
          const uint32_t a2 = j == 0 ? w1.x : w1.z;
          const uint32_t a3 = j == 0 ? w1.y : w1.w;
#pragma unroll
          for (int bt = 0; bt < kNB8; ++bt) {
            if constexpr (kInt8 && !kA16)
              ptx::mma_s8(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
            else
              ptx::mma_f16(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&hd.empty[s]);
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
    }
  }
  // part[b * ld + n] for this warp's 32 columns (n relative to the CTA tile).
  __device__ __forceinline__ void store(Acc* part, int ld, int B, int cw) const {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt) {
        const int n = cw * kWarpCols + acc_col(j, 0);  // elements 2, 3: column n + 1
        const int b = bt * 8 + 2 * t;
        if (b < B) {
          part[b * ld + n] = acc[j][bt][0];
          part[b * ld + n + 1] = acc[j][bt][2];
        }
        if (b + 1 < B) {
          part[(b + 1) * ld + n] = acc[j][bt][1];
          part[(b + 1) * ld + n + 1] = acc[j][bt][3];
        }
      }
  }
};

// ------------------------------------------------------------------ epilogue
__device__ __forceinline__ float gelu_tanh(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}

__device__ __forceinline__ void dequant_pair(const Params& p, const Header& hd, int b, int n, int s0, int s1,
                                             float& y0, float& y1) {
  const float xs = hd.xscale[b];
  y0 = __fmul_rn(__fmul_rn(static_cast<float>(s0), xs), p.w_scale[n]);
  y1 = (n + 1 < p.N) ? __fmul_rn(__fmul_rn(static_cast<float>(s1), xs), p.w_scale[n + 1]) : 0.f;
}
// Same with the two weight scales already loaded.
__device__ __forceinline__ void dequant_pair_ws(const Header& hd, int b, int s0, int s1, float2 ws, bool has1,
                                                float& y0, float& y1) {
  const float xs = hd.xscale[b];
  y0 = __fmul_rn(__fmul_rn(static_cast<float>(s0), xs), ws.x);
  y1 = has1 ? __fmul_rn(__fmul_rn(static_cast<float>(s1), xs), ws.y) : 0.f;
}

// Epilogue row statistics of one thread's outputs (registers), reduced per warp by row_stat_commit.
struct RowStat {
  long long s1 = 0, s2 = 0;  // fixed point, see kSumScale / kSqScale
  float amax = 0.f;
  __device__ __forceinline__ void add(float y) {
    s1 += __float2ll_rn(__fmul_rn(y, kSumScale));
    s2 += __float2ll_rn(__fmul_rn(__fmul_rn(y, y), kSqScale));
  }
};

// The whole warp holds row b's statistics of this CTA: reduce and store them (lane 0).
__device__ __forceinline__ void row_stat_commit(RowStat st, EpiStats& es, int b, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st.s1 += __shfl_xor_sync(0xffffffffu, st.s1, o);
    st.s2 += __shfl_xor_sync(0xffffffffu, st.s2, o);
  }
  const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(st.amax));
  if (lane == 0) {
    es.esum[b][0] = static_cast<unsigned long long>(st.s1);
    es.esum[b][1] = static_cast<unsigned long long>(st.s2);
    es.emax[b] = m;
  }
}

// Same for a group of `gp` lanes (power of two, aligned) holding row b: the group leader stores.
__device__ __forceinline__ void row_stat_commit_group(RowStat st, EpiStats& es, int b, int lane, int gp, bool valid) {
  unsigned m = __float_as_uint(st.amax);
  for (int o = gp >> 1; o > 0; o >>= 1) {
    st.s1 += __shfl_xor_sync(0xffffffffu, st.s1, o);
    st.s2 += __shfl_xor_sync(0xffffffffu, st.s2, o);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if (valid && (lane & (gp - 1)) == 0) {
    es.esum[b][0] = static_cast<unsigned long long>(st.s1);
    es.esum[b][1] = static_cast<unsigned long long>(st.s2);
    es.emax[b] = m;
  }
}

// One CTA's epilogue statistics -> the global stripes (after a block-wide barrier).
__device__ __forceinline__ void stats_flush(const Params& p, const EpiStats& es, int stripe) {
  if (p.ln_stats_out != nullptr && threadIdx.x < 2 * p.B) {
    const int b = threadIdx.x >> 1, j = threadIdx.x & 1;
    atomicAdd(reinterpret_cast<unsigned long long*>(p.ln_stats_out) + (stripe * kMaxB + b) * 2 + j, es.esum[b][j]);
  }
  if (p.amax_out != nullptr && threadIdx.x < p.B) atomicMax(p.amax_out + stripe * 32 + threadIdx.x, es.emax[threadIdx.x]);
}

// `st` (nullable) accumulates the statistics requested by p.ln_stats_out / p.amax_out;
// `rin` (nullable) holds the two residual values of EPI_RESID when the caller preloaded them.
__device__ __forceinline__ void epilogue_pair(const Params& p, int b, int n, float y0, float y1, bool has1,
                                              RowStat* st = nullptr, const float2* rin = nullptr) {
  if (p.bias) {
    y0 = __fadd_rn(y0, __half2float(p.bias[n]));
    if (has1) y1 = __fadd_rn(y1, __half2float(p.bias[n + 1]));
  }
  switch (p.epi) {
    case EPI_F32: {
      float* o = static_cast<float*>(p.out) + static_cast<size_t>(b) * p.out_ld + n;
      if (has1 && ((reinterpret_cast<uintptr_t>(o) & 7) == 0)) {
        *reinterpret_cast<float2*>(o) = make_float2(y0, y1);
      } else {
        o[0] = y0;
        if (has1) o[1] = y1;
      }
      break;
    }
    case EPI_RESID: {  // residual stream += y + bias (fp32, this column's only writer)
      float* o = static_cast<float*>(p.out) + static_cast<size_t>(b) * p.out_ld + n;
      const float r0 = __fadd_rn(rin ? rin->x : __ldcg(o), y0);
      o[0] = r0;
      if (st) st->add(r0);
      if (has1) {
        const float r1 = __fadd_rn(rin ? rin->y : __ldcg(o + 1), y1);
        o[1] = r1;
        if (st) st->add(r1);
      }
      break;
    }
    case EPI_F16:
    case EPI_GELU_F16: {
      if (p.epi == EPI_GELU_F16) {
        y0 = gelu_tanh(y0);
        y1 = gelu_tanh(y1);
      }
      __half* o = static_cast<__half*>(p.out) + static_cast<size_t>(b) * p.out_ld + n;
      const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
      if (has1 && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
        *reinterpret_cast<__half2*>(o) = __halves2half2(h0, h1);
      } else {
        o[0] = h0;
        if (has1) o[1] = h1;
      }
      if (st) {
        st->amax = fmaxf(st->amax, fabsf(__half2float(h0)));
        if (has1) st->amax = fmaxf(st->amax, fabsf(__half2float(h1)));
      }
      break;
    }
    case EPI_QKV: {
      // column n (even) -> section (0 q, 1 k, 2 v), head, dim i; (i, i+1) is a rotary pair
      const int hd = p.heads * p.head_dim;
      const int sec = n / hd;
      const int rem = n - sec * hd;
      const int head = rem / p.head_dim;
      const int i = rem - head * p.head_dim;
      const int pos = *p.pos;
      if (sec < 2) {  // GPT-J interleaved rotary embedding over the full head dim
        const float2 cs = p.rope[static_cast<size_t>(pos) * (p.head_dim / 2) + i / 2];
        const float r0 = __fsub_rn(__fmul_rn(y0, cs.x), __fmul_rn(y1, cs.y));
        const float r1 = __fadd_rn(__fmul_rn(y0, cs.y), __fmul_rn(y1, cs.x));
        y0 = r0;
        y1 = r1;
      }
      const __half2 h = __floats2half2_rn(y0, y1);
      if (sec == 0) {
        *reinterpret_cast<__half2*>(p.q_out + static_cast<size_t>(b) * hd + rem) = h;
      } else {
        __half* cache = sec == 1 ? p.k_cache : p.v_cache;
        const size_t off = ((static_cast<size_t>(b) * p.heads + head) * p.max_seq + pos) * p.head_dim + i;
        *reinterpret_cast<__half2*>(cache + off) = h;
      }
      break;
    }
    default:
      break;
  }
}

}  // namespace dev
}  // namespace gemm
}  // namespace dsinf
