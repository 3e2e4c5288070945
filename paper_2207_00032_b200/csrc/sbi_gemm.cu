// SBI-GeMM on sm_100a (infersim gemm.hpp:65-202).
//
// One CTA computes a 128-column output tile over one K split; the splits of a column tile
// form a thread-block cluster and reduce through distributed shared memory (the paper's
// "second kernel" cross-tile reduction, gemm.hpp:194-198, done in-cluster instead).
//
//   warp 0      producer: streams packed weight rows HBM -> smem with 1-D bulk async copies
//               (TMA engine) into a multi-stage mbarrier ring.  Weights do not depend on the
//               previous kernel, so the ring is filled *before* griddepcontrol.wait (PDL).
//   warps 1..4  consumers: Deep-Fusion prologue (LayerNorm / residual add / quantisation)
//               into a smem x slice, then warp MMAs over the ring.
//
// The reference packed layout [ceil(K/M)][N][M] (gemm.hpp:108-111) is used unchanged: one
// 32-bit word holds M=2 fp16 (or M=4 int8) consecutive k of one output column, which is
// exactly one A-fragment register of mma.m16n8k16.f16 (mma.m16n8k32.s8).  Row r of a stage
// is one bulk copy of 128 contiguous words; rows are padded to 136 words in smem so the
// fragment reads (row t, column g) hit 32 distinct banks.
#include <algorithm>
#include <cstdio>
#include <string>
#include <type_traits>

#include "common.h"
#include "ptx.cuh"
#include "sbi_gemm.cuh"

namespace dsinf {
namespace gemm {

namespace {

struct Header {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  float xscale[kMaxB];
  float mean[kMaxB];
  float rstd[kMaxB];
  float red[8];
};
static_assert(sizeof(Header) <= kHeaderBytes, "header too large");

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int next_pow2(int b) {
  int p = 1;
  while (p < b) p <<= 1;
  return p;
}

// Sum (or max) over the `tpr` consecutive consumer threads that own one batch row.  All
// threads of the row get the same bits (symmetric butterfly, then an in-order warp sum).
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
__device__ __forceinline__ uint32_t quant_byte(float x, float inv_unused, float scale) {
  (void)inv_unused;
  int q = __float2int_rn(__fdiv_rn(x, scale));
  q = max(-127, min(127, q));
  return static_cast<uint32_t>(q) & 0xffu;
}

__device__ __forceinline__ float act_scale(float maxabs) {
  return maxabs > 0.0f ? __fdiv_rn(maxabs, 127.0f) : 1.0f;
}

// Residual-stream element: r + (delta + delta_bias).
struct ResidualView {
  const float* r;
  const float* d;
  const __half* db;
  int K;
  __device__ __forceinline__ float4 load4(int b, int k) const {
    float4 v = *reinterpret_cast<const float4*>(r + static_cast<size_t>(b) * K + k);
    if (d) {
      float4 t = *reinterpret_cast<const float4*>(d + static_cast<size_t>(b) * K + k);
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

__device__ __forceinline__ float ln_apply(float v, float mean, float rstd, const __half* g, const __half* bta,
                                          int k) {
  return (v - mean) * rstd * __half2float(g[k]) + __half2float(bta[k]);
}

// ------------------------------------------------------------------ prologues
// Each writes this CTA's K slice of x into smem words sx[b * xrw + w], w in [0, rps).

template <bool kInt8>
__device__ void prologue_ln(const Params& p, uint32_t* sx, Header& hd, int k0, int ctid, int cw, int lane,
                            bool write_res) {
  const int Bp = next_pow2(p.B);
  const int tpr = 128 / Bp;
  const int b = ctid / tpr;
  const int j = ctid % tpr;
  const bool active = b < p.B;
  const int K = p.K;
  const ResidualView rv{p.res_in, p.res_delta, p.delta_bias, K};
  float c0 = 0.f, s1 = 0.f, s2 = 0.f;
  if (active) {
    c0 = rv.load4(b, 0).x;  // shift for a cancellation-free single pass
    for (int c = j; c < K / 4; c += tpr) {
      const float4 v = rv.load4(b, 4 * c);
      if (write_res) *reinterpret_cast<float4*>(p.res_out + static_cast<size_t>(b) * K + 4 * c) = v;
      const float d0 = v.x - c0, d1 = v.y - c0, d2 = v.z - c0, d3 = v.w - c0;
      s1 += (d0 + d1) + (d2 + d3);
      s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
  }
  s1 = row_reduce<false>(s1, tpr, hd.red, cw, lane);
  s2 = row_reduce<false>(s2, tpr, hd.red, cw, lane);
  const float inv_k = 1.0f / static_cast<float>(K);
  const float m1 = s1 * inv_k;
  const float var = fmaxf(s2 * inv_k - m1 * m1, 0.0f);
  const float mean = c0 + m1;
  const float rstd = 1.0f / sqrtf(var + p.ln_eps);
  const int rps = p.rows_per_split;
  uint32_t* row = sx + b * p.x_row_words;
  if (!kInt8) {
    if (active) {
      for (int w = j; w < rps; w += tpr) {
        const int k = k0 + 2 * w;
        uint32_t word = 0;
        if (k < K) {  // K % 8 == 0 on this path
          const float4 v = rv.load4(b, k & ~3);
          const float va = (k & 2) ? v.z : v.x, vb = (k & 2) ? v.w : v.y;
          word = pack_h2(ln_apply(va, mean, rstd, p.ln_g, p.ln_b, k), ln_apply(vb, mean, rstd, p.ln_g, p.ln_b, k + 1));
        }
        row[w] = word;
      }
    }
  } else {
    float mx = 0.f;
    if (active) {
      for (int c = j; c < K / 4; c += tpr) {
        const float4 v = rv.load4(b, 4 * c);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float y = __half2float(__float2half_rn(ln_apply(vv[i], mean, rstd, p.ln_g, p.ln_b, 4 * c + i)));
          mx = fmaxf(mx, fabsf(y));
        }
      }
    }
    mx = row_reduce<true>(mx, tpr, hd.red, cw, lane);
    const float scale = act_scale(mx);
    if (active) {
      if (j == 0) hd.xscale[b] = scale;
      for (int w = j; w < rps; w += tpr) {
        const int k = k0 + 4 * w;
        uint32_t word = 0;
        if (k < K) {
          const float4 v = rv.load4(b, k);
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float y = __half2float(__float2half_rn(ln_apply(vv[i], mean, rstd, p.ln_g, p.ln_b, k + i)));
            word |= quant_byte(y, 0.f, scale) << (8 * i);
          }
        }
        row[w] = word;
      }
    }
  }
}

__device__ __forceinline__ float ldh(const __half* x, size_t i) { return __half2float(x[i]); }

template <bool kInt8>
__device__ void prologue_load(const Params& p, uint32_t* sx, Header& hd, int k0, int ctid, int cw, int lane) {
  const int rps = p.rows_per_split;
  const int K = p.K;
  if (p.pro == PRO_F16) {
    const __half* x = static_cast<const __half*>(p.x);
    const bool vec = (p.x_ld % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0;
    for (int b = 0; b < p.B; ++b)
      for (int w = ctid; w < rps; w += 128) {
        const int k = k0 + 2 * w;
        uint32_t word = 0;
        const size_t base = static_cast<size_t>(b) * p.x_ld + k;
        if (k + 1 < K && vec) {
          word = *reinterpret_cast<const uint32_t*>(x + base);
        } else if (k < K) {
          const __half lo = x[base];
          const __half hi = (k + 1 < K) ? x[base + 1] : __float2half(0.f);
          word = static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
        }
        sx[b * p.x_row_words + w] = word;
      }
  } else if (p.pro == PRO_I8) {
    const int8_t* x = static_cast<const int8_t*>(p.x);
    const bool vec = (p.x_ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0;
    if (ctid < p.B) hd.xscale[ctid] = p.x_scale[ctid];
    for (int b = 0; b < p.B; ++b)
      for (int w = ctid; w < rps; w += 128) {
        const int k = k0 + 4 * w;
        uint32_t word = 0;
        const size_t base = static_cast<size_t>(b) * p.x_ld + k;
        if (k + 3 < K && vec) {
          word = *reinterpret_cast<const uint32_t*>(x + base);
        } else {
          for (int i = 0; i < 4; ++i)
            if (k + i < K) word |= (static_cast<uint32_t>(static_cast<uint8_t>(x[base + i]))) << (8 * i);
        }
        sx[b * p.x_row_words + w] = word;
      }
  } else {  // PRO_QUANT: fp16 in global, per-token int8 on the fly
    const __half* x = static_cast<const __half*>(p.x);
    const int Bp = next_pow2(p.B);
    const int tpr = 128 / Bp;
    const int b = ctid / tpr;
    const int j = ctid % tpr;
    const bool active = b < p.B;
    float mx = 0.f;
    if (active)
      for (int k = j; k < K; k += tpr) mx = fmaxf(mx, fabsf(ldh(x, static_cast<size_t>(b) * p.x_ld + k)));
    mx = row_reduce<true>(mx, tpr, hd.red, cw, lane);
    const float scale = act_scale(mx);
    if (active) {
      if (j == 0) hd.xscale[b] = scale;
      for (int w = j; w < rps; w += tpr) {
        const int k = k0 + 4 * w;
        uint32_t word = 0;
        for (int i = 0; i < 4; ++i)
          if (k + i < K) word |= quant_byte(ldh(x, static_cast<size_t>(b) * p.x_ld + k + i), 0.f, scale) << (8 * i);
        sx[b * p.x_row_words + w] = word;
      }
    }
  }
}

// ------------------------------------------------------------------ epilogue

__device__ __forceinline__ float gelu_tanh(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}

__device__ __forceinline__ void epilogue_pair(const Params& p, int b, int n, float y0, float y1, bool has1) {
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
    case EPI_F16:
    case EPI_GELU_F16: {
      if (p.epi == EPI_GELU_F16) {
        y0 = gelu_tanh(y0);
        y1 = gelu_tanh(y1);
      }
      __half* o = static_cast<__half*>(p.out) + static_cast<size_t>(b) * p.out_ld + n;
      if (has1 && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
        *reinterpret_cast<__half2*>(o) = __floats2half2_rn(y0, y1);
      } else {
        o[0] = __float2half_rn(y0);
        if (has1) o[1] = __float2half_rn(y1);
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

// ------------------------------------------------------------------ kernel

template <bool kInt8, int kNB8>
__global__ void __launch_bounds__(kThreads) sbi_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  Header& hd = *reinterpret_cast<Header*>(smem);
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + kHeaderBytes);
  uint32_t* ring = sx + 8 * kNB8 * p.x_row_words;  // 16-byte aligned (x_row_words % 4 == 0)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int split = blockIdx.y;
  const int nsplit = gridDim.y;
  const int n0 = tile * kColTile;
  const int row_begin = split * p.rows_per_split;
  const int row_end = min(p.rows, row_begin + p.rows_per_split);
  const int n_iters = (row_end - row_begin + kRowsPerStage - 1) / kRowsPerStage;
  const int stages = p.stages;

  ptx::pdl_trigger();  // dependents may launch and start streaming their own weights

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&hd.full[s], 1);
      ptx::mbar_init(&hd.empty[s], kConsumerWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ================= producer: weight rows -> smem ring
    const int ncols = min(kColTile, p.N - n0);
    const uint32_t row_bytes = static_cast<uint32_t>(ncols) * 4u;
    const uint64_t policy = ptx::policy_evict_first();
    for (int it = 0; it < n_iters; ++it) {
      const int s = it % stages;
      if (it == stages) ptx::pdl_wait();  // (weights never depend on the previous grid)
      if (it >= stages) ptx::mbar_wait(&hd.empty[s], ((it / stages) - 1) & 1);
      uint32_t* dst = ring + s * kStageWords;
      const int r0 = row_begin + it * kRowsPerStage;
      const int valid = min(kRowsPerStage, row_end - r0);
      if (lane >= valid) {  // K tail: zero rows so 0 * stale never yields NaN
        uint4* z = reinterpret_cast<uint4*>(dst + lane * kRowWords);
        for (int i = 0; i < kColTile / 4; ++i) z[i] = make_uint4(0, 0, 0, 0);
        ptx::fence_proxy_async_smem();
      }
      if (p.aligned) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_expect_tx(&hd.full[s], row_bytes * valid);
        __syncwarp();
        if (lane < valid)
          ptx::bulk_g2s(dst + lane * kRowWords, p.w + static_cast<size_t>(r0 + lane) * p.N + n0, row_bytes,
                        &hd.full[s], policy);
      } else {
        for (int r = 0; r < valid; ++r) {
          const uint32_t* src = p.w + static_cast<size_t>(r0 + r) * p.N + n0;
          for (int c = lane; c < ncols; c += 32) dst[r * kRowWords + c] = __ldg(src + c);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&hd.full[s]);
      }
    }
    if (n_iters <= stages) ptx::pdl_wait();
  } else {
    // ================= consumers
    const int cw = warp - 1;
    const int ctid = threadIdx.x - 32;
    ptx::pdl_wait();
    const int m = kInt8 ? 4 : 2;
    const int k0 = row_begin * m;
    if (p.pro == PRO_LN)
      prologue_ln<kInt8>(p, sx, hd, k0, ctid, cw, lane, p.res_out != nullptr && tile == 0 && split == 0);
    else
      prologue_load<kInt8>(p, sx, hd, k0, ctid, cw, lane);
    consumer_bar();

    const int g = lane >> 2;
    const int t = lane & 3;
    using Acc = typename std::conditional<kInt8, int, float>::type;
    Acc acc[2][kNB8][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][bt][e] = 0;

    const uint32_t* xrow[kNB8];
    bool xvalid[kNB8];
#pragma unroll
    for (int bt = 0; bt < kNB8; ++bt) {
      xvalid[bt] = bt * 8 + g < p.B;
      xrow[bt] = sx + (bt * 8 + g) * p.x_row_words + t;
    }
    const int colw = cw * 32 + g;
    for (int it = 0; it < n_iters; ++it) {
      const int s = it % stages;
      ptx::mbar_wait(&hd.full[s], (it / stages) & 1);
      const uint32_t* sw = ring + s * kStageWords + t * kRowWords + colw;
      const int xr0 = it * kRowsPerStage;
#pragma unroll
      for (int ks = 0; ks < kRowsPerStage / 8; ++ks) {
        uint32_t b0[kNB8], b1[kNB8];
#pragma unroll
        for (int bt = 0; bt < kNB8; ++bt) {
          b0[bt] = xvalid[bt] ? xrow[bt][xr0 + ks * 8] : 0u;
          b1[bt] = xvalid[bt] ? xrow[bt][xr0 + ks * 8 + 4] : 0u;
        }
        const uint32_t* a = sw + ks * 8 * kRowWords;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t a0 = a[j * 16];
          const uint32_t a1 = a[j * 16 + 8];
          const uint32_t a2 = a[4 * kRowWords + j * 16];
          const uint32_t a3 = a[4 * kRowWords + j * 16 + 8];
#pragma unroll
          for (int bt = 0; bt < kNB8; ++bt) {
            if constexpr (kInt8)
              ptx::mma_s8(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
            else
              ptx::mma_f16(acc[j][bt], a0, a1, a2, a3, b0[bt], b1[bt]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&hd.empty[s]);
    }
    consumer_bar();  // every consumer is done reading the ring
    // partials -> smem (reuses the ring): part[b][n]
    Acc* part = reinterpret_cast<Acc*>(ring);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt) {
        const int n = cw * 32 + j * 16 + g;
        const int b = bt * 8 + 2 * t;
        if (b < p.B) {
          part[b * kPartLd + n] = acc[j][bt][0];
          part[b * kPartLd + n + 8] = acc[j][bt][2];
        }
        if (b + 1 < p.B) {
          part[(b + 1) * kPartLd + n] = acc[j][bt][1];
          part[(b + 1) * kPartLd + n + 8] = acc[j][bt][3];
        }
      }
  }

  // ================= split-K reduction across the cluster (DSMEM) + epilogue
  if (nsplit > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  const int rank = split;  // cluster dims (1, nsplit, 1): rank == blockIdx.y
  const int cols_per_rank = kColTile / nsplit;
  const int c_begin = rank * cols_per_rank;
  const int pairs = cols_per_rank / 2;
  const uint8_t* part_base = reinterpret_cast<const uint8_t*>(ring);
  for (int item = threadIdx.x; item < p.B * pairs; item += kThreads) {
    const int b = item / pairs;
    const int c = c_begin + 2 * (item - b * pairs);
    const int n = n0 + c;
    if (n >= p.N) continue;
    const uint32_t off = static_cast<uint32_t>((b * kPartLd + c) * 4);
    float y0, y1;
    if constexpr (kInt8) {
      int s0 = 0, s1 = 0;
      for (int r = 0; r < nsplit; ++r) {
        const int2 v = ptx::ld_dsmem_i2(ptx::map_shared_rank(part_base + off, r));
        s0 += v.x;
        s1 += v.y;
      }
      const float xs = hd.xscale[b];
      y0 = __fmul_rn(__fmul_rn(static_cast<float>(s0), xs), p.w_scale[n]);
      y1 = (n + 1 < p.N) ? __fmul_rn(__fmul_rn(static_cast<float>(s1), xs), p.w_scale[n + 1]) : 0.f;
    } else {
      float2 acc2 = make_float2(0.f, 0.f);
      for (int r = 0; r < nsplit; ++r) {
        const float2 v = ptx::ld_dsmem_f2(ptx::map_shared_rank(part_base + off, r));
        acc2.x += v.x;
        acc2.y += v.y;
      }
      y0 = acc2.x;
      y1 = acc2.y;
    }
    epilogue_pair(p, b, n, y0, y1, n + 1 < p.N);
  }
  if (nsplit > 1) ptx::cluster_sync();  // keep our smem alive for remote readers
}

template <bool kInt8, int kNB8>
void launch_impl(const Params& p, const Plan& plan, cudaStream_t stream, bool pdl) {
  auto kern = sbi_gemm_kernel<kInt8, kNB8>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(plan.col_tiles, plan.ksplit, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeClusterDimension;
  attrs[na].val.clusterDim.x = 1;
  attrs[na].val.clusterDim.y = plan.ksplit;
  attrs[na].val.clusterDim.z = 1;
  ++na;
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, p));
}

template <bool kInt8, int kNB8>
void configure_one() {
  auto kern = sbi_gemm_kernel<kInt8, kNB8>;
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

}  // namespace

void configure() {
  configure_one<false, 1>();
  configure_one<false, 2>();
  configure_one<true, 1>();
  configure_one<true, 2>();
}

Plan make_plan(int N, int K, int B, bool int8_weights, int forced_split) {
  if (N < 1 || K < 1 || B < 1 || B > kMaxB) throw ConfigError("sbi_gemm: bad shape");
  const int m = int8_weights ? 4 : 2;
  const int rows = (K + m - 1) / m;
  Plan pl{};
  pl.col_tiles = (N + kColTile - 1) / kColTile;
  pl.nb8 = B <= 8 ? 1 : 2;
  const size_t x_budget = 64 * 1024;
  auto rps_for = [&](int s) {
    int r = (rows + s - 1) / s;
    return (r + kRowsPerStage - 1) / kRowsPerStage * kRowsPerStage;
  };
  auto x_bytes = [&](int rps) { return static_cast<size_t>(8 * pl.nb8) * (rps + 4) * 4; };
  auto valid = [&](int s) {
    const int rps = rps_for(s);
    if ((rows + rps - 1) / rps != s) return false;  // no empty split
    return x_bytes(rps) <= x_budget;
  };
  int chosen = 0;
  if (forced_split > 0) {
    if (forced_split != 1 && forced_split != 2 && forced_split != 4 && forced_split != 8 && forced_split != 16)
      throw ConfigError("ksplit must be one of {1, 2, 4, 8, 16}");
    if (!valid(forced_split)) throw ConfigError("ksplit not valid for this shape");
    chosen = forced_split;
  } else {
    const int target = 2 * 148;  // >= 2 resident CTAs per SM keeps enough bytes in flight
    for (int s = 1; s <= 16; s <<= 1) {
      if (!valid(s)) continue;
      chosen = s;
      if (pl.col_tiles * s >= target) break;
    }
    if (chosen == 0) throw ConfigError("sbi_gemm: K too large for the x slice budget");
  }
  pl.ksplit = chosen;
  pl.rows_per_split = rps_for(chosen);
  const int iters = pl.rows_per_split / kRowsPerStage;
  const size_t stage_bytes = static_cast<size_t>(kStageWords) * 4;
  const size_t fixed = kHeaderBytes + x_bytes(pl.rows_per_split);
  // ring depth: up to 4 stages, bounded so ~2 CTAs fit per SM
  int st = std::min(4, std::max(1, iters));
  while (st > 2 && fixed + st * stage_bytes > 110 * 1024) --st;
  pl.stages = st;
  const size_t part_bytes = static_cast<size_t>(kMaxB) * kPartLd * 4;
  pl.smem_bytes = fixed + std::max(static_cast<size_t>(st) * stage_bytes, part_bytes);
  return pl;
}

void launch(const Params& p_in, const Plan& plan, bool int8_weights, cudaStream_t stream, bool pdl) {
  Params p = p_in;
  p.rows_per_split = plan.rows_per_split;
  p.stages = plan.stages;
  p.x_row_words = plan.rows_per_split + 4;
  p.aligned = (p.N % 4) == 0 && (reinterpret_cast<uintptr_t>(p.w) & 15) == 0;
  if (p.B < 1 || p.B > kMaxB) throw ConfigError("sbi_gemm: batch must be 1..16 per launch");
  if (p.pro == PRO_LN && (p.K % 8) != 0) throw ConfigError("LayerNorm prologue needs K % 8 == 0");
  if (int8_weights) {
    if (plan.nb8 == 1)
      launch_impl<true, 1>(p, plan, stream, pdl);
    else
      launch_impl<true, 2>(p, plan, stream, pdl);
  } else {
    if (plan.nb8 == 1)
      launch_impl<false, 1>(p, plan, stream, pdl);
    else
      launch_impl<false, 2>(p, plan, stream, pdl);
  }
}

}  // namespace gemm
}  // namespace dsinf
