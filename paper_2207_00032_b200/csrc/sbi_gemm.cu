// SBI-GeMM on sm_100a (infersim gemm.hpp:65-202).
//
// One CTA computes a 128-column output tile over one K split; the splits of a column tile
// form a thread-block cluster and reduce through distributed shared memory (the paper's
// "second kernel" cross-tile reduction, gemm.hpp:194-198, done in-cluster instead).
//
//   warp 0      producer: one elected thread streams the packed weights HBM -> smem with 2-D
//               tensor TMA (4 boxes of 32 rows x 32 words per 16 KB stage) into an mbarrier
//               ring.  Weights do not depend on the previous kernel, so the ring is filled
//               *before* griddepcontrol.wait (programmatic dependent launch).
//   warps 1..4  consumers: Deep-Fusion prologue (LayerNorm / residual add / quantisation)
//               into a smem x slice, then warp MMAs over the ring.
//
// The reference packed layout [ceil(K/M)][N][M] (gemm.hpp:108-111) is used unchanged: one
// 32-bit word holds M=2 fp16 (or M=4 int8) consecutive k of one output column, which is
// exactly one A-fragment register of mma.m16n8k16.f16 (mma.m16n8k32.s8).  TMA writes each box
// with the 128-byte swizzle; inside a k-step of 8 packed rows the MMA k-slot t reads smem row
// 2t (and t+4 reads 2t+1) — a k permutation applied to both operands — which makes every
// fragment read hit 32 distinct banks under that swizzle.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>

#include <cudaTypedefs.h>

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
__device__ __forceinline__ uint32_t quant_byte(float x, float scale) {
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
#pragma unroll 4
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
#pragma unroll 2
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
            word |= quant_byte(y, scale) << (8 * i);
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
          if (k + i < K) word |= quant_byte(ldh(x, static_cast<size_t>(b) * p.x_ld + k + i), scale) << (8 * i);
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
// Dynamic smem (base rounded up to 1024 B for the 128B swizzle):
//   [ring: stages x 16 KB] [header 1 KB] [x slice: 8*kNB8 rows x x_row_words words]
// After the main loop the ring is reused for the split-K partials part[b][n].

template <bool kInt8, int kNB8>
__global__ void __launch_bounds__(kThreads) sbi_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  uint8_t* ring = smem;
  Header& hd = *reinterpret_cast<Header*>(smem + stages * kStageBytes);
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + stages * kStageBytes + kHeaderBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int split = blockIdx.y;
  const int nsplit = gridDim.y;
  const int n0 = tile * kColTile;
  const int row_begin = split * p.rows_per_split;
  const int row_end = min(p.rows, row_begin + p.rows_per_split);
  const int n_iters = (row_end - row_begin + kRowsPerStage - 1) / kRowsPerStage;

  if (threadIdx.x == 0) {
    ptx::prefetch_tensormap(&p.tmap);
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&hd.full[s], 1);
      ptx::mbar_init(&hd.empty[s], kConsumerWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ================= producer: one elected thread issues 4 TMA boxes per stage
    if (lane == 0) {
      const uint64_t policy = ptx::policy_evict_first();
      int s = 0;
      uint32_t phase = 0;
      for (int it = 0; it < n_iters; ++it) {
        if (it == stages) ptx::pdl_wait();  // first `stages` loads run ahead of the dependency
        if (it >= stages) ptx::mbar_wait(&hd.empty[s], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&hd.full[s], kStageBytes);
        const int r0 = row_begin + it * kRowsPerStage;
        uint8_t* dst = ring + s * kStageBytes;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w)
          ptx::tma_load_2d(dst + w * kBoxBytes, &p.tmap, n0 + w * kWarpCols, r0, &hd.full[s], policy);
        if (++s == stages) {
          s = 0;
          phase ^= 1;
        }
      }
      if (n_iters <= stages) ptx::pdl_wait();
    } else {
      ptx::pdl_wait();
    }
    // All of this CTA's weight loads are issued: let the next kernel launch and start streaming
    // its own weights into the tail of this one (triggering at kernel start instead lets a
    // cascade of dependents occupy SMs and steal bandwidth from the critical kernel).
    ptx::pdl_trigger();
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

    // x words: b0 = slice row 2t, b1 = row 2t+1 of each k-step (one 8-byte load)
    const uint32_t* xrow[kNB8];
    bool xvalid[kNB8];
#pragma unroll
    for (int bt = 0; bt < kNB8; ++bt) {
      xvalid[bt] = bt * 8 + g < p.B;
      xrow[bt] = sx + (bt * 8 + g) * p.x_row_words + 2 * t;
    }
    // A words inside this warp's 128B-swizzled box: row r = 8*ks + 2t + par, column c = 16j + 8h + g
    //   byte = r*128 + ((c/4) ^ (r%8))*16 + (c%4)*4, and r%8 = 2t + par does not depend on ks.
    uint32_t aoff[2][2][2];  // [j][h][par]
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int par = 0; par < 2; ++par) {
          const int r = 2 * t + par;
          const int c = 16 * j + 8 * h + g;
          aoff[j][h][par] = r * 128 + (((c >> 2) ^ r) << 4) + (c & 3) * 4;
        }
    const uint8_t* wbox = ring + cw * kBoxBytes;
    int s = 0;
    uint32_t phase = 0;
    for (int it = 0; it < n_iters; ++it) {
      ptx::mbar_wait(&hd.full[s], phase);
      const uint8_t* sw = wbox + s * kStageBytes;
      const int xr0 = it * kRowsPerStage;
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
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t a0 = *reinterpret_cast<const uint32_t*>(a + aoff[j][0][0]);
          const uint32_t a1 = *reinterpret_cast<const uint32_t*>(a + aoff[j][1][0]);
          const uint32_t a2 = *reinterpret_cast<const uint32_t*>(a + aoff[j][0][1]);
          const uint32_t a3 = *reinterpret_cast<const uint32_t*>(a + aoff[j][1][1]);
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
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
    }
    ptx::pdl_trigger();
    consumer_bar();  // every consumer is done reading the ring
    // partials -> smem (reuses the ring): part[b][n]
    Acc* part = reinterpret_cast<Acc*>(ring);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt) {
        const int n = cw * kWarpCols + j * 16 + g;
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
  const uint8_t* part_base = ring;
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable");
  return fn;
}

}  // namespace

void make_weight_map(CUtensorMap* map, const void* w_packed, int N, int rows) {
  if (N % 4 != 0) throw ConfigError("sbi_gemm: out_dim must be a multiple of 4 (16-byte TMA row stride)");
  if ((reinterpret_cast<uintptr_t>(w_packed) & 15) != 0) throw ConfigError("sbi_gemm: weights must be 16-byte aligned");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kWarpCols), static_cast<cuuint32_t>(kRowsPerStage)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(w_packed), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
}

void configure() {
  configure_one<false, 1>();
  configure_one<false, 2>();
  configure_one<true, 1>();
  configure_one<true, 2>();
}

namespace {

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Co-resident clusters of `split` CTAs for this kernel / smem (cached; 0 when unknown).
int resident_clusters(bool int8_weights, int nb8, int split, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<bool, int, int, size_t>, int> cache;
  const auto key = std::make_tuple(int8_weights, nb8, split, smem);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const void* kern = nullptr;
  if (int8_weights)
    kern = nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1>)
                    : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2>);
  else
    kern = nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<false, 1>)
                    : reinterpret_cast<const void*>(sbi_gemm_kernel<false, 2>);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, split, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 1;
  attr.val.clusterDim.y = split;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[key] = n;
  return n;
}

}  // namespace

// B200 launch plan (the device half of derive_schedule, gemm.hpp:65-96): like the reference it
// splits K only when the output tiles alone cannot occupy the machine, but it sizes the split
// so that the whole grid is ONE wave of co-resident clusters (every CTA starts streaming at
// once, no tail wave) and reduces the split in-cluster.
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
  auto x_bytes = [&](int rps) { return static_cast<size_t>(B) * (rps + 8) * 4; };
  auto valid = [&](int s) {
    const int rps = rps_for(s);
    if ((rows + rps - 1) / rps != s) return false;  // no empty split
    return x_bytes(rps) <= x_budget;
  };
  const int max_stages = std::max(1, std::min(kMaxStages, env_int("DSINF_STAGES", 4)));
  auto smem_for = [&](int s, int* stages_out) {
    const int rps = rps_for(s);
    const int iters = rps / kRowsPerStage;
    const size_t fixed = 1024 /*alignment slack*/ + kHeaderBytes + x_bytes(rps);
    int st = std::min(max_stages, std::max(1, iters));
    while (st > 2 && fixed + st * static_cast<size_t>(kStageBytes) > 110 * 1024) --st;
    if (stages_out) *stages_out = st;
    const size_t part_bytes = static_cast<size_t>(B) * kPartLd * 4;
    return fixed + std::max(static_cast<size_t>(st) * kStageBytes, part_bytes);
  };
  int chosen = 0;
  if (forced_split <= 0) forced_split = env_int("DSINF_KSPLIT", 0);
  if (forced_split > 0) {
    if (forced_split != 1 && forced_split != 2 && forced_split != 4 && forced_split != 8 && forced_split != 16)
      throw ConfigError("ksplit must be one of {1, 2, 4, 8, 16}");
    if (!valid(forced_split)) throw ConfigError("ksplit not valid for this shape");
    chosen = forced_split;
  } else {
    // largest one-wave grid; if none fits in one wave, the smallest valid split
    int best_units = -1;
    for (int s = 1; s <= 16; s <<= 1) {
      if (!valid(s)) continue;
      const int units = pl.col_tiles * s;
      const int clusters = resident_clusters(int8_weights, pl.nb8, s, smem_for(s, nullptr));
      const int capacity = clusters > 0 ? clusters * s : 2 * 148;
      if (units <= capacity && units > best_units) {
        best_units = units;
        chosen = s;
      }
    }
    if (chosen == 0)
      for (int s = 1; s <= 16 && chosen == 0; s <<= 1)
        if (valid(s)) chosen = s;
    if (chosen == 0) throw ConfigError("sbi_gemm: K too large for the x slice budget");
  }
  pl.ksplit = chosen;
  pl.rows_per_split = rps_for(chosen);
  pl.smem_bytes = smem_for(chosen, &pl.stages);
  return pl;
}

void launch(const Params& p_in, const Plan& plan, bool int8_weights, cudaStream_t stream, bool pdl) {
  Params p = p_in;
  p.rows_per_split = plan.rows_per_split;
  p.stages = plan.stages;
  p.x_row_words = plan.rows_per_split + 8;
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
