// Non-GEMM device operators: synthetic weight init / packing / quantisation, decode
// attention over the KV cache, embedding, greedy argmax and the single-device shard reduce.
#include <cstdlib>
#include <cfloat>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ops.cuh"
#include "sbi_gemm.cuh"
#include "sbi_gemm_dev.cuh"
#include "ptx.cuh"
#include "synth.h"

namespace dsinf {
namespace ops {

namespace {

inline int blocks_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

__device__ __forceinline__ int64_t global_row(const ShardMap& m, int64_t n) {
  return (n / m.sec_local) * m.sec_global + m.row_off + (n % m.sec_local);
}

__device__ __forceinline__ float synth_value(const ShardMap& m, int64_t grow, int64_t gcol) {
  if (grow >= m.valid_rows || gcol >= m.K_global) return 0.0f;
  const float w = __fmul_rn(synth_unit(m.base, static_cast<uint64_t>(grow * m.K_global + gcol)), m.amp);
  return __half2float(__float2half_rn(w));
}

__global__ void init_packed_f16_kernel(ShardMap m, uint32_t* packed) {
  const int64_t rows = (m.K_local + 1) / 2;
  const int64_t total = rows * m.N_local;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / m.N_local, n = i - r * m.N_local;
    const int64_t grow = global_row(m, n);
    const int64_t k = 2 * r;
    const float v0 = synth_value(m, grow, m.col_off + k);
    const float v1 = (k + 1 < m.K_local) ? synth_value(m, grow, m.col_off + k + 1) : 0.0f;
    const __half2 h = __floats2half2_rn(v0, v1);
    packed[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
}

// int8 row scale over the FULL global row (TP-invariant quantisation).
__global__ void init_row_scale_kernel(ShardMap m, float* scales) {
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t n = blockIdx.x * warps + (threadIdx.x >> 5); n < m.N_local; n += static_cast<int64_t>(gridDim.x) * warps) {
    const int64_t grow = global_row(m, n);
    float mx = 0.f;
    for (int64_t k = lane; k < m.K_global; k += 32) mx = fmaxf(mx, fabsf(synth_value(m, grow, k)));
    mx = ptx::warp_max(mx);
    if (lane == 0) scales[n] = mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f;
  }
}

__device__ __forceinline__ uint32_t q8(float x, float scale) {
  int q = __float2int_rn(__fdiv_rn(x, scale));
  q = max(-127, min(127, q));
  return static_cast<uint32_t>(q) & 0xffu;
}

__global__ void init_packed_i8_kernel(ShardMap m, const float* scales, uint32_t* packed, uint32_t bias) {
  const int64_t rows = (m.K_local + 3) / 4;
  const int64_t total = rows * m.N_local;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / m.N_local, n = i - r * m.N_local;
    const int64_t grow = global_row(m, n);
    const float s = scales[n];
    uint32_t word = 0;
    for (int e = 0; e < 4; ++e) {
      const int64_t k = 4 * r + e;
      if (k < m.K_local) word |= q8(synth_value(m, grow, m.col_off + k), s) << (8 * e);
    }
    packed[i] = word ^ bias;
  }
}

// The same synthetic tensor quantised per (global output row, 128-k group) (K_local and col_off
// multiples of 128, so a group never straddles TP shards): fp16 scale s = fp16(max|w| / 127), q =
// clamp(rint(w / s)); one warp per (row, group), lane l owns packed word l of the group.
__global__ void init_packed_i8_groups_kernel(ShardMap m, uint32_t* packed, __half* gscales, uint32_t bias) {
  const int64_t G = m.K_local / kI8Group;
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(warps) + (threadIdx.x >> 5); u < m.N_local * G;
       u += static_cast<int64_t>(gridDim.x) * warps) {
    const int64_t n = u / G, g = u - n * G;
    const int64_t grow = global_row(m, n);
    const int64_t k0 = g * kI8Group + 4 * lane;
    float v[4];
    float mx = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = synth_value(m, grow, m.col_off + k0 + e);
      mx = fmaxf(mx, fabsf(v[e]));
    }
    mx = ptx::warp_max(mx);
    __half sh = __float2half_rn(mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f);
    if (__half2float(sh) == 0.f) sh = __float2half_rn(1.0f);
    const float sc = __half2float(sh);
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) word |= q8(v[e], sc) << (8 * e);
    packed[(k0 / 4) * m.N_local + n] = word ^ bias;
    if (lane == 0) gscales[g * m.N_local + n] = sh;
  }
}

// Row-major [N_local][K_local] copies of the same synthetic tensor for the tensor-core
// (large-batch) path: fp16 values, or int8 quantised with the packed layout's row scales (so both
// layouts hold identical int8 weights).
__global__ void init_rowmajor_map_f16_kernel(ShardMap m, __half* out) {
  const int64_t total = m.N_local * m.K_local;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / m.K_local, k = i - n * m.K_local;
    out[i] = __float2half_rn(synth_value(m, global_row(m, n), m.col_off + k));
  }
}

__global__ void init_rowmajor_map_i8_kernel(ShardMap m, const float* scales, int8_t* out) {
  const int64_t total = m.N_local * m.K_local;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / m.K_local, k = i - n * m.K_local;
    out[i] = static_cast<int8_t>(q8(synth_value(m, global_row(m, n), m.col_off + k), scales[n]));
  }
}

__global__ void init_vector_kernel(ShardMap m, float offset, __half* out) {
  for (int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; n < m.N_local;
       n += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t grow = global_row(m, n);
    float v = 0.f;
    if (grow < m.valid_rows) v = __fadd_rn(offset, __fmul_rn(synth_unit(m.base, static_cast<uint64_t>(grow)), m.amp));
    out[n] = __float2half_rn(v);
  }
}

__global__ void init_rowmajor_kernel(uint64_t base, float amp, int64_t total, __half* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2half_rn(__fmul_rn(synth_unit(base, static_cast<uint64_t>(i)), amp));
}

__global__ void pack_f16_kernel(const void* w, bool src_f32, int64_t N, int64_t K, int M, __half* out) {
  const int64_t rows = (K + M - 1) / M;
  const int64_t total = rows * N * M;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (N * M);
    const int64_t rem = i - r * N * M;
    const int64_t n = rem / M;
    const int64_t k = r * M + (rem - n * M);
    __half v = __float2half(0.f);
    if (k < K) {
      if (src_f32)
        v = __float2half_rn(static_cast<const float*>(w)[n * K + k]);
      else
        v = static_cast<const __half*>(w)[n * K + k];
    }
    out[i] = v;
  }
}

__global__ void row_maxabs_scale_kernel(const __half* w, int64_t N, int64_t K, float* scales) {
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += static_cast<int64_t>(gridDim.x) * warps) {
    float mx = 0.f;
    for (int64_t k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(__half2float(w[n * K + k])));
    mx = ptx::warp_max(mx);
    if (lane == 0) scales[n] = mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f;
  }
}

__global__ void quant_pack_i8_kernel(const __half* w, int64_t N, int64_t K, const float* scales, uint32_t* packed) {
  const int64_t rows = (K + 3) / 4;
  const int64_t total = rows * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, n = i - r * N;
    uint32_t word = 0;
    for (int e = 0; e < 4; ++e) {
      const int64_t k = 4 * r + e;
      if (k < K) word |= q8(__half2float(w[n * K + k]), scales[n]) << (8 * e);
    }
    packed[i] = word;
  }
}

// K-group weight quantisation (group = 128 consecutive k of one output row, kI8Group): one warp per
// (row, group), lane l owns packed word l of the group (4 consecutive k).  Scale s = fp16(max|w| /
// 127) (fp32 divide, fp16 round to nearest; 1 for an all-zero group), q = clamp(rint(w / s), +-127)
// with an fp32 divide by the fp16 scale the kernels dequantise with.  Scales [ceil(K/128)][N].
__global__ void quant_groups_i8_kernel(const __half* w, int64_t N, int64_t K, uint32_t* packed, __half* gscales) {
  const int64_t G = (K + kI8Group - 1) / kI8Group;
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(warps) + (threadIdx.x >> 5); u < N * G;
       u += static_cast<int64_t>(gridDim.x) * warps) {
    const int64_t n = u / G, g = u - n * G;
    const int64_t k0 = g * kI8Group + 4 * lane;
    float v[4];
    float mx = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = k0 + e < K ? __half2float(w[n * K + k0 + e]) : 0.f;
      mx = fmaxf(mx, fabsf(v[e]));
    }
    mx = ptx::warp_max(mx);
    __half sh = __float2half_rn(mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f);
    if (__half2float(sh) == 0.f) sh = __float2half_rn(1.0f);  // fp16 underflow of a tiny group
    const float sc = __half2float(sh);
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (k0 + e < K) word |= q8(v[e], sc) << (8 * e);
    if (k0 < K) packed[(k0 / 4) * N + n] = word;
    if (lane == 0) gscales[g * N + n] = sh;
  }
}

__global__ void quant_act_kernel(const __half* x, int64_t K, int8_t* q, float* scales) {
  const int64_t b = blockIdx.x;
  __shared__ float red[32];
  float mx = 0.f;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) mx = fmaxf(mx, fabsf(__half2float(x[b * K + k])));
  mx = ptx::warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    v = ptx::warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float s = red[0] > 0.f ? __fdiv_rn(red[0], 127.0f) : 1.0f;
  if (threadIdx.x == 0) scales[b] = s;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
    q[b * K + k] = static_cast<int8_t>(static_cast<int>(q8(__half2float(x[b * K + k]), s) << 24) >> 24);
}

// ---------------------------------------------------------------- step boundary
__global__ void embed_kernel(const __grid_constant__ EmbedParams p) {
  ptx::trace_begin(p.trace);
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int b = blockIdx.x;
  const int pos = *p.pos;
  int tok = pos < p.prompt_len ? p.prompt[static_cast<size_t>(b) * p.prompt_ld + pos] : p.next_tok[b];
  if (tok < 0 || tok >= p.V) tok = 0;
  if (threadIdx.x == 0 && pos < p.max_ctx) p.hist[static_cast<size_t>(b) * p.max_ctx + pos] = tok;
  const uint4* row = reinterpret_cast<const uint4*>(p.wte + static_cast<size_t>(tok) * p.h);  // h % 8 == 0
  float4* out = reinterpret_cast<float4*>(p.res + static_cast<size_t>(b) * p.h);
  long long s1 = 0, s2 = 0;
  for (int k = threadIdx.x; k < p.h / 8; k += blockDim.x) {
    const uint4 u = __ldg(row + k);
    const __half2* hh = reinterpret_cast<const __half2*>(&u);
    float v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __low2float(hh[i]);
      v[2 * i + 1] = __high2float(hh[i]);
    }
    out[2 * k] = make_float4(v[0], v[1], v[2], v[3]);
    out[2 * k + 1] = make_float4(v[4], v[5], v[6], v[7]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s1 += __float2ll_rn(__fmul_rn(v[i], gemm::kSumScale));
      s2 += __float2ll_rn(__fmul_rn(__fmul_rn(v[i], v[i]), gemm::kSqScale));
    }
  }
  if (p.ln_stats_out != nullptr) {  // LayerNorm statistics of the first layer (integer sums: exact)
    __shared__ long long red[2][32];
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = s1;
      red[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      long long t = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
      atomicAdd(reinterpret_cast<unsigned long long*>(p.ln_stats_out) + b * 2 + threadIdx.x, static_cast<unsigned long long>(t));
    }
  }
  ptx::trace_end(p.trace);
}

__global__ void argmax_kernel(const __grid_constant__ ArgmaxParams p) {
  ptx::trace_begin(p.trace);
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int b = blockIdx.x;
  const float* row = p.logits + static_cast<size_t>(b) * p.ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < p.valid; i += blockDim.x) {
    const float v = row[i];
    if (v > best) {  // strided ascending scan: first max per thread is the lowest index
      best = v;
      bi = i;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bv = sv[0];
    int bx = si[0];
    for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bx)) {
        bv = sv[w];
        bx = si[w];
      }
    p.out_val[b] = bv;
    p.out_idx[b] = static_cast<int32_t>(bx + p.idx_offset);
  }
  ptx::trace_end(p.trace);
}

__global__ void select_kernel(const __grid_constant__ SelectParams p) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int pos = *p.pos;
  if (p.ipc_t > 1) {  // all-gather of the vocab shards' argmax keys over peer memory
    for (int b = threadIdx.x; b < p.B; b += blockDim.x) {
      const unsigned long long k = p.keys[p.ipc_rank * p.B + b];
      for (int q = 0; q < p.ipc_t; ++q)
        if (q != p.ipc_rank) p.ipc_keys[q][p.ipc_rank * p.B + b] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < p.ipc_t; ++q)
        if (q != p.ipc_rank) atomicAdd_system(p.ipc_flag[q], 1ull);
      const unsigned long long target =
          (static_cast<unsigned long long>(*p.step_ctr) + 1ull) * static_cast<unsigned long long>(p.ipc_t - 1);
      while (ptx::ld_acquire_sys(p.ipc_flag[p.ipc_rank]) < target) __nanosleep(32);
    }
    __syncthreads();
  }
  for (int b = threadIdx.x; b < p.B; b += blockDim.x) {
    float bv = 0.f;
    int32_t bx = 0;
    if (p.keys != nullptr) {  // fused LM-head argmax: the max key is the max logit, lowest index
      const volatile unsigned long long* keys = p.keys;  // peers' slots land over NVLink (IPC mode)
      unsigned long long k = keys[b];
      for (int s = 1; s < p.shards; ++s) k = max(k, keys[s * p.B + b]);
      bx = gemm::argmax_key_index(k);
    } else {
      bv = p.vals[b];
      bx = p.idxs[b];
      for (int s = 1; s < p.shards; ++s) {  // ties -> lowest vocabulary index
        const float v = p.vals[s * p.B + b];
        const int32_t x = p.idxs[s * p.B + b];
        if (v > bv || (v == bv && x < bx)) {
          bv = v;
          bx = x;
        }
      }
    }
    p.next_tok[b] = bx;
    if (pos + 1 < p.max_ctx) p.hist[static_cast<size_t>(b) * p.max_ctx + pos + 1] = bx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *p.pos = pos + 1;
    if (p.step_ctr) *p.step_ctr += 1;
  }
}

// ---------------------------------------------------------------- row preparation (x streaming)
constexpr int kPrepThreads = 512;
constexpr int kPrepVec = 8;  // float4 per thread held in registers: K <= 16384

__device__ __forceinline__ uint32_t prep_q(float y, float s) {
  int q = __float2int_rn(__fdiv_rn(y, s));
  q = max(-127, min(127, q));
  return static_cast<uint32_t>(q) & 0xffu;
}

// Cluster-wide (S CTAs of one row) integer sums and float max, in rank order; `slot` is this
// CTA's smem exchange word(s).  S == 1: the CTA's own values.
__device__ __forceinline__ void prep_cluster_sum2(long long& a, long long& b, long long* slot, int S) {
  if (S == 1) return;
  if (threadIdx.x == 0) {
    slot[0] = a;
    slot[1] = b;
  }
  ptx::cluster_sync();
  a = b = 0;
  for (int q = 0; q < S; ++q) {
    const uint32_t ad = ptx::map_shared_rank(slot, q);
    const uint2 u0 = ptx::ld_dsmem_u2(ad), u1 = ptx::ld_dsmem_u2(ad + 8);
    a += static_cast<long long>((static_cast<unsigned long long>(u0.y) << 32) | u0.x);
    b += static_cast<long long>((static_cast<unsigned long long>(u1.y) << 32) | u1.x);
  }
}
__device__ __forceinline__ float prep_cluster_max(float m, float* slot, int S) {
  if (S == 1) return m;
  if (threadIdx.x == 0) *slot = m;
  ptx::cluster_sync();
  for (int q = 0; q < S; ++q) m = fmaxf(m, ptx::ld_dsmem_f_nc(ptx::map_shared_rank(slot, q)));
  return m;
}

// One row per cluster of S = gridDim.x CTAs (S = 1 for short rows): CTA r owns the float4 columns
// r*kPrepThreads + tid + u*kPrepThreads*S; row sums and maxima are exchanged through DSMEM.
__global__ void __launch_bounds__(kPrepThreads) row_prep_kernel(const __grid_constant__ PrepParams p) {
  ptx::trace_begin(p.trace);
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int b = blockIdx.y;
  const int S = gridDim.x;
  const int c0 = blockIdx.x * kPrepThreads + threadIdx.x, cs = kPrepThreads * S;
  const int K4 = p.K / 4;
  __shared__ float red[kPrepThreads / 32];
  __shared__ long long xsum[2];
  __shared__ float xmax[2];
  auto block_max = [&](float mx) {
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < kPrepThreads / 32; ++w) mx = fmaxf(mx, red[w]);
    return mx;
  };
  if (p.mode == PREP_QUANT_I8) {
    float mx = 0.f;
    if (p.amax != nullptr) {
      for (int s = 0; s < gemm::kStatStripes; ++s) mx = fmaxf(mx, __uint_as_float(__ldcg(p.amax + s * 32 + b)));
    } else {  // row max computed here (large-batch path: rows beyond the producer's stripes)
      const uint2* row2 = reinterpret_cast<const uint2*>(p.x + static_cast<size_t>(b) * p.x_ld);
      for (int c = c0; c < K4; c += cs) {
        const uint2 u = __ldcg(row2 + c);
        const __half2 h01 = *reinterpret_cast<const __half2*>(&u.x), h23 = *reinterpret_cast<const __half2*>(&u.y);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(__low2float(h01)), fabsf(__high2float(h01))),
                             fmaxf(fabsf(__low2float(h23)), fabsf(__high2float(h23)))));
      }
      mx = prep_cluster_max(block_max(mx), &xmax[0], S);
    }
    const float scale = mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f;
    if (threadIdx.x == 0 && blockIdx.x == 0) p.out_scale[b] = scale;
    const __half* row = p.x + static_cast<size_t>(b) * p.x_ld;
    uint32_t* out = reinterpret_cast<uint32_t*>(static_cast<int8_t*>(p.out) + static_cast<size_t>(b) * p.K);
#pragma unroll 4
    for (int c = c0; c < K4; c += cs) {
      const uint2 u = __ldcg(reinterpret_cast<const uint2*>(row) + c);
      const __half2 h01 = *reinterpret_cast<const __half2*>(&u.x), h23 = *reinterpret_cast<const __half2*>(&u.y);
      out[c] = prep_q(__low2float(h01), scale) | (prep_q(__high2float(h01), scale) << 8) |
               (prep_q(__low2float(h23), scale) << 16) | (prep_q(__high2float(h23), scale) << 24);
    }
    if (S > 1 && p.amax == nullptr) ptx::cluster_sync_relaxed();  // peers' DSMEM reads of xmax are done
    ptx::trace_end(p.trace);
    return;
  }
  // LayerNorm of the residual row (same expression as the fused GEMM prologue, so both plans
  // produce identical x); statistics from the producer or summed here in the same fixed point
  const size_t rb = static_cast<size_t>(b) * p.K;
  if (p.red_flag != nullptr) {  // fused all-reduce: every rank's partial has landed
    if (threadIdx.x == 0) ptx::wait_flag(p.red_flag, p.step_ctr, p.red_per_step);
    __syncthreads();
  }
  float4 v[kPrepVec];
  long long s1 = 0, s2 = 0;
#pragma unroll
  for (int u = 0; u < kPrepVec; ++u) {
    const int c = c0 + u * cs;
    v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < K4) {
      v[u] = __ldcg(reinterpret_cast<const float4*>(p.res + rb) + c);
      if (p.res_delta) {
        float4 t = __ldcg(reinterpret_cast<const float4*>(p.res_delta + rb) + c);
        for (int q = 1; q < p.delta_slots; ++q) {
          const float4 u = __ldcg(reinterpret_cast<const float4*>(p.res_delta + q * p.delta_stride + rb) + c);
          t.x = __fadd_rn(t.x, u.x);
          t.y = __fadd_rn(t.y, u.y);
          t.z = __fadd_rn(t.z, u.z);
          t.w = __fadd_rn(t.w, u.w);
        }
        if (p.delta_bias) {
          const __half2 d01 = *reinterpret_cast<const __half2*>(p.delta_bias + 4 * c);
          const __half2 d23 = *reinterpret_cast<const __half2*>(p.delta_bias + 4 * c + 2);
          t.x = __fadd_rn(t.x, __low2float(d01));
          t.y = __fadd_rn(t.y, __high2float(d01));
          t.z = __fadd_rn(t.z, __low2float(d23));
          t.w = __fadd_rn(t.w, __high2float(d23));
        }
        v[u].x = __fadd_rn(v[u].x, t.x);
        v[u].y = __fadd_rn(v[u].y, t.y);
        v[u].z = __fadd_rn(v[u].z, t.z);
        v[u].w = __fadd_rn(v[u].w, t.w);
      }
      if (p.res_out) reinterpret_cast<float4*>(p.res_out + rb)[c] = v[u];
      if (!p.ln_stats) {
        const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          s1 += __float2ll_rn(__fmul_rn(e[i], gemm::kSumScale));
          s2 += __float2ll_rn(__fmul_rn(__fmul_rn(e[i], e[i]), gemm::kSqScale));
        }
      }
    }
  }
  __shared__ long long lred[2][kPrepThreads / 32];
  if (p.ln_stats) {
    for (int s = 0; s < gemm::kStatStripes; ++s) {
      s1 += __ldcg(p.ln_stats + (s * gemm::kMaxB + b) * 2);
      s2 += __ldcg(p.ln_stats + (s * gemm::kMaxB + b) * 2 + 1);
    }
  } else {  // integer block (then cluster) sum: exact, order-independent
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
      lred[0][threadIdx.x >> 5] = s1;
      lred[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    s1 = s2 = 0;
    for (int w = 0; w < kPrepThreads / 32; ++w) {
      s1 += lred[0][w];
      s2 += lred[1][w];
    }
    prep_cluster_sum2(s1, s2, xsum, S);
  }
  float mean, rstd;
  gemm::dev::ln_mean_rstd(s1, s2, p.inv_k, p.eps, mean, rstd);
  uint2 hv[kPrepVec];
  float mx = 0.f;
#pragma unroll
  for (int u = 0; u < kPrepVec; ++u) {
    const int c = c0 + u * cs;
    if (c < K4) {
      const uint2 g = *reinterpret_cast<const uint2*>(p.ln_g + 4 * c);
      const uint2 be = *reinterpret_cast<const uint2*>(p.ln_b + 4 * c);
      const __half2 g01 = *reinterpret_cast<const __half2*>(&g.x), g23 = *reinterpret_cast<const __half2*>(&g.y);
      const __half2 b01 = *reinterpret_cast<const __half2*>(&be.x), b23 = *reinterpret_cast<const __half2*>(&be.y);
      const __half2 h01 = __floats2half2_rn((v[u].x - mean) * rstd * __low2float(g01) + __low2float(b01),
                                            (v[u].y - mean) * rstd * __high2float(g01) + __high2float(b01));
      const __half2 h23 = __floats2half2_rn((v[u].z - mean) * rstd * __low2float(g23) + __low2float(b23),
                                            (v[u].w - mean) * rstd * __high2float(g23) + __high2float(b23));
      hv[u].x = *reinterpret_cast<const uint32_t*>(&h01);
      hv[u].y = *reinterpret_cast<const uint32_t*>(&h23);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(__low2float(h01)), fabsf(__high2float(h01))),
                           fmaxf(fabsf(__low2float(h23)), fabsf(__high2float(h23)))));
    }
  }
  if (p.mode == PREP_LN_F16) {
    uint2* out = reinterpret_cast<uint2*>(static_cast<__half*>(p.out) + static_cast<size_t>(b) * p.K);
#pragma unroll
    for (int u = 0; u < kPrepVec; ++u) {
      const int c = c0 + u * cs;
      if (c < K4) out[c] = hv[u];
    }
    if (S > 1 && !p.ln_stats) ptx::cluster_sync_relaxed();  // peers' DSMEM reads of xsum are done
    ptx::trace_end(p.trace);
    return;
  }
  mx = prep_cluster_max(block_max(mx), &xmax[1], S);
  const float scale = mx > 0.f ? __fdiv_rn(mx, 127.0f) : 1.0f;
  if (threadIdx.x == 0 && blockIdx.x == 0) p.out_scale[b] = scale;
  uint32_t* out = reinterpret_cast<uint32_t*>(static_cast<int8_t*>(p.out) + static_cast<size_t>(b) * p.K);
#pragma unroll
  for (int u = 0; u < kPrepVec; ++u) {
    const int c = c0 + u * cs;
    if (c < K4) {
      const __half2 h01 = *reinterpret_cast<const __half2*>(&hv[u].x), h23 = *reinterpret_cast<const __half2*>(&hv[u].y);
      out[c] = prep_q(__low2float(h01), scale) | (prep_q(__high2float(h01), scale) << 8) |
               (prep_q(__low2float(h23), scale) << 16) | (prep_q(__high2float(h23), scale) << 24);
    }
  }
  if (S > 1) ptx::cluster_sync_relaxed();  // peers' DSMEM reads of xmax are done
  ptx::trace_end(p.trace);
}

__global__ void local_allreduce_kernel(const __grid_constant__ LocalReduceParams p) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < p.count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = p.buf[0][i];
    for (int s = 1; s < p.shards; ++s) acc += p.buf[s][i];
    for (int s = 0; s < p.shards; ++s) p.buf[s][i] = acc;
  }
}

}  // namespace

bool carveout_max() {
  const char* v = std::getenv("DSINF_CARVEOUT");
  return v == nullptr || std::atoi(v) != 0;
}

// The small step kernels ask for the maximum shared-memory carveout like the GEMMs: an SM whose
// L1/shared split was set for a low-smem kernel cannot take a GEMM CTA (PDL-launched next to it)
// until it drains and reconfigures.
void configure_step_kernels() {
  if (!carveout_max()) return;
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(row_prep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(embed_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(select_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(local_allreduce_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}

void row_prep(const PrepParams& p_in, cudaStream_t s, bool pdl) {
  PrepParams p = p_in;
  p.inv_k = 1.0 / static_cast<double>(p.K);
  if (p.K % 8 != 0) throw ConfigError("row_prep: K must be a multiple of 8");
  // the LayerNorm modes hold the row in registers; quantisation loops over any K
  if (p.mode != PREP_QUANT_I8 && p.K / 4 > kPrepThreads * kPrepVec)
    throw ConfigError("row_prep: LayerNorm rows must be <= 16384 wide");
  if (p.mode == PREP_QUANT_I8 && (p.x_ld % 4 != 0 || (reinterpret_cast<uintptr_t>(p.x) & 7) != 0))
    throw ConfigError("row_prep: x rows must be 8-byte aligned");
  // CTAs per row (a cluster): one SM's L2 request rate bounds a single-CTA pass over a long row.
  // Measured (GPT-J, GPT3-175B t=8 rank): best S = 8 at B=1 (h=12288: 9.70 -> 8.89 ms fp16),
  // 4 at B=4 (2.91 -> 2.78 ms), 2 at B=16 (3.15 -> 3.09 ms fp16, 2.67 -> 2.58 int8); at least
  // 128 float4 per CTA.  DSINF_PREP_SPLIT overrides.
  const char* fv = std::getenv("DSINF_PREP_SPLIT");  // read at enqueue / graph capture time only
  const int forced = fv ? std::atoi(fv) : 0;
  int S = 1;
  if (forced > 0) {
    S = forced;
  } else if (p.split > 0) {
    S = p.split;
  } else {
    S = 8;
    while (S > 2 && p.B * S > 16) S >>= 1;
    // long LayerNorm rows (two float4 streams per column): <= 1024 float4 per CTA (175B B=16: 10.44 -> 10.13)
    while (p.mode != PREP_QUANT_I8 && S < 8 && p.K / 4 / S > 1024) S <<= 1;
    while (S > 1 && p.K / 4 / S < 128) S >>= 1;
  }
  if (S != 1 && S != 2 && S != 4 && S != 8) throw ConfigError("row_prep: split must be 1, 2, 4 or 8");
  launch_pdl(row_prep_kernel, dim3(S, p.B), dim3(kPrepThreads), 0, s, pdl, p, dim3(S, 1, 1));
}

void init_packed_f16(const ShardMap& m, uint32_t* packed, cudaStream_t s) {
  const int64_t total = (m.K_local + 1) / 2 * m.N_local;
  init_packed_f16_kernel<<<blocks_for(total, 256), 256, 0, s>>>(m, packed);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_packed_i8(const ShardMap& m, uint32_t* packed, float* scales, cudaStream_t s, bool biased) {
  init_row_scale_kernel<<<blocks_for(m.N_local, 8, 148 * 8), 256, 0, s>>>(m, scales);
  DSINF_CUDA_CHECK(cudaGetLastError());
  const int64_t total = (m.K_local + 3) / 4 * m.N_local;
  init_packed_i8_kernel<<<blocks_for(total, 256), 256, 0, s>>>(m, scales, packed, biased ? 0x80808080u : 0u);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_packed_i8_groups(const ShardMap& m, uint32_t* packed, __half* gscales, cudaStream_t s, bool biased) {
  if (m.K_local % kI8Group != 0 || m.col_off % kI8Group != 0)
    throw ConfigError("K-group INT8 weights need per-rank in_dim (and shard offsets) multiples of 128");
  const int64_t units = m.N_local * (m.K_local / kI8Group);
  init_packed_i8_groups_kernel<<<blocks_for(units, 8, 148 * 16), 256, 0, s>>>(m, packed, gscales,
                                                                            biased ? 0x80808080u : 0u);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_rowmajor_map_f16(const ShardMap& m, __half* out, cudaStream_t s) {
  init_rowmajor_map_f16_kernel<<<blocks_for(m.N_local * m.K_local, 256), 256, 0, s>>>(m, out);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_rowmajor_map_i8(const ShardMap& m, const float* scales, int8_t* out, cudaStream_t s) {
  init_rowmajor_map_i8_kernel<<<blocks_for(m.N_local * m.K_local, 256), 256, 0, s>>>(m, scales, out);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_vector_f16(const ShardMap& m, float offset, __half* out, cudaStream_t s) {
  init_vector_kernel<<<blocks_for(m.N_local, 256), 256, 0, s>>>(m, offset, out);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void init_rowmajor_f16(uint64_t base, float amp, int64_t rows, int64_t cols, __half* out, cudaStream_t s) {
  init_rowmajor_kernel<<<blocks_for(rows * cols, 256), 256, 0, s>>>(base, amp, rows * cols, out);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void pack_f16(const void* w, bool src_f32, int64_t N, int64_t K, int pack_M, __half* out, cudaStream_t s) {
  const int64_t total = (K + pack_M - 1) / pack_M * N * pack_M;
  pack_f16_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, src_f32, N, K, pack_M, out);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void quantize_weights_i8(const __half* w, int64_t N, int64_t K, int8_t* packed, float* scales, cudaStream_t s) {
  row_maxabs_scale_kernel<<<blocks_for(N, 8, 148 * 8), 256, 0, s>>>(w, N, K, scales);
  DSINF_CUDA_CHECK(cudaGetLastError());
  const int64_t total = (K + 3) / 4 * N;
  quant_pack_i8_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, N, K, scales, reinterpret_cast<uint32_t*>(packed));
  DSINF_CUDA_CHECK(cudaGetLastError());
}

__global__ void word_transpose_kernel(const uint32_t* __restrict__ in, int64_t rows, int64_t N,
                                      uint32_t* __restrict__ out, uint32_t xor_mask) {
  __shared__ uint32_t tile[32][33];
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && n < N) ? __ldcs(in + r * N + n) : 0u;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t n = n0 + i, r = r0 + threadIdx.x;
    if (n < N && r < rows) out[n * rows + r] = tile[threadIdx.x][i] ^ xor_mask;
  }
}

void packed_to_rowmajor(const uint32_t* packed, int64_t rows, int64_t N, uint32_t* out, cudaStream_t s,
                        uint32_t xor_mask) {
  if (rows >= (1LL << 31) / 32 * 32 || N >= (1LL << 31) / 32 * 32) throw ConfigError("packed_to_rowmajor: too large");
  const dim3 grid(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  word_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(packed, rows, N, out, xor_mask);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void quantize_weights_i8_groups(const __half* w, int64_t N, int64_t K, int8_t* packed, __half* gscales,
                                cudaStream_t s) {
  const int64_t units = N * ((K + kI8Group - 1) / kI8Group);
  quant_groups_i8_kernel<<<blocks_for(units, 8, 148 * 16), 256, 0, s>>>(w, N, K, reinterpret_cast<uint32_t*>(packed),
                                                                        gscales);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void quantize_act_i8(const __half* x, int64_t B, int64_t K, int8_t* q, float* scales, cudaStream_t s) {
  quant_act_kernel<<<static_cast<unsigned>(B), 256, 0, s>>>(x, K, q, scales);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void embed(const EmbedParams& p, cudaStream_t s, bool pdl) {
  launch_pdl(embed_kernel, dim3(p.B), dim3(256), 0, s, pdl, p);
}

void argmax(const ArgmaxParams& p, cudaStream_t s, bool pdl) {
  launch_pdl(argmax_kernel, dim3(p.B), dim3(1024), 0, s, pdl, p);
}

void select_token(const SelectParams& p, cudaStream_t s, bool pdl) {
  if (p.ipc_t > 8) throw ConfigError("select_token: at most 8 IPC ranks");
  if (p.ipc_t > 1 && (p.step_ctr == nullptr || p.keys == nullptr)) throw ConfigError("select_token: IPC needs keys and step_ctr");
  launch_pdl(select_kernel, dim3(1), dim3(32), 0, s, pdl, p);
}

void local_allreduce(const LocalReduceParams& p, cudaStream_t s, bool pdl) {
  launch_pdl(local_allreduce_kernel, dim3(blocks_for(p.count, 256, 148)), dim3(256), 0, s, pdl, p);
}

}  // namespace ops
}  // namespace dsinf
