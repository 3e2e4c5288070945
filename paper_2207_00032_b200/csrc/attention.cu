// Decode attention over the KV cache (paper Deep-Fusion region 2, "transposition plus
// attention"; canonical graph nodes attn_transpose + attention, fusion.hpp:271-277).
//
// One thread-block cluster per (batch row, head); its `C` CTAs split the context into chunks
// and merge their (max, sum, output) partials through distributed shared memory.  Inside a CTA
// TPP threads own one position (8 head dims each, one 16-byte load of K and of V), so every
// position of a round is in flight at once; each thread keeps an online-softmax accumulator
// over its positions, then slots are merged in smem and chunks across the cluster.
#include <cfloat>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ops.cuh"
#include "ptx.cuh"

namespace dsinf {
namespace ops {

namespace {

constexpr int kAttnThreads = 128;
constexpr int kUnroll = 4;

__device__ __forceinline__ void h8_to_f(const uint4& u, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __half22float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

template <int TPP>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const __grid_constant__ AttnParams p) {
  constexpr int PPR = kAttnThreads / TPP;  // positions per round
  extern __shared__ __align__(16) float asmem[];
  const int d = p.d;
  float* so = asmem;                  // [PPR][d] per-slot outputs
  float* sm = so + PPR * d;           // [PPR] per-slot max
  float* sl = sm + PPR;               // [PPR] per-slot sum
  float* co = sl + PPR;               // [d] this CTA's merged output
  float* cst = co + d;                // [2] this CTA's (max, sum)
  const int head = blockIdx.x, b = blockIdx.y, c = blockIdx.z, C = gridDim.z;
  const int tid = threadIdx.x;
  const int slot = tid / TPP, lane_in = tid % TPP;
  const int dim0 = lane_in * 8;
  const bool has_dims = dim0 < d;
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int ctx = *p.pos + 1;
  const int chunk = (ctx + C - 1) / C;
  const int j0 = c * chunk;
  const int j1 = min(ctx, j0 + chunk);
  const int len = max(0, j1 - j0);
  const int rounds = (len + PPR - 1) / PPR;
  const int hd = p.H * d;
  float q[8];
  if (has_dims) {
    const uint4 qu = *reinterpret_cast<const uint4*>(p.q + static_cast<size_t>(b) * hd + head * d + dim0);
    h8_to_f(qu, q);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] *= p.scale;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = 0.f;
  }
  const size_t kv_base = (static_cast<size_t>(b) * p.H + head) * p.max_seq * d + dim0;
  const __half* kb = p.kc + kv_base;
  const __half* vb = p.vc + kv_base;
  float m = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = 0.f;
  for (int r0 = 0; r0 < rounds; r0 += kUnroll) {  // warp-uniform trip count
    uint4 kr[kUnroll], vr[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int j = j0 + (r0 + u) * PPR + slot;
      if (j < j1 && has_dims) {
        kr[u] = *reinterpret_cast<const uint4*>(kb + static_cast<size_t>(j) * d);
        vr[u] = *reinterpret_cast<const uint4*>(vb + static_cast<size_t>(j) * d);
      } else {
        kr[u] = make_uint4(0, 0, 0, 0);
        vr[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      float kf[8];
      h8_to_f(kr[u], kf);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) s = fmaf(q[i], kf[i], s);
#pragma unroll
      for (int off = TPP / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const int j = j0 + (r0 + u) * PPR + slot;
      if (j < j1) {
        const float mn = fmaxf(m, s);
        const float corr = expf(m - mn);
        const float pj = expf(s - mn);
        float vf[8];
        h8_to_f(vr[u], vf);
        l = l * corr + pj;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = fmaf(pj, vf[i], o[i] * corr);
        m = mn;
      }
    }
  }
  // merge the PPR position slots of this CTA
  if (has_dims) {
#pragma unroll
    for (int i = 0; i < 8; ++i) so[slot * d + dim0 + i] = o[i];
  }
  if (lane_in == 0) {
    sm[slot] = m;
    sl[slot] = l;
  }
  __syncthreads();
  float M = -INFINITY;
  for (int sidx = 0; sidx < PPR; ++sidx) M = fmaxf(M, sm[sidx]);
  for (int i = tid; i < d; i += kAttnThreads) {
    float acc = 0.f;
    for (int sidx = 0; sidx < PPR; ++sidx) {
      const float w = sm[sidx] == -INFINITY ? 0.f : expf(sm[sidx] - M);
      acc = fmaf(w, so[sidx * d + i], acc);
    }
    co[i] = acc;
  }
  if (tid == 0) {
    float L = 0.f;
    for (int sidx = 0; sidx < PPR; ++sidx) L += sm[sidx] == -INFINITY ? 0.f : sl[sidx] * expf(sm[sidx] - M);
    cst[0] = M;
    cst[1] = L;
  }
  // merge the C chunks of this (b, head) across the cluster
  if (C > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  float MM = -INFINITY;
  for (int r = 0; r < C; ++r) MM = fmaxf(MM, ptx::ld_dsmem_f(ptx::map_shared_rank(&cst[0], r)));
  float wts[16];
  float LL = 0.f;
  for (int r = 0; r < C; ++r) {
    const float mr = ptx::ld_dsmem_f(ptx::map_shared_rank(&cst[0], r));
    const float lr = ptx::ld_dsmem_f(ptx::map_shared_rank(&cst[1], r));
    const float w = mr == -INFINITY ? 0.f : expf(mr - MM);
    wts[r] = w;
    LL += w * lr;
  }
  const float inv = 1.0f / LL;
  for (int i = c + C * tid; i < d; i += C * kAttnThreads) {
    float acc = 0.f;
    for (int r = 0; r < C; ++r) acc = fmaf(wts[r], ptx::ld_dsmem_f(ptx::map_shared_rank(&co[i], r)), acc);
    p.out[static_cast<size_t>(b) * hd + head * d + i] = __float2half_rn(acc * inv);
  }
  if (C > 1) ptx::cluster_sync();
}

template <int TPP>
size_t attn_smem(int d) {
  constexpr int PPR = kAttnThreads / TPP;
  return (static_cast<size_t>(PPR) * d + 2 * PPR + d + 4) * sizeof(float);
}

}  // namespace

int attention_chunks(int B, int H) {
  const int pairs = B * H;
  int c = 1;
  while (c < 8 && pairs * c < 2 * 148) c <<= 1;
  return c;
}

void configure() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

void attention(const AttnParams& p, int chunks, cudaStream_t s, bool pdl) {
  if (p.d % 8 != 0 || p.d > 256) throw ConfigError("attention: head dim must be a multiple of 8 and <= 256");
  if (chunks < 1 || chunks > 16) throw ConfigError("attention: bad chunk count");
  const dim3 grid(p.H, p.B, chunks), block(kAttnThreads), cluster(1, 1, chunks);
  if (p.d <= 64)
    launch_pdl(attention_kernel<8>, grid, block, attn_smem<8>(p.d), s, pdl, p, cluster);
  else if (p.d <= 128)
    launch_pdl(attention_kernel<16>, grid, block, attn_smem<16>(p.d), s, pdl, p, cluster);
  else
    launch_pdl(attention_kernel<32>, grid, block, attn_smem<32>(p.d), s, pdl, p, cluster);
}

}  // namespace ops
}  // namespace dsinf
