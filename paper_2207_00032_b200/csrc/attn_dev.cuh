// Device building block of decode attention (paper region 2; fusion.hpp:271-277):
// one chunk of context positions of one (batch row, head) reduced to an online-softmax partial
// (max, sum, unnormalised output).  Shared by the standalone attention kernel (chunks merged
// in-cluster through DSMEM) and the persistent step kernel (chunks merged through L2).
#pragma once

#include <cfloat>
#include <cstdint>
#include <cuda_fp16.h>

#include "ops.cuh"
#include "ptx.cuh"

namespace dsinf {
namespace ops {
namespace dev {

constexpr int kAttnThreads = 128;
constexpr int kAttnUnroll = 4;

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
__host__ __device__ constexpr size_t attn_scratch_floats(int d) {
  return static_cast<size_t>(kAttnThreads / TPP) * d + 2 * (kAttnThreads / TPP) + d + 4;
}

// Computes the partial of positions [j0, j1) into co[0..d) (output, unnormalised) and
// cst[0] = max, cst[1] = sum.  Called by kAttnThreads threads (tid in [0, 128)); `bar` is the
// barrier among them.  Loads use ld.global.cg: q / K / V may have been written by other CTAs.
// kv_pre (optional): K rows then V rows of positions [j0, j_pre) already in shared memory
// ([rows_cap][d] halves each; staged before the kernel's dependency wait), read instead of global.
template <int TPP, class Bar>
__device__ void attn_chunk(const AttnParams& p, int b, int head, int j0, int j1, int tid, float* scratch,
                           Bar bar, const __half* kv_pre = nullptr, int j_pre = 0, int rows_cap = 0) {
  constexpr int PPR = kAttnThreads / TPP;
  const int d = p.d;
  float* so = scratch;       // [PPR][d]
  float* sm = so + PPR * d;  // [PPR]
  float* sl = sm + PPR;      // [PPR]
  float* co = sl + PPR;      // [d]
  float* cst = co + d;       // [2]
  const int slot = tid / TPP, lane_in = tid % TPP;
  const int dim0 = lane_in * 8;
  const bool has_dims = dim0 < d;
  const int len = max(0, j1 - j0);
  const int rounds = (len + PPR - 1) / PPR;
  const int hd = p.H * d;
  float q[8];
  if (has_dims) {
    const uint4 qu = __ldcg(reinterpret_cast<const uint4*>(p.q + static_cast<size_t>(b) * hd + head * d + dim0));
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
  // software-pipelined: the K/V rows of batch r0 + kAttnUnroll are requested before batch r0 is
  // consumed, so two batches of loads are in flight (the loop is latency-bound, not bandwidth-bound)
  uint4 kr[kAttnUnroll], vr[kAttnUnroll];
  auto load_batch = [&](int r0, uint4 (&kk)[kAttnUnroll], uint4 (&vv)[kAttnUnroll]) {
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      const int j = j0 + (r0 + u) * PPR + slot;
      if (r0 < rounds && j < j1 && has_dims) {
        if (j < j_pre) {
          const __half* ks = kv_pre + static_cast<size_t>(j - j0) * d + dim0;
          kk[u] = *reinterpret_cast<const uint4*>(ks);
          vv[u] = *reinterpret_cast<const uint4*>(ks + static_cast<size_t>(rows_cap) * d);
        } else {
          kk[u] = __ldcg(reinterpret_cast<const uint4*>(kb + static_cast<size_t>(j) * d));
          vv[u] = __ldcg(reinterpret_cast<const uint4*>(vb + static_cast<size_t>(j) * d));
        }
      } else {
        kk[u] = make_uint4(0, 0, 0, 0);
        vv[u] = make_uint4(0, 0, 0, 0);
      }
    }
  };
  load_batch(0, kr, vr);
  for (int r0 = 0; r0 < rounds; r0 += kAttnUnroll) {  // warp-uniform trip count
    uint4 kn[kAttnUnroll], vn[kAttnUnroll];
    load_batch(r0 + kAttnUnroll, kn, vn);
    // scores of the batch's kAttnUnroll positions, then ONE online-softmax rescale per batch
    float sc[kAttnUnroll];
    float mt = -INFINITY;
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      float kf[8];
      h8_to_f(kr[u], kf);
      float sdot = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) sdot = fmaf(q[i], kf[i], sdot);
#pragma unroll
      for (int off = TPP / 2; off > 0; off >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, off);
      const int j = j0 + (r0 + u) * PPR + slot;
      sc[u] = j < j1 ? sdot : -INFINITY;
      mt = fmaxf(mt, sc[u]);
    }
    if (mt != -INFINITY) {
      const float mn = fmaxf(m, mt);
      const float corr = expf(m - mn);
      l *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] *= corr;
#pragma unroll
      for (int u = 0; u < kAttnUnroll; ++u) {
        if (sc[u] == -INFINITY) continue;
        const float pj = expf(sc[u] - mn);
        float vf[8];
        h8_to_f(vr[u], vf);
        l += pj;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = fmaf(pj, vf[i], o[i]);
      }
      m = mn;
    }
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      kr[u] = kn[u];
      vr[u] = vn[u];
    }
  }
  if (has_dims) {
#pragma unroll
    for (int i = 0; i < 8; ++i) so[slot * d + dim0 + i] = o[i];
  }
  if (lane_in == 0) {
    sm[slot] = m;
    sl[slot] = l;
  }
  bar();
  float M = -INFINITY;
  for (int s = 0; s < PPR; ++s) M = fmaxf(M, sm[s]);
  for (int i = tid; i < d; i += kAttnThreads) {
    float acc = 0.f;
    for (int s = 0; s < PPR; ++s) {
      const float w = sm[s] == -INFINITY ? 0.f : expf(sm[s] - M);
      acc = fmaf(w, so[s * d + i], acc);
    }
    co[i] = acc;
  }
  if (tid == 0) {
    float L = 0.f;
    for (int s = 0; s < PPR; ++s) L += sm[s] == -INFINITY ? 0.f : sl[s] * expf(sm[s] - M);
    cst[0] = M;
    cst[1] = L;
  }
  bar();
}

}  // namespace dev
}  // namespace ops
}  // namespace dsinf
