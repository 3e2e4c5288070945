// Prompt prefill in the large-batch regime (fusion.hpp:145-154): all B x P prompt
// tokens go through each layer at once, the GEMMs on the tcgen05 tensor cores (tc_gemm.cu), the
// non-GEMM work in the row kernels below.  Leaves the model in the state P decode steps over the
// prompt would (KV cache rows 0..P-1, history, next token, pos = P).
#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdlib>

#include "common.h"
#include "ops.cuh"
#include "ptx.cuh"
#include "sbi_gemm.cuh"
#include "sbi_gemm_dev.cuh"

namespace dsinf {
namespace ops {

namespace {

__global__ void prefill_embed_kernel(const __grid_constant__ PrefillEmbedParams p) {
  const int m = blockIdx.x;
  const int b = m / p.P, t = m - b * p.P;
  int tok = p.prompt[static_cast<size_t>(b) * p.prompt_ld + t];
  if (tok < 0 || tok >= p.V) tok = 0;  // same clamp as the decode embed
  if (threadIdx.x == 0 && t < p.max_ctx) p.hist[static_cast<size_t>(b) * p.max_ctx + t] = tok;
  const uint4* row = reinterpret_cast<const uint4*>(p.wte + static_cast<size_t>(tok) * p.h);  // h % 8 == 0
  float4* out = reinterpret_cast<float4*>(p.res + static_cast<size_t>(m) * p.h);
  for (int k = threadIdx.x; k < p.h / 8; k += blockDim.x) {
    const uint4 u = __ldg(row + k);
    const __half2* hh = reinterpret_cast<const __half2*>(&u);
    out[2 * k] = make_float4(__low2float(hh[0]), __high2float(hh[0]), __low2float(hh[1]), __high2float(hh[1]));
    out[2 * k + 1] = make_float4(__low2float(hh[2]), __high2float(hh[2]), __low2float(hh[3]), __high2float(hh[3]));
  }
}

// One CTA = kQ queries of one (sequence, head); K/V stream through shared memory in tiles of
// kT positions up to the block's causal limit.  Warp w owns queries w*4 .. w*4+3; within a tile
// lane j scores key j, the warp keeps an online softmax per query, and lane l accumulates the
// output dims l, l+32, ... (fp32; stored fp16 like the decode kernel).
constexpr int kQ = 32, kT = 32, kPThreads = 256, kQPerWarp = kQ / (kPThreads / 32);
constexpr int kMaxDimsPerLane = 8;  // d <= 256

__global__ void __launch_bounds__(kPThreads) prefill_attention_kernel(const __grid_constant__ PrefillAttnParams p) {
  extern __shared__ __align__(16) unsigned char psm[];
  const int d = p.d, ks = d + 2;  // K row stride (halves): conflict-free column reads across rows
  float* qs = reinterpret_cast<float*>(psm);                              // [kQ][d] scaled q
  __half* kt = reinterpret_cast<__half*>(qs + kQ * d);                    // [kT][d + 2]
  __half* vt = kt + kT * ks;                                              // [kT][d]
  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hd = p.H * d;
  const int q0 = qb * kQ;
  const int qn = min(kQ, p.P - q0);
  for (int i = threadIdx.x; i < qn * d; i += kPThreads) {
    const int r = i / d, c = i - r * d;
    qs[i] = __half2float(p.q[static_cast<size_t>(b * p.P + q0 + r) * hd + head * d + c]) * p.scale;
  }
  const size_t kv0 = (static_cast<size_t>(b) * p.H + head) * p.max_seq * d;
  const int dpl = d / 32;
  float o[kQPerWarp][kMaxDimsPerLane];
  float mrun[kQPerWarp], lrun[kQPerWarp];
#pragma unroll
  for (int r = 0; r < kQPerWarp; ++r) {
    mrun[r] = -INFINITY;
    lrun[r] = 0.f;
#pragma unroll
    for (int e = 0; e < kMaxDimsPerLane; ++e) o[r][e] = 0.f;
  }
  const int last = q0 + qn - 1;  // highest query position of the block
  for (int t0 = 0; t0 <= last; t0 += kT) {
    __syncthreads();
    const int tn = min(kT, last + 1 - t0);
    for (int i = threadIdx.x; i < tn * (d / 8); i += kPThreads) {
      const int j = i / (d / 8), c = (i - j * (d / 8)) * 8;
      const uint4 ku = __ldcg(reinterpret_cast<const uint4*>(p.kc + kv0 + static_cast<size_t>(t0 + j) * d + c));
      const uint4 vu = __ldcg(reinterpret_cast<const uint4*>(p.vc + kv0 + static_cast<size_t>(t0 + j) * d + c));
      uint32_t* kd = reinterpret_cast<uint32_t*>(kt + j * ks + c);  // 4-byte aligned (ks even)
      kd[0] = ku.x;
      kd[1] = ku.y;
      kd[2] = ku.z;
      kd[3] = ku.w;
      *reinterpret_cast<uint4*>(vt + j * d + c) = vu;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kQPerWarp; ++r) {
      const int qi = warp * kQPerWarp + r;
      const int tq = q0 + qi;
      if (qi >= qn) continue;  // warp-uniform
      const int tk = t0 + lane;
      const bool valid = lane < tn && tk <= tq;
      float sc = -INFINITY;
      if (valid) {
        const float* qr = qs + qi * d;
        const __half2* kr = reinterpret_cast<const __half2*>(kt + lane * ks);
        float acc = 0.f;
        for (int c = 0; c < d / 2; ++c) {
          const float2 kf = __half22float2(kr[c]);
          acc = fmaf(qr[2 * c], kf.x, acc);
          acc = fmaf(qr[2 * c + 1], kf.y, acc);
        }
        sc = acc;
      }
      const float mt = ptx::warp_max(sc);
      if (mt == -INFINITY) continue;  // no visible key in this tile (warp-uniform)
      const float mn = fmaxf(mrun[r], mt);
      const float corr = expf(mrun[r] - mn);
      const float pj = valid ? expf(sc - mn) : 0.f;
      lrun[r] = lrun[r] * corr + ptx::warp_sum(pj);
      mrun[r] = mn;
#pragma unroll
      for (int e = 0; e < kMaxDimsPerLane; ++e) o[r][e] *= corr;
      for (int j = 0; j < tn; ++j) {
        const float w = __shfl_sync(0xffffffffu, pj, j);
        if (w == 0.f) continue;  // warp-uniform (same w for every lane)
        const __half* vr = vt + j * d;
#pragma unroll
        for (int e = 0; e < kMaxDimsPerLane; ++e)
          if (e < dpl) o[r][e] = fmaf(w, __half2float(vr[lane + 32 * e]), o[r][e]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kQPerWarp; ++r) {
    const int qi = warp * kQPerWarp + r;
    if (qi >= qn) continue;
    const float inv = 1.0f / lrun[r];
    __half* orow = p.out + static_cast<size_t>(b * p.P + q0 + qi) * hd + head * d;
#pragma unroll
    for (int e = 0; e < kMaxDimsPerLane; ++e)
      if (e < dpl) orow[lane + 32 * e] = __float2half_rn(o[r][e] * inv);
  }
}

// Tensor-core variant (head_dim % 16 == 0, <= 128): FlashAttention-2 style on mma.sync.
// One CTA = 64 queries of one (sequence, head), 4 warps x 16 query rows; K/V tiles of 64 positions
// in shared memory (row stride d + 8 halves: ldmatrix conflict-free).  S = Q K^T and O += P V on
// m16n8k16 (fp16 in, fp32 accumulate), online softmax on the accumulator fragments.
constexpr int kFQ = 64, kFK = 64, kFThreads = 128, kFMaxD = 128;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// 16-byte global -> shared copy without a register round trip (zero-filled when !valid), so a CTA's
// whole tile load is in flight at once instead of one dependent L2 round trip per loop iteration
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <int D>
__global__ void __launch_bounds__(kFThreads) prefill_attention_mma_kernel(const __grid_constant__ PrefillAttnParams p) {
  constexpr int LD = D + 8;       // smem row stride (halves)
  constexpr int NT = D / 8;       // output n-tiles
  constexpr int KS = D / 16;      // k-steps of Q K^T
  extern __shared__ __align__(16) unsigned char fsm[];
  __half* qs = reinterpret_cast<__half*>(fsm);  // [kFQ][LD]
  __half* ks = qs + kFQ * LD;                   // [kFK][LD]
  __half* vs = ks + kFK * LD;                   // [kFK][LD]
  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int hd = p.H * D;
  const int q0 = qb * kFQ;
  const int qn = min(kFQ, p.P - q0);
#pragma unroll
  for (int i = threadIdx.x; i < kFQ * (D / 8); i += kFThreads) {
    const int r = i / (D / 8), c = (i - r * (D / 8)) * 8;
    cp_async16(qs + r * LD + c, p.q + static_cast<size_t>(b * p.P + q0 + min(r, qn - 1)) * hd + head * D + c, r < qn);
  }
  cp_async_wait_all();
  __syncthreads();
  // this warp's Q fragments (rows warp*16 .. +16)
  uint32_t qa[KS][4];
  {
    const uint32_t base = ptx::smem_u32(qs + (warp * 16 + (lane & 15)) * LD + (lane >> 4) * 8);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) ldsm_x4(base + kk * 32, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
  }
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int row0 = q0 + warp * 16 + g;  // query positions of this thread's two rows
  const int row1 = row0 + 8;
  const size_t kv0 = (static_cast<size_t>(b) * p.H + head) * p.max_seq * D;
  const int last = q0 + qn - 1;
  for (int t0 = 0; t0 <= last; t0 += kFK) {
    __syncthreads();
    const int tn = min(kFK, last + 1 - t0);
#pragma unroll
    for (int i = threadIdx.x; i < kFK * (D / 8); i += kFThreads) {
      const int j = i / (D / 8), c = (i - j * (D / 8)) * 8;
      const size_t off = kv0 + static_cast<size_t>(t0 + min(j, tn - 1)) * D + c;
      cp_async16(ks + j * LD + c, p.kc + off, j < tn);
      cp_async16(vs + j * LD + c, p.vc + off, j < tn);
    }
    cp_async_wait_all();
    __syncthreads();
    if (q0 + warp * 16 > last) continue;  // warp has no valid query rows (tail block)
    // S = Q K^T over 64 keys: 8 n-tiles of 8 keys
    float sc[kFK / 8][4];
#pragma unroll
    for (int n = 0; n < kFK / 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int n2 = 0; n2 < kFK / 16; ++n2) {  // two n-tiles per ldmatrix.x4
      const int key = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
      const uint32_t kb = ptx::smem_u32(ks + key * LD + ((lane >> 3) & 1) * 8);
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + kk * 32, b0, b1, b2, b3);
        ptx::mma_f16(sc[2 * n2], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
        ptx::mma_f16(sc[2 * n2 + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
      }
    }
    // scale, causal mask, online softmax (rows g and g + 8 of the warp's 16)
    float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < kFK / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = t0 + n * 8 + 2 * t + (e & 1);
        const int qrow = (e < 2) ? row0 : row1;
        float v = sc[n][e] * p.scale;
        if (key > qrow || key > last) v = -INFINITY;
        sc[n][e] = v;
        mt[e >> 1] = fmaxf(mt[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mt[r] = fmaxf(mt[r], __shfl_xor_sync(0xffffffffu, mt[r], 1));
      mt[r] = fmaxf(mt[r], __shfl_xor_sync(0xffffffffu, mt[r], 2));
      const float mn = fmaxf(mrow[r], mt[r]);
      corr[r] = mn == -INFINITY ? 1.f : expf(mrow[r] - mn);
      mrow[r] = mn;
      lrow[r] *= corr[r];
    }
    // P as a sum of two fp16 terms (hi + lo, ~22 significant bits): the P.V product then carries
    // the fp32 probabilities of the decode attention instead of fp16-rounded ones.  A 2^-11
    // relative error in the attention output is harmless in fp16 but flips int8 quantisation
    // steps of the attn-out activations (W8A8) often enough to show in the logits.
    uint32_t pa[kFK / 16][4], pl[kFK / 16][4];
#pragma unroll
    for (int n = 0; n < kFK / 8; ++n) {
      float pe[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = mrow[e >> 1];
        pe[e] = sc[n][e] == -INFINITY ? 0.f : expf(sc[n][e] - m);
        lrow[e >> 1] += pe[e];
        lo[e] = pe[e] - __half2float(__float2half_rn(pe[e]));
      }
      pa[n >> 1][(n & 1) * 2 + 0] = gemm::dev::pack_h2(pe[0], pe[1]);
      pa[n >> 1][(n & 1) * 2 + 1] = gemm::dev::pack_h2(pe[2], pe[3]);
      pl[n >> 1][(n & 1) * 2 + 0] = gemm::dev::pack_h2(lo[0], lo[1]);
      pl[n >> 1][(n & 1) * 2 + 1] = gemm::dev::pack_h2(lo[2], lo[3]);
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= corr[0];
      o[n][1] *= corr[0];
      o[n][2] *= corr[1];
      o[n][3] *= corr[1];
    }
    // O += P V: k = 64 keys (4 steps), n = D dims; V B-fragments via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < kFK / 16; ++kk) {
      const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
      for (int n2 = 0; n2 < NT / 2; ++n2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(ptx::smem_u32(vs + key * LD + n2 * 16 + (lane >> 4) * 8), b0, b1, b2, b3);
        // A fragment order (a0 a1 a2 a3) = (row g k0-7, row g+8 k0-7, row g k8-15, row g+8 k8-15)
        ptx::mma_f16(o[2 * n2], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
        ptx::mma_f16(o[2 * n2 + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
        ptx::mma_f16(o[2 * n2], pl[kk][0], pl[kk][1], pl[kk][2], pl[kk][3], b0, b1);
        ptx::mma_f16(o[2 * n2 + 1], pl[kk][0], pl[kk][1], pl[kk][2], pl[kk][3], b2, b3);
      }
      if constexpr (NT % 2 == 1) {
        uint32_t b0, b1, b2, b3;
        const int n = NT - 1;
        ldsm_x4_t(ptx::smem_u32(vs + key * LD + n * 8), b0, b1, b2, b3);
        ptx::mma_f16(o[n], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
        ptx::mma_f16(o[n], pl[kk][0], pl[kk][1], pl[kk][2], pl[kk][3], b0, b1);
      }
    }
  }
  if (q0 + warp * 16 > last) return;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = 1.0f / lrow[0], inv1 = 1.0f / lrow[1];
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int c = head * D + n * 8 + 2 * t;
    if (row0 <= last)
      *reinterpret_cast<uint32_t*>(p.out + static_cast<size_t>(b * p.P + row0) * hd + c) =
          gemm::dev::pack_h2(o[n][0] * inv0, o[n][1] * inv0);
    if (row1 <= last)
      *reinterpret_cast<uint32_t*>(p.out + static_cast<size_t>(b * p.P + row1) * hd + c) =
          gemm::dev::pack_h2(o[n][2] * inv1, o[n][3] * inv1);
  }
}

size_t prefill_mma_smem(int d) { return static_cast<size_t>(kFQ + 2 * kFK) * (d + 8) * 2; }

size_t prefill_attn_smem(int d) { return static_cast<size_t>(kQ) * d * 4 + static_cast<size_t>(kT) * (d + 2) * 2 + static_cast<size_t>(kT) * d * 2; }

__global__ void prefill_gather_kernel(const __grid_constant__ PrefillGatherParams p) {
  const int b = blockIdx.x;
  const float4* src = reinterpret_cast<const float4*>(p.res_rows + static_cast<size_t>(b * p.P + p.P - 1) * p.h);
  float4* dst = reinterpret_cast<float4*>(p.res + static_cast<size_t>(b) * p.h);
  long long s1 = 0, s2 = 0;
  for (int c = threadIdx.x; c < p.h / 4; c += blockDim.x) {
    const float4 v = src[c];
    dst[c] = v;
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // the decode epilogues' fixed-point row sums
      s1 += __float2ll_rn(__fmul_rn(e[i], gemm::kSumScale));
      s2 += __float2ll_rn(__fmul_rn(__fmul_rn(e[i], e[i]), gemm::kSqScale));
    }
  }
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
  if (threadIdx.x == 0) {
    long long a = 0, c = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
      a += red[0][w];
      c += red[1][w];
    }
    if (p.ln_stats != nullptr) {  // stripe 0 of the slot (fused-statistics mode)
      p.ln_stats[b * 2] = a;
      p.ln_stats[b * 2 + 1] = c;
    }
    if (b == 0) *p.pos = p.P - 1;
  }
}

__global__ void prefill_residual_add_kernel(float* res, const float* part, const __half* bias, int64_t count, int h) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    res[i] = __fadd_rn(res[i], __fadd_rn(part[i], __half2float(bias[i % h])));
}

}  // namespace

void prefill_residual_add(float* res, const float* part, const __half* bias, int64_t count, int h, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  prefill_residual_add_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(res, part, bias, count, h);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void prefill_embed(const PrefillEmbedParams& p, cudaStream_t s) {
  if (p.h % 8 != 0) throw ConfigError("prefill: hidden_dim must be a multiple of 8");
  prefill_embed_kernel<<<p.B * p.P, 256, 0, s>>>(p);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void configure_prefill() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(prefill_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(prefill_attn_smem(256))));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(prefill_attention_mma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(prefill_mma_smem(64))));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(prefill_attention_mma_kernel<96>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(prefill_mma_smem(96))));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(prefill_attention_mma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(prefill_mma_smem(128))));
}

void prefill_attention(const PrefillAttnParams& p, cudaStream_t s) {
  if (p.d % 32 != 0 || p.d > 32 * kMaxDimsPerLane) throw ConfigError("prefill attention: head dim must be a multiple of 32, <= 256");
  const bool use_mma = !std::getenv("DSINF_PREFILL_SIMT") && (p.d == 64 || p.d == 96 || p.d == kFMaxD);
  if (use_mma) {
    const dim3 grid((p.P + kFQ - 1) / kFQ, p.H, p.B);
    const size_t sm = prefill_mma_smem(p.d);
    if (p.d == 64)
      prefill_attention_mma_kernel<64><<<grid, kFThreads, sm, s>>>(p);
    else if (p.d == 96)
      prefill_attention_mma_kernel<96><<<grid, kFThreads, sm, s>>>(p);
    else
      prefill_attention_mma_kernel<128><<<grid, kFThreads, sm, s>>>(p);
  } else {
    const dim3 grid((p.P + kQ - 1) / kQ, p.H, p.B);
    prefill_attention_kernel<<<grid, kPThreads, prefill_attn_smem(p.d), s>>>(p);
  }
  DSINF_CUDA_CHECK(cudaGetLastError());
}

void prefill_gather(const PrefillGatherParams& p, cudaStream_t s) {
  prefill_gather_kernel<<<p.B, 256, 0, s>>>(p);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

}  // namespace ops
}  // namespace dsinf
