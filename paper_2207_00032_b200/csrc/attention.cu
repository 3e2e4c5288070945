// Decode attention over the KV cache (paper Deep-Fusion region 2, "transposition plus
// attention"; canonical graph nodes attn_transpose + attention, fusion.hpp:271-277).
//
// One thread-block cluster per (batch row, head); its `C` CTAs split the context into chunks
// (attn_dev.cuh) and merge their (max, sum, output) partials through distributed shared memory.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "attn_dev.cuh"
#include "common.h"
#include "launch.cuh"
#include "ops.cuh"
#include "sbi_gemm.cuh"
#include "ptx.cuh"

namespace dsinf {
namespace ops {

namespace {

using dev::kAttnThreads;

template <int TPP>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const __grid_constant__ AttnParams p) {
  constexpr int PPR = kAttnThreads / TPP;
  extern __shared__ __align__(16) float asmem[];
  const int d = p.d;
  float* co = asmem + PPR * d + 2 * PPR;  // layout of attn_chunk's scratch
  float* cst = co + d;
  const int head = blockIdx.x, b = blockIdx.y, c = blockIdx.z, C = gridDim.z;
  const int tid = threadIdx.x;
  ptx::trace_begin(p.trace);
  ptx::pdl_trigger();
  // the position counter and the K/V rows of earlier positions were written by earlier steps (the
  // previous graph launch has completed): they are read before the wait on this step's QKV GEMM
  const int pos = *reinterpret_cast<const volatile int*>(p.pos);
  const int ctx = pos + 1;
  const int chunk = (ctx + C - 1) / C;
  const int j0 = c * chunk;
  const int j1 = min(ctx, j0 + chunk);
  const int j_pre = p.kv_rows_cap > 0 ? max(j0, min(j1, pos)) : 0;
  __half* kv = reinterpret_cast<__half*>(asmem + dev::attn_scratch_floats<TPP>(d));
  if (j_pre > j0) {  // cp.async 16-byte pieces of rows [j0, j_pre) of K and V
    const int per_row = d / 8, n = (j_pre - j0) * per_row;
    const size_t kv_base = (static_cast<size_t>(b) * p.H + head) * p.max_seq * d;
    for (int i = tid; i < 2 * n; i += kAttnThreads) {
      const int v = i >= n, ii = v ? i - n : i;
      const int r = ii / per_row, q = ii - r * per_row;
      const __half* src = (v ? p.vc : p.kc) + kv_base + static_cast<size_t>(j0 + r) * d + q * 8;
      __half* dst = kv + (static_cast<size_t>(v) * p.kv_rows_cap + r) * d + q * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  ptx::pdl_wait();
  if (j_pre > j0) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  dev::attn_chunk<TPP>(p, b, head, j0, j1, tid, asmem, [] { __syncthreads(); }, kv, j_pre, p.kv_rows_cap);
  // merge the C chunks of this (b, head) across the cluster
  if (C > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  // every rank's (max, sum) in one DSMEM round trip, then this CTA's output dims (all ranks'
  // partials requested before the first is used)
  constexpr int kMaxC = 16;
  float mr[kMaxC], lr[kMaxC];
#pragma unroll
  for (int r = 0; r < kMaxC; ++r)
    if (r < C) {
      const uint32_t a = ptx::map_shared_rank(&cst[0], r);
      const float2 v = ptx::ld_dsmem_f2_nc(a);
      mr[r] = v.x;
      lr[r] = v.y;
    }
  float MM = -INFINITY;
#pragma unroll
  for (int r = 0; r < kMaxC; ++r)
    if (r < C) MM = fmaxf(MM, mr[r]);
  float wts[kMaxC];
  float LL = 0.f;
#pragma unroll
  for (int r = 0; r < kMaxC; ++r)
    if (r < C) {
      const float w = mr[r] == -INFINITY ? 0.f : expf(mr[r] - MM);
      wts[r] = w;
      LL += w * lr[r];
    }
  const float inv = 1.0f / LL;
  const int hd = p.H * d;
  float amax = 0.f;
  for (int i = c + C * tid; i < d; i += C * kAttnThreads) {
    float part[kMaxC];
#pragma unroll
    for (int r = 0; r < kMaxC; ++r)
      if (r < C) part[r] = ptx::ld_dsmem_f_nc(ptx::map_shared_rank(&co[i], r));
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < kMaxC; ++r)
      if (r < C) acc = fmaf(wts[r], part[r], acc);
    const __half o = __float2half_rn(acc * inv);
    p.out[static_cast<size_t>(b) * hd + head * d + i] = o;
    amax = fmaxf(amax, fabsf(__half2float(o)));
  }
  if (p.amax_out != nullptr) {  // per-token int8 scale input of the attn-out GEMM
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
    if ((tid & 31) == 0 && m != 0)
      atomicMax(p.amax_out + ((head + c) % gemm::kStatStripes) * 32 + b, m);
  }
  if (C > 1) ptx::cluster_sync_relaxed();  // peers' DSMEM reads of our partials are consumed
  ptx::trace_end(p.trace);
}

}  // namespace

int attention_chunks(int B, int H) {
  // enough CTAs for the KV stream's memory parallelism: (batch, head) pairs x chunks >= target
  static const int target = [] {
    const char* v = std::getenv("DSINF_ATTN_CTAS");
    return v ? std::atoi(v) : 2 * 148;
  }();
  const int pairs = B * H;
  int c = 1;
  while (c < 8 && pairs * c < target) c <<= 1;
  return c;
}

void configure() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // the K/V staging area (<= 48 KB) on top of the softmax scratch
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  if (carveout_max()) {
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  configure_step_kernels();
}

void attention(const AttnParams& p_in, int chunks, cudaStream_t s, bool pdl) {
  AttnParams p = p_in;
  if (p.d % 8 != 0 || p.d > 256) throw ConfigError("attention: head dim must be a multiple of 8 and <= 256");
  if (chunks < 1 || chunks > 16) throw ConfigError("attention: bad chunk count");
  const dim3 grid(p.H, p.B, chunks), block(kAttnThreads), cluster(1, 1, chunks);
  // DSINF_ATTN_PREFETCH=1: K/V staging before the dependency wait (a chunk's rows at the largest
  // context must fit a 48 KB budget).  Measured slower and off by default: GPT-J B=1 int8 2.062 ->
  // 2.100 ms, fp16 2.671 -> 2.706; with attention PDL-launched (DSINF_PDL_MASK=0x8f) 2.150 / 2.691
  static const int pre = [] { const char* v = std::getenv("DSINF_ATTN_PREFETCH"); return v ? std::atoi(v) : 0; }();
  const int rows_cap = (p.max_seq + chunks - 1) / chunks;
  const size_t kv_bytes = static_cast<size_t>(2) * rows_cap * p.d * 2;
  p.kv_rows_cap = pre && kv_bytes <= 48 * 1024 ? rows_cap : 0;
  const size_t extra = p.kv_rows_cap > 0 ? kv_bytes : 0;
  if (p.d <= 64)
    launch_pdl(attention_kernel<8>, grid, block, dev::attn_scratch_floats<8>(p.d) * 4 + extra, s, pdl, p, cluster);
  else if (p.d <= 128)
    launch_pdl(attention_kernel<16>, grid, block, dev::attn_scratch_floats<16>(p.d) * 4 + extra, s, pdl, p, cluster);
  else
    launch_pdl(attention_kernel<32>, grid, block, dev::attn_scratch_floats<32>(p.d) * 4 + extra, s, pdl, p, cluster);
}

}  // namespace ops
}  // namespace dsinf
