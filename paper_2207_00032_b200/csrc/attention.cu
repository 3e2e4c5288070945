// Decode attention over the KV cache (paper Deep-Fusion region 2, "transposition plus
// attention"; canonical graph nodes attn_transpose + attention, fusion.hpp:271-277).
//
// One thread-block cluster per (batch row, head); its `C` CTAs split the context into chunks
// (attn_dev.cuh) and merge their (max, sum, output) partials through distributed shared memory.
#include <algorithm>
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

// Merge the C chunk partials of (b, head) across the cluster through DSMEM and write the output
// row (and the int8 row max).  co / cst: this CTA's partial (unnormalised output, max, sum).
__device__ __forceinline__ void merge_chunks_and_store(const AttnParams& p, float* co, float* cst, int head, int b,
                                                       int c, int C, int tid, int nthreads = kAttnThreads) {
  const int d = p.d;
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
  for (int i = c + C * tid; i < d; i += C * nthreads) {
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
  merge_chunks_and_store(p, co, cst, head, b, c, C, tid);
}

// Bulk-copy (TMA, 1-D) variant: the chunk's K and V rows are contiguous in the cache
// ([B][H][max_seq][d]), so one elected thread streams them into a 2-stage shared-memory ring of
// kTmaRows positions (two cp.async.bulk per stage, completion as mbarrier transaction bytes) while
// the CTA scores the previous stage from shared memory: a handful of large DMA requests per CTA
// instead of 16-byte loads on every thread's dependency chain.  Same online softmax and merge
// as attn_chunk / attention_kernel.
constexpr int kTmaRows = 32;

constexpr int kTmaMaxRing = 4;
template <int TPP>
__host__ __device__ constexpr size_t tma_ring_bytes(int d, int ring = 2) {
  return static_cast<size_t>(ring) * 2 * kTmaRows * d * 2;
}

// NT threads per CTA: 128 (default), or 256 (DSINF_ATTN_NT; twice the warps per SM, measured slower)
template <int TPP, int NT>
__host__ __device__ constexpr size_t tma_scratch_floats(int d) {
  return static_cast<size_t>(NT / TPP) * d + 2 * (NT / TPP) + d + 4;
}

template <int TPP, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 4 : 1) attention_tma_kernel(const __grid_constant__ AttnParams p) {
  constexpr int PPR = NT / TPP;  // positions scored in parallel
  constexpr int kU = kTmaRows / PPR;       // positions per thread per stage
  extern __shared__ __align__(128) uint8_t araw[];
  const int d = p.d;
  const size_t stage_halves = static_cast<size_t>(2) * kTmaRows * d;  // K rows then V rows
  __half* ring = reinterpret_cast<__half*>(araw);
  const int R = p.tma_ring;  // ring slots (2..kTmaMaxRing)
  float* scratch = reinterpret_cast<float*>(araw + tma_ring_bytes<TPP>(d, R));
  float* so = scratch;       // [PPR][d]
  float* sm = so + PPR * d;  // [PPR]
  float* sl = sm + PPR;      // [PPR]
  float* co = sl + PPR;      // [d]
  float* cst = co + d;       // [2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      araw + tma_ring_bytes<TPP>(d, R) + (tma_scratch_floats<TPP, NT>(d) * 4 + 7) / 8 * 8);
  const int head = blockIdx.x, b = blockIdx.y, c = blockIdx.z, C = gridDim.z;
  const int tid = threadIdx.x;
  ptx::trace_begin(p.trace);
  if (!p.late_trigger) ptx::pdl_trigger();
  if (tid == 0) {
    for (int r = 0; r < R; ++r) ptx::mbar_init(&bars[r], 1);
    ptx::fence_mbar_init();
  }
  // the position counter and the K/V rows of earlier positions were written by earlier steps (the
  // previous graph launch has completed): with p.early_kv the stages holding only such rows are
  // requested before the wait on this step's QKV GEMM
  const int ctx = *reinterpret_cast<const volatile int*>(p.pos) + 1;
  const int chunk = (ctx + C - 1) / C;
  const int j0 = c * chunk;
  const int j1 = min(ctx, j0 + chunk);
  const int n = max(0, j1 - j0);
  const int nst = (n + kTmaRows - 1) / kTmaRows;
  const size_t kv_base = (static_cast<size_t>(b) * p.H + head) * p.max_seq * d;
  const uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](int st) {
    const int rows = min(kTmaRows, n - st * kTmaRows);
    const uint32_t bytes = static_cast<uint32_t>(rows) * d * 2;
    __half* dst = ring + (st % R) * stage_halves;
    const size_t src = kv_base + static_cast<size_t>(j0 + st * kTmaRows) * d;
    ptx::mbar_arrive_expect_tx(&bars[st % R], 2 * bytes);
    ptx::bulk_g2s(dst, p.kc + src, bytes, &bars[st % R], pol);
    ptx::bulk_g2s(dst + static_cast<size_t>(kTmaRows) * d, p.vc + src, bytes, &bars[st % R], pol);
  };
  __syncthreads();  // barrier init visible
  int issued = 0;
  if (p.early_kv && tid == 0)
    while (issued < min(R, nst) && j0 + (issued + 1) * kTmaRows <= ctx - 1) issue(issued++);  // rows < pos
  ptx::pdl_wait();
  if (p.late_trigger) ptx::pdl_trigger();  // dependents launch once our inputs are complete
  if (tid == 0) {
    for (int st = issued; st < min(R, nst); ++st) issue(st);
  }
  const int slot = tid / TPP, lane_in = tid % TPP;
  const int dim0 = lane_in * 8;
  const bool has_dims = dim0 < d;
  // scores in the log2 domain (q pre-scaled by log2(e)): exp2f is one MUFU.EX2, expf a longer sequence;
  // the CTA's (max, sum) go back to the natural domain before the chunk merge
  constexpr float kLog2e = 1.4426950408889634f;
  float q[8];
  if (has_dims) {
    const uint4 qu = __ldcg(reinterpret_cast<const uint4*>(p.q + static_cast<size_t>(b) * p.H * d + head * d + dim0));
    dev::h8_to_f(qu, q);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] *= p.scale * kLog2e;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = 0.f;
  const bool all_dims = TPP * 8 == d;  // every lane owns 8 dims (d = 64 / 128 / 256)
  int rs = 0;                          // ring slot and its parity, advanced per stage
  uint32_t rph = 0;
  for (int st = 0; st < nst; ++st) {
    ptx::mbar_wait(&bars[rs], rph);
    const __half* ks = ring + rs * stage_halves;
    const __half* vs = ks + static_cast<size_t>(kTmaRows) * d;
    const int rows = min(kTmaRows, n - st * kTmaRows);
    if (rows == kTmaRows && all_dims) {
      // full stage, every lane with dims: no per-position predicates
      float sc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float kf[8];
        dev::h8_to_f(*reinterpret_cast<const uint4*>(ks + static_cast<size_t>(u * PPR + slot) * d + dim0), kf);
        float sdot = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) sdot = fmaf(q[i], kf[i], sdot);
        sc[u] = sdot;
      }
#pragma unroll
      for (int off = TPP / 2; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < kU; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], off);
      float mt = sc[0];
#pragma unroll
      for (int u = 1; u < kU; ++u) mt = fmaxf(mt, sc[u]);
      const float mn = fmaxf(m, mt);
      const float corr = exp2f(m - mn);  // m = -inf on the first stage: 0
      l *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] *= corr;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const float pj = exp2f(sc[u] - mn);
        l += pj;
        float vf[8];
        dev::h8_to_f(*reinterpret_cast<const uint4*>(vs + static_cast<size_t>(u * PPR + slot) * d + dim0), vf);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = fmaf(pj, vf[i], o[i]);
      }
      m = mn;
    } else {
      float sc[kU];
      float mt = -INFINITY;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int r = u * PPR + slot;
        float sdot = 0.f;
        if (r < rows && has_dims) {
          float kf[8];
          dev::h8_to_f(*reinterpret_cast<const uint4*>(ks + static_cast<size_t>(r) * d + dim0), kf);
#pragma unroll
          for (int i = 0; i < 8; ++i) sdot = fmaf(q[i], kf[i], sdot);
        }
#pragma unroll
        for (int off = TPP / 2; off > 0; off >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, off);
        sc[u] = r < rows ? sdot : -INFINITY;
        mt = fmaxf(mt, sc[u]);
      }
      if (mt != -INFINITY) {
        const float mn = fmaxf(m, mt);
        const float corr = exp2f(m - mn);
        l *= corr;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] *= corr;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (sc[u] == -INFINITY) continue;
          const float pj = exp2f(sc[u] - mn);
          l += pj;
          if (has_dims) {
            float vf[8];
            dev::h8_to_f(*reinterpret_cast<const uint4*>(vs + static_cast<size_t>(u * PPR + slot) * d + dim0), vf);
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = fmaf(pj, vf[i], o[i]);
          }
        }
        m = mn;
      }
    }
    __syncthreads();  // every thread is done with this ring slot
    if (tid == 0 && st + R < nst) issue(st + R);
    if (++rs == R) {
      rs = 0;
      rph ^= 1u;
    }
  }
  m = m == -INFINITY ? m : m * 0.69314718055994531f;  // back to the natural-log domain
  // merge the PPR position slots of this CTA (attn_chunk's tail)
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
  for (int i = tid; i < d; i += NT) {
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
  __syncthreads();
  merge_chunks_and_store(p, co, cst, head, b, c, C, tid, NT);
}

// Tensor-core variant (DSINF_ATTN_MMA=1; d in {64, 96, 128}): the bulk-copy ring with K/V rows
// landing at a padded stride (d + 8 halves: the mma fragment loads are conflict-free), scores
// S = K q on mma.m16n8k16 (q in column 0 of B; warps 0-1 take 16 positions each), the online softmax
// on 32 lanes (one position each), and O += P V on mma (P in row 0 of A; each warp 32 dims, V
// fragments by ldmatrix.trans).  q and P are rounded to fp16 for the MMAs, accumulation is fp32.
// row padding in halves: 8 = conflict-free fragment loads but one bulk copy per row (measured 2x
// slower: the single issuing thread serialises 64 copies per stage); 0 = two bulk copies per stage
constexpr int kMmaPad = 0;
__device__ __forceinline__ uint32_t ptx_pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void att_ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__host__ __device__ constexpr size_t mma_stage_halves(int d) { return static_cast<size_t>(2) * kTmaRows * (d + kMmaPad); }
size_t mma_smem_bytes(int d) {
  // ring (2 stages) + q (d halves) + raw scores [32] + co [d] + cst [2] + 2 barriers
  return 2 * mma_stage_halves(d) * 2 + static_cast<size_t>(d) * 2 + 32 * 4 + static_cast<size_t>(d) * 4 + 16 + 16;
}

__global__ void __launch_bounds__(128) attention_mma_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ __align__(128) uint8_t araw[];
  const int d = p.d, SP = d + kMmaPad;
  const size_t stage_halves = mma_stage_halves(d);
  __half* ring = reinterpret_cast<__half*>(araw);
  __half* sq = ring + 2 * stage_halves;
  float* ssc = reinterpret_cast<float*>(sq + d);
  float* co = ssc + 32;
  float* cst = co + d;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(cst + 4) + 0);
  const int head = blockIdx.x, b = blockIdx.y, c = blockIdx.z, C = gridDim.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  ptx::trace_begin(p.trace);
  ptx::pdl_trigger();
  if (tid == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_mbar_init();
  }
  const int ctx = *reinterpret_cast<const volatile int*>(p.pos) + 1;
  const int chunk = (ctx + C - 1) / C;
  const int j0 = c * chunk;
  const int j1 = min(ctx, j0 + chunk);
  const int n = max(0, j1 - j0);
  const int nst = (n + kTmaRows - 1) / kTmaRows;
  const size_t kv_base = (static_cast<size_t>(b) * p.H + head) * p.max_seq * d;
  const uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](int st) {  // one bulk copy per K and V row into the padded stage
    const int rows = min(kTmaRows, n - st * kTmaRows);
    const uint32_t bytes = static_cast<uint32_t>(d) * 2;
    __half* dst = ring + (st & 1) * stage_halves;
    const size_t src = kv_base + static_cast<size_t>(j0 + st * kTmaRows) * d;
    ptx::mbar_arrive_expect_tx(&bars[st & 1], 2 * bytes * rows);
    if (kMmaPad == 0) {  // contiguous rows: one bulk copy each for K and V
      ptx::bulk_g2s(dst, p.kc + src, bytes * rows, &bars[st & 1], pol);
      ptx::bulk_g2s(dst + kTmaRows * SP, p.vc + src, bytes * rows, &bars[st & 1], pol);
    } else {
      for (int r = 0; r < rows; ++r) {
        ptx::bulk_g2s(dst + r * SP, p.kc + src + static_cast<size_t>(r) * d, bytes, &bars[st & 1], pol);
        ptx::bulk_g2s(dst + (kTmaRows + r) * SP, p.vc + src + static_cast<size_t>(r) * d, bytes, &bars[st & 1], pol);
      }
    }
  };
  __syncthreads();  // barrier init visible
  ptx::pdl_wait();
  if (tid == 0) {
    if (nst > 0) issue(0);
    if (nst > 1) issue(1);
  }
  constexpr float kLog2e = 1.4426950408889634f;
  for (int i = tid; i < d; i += 128)
    sq[i] = __float2half_rn(__half2float(__ldcg(p.q + static_cast<size_t>(b) * p.H * d + head * d + i)) * p.scale * kLog2e);
  __syncthreads();
  float m = -INFINITY, l = 0.f;
  float o[4][4];  // this warp's 32 dims: 4 n-tiles (row 0 of the accumulator is the output)
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
  const bool pv_warp = warp * 32 < d;
  for (int st = 0; st < nst; ++st) {
    ptx::mbar_wait(&bars[st & 1], static_cast<uint32_t>((st >> 1) & 1));
    const __half* ks = ring + (st & 1) * stage_halves;
    const __half* vs = ks + kTmaRows * SP;
    const int rows = min(kTmaRows, n - st * kTmaRows);
    if (rows < kTmaRows) {  // rows past the context hold stale bytes: zero their V (P is 0 there)
      __half* vz = const_cast<__half*>(vs);
      for (int i = tid; i < (kTmaRows - rows) * d; i += 128) vz[(rows + i / d) * SP + i % d] = __ushort_as_half(0);
    }
    if (warp < 2) {  // S[16 positions] = K q, k over d in steps of 16
      float sacc[4] = {0.f, 0.f, 0.f, 0.f};
      const __half* kr = ks + (warp * 16) * SP;
      for (int k0 = 0; k0 < d; k0 += 16) {
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(kr + g * SP + k0 + 2 * t);
        const uint32_t a1 = *reinterpret_cast<const uint32_t*>(kr + (g + 8) * SP + k0 + 2 * t);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(kr + g * SP + k0 + 8 + 2 * t);
        const uint32_t a3 = *reinterpret_cast<const uint32_t*>(kr + (g + 8) * SP + k0 + 8 + 2 * t);
        const uint32_t b0 = g == 0 ? *reinterpret_cast<const uint32_t*>(sq + k0 + 2 * t) : 0u;
        const uint32_t b1 = g == 0 ? *reinterpret_cast<const uint32_t*>(sq + k0 + 8 + 2 * t) : 0u;
        ptx::mma_f16(sacc, a0, a1, a2, a3, b0, b1);
      }
      if (t == 0) {  // column 0: positions g and g + 8 of this warp's 16
        ssc[warp * 16 + g] = sacc[0];
        ssc[warp * 16 + g + 8] = sacc[2];
      }
    }
    __syncthreads();
    // online softmax: lane j owns position j of the stage (every warp computes the same values)
    const float sj = lane < rows ? ssc[lane] : -INFINITY;
    float mt = sj;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
    const float mn = fmaxf(m, mt);
    const float corr = exp2f(m - mn);
    const float pj = lane < rows ? exp2f(sj - mn) : 0.f;
    float ps = pj;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l = l * corr + ps;
    m = mn;
    if (pv_warp) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[nt][e] *= corr;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {  // 16 positions per k step
        const float p0 = __shfl_sync(0xffffffffu, pj, kk * 16 + 2 * t);
        const float p1 = __shfl_sync(0xffffffffu, pj, kk * 16 + 2 * t + 1);
        const float p2 = __shfl_sync(0xffffffffu, pj, kk * 16 + 8 + 2 * t);
        const float p3 = __shfl_sync(0xffffffffu, pj, kk * 16 + 8 + 2 * t + 1);
        const uint32_t pa0 = g == 0 ? ptx_pack_h2(p0, p1) : 0u;
        const uint32_t pa2 = g == 0 ? ptx_pack_h2(p2, p3) : 0u;
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
        for (int n2 = 0; n2 < 2; ++n2) {
          uint32_t b0, b1, b2, b3;
          att_ldsm_x4_t(ptx::smem_u32(vs + key * SP + warp * 32 + n2 * 16 + (lane >> 4) * 8), b0, b1, b2, b3);
          ptx::mma_f16(o[2 * n2], pa0, 0u, pa2, 0u, b0, b1);
          ptx::mma_f16(o[2 * n2 + 1], pa0, 0u, pa2, 0u, b2, b3);
        }
      }
    }
    __syncthreads();  // the ring slot and the raw scores are free
    if (tid == 0 && st + 2 < nst) issue(st + 2);
  }
  if (pv_warp && g == 0) {
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      co[warp * 32 + nt * 8 + 2 * t] = o[nt][0];
      co[warp * 32 + nt * 8 + 2 * t + 1] = o[nt][1];
    }
  }
  if (tid == 0) {
    cst[0] = m == -INFINITY ? m : m * 0.69314718055994531f;  // natural-log domain for the merge
    cst[1] = l;
  }
  __syncthreads();
  merge_chunks_and_store(p, co, cst, head, b, c, C, tid, 128);
}

template <int TPP, int NT>
size_t tma_smem_bytes(int d, int ring) {
  return tma_ring_bytes<TPP>(d, ring) + (tma_scratch_floats<TPP, NT>(d) * 4 + 7) / 8 * 8 + 8 * kTmaMaxRing;
}

template <int TPP, int NT>
void configure_tma() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_tma_kernel<TPP, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_tma_kernel<TPP, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  if (carveout_max())
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_tma_kernel<TPP, NT>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}

template <int NT>
void launch_tma(const AttnParams& p, dim3 grid, dim3 cluster, cudaStream_t s, bool pdl) {
  const dim3 block(NT);
  if (p.d <= 64)
    launch_pdl(attention_tma_kernel<8, NT>, grid, block, tma_smem_bytes<8, NT>(p.d, p.tma_ring), s, pdl, p, cluster);
  else if (p.d <= 128)
    launch_pdl(attention_tma_kernel<16, NT>, grid, block, tma_smem_bytes<16, NT>(p.d, p.tma_ring), s, pdl, p, cluster);
  else
    launch_pdl(attention_tma_kernel<32, NT>, grid, block, tma_smem_bytes<32, NT>(p.d, p.tma_ring), s, pdl, p, cluster);
}

}  // namespace

int attention_chunks(int B, int H) {
  // enough CTAs for the KV stream's memory parallelism: (batch, head) pairs x chunks >= target
  const int target = [] {  // read per model (DSINF_ATTN_CTAS)
    const char* v = std::getenv("DSINF_ATTN_CTAS");
    return v ? std::atoi(v) : 2 * 148;
  }();
  const int max_c = [] {
    const char* v = std::getenv("DSINF_ATTN_MAXC");
    return v ? std::max(1, std::min(16, std::atoi(v))) : 8;
  }();
  const int pairs = B * H;
  int c = 1;
  while (c < max_c && pairs * c < target) c <<= 1;
  return c;
}

void configure() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_mma_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  if (carveout_max())
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(attention_mma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  configure_tma<8, 128>();
  configure_tma<16, 128>();
  configure_tma<32, 128>();
  configure_tma<8, 256>();
  configure_tma<16, 256>();
  configure_tma<32, 256>();
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
  // the bulk-copy K/V ring variant (16-byte aligned rows: d % 8 == 0), default; DSINF_ATTN_TMA=0 selects
  // the per-thread pipelined loads.  GPT-J ms/token (per-thread -> bulk): int8 B=1 1.893 -> 1.867,
  // B=8 2.209 -> 2.190; fp16 B=1 2.564 -> 2.554, B=16 3.137 -> 3.123; GPT-2 B=1 fp16 1.650 -> 1.626
  const int tma = [] { const char* v = std::getenv("DSINF_ATTN_TMA"); return v ? std::atoi(v) : 1; }();  // read per enqueue
  if (tma && (reinterpret_cast<uintptr_t>(p.kc) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.vc) & 15) == 0) {
    p.kv_rows_cap = 0;
    // ring slots: enough for a chunk's stages at the largest context, 2..4 (DSINF_ATTN_RING overrides)
    const int max_st = ((p.max_seq + chunks - 1) / chunks + kTmaRows - 1) / kTmaRows;
    const char* rv = std::getenv("DSINF_ATTN_RING");
    p.tma_ring = rv ? std::max(2, std::min(kTmaMaxRing, std::atoi(rv))) : 2;
    p.tma_ring = std::max(2, std::min(p.tma_ring, max_st));
    const char* ev = std::getenv("DSINF_ATTN_EARLY");
    p.early_kv = ev != nullptr && std::atoi(ev) != 0;
    const char* ltv = std::getenv("DSINF_ATTN_LATE_TRIGGER");  // overrides the model's choice
    if (ltv != nullptr) p.late_trigger = std::atoi(ltv) != 0;
    // DSINF_ATTN_NT=256: 256 threads per CTA (measured slower at B = 8 / 16: GPT-J int8 B=16 attention
    // 13.8 -> 15.5 us per layer, fp16 B=8 10.8 -> 12.8; profiles/r2_attn_fastpath_ab.log)
    const char* mmv = std::getenv("DSINF_ATTN_MMA");
    if (mmv != nullptr && std::atoi(mmv) != 0 && (p.d == 64 || p.d == 96 || p.d == 128)) {
      launch_pdl(attention_mma_kernel, grid, dim3(128), mma_smem_bytes(p.d), s, pdl, p, cluster);
      return;
    }
    const char* ntv = std::getenv("DSINF_ATTN_NT");
    const int nt = ntv ? std::atoi(ntv) : 128;
    if (nt == 256)
      launch_tma<256>(p, grid, cluster, s, pdl);
    else
      launch_tma<128>(p, grid, cluster, s, pdl);
    return;
  }
  // DSINF_ATTN_PREFETCH=1 (with DSINF_ATTN_TMA=0): K/V staging before the dependency wait (a chunk's
  // rows at the largest context must fit a 48 KB budget).  Measured slower and off by default: GPT-J
  // B=1 int8 1.929 -> 1.944 ms, fp16 2.564 -> 2.589
  const int pre = [] { const char* v = std::getenv("DSINF_ATTN_PREFETCH"); return v ? std::atoi(v) : 0; }();
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
