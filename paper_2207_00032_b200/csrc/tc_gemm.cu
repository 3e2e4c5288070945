// tcgen05 / TMEM large-batch GEMM for sm_100a (see tc_gemm.cuh).
//
// One CTA = one 128 x 256 output tile, warp-specialised:
//   warp 0      one elected thread streams x and W K-blocks (128 B wide) with 2-D TMA into a
//               4-stage mbarrier ring (128B swizzle, the canonical K-major UMMA layout);
//   warp 1      allocates 256 TMEM columns (the fp32 / int32 accumulator: lane = row, column = n);
//               one elected thread issues tcgen05.mma (M=128, N=256, K=16 fp16 / 32 int8) four
//               times per stage and frees the stage with tcgen05.commit;
//   warps 2..5  epilogue: wait for the final commit, tcgen05.ld 32 columns at a time (each warp
//               owns the 32 TMEM lanes of its quarter), dequantise / bias / GeLU / RoPE / residual,
//               store straight to global.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include <cudaTypedefs.h>

#include "common.h"
#include "ptx.cuh"
#include "sbi_gemm_dev.cuh"
#include "tc_gemm.cuh"

namespace dsinf {
namespace tc {

namespace {

// ---------------------------------------------------------------- tcgen05 wrappers
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(slot)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major operand in the 128B-swizzle canonical layout:
// rows of 128 B, 8-row core groups 1024 B apart (SBO), descriptor version 1, layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);       // start address
  d |= static_cast<uint64_t>(1) << 16;                      // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;              // SBO
  d |= static_cast<uint64_t>(1) << 46;                      // version
  d |= static_cast<uint64_t>(2) << 61;                      // SWIZZLE_128B
  return d;
}

// Instruction descriptor: K-major A and B, M = 128, N = 256.
//   kind::f16: D f32 (1), A/B f16 (0);  kind::i8: D s32 (2), A/B s8 (1).
template <bool kInt8>
__host__ __device__ constexpr uint32_t instr_desc() {
  return (kInt8 ? 2u : 1u) << 4 | (kInt8 ? 1u : 0u) << 7 | (kInt8 ? 1u : 0u) << 10 |
         static_cast<uint32_t>(kBN >> 3) << 17 | static_cast<uint32_t>(kBM >> 4) << 24;
}

template <bool kInt8>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  if constexpr (kInt8)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}
// Commit to the same barrier in every CTA of `mask` (cluster pair: both CTAs' empty slots).
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   ptx::smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// 2-D TMA box multicast to the same smem offset (and barrier) of every CTA in `mask`.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* map, int c0, int c1, uint64_t* bar, uint16_t mask,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(ptx::smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint4 ld_dsmem_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// 32 lanes x 32 columns of 32-bit: thread t of the warp gets lane (base + t), columns [col, col + 32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- epilogue of one row's 32 columns
template <bool kInt8>
__device__ __forceinline__ void epilogue32(const Params& p, int row, int n0, const uint32_t (&v)[32]) {
  float y[32];
  if constexpr (kInt8) {
    const float xs = p.x_scale[row];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      const float ws = n < p.N ? __ldg(p.w_scale + n) : 0.f;
      y[j] = __fmul_rn(__fmul_rn(static_cast<float>(static_cast<int>(v[j])), xs), ws);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
  }
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < p.N) y[j] = __fadd_rn(y[j], __half2float(p.bias[n0 + j]));
  }
  const bool full = n0 + 32 <= p.N;
  switch (p.epi) {
    case EPI_F32: {
      float* o = static_cast<float*>(p.out) + static_cast<size_t>(row) * p.out_ld + n0;
      if (full && (p.out_ld % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
      } else {
        for (int j = 0; j < 32; ++j)
          if (n0 + j < p.N) o[j] = y[j];
      }
      break;
    }
    case EPI_RESID: {
      float* o = static_cast<float*>(p.out) + static_cast<size_t>(row) * p.out_ld + n0;
      for (int j = 0; j < 32; ++j)
        if (n0 + j < p.N) o[j] = __fadd_rn(o[j], y[j]);
      break;
    }
    case EPI_F16:
    case EPI_GELU_F16: {
      if (p.epi == EPI_GELU_F16) {
#pragma unroll
        for (int j = 0; j < 32; ++j) y[j] = gemm::dev::gelu_tanh(y[j]);
      }
      __half* o = static_cast<__half*>(p.out) + static_cast<size_t>(row) * p.out_ld + n0;
      if (full && (p.out_ld % 8) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 u;
          u.x = gemm::dev::pack_h2(y[j], y[j + 1]);
          u.y = gemm::dev::pack_h2(y[j + 2], y[j + 3]);
          u.z = gemm::dev::pack_h2(y[j + 4], y[j + 5]);
          u.w = gemm::dev::pack_h2(y[j + 6], y[j + 7]);
          *reinterpret_cast<uint4*>(o + j) = u;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (n0 + j < p.N) o[j] = __float2half_rn(y[j]);
      }
      break;
    }
    case EPI_QKV: {
      const int hd = p.heads * p.head_dim;
      const int b = row / p.seq_len;
      const int pos = p.pos0 + (row - b * p.seq_len);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int n = n0 + j;
        if (n >= p.N) break;
        const int sec = n / hd;
        const int rem = n - sec * hd;
        const int head = rem / p.head_dim;
        const int i = rem - head * p.head_dim;
        float y0 = y[j], y1 = y[j + 1];
        if (sec < 2) {  // GPT-J interleaved rotary embedding (same arithmetic as the decode epilogue)
          const float2 cs = p.rope[static_cast<size_t>(pos) * (p.head_dim / 2) + i / 2];
          const float r0 = __fsub_rn(__fmul_rn(y0, cs.x), __fmul_rn(y1, cs.y));
          const float r1 = __fadd_rn(__fmul_rn(y0, cs.y), __fmul_rn(y1, cs.x));
          y0 = r0;
          y1 = r1;
        }
        const __half2 h = __floats2half2_rn(y0, y1);
        if (sec == 0) {
          *reinterpret_cast<__half2*>(p.q_out + static_cast<size_t>(row) * hd + rem) = h;
        } else {
          __half* cache = sec == 1 ? p.k_cache : p.v_cache;
          const size_t off = ((static_cast<size_t>(b) * p.heads + head) * p.max_seq + pos) * p.head_dim + i;
          *reinterpret_cast<__half2*>(cache + off) = h;
        }
      }
      break;
    }
    default:
      break;
  }
}

// Persistent: one CTA per SM walks the tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... (m
// fastest, so the CTAs in flight share a weight tile: W streams from HBM about once, x stays in
// L2).  The accumulator is double-buffered in TMEM (2 x 256 columns): the epilogue warps drain
// tile j while the MMA thread already accumulates tile j + 1, and the TMA ring runs across tile
// boundaries.
// kPair: clusters of 2 CTAs on row tiles (m, m+1) of the same weight tile; each CTA TMA-loads one
// 128-row half of the weight tile and multicasts it to both, halving the L2 -> SM weight traffic;
// both CTAs' MMA commits free a stage in both (the halves live in both CTAs' smem).
template <bool kInt8, bool kPair>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;   // [2] MMA -> epilogue (tcgen05.commit)
  uint64_t* acc_empty = acc_full + 2;     // [2] epilogue -> MMA (128 epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = p.k_blocks;
  const int m_tiles = (p.M + kBM - 1) / kBM;
  // units: single tiles, or (kPair) row-tile pairs handled by the two CTAs of a cluster
  const int m_units = kPair ? (m_tiles + 1) / 2 : m_tiles;
  const int units = m_units * ((p.N + kBN - 1) / kBN);
  const int rank = kPair ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int unit0 = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int ustride = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  auto m_of = [&](int u) { return ((kPair ? 2 * (u % m_units) + rank : u % m_units)) * kBM; };
  auto n_of = [&](int u) { return (u / m_units) * kBN; };

  if (threadIdx.x == 0) {
    ptx::prefetch_tensormap(&p.amap);
    ptx::prefetch_tensormap(&p.bmap);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kPair ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], kEpiThreads);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * kBN);
  tc_fence_before();
  if (kPair)
    ptx::cluster_sync();  // both CTAs' barriers initialised before any multicast lands
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ================= TMA producer (ring continuous across tiles)
      ptx::pdl_wait();
      const uint64_t pol_a = ptx::policy_evict_last();   // x tiles are re-read by every column tile
      const uint64_t pol_b = ptx::policy_evict_normal();
      int it = 0;
      for (int u = unit0; u < units; u += ustride) {
        const int m0 = m_of(u), n0 = n_of(u);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], kStageBytes);
          uint8_t* sa = smem + s * kStageBytes;
          ptx::tma_load_2d(sa, &p.amap, kb * kBK, m0, &full[s], pol_a);
          if constexpr (kPair)  // my half of the weight tile, into both CTAs
            tma_load_2d_mc(sa + kABytes + rank * (kBBytes / 2), &p.bmap, kb * kBK, n0 + rank * (kBN / 2), &full[s],
                           0x3, pol_b);
          else
            ptx::tma_load_2d(sa + kABytes, &p.bmap, kb * kBK, n0, &full[s], pol_b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ================= MMA issuer
      const uint32_t idesc = instr_desc<kInt8>() | (!kInt8 && p.bf16 ? (1u << 7) | (1u << 10) : 0u);
      int it = 0, j = 0;
      for (int u = unit0; u < units; u += ustride, ++j) {
        const int a = j & 1;
        ptx::mbar_wait(&acc_empty[a], ((j >> 1) & 1) ^ 1);  // the epilogue has drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(a * kBN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          ptx::mbar_wait(&full[s], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * kStageBytes);
          const uint64_t da = smem_desc(sa), db = smem_desc(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k)  // 32 bytes of K per MMA (16 fp16 / 32 int8)
            mma<kInt8>(acc, da + static_cast<uint64_t>(k * 2), db + static_cast<uint64_t>(k * 2), idesc,
                       (kb | k) != 0 ? 1u : 0u);
          if constexpr (kPair)
            mma_commit_mc(&empty[s], 0x3);  // both CTAs hold halves of this stage's weight tile
          else
            mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        }
        mma_commit(&acc_full[a]);
      }
    }
  } else {
    // ================= epilogue: warp w owns TMEM lanes [32 (w % 4), +32)
    const int quarter = warp & 3;
    int j = 0;
    for (int u = unit0; u < units; u += ustride, ++j) {
      const int a = j & 1;
      const int m0 = m_of(u), n0 = n_of(u);
      const int row = m0 + quarter * 32 + lane;
      ptx::mbar_wait(&acc_full[a], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(a * kBN + c * 32), v);
        if (row < p.M && n0 + c * 32 < p.N) epilogue32<kInt8>(p, row, n0 + c * 32, v);
      }
      tc_fence_before();
      ptx::mbar_arrive(&acc_empty[a]);  // buffer a may be overwritten by tile j + 2
    }
    ptx::pdl_trigger();
  }
  tc_fence_before();
  if (kPair)
    ptx::cluster_sync();  // the peer's last commits / multicasts into our smem have landed
  else
    __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * kBN);
}

#ifdef DSINF_DIAG
// per-CTA phase stamps of the last split-K launch (`make DIAG=1`, tools/tc_stamps.py)
__device__ unsigned long long g_tc_stamps[4096 * 8];
#define TC_STAMP(k) (g_tc_stamps[blockIdx.x * 8 + (k)] = ptx::gtimer())
#else
#define TC_STAMP(k) ((void)0)
#endif

// Split-K mode for one row tile (M <= 128, the B = 1 prompt): the weights must stream at HBM rate,
// so a 128-column tile is split over a cluster of `split` CTAs along K; each accumulates its K range
// in TMEM, stages the partial tile in its (drained) ring smem, and after a cluster barrier rank r
// sums the ranks' partials for column chunks r, r + split, ... through DSMEM (rank order) and runs
// the fused epilogue on them.
template <bool kInt8, int kSBN>
__global__ void __launch_bounds__(kThreads, kSBN == 128 ? 2 : 1) tc_gemm_splitk_kernel(const __grid_constant__ Params p) {
  constexpr int kSStages = SplitCfg<kSBN>::kStagesS, kSStageBytes = SplitCfg<kSBN>::kStageBytesS;
  constexpr int kSPartLd = SplitCfg<kSBN>::kPartLd;
  constexpr int kQ = kSBN == 128 ? 2 : 4;  // ranks whose partial loads are in flight at once (register budget)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSStages * kSStageBytes);
  uint64_t* empty = full + kSStages;
  uint64_t* acc_ready = empty + kSStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.split;
  const int rank = static_cast<int>(ptx::cluster_ctarank());
  const int n0 = static_cast<int>(blockIdx.x / S) * kSBN;
  const int kps = (p.k_blocks + S - 1) / S;
  const int kb0 = rank * kps, kb1 = min(p.k_blocks, kb0 + kps);
  const int nk = max(0, kb1 - kb0);
  if (threadIdx.x == 0) TC_STAMP(0);
  if (threadIdx.x == 0) {
    ptx::prefetch_tensormap(&p.amap);
    ptx::prefetch_tensormap(&p.bmap);
    for (int st = 0; st < kSStages; ++st) {
      ptx::mbar_init(&full[st], 1);
      ptx::mbar_init(&empty[st], 1);
    }
    ptx::mbar_init(acc_ready, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kSBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TC_STAMP(1);
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = ptx::policy_evict_last();
      const uint64_t pol_b = ptx::policy_evict_first();  // each weight byte is read once
      // weights never depend on the previous kernel: the first ring stages stream before the wait
      const int pre = p.w_early ? min(nk, kSStages) : 0;
      for (int i = 0; i < pre; ++i) {
        ptx::mbar_arrive_expect_tx(&full[i], kSStageBytes);
        ptx::tma_load_2d(smem + i * kSStageBytes + kABytes, &p.bmap, (kb0 + i) * kBK, n0, &full[i], pol_b);
      }
      ptx::pdl_wait();
      TC_STAMP(2);
      for (int i = 0; i < nk; ++i) {
        const int st = i % kSStages;
        uint8_t* sa = smem + st * kSStageBytes;
        if (i >= pre) {
          ptx::mbar_wait(&empty[st], ((i / kSStages) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full[st], kSStageBytes);
          ptx::tma_load_2d(sa + kABytes, &p.bmap, (kb0 + i) * kBK, n0, &full[st], pol_b);
        }
        ptx::tma_load_2d(sa, &p.amap, (kb0 + i) * kBK, 0, &full[st], pol_a);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // instruction descriptor with N = 128
      const uint32_t idesc = ((instr_desc<kInt8>() & ~(0x3fu << 17)) | (static_cast<uint32_t>(kSBN >> 3) << 17)) |
                             (!kInt8 && p.bf16 ? (1u << 7) | (1u << 10) : 0u);
      for (int i = 0; i < nk; ++i) {
        const int st = i % kSStages;
        ptx::mbar_wait(&full[st], (i / kSStages) & 1);
        tc_fence_after();
        if (i == 0) TC_STAMP(3);
        const uint32_t sa = ptx::smem_u32(smem + st * kSStageBytes);
        const uint64_t da = smem_desc(sa), db = smem_desc(sa + kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 32; ++k)
          mma<kInt8>(tmem, da + static_cast<uint64_t>(k * 2), db + static_cast<uint64_t>(k * 2), idesc,
                     (i | k) != 0 ? 1u : 0u);
        mma_commit(&empty[st]);
      }
      TC_STAMP(4);
      mma_commit(acc_ready);
    }
  }
  // partial tile -> own smem (the ring is drained once every MMA has completed)
  uint32_t* part = reinterpret_cast<uint32_t*>(smem);
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;  // epilogue warps 2..5: TMEM lane quarter = warp % 4
  if (warp >= 2) {
    ptx::pdl_wait();  // the epilogue reads / writes activations of the previous kernels
    if (nk > 0) {
      ptx::mbar_wait(acc_ready, 0);
      tc_fence_after();
    }
    if (threadIdx.x == 64) TC_STAMP(5);
#pragma unroll 1
    for (int c = 0; c < kSBN / 32; ++c) {
      uint32_t v[32];
      if (nk > 0) {
        tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<uint4*>(part + row * kSPartLd + c * 32 + j) = make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  tc_fence_before();
  ptx::cluster_sync();  // every rank's partial tile is in its smem
  if (threadIdx.x == 64) TC_STAMP(6);
  if (warp >= 2 && row < p.M) {
    for (int c = rank; c < kSBN / 32; c += S) {
      if (n0 + c * 32 >= p.N) break;
      uint32_t v[32];
      // sum of the S partials of this 32-column chunk, in the fixed order rank, rank + 1, ... (mod S):
      // every rank starts on a different peer, so no CTA's shared memory serves the whole cluster at
      // once; 16 columns x up to 4 ranks of loads in flight per round (deterministic: the chunk's
      // owner and order never change)
      uint32_t acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0u;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        for (int r0 = 0; r0 < S; r0 += 4) {
          uint4 u[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (r0 + q < S) {
              int peer = rank + r0 + q;
              peer -= peer >= S ? S : 0;
              const uint32_t base = ptx::map_shared_rank(part + row * kSPartLd + c * 32 + hh * 16, peer);
#pragma unroll
              for (int j = 0; j < 4; ++j) u[q][j] = ld_dsmem_u4(base + j * 16);
            }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (r0 + q < S) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t w4[4] = {u[q][j].x, u[q][j].y, u[q][j].z, u[q][j].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  uint32_t& d = acc[hh * 16 + 4 * j + e];
                  if constexpr (kInt8)
                    d = static_cast<uint32_t>(static_cast<int>(d) + static_cast<int>(w4[e]));
                  else
                    d = __float_as_uint(__uint_as_float(d) + __uint_as_float(w4[e]));
                }
              }
            }
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = acc[j];
      if (threadIdx.x == 64 && c == rank) TC_STAMP(7);
      epilogue32<kInt8>(p, row, n0 + c * 32, v);
    }
  }
  if (warp >= 2) ptx::pdl_trigger();
  ptx::cluster_sync_relaxed();  // peers are done reading our partials
  if (warp == 1) tmem_dealloc(tmem, kSBN);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable");
  return fn;
}

void byte_map(CUtensorMap* map, const void* base, int rows, int row_bytes, int ld_bytes, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld_bytes % 16) != 0)
    throw ConfigError("tc_gemm: operands need 16-byte aligned bases and row strides");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_bytes), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_bytes)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (tc_gemm) failed: " + std::to_string(static_cast<int>(r)));
}

}  // namespace

int sm_count();

void configure();

// co-resident clusters of `sp` CTAs of the 256-column split-K kernel (cached per size)
int split_clusters(int sp) {
  static int cache[9] = {0};
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (cache[sp] == 0) {
    configure();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sp * 64);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SplitCfg<256>::kSmem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = sp;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    DSINF_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&n, tc_gemm_splitk_kernel<false, 256>, &cfg));
    cache[sp] = std::max(1, n);
  }
  return cache[sp];
}

void make_maps(Params& p, const void* x, int x_ld_bytes, const void* w, int w_ld_bytes, int elem_bytes) {
  if (p.M < 1 || p.N < 1 || p.K < 1) throw ConfigError("tc_gemm: gemm shape dims must be positive");
  const int kbytes = p.K * elem_bytes;
  p.k_blocks = (kbytes + kBK - 1) / kBK;
  byte_map(&p.amap, x, p.M, kbytes, x_ld_bytes, kBM);
  const int m_tiles = (p.M + kBM - 1) / kBM;
  p.pair = m_tiles >= 2 && !std::getenv("DSINF_TC_NOPAIR");
  // one row tile: split K over a cluster so that the weight stream fills every SM
  p.split = 1;
  // measured (tools/tc_kscan.py, M = 128): the 256-column tile at one CTA per SM matches the 128-column
  // tile on QKV / MLP-up and loses on the N = 4096 GEMMs (cluster packing leaves 96-132 CTAs), so 128
  // is the default and DSINF_TC_SBN=256 selects the other
  p.sbn = 128;
  if (const char* v = std::getenv("DSINF_TC_SBN")) p.sbn = std::atoi(v) == 256 ? 256 : 128;
  if (m_tiles == 1 && !std::getenv("DSINF_TC_NOSPLIT")) {
    const int nt = (p.N + p.sbn - 1) / p.sbn;
    if (p.sbn == 128) {
      // measured: clusters of up to 4 keep two CTAs per SM co-resident; 8-CTA clusters and second
      // waves are slower
      while (p.split < 4 && nt * (2 * p.split) <= 2 * sm_count() && p.k_blocks >= 4 * (2 * p.split)) p.split *= 2;
    } else {
      // one CTA per SM: the largest cluster (<= 8) whose nt clusters are co-resident in one wave
      // (cudaOccupancyMaxActiveClusters: clusters are packed per GPC), >= 4 stages per CTA
      p.split = 1;
      for (int sp = 2; sp <= 8; ++sp)
        if (p.k_blocks >= 4 * sp && nt <= split_clusters(sp)) p.split = sp;
    }
    if (const char* v = std::getenv("DSINF_TC_SPLIT")) p.split = std::max(1, std::min(8, std::atoi(v)));
    if (std::getenv("DSINF_TC_DEBUG"))
      std::fprintf(stderr, "tc split-K N=%d K=%d: tile %d split %d clusters(split)=%d\n", p.N, p.K, p.sbn, p.split,
                   p.sbn == 256 ? split_clusters(std::max(1, p.split)) : -1);
  }
  byte_map(&p.bmap, w, p.N, kbytes, w_ld_bytes, p.pair || (p.split > 1 && p.sbn == 128) ? 128 : kBN);
}

void configure() {
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(tc_gemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(tc_gemm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(tc_gemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(tc_gemm_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  auto split_attrs = [](auto kern, int smem) {
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  };
  split_attrs(tc_gemm_splitk_kernel<false, 128>, SplitCfg<128>::kSmem);
  split_attrs(tc_gemm_splitk_kernel<true, 128>, SplitCfg<128>::kSmem);
  split_attrs(tc_gemm_splitk_kernel<false, 256>, SplitCfg<256>::kSmem);
  split_attrs(tc_gemm_splitk_kernel<true, 256>, SplitCfg<256>::kSmem);
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    DSINF_CUDA_CHECK(cudaGetDevice(&dev));
    DSINF_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

void launch(const Params& p, bool int8, cudaStream_t s, bool pdl) {
  const int m_tiles = (p.M + kBM - 1) / kBM, n_tiles = (p.N + kBN - 1) / kBN;
  if (p.split > 1) {
    const int nt = (p.N + p.sbn - 1) / p.sbn;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nt * p.split);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.sbn == 128 ? SplitCfg<128>::kSmem : SplitCfg<256>::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = p.split;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cudaLaunchAttribute attrs[2] = {attr, {}};
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = pdl ? 2 : 1;
    if (p.sbn == 128) {
      if (int8)
        DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_splitk_kernel<true, 128>, p));
      else
        DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_splitk_kernel<false, 128>, p));
    } else {
      if (int8)
        DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_splitk_kernel<true, 256>, p));
      else
        DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_splitk_kernel<false, 256>, p));
    }
    return;
  }
  if (p.pair) {
    const int units = (m_tiles + 1) / 2 * n_tiles;
    const int ctas = 2 * std::min(units, sm_count() / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (int8)
      DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<true, true>, p));
    else
      DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<false, true>, p));
    return;
  }
  const dim3 grid(std::min(m_tiles * n_tiles, sm_count()));
  if (int8)
    tc_gemm_kernel<true, false><<<grid, kThreads, kSmemBytes, s>>>(p);
  else
    tc_gemm_kernel<false, false><<<grid, kThreads, kSmemBytes, s>>>(p);
  DSINF_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tc
}  // namespace dsinf

#ifdef DSINF_DIAG
extern "C" int dsinf_debug_tc_stamps(unsigned long long* host, int n) {
  if (n > 4096 * 8) n = 4096 * 8;
  return cudaMemcpyFromSymbol(host, dsinf::tc::g_tc_stamps, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
#endif
