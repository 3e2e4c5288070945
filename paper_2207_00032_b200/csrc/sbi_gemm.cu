// SBI-GeMM on sm_100a (infersim gemm.hpp:65-202): the standalone kernel.
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
// exactly one A-fragment register of mma.m16n8k16.f16 (mma.m16n8k32.s8).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include <cudaTypedefs.h>

#include "common.h"
#include "ptx.cuh"
#include "sbi_gemm.cuh"
#include "sbi_gemm_dev.cuh"
#include "attn_dev.cuh"

namespace dsinf {
namespace gemm {

namespace {

using dev::Header;

// ---------------------------------------------------------------- QKV attention tail (kXS == 3)
// Deep-Fusion region 2 inside the QKV launch: the cluster whose epilogue
// completes a head's q, k and v columns runs that head's decode attention (the standalone kernel's
// online-softmax chunk, attn_dev.cuh, and its DSMEM chunk merge), so no attention launch and no
// grid drain sit between QKV and attn-out.
constexpr int kTailMaxHeads = 16;  // heads one column tile can complete (q/k/v sections, d >= 8)

// column tiles overlapping columns [lo, hi) of the QKV output
__device__ __forceinline__ int tiles_over(int lo, int hi) { return (hi - 1) / kColTile - lo / kColTile + 1; }

// One (head, batch row): this CTA's context chunk, then the nsplit chunks merged through DSMEM
// (merge_chunks_and_store's arithmetic, attention.cu) into attn_out.  Every thread of the CTA
// calls it (the cluster barriers); the 128 consumer threads compute.
template <int TPP>
__device__ __forceinline__ void attn_tail_one(const Params& p, int head, int b, int split, int nsplit, float* scr, int ctx) {
  constexpr int PPR = ops::dev::kAttnThreads / TPP;
  ops::AttnParams a{};
  a.q = p.q_out;
  a.kc = p.k_cache;
  a.vc = p.v_cache;
  a.pos = p.pos;
  a.B = p.B;
  a.H = p.heads;
  a.d = p.head_dim;
  a.max_seq = p.max_seq;
  a.scale = p.attn_scale;
  const int d = p.head_dim;
  const int tid = static_cast<int>(threadIdx.x) - 32;  // consumer index, < 0 on the producer warp
  const int chunk = (ctx + nsplit - 1) / nsplit;
  const int j0 = split * chunk, j1 = min(ctx, j0 + chunk);
  if (tid >= 0) ops::dev::attn_chunk<TPP>(a, b, head, j0, j1, tid, scr, [] { dev::consumer_bar(); });
  float* co = scr + PPR * d + 2 * PPR;
  float* cst = co + d;
  if (nsplit > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  if (tid >= 0) {
    // the ranks' (max, sum) re-read from DSMEM where needed: no per-rank register arrays (the
    // kernel's register budget is the GEMM main loop's, 3 CTAs per SM)
    float MM = -INFINITY;
    for (int r = 0; r < nsplit; ++r) MM = fmaxf(MM, ptx::ld_dsmem_f2_nc(ptx::map_shared_rank(&cst[0], r)).x);
    float LL = 0.f;
    for (int r = 0; r < nsplit; ++r) {
      const float2 v = ptx::ld_dsmem_f2_nc(ptx::map_shared_rank(&cst[0], r));
      LL += (v.x == -INFINITY ? 0.f : expf(v.x - MM)) * v.y;
    }
    const float inv = 1.0f / LL;
    const int hd = p.heads * d;
    float amax = 0.f;
    for (int i = split + nsplit * tid; i < d; i += nsplit * ops::dev::kAttnThreads) {
      float acc = 0.f;
      for (int r = 0; r < nsplit; ++r) {
        const float mr = ptx::ld_dsmem_f2_nc(ptx::map_shared_rank(&cst[0], r)).x;
        const float w = mr == -INFINITY ? 0.f : expf(mr - MM);
        acc = fmaf(w, ptx::ld_dsmem_f_nc(ptx::map_shared_rank(&co[i], r)), acc);
      }
      const __half o = __float2half_rn(acc * inv);
      p.attn_out[static_cast<size_t>(b) * hd + head * d + i] = o;
      amax = fmaxf(amax, fabsf(__half2float(o)));
    }
    if (p.attn_amax != nullptr) {  // per-token int8 scale input of the attn-out GEMM
      const unsigned mx = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
      if ((tid & 31) == 0 && mx != 0) atomicMax(p.attn_amax + ((head + split) % kStatStripes) * 32 + b, mx);
    }
  }
  // peers' DSMEM reads of our partials are consumed before the scratch is reused
  if (nsplit > 1)
    ptx::cluster_sync_relaxed();
  else
    __syncthreads();
}

// After the epilogue: count this tile's (section, head) pieces; run the heads it completes.
__device__ __forceinline__ void attn_tail(const Params& p, uint8_t* ring, int tile, int split, int nsplit) {
  __shared__ int s_heads[kTailMaxHeads + 1];  // [0] = count (read by the peers through DSMEM)
  if (nsplit > 1)
    ptx::cluster_sync();  // every CTA's epilogue stores precede rank 0's release below
  else
    __syncthreads();
  if (split == 0 && threadIdx.x == 0) {
    const int d = p.head_dim, hd = p.heads * d, n0 = tile * kColTile;
    int cnt = 0;
    __threadfence();
    for (int sec = 0; sec < 3; ++sec) {
      const int lo = max(n0, sec * hd), hi = min(min(n0 + kColTile, p.N), (sec + 1) * hd);
      if (lo >= hi) continue;
      for (int h = (lo - sec * hd) / d; h <= (hi - 1 - sec * hd) / d; ++h) {
        int need = 0;
        for (int s2 = 0; s2 < 3; ++s2) need += tiles_over(s2 * hd + h * d, s2 * hd + (h + 1) * d);
        const unsigned old = atomicAdd(p.head_ctr + h, 1u);
        if (old + 1 == static_cast<unsigned>(need)) {
          p.head_ctr[h] = 0u;  // every piece of this step arrived: reset for the next step
          if (cnt < kTailMaxHeads) s_heads[1 + cnt++] = h;
        }
      }
    }
    __threadfence();  // acquire the other clusters' q / k / v stores before the peers read them
    s_heads[0] = cnt;
  }
  if (nsplit > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  // rank 0's head list (read per head below: no dynamically indexed local array)
  auto list_at = [&](int i) {
    return nsplit > 1 ? __float_as_int(ptx::ld_dsmem_f_nc(ptx::map_shared_rank(&s_heads[i], 0))) : s_heads[i];
  };
  const int cnt = list_at(0);
  if (cnt == 0) {
    if (nsplit > 1) ptx::cluster_sync_relaxed();  // rank 0's head list is read before it exits
    return;
  }
  const int ctx = *p.pos + 1;
  float* scr = reinterpret_cast<float*>(ring + 16 * 1024);  // past the split-K partials (<= 8.4 KB)
  for (int i = 0; i < cnt; ++i) {
    const int head = list_at(1 + i);
    for (int b = 0; b < p.B; ++b) {
      if (p.head_dim <= 64)
        attn_tail_one<8>(p, head, b, split, nsplit, scr, ctx);
      else if (p.head_dim <= 128)
        attn_tail_one<16>(p, head, b, split, nsplit, scr, ctx);
      else
        attn_tail_one<32>(p, head, b, split, nsplit, scr, ctx);
    }
  }
}

// Dynamic smem (base rounded up to 1024 B for the 128B swizzle):
//   [ring: stages x 16 KB] [header 1 KB] [x slice: B rows x x_row_words words]
// After the main loop the ring is reused for the split-K partials part[b][n].
// kXS (x-streaming, large batch): stages are 18 KB (weights + the x box), no x slice.
// kA16 (int8 weights only): W8A16 -- x stays fp16 (slice of fp16 pairs, or two x boxes per
// 128-k stage when streamed), weights widened in registers, fp32 accumulate, y = acc * w_scale.
// kXS: 0 smem x slice, 1 x-streaming, 2 LayerNorm-streaming (fp32 residual boxes per stage,
// normalised by the consumers into the stage's fp16 x boxes; fp16 or W8A16 weights).
template <bool kInt8, int kNB8, int kXS, int kA16>
__global__ void __launch_bounds__(kThreads, kXS == 3 ? 3 : 1) sbi_gemm_kernel(const __grid_constant__ Params p) {
  static_assert(!kA16 || kInt8, "W8A16 needs int8 weights");
  constexpr bool kLN = kXS >= 2;  // 3: LayerNorm-streaming + the QKV attention tail
  static_assert(!kLN || !kInt8 || kA16, "LayerNorm-streaming takes fp16 or W8A16 weights");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  constexpr int kXBoxes = kA16 ? 2 : 1;           // fp16 x boxes per streamed stage
  constexpr int kRBoxes = kLN ? 2 * kXBoxes : 0;  // fp32 residual boxes per stage (LayerNorm-streaming)
  // activation box slot: kXBoxBytes (16 rows), or for LayerNorm-streaming 1 KB when B <= 8 (one
  // 128B-swizzle atom), so the small-batch ring keeps 4 stages (p.box_bytes, set by launch)
  const int kBoxSlot = kLN ? p.box_bytes : kXBoxBytes;
  const int kSB = kLN ? kStageBytes + (kRBoxes + kXBoxes) * kBoxSlot
                      : (kXS ? (kA16 ? kStageBytesXS16 : kStageBytesXS) : kStageBytes);
  const int kXOff = kStageBytes + kRBoxes * kBoxSlot;  // the x boxes within a stage
  constexpr int kKPerRow = kInt8 ? 4 : 2;        // k per packed weight row
  uint8_t* ring = smem;
  Header& hd = *reinterpret_cast<Header*>(smem + stages * kSB);
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + stages * kSB + kHeaderBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int split = blockIdx.y;
  const int nsplit = gridDim.y;
  const int n0 = tile * kColTile;
  const int row_begin = split * p.rows_per_split;
  const int row_end = min(p.rows, row_begin + p.rows_per_split);
  const int n_iters = (row_end - row_begin + kRowsPerStage - 1) / kRowsPerStage;

  __shared__ dev::EpiStats es;
  ptx::trace_begin(p.trace);
#ifdef DSINF_DIAG
  unsigned long long* clog = p.cta_log ? p.cta_log + 6 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
#else
  constexpr unsigned long long* clog = nullptr;
#endif
  if (clog && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    clog[0] = smid;
    clog[1] = ptx::gtimer();
  }
  if (threadIdx.x == 0) {
    ptx::prefetch_tensormap(&p.tmap);
    if (kXS) ptx::prefetch_tensormap(&p.xmap);
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&hd.full[s], 1);
      ptx::mbar_init(&hd.empty[s], kConsumerWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ================= producer: one elected thread issues 4 TMA boxes per stage
    if (kXS && lane == 0) {
      // weights of the first `stages` stages before the dependency, their x boxes after it
      const uint64_t policy = ptx::policy_evict_first();
      const uint64_t xpolicy = ptx::policy_evict_last();  // x is re-read by every column tile
      const uint32_t tx = kStageBytes + (kLN ? kRBoxes : kXBoxes) * p.B * 128;
      // the stage's activation boxes: GEMM-ready x words, or (kLN) the fp32 residual of its k range
      auto load_x = [&](int it, uint8_t* st) {
        const int r0 = row_begin + it * kRowsPerStage;
        if constexpr (kLN) {
#pragma unroll
          for (int rb = 0; rb < kRBoxes; ++rb)
            ptx::tma_load_2d(st + kStageBytes + rb * kBoxSlot, &p.xmap, kKPerRow * r0 + rb * 32, 0,
                             &hd.full[it % stages], xpolicy);
        } else {
#pragma unroll
          for (int xb = 0; xb < kXBoxes; ++xb)
            ptx::tma_load_2d(st + kStageBytes + xb * kXBoxBytes, &p.xmap, kXBoxes * r0 + xb * kRowsPerStage, 0,
                             &hd.full[it % stages], xpolicy);
        }
      };
      const int pre = min(stages, n_iters);
      for (int it = 0; it < pre; ++it) {
        ptx::mbar_arrive_expect_tx(&hd.full[it], tx);
        const int r0 = row_begin + it * kRowsPerStage;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w)
          ptx::tma_load_2d(ring + it * kSB + w * kBoxBytes, &p.tmap, n0 + w * kWarpCols, r0, &hd.full[it], policy);
      }
      if (p.dep_flags != nullptr) {  // only the x-producing tiles of this split's k range
        const long long step = *reinterpret_cast<const volatile long long*>(p.dep_step);
        const unsigned target = static_cast<unsigned>(step + 1) * p.dep_per_step;
        const int t0 = (row_begin * kKPerRow) / kColTile, t1 = (row_end * kKPerRow - 1) / kColTile;
        for (int t = t0; t <= t1; ++t) {
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.dep_flags + t) : "memory");
          } while (static_cast<int>(v - target) < 0);
        }
        ptx::fence_proxy_async_global();  // the TMA (async proxy) reads what the flags published
      } else {
        ptx::pdl_wait();
      }
      for (int it = 0; it < pre; ++it) load_x(it, ring + it * kSB);
      int s = pre % stages;
      uint32_t phase = pre == stages ? 1u : 0u;
      for (int it = pre; it < n_iters; ++it) {
        ptx::mbar_wait(&hd.empty[s], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&hd.full[s], tx);
        const int r0 = row_begin + it * kRowsPerStage;
        uint8_t* dst = ring + s * kSB;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w)
          ptx::tma_load_2d(dst + w * kBoxBytes, &p.tmap, n0 + w * kWarpCols, r0, &hd.full[s], policy);
        load_x(it, dst);
        if (++s == stages) {
          s = 0;
          phase ^= 1;
        }
      }
    } else if (lane == 0) {
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
    // All of this CTA's weight loads are issued: let the next kernel launch and stream its own
    // weights into our tail (triggering at kernel start lets a cascade of dependents occupy SMs).
    ptx::pdl_trigger();
  } else {
    // ================= consumers
    const int cw = warp - 1;
    const int ctid = threadIdx.x - 32;
    const bool flag_dep = kXS == 1 && p.dep_flags != nullptr;  // x by TMA after the producer's flag wait
    // LayerNorm-streaming: gamma / beta of this split's k range into smem (weights: before the wait)
    __half* sg = reinterpret_cast<__half*>(sx);
    __half* sb = sg + p.rows_per_split * kKPerRow;
    if constexpr (kLN) {
      const int k0 = row_begin * kKPerRow, nk = p.rows_per_split * kKPerRow;  // nk % 64 == 0
      for (int i = ctid; i < nk / 8; i += 128) {
        const int k = k0 + 8 * i;
        uint4 g = make_uint4(0u, 0u, 0u, 0u), b = make_uint4(0u, 0u, 0u, 0u);
        if (k < p.K) {  // K % 8 == 0 on this plan
          g = __ldg(reinterpret_cast<const uint4*>(p.ln_g + k));
          b = __ldg(reinterpret_cast<const uint4*>(p.ln_b + k));
        }
        reinterpret_cast<uint4*>(sg)[i] = g;
        reinterpret_cast<uint4*>(sb)[i] = b;
      }
    }
    // K-group scales of this CTA's stages -> smem [stage][128 columns] (weights: before the wait)
    const int x_region = kLN ? 2 * p.rows_per_split * kKPerRow * 2 : (kXS ? 0 : p.B * p.x_row_words * 4);
    __half* sgs = reinterpret_cast<__half*>(reinterpret_cast<uint8_t*>(sx) + x_region);
    if constexpr ((kA16 & 4) != 0) {
      {
        const int g0 = row_begin / kRowsPerStage;
        for (int i = ctid; i < n_iters * (kColTile / 8); i += 128) {  // 8 columns (16 B) per item
          const int it = i / (kColTile / 8), c8 = (i - it * (kColTile / 8)) * 8;
          const int n = n0 + c8;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          const __half* src = p.w_gscale + static_cast<size_t>(g0 + it) * p.N + n;
          if (n + 8 <= p.N && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            v = __ldg(reinterpret_cast<const uint4*>(src));
          } else {
            unsigned short h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int e = 0; e < 8; ++e)
              if (n + e < p.N) h[e] = __half_as_ushort(src[e]);
            v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
          }
          *reinterpret_cast<uint4*>(sgs + it * kColTile + c8) = v;
        }
      }
    }
    if (!flag_dep) ptx::pdl_wait();
#ifdef DSINF_DIAG
    const unsigned long long t_rel = ptx::trace_release(p.trace, 32);
    const long long c_rel = ptx::clk();
#else
    constexpr long long c_rel = 0;
#endif
    if (clog && threadIdx.x == 32) clog[2] = ptx::gtimer();
    if (p.red_flag != nullptr) {  // fused all-reduce: every rank's partial has landed
      if (ctid == 0) ptx::wait_flag(p.red_flag, p.step_ctr, p.red_per_step);
      dev::consumer_bar();
    }
    if (kLN) {  // the residual arrives with the weights; the row statistics come from the producer
      if (ctid < p.B) dev::ln_from_sums(p.ln_stats_in, ctid, p.ln_inv_k, p.ln_eps, hd.mean[ctid], hd.rstd[ctid]);
    } else if (kXS) {  // x arrives with the weights; only the per-token int8 scales are needed
      if (kInt8 && !kA16 && ctid < p.B) hd.xscale[ctid] = p.x_scale[ctid];
    } else if (kA16) {  // fp16 x slice, in units of fp16 pairs: twice the packed int8 rows
      if (p.pro == PRO_LN && p.ln_stats_in != nullptr) {
        dev::fill_x_ln_f16_pre(p, sx, hd, 2 * row_begin, 2 * p.rows_per_split, ctid, c_rel);
      } else {
        if (p.pro == PRO_LN) dev::ln_row_stats<false>(p, hd, ctid, cw, lane, p.res_out != nullptr && tile == 0 && split == 0);
        dev::consumer_bar();
        dev::fill_x_slice<false>(p, sx, hd, 2 * row_begin, 2 * p.rows_per_split, ctid);
      }
    } else if (!kInt8 && p.pro == PRO_LN && p.ln_stats_in != nullptr) {
      dev::fill_x_ln_f16_pre(p, sx, hd, row_begin, p.rows_per_split, ctid, c_rel);
    } else if (kInt8 && p.pro == PRO_LN && p.ln_stats_in != nullptr && dev::ln_i8_fits(p.B, p.K)) {
      dev::fill_x_ln_i8_regs(p, sx, hd, row_begin, p.rows_per_split, ctid, cw, lane);
    } else if (kInt8 && p.pro == PRO_QUANT && p.amax_in != nullptr && (p.x_ld % 4) == 0 && (p.K % 4) == 0 &&
               (reinterpret_cast<uintptr_t>(p.x) & 7) == 0) {
      dev::fill_x_quant_pre(p, sx, hd, row_begin, p.rows_per_split, ctid, c_rel);
    } else {
      if (p.pro == PRO_LN)
        dev::ln_row_stats<kInt8>(p, hd, ctid, cw, lane, p.res_out != nullptr && tile == 0 && split == 0);
      else if (p.pro == PRO_QUANT)
        dev::quant_row_scale(p, hd, ctid, cw, lane);
      else if (p.pro == PRO_I8 && ctid < p.B)
        hd.xscale[ctid] = p.x_scale[ctid];
      dev::consumer_bar();
      dev::fill_x_slice<kInt8>(p, sx, hd, row_begin, p.rows_per_split, ctid);
    }
    dev::consumer_bar();
#ifdef DSINF_DIAG
    ptx::trace_prologue_end(p.trace, 32, t_rel);
#endif
    if (clog && threadIdx.x == 32) clog[3] = ptx::gtimer();

    dev::Consumer<kInt8, kNB8, kA16> c;
    c.init(lane);
    c.zero();
    int s = 0;
    uint32_t phase = 0;
    // LayerNorm-streaming: the 128 consumer threads turn stage st's fp32 residual boxes into its fp16
    // x boxes ((v - mean) rstd g + b, row_prep's expression), then a consumer barrier
    auto ln_pre = [&](int st, int it) {
      if constexpr (kLN) {
        uint8_t* stg = ring + st * kSB;
        const int kl0 = it * kRowsPerStage * kKPerRow;  // k offset of the stage within the split
        constexpr int W = kXBoxes * 32;               // fp16 x words per row per stage
        for (int i = ctid; i < p.B * W; i += 128) {
          const int r = i / W, w = i - r * W;
          const int e = 2 * w, rb = e >> 5, ee = e & 31;
          const float2 v = *reinterpret_cast<const float2*>(stg + kStageBytes + rb * kBoxSlot + r * 128 +
                                                            (((ee >> 2) ^ (r & 7)) << 4) + (ee & 3) * 4);
          const __half2 g2 = *reinterpret_cast<const __half2*>(sg + kl0 + e);
          const __half2 b2 = *reinterpret_cast<const __half2*>(sb + kl0 + e);
          const float mean = hd.mean[r], rstd = hd.rstd[r];
          const uint32_t word = dev::pack_h2((v.x - mean) * rstd * __low2float(g2) + __low2float(b2),
                                             (v.y - mean) * rstd * __high2float(g2) + __high2float(b2));
          const int xb = w >> 5, ww = w & 31;
          *reinterpret_cast<uint32_t*>(stg + kXOff + xb * kBoxSlot + r * 128 + (((ww >> 2) ^ (r & 7)) << 4) +
                                       (ww & 3) * 4) = word;
        }
        dev::consumer_bar();
      }
    };
    if constexpr (kA16) {
      const int g = lane >> 2, t = lane & 3;
      // K-group scales: stage i of this split is group row_begin / kRowsPerStage + i
      // K-group scales from the staged smem copy ([stage][128]; written before the consumer barrier)
      const __half* gs = (kA16 & 4) != 0 ? sgs + cw * kWarpCols : nullptr;
      const int gs_valid = kWarpCols;  // out-of-range columns were staged as 0
      if constexpr (kXS) {  // x word pair 2 * (4 kk + t) of batch row r in the stage's two boxes
        c.run_a16(ring, kSB, hd, stages, s, phase, n_iters, cw, lane, [&](int st, int, int kk, int bt) {
          const int r = bt * 8 + g;
          if (r >= p.B) return make_uint2(0u, 0u);
          const int w = 8 * kk + 2 * t, ww = w & 31;
          const uint8_t* xb = ring + st * kSB + kXOff + (w >> 5) * kBoxSlot;
          return *reinterpret_cast<const uint2*>(xb + r * 128 + (((ww >> 2) ^ (r & 7)) << 4) + (ww & 3) * 4);
        }, 1, gs, kColTile, gs_valid, ln_pre);
      } else {
        const int xrw = p.x_row_words;
        c.run_a16(ring, kSB, hd, stages, s, phase, n_iters, cw, lane, [&](int, int it, int kk, int bt) {
          const int r = bt * 8 + g;
          if (r >= p.B) return make_uint2(0u, 0u);
          return *reinterpret_cast<const uint2*>(sx + r * xrw + it * 2 * kRowsPerStage + 8 * kk + 2 * t);
        }, 1, gs, kColTile, gs_valid);
      }
    } else if constexpr (kXS) {
      c.run_xs(ring, hd, stages, s, phase, n_iters, p.B, cw, lane, kSB, kXOff, ln_pre);
    } else {
      c.run(ring, hd, stages, s, phase, n_iters, sx, p.x_row_words, p.B, cw, lane);
    }
#ifdef DSINF_DIAG
    ptx::trace_phase_max(p.trace, 4, 32);
#endif
    if (clog && threadIdx.x == 32) clog[4] = ptx::gtimer();
    ptx::pdl_trigger();
    dev::consumer_bar();  // every consumer is done reading the ring
    c.store(reinterpret_cast<typename dev::Consumer<kInt8, kNB8, kA16>::Acc*>(ring), kPartLd, p.B, cw);
  }

  // ================= split-K reduction across the cluster (DSMEM) + epilogue
  if (p.dep_flags != nullptr) ptx::pdl_wait();  // the epilogue's residual / outputs: whole previous grid
  if (nsplit > 1)
    ptx::cluster_sync();
  else
    __syncthreads();
  const int rank = split;  // cluster dims (1, nsplit, 1): rank == blockIdx.y
  const int cols_per_rank = kColTile / nsplit;
  const int c_begin = rank * cols_per_rank;
  const int pairs = cols_per_rank / 2;
  const uint8_t* part_base = ring;
  const bool want_stats = p.ln_stats_out != nullptr || p.amax_out != nullptr;
  // lane groups of gp = min(32, pow2 >= pairs) lanes per batch row (lanes over column pairs), so
  // a warp covers 32 / gp rows at once and the row statistics reduce with in-group shuffles
  const int gp = pairs >= 32 ? 32 : dev::next_pow2(pairs);
  const int rpw = 32 / gp;                      // rows per warp per pass
  const int rows_per_pass = rpw * (kThreads / 32);
  for (int b0 = 0; b0 < p.B; b0 += rows_per_pass) {
    const int b = b0 + warp * rpw + lane / gp;  // this lane's row (may be >= B: shuffles only)
    const bool brow = b < p.B;
    dev::RowStat st;
    unsigned long long best = 0;  // fused argmax (p.am_out)
    for (int q = lane & (gp - 1); brow && q < pairs; q += gp) {
      const int c = c_begin + 2 * q;
      const int n = n0 + c;
      if (n >= p.N) continue;
      const bool has1 = n + 1 < p.N;
      float2 rin = make_float2(0.f, 0.f);  // issue the residual / scale reads ahead of the DSMEM reads
      if (p.epi == EPI_RESID) {
        const float* o = static_cast<const float*>(p.out) + static_cast<size_t>(b) * p.out_ld + n;
        rin.x = __ldcg(o);
        if (has1) rin.y = __ldcg(o + 1);
      }
      float2 ws = make_float2(0.f, 0.f);
      if constexpr (kInt8) {
        if ((kA16 & 4) != 0) {  // K-group scales were applied in the main loop
          ws = make_float2(1.f, 1.f);
        } else {
          ws.x = __ldg(p.w_scale + n);
          if (has1) ws.y = __ldg(p.w_scale + n + 1);
        }
      }
      const uint32_t off = static_cast<uint32_t>((b * kPartLd + c) * 4);
      // the ranks' partials in batches of 4 DSMEM loads in flight, summed in rank order
      float y0, y1;
      if constexpr (kInt8 && !kA16) {
        int s0 = 0, s1 = 0;
        for (int r0 = 0; r0 < nsplit; r0 += 4) {
          uint2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + u < nsplit) v[u] = ptx::ld_dsmem_u2(ptx::map_shared_rank(part_base + off, r0 + u));
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + u < nsplit) {
              s0 += static_cast<int>(v[u].x);
              s1 += static_cast<int>(v[u].y);
            }
        }
        dev::dequant_pair_ws(hd, b, s0, s1, ws, has1, y0, y1);
      } else {
        float2 acc2 = make_float2(0.f, 0.f);
        for (int r0 = 0; r0 < nsplit; r0 += 4) {
          uint2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + u < nsplit) v[u] = ptx::ld_dsmem_u2(ptx::map_shared_rank(part_base + off, r0 + u));
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + u < nsplit) {
              acc2.x += __uint_as_float(v[u].x);
              acc2.y += __uint_as_float(v[u].y);
            }
        }
        y0 = acc2.x;
        y1 = acc2.y;
        if constexpr (kA16) {  // weight-only dequant: per output row scale
          y0 = __fmul_rn(y0, ws.x);
          y1 = has1 ? __fmul_rn(y1, ws.y) : 0.f;
        }
      }
      if (p.push_n > 0) {  // fused all-reduce: this rank's partial into every rank's slot
        const size_t o = static_cast<size_t>(b) * p.out_ld + n;
        for (int q = 0; q < p.push_n; ++q) {
          if (has1)
            *reinterpret_cast<float2*>(p.push_dst[q] + o) = make_float2(y0, y1);
          else
            p.push_dst[q][o] = y0;
        }
        continue;
      }
      dev::epilogue_pair(p, b, n, y0, y1, has1, &st, p.epi == EPI_RESID ? &rin : nullptr);
      if (p.am_out != nullptr) {
        if (n < p.am_valid) best = max(best, argmax_key(y0, p.am_offset + n));
        if (has1 && n + 1 < p.am_valid) best = max(best, argmax_key(y1, p.am_offset + n + 1));
      }
    }
    if (p.am_out != nullptr) {
      for (int o = gp >> 1; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (brow && (lane & (gp - 1)) == 0 && best != 0) atomicMax(p.am_out + b, best);
    }
    if (want_stats) dev::row_stat_commit_group(st, es, brow ? b : 0, lane, gp, brow);
  }
  if (want_stats) {
    __syncthreads();
    dev::stats_flush(p, es, (tile + split) % kStatStripes);
  }
  if (p.out_flags != nullptr) {  // column-tile counter for flag-granular consumers (DSINF_DOWN_FLAGS)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.out_flags + tile) : "memory");
    }
  }
  if (p.push_n > 0) {  // publish the pushed partials: one system-scope release per destination rank
    __syncthreads();
    if (threadIdx.x == 0) {
      // one system-scope fence, then fire-and-forget reductions: returning atomics serialised one
      // round trip per destination (t of them) at the end of every CTA, on the consumers' critical path
      if (p.push_gpu_scope) {
        __threadfence();
        for (int q = 0; q < p.push_n; ++q)
          asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(p.push_flag[q]) : "memory");
      } else if (p.push_done != nullptr) {
        // every CTA's pushes ordered at gpu scope before its counter bump; the last CTA acquires them
        // all, fences at system scope once and signals each destination rank once
        __threadfence();
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(p.push_done) : "memory");
        const unsigned long long step = static_cast<unsigned long long>(*reinterpret_cast<const volatile long long*>(p.push_step));
        if (old + 1 == (step + 1) * p.push_ctas) {
          __threadfence_system();
          for (int q = 0; q < p.push_n; ++q)
            asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(p.push_flag[q]) : "memory");
        }
      } else {
        __threadfence_system();
        for (int q = 0; q < p.push_n; ++q)
          asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(p.push_flag[q]) : "memory");
      }
    }
  }
  // keep our smem alive until the peers' DSMEM reads are done (their values are consumed before
  // they arrive, so no release ordering -- and no GPU-scope fence over our epilogue stores -- needed)
  if constexpr (kXS == 3) {
    attn_tail(p, ring, tile, split, nsplit);  // its cluster barriers also keep our partials alive
  } else {
    if (nsplit > 1) ptx::cluster_sync_relaxed();
  }
  ptx::trace_end(p.trace);
  if (clog && threadIdx.x == 0) clog[5] = ptx::gtimer();
}

template <bool kInt8, int kNB8, int kXS, int kA16 = 0>
void launch_impl(const Params& p, const Plan& plan, cudaStream_t stream, bool pdl) {
  auto kern = sbi_gemm_kernel<kInt8, kNB8, kXS, kA16>;
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

template <bool kInt8, int kNB8, int kXS, int kA16 = 0>
void configure_one() {
  auto kern = sbi_gemm_kernel<kInt8, kNB8, kXS, kA16>;
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
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

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Co-resident clusters of `split` CTAs for this kernel / smem (cached; 0 when unknown).
const void* kernel_ptr(bool int8_weights, int nb8, bool xs, bool a16, bool ln = false) {
  if (ln) {
    if (a16) return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1, 2, true>)
                             : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2, 2, true>);
    return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<false, 1, 2, false>)
                    : reinterpret_cast<const void*>(sbi_gemm_kernel<false, 2, 2, false>);
  }
  if (a16) {
    if (xs) return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1, true, true>)
                            : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2, true, true>);
    return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1, false, true>)
                    : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2, false, true>);
  }
  if (int8_weights) {
    if (xs) return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1, true, false>)
                            : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2, true, false>);
    return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<true, 1, false, false>)
                    : reinterpret_cast<const void*>(sbi_gemm_kernel<true, 2, false, false>);
  }
  if (xs) return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<false, 1, true, false>)
                          : reinterpret_cast<const void*>(sbi_gemm_kernel<false, 2, true, false>);
  return nb8 == 1 ? reinterpret_cast<const void*>(sbi_gemm_kernel<false, 1, false, false>)
                  : reinterpret_cast<const void*>(sbi_gemm_kernel<false, 2, false, false>);
}

int resident_clusters(bool int8_weights, int nb8, bool xs, bool a16, int split, size_t smem, bool ln = false) {
  static std::mutex mu;
  static std::map<std::tuple<bool, int, bool, bool, int, size_t, bool>, int> cache;
  const auto key = std::make_tuple(int8_weights, nb8, xs, a16, split, smem, ln);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const void* kern = kernel_ptr(int8_weights, nb8, xs, a16, ln);
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
  configure_one<false, 1, false>();
  configure_one<false, 2, false>();
  configure_one<true, 1, false>();
  configure_one<true, 2, false>();
  configure_one<false, 1, true>();
  configure_one<false, 2, true>();
  configure_one<true, 1, true>();
  configure_one<true, 2, true>();
  configure_one<true, 1, false, true>();
  configure_one<true, 2, false, true>();
  configure_one<true, 1, true, true>();
  configure_one<true, 2, true, true>();
  configure_one<false, 1, 2>();
  configure_one<false, 2, 2>();
  configure_one<true, 1, 2, true>();
  configure_one<true, 2, 2, true>();
  // biased-weight W8A16 (the decode model's weights)
  configure_one<true, 1, 0, 2>();
  configure_one<true, 2, 0, 2>();
  configure_one<true, 1, 1, 2>();
  configure_one<true, 2, 1, 2>();
  configure_one<true, 1, 2, 2>();
  configure_one<true, 2, 2, 2>();
  // LayerNorm-streaming QKV with the attention tail (kXS = 3): fp16 and biased W8A16
  configure_one<false, 1, 3, 0>();
  configure_one<false, 2, 3, 0>();
  configure_one<true, 1, 3, 2>();
  configure_one<true, 2, 3, 2>();
  // W8A16 with K-group scales (kA16 | 4): signed (drop-in) and biased (model) weights
  configure_one<true, 1, 0, 5>();
  configure_one<true, 2, 0, 5>();
  configure_one<true, 1, 1, 5>();
  configure_one<true, 2, 1, 5>();
  configure_one<true, 1, 0, 6>();
  configure_one<true, 2, 0, 6>();
  configure_one<true, 1, 1, 6>();
  configure_one<true, 2, 1, 6>();
  configure_one<true, 1, 2, 6>();
  configure_one<true, 2, 2, 6>();
}

void make_x_map(CUtensorMap* map, const void* x, int words, int B, int ld_words) {
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 || (ld_words % 4) != 0)
    throw ConfigError("sbi_gemm: streamed x needs a 16-byte aligned base and row stride");
  if (B < 1 || B > kMaxB) throw ConfigError("sbi_gemm: batch must be 1..16 per launch");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(words), static_cast<cuuint64_t>(B)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_words) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kRowsPerStage), static_cast<cuuint32_t>(B)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(x), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (x) failed: " + std::to_string(static_cast<int>(r)));
}

bool prefer_x_stream(int B, bool tp) {
  const int v = env_int("DSINF_XS", -1);
  return v < 0 ? (B >= kXsMinBatch || tp) : v != 0;
}

bool x_streamable(const void* x, int x_ld, int K, bool int8_x) {
  const int m = int8_x ? 4 : 2;
  const size_t row_bytes = static_cast<size_t>(x_ld) * (int8_x ? 1 : 2);
  return x != nullptr && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (row_bytes % 16) == 0 && (K % m) == 0;
}

// B200 launch plan (the device half of derive_schedule, gemm.hpp:65-96): like the reference it
// splits K only when the output tiles alone cannot occupy the machine, but it sizes the split
// so that the whole grid is ONE wave of co-resident clusters (every CTA starts streaming at
// once, no tail wave) and reduces the split in-cluster.
Plan make_plan(int N, int K, int B, bool int8_weights, int forced_split, bool x_stream, bool a16, bool ln_stream,
               bool a16_biased, bool k_groups, int stage_cap) {
  if (N < 1 || K < 1 || B < 1 || B > kMaxB) throw ConfigError("sbi_gemm: bad shape");
  if (a16 && !int8_weights) throw ConfigError("sbi_gemm: W8A16 needs int8 weights");
  if (ln_stream && (!x_stream || (int8_weights && !a16)))
    throw ConfigError("sbi_gemm: LayerNorm-streaming needs the x-streaming plan with fp16 or W8A16 weights");
  const int m = int8_weights ? 4 : 2;
  const int rows = (K + m - 1) / m;
  const int xw = a16 ? 2 : 1;  // x-slice words per packed row
  Plan pl{};
  pl.x_stream = x_stream ? 1 : 0;
  pl.ln_stream = ln_stream ? 1 : 0;
  pl.k_groups = k_groups && a16 ? 1 : 0;
  pl.a16 = a16 ? (a16_biased ? 2 : 1) : 0;
  pl.col_tiles = (N + kColTile - 1) / kColTile;
  pl.nb8 = B <= 8 ? 1 : 2;
  const size_t x_budget = 64 * 1024;
  const size_t stage_bytes = ln_stream ? kStageBytes + (a16 ? 6 : 3) * ln_box_bytes(B)
                                       : (x_stream ? (a16 ? kStageBytesXS16 : kStageBytesXS) : kStageBytes);
  auto rps_for = [&](int s) {
    int r = (rows + s - 1) / s;
    return (r + kRowsPerStage - 1) / kRowsPerStage * kRowsPerStage;
  };
  // smem x slice of the non-streaming mode (the streaming mode keeps x in the ring stages)
  // (LayerNorm-streaming: the split's gamma and beta, fp16, in place of the slice)
  // (+ the K-group scales of the CTA's stages: 128 fp16 per stage)
  auto x_bytes = [&](int rps) {
    const size_t gbytes = pl.k_groups ? static_cast<size_t>(rps / kRowsPerStage) * kColTile * 2 : 0;
    if (ln_stream) return static_cast<size_t>(2) * rps * m * 2 + gbytes;
    return (x_stream ? size_t{0} : static_cast<size_t>(B) * (xw * rps + 8) * 4) + gbytes;
  };
  auto valid = [&](int s) {
    const int rps = rps_for(s);
    if ((rows + rps - 1) / rps != s) return false;  // no empty split
    return x_bytes(rps) <= x_budget;
  };
  // ring depth: 4 stages; W8A16 at B <= 2 takes 3 (GPT-J int8 B=1 1.868 -> 1.838 ms; B=8: 2.187 -> 2.237
  // and B=16: 2.587 -> 2.747 with 3, so larger batches keep 4).  DSINF_STAGES overrides.
  int max_stages = std::max(1, std::min(kMaxStages, env_int("DSINF_STAGES", a16 && B <= 2 ? 3 : 4)));
  if (stage_cap > 0) max_stages = std::min(kMaxStages, stage_cap);  // per-GEMM ring depth request
  const int cap_per_sm = env_int("DSINF_CTA_PER_SM", 0);
  auto smem_for = [&](int s, int* stages_out) {
    const int rps = rps_for(s);
    const int iters = rps / kRowsPerStage;
    const size_t fixed = 1024 /*alignment slack*/ + kHeaderBytes + x_bytes(rps);
    int st = std::min(max_stages, std::max(1, iters));
    while (st > 2 && fixed + st * stage_bytes > 110 * 1024) --st;
    if (stages_out) *stages_out = st;
    const size_t part_bytes = static_cast<size_t>(B) * kPartLd * 4;
    return fixed + std::max(static_cast<size_t>(st) * stage_bytes, part_bytes);
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
      const int clusters = resident_clusters(int8_weights, pl.nb8, x_stream, a16, s, smem_for(s, nullptr), ln_stream);
      int capacity = clusters > 0 ? clusters * s : 2 * 148;
      if (cap_per_sm > 0) capacity = std::min(capacity, cap_per_sm * 148);  // leave room for PDL overlap
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
  p.a16 = plan.a16;
  if (p.w_gscale != nullptr && !(int8_weights && plan.a16 && plan.k_groups))
    throw ConfigError("sbi_gemm: K-group scales need int8 weights on a W8A16 plan made with k_groups");
  if (plan.k_groups && p.w_gscale == nullptr) throw ConfigError("sbi_gemm: a k_groups plan needs the K-group scales");
  p.x_row_words = (plan.a16 ? 2 : 1) * plan.rows_per_split + 8;
  p.ln_inv_k = 1.0 / static_cast<double>(p.K);
  if (p.B < 1 || p.B > kMaxB) throw ConfigError("sbi_gemm: batch must be 1..16 per launch");
  if (p.pro == PRO_LN && (p.K % 8) != 0) throw ConfigError("LayerNorm prologue needs K % 8 == 0");
  if (p.push_n > 0 && (p.epi != EPI_F32 || p.bias != nullptr || p.push_n > 8 || (p.out_ld % 2) != 0))
    throw ConfigError("sbi_gemm: the fused all-reduce pushes the plain fp32 partial (no bias)");
  if (p.am_out != nullptr && (p.epi != EPI_F32 || p.bias != nullptr))
    throw ConfigError("sbi_gemm: the fused argmax needs the plain fp32 epilogue without bias");
  const bool xs = plan.x_stream != 0;
  const bool i8x = int8_weights && !plan.a16;  // int8 activations
  if (plan.a16 && p.pro != PRO_F16 && p.pro != PRO_LN) throw ConfigError("sbi_gemm: W8A16 takes fp16 x (PRO_F16 / PRO_LN)");
  if (p.dep_flags != nullptr && !(xs && !plan.ln_stream && !i8x))
    throw ConfigError("sbi_gemm: flag-granular dependencies need the fp16 / W8A16 x-streaming plan");
  if (plan.ln_stream) {
    if (p.pro != PRO_LN || p.ln_stats_in == nullptr || p.res_in == nullptr || p.ln_g == nullptr || p.ln_b == nullptr)
      throw ConfigError("sbi_gemm: LayerNorm-streaming needs PRO_LN with the producer's row sums");
    if (p.K % 8 != 0 || p.res_delta != nullptr || p.res_out != nullptr)
      throw ConfigError("sbi_gemm: LayerNorm-streaming takes a final residual row (K % 8 == 0)");
    if ((reinterpret_cast<uintptr_t>(p.ln_g) & 15) != 0 || (reinterpret_cast<uintptr_t>(p.ln_b) & 15) != 0)
      throw ConfigError("sbi_gemm: LayerNorm-streaming needs 16-byte aligned gamma / beta");
    make_x_map(&p.xmap, p.res_in, p.K, p.B, p.K);  // fp32 residual [B][K] as 32-bit words
    p.box_bytes = ln_box_bytes(p.B);
  } else if (xs) {
    if (p.pro != (i8x ? PRO_I8 : PRO_F16))
      throw ConfigError("sbi_gemm: the x-streaming plan needs GEMM-ready x (fp16, or int8 for W8A8)");
    if (!x_streamable(p.x, p.x_ld, p.K, i8x)) throw ConfigError("sbi_gemm: x cannot be streamed (alignment)");
    // words: W8A8 int8 quads (= packed rows); fp16 pairs otherwise (W8A16: 2 per packed row)
    make_x_map(&p.xmap, p.x, plan.a16 ? 2 * p.rows : p.rows, p.B, p.x_ld / (i8x ? 4 : 2));
  }
#define DSINF_LAUNCH(I8, NB, XS, A16) launch_impl<I8, NB, XS, A16>(p, plan, stream, pdl)
  if (p.attn_tail) {  // QKV + attention tail: LayerNorm-streaming fp16 or biased W8A16 only
    if (!plan.ln_stream || plan.k_groups || (plan.a16 != 0 && plan.a16 != 2) || (int8_weights && !plan.a16) ||
        p.epi != EPI_QKV || p.head_ctr == nullptr || p.attn_out == nullptr || p.head_dim % 8 != 0 ||
        p.head_dim > 256)
      throw ConfigError("sbi_gemm: the attention tail needs the LayerNorm-streaming QKV plan (fp16 / biased W8A16)");
    if (plan.a16) {
      if (plan.nb8 == 1) DSINF_LAUNCH(true, 1, 3, 2); else DSINF_LAUNCH(true, 2, 3, 2);
    } else {
      if (plan.nb8 == 1) DSINF_LAUNCH(false, 1, 3, 0); else DSINF_LAUNCH(false, 2, 3, 0);
    }
  } else if (plan.k_groups) {  // W8A16 with K-group scales: kA16 = 5 (signed) / 6 (biased)
    const int x = plan.ln_stream ? 2 : (xs ? 1 : 0);
    if (plan.a16 == 2) {
      if (plan.nb8 == 1) {
        if (x == 2) DSINF_LAUNCH(true, 1, 2, 6); else if (x == 1) DSINF_LAUNCH(true, 1, 1, 6); else DSINF_LAUNCH(true, 1, 0, 6);
      } else {
        if (x == 2) DSINF_LAUNCH(true, 2, 2, 6); else if (x == 1) DSINF_LAUNCH(true, 2, 1, 6); else DSINF_LAUNCH(true, 2, 0, 6);
      }
    } else {
      if (x == 2) throw ConfigError("sbi_gemm: LayerNorm-streaming K-group plans take biased weights");
      if (plan.nb8 == 1) {
        if (x == 1) DSINF_LAUNCH(true, 1, 1, 5); else DSINF_LAUNCH(true, 1, 0, 5);
      } else {
        if (x == 1) DSINF_LAUNCH(true, 2, 1, 5); else DSINF_LAUNCH(true, 2, 0, 5);
      }
    }
  } else if (plan.a16 == 2) {  // biased-weight W8A16
    const int x = plan.ln_stream ? 2 : (xs ? 1 : 0);
    if (plan.nb8 == 1) {
      if (x == 2) DSINF_LAUNCH(true, 1, 2, 2); else if (x == 1) DSINF_LAUNCH(true, 1, 1, 2); else DSINF_LAUNCH(true, 1, 0, 2);
    } else {
      if (x == 2) DSINF_LAUNCH(true, 2, 2, 2); else if (x == 1) DSINF_LAUNCH(true, 2, 1, 2); else DSINF_LAUNCH(true, 2, 0, 2);
    }
  } else if (plan.ln_stream) {
    if (plan.a16) {
      if (plan.nb8 == 1) DSINF_LAUNCH(true, 1, 2, true); else DSINF_LAUNCH(true, 2, 2, true);
    } else {
      if (plan.nb8 == 1) DSINF_LAUNCH(false, 1, 2, false); else DSINF_LAUNCH(false, 2, 2, false);
    }
  } else if (plan.a16) {
    if (plan.nb8 == 1) {
      if (xs) DSINF_LAUNCH(true, 1, true, true); else DSINF_LAUNCH(true, 1, false, true);
    } else {
      if (xs) DSINF_LAUNCH(true, 2, true, true); else DSINF_LAUNCH(true, 2, false, true);
    }
  } else if (int8_weights) {
    if (plan.nb8 == 1) {
      if (xs) DSINF_LAUNCH(true, 1, true, false); else DSINF_LAUNCH(true, 1, false, false);
    } else {
      if (xs) DSINF_LAUNCH(true, 2, true, false); else DSINF_LAUNCH(true, 2, false, false);
    }
  } else {
    if (plan.nb8 == 1) {
      if (xs) DSINF_LAUNCH(false, 1, true, false); else DSINF_LAUNCH(false, 1, false, false);
    } else {
      if (xs) DSINF_LAUNCH(false, 2, true, false); else DSINF_LAUNCH(false, 2, false, false);
    }
  }
#undef DSINF_LAUNCH
}

}  // namespace gemm
}  // namespace dsinf
