// Persistent decode-step kernel (PAPER.md:1004-1006 taken to its limit): ONE
// launch per decode step runs the embedding, every layer's Deep-Fusion regions
// and the LM head + greedy argmax, for tensor-parallel degree 1.
//
// Warp roles per CTA (all CTAs co-resident, cooperative launch):
//   warp 0      producer: claims work units (one 128-column tile x a chunk of 32-row weight
//               stages) with an atomic ticket, warms them into L2, and streams their stages
//               through the TMA ring.  It runs ahead across phase boundaries (weights never
//               depend on activations) and never waits for a dependency.
//   warps 1..4  consumers: per phase wait for the previous phase, build the x vector (LayerNorm /
//               quantisation prologue), then per unit run the warp MMAs and push the unit's
//               partial sums straight to the tile accumulator in L2 with fire-and-forget integer
//               reductions (exact int32 for INT8; 2^-32 fixed point in int64 for FP16), so the
//               sum is independent of arrival order: deterministic without ordering.
//   warp 5      sync warp: per unit, fence + ticket; the unit that completes a tile reads the
//               accumulator back, resets it and runs the fused epilogue (bias, RoPE + KV append,
//               GeLU, residual add, LM-head argmax).  Global synchronisation never stalls the
//               MMA warps.
// Dynamic claiming balances the phase: a CTA that falls behind simply claims fewer units, so
// nobody idles at the phase boundary waiting for a statically assigned straggler.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "attn_dev.cuh"
#include "common.h"
#include "ptx.cuh"
#include "sbi_gemm.cuh"
#include "sbi_gemm_dev.cuh"
#include "step_kernel.cuh"

namespace dsinf {
namespace step {

namespace {

using gemm::kColTile;
using gemm::kRowsPerStage;
using gemm::kStageBytes;
using gemm::dev::consumer_bar;
using gemm::dev::Header;

enum Kind : int { K_EMBED = 0, K_GEMM = 1, K_ATTN = 2, K_LM = 3 };
constexpr int kMaxLookahead = 4;
constexpr int kUnitQueue = 8;
constexpr int kThreadsStep = 32 * (gemm::kConsumerWarps + 2);
constexpr float kFix = 4294967296.0f;  // 2^32 fixed-point scale of FP16-path partials

struct Phase {
  int kind;
  int idx;       // gemm params index / attention layer index
  int tiles;     // 128-column tiles
  int spt;       // 32-row stages per tile
  int cs;        // stages per unit
  int cpt;       // units (chunks) per tile
  int units;     // tiles * cpt
  int full_x;    // the whole x vector of this phase is staged in smem once
  unsigned target;  // completion-counter increments per step
  int chunk_major;  // claim order: 1 = chunk-major (units in flight spread over all tiles)
};

// Unit -> (tile, chunk) in claim order.
__device__ __forceinline__ int unit_tile(const Phase& f, int u) { return f.chunk_major ? u % f.tiles : u / f.cpt; }
__device__ __forceinline__ int unit_chunk(const Phase& f, int u) { return f.chunk_major ? u / f.tiles : u % f.cpt; }

struct Prog {
  const Phase* phases;
  int n_phases;
  const gemm::Params* params;
  const ops::AttnParams* attn;
  int attn_chunks;
  ops::EmbedParams embed;
  void* acc;          // tile accumulators [tiles][B][128] (int64 fixed point or int32), kept zero
  float* attn_ws;
  int* tile_cnt;
  int* attn_cnt;
  unsigned* claim;    // per phase
  unsigned* done;     // per phase
  unsigned* arrived;
  unsigned* epoch;
  float* am_val;
  int* am_idx;
  int lm_tiles;
  int lm_valid;
  float* logits;
  int logits_ld;
  int32_t* next_tok;
  int32_t* hist;
  int* pos;
  int max_ctx;
  int B, stages, lookahead;
  size_t x_bytes_;            // smem bytes reserved for the x vector
  unsigned long long* trace;  // optional [G][n_phases][4] globaltimer stamps (DSINF_STEP_TRACE)
};

// Per-CTA bookkeeping shared between the warp roles (lives in the 1 KB header region).
struct Extra {
  uint64_t ufull[kUnitQueue];
  uint64_t uempty[kUnitQueue];
  int ent_phase[kUnitQueue];
  int ent_tile[kUnitQueue];
  int meta[gemm::kMaxStages];
  int meta_last[gemm::kMaxStages];  // stage belongs to the CTA's last unit of its phase
  float xs[2][gemm::kMaxB];  // per-token activation scales by phase parity (sync warp dequant)
  int sflag[4];
};
static_assert(sizeof(Header) + sizeof(Extra) <= gemm::kHeaderBytes, "header region too small");

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// slot: 0 consumer reaches the phase, 1 dependency satisfied, 2 consumer done, 3 producer moved on,
//       4 sync warp took a unit of the phase, 5 sync warp finished a tile, 6 sync warp published done
__device__ __forceinline__ void trace_rec(const Prog& P, int cta, int p, int slot) {
  if (P.trace) P.trace[(static_cast<size_t>(cta) * P.n_phases + p) * 8 + slot] = gtime();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Consumers of a phase wait until the previous phase has completed this step's work.
__device__ __forceinline__ void wait_phase(const Prog& P, int p, unsigned epoch, int ctid) {
  if (p < 0) return;
  const unsigned target = (epoch + 1u) * P.phases[p].target;
  if (ctid == 0)
    while (static_cast<int>(ld_relaxed(P.done + p) - target) < 0) __nanosleep(20);
  consumer_bar();
  (void)ld_acquire(P.done + p);
}

// ------------------------------------------------------------------ producer (one thread)
__device__ void producer(const Prog& P, uint8_t* ring, Header& hd, Extra& ex, unsigned epoch, int cta, int G) {
  const uint64_t pol = ptx::policy_evict_first();
  const int stages = P.stages;
  int s = 0;
  uint32_t ph = 0;
  int it = 0;
  int qp[kMaxLookahead], qu[kMaxLookahead];
  int qh = 0, qn = 0;
  int cp = 0;  // phase being claimed
  auto claim = [&]() -> bool {
    while (cp < P.n_phases) {
      const Phase f = P.phases[cp];
      if (f.kind == K_GEMM || f.kind == K_LM) {
        const unsigned c = atomicAdd(P.claim + cp, 1u);
        const int u = static_cast<int>(c - epoch * static_cast<unsigned>(f.units + G));
        if (u < f.units) {
          const int slot = (qh + qn) % kMaxLookahead;
          qp[slot] = cp;
          qu[slot] = u;
          ++qn;
          // warm the unit's weights into L2 now; the ring loads follow when slots free up
          const gemm::Params& gp = P.params[f.idx];
          const int tile = unit_tile(f, u), st0 = unit_chunk(f, u) * f.cs, st1 = min(f.spt, st0 + f.cs);
          for (int st = st0; st < st1; ++st)
#pragma unroll
            for (int w = 0; w < gemm::kConsumerWarps; ++w)
              ptx::tma_prefetch_l2_2d(&gp.tmap, tile * kColTile + w * gemm::kWarpCols, st * kRowsPerStage);
          return true;
        }
        trace_rec(P, cta, cp, 3);
      }
      ++cp;
    }
    return false;
  };
  while (qn < P.lookahead && claim()) {
  }
  while (qn > 0) {
    const int p = qp[qh], u = qu[qh];
    qh = (qh + 1) % kMaxLookahead;
    --qn;
    while (qn < P.lookahead && claim()) {
    }
    // is this the CTA's last unit of phase p?  (the refill above already tried to claim more)
    const int last = (qn == 0 || qp[qh] != p) ? 1 : 0;
    const Phase f = P.phases[p];
    const gemm::Params& gp = P.params[f.idx];
    const int tile = unit_tile(f, u), st0 = unit_chunk(f, u) * f.cs, st1 = min(f.spt, st0 + f.cs);
    for (int st = st0; st < st1; ++st) {
      if (it >= stages) ptx::mbar_wait(&hd.empty[s], ph ^ 1);
      ex.meta[s] = (p << 20) | u;
      ex.meta_last[s] = last;
      ptx::mbar_arrive_expect_tx(&hd.full[s], kStageBytes);
      uint8_t* dst = ring + s * kStageBytes;
#pragma unroll
      for (int w = 0; w < gemm::kConsumerWarps; ++w)
        ptx::tma_load_2d(dst + w * gemm::kBoxBytes, &gp.tmap, tile * kColTile + w * gemm::kWarpCols,
                         st * kRowsPerStage, &hd.full[s], pol);
      ++it;
      if (++s == stages) {
        s = 0;
        ph ^= 1;
      }
    }
  }
  // end-of-step sentinel: a stage with no bytes
  if (it >= stages) ptx::mbar_wait(&hd.empty[s], ph ^ 1);
  ex.meta[s] = -1;
  ptx::mbar_arrive(&hd.full[s]);
}

// ------------------------------------------------------------------ sync warp
// Greedy token of the step from the per-tile argmaxes (tile order == vocabulary order, so
// keeping the first maximum keeps the lowest id), then publish the next position / epoch.
__device__ void finalize_step(const Prog& P, unsigned epoch, int pos, int G, int lane) {
  if (lane == 0)
    while (static_cast<int>(ld_relaxed(P.arrived) - (epoch + 1u) * static_cast<unsigned>(G)) < 0) __nanosleep(64);
  __syncwarp();
  (void)ld_acquire(P.arrived);
  for (int b = lane; b < P.B; b += 32) {
    float bv = -INFINITY;
    int bi = 0;
    for (int t = 0; t < P.lm_tiles; ++t) {
      const float v = __ldcg(P.am_val + t * P.B + b);
      const int i = __ldcg(P.am_idx + t * P.B + b);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
    P.next_tok[b] = bi;
    if (pos + 1 < P.max_ctx) P.hist[static_cast<size_t>(b) * P.max_ctx + pos + 1] = bi;
  }
  __threadfence();
  __syncwarp();
  if (lane == 0) {
    *P.pos = pos + 1;
    __threadfence();
    atomicExch(P.epoch, epoch + 1u);
  }
}

template <bool I8>
__device__ void finish_tile(const Prog& P, const Phase& f, int p, int tile, const Extra& ex, unsigned epoch,
                            int pos, int G, int lane) {
  const gemm::Params& gp = P.params[f.idx];
  const int B = gp.B;
  const int n0 = tile * kColTile;
  Header dq{};  // dequant scales for dev::dequant_pair
  if (I8)
    for (int b = 0; b < B; ++b) dq.xscale[b] = ex.xs[p & 1][b];
  for (int item = lane; item < B * (kColTile / 2); item += 32) {
    const int b = item / (kColTile / 2);
    const int cc = 2 * (item - b * (kColTile / 2));
    const int n = n0 + cc;
    float y0, y1;
    if constexpr (I8) {
      int* a = static_cast<int*>(P.acc) + (static_cast<size_t>(tile) * B + b) * kColTile + cc;
      const int2 v = __ldcg(reinterpret_cast<const int2*>(a));
      *reinterpret_cast<int2*>(a) = make_int2(0, 0);
      if (n >= gp.N) continue;
      gemm::dev::dequant_pair(gp, dq, b, n, v.x, v.y, y0, y1);
    } else {
      long long* a = static_cast<long long*>(P.acc) + (static_cast<size_t>(tile) * B + b) * kColTile + cc;
      const longlong2 v = __ldcg(reinterpret_cast<const longlong2*>(a));
      *reinterpret_cast<longlong2*>(a) = make_longlong2(0, 0);
      if (n >= gp.N) continue;
      y0 = static_cast<float>(static_cast<double>(v.x) * (1.0 / 4294967296.0));
      y1 = static_cast<float>(static_cast<double>(v.y) * (1.0 / 4294967296.0));
    }
    gemm::dev::epilogue_pair(gp, b, n, y0, y1, n + 1 < gp.N);
  }
  if (f.kind == K_LM) {  // per-tile greedy argmax over this tile's valid vocabulary columns
    __threadfence();
    __syncwarp();
    for (int b = 0; b < B; ++b) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int cc = lane; cc < kColTile; cc += 32) {
        const int n = n0 + cc;
        if (n >= P.lm_valid) break;
        const float v = __ldcg(P.logits + static_cast<size_t>(b) * P.logits_ld + n);
        if (v > bv) {
          bv = v;
          bi = n;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        P.am_val[tile * B + b] = bv;
        P.am_idx[tile * B + b] = bi;
      }
    }
  }
  __syncwarp();
  unsigned prev = 0;
  if (lane == 0) {
    P.tile_cnt[tile] = 0;
    prev = atom_add_acq_rel(P.done + p, 1u);
    trace_rec(P, blockIdx.x, p, 6);
  }
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (f.kind == K_LM && prev + 1u == (epoch + 1u) * f.target) finalize_step(P, epoch, pos, G, lane);
}

// Drains the unit queue in batches: one lane per queued unit issues its tile ticket, so the
// ticket round trips overlap; the unit that completes a tile runs the fused epilogue.  (The
// consumers fenced their reductions before queueing the unit.)
template <bool kInt8>
__device__ void sync_warp(const Prog& P, Extra& ex, unsigned epoch, int pos, int cta, int G, int lane) {
  int q = 0;
  uint32_t qph = 0;
  for (;;) {
    ptx::mbar_wait(&ex.ufull[q], qph);
    int n = 1;
    if (lane == 0) {
      int qq = q + 1;
      uint32_t pp = qph;
      if (qq == kUnitQueue) {
        qq = 0;
        pp ^= 1;
      }
      while (n < kUnitQueue && ptx::mbar_test_wait(&ex.ufull[qq], pp)) {
        ++n;
        if (++qq == kUnitQueue) {
          qq = 0;
          pp ^= 1;
        }
      }
    }
    n = __shfl_sync(0xffffffffu, n, 0);
    int my_p = -2, my_tile = 0;
    if (lane < n) {
      const int slot = (q + lane) % kUnitQueue;
      my_p = ex.ent_phase[slot];
      my_tile = ex.ent_tile[slot];
    }
    unsigned old = 0;
    // The queued units' reductions were observed through the unit mbarriers (acquire at CTA
    // scope); one GPU-scope fence here makes them visible before the relaxed tickets (cumulative
    // release), and the finisher fences again (acquire) before reading the accumulator.
    if (lane == 0) __threadfence();
    __syncwarp();
    if (lane < n && my_p >= 0) old = atomicAdd(reinterpret_cast<unsigned*>(P.tile_cnt + my_tile), 1u);
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < n; ++i) ptx::mbar_arrive(&ex.uempty[(q + i) % kUnitQueue]);
    for (int i = 0; i < n; ++i) {
      if (++q == kUnitQueue) {
        q = 0;
        qph ^= 1;
      }
    }
    bool terminal = false;
    for (int i = 0; i < n; ++i) {
      const int p = __shfl_sync(0xffffffffu, my_p, i);
      const int tile = __shfl_sync(0xffffffffu, my_tile, i);
      const unsigned o = __shfl_sync(0xffffffffu, old, i);
      if (p < 0) {
        terminal = true;
        continue;
      }
      const Phase& f = P.phases[p];
      if (lane == 0) trace_rec(P, cta, p, 4);
      if (o != static_cast<unsigned>(f.cpt - 1)) continue;
      if (lane == 0) trace_rec(P, cta, p, 5);
      __threadfence();
      if (f.kind == K_LM)
        finish_tile<false>(P, f, p, tile, ex, epoch, pos, G, lane);
      else
        finish_tile<kInt8>(P, f, p, tile, ex, epoch, pos, G, lane);
    }
    if (terminal) return;  // end of step
  }
}

// ------------------------------------------------------------------ consumers
struct RingPos {
  int s;
  uint32_t ph;
  int uq;
  uint32_t uph;
};

// Hand a finished unit (or the end-of-step marker, phase < 0) to the sync warp.
__device__ __forceinline__ void push_unit(Extra& ex, RingPos& rp, int phase, int tile, int cw, int lane) {
  __syncwarp();
  if (lane == 0) {
    ptx::mbar_wait(&ex.uempty[rp.uq], rp.uph ^ 1);
    if (cw == 0) {
      ex.ent_phase[rp.uq] = phase;
      ex.ent_tile[rp.uq] = tile;
    }
  }
  consumer_bar();  // entry written before any warp arrives
  if (lane == 0) ptx::mbar_arrive(&ex.ufull[rp.uq]);
  if (++rp.uq == kUnitQueue) {
    rp.uq = 0;
    rp.uph ^= 1;
  }
}

template <bool I8, int kNB8>
__device__ void gemm_phase(const Prog& P, const Phase& f, int p, unsigned epoch, int cta, Header& hd, Extra& ex,
                           uint8_t* ring, uint32_t* sx, RingPos& rp, int cw, int lane, int ctid) {
  auto peek = [&]() -> int {
    ptx::mbar_wait(&hd.full[rp.s], rp.ph);
    return ex.meta[rp.s];
  };
  int m = peek();
  if (m < 0 || (m >> 20) != p) return;  // this CTA claimed no unit of phase p
  if (ctid == 0) trace_rec(P, cta, p, 0);
  wait_phase(P, p - 1, epoch, ctid);
  if (ctid == 0) trace_rec(P, cta, p, 1);
  const gemm::Params& gp = P.params[f.idx];
  const int B = gp.B;
  if (gp.pro == gemm::PRO_LN)
    gemm::dev::ln_row_stats<I8>(gp, hd, ctid, cw, lane, false);
  else if (gp.pro == gemm::PRO_QUANT)
    gemm::dev::quant_row_scale(gp, hd, ctid, cw, lane);
  consumer_bar();
  if (I8 && ctid < B) ex.xs[p & 1][ctid] = hd.xscale[ctid];
  if (f.full_x) {
    gemm::dev::fill_x_slice<I8, 1>(gp, sx, hd, 0, f.spt * kRowsPerStage, ctid);
    consumer_bar();
  }
  using C = gemm::dev::Consumer<I8, kNB8>;
  C c;
  c.init(lane);
  while (m >= 0 && (m >> 20) == p) {
    const int u = m & 0xFFFFF;
    const int tile = unit_tile(f, u), chunk = unit_chunk(f, u);
    const int st0 = chunk * f.cs, nst = min(f.spt, st0 + f.cs) - st0;
    if (!f.full_x) {
      gemm::dev::fill_x_slice<I8, 1>(gp, sx, hd, st0 * kRowsPerStage, nst * kRowsPerStage, ctid);
      consumer_bar();
    }
    c.zero();
    c.run(ring, hd, P.stages, rp.s, rp.ph, nst, sx + (f.full_x ? st0 * kRowsPerStage : 0), gp.x_row_words, B, cw,
          lane);
    if (!f.full_x) consumer_bar();  // x slice is refilled for the next unit
    // partials -> tile accumulator (fire-and-forget integer reductions, order independent); the
    // sync warp fences them at GPU scope before the tile ticket

#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n = cw * gemm::kWarpCols + j * 16 + c.g + (e >= 2 ? 8 : 0);
          const int b = bt * 8 + 2 * c.t + (e & 1);
          if (b >= B) continue;
          const size_t off = (static_cast<size_t>(tile) * B + b) * kColTile + n;
          if constexpr (I8)
            red_add(static_cast<int*>(P.acc) + off, c.acc[j][bt][e]);
          else
            red_add(static_cast<long long*>(P.acc) + off, __float2ll_rn(c.acc[j][bt][e] * kFix));
        }
    push_unit(ex, rp, p, tile, cw, lane);
    m = peek();
  }
  if (ctid == 0) trace_rec(P, cta, p, 2);
}

template <int kTPP>
__device__ void attn_phase(const Prog& P, const Phase& f, int p, unsigned epoch, int pos, int cta, int G, Header& hd,
                           float* ascr, int ctid) {
  constexpr int PPR = ops::dev::kAttnThreads / kTPP;
  const ops::AttnParams& ap = P.attn[f.idx];
  const int C = P.attn_chunks;
  const int items = ap.B * ap.H * C;
  if (cta >= items) return;
  if (ctid == 0) trace_rec(P, cta, p, 0);
  wait_phase(P, p - 1, epoch, ctid);
  if (ctid == 0) trace_rec(P, cta, p, 1);
  const int d = ap.d;
  const int ctx = pos + 1;
  const int chunk = (ctx + C - 1) / C;
  float* co = ascr + PPR * d + 2 * PPR;
  float* cst = co + d;
  for (int item = cta; item < items; item += G) {
    const int bh = item / C, c = item - bh * C;
    const int b = bh / ap.H, head = bh - b * ap.H;
    const int j0 = c * chunk, j1 = min(ctx, j0 + chunk);
    ops::dev::attn_chunk<kTPP>(ap, b, head, j0, j1, ctid, ascr, [] { consumer_bar(); });
    float* dst = P.attn_ws + static_cast<size_t>(item) * (d + 2);
    for (int i = ctid; i < d; i += 128) dst[i] = co[i];
    if (ctid == 0) {
      dst[d] = cst[0];
      dst[d + 1] = cst[1];
    }
    consumer_bar();
    if (ctid == 0)
      hd.flag[0] = atom_add_acq_rel(reinterpret_cast<unsigned*>(P.attn_cnt + bh), 1u) == static_cast<unsigned>(C - 1);
    consumer_bar();
    if (!hd.flag[0]) continue;
    (void)ld_acquire(reinterpret_cast<unsigned*>(P.attn_cnt + bh));
    const float* base = P.attn_ws + static_cast<size_t>(bh) * C * (d + 2);
    float M = -INFINITY;
    for (int r = 0; r < C; ++r) M = fmaxf(M, __ldcg(base + r * (d + 2) + d));
    float Lsum = 0.f;
    for (int r = 0; r < C; ++r) {
      const float mr = __ldcg(base + r * (d + 2) + d);
      Lsum += mr == -INFINITY ? 0.f : __ldcg(base + r * (d + 2) + d + 1) * expf(mr - M);
    }
    const float inv = 1.0f / Lsum;
    for (int i = ctid; i < d; i += 128) {
      float acc = 0.f;
      for (int r = 0; r < C; ++r) {
        const float mr = __ldcg(base + r * (d + 2) + d);
        const float w = mr == -INFINITY ? 0.f : expf(mr - M);
        acc = fmaf(w, __ldcg(base + r * (d + 2) + i), acc);
      }
      ap.out[static_cast<size_t>(b) * ap.H * d + head * d + i] = __float2half_rn(acc * inv);
    }
    consumer_bar();
    if (ctid == 0) {
      P.attn_cnt[bh] = 0;
      red_release(P.done + p, 1u);
    }
  }
  if (ctid == 0) trace_rec(P, cta, p, 2);
}

__device__ void embed_phase(const Prog& P, int p, int pos, int cta, int ctid) {
  if (cta != 0) return;
  const ops::EmbedParams& e = P.embed;
  for (int b = 0; b < e.B; ++b) {
    int tok = pos < e.prompt_len ? e.prompt[static_cast<size_t>(b) * e.prompt_ld + pos] : e.next_tok[b];
    if (tok < 0 || tok >= e.V) tok = 0;
    if (ctid == 0 && pos < e.max_ctx) e.hist[static_cast<size_t>(b) * e.max_ctx + pos] = tok;
    const __half* row = e.wte + static_cast<size_t>(tok) * e.h;
    float* out = e.res + static_cast<size_t>(b) * e.h;
    if ((e.h & 7) == 0) {  // 16-byte loads, all in flight at once
#pragma unroll 4
      for (int k = 8 * ctid; k < e.h; k += 8 * 128) {
        const uint4 u = *reinterpret_cast<const uint4*>(row + k);
        const __half2* h = reinterpret_cast<const __half2*>(&u);
        const float2 a = __half22float2(h[0]), c = __half22float2(h[1]), d = __half22float2(h[2]),
                     f = __half22float2(h[3]);
        *reinterpret_cast<float4*>(out + k) = make_float4(a.x, a.y, c.x, c.y);
        *reinterpret_cast<float4*>(out + k + 4) = make_float4(d.x, d.y, f.x, f.y);
      }
    } else {
      for (int k = ctid; k < e.h; k += 128) out[k] = __half2float(row[k]);
    }
  }
  consumer_bar();
  if (ctid == 0) red_release(P.done + p, 1u);
}

template <bool kInt8, int kNB8, int kTPP>
__global__ void __launch_bounds__(kThreadsStep, 1) step_kernel(const __grid_constant__ Prog P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  Header& hd = *reinterpret_cast<Header*>(smem + P.stages * kStageBytes);
  Extra& ex = *reinterpret_cast<Extra*>(smem + P.stages * kStageBytes + sizeof(Header));
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + P.stages * kStageBytes + gemm::kHeaderBytes);
  float* ascr = reinterpret_cast<float*>(smem + P.stages * kStageBytes + gemm::kHeaderBytes + P.x_bytes_);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x, G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) {
      ptx::mbar_init(&hd.full[s], 1);
      ptx::mbar_init(&hd.empty[s], gemm::kConsumerWarps);
    }
    for (int q = 0; q < kUnitQueue; ++q) {
      ptx::mbar_init(&ex.ufull[q], gemm::kConsumerWarps);
      ptx::mbar_init(&ex.uempty[q], 1);
    }
    ptx::fence_mbar_init();
    hd.flag[1] = static_cast<int>(ld_acquire(P.epoch));
    hd.flag[2] = *P.pos;
    red_release(P.arrived, 1u);  // check in: (epoch, pos) of this step have been read
  }
  __syncthreads();
  const unsigned epoch = static_cast<unsigned>(hd.flag[1]);
  const int pos = hd.flag[2];
  if (warp == 0) {
    if (lane == 0) producer(P, ring, hd, ex, epoch, cta, G);
    return;
  }
  if (warp == gemm::kConsumerWarps + 1) {
    sync_warp<kInt8>(P, ex, epoch, pos, cta, G, lane);
    return;
  }
  const int cw = warp - 1, ctid = threadIdx.x - 32;
  RingPos rp{0, 0, 0, 0};
  for (int p = 0; p < P.n_phases; ++p) {
    const Phase& f = P.phases[p];
    switch (f.kind) {
      case K_EMBED: embed_phase(P, p, pos, cta, ctid); break;
      case K_GEMM: gemm_phase<kInt8, kNB8>(P, f, p, epoch, cta, hd, ex, ring, sx, rp, cw, lane, ctid); break;
      case K_LM: gemm_phase<false, kNB8>(P, f, p, epoch, cta, hd, ex, ring, sx, rp, cw, lane, ctid); break;
      case K_ATTN: attn_phase<kTPP>(P, f, p, epoch, pos, cta, G, hd, ascr, ctid); break;
      default: break;
    }
  }
  push_unit(ex, rp, -1, 0, cw, lane);  // release the sync warp
}

using KernelFn = void (*)(Prog);

KernelFn pick(int variant) {
  // variant = int8 * 6 + (nb8 - 1) * 3 + tpp index (8, 16, 32)
  static const KernelFn table[12] = {
      step_kernel<false, 1, 8>, step_kernel<false, 1, 16>, step_kernel<false, 1, 32>,
      step_kernel<false, 2, 8>, step_kernel<false, 2, 16>, step_kernel<false, 2, 32>,
      step_kernel<true, 1, 8>,  step_kernel<true, 1, 16>,  step_kernel<true, 1, 32>,
      step_kernel<true, 2, 8>,  step_kernel<true, 2, 16>,  step_kernel<true, 2, 32>};
  return table[variant];
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

}  // namespace

struct StepProgram::ProgHost {
  Prog prog;
};

void StepProgram::release() {
  for (void* p : allocs_) cudaFree(p);
  allocs_.clear();
  built_ = false;
}

size_t StepProgram::trace(unsigned long long* host, size_t len) const {
  if (!trace_ptr_) return 0;
  const size_t n = std::min(len, trace_len_);
  if (host && n) DSINF_CUDA_CHECK(cudaMemcpy(host, trace_ptr_, n * 8, cudaMemcpyDeviceToHost));
  return trace_len_;
}

void StepProgram::build(const StepDesc& D) {
  release();
  require(D.B >= 1 && D.B <= gemm::kMaxB, "step kernel: batch must be 1..16");
  require(D.d % 8 == 0 && D.d <= 256, "step kernel: head dim must be a multiple of 8 and <= 256");
  require(static_cast<int>(D.gemms.size()) == 4 * D.L + 1, "step kernel: expected 4 GEMMs per layer + LM head");
  require(static_cast<int>(D.attn.size()) == D.L, "step kernel: one attention descriptor per layer");
  const int tpp = D.d <= 64 ? 8 : (D.d <= 128 ? 16 : 32);
  const int tpp_idx = tpp == 8 ? 0 : (tpp == 16 ? 1 : 2);
  const int nb8 = D.B <= 8 ? 1 : 2;
  variant_ = (D.int8 ? 6 : 0) + (nb8 - 1) * 3 + tpp_idx;
  const int stages = std::max(2, std::min(gemm::kMaxStages, env_int("DSINF_STEP_STAGES", 4)));
  const int lookahead = std::max(1, std::min(kMaxLookahead, env_int("DSINF_STEP_LA", 2)));
  const size_t x_budget = static_cast<size_t>(env_int("DSINF_STEP_XKB", 36)) * 1024;
  const int cs = std::max(1, env_int("DSINF_STEP_CS", 4));

  // ---- phases
  std::vector<Phase> phases;
  std::vector<gemm::Params> params = D.gemms;
  size_t x_words_max = 0;
  int max_tiles = 1, lm_tiles = 0;
  auto add_gemm = [&](int idx, int kind) {
    gemm::Params& gp = params[idx];
    require(gp.N % 4 == 0, "step kernel: out_dim must be a multiple of 4");
    Phase f{};
    f.kind = kind;
    f.idx = idx;
    f.tiles = (gp.N + kColTile - 1) / kColTile;
    f.spt = (gp.rows + kRowsPerStage - 1) / kRowsPerStage;
    f.cs = std::min(cs, f.spt);
    f.cpt = (f.spt + f.cs - 1) / f.cs;
    f.units = f.tiles * f.cpt;
    require(f.units < (1 << 20), "step kernel: too many units in one phase");
    f.target = static_cast<unsigned>(f.tiles);
    f.chunk_major = env_int("DSINF_STEP_ORDER", 1);
    const size_t full_words = static_cast<size_t>(f.spt) * kRowsPerStage + 8;  // row stride == 8 mod 32
    f.full_x = static_cast<size_t>(D.B) * full_words * 4 <= x_budget;
    gp.x_row_words = static_cast<int>(f.full_x ? full_words : static_cast<size_t>(f.cs) * kRowsPerStage + 8);
    gp.stages = stages;
    gp.rows_per_split = 0;
    x_words_max = std::max(x_words_max, static_cast<size_t>(D.B) * gp.x_row_words);
    max_tiles = std::max(max_tiles, f.tiles);
    if (kind == K_LM) lm_tiles = f.tiles;
    phases.push_back(f);
  };
  {
    Phase e{};
    e.kind = K_EMBED;
    e.target = 1;
    phases.push_back(e);
  }
  int sms = 0, dev = 0;
  DSINF_CUDA_CHECK(cudaGetDevice(&dev));
  DSINF_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int cps_req = std::max(1, env_int("DSINF_STEP_CPS", 2));
  const int C = std::max(1, std::min(8, (sms * cps_req) / std::max(1, D.B * D.H)));
  for (int l = 0; l < D.L; ++l) {
    add_gemm(4 * l + 0, K_GEMM);
    Phase a{};
    a.kind = K_ATTN;
    a.idx = l;
    a.target = static_cast<unsigned>(D.B * D.H);
    phases.push_back(a);
    add_gemm(4 * l + 1, K_GEMM);
    add_gemm(4 * l + 2, K_GEMM);
    add_gemm(4 * l + 3, K_GEMM);
  }
  add_gemm(4 * D.L, K_LM);

  // ---- launch geometry
  const size_t x_bytes = (x_words_max * 4 + 127) / 128 * 128;
  const size_t attn_floats = static_cast<size_t>(128 / tpp) * D.d + 2 * (128 / tpp) + D.d + 4;
  smem_ = 1024 + static_cast<size_t>(stages) * kStageBytes + gemm::kHeaderBytes + x_bytes + attn_floats * 4;
  KernelFn kern = pick(variant_);
  DSINF_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
  int per_sm = 0;
  DSINF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(kern),
                                                                 kThreadsStep, smem_));
  require(per_sm >= 1, "step kernel: does not fit on an SM");
  const int G = sms * std::min(per_sm, cps_req);
  grid_ = G;

  // ---- device buffers
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    DSINF_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    allocs_.push_back(p);
    return p;
  };
  auto upload = [&](const void* src, size_t bytes) {
    void* p = dalloc(bytes);
    DSINF_CUDA_CHECK(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
    return p;
  };
  auto zeros = [&](size_t bytes) {
    void* p = dalloc(bytes);
    DSINF_CUDA_CHECK(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
    return p;
  };
  Prog P{};
  P.phases = static_cast<const Phase*>(upload(phases.data(), phases.size() * sizeof(Phase)));
  P.n_phases = static_cast<int>(phases.size());
  P.params = static_cast<const gemm::Params*>(upload(params.data(), params.size() * sizeof(gemm::Params)));
  P.attn = static_cast<const ops::AttnParams*>(upload(D.attn.data(), D.attn.size() * sizeof(ops::AttnParams)));
  P.attn_chunks = C;
  P.embed = D.embed;
  P.acc = zeros(static_cast<size_t>(max_tiles) * D.B * kColTile * 8);  // int64 (fp16) or int32 (int8)
  P.attn_ws = static_cast<float*>(dalloc(static_cast<size_t>(D.B) * D.H * C * (D.d + 2) * 4));
  P.tile_cnt = static_cast<int*>(zeros(static_cast<size_t>(max_tiles) * 4));
  P.attn_cnt = static_cast<int*>(zeros(static_cast<size_t>(D.B) * D.H * 4));
  P.claim = static_cast<unsigned*>(zeros(phases.size() * 4));
  P.done = static_cast<unsigned*>(zeros(phases.size() * 4));
  P.arrived = static_cast<unsigned*>(zeros(4));
  P.epoch = static_cast<unsigned*>(zeros(4));
  P.am_val = static_cast<float*>(dalloc(static_cast<size_t>(lm_tiles) * D.B * 4));
  P.am_idx = static_cast<int*>(dalloc(static_cast<size_t>(lm_tiles) * D.B * 4));
  P.lm_tiles = lm_tiles;
  P.lm_valid = D.V;
  P.logits = D.logits;
  P.logits_ld = D.Vl;
  P.next_tok = D.next_tok;
  P.hist = D.hist;
  P.pos = D.pos;
  P.max_ctx = D.max_ctx;
  P.B = D.B;
  P.stages = stages;
  P.lookahead = lookahead;
  P.x_bytes_ = x_bytes;
  P.trace = nullptr;
  trace_len_ = 0;
  if (env_int("DSINF_STEP_TRACE", 0)) {
    trace_len_ = static_cast<size_t>(G) * phases.size() * 8;
    P.trace = static_cast<unsigned long long*>(zeros(trace_len_ * 8));
  }
  trace_ptr_ = P.trace;
  n_phases_ = static_cast<int>(phases.size());
  prog_host_.resize(sizeof(Prog));
  std::memcpy(prog_host_.data(), &P, sizeof(Prog));
  built_ = true;
}

void StepProgram::set_embed(const ops::EmbedParams& e) {
  require(built_, "step kernel not built");
  Prog P;
  std::memcpy(&P, prog_host_.data(), sizeof(Prog));
  P.embed = e;
  std::memcpy(prog_host_.data(), &P, sizeof(Prog));
}

void StepProgram::launch(cudaStream_t s) const {
  require(built_, "step kernel not built");
  Prog P;
  std::memcpy(&P, prog_host_.data(), sizeof(Prog));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_);
  cfg.blockDim = dim3(kThreadsStep);
  cfg.dynamicSmemBytes = smem_;
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (phase waits span CTAs)
  attr.val.cooperative = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, pick(variant_), P));
}

}  // namespace step
}  // namespace dsinf
