// Persistent decode-step kernel (PAPER.md:1004-1006 taken to its limit): ONE
// launch per decode step runs the embedding, every layer's Deep-Fusion regions
// and the LM head + greedy argmax, tensor-parallel degree 1, fp16 or INT8 weight-only (W8A16)
// weights in the reference packed layout (gemm.hpp:108-111).
//
// Static schedule.  The 16 KB weight stages (128 output columns x 32 packed rows) of every GEMM
// phase are numbered in (column tile, k) order and cut into G equal contiguous ranges, one per CTA
// (rotated per phase so the +1 remainders move around the grid).  One CTA per SM:
//   warp 0      producer: streams the CTA's stages of ALL phases, in program order, through a deep
//               TMA ring.  Weights never depend on activations, so it only ever waits for a free
//               ring slot: HBM keeps streaming while the consumers wait for a dependency, and the
//               ring (up to ~200 KB per SM, ~4 us of HBM time over the grid) absorbs the wait.
//   warps 1..4  consumers: per segment (the part of the CTA's range inside one column tile) wait
//               for exactly the data they read, build the x slice in shared memory (LayerNorm from
//               the producer's fixed-point row sums, or plain fp16 loads), run the warp MMAs over
//               the ring and push the partial sums into the tile accumulator with integer
//               reductions (2^-32 fixed point: order-independent, so the step is deterministic).
//   warp 5      epilogue warp: per segment a tile ticket; the segment that completes a tile runs
//               the fused epilogue (bias, RoPE + KV-cache append, GeLU, residual add + the next
//               LayerNorm's row sums, LM-head logits + greedy argmax key) and publishes the tile.
// Dependencies are as fine as the math allows: decode attention of (row, head) waits for that
// head's q/k/v tiles; an attn-out segment for the attention outputs of the heads in its K range;
// an MLP-down segment for the MLP-up tiles of its K range.  Only the LayerNorm consumers (QKV,
// MLP-up, LM head) wait for a whole phase: the row statistics need the complete row.
#include <algorithm>
#include <cfloat>
#include <cmath>
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
using gemm::kConsumerWarps;
using gemm::kRowsPerStage;
using gemm::kStageBytes;
using gemm::dev::consumer_bar;
using gemm::dev::Header;

enum Kind : int { K_EMBED = 0, K_GEMM = 1, K_ATTN = 2, K_LM = 3 };
enum Dep : int { DEP_NONE = 0, DEP_FULL = 1, DEP_HEADS = 2, DEP_TILES = 3 };
enum AccKind : int { ACC_QKV = 0, ACC_O = 1, ACC_UP = 2, ACC_DOWN = 3, ACC_LM = 4, kAccKinds = 5 };
constexpr int kUnitQueue = 16;
// Consumer warp groups: 4 warps (one 128-column tile) each; group g consumes the ring slots
// s = g mod kGroups.  One group of 4 warps cannot hide the per-warp latency of the W8A16 / fp16
// MMA loop (~0.7 us per 16 KB stage, ~20 GB/s per SM); interleaved groups double it.
constexpr int kGroups = 1;
constexpr int kConsumerThreads = 128 * kGroups;
constexpr int kThreadsStep = 32 * (2 + kConsumerWarps * kGroups);
constexpr int kEpilogueWarp = 1 + kConsumerWarps * kGroups;

// All consumer threads of every group (named barrier 2; barrier 1 = group 0's 128 threads, used by
// the shared prologue helpers).
__device__ __forceinline__ void all_bar() { asm volatile("bar.sync 2, %0;" ::"n"(kConsumerThreads) : "memory"); }
constexpr float kFix = 4294967296.0f;  // 2^32: fixed-point scale of the partial sums
constexpr double kFixInv = 1.0 / 4294967296.0;

struct Phase {
  int kind;
  int idx;        // GEMM params index / layer (attention)
  int tiles;      // 128-column tiles
  int spt;        // 32-row stages per tile
  int total;      // tiles * spt
  int rot;        // range rotation
  int xw;         // x words per packed weight row: 1 (fp16 weights), 2 (W8A16)
  int kpr;        // k per packed weight row: 2 (fp16), 4 (int8)
  int dep;        // Dep
  int dep_phase;  // phase waited on
  int dep_base;   // DEP_HEADS: first head counter; DEP_TILES: first tile flag of dep_phase
  unsigned dep_target;  // DEP_FULL: done[dep_phase] increments per step
  unsigned target;      // done[this] increments per step
  int tile_base;        // first entry of nseg / tile_cnt / tile_flag
  int acc;              // AccKind
};

struct Prog {
  const Phase* phases;
  int n_phases;
  const gemm::Params* params;
  const ops::AttnParams* attn;
  int attn_chunks;
  ops::EmbedParams embed;
  long long* acc[kAccKinds];  // [tiles][B][128] fixed point, zero between uses
  const int* nseg;            // per global tile: CTA segments contributing to it
  unsigned* tile_cnt;         // per global tile: tickets (monotonic)
  unsigned* tile_flag;        // per global tile: epoch + 1 once published
  unsigned* done;             // per phase (monotonic)
  unsigned* head_cnt;         // [L][H]: (row, head) attention outputs published (monotonic)
  float* attn_ws;             // chunk partials [B * H * C][d + 2]
  unsigned* arrived;
  unsigned* epoch;
  unsigned long long* am_key;  // [B] greedy-argmax keys (zeroed per step by the graph)
  int lm_valid;
  int32_t* next_tok;
  int32_t* hist;
  int* pos;
  int max_ctx;
  int B, H, d, stages;
  int nomma;     // timing experiment: consumers only drain the ring
  int inflight;  // producer in-flight cap (stages; 0 = ring depth)
  int l2_ahead;  // stages warmed into L2 beyond the ring while the ring is full
  int xrw;    // x slice row stride (words, == 8 mod 32)
  int x_cap;  // x words per row per chunk (multiple of 64)
  int x_bytes;  // x slice region (the attention merge weights follow it)
  unsigned long long* trace;  // optional [G][n_phases][8] globaltimer stamps (DSINF_STEP_TRACE)
};

// Per-CTA bookkeeping shared between the warp roles (in the 1 KB header region after Header).
struct Extra {
  uint64_t ufull[kUnitQueue];
  uint64_t uempty[kUnitQueue];
  int ent_phase[kUnitQueue];
  int ent_tile[kUnitQueue];
  long long red64[2 * kConsumerWarps];
  int flag[4];
};
static_assert(sizeof(Header) + sizeof(Extra) <= gemm::kHeaderBytes, "header region too small");

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// slot: 0 consumer reaches the phase, 1 dependency satisfied, 2 consumer done, 3 producer issued the
//       phase, 4 epilogue warp took a unit of the phase, 5 first x slice built, 6 a tile of the phase published
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
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool reached(unsigned v, unsigned target) { return static_cast<int>(v - target) >= 0; }

// First stage of virtual CTA v's range of a phase with `total` stages.
__host__ __device__ __forceinline__ int range_start(int total, int v, int G) {
  return static_cast<int>((static_cast<long long>(total) * v) / G);
}

// All 128 consumer threads: wait until counter(i) >= target(i) for every i < n (thread i polls
// counter i), then a consumer barrier.  The pollers' acquire loads + the barrier order every later
// read of the published data after its publication.
__device__ int g_step_nodep;  // timing experiment (DSINF_STEP_NODEP): dependency waits skipped

template <class F>
__device__ __forceinline__ void wait_all(int n, int ctid, F counter) {
  if (g_step_nodep) {
    consumer_bar();
    return;
  }
  for (int i = ctid; i < n; i += 128) {
    const unsigned* c;
    unsigned t;
    counter(i, c, t);
    if (!reached(ld_acquire(c), t)) {
      while (!reached(ld_relaxed(c), t)) __nanosleep(32);
      (void)ld_acquire(c);
    }
  }
  consumer_bar();
}

// ------------------------------------------------------------------ producer (one thread)
// Walks the CTA's stages of every GEMM phase in program order with phase fields in registers and
// no divisions in the per-stage path (one producer thread per SM must issue ~45 GB/s of stages).
struct StageWalk {
  int p = -1, i = 0, e = 0, st = 0, spt = 1, c0 = 0;
  const CUtensorMap* map = nullptr;
  __device__ __forceinline__ bool next(const Prog& P, int cta, int G) {
    if (i >= e) {
      for (;;) {
        if (++p >= P.n_phases) return false;
        const Phase& f = P.phases[p];
        if (f.kind != K_GEMM && f.kind != K_LM) continue;
        const int v = (cta + f.rot) % G;
        i = range_start(f.total, v, G);
        e = range_start(f.total, v + 1, G);
        if (i >= e) continue;
        spt = f.spt;
        const int tile = i / spt;
        st = i - tile * spt;
        c0 = tile * kColTile;
        map = &P.params[f.idx].tmap;
        break;
      }
    } else if (++st == spt) {
      st = 0;
      c0 += kColTile;
    }
    ++i;
    return true;
  }
};

// Ring loads; while the ring is full (the consumers wait for a dependency) the producer warms up
// to P.l2_ahead further stages into L2 (cp.async.bulk.prefetch.tensor), so HBM keeps streaming
// through the wait and the ring refills from L2 afterwards.
__device__ void producer(const Prog& P, uint8_t* ring, Header& hd, int cta, int G) {
  const uint64_t pol = ptx::policy_evict_first();
  const int S = P.stages;
  int s = 0;
  uint32_t ph = 0;
  int it = 0;
  StageWalk ld, pf;
  int pf_it = 0;  // stages the prefetch walk has passed (prefetched beyond the first S)
  bool pf_more = P.l2_ahead > 0;
  int last_p = -1;
  while (ld.next(P, cta, G)) {
    if (ld.p != last_p) {
      if (last_p >= 0) trace_rec(P, cta, last_p, 3);
      last_p = ld.p;
    }
    // in-flight cap: stage it - inflight must have landed before stage it is issued, so at most
    // `inflight` stages per SM sit in the memory system's queues (the ring still buffers up to S
    // landed stages); dependent loads of the consumers then queue behind ~inflight x 148 x 16 KB
    // instead of S x 148 x 16 KB
    if (P.inflight > 0 && it >= P.inflight) {
      const int j = it - P.inflight;
      const int sj = j % S;
      const uint32_t pj = static_cast<uint32_t>((j / S) & 1);
      while (!ptx::mbar_test_wait(&hd.full[sj], pj)) {
      }
    }
    if (it >= S) {
      while (!ptx::mbar_test_wait(&hd.empty[s], ph ^ 1)) {
        if (pf_more && pf_it < it + S + P.l2_ahead) {
          if (!pf.next(P, cta, G)) {
            pf_more = false;
          } else if (pf_it++ >= it + S) {  // beyond what the ring will hold
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w)
              ptx::tma_prefetch_l2_2d(pf.map, pf.c0 + w * gemm::kWarpCols, pf.st * kRowsPerStage);
          }
        }
      }
    }
    ptx::mbar_arrive_expect_tx(&hd.full[s], kStageBytes);
    uint8_t* dst = ring + s * kStageBytes;
    const int r0 = ld.st * kRowsPerStage;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w)
      ptx::tma_load_2d(dst + w * gemm::kBoxBytes, ld.map, ld.c0 + w * gemm::kWarpCols, r0, &hd.full[s], pol);
    ++it;
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }
  if (last_p >= 0) trace_rec(P, cta, last_p, 3);
}

// ------------------------------------------------------------------ epilogue warp
// End of the step (the warp that published the last LM-head tile): greedy tokens from the argmax
// keys, history, next position, epoch.
__device__ void finalize_step(const Prog& P, int p, unsigned epoch, int pos, int G, int lane) {
  if (lane == 0)
    while (!reached(ld_relaxed(P.arrived), (epoch + 1u) * static_cast<unsigned>(G))) __nanosleep(64);
  __syncwarp();
  (void)ld_acquire(P.arrived);
  (void)ld_acquire(P.done + p);
  for (int b = lane; b < P.B; b += 32) {
    const int tok = gemm::argmax_key_index(__ldcg(P.am_key + b));
    P.next_tok[b] = tok;
    if (pos + 1 < P.max_ctx) P.hist[static_cast<size_t>(b) * P.max_ctx + pos + 1] = tok;
  }
  __syncwarp();
  if (lane == 0) {
    fence_acq_rel();
    *P.pos = pos + 1;
    fence_acq_rel();
    atomicExch(P.epoch, epoch + 1u);
  }
}

// The segment that completed `tile` of phase p: reduce (read + re-zero the accumulator), fused
// epilogue, publish.  One warp; lane l owns column pairs l and l + 32 of the tile.  Rows go in
// batches of kFinRows whose loads are all issued before any is used (the finish of the last tile
// of a phase is on the dependency critical path: its latency is a few L2 round trips, not B).
constexpr int kFinRows = 2;

// Per-column epilogue operands of one lane (column pairs lane and lane + 32 of the tile): loaded
// by the epilogue warp while its tile ticket is in flight.
struct ColOps {
  int n[2];
  bool ok[2], has1[2];
  float2 bias[2], ws[2], cs[2];
  int sec[2], head[2], dim[2], rem[2];
  __device__ __forceinline__ void load(const gemm::Params& gp, int tile, int pos, int lane) {
    const int hdq = gp.heads * gp.head_dim;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      n[hh] = tile * kColTile + 2 * (lane + 32 * hh);
      ok[hh] = n[hh] < gp.N;
      has1[hh] = n[hh] + 1 < gp.N;
      bias[hh] = make_float2(0.f, 0.f);
      ws[hh] = make_float2(1.f, 1.f);
      cs[hh] = make_float2(1.f, 0.f);
      sec[hh] = head[hh] = dim[hh] = rem[hh] = 0;
      if (!ok[hh]) continue;
      if (gp.bias) {
        bias[hh].x = __half2float(gp.bias[n[hh]]);
        if (has1[hh]) bias[hh].y = __half2float(gp.bias[n[hh] + 1]);
      }
      if (gp.a16) {
        ws[hh].x = gp.w_scale[n[hh]];
        if (has1[hh]) ws[hh].y = gp.w_scale[n[hh] + 1];
      }
      if (gp.epi == gemm::EPI_QKV) {
        sec[hh] = n[hh] / hdq;
        rem[hh] = n[hh] - sec[hh] * hdq;
        head[hh] = rem[hh] / gp.head_dim;
        dim[hh] = rem[hh] - head[hh] * gp.head_dim;
        if (sec[hh] < 2) cs[hh] = gp.rope[static_cast<size_t>(pos) * (gp.head_dim / 2) + dim[hh] / 2];
      }
    }
  }
};

__device__ void finish_tile(const Prog& P, const Phase& f, int p, int tile, const ColOps& co, unsigned epoch,
                            int pos, int G, int lane) {
  const gemm::Params& gp = P.params[f.idx];
  const int B = gp.B;
  long long* acc = P.acc[f.acc] + static_cast<size_t>(tile) * B * kColTile;
  const bool lm = f.kind == K_LM;
  const int epi = gp.epi;
  const int hdq = gp.heads * gp.head_dim;
  const int* n = co.n;
  const bool* ok = co.ok;
  const bool* has1 = co.has1;
  const float2* bias = co.bias;
  const float2* ws = co.ws;
  const float2* cs = co.cs;
  const int* sec = co.sec;
  const int* head = co.head;
  const int* dim = co.dim;
  const int* rem = co.rem;
  for (int b0 = 0; b0 < B; b0 += kFinRows) {
    longlong2 v[kFinRows][2];
    float2 rin[kFinRows][2];
#pragma unroll
    for (int r = 0; r < kFinRows; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        v[r][hh] = make_longlong2(0, 0);
        rin[r][hh] = make_float2(0.f, 0.f);
        const int b = b0 + r;
        if (b >= B) continue;
        long long* a = acc + static_cast<size_t>(b) * kColTile + 2 * (lane + 32 * hh);
        v[r][hh] = __ldcg(reinterpret_cast<const longlong2*>(a));
        if (epi == gemm::EPI_RESID && ok[hh])
          rin[r][hh] = __ldcg(reinterpret_cast<const float2*>(static_cast<const float*>(gp.out) +
                                                              static_cast<size_t>(b) * gp.out_ld + n[hh]));
      }
#pragma unroll
    for (int r = 0; r < kFinRows; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        if (b0 + r < B)
          *reinterpret_cast<longlong2*>(acc + static_cast<size_t>(b0 + r) * kColTile + 2 * (lane + 32 * hh)) =
              make_longlong2(0, 0);
#pragma unroll
    for (int r = 0; r < kFinRows; ++r) {
      const int b = b0 + r;
      if (b >= B) break;
      gemm::dev::RowStat st;
      unsigned long long key = 0ull;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (!ok[hh]) continue;
        float y0 = static_cast<float>(static_cast<double>(v[r][hh].x) * kFixInv);
        float y1 = has1[hh] ? static_cast<float>(static_cast<double>(v[r][hh].y) * kFixInv) : 0.f;
        if (gp.a16) {  // W8A16: y = acc * w_scale (the standalone kernel's dequant)
          y0 = __fmul_rn(y0, ws[hh].x);
          if (has1[hh]) y1 = __fmul_rn(y1, ws[hh].y);
        }
        if (gp.bias) {
          y0 = __fadd_rn(y0, bias[hh].x);
          if (has1[hh]) y1 = __fadd_rn(y1, bias[hh].y);
        }
        const int nc = n[hh];
        switch (epi) {
          case gemm::EPI_RESID: {  // residual += y + bias; the next LayerNorm's row sums
            float* o = static_cast<float*>(gp.out) + static_cast<size_t>(b) * gp.out_ld + nc;
            const float r0 = __fadd_rn(rin[r][hh].x, y0), r1 = __fadd_rn(rin[r][hh].y, y1);
            if (has1[hh]) {
              *reinterpret_cast<float2*>(o) = make_float2(r0, r1);
            } else {
              o[0] = r0;
            }
            st.add(r0);
            if (has1[hh]) st.add(r1);
            break;
          }
          case gemm::EPI_GELU_F16: {
            __half* o = static_cast<__half*>(gp.out) + static_cast<size_t>(b) * gp.out_ld + nc;
            const __half h0 = __float2half_rn(gemm::dev::gelu_tanh(y0)), h1 = __float2half_rn(gemm::dev::gelu_tanh(y1));
            if (has1[hh]) {
              *reinterpret_cast<__half2*>(o) = __halves2half2(h0, h1);
            } else {
              o[0] = h0;
            }
            break;
          }
          case gemm::EPI_QKV: {
            if (sec[hh] < 2) {  // GPT-J interleaved rotary embedding (as gemm::dev::epilogue_pair)
              const float a0 = __fsub_rn(__fmul_rn(y0, cs[hh].x), __fmul_rn(y1, cs[hh].y));
              const float a1 = __fadd_rn(__fmul_rn(y0, cs[hh].y), __fmul_rn(y1, cs[hh].x));
              y0 = a0;
              y1 = a1;
            }
            const __half2 hv = __floats2half2_rn(y0, y1);
            if (sec[hh] == 0) {
              *reinterpret_cast<__half2*>(gp.q_out + static_cast<size_t>(b) * hdq + rem[hh]) = hv;
            } else {
              __half* cache = sec[hh] == 1 ? gp.k_cache : gp.v_cache;
              const size_t off =
                  ((static_cast<size_t>(b) * gp.heads + head[hh]) * gp.max_seq + pos) * gp.head_dim + dim[hh];
              *reinterpret_cast<__half2*>(cache + off) = hv;
            }
            break;
          }
          default: {  // EPI_F32 (LM head logits) + greedy argmax key
            float* o = static_cast<float*>(gp.out) + static_cast<size_t>(b) * gp.out_ld + nc;
            if (has1[hh]) {
              *reinterpret_cast<float2*>(o) = make_float2(y0, y1);
            } else {
              o[0] = y0;
            }
            if (lm) {
              if (nc < P.lm_valid) key = max(key, gemm::argmax_key(y0, nc));
              if (has1[hh] && nc + 1 < P.lm_valid) key = max(key, gemm::argmax_key(y1, nc + 1));
            }
            break;
          }
        }
      }
      if (epi == gemm::EPI_RESID && gp.ln_stats_out != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          st.s1 += __shfl_xor_sync(0xffffffffu, st.s1, o);
          st.s2 += __shfl_xor_sync(0xffffffffu, st.s2, o);
        }
        if (lane == 0) {
          unsigned long long* dst = reinterpret_cast<unsigned long long*>(gp.ln_stats_out) +
                                    ((tile & (gemm::kStatStripes - 1)) * gemm::kMaxB + b) * 2;
          atomicAdd(dst, static_cast<unsigned long long>(st.s1));
          atomicAdd(dst + 1, static_cast<unsigned long long>(st.s2));
        }
      }
      if (lm) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
        if (lane == 0 && key != 0ull) atomicMax(P.am_key + b, key);
      }
    }
  }
  __syncwarp();  // the warp's epilogue stores before lane 0's (cumulative) release
  unsigned prev = 0;
  if (lane == 0) {
    st_release(P.tile_flag + f.tile_base + tile, epoch + 1u);
    if (lm)
      prev = atom_add_acq_rel(P.done + p, 1u);
    else
      red_release(P.done + p, 1u);
    trace_rec(P, blockIdx.x, p, 6);
  }
  if (!lm) return;
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev + 1u == (epoch + 1u) * f.target) finalize_step(P, p, epoch, pos, G, lane);
}

__device__ void epilogue_warp(const Prog& P, Extra& ex, unsigned epoch, int pos, int cta, int G, int lane) {
  int q = 0;
  uint32_t qph = 0;
  for (;;) {
    ptx::mbar_wait(&ex.ufull[q], qph);
    const int p = ex.ent_phase[q], tile = ex.ent_tile[q];
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&ex.uempty[q]);
    if (++q == kUnitQueue) {
      q = 0;
      qph ^= 1;
    }
    if (p < 0) return;  // end of step
    const Phase& f = P.phases[p];
    const int gt = f.tile_base + tile;
    unsigned old = 0;
    if (lane == 0) {
      // the consumers' reductions were observed through the unit mbarrier (CTA scope); the
      // acq_rel ticket releases them at GPU scope (cumulativity) and acquires the other segments'
      old = atom_add_acq_rel(P.tile_cnt + gt, 1u);
    }
    ColOps co;  // independent of the ticket: in flight with it
    co.load(P.params[f.idx], tile, pos, lane);
    const unsigned ns = static_cast<unsigned>(__ldg(P.nseg + gt));
    old = __shfl_sync(0xffffffffu, old, 0);
    if (lane == 0) trace_rec(P, cta, p, 4);
    if ((old + 1u) % ns != 0u) continue;
    __syncwarp();
    finish_tile(P, f, p, tile, co, epoch, pos, G, lane);
  }
}

// ------------------------------------------------------------------ consumers
struct RingPos {
  int s;         // this group's next ring slot
  uint32_t ph;
  int uq;
  uint32_t uph;
  int gidx;      // stages of the CTA consumed so far (all groups; its parity picks the group)
};

// Hand a finished segment (or the end-of-step marker, phase < 0) to the epilogue warp (every
// consumer warp of every group arrives: the unit's reductions of both groups precede).
__device__ __forceinline__ void push_unit(Extra& ex, RingPos& rp, int phase, int tile, int grp, int cw, int lane) {
  __syncwarp();
  if (lane == 0) {
    ptx::mbar_wait(&ex.uempty[rp.uq], rp.uph ^ 1);
    if (cw == 0 && grp == 0) {
      ex.ent_phase[rp.uq] = phase;
      ex.ent_tile[rp.uq] = tile;
    }
  }
  all_bar();  // entry written before any warp arrives
  if (lane == 0) ptx::mbar_arrive(&ex.ufull[rp.uq]);
  if (++rp.uq == kUnitQueue) {
    rp.uq = 0;
    rp.uph ^= 1;
  }
}

__device__ void fill_x_attn(const Prog& P, const gemm::Params& gp, uint32_t* sx, float* mw, int row0, int nrows,
                            int ctid);
template <int kR = 8>
__device__ void fill_x_ln_fast(const gemm::Params& gp, uint32_t* sx, Header& hd, int row0, int nrows, int xrw,
                               int ctid);
template <int kR = 8>
__device__ void fill_x_f16_fast(const gemm::Params& gp, uint32_t* sx, int row0, int nrows, int xrw, int ctid);

template <bool kA16, int kNB8>
__device__ void gemm_phase(const Prog& P, const Phase& f, int p, unsigned epoch, int cta, int G, Header& hd,
                           Extra& ex, uint8_t* ring, uint32_t* sx, float* mw, RingPos& rp, int grp, int cw, int lane,
                           int ctid) {
  const int v = (cta + f.rot) % G;
  const int a = range_start(f.total, v, G), e = range_start(f.total, v + 1, G);
  if (a >= e) return;
  const bool lead = grp == 0 && ctid == 0;
  if (lead) trace_rec(P, cta, p, 0);
  // this group's share of a run of n ring stages starting at CTA stage index gidx
  auto my_first = [&](int gidx) { return (grp - gidx) & (kGroups - 1); };
  auto my_count = [&](int gidx, int n) { const int j0 = my_first(gidx); return n > j0 ? (n - j0 + kGroups - 1) / kGroups : 0; };
  if (P.nomma) {  // DSINF_STEP_NOMMA: pure weight streaming of the schedule (timing experiment)
    const int cnt = my_count(rp.gidx, e - a);
    for (int i = 0; i < cnt; ++i) {
      ptx::mbar_wait(&hd.full[rp.s], rp.ph);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&hd.empty[rp.s]);
      if ((rp.s += kGroups) >= P.stages) {
        rp.s -= P.stages;
        rp.ph ^= 1;
      }
    }
    rp.gidx += e - a;
    if (lead) trace_rec(P, cta, p, 2);
    return;
  }
  const gemm::Params& gp = P.params[f.idx];
  const int B = gp.B;
  const int kps = kRowsPerStage * f.kpr;  // k per stage
  // LayerNorm phases: the whole normalised row is the same for every segment -- built once per
  // phase when it fits the slice (fp16 words: K / 2 per row)
  // (the whole-row slice covers every stage of the phase: K/2 words rounded up to whole stages,
  // zero past K -- the weights of a partial last stage are zero-filled by TMA, but 0 x stale smem
  // could be NaN)
  const int full_words = f.spt * kRowsPerStage * f.xw;
  const bool full_x = gp.pro == gemm::PRO_LN && full_words <= P.x_cap;
  if (grp == 0) {
    if (f.dep == DEP_FULL) {
      const unsigned t = (epoch + 1u) * f.dep_target;
      wait_all(1, ctid, [&](int, const unsigned*& c, unsigned& tt) {
        c = P.done + f.dep_phase;
        tt = t;
      });
    }
    if (lead) trace_rec(P, cta, p, 1);
    if (full_x) fill_x_ln_fast(gp, sx, hd, 0, full_words, P.xrw, ctid);
  }
  if (full_x) all_bar();
  if (full_x && lead) trace_rec(P, cta, p, 5);
  const int cap = full_x ? f.spt : P.x_cap / (kRowsPerStage * f.xw);  // stages per x chunk
  using Cons = gemm::dev::Consumer<kA16, kNB8, kA16 ? 2 : 0>;  // the model's W8A16 weights are biased
  Cons c;
  c.init(lane);
  for (int i = a; i < e;) {
    const int tile = i / f.spt, st0 = i - tile * f.spt;
    const int n = min(e - i, f.spt - st0);
    c.zero();
    for (int c0 = 0; c0 < n; c0 += cap) {
      const int nn = min(cap, n - c0);
      const int row0 = (st0 + c0) * kRowsPerStage * f.xw, nrows = nn * kRowsPerStage * f.xw;
      if (!full_x) {
        if (grp == 0) {
          if (c0 == 0 && (f.dep == DEP_HEADS || f.dep == DEP_TILES)) {
            const int k0 = st0 * kps, k1 = min(gp.K, (st0 + n) * kps);
            const int unit = f.dep == DEP_HEADS ? P.d : kColTile;
            const int u0 = k0 / unit, u1 = (k1 - 1) / unit;
            const unsigned t = f.dep == DEP_HEADS ? (epoch + 1u) * f.dep_target : epoch + 1u;
            const unsigned* base = (f.dep == DEP_HEADS ? P.head_cnt : P.tile_flag) + f.dep_base + u0;
            wait_all(u1 - u0 + 1, ctid, [&](int j, const unsigned*& cc, unsigned& tt) {
              cc = base + j;
              tt = t;
            });
          }
          if (gp.pro == gemm::PRO_LN)
            fill_x_ln_fast(gp, sx, hd, row0, nrows, P.xrw, ctid);
          else if (f.dep == DEP_HEADS)
            fill_x_attn(P, gp, sx, mw, row0, nrows, ctid);
          else
            fill_x_f16_fast(gp, sx, row0, nrows, P.xrw, ctid);
        }
        all_bar();
        if (lead && i == a && c0 == 0) trace_rec(P, cta, p, 5);
      }
      const uint32_t* xs = (full_x ? sx + row0 : sx);
      const int j0 = my_first(rp.gidx), cnt = my_count(rp.gidx, nn);
      if (cnt > 0) {
        if constexpr (kA16) {
          const int g = lane >> 2, t = lane & 3, xrw = P.xrw;
          c.run_a16(ring, kStageBytes, hd, P.stages, rp.s, rp.ph, cnt, cw, lane, [&](int, int it, int kk, int bt) {
            const int r = bt * 8 + g;
            if (r >= B) return make_uint2(0u, 0u);
            return *reinterpret_cast<const uint2*>(xs + r * xrw + (j0 + kGroups * it) * 2 * kRowsPerStage + 8 * kk + 2 * t);
          }, kGroups);
        } else {
          c.run(ring, hd, P.stages, rp.s, rp.ph, cnt, xs + j0 * kRowsPerStage, P.xrw, B, cw, lane, kGroups);
        }
      }
      rp.gidx += nn;
      if (!full_x) all_bar();  // the x slice is refilled next
    }
    // partials -> tile accumulator (fire-and-forget integer reductions, order independent); the
    // epilogue warp's acq_rel ticket releases them at GPU scope
    long long* acc = P.acc[f.acc] + static_cast<size_t>(tile) * B * kColTile;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int bt = 0; bt < kNB8; ++bt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = cw * gemm::kWarpCols + c.acc_col(j, q);
          const int b = bt * 8 + 2 * c.t + (q & 1);
          if (b < B) red_add(acc + static_cast<size_t>(b) * kColTile + col, __float2ll_rn(c.acc[j][bt][q] * kFix));
        }
    push_unit(ex, rp, p, tile, grp, cw, lane);
    i += n;
  }
  if (lead) trace_rec(P, cta, p, 2);
}

// Decode attention of layer f.idx: items (row, head, context chunk) over the grid.  Each item
// writes its online-softmax partial (unnormalised output, max, sum) to L2 and publishes it; the
// attn-out consumers merge the C partials of the heads they read while building their x slice
// (fill_x_attn), so no merge hop sits between attention and attn-out.
template <int kTPP>
__device__ void attn_phase(const Prog& P, const Phase& f, int p, unsigned epoch, int pos, int cta, int G,
                           float* ascr, int ctid) {
  constexpr int PPR = ops::dev::kAttnThreads / kTPP;
  const ops::AttnParams& ap = P.attn[f.idx];
  const int C = P.attn_chunks, H = ap.H, d = ap.d, hd = H * d;
  const int items = ap.B * H * C;
  const int v = (cta + f.rot) % G;
  if (v >= items) return;
  if (ctid == 0) trace_rec(P, cta, p, 0);
  const Phase& fq = P.phases[f.dep_phase];
  const int ctx = pos + 1;
  const int chunk = (ctx + C - 1) / C;
  float* co = ascr + PPR * d + 2 * PPR;
  float* cst = co + d;
  bool first = true;
  for (int item = v; item < items; item += G) {
    const int bh = item / C, c = item - bh * C;
    const int b = bh / H, head = bh - b * H;
    // q, k and v columns of this head: up to 3 tiles per section (d <= 256)
    int tb[3], tn[3];
#pragma unroll
    for (int sec = 0; sec < 3; ++sec) {
      tb[sec] = (sec * hd + head * d) / kColTile;
      tn[sec] = (sec * hd + head * d + d - 1) / kColTile - tb[sec] + 1;
    }
    wait_all(tn[0] + tn[1] + tn[2], ctid, [&](int j, const unsigned*& cc, unsigned& tt) {
      const int sec = j < tn[0] ? 0 : (j < tn[0] + tn[1] ? 1 : 2);
      const int k = j - (sec > 0 ? tn[0] : 0) - (sec > 1 ? tn[1] : 0);
      cc = P.tile_flag + fq.tile_base + tb[sec] + k;
      tt = epoch + 1u;
    });
    if (first && ctid == 0) trace_rec(P, cta, p, 1);
    first = false;
    const int j0 = c * chunk, j1 = min(ctx, j0 + chunk);
    ops::dev::attn_chunk<kTPP>(ap, b, head, j0, j1, ctid, ascr, [] { consumer_bar(); });
    float* dst = P.attn_ws + static_cast<size_t>(item) * (d + 2);
    for (int i = ctid; i < d; i += 128) dst[i] = co[i];
    if (ctid == 0) {
      dst[d] = cst[0];
      dst[d + 1] = cst[1];
    }
    consumer_bar();
    if (ctid == 0) red_release(P.head_cnt + f.dep_base + head, 1u);
  }
  if (ctid == 0) trace_rec(P, cta, p, 2);
}

// x builders: every load of a round is issued before any is used, so a build costs ONE dependent
// L2 round trip (a round trip under full HBM streaming is a few microseconds: the generic
// chunked builders' 3-5 sequential round trips made the x build the longest part of a phase).

// LayerNorm'd fp16 words [row0, row0 + nrows) of every row (nrows, row0 even): the residual /
// gamma / beta loads of a round (kR float4 per thread) are in flight together with the read of
// the producer's fixed-point row sums.
template <int kR>
__device__ void fill_x_ln_fast(const gemm::Params& gp, uint32_t* sx, Header& hd, int row0, int nrows, int xrw,
                               int ctid) {
  const int K = gp.K, B = gp.B;
  const int n2 = nrows / 2;  // float4 units (4 k = 2 fp16 words)
  const int total = B * n2;
  bool have_stats = false;
  for (int base = ctid;; base += 128 * kR) {
    float4 r[kR];
    uint2 g[kR], be[kR];
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int i = base + 128 * j;
      r[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      g[j] = be[j] = make_uint2(0u, 0u);
      if (i < total) {
        const int b = i / n2;
        const int k = 2 * row0 + 4 * (i - b * n2);
        if (k < K) {  // K % 8 == 0
          r[j] = __ldcg(reinterpret_cast<const float4*>(gp.res_in + static_cast<size_t>(b) * K + k));
          g[j] = __ldg(reinterpret_cast<const uint2*>(gp.ln_g + k));
          be[j] = __ldg(reinterpret_cast<const uint2*>(gp.ln_b + k));
        }
      }
    }
    if (!have_stats) {
      if (ctid < B) gemm::dev::ln_from_sums(gp.ln_stats_in, ctid, gp.ln_inv_k, gp.ln_eps, hd.mean[ctid], hd.rstd[ctid]);
      consumer_bar();
      have_stats = true;
    }
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int i = base + 128 * j;
      if (i < total) {
        const int b = i / n2, u = i - b * n2;
        const int k = 2 * row0 + 4 * u;
        uint2 w = make_uint2(0u, 0u);
        if (k < K) {
          const float mean = hd.mean[b], rstd = hd.rstd[b];
          const __half2 g01 = *reinterpret_cast<const __half2*>(&g[j].x), g23 = *reinterpret_cast<const __half2*>(&g[j].y);
          const __half2 b01 = *reinterpret_cast<const __half2*>(&be[j].x), b23 = *reinterpret_cast<const __half2*>(&be[j].y);
          w.x = gemm::dev::pack_h2((r[j].x - mean) * rstd * __low2float(g01) + __low2float(b01),
                                   (r[j].y - mean) * rstd * __high2float(g01) + __high2float(b01));
          w.y = gemm::dev::pack_h2((r[j].z - mean) * rstd * __low2float(g23) + __low2float(b23),
                                   (r[j].w - mean) * rstd * __high2float(g23) + __high2float(b23));
        }
        *reinterpret_cast<uint2*>(sx + b * xrw + 2 * u) = w;
      }
    }
    if (base + 128 * kR >= total) break;
  }
}

// Plain fp16 x (PRO_F16, x_ld % 8 == 0, 16-byte aligned base) words [row0, row0 + nrows)
// (row0, nrows multiples of 4): 16-byte loads, kR per thread per round.
template <int kR>
__device__ void fill_x_f16_fast(const gemm::Params& gp, uint32_t* sx, int row0, int nrows, int xrw, int ctid) {
  const int K = gp.K, B = gp.B;
  const __half* x = static_cast<const __half*>(gp.x);
  const int n4 = nrows / 4;  // uint4 units (8 k)
  const int total = B * n4;
  for (int base = ctid; base < total; base += 128 * kR) {
    uint4 v[kR];
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int i = base + 128 * j;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (i < total) {
        const int b = i / n4;
        const int k = 2 * row0 + 8 * (i - b * n4);
        if (k < K) v[j] = __ldcg(reinterpret_cast<const uint4*>(x + static_cast<size_t>(b) * gp.x_ld + k));
      }
    }
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int i = base + 128 * j;
      if (i < total) {
        const int b = i / n4;
        *reinterpret_cast<uint4*>(sx + b * xrw + 4 * (i - b * n4)) = v[j];
      }
    }
  }
}

// attn-out x slice (fp16 words [row0, row0 + nrows) of every row) from the attention partials:
// per (row, head) the C chunks merge as exp(m_c - M)-weighted sums divided by the total sum --
// the standalone attention kernel's merge, in the same order.  `mw` holds the merge weights.
__device__ void fill_x_attn(const Prog& P, const gemm::Params& gp, uint32_t* sx, float* mw, int row0, int nrows,
                            int ctid) {
  constexpr int kW = 4, kMaxC = 8;
  const int C = P.attn_chunks, d = P.d, H = P.H, B = gp.B;
  const int k0 = 2 * row0, k1 = min(gp.K, 2 * (row0 + nrows));
  const int h0 = k0 / d, nh = (k1 - 1) / d - h0 + 1;
  const int xrw = P.xrw;
  const int total = B * nrows;
  bool have_w = false;
  for (int base = ctid;; base += 128 * kW) {
    // the partial outputs of this round's words, issued before the merge weights are read
    float2 o[kW][kMaxC];
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int i = base + 128 * j;
      const int b = i / nrows, w = i - b * nrows;
      const int k = 2 * (row0 + w);
      const bool ok = i < total && k < gp.K;
      const int h = ok ? k / d : 0, dim = k - h * d;
      const float* pb = P.attn_ws + (static_cast<size_t>(b) * H + h) * C * (d + 2) + dim;
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)
        o[j][c] = (ok && c < C) ? __ldcg(reinterpret_cast<const float2*>(pb + c * (d + 2))) : make_float2(0.f, 0.f);
    }
    if (!have_w) {
      // per (row, head): chunk weights exp(m_c - M) and 1 / sum (the standalone kernel's merge)
      for (int i = ctid; i < B * nh; i += 128) {
        const int b = i / nh, h = h0 + (i - b * nh);
        const float* pb = P.attn_ws + (static_cast<size_t>(b) * H + h) * C * (d + 2);
        float mc[kMaxC], lc[kMaxC];
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
          mc[c] = c < C ? __ldcg(pb + c * (d + 2) + d) : -INFINITY;
          lc[c] = c < C ? __ldcg(pb + c * (d + 2) + d + 1) : 0.f;
        }
        float M = -INFINITY;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) M = fmaxf(M, mc[c]);
        float L = 0.f;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
          if (c >= C) break;
          const float wgt = mc[c] == -INFINITY ? 0.f : expf(mc[c] - M);
          mw[i * (C + 1) + c] = wgt;
          L += mc[c] == -INFINITY ? 0.f : lc[c] * wgt;
        }
        mw[i * (C + 1) + C] = 1.0f / L;
      }
      consumer_bar();
      have_w = true;
    }
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int i = base + 128 * j;
      if (i >= total) break;
      const int b = i / nrows, w = i - b * nrows;
      const int k = 2 * (row0 + w);
      uint32_t word = 0u;
      if (k < gp.K) {
        const int h = k / d;
        const float* wt = mw + (b * nh + (h - h0)) * (C + 1);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
          if (c >= C) break;
          a0 = fmaf(wt[c], o[j][c].x, a0);
          a1 = fmaf(wt[c], o[j][c].y, a1);
        }
        word = gemm::dev::pack_h2(a0 * wt[C], a1 * wt[C]);
      }
      sx[b * xrw + w] = word;
    }
    if (base + 128 * kW >= total) break;
  }
}

// Token row -> fp32 residual + the first LayerNorm's fixed-point row sums (one CTA per row).
__device__ void embed_phase(const Prog& P, const Phase& f, int p, int pos, int cta, int G, Extra& ex, int cw,
                            int lane, int ctid) {
  const ops::EmbedParams& e = P.embed;
  const int v = (cta + f.rot) % G;
  if (v >= e.B) return;
  for (int b = v; b < e.B; b += G) {
    int tok = pos < e.prompt_len ? e.prompt[static_cast<size_t>(b) * e.prompt_ld + pos] : e.next_tok[b];
    if (tok < 0 || tok >= e.V) tok = 0;
    if (ctid == 0 && pos < e.max_ctx) e.hist[static_cast<size_t>(b) * e.max_ctx + pos] = tok;
    const __half* row = e.wte + static_cast<size_t>(tok) * e.h;
    float* out = e.res + static_cast<size_t>(b) * e.h;
    gemm::dev::RowStat st;
    for (int k = ctid; k < e.h; k += 128) {
      const float r = __half2float(row[k]);
      out[k] = r;
      st.add(r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st.s1 += __shfl_xor_sync(0xffffffffu, st.s1, o);
      st.s2 += __shfl_xor_sync(0xffffffffu, st.s2, o);
    }
    if (lane == 0) {
      ex.red64[2 * cw] = st.s1;
      ex.red64[2 * cw + 1] = st.s2;
    }
    consumer_bar();
    if (ctid == 0 && e.ln_stats_out) {
      long long s1 = 0, s2 = 0;
      for (int w = 0; w < kConsumerWarps; ++w) {
        s1 += ex.red64[2 * w];
        s2 += ex.red64[2 * w + 1];
      }
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(e.ln_stats_out) + b * 2;
      atomicAdd(dst, static_cast<unsigned long long>(s1));
      atomicAdd(dst + 1, static_cast<unsigned long long>(s2));
    }
    consumer_bar();
  }
  if (ctid == 0) {
    fence_acq_rel();
    red_release(P.done + p, 1u);
  }
}

template <int kNB8, int kTPP>
__global__ void __launch_bounds__(kThreadsStep, 1) step_kernel(const __grid_constant__ Prog P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  Header& hd = *reinterpret_cast<Header*>(smem + P.stages * kStageBytes);
  Extra& ex = *reinterpret_cast<Extra*>(smem + P.stages * kStageBytes + sizeof(Header));
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + P.stages * kStageBytes + gemm::kHeaderBytes);
  float* ascr = reinterpret_cast<float*>(sx);  // attention scratch aliases the x slice
  float* mw = reinterpret_cast<float*>(smem + P.stages * kStageBytes + gemm::kHeaderBytes + P.x_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x, G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) {
      ptx::mbar_init(&hd.full[s], 1);
      ptx::mbar_init(&hd.empty[s], kConsumerWarps);  // one group consumes a slot
    }
    for (int q = 0; q < kUnitQueue; ++q) {
      ptx::mbar_init(&ex.ufull[q], kConsumerWarps * kGroups);
      ptx::mbar_init(&ex.uempty[q], 1);
    }
    ptx::fence_mbar_init();
    ex.flag[1] = static_cast<int>(ld_acquire(P.epoch));
    ex.flag[2] = *P.pos;
    red_release(P.arrived, 1u);  // check in: (epoch, pos) of this step have been read
    trace_rec(P, cta, 0, 7);     // CTA start
  }
  __syncthreads();
  const unsigned epoch = static_cast<unsigned>(ex.flag[1]);
  const int pos = ex.flag[2];
  if (warp == 0) {
    if (lane == 0) producer(P, ring, hd, cta, G);
    return;
  }
  if (warp == kEpilogueWarp) {
    epilogue_warp(P, ex, epoch, pos, cta, G, lane);
    return;
  }
  const int grp = (warp - 1) / kConsumerWarps, cw = (warp - 1) % kConsumerWarps;
  const int ctid = threadIdx.x - 32 - 128 * grp;
  RingPos rp{grp, 0, 0, 0, 0};
  for (int p = 0; p < P.n_phases; ++p) {
    const Phase& f = P.phases[p];
    switch (f.kind) {
      case K_EMBED:  // group 0 (the prologue helpers run on 128 threads)
        if (!P.nomma && grp == 0) embed_phase(P, f, p, pos, cta, G, ex, cw, lane, ctid);
        break;
      case K_GEMM:
      case K_LM:
        if (f.xw == 2)
          gemm_phase<true, kNB8>(P, f, p, epoch, cta, G, hd, ex, ring, sx, mw, rp, grp, cw, lane, ctid);
        else
          gemm_phase<false, kNB8>(P, f, p, epoch, cta, G, hd, ex, ring, sx, mw, rp, grp, cw, lane, ctid);
        break;
      case K_ATTN:
        if (!P.nomma && grp == 0) attn_phase<kTPP>(P, f, p, epoch, pos, cta, G, ascr, ctid);
        break;
      default: break;
    }
  }
  push_unit(ex, rp, -1, 0, grp, cw, lane);  // release the epilogue warp
}

using KernelFn = void (*)(Prog);

KernelFn pick(int variant) {
  // variant = (nb8 - 1) * 3 + tpp index (8, 16, 32)
  static const KernelFn table[6] = {step_kernel<1, 8>, step_kernel<1, 16>, step_kernel<1, 32>,
                                    step_kernel<2, 8>, step_kernel<2, 16>, step_kernel<2, 32>};
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
  for (int i = 0; i < 4 * D.L; ++i)
    require(!D.int8 || D.gemms[i].a16, "step kernel: INT8 weights run weight-only (W8A16) only");
  const int tpp = D.d <= 64 ? 8 : (D.d <= 128 ? 16 : 32);
  const int tpp_idx = tpp == 8 ? 0 : (tpp == 16 ? 1 : 2);
  const int nb8 = D.B <= 8 ? 1 : 2;
  variant_ = (nb8 - 1) * 3 + tpp_idx;
  KernelFn kern = pick(variant_);

  int sms = 0, dev = 0, optin = 0;
  DSINF_CUDA_CHECK(cudaGetDevice(&dev));
  DSINF_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DSINF_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int G = sms;  // one CTA per SM (cooperative: all co-resident)

  // ---- shared memory: [ring][header][x slice | attention scratch]
  const size_t attn_bytes = ops::dev::attn_scratch_floats<32>(D.d) * 4;  // largest TPP variant bound
  size_t x_bytes = static_cast<size_t>(std::max(8, env_int("DSINF_STEP_XKB", 32))) * 1024;
  int xrw_max = static_cast<int>(x_bytes / (4 * static_cast<size_t>(D.B)));
  const int x_cap = (xrw_max - 8) / 64 * 64;
  require(x_cap >= 64, "step kernel: x slice budget too small for this batch");
  const int xrw = x_cap + 8;
  x_bytes = std::max(static_cast<size_t>(xrw) * 4 * D.B, attn_bytes);
  x_bytes = (x_bytes + 127) / 128 * 128;
  const int C = std::max(1, std::min(8, (G * std::max(1, env_int("DSINF_STEP_CPS", 1))) / std::max(1, D.B * D.H)));
  const size_t mw_bytes = (static_cast<size_t>(2 * x_cap / D.d + 2) * D.B * (C + 1) * 4 + 127) / 128 * 128;
  cudaFuncAttributes fa{};
  DSINF_CUDA_CHECK(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kern)));
  const size_t fixed = 1024 + gemm::kHeaderBytes + x_bytes + mw_bytes + fa.sharedSizeBytes;
  int stages = static_cast<int>((static_cast<size_t>(optin) - fixed) / kStageBytes);
  stages = std::min(stages, gemm::kMaxStages);
  if (const int e = env_int("DSINF_STEP_STAGES", 0); e > 0) stages = std::min(stages, e);
  stages -= stages % kGroups;  // the groups' interleaved sub-rings
  require(stages >= 2 * kGroups, "step kernel: shared memory too small for the ring");
  smem_ = fixed - fa.sharedSizeBytes + static_cast<size_t>(stages) * kStageBytes;  // dynamic part

  // ---- phases
  std::vector<Phase> phases;
  std::vector<gemm::Params> params = D.gemms;
  std::vector<int> nseg;
  int acc_tiles[kAccKinds] = {0, 0, 0, 0, 0};
  long long stage_cursor = 0;  // rotation: the ranges continue across phases
  auto add_gemm = [&](int idx, int kind, int acc, int dep, int dep_phase, int dep_base, unsigned dep_target) {
    gemm::Params& gp = params[idx];
    require(gp.N % 4 == 0, "step kernel: out_dim must be a multiple of 4");
    require(gp.K % 8 == 0, "step kernel: in_dim must be a multiple of 8");
    if (gp.pro == gemm::PRO_F16 && dep == DEP_TILES)
      require(gp.x_ld % 8 == 0 && (reinterpret_cast<uintptr_t>(gp.x) & 15) == 0,
              "step kernel: fp16 x rows must be 16-byte aligned");
    Phase f{};
    f.kind = kind;
    f.idx = idx;
    f.tiles = (gp.N + kColTile - 1) / kColTile;
    f.spt = (gp.rows + kRowsPerStage - 1) / kRowsPerStage;
    f.total = f.tiles * f.spt;
    f.rot = static_cast<int>(stage_cursor % G);
    stage_cursor += f.total;
    f.xw = gp.a16 ? 2 : 1;
    f.kpr = (D.int8 && kind == K_GEMM) ? 4 : 2;
    f.dep = dep;
    f.dep_phase = dep_phase;
    f.dep_base = dep_base;
    f.dep_target = dep_target;
    f.target = static_cast<unsigned>(f.tiles);
    f.tile_base = static_cast<int>(nseg.size());
    f.acc = acc;
    acc_tiles[acc] = std::max(acc_tiles[acc], f.tiles);
    // contributors per tile: the CTA ranges that intersect it
    std::vector<int> cnt(f.tiles, 0);
    for (int v = 0; v < G; ++v) {
      const int a = range_start(f.total, v, G), e = range_start(f.total, v + 1, G);
      if (a >= e) continue;
      for (int t = a / f.spt; t <= (e - 1) / f.spt; ++t) ++cnt[t];
    }
    nseg.insert(nseg.end(), cnt.begin(), cnt.end());
    gp.x_row_words = xrw;
    gp.ln_inv_k = 1.0 / static_cast<double>(gp.K);
    gp.stages = stages;
    gp.rows_per_split = 0;
    phases.push_back(f);
    return static_cast<int>(phases.size()) - 1;
  };
  Phase e{};
  e.kind = K_EMBED;
  e.target = static_cast<unsigned>(D.B);
  e.rot = 0;
  phases.push_back(e);
  int resid = 0;  // phase whose completion makes the residual (and its row sums) final
  for (int l = 0; l < D.L; ++l) {
    const int q = add_gemm(4 * l + 0, K_GEMM, ACC_QKV, DEP_FULL, resid, 0, phases[resid].target);
    Phase a{};
    a.kind = K_ATTN;
    a.idx = l;
    a.dep_phase = q;
    a.dep_base = l * D.H;
    a.rot = static_cast<int>(stage_cursor % G);
    a.target = static_cast<unsigned>(D.B * D.H);
    phases.push_back(a);
    const int o = add_gemm(4 * l + 1, K_GEMM, ACC_O, DEP_HEADS, q + 1, l * D.H, static_cast<unsigned>(D.B * C));
    const int u = add_gemm(4 * l + 2, K_GEMM, ACC_UP, DEP_FULL, o, 0, phases[o].target);
    resid = add_gemm(4 * l + 3, K_GEMM, ACC_DOWN, DEP_TILES, u, phases[u].tile_base, 0);
  }
  const int lm = add_gemm(4 * D.L, K_LM, ACC_LM, DEP_FULL, resid, 0, phases[resid].target);
  (void)lm;

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
  for (int k = 0; k < kAccKinds; ++k)
    P.acc[k] = static_cast<long long*>(zeros(static_cast<size_t>(std::max(1, acc_tiles[k])) * D.B * kColTile * 8));
  P.nseg = static_cast<const int*>(upload(nseg.data(), nseg.size() * sizeof(int)));
  P.tile_cnt = static_cast<unsigned*>(zeros(nseg.size() * 4));
  P.tile_flag = static_cast<unsigned*>(zeros(nseg.size() * 4));
  P.done = static_cast<unsigned*>(zeros(phases.size() * 4));
  P.head_cnt = static_cast<unsigned*>(zeros(static_cast<size_t>(D.L) * D.H * 4));
  P.attn_ws = static_cast<float*>(dalloc(static_cast<size_t>(D.B) * D.H * C * (D.d + 2) * 4));
  P.arrived = static_cast<unsigned*>(zeros(4));
  P.epoch = static_cast<unsigned*>(zeros(4));
  P.am_key = D.am_key;
  P.lm_valid = D.V;
  P.next_tok = D.next_tok;
  P.hist = D.hist;
  P.pos = D.pos;
  P.max_ctx = D.max_ctx;
  P.B = D.B;
  P.H = D.H;
  P.d = D.d;
  P.stages = stages;
  P.nomma = env_int("DSINF_STEP_NOMMA", 0);
  P.l2_ahead = std::max(0, env_int("DSINF_STEP_L2", 0));
  P.inflight = std::max(0, env_int("DSINF_STEP_INFLIGHT", 0));
  P.xrw = xrw;
  P.x_cap = x_cap;
  P.x_bytes = static_cast<int>(x_bytes);
  P.trace = nullptr;
  trace_len_ = 0;
  if (env_int("DSINF_STEP_TRACE", 0)) {
    trace_len_ = static_cast<size_t>(G) * phases.size() * 8;
    P.trace = static_cast<unsigned long long*>(zeros(trace_len_ * 8));
  }
  trace_ptr_ = P.trace;
  n_phases_ = static_cast<int>(phases.size());

  DSINF_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
  int per_sm = 0;
  DSINF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(kern),
                                                                 kThreadsStep, smem_));
  require(per_sm >= 1, "step kernel: does not fit on an SM");
  grid_ = G;
  stages_ = stages;
  {
    const int nodep = env_int("DSINF_STEP_NODEP", 0);
    DSINF_CUDA_CHECK(cudaMemcpyToSymbol(g_step_nodep, &nodep, sizeof(int)));
  }
  prog_host_.resize(sizeof(Prog));
  std::memcpy(prog_host_.data(), &P, sizeof(Prog));
  built_ = true;
}

void StepProgram::set_embed(const ops::EmbedParams& e) {
  require(built_, "step kernel not built");
  Prog P;
  std::memcpy(&P, prog_host_.data(), sizeof(Prog));
  long long* stats = P.embed.ln_stats_out;  // the first LayerNorm's slot stays the program's
  P.embed = e;
  if (P.embed.ln_stats_out == nullptr) P.embed.ln_stats_out = stats;
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
  attr.id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (cross-CTA waits)
  attr.val.cooperative = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, pick(variant_), P));
}

}  // namespace step
}  // namespace dsinf
