// Decoder-model runtime: synthetic weights on device, the per-step kernel schedule (Deep-Fusion
// regions of PAPER.md:988-993 around SBI-GeMM), tensor-parallel sharding with NCCL (or all
// shards on one device), and whole-step CUDA-graph capture.
//
// Step schedule per shard (t = TP degree; "AR" = all-reduce of a fp32 [B][h] partial):
//   embed                                  res0 = wte[token]
//   per layer:
//     K1 LN1+QKV+bias+RoPE+KV-append       prologue: res1 = res0 (+ d_mlp + b_down[l-1]) ; LN1
//     K2 attention over the KV cache
//     K3 attn-out GEMM                     -> d_attn (partial when t > 1)         AR(d_attn)
//     K4 LN2+MLP-up+bias+GeLU              prologue: res0 = res1 + d_attn + b_o ; LN2
//     K5 MLP-down GEMM                     -> d_mlp                               AR(d_mlp)
//   LM head (final LN prologue: res0 + d_mlp + b_down[L-1]) -> logits + fused argmax keys  AG(keys)
//   select: greedy token (ties -> lowest id), pos += 1
// The residual bias+add (paper region 4) lives in the next LayerNorm's prologue, which is
// also where the TP all-reduced partial is folded in, so t = 1 and t > 1 share one path.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "nccl_dl.h"
#include "ops.cuh"
#include "ptx.cuh"
#include "sbi_gemm.cuh"
#include "step_kernel.cuh"
#include "tc_gemm.cuh"
#include "synth.h"

namespace dsinf {

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct LayerW {
  uint32_t* wqkv = nullptr;
  float* sqkv = nullptr;
  __half* bqkv = nullptr;
  __half *ln1g = nullptr, *ln1b = nullptr;
  uint32_t* wo = nullptr;
  float* so = nullptr;
  __half* bo = nullptr;
  __half *ln2g = nullptr, *ln2b = nullptr;
  uint32_t* wup = nullptr;
  float* sup = nullptr;
  __half* bup = nullptr;
  uint32_t* wdown = nullptr;
  float* sdown = nullptr;
  __half* bdown = nullptr;
  unsigned* up_flags = nullptr;  // DSINF_DOWN_FLAGS: [L][MLP-up column tiles] completion counters (monotonic)
  // int8 K-group scales (dsinf_runtime_config.int8_group = 128): fp16 [K_local/128][N_local]
  __half *gqkv = nullptr, *go = nullptr, *gup = nullptr, *gdown = nullptr;
  // row-major [N][K] copies for the tensor-core prefill (fp16, or int8 with the scales above);
  // generated on the first dsinf_model_prefill
  void *rqkv = nullptr, *ro = nullptr, *rup = nullptr, *rdown = nullptr;
};

// Prefill activations for M = B x P rows (grown on demand).
struct PrefillBufs {
  int64_t cap = 0;
  float* res = nullptr;    // [M][h]
  __half* xn = nullptr;    // [M][h] LayerNorm output (fp16 path)
  int8_t* xq = nullptr;    // [M][max(h, F/t)] int8 GEMM input
  float* xs = nullptr;     // [M] its per-row scales
  __half* q = nullptr;     // [M][Hl*d]
  __half* a = nullptr;     // [M][Hl*d] attention output
  __half* u = nullptr;     // [M][F/t] GeLU output
  float* part = nullptr;   // TP > 1: [M][h] row-parallel partial (all-reduced in place)
};

struct Shard {
  int rank = 0;
  std::vector<LayerW> layers;
  uint32_t* wlm = nullptr;  // fp16 packed [h/2][Vl][2]
  __half *lnfg = nullptr, *lnfb = nullptr;
  __half* wte = nullptr;    // row-major [V][h] (replicated)
  float* res[2] = {nullptr, nullptr};
  float* d_attn = nullptr;
  float* d_mlp = nullptr;
  __half* q = nullptr;
  __half* a = nullptr;
  __half* u = nullptr;
  float* logits = nullptr;
  __half* kc = nullptr;
  __half* vc = nullptr;
  __half* xn = nullptr;    // x-streaming plan: LayerNorm output fp16 [B][h]
  int8_t* xq = nullptr;    // x-streaming plan, int8: quantised x [B][max(h, F/t)]
  float* xsc = nullptr;    // its per-token scales [B]
  long long* lnstats = nullptr;  // [2L+1][kLnSlotWords]: LayerNorm row sums from the producing epilogue
  unsigned* amax = nullptr;      // [2L][kAmaxSlotWords]: int8 activation row max from the producer
  unsigned* head_ctr = nullptr;  // [L][Hl]: QKV attention-tail piece counters (m.attn_fuse; zero at rest)
  gemm::Plan plan_qkv{}, plan_o{}, plan_up{}, plan_down{}, plan_lm{};
  PrefillBufs pf;
  bool rm_ready = false;
  // prefill weights when the row-major copies of every layer do not fit (or DSINF_PREFILL_REPACK=1):
  // ONE layer's four row-major tensors, re-filled from the packed decode weights before each
  // layer's GEMMs (packed_to_rowmajor), so the model keeps a single resident weight copy
  bool rm_per_layer = false;
  void* rm_scratch[4] = {nullptr, nullptr, nullptr, nullptr};
  // fused tensor-parallel all-reduce: [2 points][t source ranks][B*h] partial slots written by every
  // rank's attn-out (point 0) / MLP-down (point 1) epilogue, and their arrival counters [2][L]
  float* red = nullptr;
  unsigned long long* red_flag = nullptr;
  unsigned long long* push_done = nullptr;  // [2][L] gpu-local CTA counters of the last-CTA signalling
  // every rank's red / red_flag as addressable from this rank: the other on-device shards
  // (DSINF_TP_LOCAL) or CUDA-IPC mappings of the peer processes' allocations over NVLink (NCCL mode)
  std::vector<float*> peer_red;
  std::vector<unsigned long long*> peer_flag;
};

}  // namespace

}  // namespace dsinf

struct dsinf_model {
  dsinf_model_config cfg{};
  dsinf_runtime_config rt{};
  int64_t h = 0, L = 0, H = 0, d = 0, Hl = 0, V = 0, Vpad = 0, Vl = 0, F = 0, Fl = 0;
  int B = 0, t = 1, max_ctx = 0;
  bool int8 = false;
  bool a16 = false;  // int8 weights with fp16 activations (W8A16) in some decode GEMM
  int a16_mask = 0;  // which: bit 0 QKV, 1 attn-out, 2 MLP-up, 3 MLP-down
  bool a16g(int g) const { return int8 && ((a16_mask >> g) & 1); }
  bool q8g(int g) const { return int8 && !a16g(g); }  // GEMM g takes int8 activations (W8A8)
  bool q8() const { return q8g(0) || q8g(1) || q8g(2) || q8g(3); }  // any W8A8 GEMM
  std::vector<dsinf::DevBuf> allocs;
  std::vector<dsinf::Shard> shards;
  float2* rope = nullptr;
  int32_t* prompt = nullptr;
  int prompt_cap = 0, prompt_len = 0;
  int32_t* next_tok = nullptr;
  int32_t* hist = nullptr;
  int* pos = nullptr;
  float* am_val = nullptr;  // [t][B]
  int32_t* am_idx = nullptr;
  unsigned long long* am_key = nullptr;  // [t][B] fused LM-head argmax keys (zeroed per step)
  dsinf::nccl::Comm comm = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t host_pos = 0;
  int64_t weight_bytes = 0;
  int64_t kernels_per_step = 0;
  int attn_chunks = 1;
  dsinf::step::StepProgram step_prog;  // persistent whole-step kernel (TP = 1)
  // TP = 1: the attn-out / MLP-down epilogues add the residual and emit the next LayerNorm's
  // row sums, so the LN prologues skip their full-row statistics pass (DSINF_FUSE_STATS=0: off)
  bool fuse_ln = false;
  // QKV attention tail (Deep-Fusion region 2 in the QKV launch, LayerNorm-streaming plan): no
  // standalone attention launch.  Opt-in (DSINF_ATTN_FUSE=1; DSINF_ATTN_FUSE_MAXB batch cap, 8)
  bool attn_fuse = false;
  // attention PDL-launched with its dependents released after its own dependency wait (and MLP-down
  // early): fp16 at h <= 4096 and INT8 at h < 4096, TP = 1 (GPT-J fp16 B=1 2.501 -> 2.458 ms, B=8
  // 2.707 -> 2.670; GPT-2 int8 B=8 1.818 -> 1.764; slower for GPT-J INT8 and NeoX fp16;
  // profiles/r2_attn_late_trigger.log)
  bool attn_late = false;
  // TP > 1 without NCCL kernels between the GEMMs: the row-parallel GEMMs push their partials into
  // every rank's slots and signal a counter; the next LayerNorm prologue waits and sums the slots
  bool fused_ar = false;
  // fused all-reduce signalling: gpu-scope fences when every destination is on this GPU (TP_LOCAL,
  // TP_SLICE; DSINF_FAR_SYS=1 forces system scope for measurement); with system scope the grid's last
  // CTA signals each rank once (DSINF_FAR_LASTCTA=0: every CTA signals)
  bool far_gpu_scope = false, far_last_cta = false;
  long long* step_ctr = nullptr;  // decode steps taken (fused all-reduce counter targets)
  // DSINF_TP_IPC: argmax-key arrival counter (bumped by the peers' select kernels) and the peers'
  // key arrays / counters as mapped into this process; ipc_ready once dsinf_model_ipc_attach ran
  unsigned long long* key_flag = nullptr;
  std::vector<unsigned long long*> peer_keys, peer_key_flag;
  bool ipc_ready = false;
  std::vector<void*> ipc_maps;    // peer allocations opened with cudaIpcOpenMemHandle
  // x-streaming GEMM plans (gemm::Plan::x_stream): x reaches each stage by TMA next to the
  // weights instead of a per-CTA smem slice.  xs_ln: the LayerNorm GEMMs (QKV, MLP-up, LM head)
  // take x from a row_prep launch; xs_od: attn-out / MLP-down (int8: after a quantise prep).
  bool xs_ln = false, xs_od = false, xs_lm = false;
  // LayerNorm-streaming (gemm::Plan::ln_stream; TP = 1 with producer-fused statistics): the
  // LayerNorm GEMMs stream the fp32 residual and normalise it per stage -- no row_prep launch.
  // Not for W8A8 GEMMs (their per-token scale needs the whole normalised row).  DSINF_LN_STREAM=0: off
  bool ln_stream = false;
  // DSINF_DOWN_FLAGS=1 (TP = 1, x-streamed fp16 / W8A16 MLP-down): MLP-down is PDL-launched and its
  // producer waits only for the MLP-up column tiles of its k range (per-tile counters) instead of
  // the whole MLP-up grid; its epilogue still waits for the grid
  bool down_flags = false;
  bool ln_use(int g) const { return ln_stream && !q8g(g); }  // g: 0 QKV, 2 MLP-up, 4 LM head (fp16)
  unsigned long long* ltrace = nullptr;
  std::vector<int> ltrace_kinds;  // DSINF_LAUNCH_TRACE: [2][ptx::kTraceEnd] start / end stamps
  int64_t ltrace_n = 0;
  unsigned long long* cta_log = nullptr;  // DSINF_CTA_LOG=<n>: per-CTA stamps of the n-th SBI-GeMM launch of a step
  int cta_log_launch = -1;

  void* alloc(size_t bytes) {
    void* p = nullptr;
    DSINF_CUDA_CHECK(cudaMalloc(&p, bytes));
    allocs.push_back({p, bytes});
    return p;
  }
  template <class T>
  T* alloc_n(int64_t n) {
    return static_cast<T*>(alloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T)));
  }
  // NCCL mode: the per-layer all-reduce buffers in NCCL symmetric memory (ncclMemAlloc, registered as
  // NCCL_WIN_COLL_SYMMETRIC windows) when the library has them; released before the communicator
  std::vector<std::pair<void*, dsinf::nccl::Window>> nccl_windows;
  ~dsinf_model() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& w : nccl_windows) {
      dsinf::nccl::window_deregister(comm, w.second);
      dsinf::nccl::mem_free(w.first);
    }
    for (void* p : ipc_maps) cudaIpcCloseMemHandle(p);
    for (auto& a : allocs) cudaFree(a.p);
    if (cta_log) cudaFree(cta_log);
  }
};

namespace dsinf {

namespace {

using Model = dsinf_model;

ops::ShardMap make_map(uint64_t seed, int64_t N_local, int64_t K_local, int64_t N_global, int64_t K_global,
                       int64_t sec_local, int64_t sec_global, int64_t row_off, int64_t col_off, int layer,
                       int tensor, float amp, int64_t valid_rows = -1) {
  ops::ShardMap s{};
  s.N_local = N_local;
  s.K_local = K_local;
  s.N_global = N_global;
  s.K_global = K_global;
  s.sec_local = sec_local;
  s.sec_global = sec_global;
  s.row_off = row_off;
  s.col_off = col_off;
  s.valid_rows = valid_rows < 0 ? N_global : valid_rows;
  s.base = synth_base(seed, layer, tensor);
  s.amp = amp;
  return s;
}

float tensor_amp(int tensor, float* offset) {
  *offset = 0.f;
  switch (tensor) {
    case DSINF_T_QKV_BIAS:
    case DSINF_T_O_BIAS:
    case DSINF_T_UP_BIAS:
    case DSINF_T_DOWN_BIAS: return SynthScale::kBias;
    case DSINF_T_LN1_G:
    case DSINF_T_LN2_G:
    case DSINF_T_LNF_G: *offset = 1.f; return SynthScale::kLnGamma;
    case DSINF_T_LN1_B:
    case DSINF_T_LN2_B:
    case DSINF_T_LNF_B: return SynthScale::kLnBeta;
    default: return SynthScale::kWeight;
  }
}

// Megatron tensor-parallel shard of one synthetic tensor for rank r of t:
// QKV column-parallel by head (local rows [q_r | k_r | v_r]); attn-out row-parallel over this
// rank's heads; MLP-up column-parallel; MLP-down row-parallel; LM head vocab-parallel over the
// vocab padded to 128*t rows; biases / LayerNorm replicated.  The device generator and the host
// dsinf_shard_tensor both use this map.
ops::ShardMap tensor_map(int64_t h, int64_t H, int64_t V, int t, int r, uint64_t seed, int layer, int tensor) {
  const int64_t d = h / H, Hl = H / t, F = 4 * h, Fl = F / t;
  const int64_t vq = 128LL * t, Vpad = (V + vq - 1) / vq * vq, Vl = Vpad / t;
  float off = 0.f;
  const float amp = tensor_amp(tensor, &off);
  switch (tensor) {
    case DSINF_T_QKV: return make_map(seed, 3 * Hl * d, h, 3 * h, h, Hl * d, h, r * Hl * d, 0, layer, tensor, amp);
    case DSINF_T_QKV_BIAS: return make_map(seed, 3 * Hl * d, 1, 3 * h, 1, Hl * d, h, r * Hl * d, 0, layer, tensor, amp);
    case DSINF_T_O: return make_map(seed, h, Hl * d, h, h, h, h, 0, r * Hl * d, layer, tensor, amp);
    case DSINF_T_UP: return make_map(seed, Fl, h, F, h, Fl, F, r * Fl, 0, layer, tensor, amp);
    case DSINF_T_UP_BIAS: return make_map(seed, Fl, 1, F, 1, Fl, F, r * Fl, 0, layer, tensor, amp);
    case DSINF_T_DOWN: return make_map(seed, h, Fl, h, F, h, h, 0, r * Fl, layer, tensor, amp);
    case DSINF_T_WTE: return make_map(seed, Vl, h, Vpad, h, Vl, Vpad, r * Vl, 0, layer, tensor, amp, V);
    default: return make_map(seed, h, 1, h, 1, h, h, 0, 0, layer, tensor, amp);  // replicated vectors
  }
}

// Allocates and generates one GEMM weight in the packed layout (fp16 M=2 or int8 M=4).
// biased: int8 bytes stored as s + 128 for the W8A16 GEMMs (gemm::Plan::a16 == 2)
uint32_t* make_weight(Model& m, const ops::ShardMap& map, float** scales, cudaStream_t s, __half** gscales = nullptr,
                      bool biased = false) {
  const int M = m.int8 ? 4 : 2;
  const int64_t words = (map.K_local + M - 1) / M * map.N_local;
  uint32_t* w = m.alloc_n<uint32_t>(words);
  m.weight_bytes += words * 4;
  if (m.int8 && m.rt.int8_group != 0) {  // K-group scales: the W8A16 GEMMs dequantise per group
    const int64_t ng = map.K_local / ops::kI8Group * map.N_local;
    *gscales = m.alloc_n<__half>(ng);
    m.weight_bytes += ng * 2;
    *scales = nullptr;
    ops::init_packed_i8_groups(map, w, *gscales, s, biased);
  } else if (m.int8) {
    *scales = m.alloc_n<float>(map.N_local);
    m.weight_bytes += map.N_local * 4;
    ops::init_packed_i8(map, w, *scales, s, biased);
  } else {
    *scales = nullptr;
    ops::init_packed_f16(map, w, s);
  }
  return w;
}

__half* make_vec(Model& m, const ops::ShardMap& map, float offset, cudaStream_t s) {
  __half* v = m.alloc_n<__half>(map.N_local);
  m.weight_bytes += map.N_local * 2;
  ops::init_vector_f16(map, offset, v, s);
  return v;
}

void build_shard(Model& m, Shard& sh, cudaStream_t s) {
  const int r = sh.rank;
  const int64_t h = m.h, Hl = m.Hl, d = m.d, Fl = m.Fl;
  sh.layers.resize(m.L);
  for (int l = 0; l < m.L; ++l) {
    LayerW& w = sh.layers[l];
    auto map = [&](int tensor) { return tensor_map(h, m.H, m.V, m.t, r, m.rt.seed, l, tensor); };
    auto vec = [&](int tensor) {
      float off = 0.f;
      tensor_amp(tensor, &off);
      return make_vec(m, map(tensor), off, s);
    };
    w.wqkv = make_weight(m, map(DSINF_T_QKV), &w.sqkv, s, &w.gqkv, m.a16g(0));
    w.bqkv = vec(DSINF_T_QKV_BIAS);
    w.wo = make_weight(m, map(DSINF_T_O), &w.so, s, &w.go, m.a16g(1));
    w.bo = vec(DSINF_T_O_BIAS);
    w.wup = make_weight(m, map(DSINF_T_UP), &w.sup, s, &w.gup, m.a16g(2));
    w.bup = vec(DSINF_T_UP_BIAS);
    w.wdown = make_weight(m, map(DSINF_T_DOWN), &w.sdown, s, &w.gdown, m.a16g(3));
    w.bdown = vec(DSINF_T_DOWN_BIAS);
    w.ln1g = vec(DSINF_T_LN1_G);
    w.ln1b = vec(DSINF_T_LN1_B);
    w.ln2g = vec(DSINF_T_LN2_G);
    w.ln2b = vec(DSINF_T_LN2_B);
  }
  // LM head (tied with the embedding, fp16 in both modes): vocab parallel, padded rows are 0
  {
    const ops::ShardMap lm = tensor_map(h, m.H, m.V, m.t, r, m.rt.seed, -1, DSINF_T_WTE);
    const int64_t words = (h + 1) / 2 * m.Vl;
    sh.wlm = m.alloc_n<uint32_t>(words);
    m.weight_bytes += words * 4;
    ops::init_packed_f16(lm, sh.wlm, s);
  }
  sh.lnfg = make_vec(m, tensor_map(h, m.H, m.V, m.t, r, m.rt.seed, -1, DSINF_T_LNF_G), 1.f, s);
  sh.lnfb = make_vec(m, tensor_map(h, m.H, m.V, m.t, r, m.rt.seed, -1, DSINF_T_LNF_B), 0.f, s);
  if (r == 0 || m.rt.tp_mode != DSINF_TP_LOCAL) {
    sh.wte = m.alloc_n<__half>(m.V * h);
    ops::init_rowmajor_f16(synth_base(m.rt.seed, -1, DSINF_T_WTE), SynthScale::kWeight, m.V, h, sh.wte, s);
  } else {
    sh.wte = m.shards[0].wte;
  }
  const int B = m.B;
  sh.res[0] = m.alloc_n<float>(B * h);
  sh.res[1] = m.alloc_n<float>(B * h);
  const char* wv = std::getenv("DSINF_NCCL_WINDOWS");
  if (m.rt.tp_mode == DSINF_TP_NCCL && m.t > 1 && !m.fused_ar && m.comm != nullptr && nccl::has_windows() &&
      (wv == nullptr || std::atoi(wv) != 0)) {
    // latency-bound B x h fp32 messages (16-786 KB): symmetric windows let NCCL use its symmetric-memory
    // all-reduce kernels (collective registration, same order on every rank)
    for (float** d : {&sh.d_attn, &sh.d_mlp}) {
      void* p = nccl::mem_alloc(static_cast<size_t>(B * h) * 4);
      m.nccl_windows.emplace_back(p, nccl::window_register(m.comm, p, static_cast<size_t>(B * h) * 4));
      *d = static_cast<float*>(p);
    }
  } else {
    sh.d_attn = m.alloc_n<float>(B * h);
    sh.d_mlp = m.alloc_n<float>(B * h);
  }
  sh.q = m.alloc_n<__half>(B * Hl * d);
  sh.a = m.alloc_n<__half>(B * Hl * d);
  sh.u = m.alloc_n<__half>(B * Fl);
  sh.logits = m.alloc_n<float>(B * m.Vl);
  const int64_t kv = m.L * B * Hl * static_cast<int64_t>(m.max_ctx) * d;
  sh.kc = m.alloc_n<__half>(kv);
  sh.vc = m.alloc_n<__half>(kv);
  DSINF_CUDA_CHECK(cudaMemsetAsync(sh.kc, 0, kv * 2, s));
  DSINF_CUDA_CHECK(cudaMemsetAsync(sh.vc, 0, kv * 2, s));
  DSINF_CUDA_CHECK(cudaMemsetAsync(sh.d_mlp, 0, B * h * 4, s));
  if (m.fused_ar) {
    sh.red = m.alloc_n<float>(2LL * m.t * B * h);
    sh.red_flag = m.alloc_n<unsigned long long>(2 * std::max<int64_t>(1, m.L));
    DSINF_CUDA_CHECK(cudaMemsetAsync(sh.red_flag, 0, 2 * std::max<int64_t>(1, m.L) * 8, s));
    DSINF_CUDA_CHECK(cudaMemsetAsync(sh.red, 0, 2LL * m.t * B * h * 4, s));  // TP_SLICE reads unpushed slots
    sh.push_done = m.alloc_n<unsigned long long>(2 * std::max<int64_t>(1, m.L));
    DSINF_CUDA_CHECK(cudaMemsetAsync(sh.push_done, 0, 2 * std::max<int64_t>(1, m.L) * 8, s));
  }
  if (m.fuse_ln) sh.lnstats = m.alloc_n<long long>((2 * m.L + 1) * gemm::kLnSlotWords);
  if (m.xs_ln || m.xs_lm) sh.xn = m.alloc_n<__half>(static_cast<int64_t>(B) * h);
  if (m.q8() && (m.xs_ln || m.xs_od)) {
    sh.xq = m.alloc_n<int8_t>(static_cast<int64_t>(B) * std::max(h, Fl));
    sh.xsc = m.alloc_n<float>(B);
  }
  if (m.q8()) sh.amax = m.alloc_n<unsigned>(std::max<int64_t>(1, 2 * m.L) * gemm::kAmaxSlotWords);
  if (m.attn_fuse) {
    sh.head_ctr = m.alloc_n<unsigned>(std::max<int64_t>(1, m.L) * Hl);
    DSINF_CUDA_CHECK(cudaMemsetAsync(sh.head_ctr, 0, std::max<int64_t>(1, m.L) * Hl * sizeof(unsigned), s));
  }
  const bool i8 = m.int8;
  const bool kg = m.rt.int8_group != 0;
  // per-GEMM ring depth requests (DSINF_STAGES_{QKV,O,UP,DOWN}; 0 = the plan's own).  Measured
  // defaults at TP = 1, h >= 4096 (GPT-J; profiles/r2_stage_sweep.log): QKV 3 stages for fp16 (B=1
  // 2.520 -> 2.501 ms, B=8 2.797 -> 2.752, B=16 with MLP-up 2: 3.154 -> 3.123) and W8A16 at B > 2
  // (B=8 2.185 -> 2.148; B=16 W8A16 QKV 2.602 -> 2.508, profiles/r2_b16_sweep.log); the LayerNorm-streaming W8A16 MLP-up 4 stages at B <= 2 (B=1 1.723 -> 1.685,
  // B=2 1.808 -> 1.777).  GPT-2 (h 1600) keeps the plan's own depths (both measured slower there).
  const bool big = m.t == 1 && h >= 4096;
  auto st_req = [](const char* name, int dflt) { const char* v = std::getenv(name); return v ? std::atoi(v) : dflt; };
  // per-GEMM K-split requests (DSINF_KSPLIT_{QKV,O,UP,DOWN}; 0 = the plan's one-wave choice)
  auto ks_req = [](const char* name) { const char* v = std::getenv(name); return v ? std::atoi(v) : 0; };
  const int qkv_st = big && (!i8 || (m.a16g(0) && B > 2)) ? 3 : 0;
  const int up_st = big && i8 && m.a16g(2) && m.ln_use(2) && B <= 2 ? 4 : (big && !i8 && B > 8 ? 2 : 0);
  sh.plan_qkv = gemm::make_plan(static_cast<int>(3 * Hl * d), static_cast<int>(h), B, i8, ks_req("DSINF_KSPLIT_QKV"), m.xs_ln, m.a16g(0),
                                m.ln_use(0), m.a16g(0), kg, st_req("DSINF_STAGES_QKV", qkv_st));
  sh.plan_o = gemm::make_plan(static_cast<int>(h), static_cast<int>(Hl * d), B, i8, ks_req("DSINF_KSPLIT_O"), m.xs_od, m.a16g(1), false,
                              m.a16g(1), kg, st_req("DSINF_STAGES_O", 0));
  sh.plan_up = gemm::make_plan(static_cast<int>(Fl), static_cast<int>(h), B, i8, ks_req("DSINF_KSPLIT_UP"), m.xs_ln, m.a16g(2), m.ln_use(2),
                               m.a16g(2), kg, st_req("DSINF_STAGES_UP", up_st));
  sh.plan_down = gemm::make_plan(static_cast<int>(h), static_cast<int>(Fl), B, i8, ks_req("DSINF_KSPLIT_DOWN"), m.xs_od, m.a16g(3), false,
                                 m.a16g(3), kg, st_req("DSINF_STAGES_DOWN", 0));
  if (m.down_flags) {
    for (LayerW& w : sh.layers) {
      w.up_flags = m.alloc_n<unsigned>(sh.plan_up.col_tiles);
      DSINF_CUDA_CHECK(cudaMemsetAsync(w.up_flags, 0, sizeof(unsigned) * sh.plan_up.col_tiles, s));
    }
  }
  // LM head ring depth (DSINF_LM_STAGES; 0 = the plan's own): 2 at B <= 8, where the shallower ring
  // fits more CTAs per SM (GPT-J int8 B=1 1.738 -> 1.724 ms, fp16 2.531 -> 2.521, fp16 B=8 2.811 ->
  // 2.797; B=16 neutral; profiles/r2_lm_stages_sweep.log)
  const int lm_stages = [&] { const char* v = std::getenv("DSINF_LM_STAGES"); return v ? std::atoi(v) : (B <= 8 ? 2 : 0); }();
  sh.plan_lm = gemm::make_plan(static_cast<int>(m.Vl), static_cast<int>(h), B, false, 0, m.xs_lm, false,
                               m.ln_stream && m.xs_lm, false, false, lm_stages);
}

// Row-major copies of the layer GEMM weights for the tensor-core prefill (same synthetic values;
// int8 quantised with the packed layout's row scales).
void build_rowmajor(Model& m, Shard& sh, cudaStream_t s) {
  const int r = sh.rank;
  const int64_t h = m.h;
  {
    const int64_t eb = m.int8 ? 1 : 2;
    const int64_t layer_bytes = (3 * m.Hl * m.d * h + h * m.Hl * m.d + 2 * m.Fl * h) * eb;
    size_t free_b = 0, total_b = 0;
    DSINF_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const char* rp = std::getenv("DSINF_PREFILL_REPACK");
    const int64_t shards_left = static_cast<int64_t>(m.shards.size());  // copies still to build (worst case)
    const bool fits = static_cast<double>(layer_bytes) * m.L * shards_left + (4LL << 30) < static_cast<double>(free_b);
    sh.rm_per_layer = rp ? std::atoi(rp) != 0 : !fits;
    if (sh.rm_per_layer) {
      const int64_t qkv = 3 * m.Hl * m.d * h, o = h * m.Hl * m.d, f = m.Fl * h;
      sh.rm_scratch[0] = m.alloc(static_cast<size_t>(qkv * eb));
      sh.rm_scratch[1] = m.alloc(static_cast<size_t>(o * eb));
      sh.rm_scratch[2] = m.alloc(static_cast<size_t>(f * eb));
      sh.rm_scratch[3] = m.alloc(static_cast<size_t>(f * eb));
      for (int l = 0; l < m.L; ++l) {
        LayerW& w = sh.layers[l];
        w.rqkv = sh.rm_scratch[0];
        w.ro = sh.rm_scratch[1];
        w.rup = sh.rm_scratch[2];
        w.rdown = sh.rm_scratch[3];
      }
      sh.rm_ready = true;
      return;
    }
  }
  for (int l = 0; l < m.L; ++l) {
    LayerW& w = sh.layers[l];
    auto make = [&](int tensor, const float* scales) -> void* {
      const ops::ShardMap map = tensor_map(h, m.H, m.V, m.t, r, m.rt.seed, l, tensor);
      const int64_t n = map.N_local * map.K_local;
      if (m.int8) {
        int8_t* out = m.alloc_n<int8_t>(n);
        ops::init_rowmajor_map_i8(map, scales, out, s);
        return out;
      }
      __half* out = m.alloc_n<__half>(n);
      ops::init_rowmajor_map_f16(map, out, s);
      return out;
    };
    w.rqkv = make(DSINF_T_QKV, w.sqkv);
    w.ro = make(DSINF_T_O, w.so);
    w.rup = make(DSINF_T_UP, w.sup);
    w.rdown = make(DSINF_T_DOWN, w.sdown);
  }
  sh.rm_ready = true;
}

void ensure_prefill_bufs(Model& m, Shard& sh, int64_t M) {
  PrefillBufs& pf = sh.pf;
  if (pf.cap >= M) return;
  const int64_t h = m.h, Hd = m.Hl * m.d, Fl = m.Fl;
  pf.res = m.alloc_n<float>(M * h);
  pf.xn = m.alloc_n<__half>(M * h);
  if (m.int8) {
    pf.xq = m.alloc_n<int8_t>(M * std::max(h, Fl));
    pf.xs = m.alloc_n<float>(M);
  }
  pf.q = m.alloc_n<__half>(M * Hd);
  pf.a = m.alloc_n<__half>(M * Hd);
  pf.u = m.alloc_n<__half>(M * Fl);
  if (m.t > 1) pf.part = m.alloc_n<float>(M * h);
  pf.cap = M;
}

gemm::Params base_params(const Model& m, const uint32_t* w, const float* ws, int N, int K, bool int8_w,
                         const __half* gs = nullptr) {
  gemm::Params p{};
  p.rows = int8_w ? (K + 3) / 4 : (K + 1) / 2;
  gemm::make_weight_map(&p.tmap, w, N, p.rows);
  p.w_scale = ws;
  p.w_gscale = int8_w ? gs : nullptr;
  p.N = N;
  p.K = K;
  p.B = m.B;
  p.ln_eps = m.rt.ln_eps;
  p.out_ld = N;
  return p;
}

ops::EmbedParams embed_params(const Model& m, const Shard& sh) {
  ops::EmbedParams e{};
  e.wte = sh.wte;
  e.prompt = m.prompt;
  e.prompt_len = m.prompt_len;
  e.prompt_ld = m.prompt_cap;
  e.next_tok = m.next_tok;
  e.pos = m.pos;
  e.hist = m.hist;
  e.max_ctx = m.max_ctx;
  e.res = sh.res[0];
  e.B = m.B;
  e.h = static_cast<int>(m.h);
  e.V = static_cast<int>(m.V);
  return e;
}

ops::AttnParams attn_params(const Model& m, const Shard& sh, int l) {
  ops::AttnParams a{};
  const size_t layer_kv = static_cast<size_t>(m.B) * m.Hl * m.max_ctx * m.d;
  a.q = sh.q;
  a.kc = sh.kc + l * layer_kv;
  a.vc = sh.vc + l * layer_kv;
  a.pos = m.pos;
  a.out = sh.a;
  a.B = m.B;
  a.H = static_cast<int>(m.Hl);
  a.d = static_cast<int>(m.d);
  a.max_seq = m.max_ctx;
  a.scale = 1.0f / std::sqrt(static_cast<float>(m.d));
  return a;
}

// The persistent whole-step kernel's program (TP = 1): one fp32 residual stream updated in place by
// the attn-out / MLP-down epilogues (EPI_RESID), LayerNorm prologues without a pending delta.
void build_step_program(Model& m) {
  Shard& sh = m.shards[0];
  step::StepDesc D;
  D.B = m.B;
  D.L = static_cast<int>(m.L);
  D.H = static_cast<int>(m.Hl);
  D.d = static_cast<int>(m.d);
  D.max_ctx = m.max_ctx;
  D.V = static_cast<int>(m.V);
  D.Vl = static_cast<int>(m.Vl);
  D.int8 = m.int8;
  float* r = sh.res[0];
  const int h = static_cast<int>(m.h), HD = static_cast<int>(m.Hl * m.d), Fl = static_cast<int>(m.Fl);
  const size_t layer_kv = static_cast<size_t>(m.B) * m.Hl * m.max_ctx * m.d;
  require(sh.lnstats != nullptr, "the persistent step kernel needs the producer-fused LayerNorm sums (DSINF_FUSE_STATS)");
  auto slot = [&](int i) { return sh.lnstats + static_cast<int64_t>(i) * gemm::kLnSlotWords; };
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = sh.layers[l];
    gemm::Params q = base_params(m, w.wqkv, w.sqkv, 3 * HD, h, m.int8);
    q.a16 = m.int8 ? 1 : 0;
    q.pro = gemm::PRO_LN;
    q.ln_stats_in = slot(2 * l);
    q.res_in = r;
    q.ln_g = w.ln1g;
    q.ln_b = w.ln1b;
    q.epi = gemm::EPI_QKV;
    q.bias = w.bqkv;
    q.q_out = sh.q;
    q.k_cache = sh.kc + l * layer_kv;
    q.v_cache = sh.vc + l * layer_kv;
    q.rope = m.rope;
    q.pos = m.pos;
    q.heads = static_cast<int>(m.Hl);
    q.head_dim = static_cast<int>(m.d);
    q.max_seq = m.max_ctx;
    gemm::Params o = base_params(m, w.wo, w.so, h, HD, m.int8);
    o.a16 = q.a16;
    o.pro = gemm::PRO_F16;
    o.x = sh.a;
    o.x_ld = HD;
    o.epi = gemm::EPI_RESID;
    o.out = r;
    o.bias = w.bo;
    o.ln_stats_out = slot(2 * l + 1);
    gemm::Params u = base_params(m, w.wup, w.sup, Fl, h, m.int8);
    u.a16 = q.a16;
    u.pro = gemm::PRO_LN;
    u.ln_stats_in = slot(2 * l + 1);
    u.res_in = r;
    u.ln_g = w.ln2g;
    u.ln_b = w.ln2b;
    u.epi = gemm::EPI_GELU_F16;
    u.bias = w.bup;
    u.out = sh.u;
    gemm::Params dn = base_params(m, w.wdown, w.sdown, h, Fl, m.int8);
    dn.a16 = q.a16;
    dn.pro = gemm::PRO_F16;
    dn.x = sh.u;
    dn.x_ld = Fl;
    dn.epi = gemm::EPI_RESID;
    dn.out = r;
    dn.bias = w.bdown;
    dn.ln_stats_out = slot(2 * l + 2);
    D.gemms.push_back(q);
    D.gemms.push_back(o);
    D.gemms.push_back(u);
    D.gemms.push_back(dn);
    D.attn.push_back(attn_params(m, sh, l));
  }
  gemm::Params lm = base_params(m, sh.wlm, nullptr, static_cast<int>(m.Vl), h, false);
  lm.pro = gemm::PRO_LN;
  lm.ln_stats_in = slot(2 * static_cast<int>(m.L));
  lm.res_in = r;
  lm.ln_g = sh.lnfg;
  lm.ln_b = sh.lnfb;
  lm.epi = gemm::EPI_F32;
  lm.out = sh.logits;
  D.gemms.push_back(lm);
  D.embed = embed_params(m, sh);
  D.embed.ln_stats_out = slot(0);
  D.am_key = m.am_key;
  D.logits = sh.logits;
  D.next_tok = m.next_tok;
  D.hist = m.hist;
  D.pos = m.pos;
  m.step_prog.build(D);
}

struct Enqueuer {
  Model& m;
  cudaStream_t s;
  bool pdl;
  int64_t launches = 0;

  // DSINF_PDL_MASK bits: 0 qkv, 1 attention, 2 attn-out, 3 up, 4 down, 5 lm head, 6 the rest,
  // 7 row_prep.
  // Default 0xad: QKV, attn-out, MLP-up, the LM head and row_prep launch early (their weight
  // streams / launch latency overlap the kernels before them; LM head: -2.7 us per step at B=1).
  // MLP-down launches early only on the 3-stage W8A16 plans (INT8 at B <= 2: GPT-J B=1 1.775 ->
  // 1.748 ms); elsewhere its early CTAs steal SM slots from MLP-up (int8 B=16 2.62 -> 2.79 ms).
  // Attention early measured slower everywhere (tools/mask_sweep.sh, profiles/r2_pdl_mask_sweep.log).
  int mask = [this] {
    const char* v = std::getenv("DSINF_PDL_MASK");
    if (v) return static_cast<int>(std::strtol(v, nullptr, 0));
    // small fp16 layers (h < 4096, TP = 1, B <= 8: GPT-2 1.5B) leave room for early MLP-down and
    // attention CTAs: B=1 1.642 -> 1.593 ms, B=8 1.843 -> 1.796 (profiles/r2_gpt2_sweep.log)
    const bool small16 = !m.int8 && m.h < 4096 && m.t == 1 && m.B <= 8;
    // INT8 at B > 8 (W8A16 since the tuning pass): attention early too (GPT-J B=16 2.502 -> 2.476 ms)
    const bool i8big = m.int8 && m.B > 8 && m.t == 1;
    return 0xad | (m.a16g(3) && m.B <= 2 ? 0x10 : 0) | (small16 ? 0x12 : 0) | (i8big ? 0x02 : 0) |
           (m.attn_late ? 0x12 : 0);
  }();
  bool P(int bit) const { return pdl && ((mask >> bit) & 1); }

  int64_t pdl_launches = 0;
  int gemm_index = 0;

  // DSINF_LAUNCH_TRACE: per-launch [first CTA start, last CTA end] stamps, in launch order
  int slot = 0;
  unsigned long long* tslot(int kind) {
    if (!m.ltrace || slot >= ptx::kTraceEnd) return nullptr;
    if (static_cast<int>(m.ltrace_kinds.size()) <= slot) m.ltrace_kinds.resize(slot + 1);
    m.ltrace_kinds[slot] = kind;
    return m.ltrace + slot++;
  }

  // ---- fused all-reduce plumbing (m.fused_ar)
  struct RedIn {
    const float* slots = nullptr;
    int n = 0;
    long long stride = 0;
    const unsigned long long* flag = nullptr;
    unsigned long long per_step = 0;
  };
  static int64_t ctas(const gemm::Plan& pl) { return static_cast<int64_t>(pl.col_tiles) * pl.ksplit; }
  // consumer view of reduction point `pt` (0 attn-out, 1 MLP-down) of layer l on shard sh
  RedIn red_in(Shard& sh, int pt, int l) const {
    RedIn r;
    const long long bh = static_cast<long long>(m.B) * m.h;
    r.slots = sh.red + pt * m.t * bh;
    r.n = m.t;
    r.stride = bh;
    r.flag = sh.red_flag + pt * m.L + l;
    r.per_step = static_cast<unsigned long long>(m.t) * (m.far_last_cta ? 1 : ctas(pt == 0 ? sh.plan_o : sh.plan_down));
    return r;
  }
  void use_red(gemm::Params& p, const RedIn& r) const {
    p.res_delta = r.slots;
    p.delta_slots = r.n;
    p.delta_stride = r.stride;
    p.red_flag = r.flag;
    p.step_ctr = m.step_ctr;
    p.red_per_step = r.per_step;
  }
  // producer side: this shard's partial into every rank's slot `rank` of point pt, layer l
  void push_to_all(Shard& sh, gemm::Params& p, int pt, int l) const {
    const long long bh = static_cast<long long>(m.B) * m.h;
    p.epi = gemm::EPI_F32;
    p.bias = nullptr;
    p.push_n = m.t;
    p.push_gpu_scope = m.far_gpu_scope ? 1 : 0;
    if (m.far_last_cta) {
      p.push_done = sh.push_done + pt * m.L + l;
      p.push_step = m.step_ctr;
      p.push_ctas = static_cast<unsigned long long>(ctas(pt == 0 ? sh.plan_o : sh.plan_down));
    }
    for (int q = 0; q < m.t; ++q) {
      p.push_dst[q] = sh.peer_red[q] + (pt * m.t + sh.rank) * bh;
      p.push_flag[q] = sh.peer_flag[q] + pt * m.L + l;
    }
  }

  void prep(Shard& sh, int mode, const float* res, const long long* stats, const float* delta, const __half* dbias,
            float* res_out, const __half* g, const __half* b, const __half* x, int x_ld, const unsigned* amax, int K,
            bool to_int8, const RedIn* red = nullptr) {
    ops::PrepParams pp{};
    if (red) {
      delta = red->slots;
      pp.delta_slots = red->n;
      pp.delta_stride = red->stride;
      pp.red_flag = red->flag;
      pp.step_ctr = m.step_ctr;
      pp.red_per_step = red->per_step;
    }
    pp.mode = mode;
    pp.res = res;
    pp.ln_stats = stats;
    pp.res_delta = delta;
    pp.delta_bias = dbias;
    pp.res_out = res_out;
    pp.ln_g = g;
    pp.ln_b = b;
    pp.eps = m.rt.ln_eps;
    pp.x = x;
    pp.x_ld = x_ld;
    pp.amax = amax;
    pp.out = to_int8 ? static_cast<void*>(sh.xq) : static_cast<void*>(sh.xn);
    pp.out_scale = sh.xsc;
    pp.B = m.B;
    pp.K = K;
    pp.trace = tslot(DSINF_LK_PREP);
    ops::row_prep(pp, s, P(7));
    ++launches;
  }

  // LayerNorm GEMM x via row_prep (x-streaming plan): fp16 xn, or int8 xq + scales
  void ln_x(Shard& sh, gemm::Params& p, const float* res, const long long* stats, const float* delta,
            const __half* dbias, float* res_out, const __half* g, const __half* b, bool int8_w,
            const RedIn* red = nullptr) {
    const int h = static_cast<int>(m.h);
    prep(sh, int8_w ? ops::PREP_LN_I8 : ops::PREP_LN_F16, res, stats, delta, dbias, res_out, g, b, nullptr, 0, nullptr,
         h, int8_w, red);
    p.pro = int8_w ? gemm::PRO_I8 : gemm::PRO_F16;
    p.x = int8_w ? static_cast<const void*>(sh.xq) : static_cast<const void*>(sh.xn);
    p.x_ld = h;
    p.x_scale = sh.xsc;
  }

  long long* lnslot(Shard& sh, int i) const { return sh.lnstats ? sh.lnstats + static_cast<int64_t>(i) * gemm::kLnSlotWords : nullptr; }
  unsigned* amslot(Shard& sh, int i) const { return sh.amax ? sh.amax + static_cast<int64_t>(i) * gemm::kAmaxSlotWords : nullptr; }

  void gemm_launch(const gemm::Params& p_in, const gemm::Plan& plan, bool int8_w, int bit, bool force_pdl = false) {
    gemm::Params p = p_in;
    p.trace = tslot(bit == 0 ? DSINF_LK_QKV : bit == 2 ? DSINF_LK_O : bit == 3 ? DSINF_LK_UP : bit == 4 ? DSINF_LK_DOWN
                                                                                                  : DSINF_LK_LM);
    if (m.cta_log && gemm_index++ == m.cta_log_launch) p.cta_log = m.cta_log;
    const bool pl = P(bit) || (force_pdl && pdl);
    pdl_launches += pl;
    gemm::launch(p, plan, int8_w, s, pl);
    ++launches;
  }

  void k1_qkv(Shard& sh, int l) {
    const LayerW& w = sh.layers[l];
    const int N = static_cast<int>(3 * m.Hl * m.d);
    gemm::Params p = base_params(m, w.wqkv, w.sqkv, N, static_cast<int>(m.h), m.int8, w.gqkv);
    if (m.ln_use(0)) {  // the residual streamed and LayerNorm'd per stage (Deep-Fusion region 1)
      p.pro = gemm::PRO_LN;
      p.res_in = sh.res[0];
      p.ln_stats_in = lnslot(sh, 2 * l);
      p.ln_g = w.ln1g;
      p.ln_b = w.ln1b;
    } else if (m.xs_ln) {
      RedIn red;  // fused all-reduce: row_prep sums the ranks' MLP-down slots of layer l - 1
      const bool use_slots = m.fused_ar && l > 0;
      if (use_slots) red = red_in(sh, 1, l - 1);
      ln_x(sh, p, sh.res[0], lnslot(sh, 2 * l), m.fuse_ln || l == 0 ? nullptr : sh.d_mlp,
           m.fuse_ln || l == 0 ? nullptr : sh.layers[l - 1].bdown, m.fuse_ln ? nullptr : sh.res[1], w.ln1g, w.ln1b,
           m.q8g(0), use_slots ? &red : nullptr);
    } else {
      p.pro = gemm::PRO_LN;
      p.res_in = sh.res[0];
      if (m.fuse_ln) {
        p.ln_stats_in = lnslot(sh, 2 * l);
      } else {
        p.res_delta = l > 0 ? sh.d_mlp : nullptr;
        p.delta_bias = l > 0 ? sh.layers[l - 1].bdown : nullptr;
        if (m.fused_ar && l > 0) use_red(p, red_in(sh, 1, l - 1));
        p.res_out = sh.res[1];
      }
      p.ln_g = w.ln1g;
      p.ln_b = w.ln1b;
    }
    p.epi = gemm::EPI_QKV;
    p.bias = w.bqkv;
    p.q_out = sh.q;
    const size_t layer_kv = static_cast<size_t>(m.B) * m.Hl * m.max_ctx * m.d;
    p.k_cache = sh.kc + l * layer_kv;
    p.v_cache = sh.vc + l * layer_kv;
    p.rope = m.rope;
    p.pos = m.pos;
    p.heads = static_cast<int>(m.Hl);
    p.head_dim = static_cast<int>(m.d);
    p.max_seq = m.max_ctx;
    if (m.attn_fuse) {  // the attention of every head runs in the tail of the cluster completing it
      p.attn_tail = 1;
      p.head_ctr = sh.head_ctr + static_cast<int64_t>(l) * m.Hl;
      p.attn_out = sh.a;
      p.attn_amax = amslot(sh, 2 * l);
      p.attn_scale = 1.0f / std::sqrt(static_cast<float>(m.d));
    }
    gemm_launch(p, sh.plan_qkv, m.int8, 0);
  }

  void k2_attn(Shard& sh, int l) {
    if (m.attn_fuse) return;  // ran in the QKV launch's tail
    ops::AttnParams a{};
    const size_t layer_kv = static_cast<size_t>(m.B) * m.Hl * m.max_ctx * m.d;
    a.q = sh.q;
    a.kc = sh.kc + l * layer_kv;
    a.vc = sh.vc + l * layer_kv;
    a.pos = m.pos;
    a.out = sh.a;
    a.B = m.B;
    a.H = static_cast<int>(m.Hl);
    a.d = static_cast<int>(m.d);
    a.max_seq = m.max_ctx;
    a.scale = 1.0f / std::sqrt(static_cast<float>(m.d));
    a.amax_out = amslot(sh, 2 * l);
    a.trace = tslot(DSINF_LK_ATTN);
    a.late_trigger = m.attn_late ? 1 : 0;
    ops::attention(a, m.attn_chunks, s, P(1));
    ++launches;
  }

  void k3_attn_out(Shard& sh, int l) {
    const LayerW& w = sh.layers[l];
    gemm::Params p = base_params(m, w.wo, w.so, static_cast<int>(m.h), static_cast<int>(m.Hl * m.d), m.int8, w.go);
    p.pro = m.q8g(1) ? gemm::PRO_QUANT : gemm::PRO_F16;
    p.x = sh.a;
    p.x_ld = static_cast<int>(m.Hl * m.d);
    p.amax_in = amslot(sh, 2 * l);
    if (m.xs_od && m.q8g(1)) {  // quantise once (row max from attention), then stream int8 x
      prep(sh, ops::PREP_QUANT_I8, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sh.a, p.x_ld,
           amslot(sh, 2 * l), p.x_ld, true);
      p.pro = gemm::PRO_I8;
      p.x = sh.xq;
      p.x_scale = sh.xsc;
    }
    if (m.fuse_ln) {  // residual += attn-out + bias; emits LN2's row sums
      p.epi = gemm::EPI_RESID;
      p.out = sh.res[0];
      p.bias = w.bo;
      p.ln_stats_out = lnslot(sh, 2 * l + 1);
    } else {
      p.epi = gemm::EPI_F32;
      p.out = sh.d_attn;
      if (m.fused_ar) push_to_all(sh, p, 0, l);
    }
    gemm_launch(p, sh.plan_o, m.int8, 2);
  }

  void k4_up(Shard& sh, int l) {
    const LayerW& w = sh.layers[l];
    gemm::Params p = base_params(m, w.wup, w.sup, static_cast<int>(m.Fl), static_cast<int>(m.h), m.int8, w.gup);
    if (m.ln_use(2)) {  // Deep-Fusion region 3: LayerNorm per streamed stage, no row_prep
      p.pro = gemm::PRO_LN;
      p.res_in = sh.res[0];
      p.ln_stats_in = lnslot(sh, 2 * l + 1);
      p.ln_g = w.ln2g;
      p.ln_b = w.ln2b;
    } else if (m.xs_ln) {
      if (m.fuse_ln)
        ln_x(sh, p, sh.res[0], lnslot(sh, 2 * l + 1), nullptr, nullptr, nullptr, w.ln2g, w.ln2b, m.q8g(2));
      else if (m.fused_ar) {
        RedIn red = red_in(sh, 0, l);  // row_prep sums the ranks' attn-out slots
        ln_x(sh, p, sh.res[1], nullptr, sh.d_attn, w.bo, sh.res[0], w.ln2g, w.ln2b, m.q8g(2), &red);
      } else {
        ln_x(sh, p, sh.res[1], nullptr, sh.d_attn, w.bo, sh.res[0], w.ln2g, w.ln2b, m.q8g(2));
      }
    } else {
      p.pro = gemm::PRO_LN;
      if (m.fuse_ln) {
        p.res_in = sh.res[0];
        p.ln_stats_in = lnslot(sh, 2 * l + 1);
      } else {
        p.res_in = sh.res[1];
        p.res_delta = sh.d_attn;
        p.delta_bias = w.bo;
        if (m.fused_ar) use_red(p, red_in(sh, 0, l));
        p.res_out = sh.res[0];
      }
      p.ln_g = w.ln2g;
      p.ln_b = w.ln2b;
    }
    p.epi = gemm::EPI_GELU_F16;
    p.bias = w.bup;
    p.out = sh.u;
    p.out_flags = w.up_flags;
    p.amax_out = amslot(sh, 2 * l + 1);
    gemm_launch(p, sh.plan_up, m.int8, 3);
  }

  void k5_down(Shard& sh, int l) {
    const LayerW& w = sh.layers[l];
    gemm::Params p = base_params(m, w.wdown, w.sdown, static_cast<int>(m.h), static_cast<int>(m.Fl), m.int8, w.gdown);
    p.pro = m.q8g(3) ? gemm::PRO_QUANT : gemm::PRO_F16;
    p.x = sh.u;
    p.x_ld = static_cast<int>(m.Fl);
    p.amax_in = amslot(sh, 2 * l + 1);
    if (m.xs_od && m.q8g(3)) {
      prep(sh, ops::PREP_QUANT_I8, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sh.u, p.x_ld,
           amslot(sh, 2 * l + 1), p.x_ld, true);
      p.pro = gemm::PRO_I8;
      p.x = sh.xq;
      p.x_scale = sh.xsc;
    }
    if (m.fuse_ln) {  // residual += mlp-down + bias; emits the next LayerNorm's row sums
      p.epi = gemm::EPI_RESID;
      p.out = sh.res[0];
      p.bias = w.bdown;
      p.ln_stats_out = lnslot(sh, 2 * l + 2);
    } else {
      p.epi = gemm::EPI_F32;
      p.out = sh.d_mlp;
      if (m.fused_ar) push_to_all(sh, p, 1, l);
    }
    if (w.up_flags != nullptr) {
      p.dep_flags = w.up_flags;
      p.dep_per_step = static_cast<unsigned>(sh.plan_up.ksplit);
      p.dep_step = m.step_ctr;
      gemm_launch(p, sh.plan_down, m.int8, 4, /*force_pdl=*/true);
    } else {
      gemm_launch(p, sh.plan_down, m.int8, 4);
    }
  }

  // complete_res: res[0] already holds the final residual (prefill); else the decode step's last
  // MLP-down partial and bias are folded in here when the statistics are not fused (TP > 1).
  void lm_head(Shard& sh, bool complete_res = false) {
    gemm::Params p = base_params(m, sh.wlm, nullptr, static_cast<int>(m.Vl), static_cast<int>(m.h), false);
    const bool fold = !m.fuse_ln && !complete_res && m.L > 0;
    RedIn red;
    const bool fold_red = fold && m.fused_ar;
    if (fold_red) red = red_in(sh, 1, static_cast<int>(m.L) - 1);
    if (m.ln_stream && m.xs_lm) {
      p.pro = gemm::PRO_LN;
      p.res_in = sh.res[0];
      p.ln_stats_in = lnslot(sh, 2 * static_cast<int>(m.L));
      p.ln_g = sh.lnfg;
      p.ln_b = sh.lnfb;
    } else if (m.xs_lm) {
      ln_x(sh, p, sh.res[0], m.fuse_ln ? lnslot(sh, 2 * static_cast<int>(m.L)) : nullptr, fold ? sh.d_mlp : nullptr,
           fold ? sh.layers[m.L - 1].bdown : nullptr, nullptr, sh.lnfg, sh.lnfb, false, fold_red ? &red : nullptr);
    } else {
      p.pro = gemm::PRO_LN;
      p.res_in = sh.res[0];
      if (m.fuse_ln) {
        p.ln_stats_in = lnslot(sh, 2 * static_cast<int>(m.L));
      } else if (fold) {
        p.res_delta = m.L > 0 ? sh.d_mlp : nullptr;
        p.delta_bias = m.L > 0 ? sh.layers[m.L - 1].bdown : nullptr;
        if (fold_red) use_red(p, red);
      }
      p.res_out = nullptr;
      p.ln_g = sh.lnfg;
      p.ln_b = sh.lnfb;
    }
    p.epi = gemm::EPI_F32;
    p.out = sh.logits;
    // greedy argmax fused into the epilogue: one key per (shard, row), ties -> lowest index
    const int64_t first = sh.rank * m.Vl;
    p.am_out = m.am_key + sh.rank * m.B;
    p.am_valid = static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(m.Vl, m.V - first)));
    p.am_offset = first;
    gemm_launch(p, sh.plan_lm, false, 5);
  }

  // Sum of the t partials of `which` (0 = d_attn, 1 = d_mlp).
  void allreduce(int which) {
    // fused: pushed by the GEMM epilogues, summed by the consumers; slice: no peers to sum with
    if (m.t == 1 || m.fused_ar || m.rt.tp_mode == DSINF_TP_SLICE) return;
    const int64_t count = static_cast<int64_t>(m.B) * m.h;
    if (m.rt.tp_mode == DSINF_TP_NCCL) {
      Shard& sh = m.shards[0];
      nccl::allreduce_sum_f32(which == 0 ? sh.d_attn : sh.d_mlp, count, m.comm, s);
    } else {
      ops::LocalReduceParams p{};
      p.shards = m.t;
      p.count = count;
      for (int i = 0; i < m.t; ++i) p.buf[i] = which == 0 ? m.shards[i].d_attn : m.shards[i].d_mlp;
      ops::local_allreduce(p, s, P(6));
      ++launches;
    }
  }

  // Prompt prefill (large-batch regime, TP = 1): every layer over all B x P prompt tokens with
  // the tcgen05 GEMMs, then the decode path's LM head / argmax / select on the last token.
  void prefill(int P) {
    const int M = m.B * P;
    const int h = static_cast<int>(m.h), Hd = static_cast<int>(m.Hl * m.d), Fl = static_cast<int>(m.Fl);
    const bool i8 = m.int8;
    const int eb = i8 ? 1 : 2;
    const bool tp = m.t > 1;  // row-parallel GEMMs produce partials: all-reduce, then residual add
    for (Shard& sh : m.shards) {
      ops::PrefillEmbedParams pe{};
      pe.wte = sh.wte;
      pe.prompt = m.prompt;
      pe.prompt_ld = m.prompt_cap;
      pe.P = P;
      pe.hist = m.hist;
      pe.max_ctx = m.max_ctx;
      pe.res = sh.pf.res;
      pe.B = m.B;
      pe.h = h;
      pe.V = static_cast<int>(m.V);
      ops::prefill_embed(pe, s);
      ++launches;
    }
    const bool pf_pdl = std::getenv("DSINF_PREFILL_NOPDL") == nullptr;
    auto ln = [&](Shard& sh, const __half* g, const __half* b) {  // LayerNorm rows -> GEMM-ready x
      ops::PrepParams pp{};
      pp.mode = i8 ? ops::PREP_LN_I8 : ops::PREP_LN_F16;
      pp.res = sh.pf.res;
      pp.ln_g = g;
      pp.ln_b = b;
      pp.eps = m.rt.ln_eps;
      pp.out = i8 ? static_cast<void*>(sh.pf.xq) : static_cast<void*>(sh.pf.xn);
      pp.out_scale = sh.pf.xs;
      pp.B = M;
      pp.K = h;
      ops::row_prep(pp, s, pf_pdl);
      ++launches;
    };
    auto quant = [&](Shard& sh, const __half* x, int K) {  // int8: per-row quantisation of an fp16 activation
      ops::PrepParams pp{};
      pp.mode = ops::PREP_QUANT_I8;
      pp.x = x;
      pp.x_ld = K;
      pp.out = sh.pf.xq;
      pp.out_scale = sh.pf.xs;
      pp.B = M;
      pp.K = K;
      ops::row_prep(pp, s, pf_pdl);
      ++launches;
    };
    auto gemm = [&](Shard& sh, tc::Params& p, const void* x, const void* w, const float* ws, int N, int K) {
      p.M = M;
      p.N = N;
      p.K = K;
      tc::make_maps(p, x, K * eb, w, K * eb, eb);
      p.x_scale = sh.pf.xs;
      p.w_scale = ws;
      // split-K (one row tile) launches under PDL: the weight ring fills during the previous kernel's
      // tail, except when this layer's row-major weights were just rewritten by the repack
      p.w_early = sh.rm_per_layer ? 0 : 1;
      tc::launch(p, i8, s, pf_pdl);
      ++launches;
    };
    // row-parallel output: t == 1 -> residual += y + bias in the epilogue; t > 1 -> partial, all-reduce,
    // then residual += (sum + bias) (the decode path's order)
    auto row_parallel = [&](Shard& sh, tc::Params& p, const __half* bias) {
      if (tp) {
        p.epi = tc::EPI_F32;
        p.out = sh.pf.part;
      } else {
        p.epi = tc::EPI_RESID;
        p.bias = bias;
        p.out = sh.pf.res;
      }
      p.out_ld = h;
    };
    auto reduce_add = [&](auto bias_of) {
      if (!tp) return;
      const int64_t count = static_cast<int64_t>(M) * h;
      if (m.rt.tp_mode == DSINF_TP_NCCL) {
        nccl::allreduce_sum_f32(m.shards[0].pf.part, count, m.comm, s);
      } else if (m.rt.tp_mode == DSINF_TP_LOCAL) {
        ops::LocalReduceParams lr{};
        lr.shards = m.t;
        lr.count = count;
        for (int i = 0; i < m.t; ++i) lr.buf[i] = m.shards[i].pf.part;
        ops::local_allreduce(lr, s, false);
        ++launches;
      }
      for (Shard& sh : m.shards) {
        ops::prefill_residual_add(sh.pf.res, sh.pf.part, bias_of(sh), count, h, s);
        ++launches;
      }
    };
    const size_t layer_kv = static_cast<size_t>(m.B) * m.Hl * m.max_ctx * m.d;
    for (int l = 0; l < m.L; ++l) {
      for (Shard& sh : m.shards) {
        if (!sh.rm_per_layer) continue;
        const LayerW& w = sh.layers[l];
        const int64_t pm = m.int8 ? 4 : 2, h64 = m.h;
        auto unbias = [&](int g) { return m.a16g(g) ? 0x80808080u : 0u; };  // W8A16 weights are stored biased
        ops::packed_to_rowmajor(w.wqkv, h64 / pm, 3 * m.Hl * m.d, static_cast<uint32_t*>(w.rqkv), s, unbias(0));
        ops::packed_to_rowmajor(w.wo, m.Hl * m.d / pm, h64, static_cast<uint32_t*>(w.ro), s, unbias(1));
        ops::packed_to_rowmajor(w.wup, h64 / pm, m.Fl, static_cast<uint32_t*>(w.rup), s, unbias(2));
        ops::packed_to_rowmajor(w.wdown, m.Fl / pm, h64, static_cast<uint32_t*>(w.rdown), s, unbias(3));
        launches += 4;
      }
      for (Shard& sh : m.shards) {
        const LayerW& w = sh.layers[l];
        PrefillBufs& pf = sh.pf;
        ln(sh, w.ln1g, w.ln1b);
        tc::Params q{};
        q.epi = tc::EPI_QKV;
        q.bias = w.bqkv;
        q.q_out = pf.q;
        q.k_cache = sh.kc + l * layer_kv;
        q.v_cache = sh.vc + l * layer_kv;
        q.rope = m.rope;
        q.seq_len = P;
        q.pos0 = 0;
        q.heads = static_cast<int>(m.Hl);
        q.head_dim = static_cast<int>(m.d);
        q.max_seq = m.max_ctx;
        gemm(sh, q, i8 ? static_cast<const void*>(pf.xq) : pf.xn, w.rqkv, w.sqkv, 3 * Hd, h);
        ops::PrefillAttnParams a{};
        a.q = pf.q;
        a.kc = q.k_cache;
        a.vc = q.v_cache;
        a.out = pf.a;
        a.B = m.B;
        a.P = P;
        a.H = static_cast<int>(m.Hl);
        a.d = static_cast<int>(m.d);
        a.max_seq = m.max_ctx;
        a.scale = 1.0f / std::sqrt(static_cast<float>(m.d));
        ops::prefill_attention(a, s);
        ++launches;
        if (i8) quant(sh, pf.a, Hd);
        tc::Params o{};
        row_parallel(sh, o, w.bo);
        gemm(sh, o, i8 ? static_cast<const void*>(pf.xq) : pf.a, w.ro, w.so, h, Hd);
      }
      reduce_add([&](Shard& sh) { return sh.layers[l].bo; });
      for (Shard& sh : m.shards) {
        const LayerW& w = sh.layers[l];
        PrefillBufs& pf = sh.pf;
        ln(sh, w.ln2g, w.ln2b);
        tc::Params u{};
        u.epi = tc::EPI_GELU_F16;
        u.bias = w.bup;
        u.out = pf.u;
        u.out_ld = Fl;
        gemm(sh, u, i8 ? static_cast<const void*>(pf.xq) : pf.xn, w.rup, w.sup, Fl, h);
        if (i8) quant(sh, pf.u, Fl);
        tc::Params dn{};
        row_parallel(sh, dn, w.bdown);
        gemm(sh, dn, i8 ? static_cast<const void*>(pf.xq) : pf.u, w.rdown, w.sdown, h, Fl);
      }
      reduce_add([&](Shard& sh) { return sh.layers[l].bdown; });
    }
    // last prompt token of every sequence -> the decode state, then LM head (+ fused argmax) / select
    DSINF_CUDA_CHECK(cudaMemsetAsync(m.am_key, 0, sizeof(unsigned long long) * m.t * m.B, s));
    for (Shard& sh : m.shards) {
      long long* lslot = lnslot(sh, 2 * static_cast<int>(m.L));
      if (lslot) DSINF_CUDA_CHECK(cudaMemsetAsync(lslot, 0, gemm::kLnSlotWords * sizeof(long long), s));
      ops::PrefillGatherParams g{};
      g.res_rows = sh.pf.res;
      g.P = P;
      g.res = sh.res[0];
      g.ln_stats = lslot;
      g.pos = m.pos;
      g.B = m.B;
      g.h = h;
      ops::prefill_gather(g, s);
      ++launches;
      lm_head(sh, /*complete_res=*/true);
    }
    if (m.t > 1 && m.rt.tp_mode == DSINF_TP_NCCL)
      nccl::allgather_bytes(m.am_key + m.shards[0].rank * m.B, m.am_key, m.B * sizeof(unsigned long long), m.comm, s);
    ops::SelectParams sp{};
    const bool slice = m.rt.tp_mode == DSINF_TP_SLICE;  // only this rank's vocab slice has a key
    sp.keys = slice ? m.am_key + m.shards[0].rank * m.B : m.am_key;
    sp.shards = slice ? 1 : m.t;
    sp.B = m.B;
    sp.next_tok = m.next_tok;
    sp.pos = m.pos;
    sp.hist = m.hist;
    sp.max_ctx = m.max_ctx;
    ops::select_token(sp, s, false);
    ++launches;
  }

  void step() {
    if (m.step_prog.ready()) {  // TP = 1: the whole step is one persistent kernel
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.am_key, 0, sizeof(unsigned long long) * m.B, s));
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.shards[0].lnstats, 0,
                                       (2 * m.L + 1) * gemm::kLnSlotWords * sizeof(long long), s));
      m.step_prog.launch(s);
      ++launches;
      return;
    }
    if (m.ltrace) {
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.ltrace, 0xff, ptx::kTraceEnd * sizeof(unsigned long long), s));
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.ltrace + ptx::kTraceEnd, 0, ptx::kTraceEnd * sizeof(unsigned long long), s));
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.ltrace + 2 * ptx::kTraceEnd, 0xff, ptx::kTraceEnd * sizeof(unsigned long long), s));
      DSINF_CUDA_CHECK(cudaMemsetAsync(m.ltrace + 3 * ptx::kTraceEnd, 0, (ptx::kTracePhases - 3) * ptx::kTraceEnd * sizeof(unsigned long long), s));
    }
    DSINF_CUDA_CHECK(cudaMemsetAsync(m.am_key, 0, sizeof(unsigned long long) * m.t * m.B, s));
    for (Shard& sh : m.shards) {  // per-step statistics slots
      if (sh.lnstats)
        DSINF_CUDA_CHECK(cudaMemsetAsync(sh.lnstats, 0, (2 * m.L + 1) * gemm::kLnSlotWords * sizeof(long long), s));
      if (sh.amax)
        DSINF_CUDA_CHECK(cudaMemsetAsync(sh.amax, 0, std::max<int64_t>(1, 2 * m.L) * gemm::kAmaxSlotWords * sizeof(unsigned), s));
    }
    for (Shard& sh : m.shards) {
      ops::EmbedParams e{};
      e.wte = sh.wte;
      e.prompt = m.prompt;
      e.prompt_len = m.prompt_len;
      e.prompt_ld = m.prompt_cap;
      e.next_tok = m.next_tok;
      e.pos = m.pos;
      e.hist = m.hist;
      e.max_ctx = m.max_ctx;
      e.res = sh.res[0];
      e.B = m.B;
      e.h = static_cast<int>(m.h);
      e.V = static_cast<int>(m.V);
      e.ln_stats_out = lnslot(sh, 0);
      e.trace = tslot(DSINF_LK_EMBED);
      ops::embed(e, s, P(6));
      ++launches;
    }
    for (int l = 0; l < m.L; ++l) {
      for (Shard& sh : m.shards) {
        k1_qkv(sh, l);
        k2_attn(sh, l);
        k3_attn_out(sh, l);
      }
      allreduce(0);
      for (Shard& sh : m.shards) {
        k4_up(sh, l);
        k5_down(sh, l);
      }
      allreduce(1);
    }
    for (Shard& sh : m.shards) lm_head(sh);
    if (m.t > 1 && m.rt.tp_mode == DSINF_TP_NCCL) {
      // gather every rank's (value, index) pair; slots are laid out [rank][B]
      nccl::allgather_bytes(m.am_key + m.shards[0].rank * m.B, m.am_key, m.B * sizeof(unsigned long long), m.comm, s);
    }
    ops::SelectParams sp{};
    const bool slice = m.rt.tp_mode == DSINF_TP_SLICE;  // only this rank's vocab slice has a key
    sp.keys = slice ? m.am_key + m.shards[0].rank * m.B : m.am_key;
    sp.shards = slice ? 1 : m.t;
    sp.B = m.B;
    sp.next_tok = m.next_tok;
    sp.pos = m.pos;
    sp.hist = m.hist;
    sp.max_ctx = m.max_ctx;
    sp.step_ctr = m.step_ctr;
    if (m.rt.tp_mode == DSINF_TP_IPC && m.t > 1) {
      sp.ipc_t = m.t;
      sp.ipc_rank = m.shards[0].rank;
      for (int q = 0; q < m.t; ++q) {
        sp.ipc_keys[q] = m.peer_keys[q];
        sp.ipc_flag[q] = m.peer_key_flag[q];
      }
    }
    ops::select_token(sp, s, P(6));
    ++launches;
    m.ltrace_n = slot;
  }
};

// Fused all-reduce peers: on-device shards directly; across processes (NCCL mode, one shard per
// rank) every rank exports CUDA-IPC handles of its slot and counter allocations, the handles are
// all-gathered over the NCCL communicator, and each rank maps its peers' allocations (NVLink P2P).
void map_reduction_peers(Model& m, cudaStream_t s) {
  if (m.rt.tp_mode == DSINF_TP_SLICE) {  // every "peer" is this rank's own slot set
    Shard& sh = m.shards[0];
    sh.peer_red.assign(m.t, sh.red);
    sh.peer_flag.assign(m.t, sh.red_flag);
    return;
  }
  if (m.rt.tp_mode != DSINF_TP_NCCL) {
    for (Shard& sh : m.shards) {
      sh.peer_red.clear();
      sh.peer_flag.clear();
      for (Shard& q : m.shards) {
        sh.peer_red.push_back(q.red);
        sh.peer_flag.push_back(q.red_flag);
      }
    }
    return;
  }
  Shard& sh = m.shards[0];
  struct Handles {
    cudaIpcMemHandle_t red, flag;
  };
  Handles mine{};
  DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&mine.red, sh.red));
  DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&mine.flag, sh.red_flag));
  const size_t hb = sizeof(Handles);
  uint8_t* dev = static_cast<uint8_t*>(m.alloc(hb * (m.t + 1)));
  DSINF_CUDA_CHECK(cudaMemcpyAsync(dev + hb * m.t, &mine, hb, cudaMemcpyHostToDevice, s));
  nccl::allgather_bytes(dev + hb * m.t, dev, hb, m.comm, s);
  std::vector<Handles> all(m.t);
  DSINF_CUDA_CHECK(cudaMemcpyAsync(all.data(), dev, hb * m.t, cudaMemcpyDeviceToHost, s));
  DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
  sh.peer_red.assign(m.t, nullptr);
  sh.peer_flag.assign(m.t, nullptr);
  for (int q = 0; q < m.t; ++q) {
    if (q == sh.rank) {
      sh.peer_red[q] = sh.red;
      sh.peer_flag[q] = sh.red_flag;
      continue;
    }
    void* pr = nullptr;
    void* pf = nullptr;
    DSINF_CUDA_CHECK(cudaIpcOpenMemHandle(&pr, all[q].red, cudaIpcMemLazyEnablePeerAccess));
    DSINF_CUDA_CHECK(cudaIpcOpenMemHandle(&pf, all[q].flag, cudaIpcMemLazyEnablePeerAccess));
    sh.peer_red[q] = static_cast<float*>(pr);
    sh.peer_flag[q] = static_cast<unsigned long long*>(pf);
    m.ipc_maps.push_back(pr);
    m.ipc_maps.push_back(pf);
  }
}

// true iff every rank of `comm` passes true (a sum all-reduce of one flag, synchronous).
bool nccl_vote_all(nccl::Comm comm, bool mine, int t) {
  float* d = nullptr;
  DSINF_CUDA_CHECK(cudaMalloc(&d, sizeof(float)));
  const float v = mine ? 1.f : 0.f;
  float all = 0.f;
  DSINF_CUDA_CHECK(cudaMemcpy(d, &v, sizeof(float), cudaMemcpyHostToDevice));
  nccl::allreduce_sum_f32(d, 1, comm, nullptr);
  DSINF_CUDA_CHECK(cudaMemcpy(&all, d, sizeof(float), cudaMemcpyDeviceToHost));
  DSINF_CUDA_CHECK(cudaFree(d));
  return all == static_cast<float>(t);
}

void validate_configs(const dsinf_model_config& c, const dsinf_runtime_config& r) {
  require(c.hidden_dim > 0 && c.num_layers >= 0 && c.num_heads > 0 && c.vocab_size > 0, "bad model dims");
  require(c.hidden_dim % c.num_heads == 0, "hidden_dim must be divisible by num_heads");
  require(c.dtype_bytes == 1 || c.dtype_bytes == 2, "dtype_bytes must be 2 (fp16) or 1 (int8)");
  require(r.batch >= 1 && r.batch <= gemm::kMaxB, "batch must be in [1, 16]");
  require(r.tp_size >= 1 && r.tp_size <= 8, "tp_size must be in [1, 8]");
  require(c.num_heads % r.tp_size == 0, "num_heads must be divisible by tp_size");
  require((4 * c.hidden_dim) % r.tp_size == 0, "4*hidden must be divisible by tp_size");
  require(c.hidden_dim % 8 == 0, "hidden_dim must be a multiple of 8");
  require((c.hidden_dim / c.num_heads) % 2 == 0, "head dim must be even (rotary pairs)");
  require(r.max_ctx >= 1 && r.max_ctx <= c.max_seq, "max_ctx must be in [1, max_seq]");
  if (r.tp_size > 1)
    require(r.tp_mode == DSINF_TP_NCCL || r.tp_mode == DSINF_TP_LOCAL || r.tp_mode == DSINF_TP_SLICE ||
                r.tp_mode == DSINF_TP_IPC,
            "tp_size > 1 needs a TP mode");
  if (r.tp_mode == DSINF_TP_NCCL || r.tp_mode == DSINF_TP_SLICE || r.tp_mode == DSINF_TP_IPC)
    require(r.tp_rank >= 0 && r.tp_rank < r.tp_size, "bad tp_rank");
  if (r.tp_mode == DSINF_TP_IPC) require(r.use_step_kernel == 0, "the persistent step kernel is TP = 1 only");
  require(r.int8_group == 0 || r.int8_group == 128, "int8_group must be 0 (row scales) or 128");
  if (r.int8_group != 0) {
    require(c.dtype_bytes == 1, "int8_group needs int8 weights (dtype_bytes 1)");
    require(r.use_step_kernel == 0, "int8_group: the persistent step kernel takes row scales only");
  }
}

void build_rope(Model& m, cudaStream_t s) {
  const int64_t half = m.d / 2;
  std::vector<float2> tab(static_cast<size_t>(m.max_ctx) * half);
  for (int64_t p = 0; p < m.max_ctx; ++p)
    for (int64_t i = 0; i < half; ++i) {
      const double inv = std::pow(static_cast<double>(m.rt.rope_base), -2.0 * static_cast<double>(i) / static_cast<double>(m.d));
      const double ang = static_cast<double>(p) * inv;
      tab[p * half + i] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
  m.rope = m.alloc_n<float2>(tab.size());
  DSINF_CUDA_CHECK(cudaMemcpyAsync(m.rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice, s));
}

void require_ipc_ready(const Model& m) {
  require(m.rt.tp_mode != DSINF_TP_IPC || m.t == 1 || m.ipc_ready,
          "DSINF_TP_IPC: call dsinf_model_ipc_attach with every rank's handles before decoding");
}

void enqueue_eager(Model& m, cudaStream_t s) {
  require_ipc_ready(m);
  Enqueuer e{m, s, m.rt.use_pdl != 0};
  e.step();
  m.kernels_per_step = e.launches;
}

void ensure_graph(Model& m) {
  if (m.exec) return;
  require_ipc_ready(m);
  DSINF_CUDA_CHECK(cudaStreamBeginCapture(m.cap_stream, cudaStreamCaptureModeThreadLocal));
  Enqueuer e{m, m.cap_stream, m.rt.use_pdl != 0};
  try {
    e.step();
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(m.cap_stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  DSINF_CUDA_CHECK(cudaStreamEndCapture(m.cap_stream, &m.graph));
  DSINF_CUDA_CHECK(cudaGraphInstantiate(&m.exec, m.graph, 0));
  if (std::getenv("DSINF_DEBUG")) fprintf(stderr, "[dsinf] captured %lld launches, %lld gemm launches with PDL (mask 0x%x, pdl %d)\n", (long long)e.launches, (long long)e.pdl_launches, e.mask, (int)e.pdl);
  m.kernels_per_step = e.launches;
}

}  // namespace
}  // namespace dsinf

using namespace dsinf;

extern "C" {

int dsinf_model_create(const dsinf_model_config* cfg, const dsinf_runtime_config* rt, void* nccl_comm,
                       dsinf_model** out) {
  return guarded([&] {
    require(cfg && rt && out, "null argument");
    validate_configs(*cfg, *rt);
    auto m = std::make_unique<dsinf_model>();
    m->cfg = *cfg;
    m->rt = *rt;
    if (m->rt.ln_eps <= 0.f) m->rt.ln_eps = 1e-5f;
    if (m->rt.rope_base <= 0.f) m->rt.rope_base = 10000.f;
    DSINF_CUDA_CHECK(cudaSetDevice(rt->device));
    gemm::configure();
    ops::configure();
    m->h = cfg->hidden_dim;
    m->L = cfg->num_layers;
    m->H = cfg->num_heads;
    m->d = m->h / m->H;
    m->t = rt->tp_size;
    m->Hl = m->H / m->t;
    m->V = cfg->vocab_size;
    const int64_t vq = 128LL * m->t;
    m->Vpad = (m->V + vq - 1) / vq * vq;
    m->Vl = m->Vpad / m->t;
    m->F = 4 * m->h;
    m->Fl = m->F / m->t;
    m->B = rt->batch;
    m->max_ctx = static_cast<int>(rt->max_ctx);
    m->int8 = cfg->dtype_bytes == 1;
    require(rt->int8_act == DSINF_INT8_W8A8 || rt->int8_act == DSINF_INT8_W8A16 || rt->int8_act == DSINF_INT8_AUTO,
            "unknown int8_act");
    // INT8 activation mode per GEMM (mask): W8A8 everywhere, W8A16 everywhere, or AUTO -- measured
    // on B200 with the x-streaming plans: W8A16 everywhere up to B = 8 (GPT-J B=8 2.40 -> 2.20 ms);
    // at B = 16 W8A8 QKV + W8A16 attn-out / MLP at TP = 1 (GPT-J 2.62 -> 2.55, GPT-2 2.44 -> 2.35),
    // W8A8 everywhere at TP > 1 (175B t=8 rank 8.04 vs 8.23, NeoX t=2 3.84 vs 4.05).
    // DSINF_A16_MASK overrides for experiments.
    if (m->int8) {
      if (rt->int8_act == DSINF_INT8_W8A16) m->a16_mask = 0xf;
      else if (rt->int8_act == DSINF_INT8_AUTO) m->a16_mask = rt->batch <= 8 || m->t == 1 ? 0xf : 0x0;  // W8A16 QKV at B=16 with 3 stages: 2.587 -> 2.508 ms
      if (const char* am = std::getenv("DSINF_A16_MASK")) m->a16_mask = static_cast<int>(std::strtol(am, nullptr, 0)) & 0xf;
    }
    m->a16 = m->a16_mask != 0;
    if (m->int8 && rt->int8_group != 0)  // K-group scales are dequantised by the W8A16 main loop
      require(m->a16_mask == 0xf, "int8_group: every decode GEMM must be W8A16 (int8_act W8A16, or AUTO at batch <= 8)");
    if (rt->use_step_kernel && m->int8) {  // the persistent step kernel runs INT8 weight-only
      require(rt->int8_act != DSINF_INT8_W8A8, "the persistent step kernel runs INT8 as W8A16 (weight-only)");
      m->a16_mask = 0xf;
      m->a16 = true;
    }
    m->attn_chunks = ops::attention_chunks(m->B, static_cast<int>(m->Hl));
    {
      const char* fs = std::getenv("DSINF_FUSE_STATS");
      m->fuse_ln = m->t == 1 && (fs == nullptr || std::atoi(fs) != 0);
      // x-streaming plans need 16-byte rows of GEMM-ready x
      const int64_t Fl = 4 * m->h / m->t, Ol = m->h / m->t;
      const bool rows16 = m->q8() ? (m->h % 16 == 0 && Fl % 16 == 0 && Ol % 16 == 0) : (Ol % 8 == 0 && Fl % 8 == 0);
      // a fused all-reduce request (below) selects the slice plan: its slots are summed by the
      // per-CTA LayerNorm prologues
      const char* far_req = std::getenv("DSINF_FUSED_AR");
      // (TP_SLICE: the rank's pushes all land in its own slots and it is its own only signaller -- a
      // timing model of the fused all-reduce's per-rank cost without the NVLink hop)
      bool want_far = m->t > 1 &&
                      (rt->tp_mode == DSINF_TP_LOCAL || rt->tp_mode == DSINF_TP_NCCL || rt->tp_mode == DSINF_TP_SLICE) &&
                      far_req != nullptr && std::atoi(far_req) != 0;
      if (rt->tp_mode == DSINF_TP_IPC && m->t > 1) want_far = true;  // the only exchange IPC mode has
      if (rt->tp_mode == DSINF_TP_NCCL && m->t > 1) {
        // the request is per process (environment) but every rank must pick the same plan, or one
        // rank waits on slot counters the others never bump: fused only if all t ranks ask for it
        require(nccl_comm != nullptr, "NCCL mode needs a communicator");
        want_far = nccl_vote_all(static_cast<nccl::Comm>(nccl_comm), want_far, m->t);
      }
      // the fused all-reduce runs on either plan: row_prep (x-streaming) or the per-CTA LayerNorm
      // prologues (slice plan) sum the ranks' slots
      m->xs_ln = rows16 && gemm::prefer_x_stream(m->B, m->t > 1);
      const char* od = std::getenv("DSINF_XS_OD");
      const int od_v = od ? std::atoi(od) : -1;
      m->xs_od = rows16 && (m->q8() ? (od_v < 0 ? m->xs_ln : od_v != 0) : (od_v < 0 ? true : od_v != 0));
      const char* lm = std::getenv("DSINF_XS_LM");
      m->xs_lm = m->h % 8 == 0 && (lm ? std::atoi(lm) != 0 : true);
      // default by batch (GPT-J, ms/token without -> with): fp16 B=1 2.678 -> 2.571, B=4 2.789 -> 2.647,
      // B=8 2.893 -> 2.804, B=16 3.155 -> 3.496 (every column tile re-normalises the fp32 rows);
      // W8A16 B=1 1.976 -> 1.910, B=4 2.083 -> 2.092, B=8 2.220 -> 2.417 (its consumers are the busier);
      // GPT-2 B=1 fp16 1.797 -> 1.649, int8 1.658 -> 1.521.  DSINF_LN_STREAM=0/1 forces it.
      const char* lsv = std::getenv("DSINF_LN_STREAM");
      const char* dfv = std::getenv("DSINF_DOWN_FLAGS");
      m->down_flags = m->t == 1 && m->xs_od && !m->q8g(3) && dfv != nullptr && std::atoi(dfv) != 0;
      const bool ls_default = m->int8 ? m->B <= 2 : m->B <= 8;
      m->ln_stream = m->fuse_ln && m->xs_ln && m->h % 8 == 0 && (lsv ? std::atoi(lsv) != 0 : ls_default);
      m->attn_late = m->t == 1 && (m->int8 ? m->h < 4096 : m->h <= 4096);
      {
        const char* afv = std::getenv("DSINF_ATTN_FUSE");
        const char* amb = std::getenv("DSINF_ATTN_FUSE_MAXB");
        const int maxb = amb ? std::atoi(amb) : 8;
        m->attn_fuse = m->ln_stream && !m->q8g(0) && rt->int8_group == 0 && !rt->use_step_kernel && m->B <= maxb &&
                       m->d % 8 == 0 && m->d <= 256 && (m->int8 ? m->a16g(0) : true) &&
                       afv != nullptr && std::atoi(afv) != 0;  // opt-in: measured slower (DESIGN 3.2)
      }
      // fused all-reduce: on-device shards (DSINF_TP_LOCAL) or CUDA-IPC peer mappings across
      // processes; the per-CTA LayerNorm prologue path (slice plan) consumes the slots, the row_prep
      // path handles the LM head.  Opt-in (DSINF_FUSED_AR=1): on one device the explicit local reduction is cheaper (every
      // consumer CTA re-reads t slots), the win is hiding the NVLink exchange across GPUs
      m->fused_ar = want_far && !m->fuse_ln;
      {
        const char* fsys = std::getenv("DSINF_FAR_SYS");
        const char* flast = std::getenv("DSINF_FAR_LASTCTA");
        m->far_gpu_scope = (rt->tp_mode == DSINF_TP_LOCAL || rt->tp_mode == DSINF_TP_SLICE) &&
                           !(fsys != nullptr && std::atoi(fsys) != 0);
        m->far_last_cta = m->fused_ar && !m->far_gpu_scope && (flast == nullptr || std::atoi(flast) != 0);
      }
    }
    if (rt->tp_mode == DSINF_TP_NCCL && m->t > 1) {
      require(nccl_comm != nullptr, "NCCL mode needs a communicator");
      m->comm = static_cast<nccl::Comm>(nccl_comm);
    }
    DSINF_CUDA_CHECK(cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking));
    cudaStream_t s = m->cap_stream;
    const int nshards = (rt->tp_mode == DSINF_TP_LOCAL) ? m->t : 1;
    m->shards.resize(nshards);
    for (int i = 0; i < nshards; ++i) m->shards[i].rank = (rt->tp_mode == DSINF_TP_LOCAL) ? i : rt->tp_rank;
    build_rope(*m, s);
    m->prompt_cap = m->max_ctx;
    m->prompt = m->alloc_n<int32_t>(static_cast<int64_t>(m->B) * m->prompt_cap);
    m->next_tok = m->alloc_n<int32_t>(m->B);
    m->hist = m->alloc_n<int32_t>(static_cast<int64_t>(m->B) * m->max_ctx);
    m->pos = m->alloc_n<int>(1);
    m->step_ctr = m->alloc_n<long long>(1);
    DSINF_CUDA_CHECK(cudaMemsetAsync(m->step_ctr, 0, sizeof(long long), s));
    m->am_val = m->alloc_n<float>(static_cast<int64_t>(m->t) * m->B);
    m->am_idx = m->alloc_n<int32_t>(static_cast<int64_t>(m->t) * m->B);
    m->am_key = m->alloc_n<unsigned long long>(static_cast<int64_t>(m->t) * m->B);
    DSINF_CUDA_CHECK(cudaMemsetAsync(m->prompt, 0, sizeof(int32_t) * m->B * m->prompt_cap, s));
    DSINF_CUDA_CHECK(cudaMemsetAsync(m->next_tok, 0, sizeof(int32_t) * m->B, s));
    DSINF_CUDA_CHECK(cudaMemsetAsync(m->hist, 0, sizeof(int32_t) * m->B * m->max_ctx, s));
    DSINF_CUDA_CHECK(cudaMemsetAsync(m->pos, 0, sizeof(int), s));
    for (auto& sh : m->shards) build_shard(*m, sh, s);
    DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
    if (rt->tp_mode == DSINF_TP_IPC && m->t > 1) {
      require(m->fused_ar, "DSINF_TP_IPC needs the fused all-reduce (slice plan)");
      m->key_flag = m->alloc_n<unsigned long long>(1);
      DSINF_CUDA_CHECK(cudaMemset(m->key_flag, 0, sizeof(unsigned long long)));
    } else if (m->fused_ar) {
      map_reduction_peers(*m, s);
    }
    if (m->t == 1 && rt->use_step_kernel) build_step_program(*m);
    if (const char* cl = std::getenv("DSINF_CTA_LOG")) {
      m->cta_log_launch = std::atoi(cl);
      DSINF_CUDA_CHECK(cudaMallocManaged(&m->cta_log, 6 * 4096 * sizeof(unsigned long long)));
    }
    if (const char* lt = std::getenv("DSINF_LAUNCH_TRACE"); lt && std::atoi(lt) != 0)
      m->ltrace = m->alloc_n<unsigned long long>(ptx::kTracePhases * ptx::kTraceEnd);
    *out = m.release();
  });
}

int dsinf_model_destroy(dsinf_model* m) {
  return guarded([&] { delete m; });
}

static void set_prompt_common(dsinf_model* m, const int32_t* src, int64_t prompt_len, bool host, cudaStream_t s) {
  require(m != nullptr, "null model");
  require(prompt_len >= 0 && prompt_len <= m->prompt_cap, "prompt_len exceeds the KV-cache capacity");
  const size_t bytes = sizeof(int32_t) * m->B * prompt_len;
  if (prompt_len > 0) {
    require(src != nullptr, "null prompt");
    DSINF_CUDA_CHECK(cudaMemcpy2DAsync(m->prompt, sizeof(int32_t) * m->prompt_cap, src, sizeof(int32_t) * prompt_len,
                                       sizeof(int32_t) * prompt_len, m->B,
                                       host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  }
  (void)bytes;
  m->prompt_len = static_cast<int>(prompt_len);
  if (m->step_prog.ready()) m->step_prog.set_embed(embed_params(*m, m->shards[0]));
  DSINF_CUDA_CHECK(cudaMemsetAsync(m->pos, 0, sizeof(int), s));
  DSINF_CUDA_CHECK(cudaMemsetAsync(m->next_tok, 0, sizeof(int32_t) * m->B, s));
  m->host_pos = 0;
  // prompt_len is a kernel argument: re-capture the step graph
  if (m->exec) {
    cudaGraphExecDestroy(m->exec);
    m->exec = nullptr;
  }
  if (m->graph) {
    cudaGraphDestroy(m->graph);
    m->graph = nullptr;
  }
}

namespace {
struct IpcBlob {
  uint32_t magic, rank, t, pad;
  cudaIpcMemHandle_t red, flag, keys, key_flag;
};
constexpr uint32_t kIpcMagic = 0x64736970u;  // "dsip"
}  // namespace

int dsinf_model_ipc_handle(dsinf_model* m, void* out, int64_t cap, int64_t* len) {
  return guarded([&] {
    require(m != nullptr && len != nullptr, "null argument");
    require(m->rt.tp_mode == DSINF_TP_IPC && m->t > 1, "dsinf_model_ipc_handle: model is not in DSINF_TP_IPC mode");
    *len = static_cast<int64_t>(sizeof(IpcBlob));
    if (out == nullptr) return;
    require(cap >= static_cast<int64_t>(sizeof(IpcBlob)), "dsinf_model_ipc_handle: buffer too small");
    const dsinf::Shard& sh = m->shards[0];
    IpcBlob b{};
    b.magic = kIpcMagic;
    b.rank = static_cast<uint32_t>(sh.rank);
    b.t = static_cast<uint32_t>(m->t);
    DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&b.red, sh.red));
    DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&b.flag, sh.red_flag));
    DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&b.keys, m->am_key));
    DSINF_CUDA_CHECK(cudaIpcGetMemHandle(&b.key_flag, m->key_flag));
    std::memcpy(out, &b, sizeof(b));
  });
}

int dsinf_model_ipc_attach(dsinf_model* m, const void* all, int64_t len) {
  return guarded([&] {
    require(m != nullptr && all != nullptr, "null argument");
    require(m->rt.tp_mode == DSINF_TP_IPC && m->t > 1, "dsinf_model_ipc_attach: model is not in DSINF_TP_IPC mode");
    require(!m->ipc_ready, "dsinf_model_ipc_attach: already attached");
    require(len == static_cast<int64_t>(sizeof(IpcBlob)) * m->t, "dsinf_model_ipc_attach: expected t handle blobs");
    dsinf::Shard& sh = m->shards[0];
    const auto* blobs = static_cast<const IpcBlob*>(all);
    sh.peer_red.assign(m->t, nullptr);
    sh.peer_flag.assign(m->t, nullptr);
    m->peer_keys.assign(m->t, nullptr);
    m->peer_key_flag.assign(m->t, nullptr);
    for (int q = 0; q < m->t; ++q) {
      IpcBlob b;
      std::memcpy(&b, blobs + q, sizeof(b));
      require(b.magic == kIpcMagic && b.rank == static_cast<uint32_t>(q) && b.t == static_cast<uint32_t>(m->t),
              "dsinf_model_ipc_attach: blobs must be every rank's dsinf_model_ipc_handle, in rank order");
      if (q == sh.rank) {
        sh.peer_red[q] = sh.red;
        sh.peer_flag[q] = sh.red_flag;
        m->peer_keys[q] = m->am_key;
        m->peer_key_flag[q] = m->key_flag;
        continue;
      }
      void* p[4] = {nullptr, nullptr, nullptr, nullptr};
      const cudaIpcMemHandle_t* hs[4] = {&b.red, &b.flag, &b.keys, &b.key_flag};
      for (int i = 0; i < 4; ++i) {
        DSINF_CUDA_CHECK(cudaIpcOpenMemHandle(&p[i], *hs[i], cudaIpcMemLazyEnablePeerAccess));
        m->ipc_maps.push_back(p[i]);
      }
      sh.peer_red[q] = static_cast<float*>(p[0]);
      sh.peer_flag[q] = static_cast<unsigned long long*>(p[1]);
      m->peer_keys[q] = static_cast<unsigned long long*>(p[2]);
      m->peer_key_flag[q] = static_cast<unsigned long long*>(p[3]);
    }
    m->ipc_ready = true;
  });
}

int dsinf_model_set_prompt(dsinf_model* m, const int32_t* prompt_host, int64_t prompt_len, void* stream) {
  return guarded([&] { set_prompt_common(m, prompt_host, prompt_len, true, static_cast<cudaStream_t>(stream)); });
}

int dsinf_model_set_prompt_device(dsinf_model* m, const int32_t* prompt_dev, int64_t prompt_len, void* stream) {
  return guarded([&] { set_prompt_common(m, prompt_dev, prompt_len, false, static_cast<cudaStream_t>(stream)); });
}

int dsinf_model_prefill(dsinf_model* m, void* stream) {
  return guarded([&] {
    require(m != nullptr, "null model");
    require(m->prompt_len >= 1, "prefill needs a prompt (dsinf_model_set_prompt)");
    require(m->host_pos == 0, "prefill must start at position 0 (call dsinf_model_set_prompt first)");
    require(m->rt.tp_mode != DSINF_TP_IPC || m->t == 1,
            "prefill: DSINF_TP_IPC has no all-reduce for the large-batch GEMMs (use decode steps)");
    require(m->rt.int8_group == 0, "prefill: the tensor-core prefill takes per-row INT8 scales (int8_group = 0)");
    require(m->d % 32 == 0 && m->d <= 256, "prefill attention needs head_dim % 32 == 0 and <= 256");
    require(m->h % 16 == 0 && (m->Hl * m->d) % 16 == 0 && m->Fl % 16 == 0,
            "prefill needs 16-byte TMA rows (hidden, per-rank head and MLP widths % 16 == 0)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    tc::configure();
    ops::configure_prefill();
    for (Shard& sh : m->shards) {
      if (!sh.rm_ready) build_rowmajor(*m, sh, s);
      ensure_prefill_bufs(*m, sh, static_cast<int64_t>(m->B) * m->prompt_len);
    }
    Enqueuer e{*m, s, m->rt.use_pdl != 0};
    e.prefill(m->prompt_len);
    m->host_pos = m->prompt_len;
  });
}

int dsinf_decode_step(dsinf_model* m, void* stream) { return dsinf_decode_steps(m, 1, stream); }

int dsinf_decode_steps(dsinf_model* m, int64_t steps, void* stream) {
  return guarded([&] {
    require(m != nullptr, "null model");
    require(steps >= 0, "negative step count");
    if (m->host_pos + steps > m->max_ctx)
      throw InfeasibleError("decode would run past the KV-cache capacity (max_ctx)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (m->rt.use_cuda_graph) {
      ensure_graph(*m);
      for (int64_t i = 0; i < steps; ++i) DSINF_CUDA_CHECK(cudaGraphLaunch(m->exec, s));
    } else {
      for (int64_t i = 0; i < steps; ++i) enqueue_eager(*m, s);
    }
    m->host_pos += steps;
  });
}

int dsinf_decode_step_host(dsinf_model* m, const int32_t* tokens_in, int32_t* tokens_out, void* stream) {
  return guarded([&] {
    require(m && tokens_in && tokens_out, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DSINF_CUDA_CHECK(cudaMemcpyAsync(m->next_tok, tokens_in, sizeof(int32_t) * m->B, cudaMemcpyHostToDevice, s));
    const int rc = dsinf_decode_steps(m, 1, stream);
    if (rc == DSINF_ERR_INFEASIBLE) throw InfeasibleError(dsinf_last_error());
    if (rc == DSINF_ERR_CONFIG) throw ConfigError(dsinf_last_error());
    if (rc != DSINF_OK) throw CudaError(dsinf_last_error());
    DSINF_CUDA_CHECK(cudaMemcpyAsync(tokens_out, m->next_tok, sizeof(int32_t) * m->B, cudaMemcpyDeviceToHost, s));
    DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int dsinf_model_step_trace(dsinf_model* m, uint64_t* out, int64_t len, int64_t* needed, int32_t* grid,
                           int32_t* phases) {
  return guarded([&] {
    require(m != nullptr, "null model");
    require(m->step_prog.ready(), "the persistent step kernel is not in use");
    const size_t n = m->step_prog.trace(nullptr, 0);
    require(n > 0, "step trace disabled (set DSINF_STEP_TRACE=1 before model creation)");
    if (needed) *needed = static_cast<int64_t>(n);
    if (grid) *grid = m->step_prog.grid();
    if (phases) *phases = m->step_prog.phases();
    if (out) m->step_prog.trace(reinterpret_cast<unsigned long long*>(out), static_cast<size_t>(len));
  });
}

int dsinf_model_set_launch_trace(dsinf_model* m, int on) {
  return guarded([&] {
    require(m != nullptr, "null model");
    if (on && !m->ltrace) m->ltrace = m->alloc_n<unsigned long long>(ptx::kTracePhases * ptx::kTraceEnd);
    if (!on) m->ltrace = nullptr;  // the buffer stays owned by the model until destroy
    m->ltrace_n = 0;
    if (m->exec) {  // launch parameters changed: re-capture the step graph
      cudaGraphExecDestroy(m->exec);
      m->exec = nullptr;
    }
    if (m->graph) {
      cudaGraphDestroy(m->graph);
      m->graph = nullptr;
    }
  });
}

int dsinf_model_launch_trace(dsinf_model* m, uint64_t* out, int64_t len, int64_t* launches) {
  return guarded([&] {
    require(m != nullptr, "null model");
    require(m->ltrace != nullptr, "launch trace disabled (set DSINF_LAUNCH_TRACE=1 before model creation)");
    if (launches) *launches = m->ltrace_n;
    if (out) {
      require(len >= 3 * m->ltrace_n, "trace buffer too small");
      std::vector<unsigned long long> st(m->ltrace_n), en(m->ltrace_n);
      DSINF_CUDA_CHECK(cudaDeviceSynchronize());
      DSINF_CUDA_CHECK(cudaMemcpy(st.data(), m->ltrace, m->ltrace_n * 8, cudaMemcpyDeviceToHost));
      DSINF_CUDA_CHECK(cudaMemcpy(en.data(), m->ltrace + ptx::kTraceEnd, m->ltrace_n * 8, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < m->ltrace_n; ++i) {
        out[3 * i] = st[i];
        out[3 * i + 1] = en[i];
        out[3 * i + 2] = i < static_cast<int64_t>(m->ltrace_kinds.size()) ? m->ltrace_kinds[i] : ~0ull;
      }
    }
  });
}

int dsinf_model_launch_phases(dsinf_model* m, uint64_t* out, int64_t len) {
  return guarded([&] {
    require(m != nullptr, "null model");
    require(m->ltrace != nullptr, "launch trace disabled");
    require(out != nullptr && len >= 8 * m->ltrace_n, "phase buffer too small");
    std::vector<unsigned long long> ph(8 * ptx::kTraceEnd);
    DSINF_CUDA_CHECK(cudaDeviceSynchronize());
    DSINF_CUDA_CHECK(cudaMemcpy(ph.data(), m->ltrace + 2 * ptx::kTraceEnd, ph.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < m->ltrace_n; ++i)
      for (int j = 0; j < 8; ++j) out[8 * i + j] = ph[j * ptx::kTraceEnd + i];
  });
}

int dsinf_model_cta_log(dsinf_model* m, uint64_t* out, int64_t len) {
  return guarded([&] {
    require(m != nullptr && m->cta_log != nullptr, "cta log disabled (set DSINF_CTA_LOG=<launch> before model creation)");
    DSINF_CUDA_CHECK(cudaDeviceSynchronize());
    for (int64_t i = 0; i < std::min<int64_t>(len, 6 * 4096); ++i) out[i] = m->cta_log[i];
  });
}

int dsinf_model_outputs(dsinf_model* m, float** logits, int64_t* logits_ld, int32_t** next_tokens, int32_t** history,
                        int32_t** pos) {
  return guarded([&] {
    require(m != nullptr, "null model");
    if (logits) *logits = m->shards[0].logits;
    if (logits_ld) *logits_ld = m->Vl;
    if (next_tokens) *next_tokens = m->next_tok;
    if (history) *history = m->hist;
    if (pos) *pos = m->pos;
  });
}

int dsinf_model_read_logits(dsinf_model* m, float* host, int64_t len, void* stream) {
  return guarded([&] {
    require(m && host, "null argument");
    const int64_t per = static_cast<int64_t>(m->B) * m->Vl;
    require(len == per * static_cast<int64_t>(m->shards.size()), "logits buffer must be shards*B*vocab_local");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (size_t i = 0; i < m->shards.size(); ++i)
      DSINF_CUDA_CHECK(cudaMemcpyAsync(host + i * per, m->shards[i].logits, per * 4, cudaMemcpyDeviceToHost, s));
    DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int dsinf_model_read_tokens(dsinf_model* m, int32_t* next_host, int32_t* history_host, int64_t history_len,
                            void* stream) {
  return guarded([&] {
    require(m != nullptr, "null model");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (next_host) DSINF_CUDA_CHECK(cudaMemcpyAsync(next_host, m->next_tok, 4 * m->B, cudaMemcpyDeviceToHost, s));
    if (history_host) {
      require(history_len == static_cast<int64_t>(m->B) * m->max_ctx, "history buffer must be B*max_ctx");
      DSINF_CUDA_CHECK(cudaMemcpyAsync(history_host, m->hist, 4 * history_len, cudaMemcpyDeviceToHost, s));
    }
    DSINF_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int64_t dsinf_model_bytes_per_step(const dsinf_model* m, int64_t pos) {
  if (!m) return -1;
  const int64_t ctx = pos + 1;
  const int64_t kv_read = 2LL * m->B * ctx * m->Hl * m->d * 2;
  const int64_t kv_write = 2LL * m->B * m->Hl * m->d * 2;
  const int64_t per_shard = m->weight_bytes / static_cast<int64_t>(m->shards.size()) + m->L * (kv_read + kv_write) +
                            static_cast<int64_t>(m->B) * m->h * 2;
  return per_shard * static_cast<int64_t>(m->shards.size());
}

int dsinf_model_get_info(const dsinf_model* m, dsinf_model_info* out) {
  return guarded([&] {
    require(m && out, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->weight_bytes = m->weight_bytes;
    out->bytes_per_token = dsinf_model_bytes_per_step(m, m->host_pos);
    out->kernels_per_step = m->kernels_per_step;
    out->vocab_local = m->Vl;
    out->heads_local = m->Hl;
    out->kv_bytes = 2LL * m->L * m->B * m->Hl * m->max_ctx * m->d * 2 * static_cast<int64_t>(m->shards.size());
    out->shards = static_cast<int32_t>(m->shards.size());
    out->graph_ready = m->exec != nullptr;
    out->fused_allreduce = m->fused_ar ? 1 : 0;
    out->plan_flags = (m->xs_ln ? DSINF_PLAN_X_STREAM : 0) | (m->fuse_ln ? DSINF_PLAN_FUSED_STATS : 0) |
                      (m->step_prog.ready() ? DSINF_PLAN_STEP_KERNEL : 0);
  });
}

int dsinf_synthetic_tensor(uint64_t seed, int32_t layer, int32_t tensor, int64_t rows, int64_t cols,
                           float* out) {
  return guarded([&] {
    require(out != nullptr && rows >= 0 && cols >= 0, "bad arguments");
    float offset = 0.f;
    const float amp = tensor_amp(tensor, &offset);
    const uint64_t base = synth_base(seed, layer, tensor);
    for (int64_t i = 0; i < rows * cols; ++i) {
      const float t = synth_unit(base, static_cast<uint64_t>(i)) * amp;
      out[i] = f16_bits_to_f32(f32_to_f16_bits(offset + t));
    }
  });
}

int dsinf_shard_tensor(const dsinf_model_config* cfg, int32_t tp, int32_t rank, int32_t layer, int32_t tensor,
                       uint64_t seed, float* out, int64_t out_len, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    require(cfg != nullptr, "null config");
    require(tp >= 1 && rank >= 0 && rank < tp, "bad tp rank");
    require(cfg->num_heads % tp == 0 && cfg->hidden_dim % cfg->num_heads == 0, "heads must divide by tp");
    require(tensor >= DSINF_T_QKV && tensor <= DSINF_T_LNF_B, "unknown tensor id");
    const ops::ShardMap mp =
        tensor_map(cfg->hidden_dim, cfg->num_heads, cfg->vocab_size, tp, rank, seed, layer, tensor);
    if (rows) *rows = mp.N_local;
    if (cols) *cols = mp.K_local;
    if (!out) return;  // size query
    require(out_len == mp.N_local * mp.K_local, "output buffer size mismatch");
    float offset = 0.f;
    tensor_amp(tensor, &offset);
    const bool vector = mp.K_global == 1;
    for (int64_t n = 0; n < mp.N_local; ++n) {
      const int64_t grow = (n / mp.sec_local) * mp.sec_global + mp.row_off + (n % mp.sec_local);
      for (int64_t k = 0; k < mp.K_local; ++k) {
        const int64_t gcol = mp.col_off + k;
        float v = 0.f;
        if (grow < mp.valid_rows && gcol < mp.K_global) {
          const float t = synth_unit(mp.base, static_cast<uint64_t>(grow * mp.K_global + gcol)) * mp.amp;
          v = f16_bits_to_f32(f32_to_f16_bits(vector ? offset + t : t));
        }
        out[n * mp.K_local + k] = v;
      }
    }
  });
}

int dsinf_nccl_get_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    require(id_out != nullptr, "null id");
    nccl::UniqueId id;
    nccl::get_unique_id(&id);
    std::memcpy(id_out, id.internal, 128);
  });
}

int dsinf_nccl_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, void** comm_out) {
  return guarded([&] {
    require(id && comm_out, "null argument");
    DSINF_CUDA_CHECK(cudaSetDevice(device));
    nccl::UniqueId uid;
    std::memcpy(uid.internal, id, 128);
    *comm_out = nccl::init_rank(nranks, uid, rank);
  });
}

int dsinf_nccl_comm_destroy(void* comm) {
  return guarded([&] { nccl::destroy(static_cast<nccl::Comm>(comm)); });
}

int dsinf_nccl_window_check(void* comm, int64_t count, int32_t* symmetric, float* first_out) {
  return guarded([&] {
    require(comm && symmetric && first_out && count >= 1, "bad argument");
    const auto c = static_cast<nccl::Comm>(comm);
    *symmetric = nccl::has_windows() ? 1 : 0;
    void* buf = nullptr;
    nccl::Window w = nullptr;
    if (*symmetric) {
      buf = nccl::mem_alloc(static_cast<size_t>(count) * 4);
      w = nccl::window_register(c, buf, static_cast<size_t>(count) * 4);
    } else {
      DSINF_CUDA_CHECK(cudaMalloc(&buf, static_cast<size_t>(count) * 4));
    }
    std::vector<float> ones(static_cast<size_t>(count), 1.0f);
    DSINF_CUDA_CHECK(cudaMemcpy(buf, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice));
    nccl::allreduce_sum_f32(static_cast<float*>(buf), static_cast<size_t>(count), c, nullptr);
    DSINF_CUDA_CHECK(cudaMemcpy(first_out, buf, 4, cudaMemcpyDeviceToHost));
    if (*symmetric) {
      nccl::window_deregister(c, w);
      nccl::mem_free(buf);
    } else {
      cudaFree(buf);
    }
  });
}

}  // extern "C"
