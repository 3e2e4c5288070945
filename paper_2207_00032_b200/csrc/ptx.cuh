// Thin inline-PTX wrappers for sm_100a: mbarrier, bulk async copies (TMA 1-D), cluster
// distributed shared memory, programmatic dependent launch, warp-level MMA.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace dsinf {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe (try_wait may suspend the thread for a while when the phase is pending).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------- bulk async copy (TMA, 1-D)
// global -> shared::cta, completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 2-D tensor TMA: box at coordinates {c0 (inner), c1} of `map` -> smem, tx bytes on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst_smem, const void* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst_smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 2-D tensor box -> L2 only (no smem, no barrier): warms L2 ahead of the ring.
__device__ __forceinline__ void tma_prefetch_l2_2d(const void* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const void* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---------------------------------------------------------------- clusters / DSMEM
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive without release semantics (no fence over this thread's outstanding global stores).
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_shared_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float2 ld_dsmem_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ int2 ld_dsmem_i2(uint32_t addr) {
  int2 v;
  asm volatile("ld.shared::cluster.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
// No memory clobber: several of these may be in flight before the first result is used.
__device__ __forceinline__ uint2 ld_dsmem_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared::cluster.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 ld_dsmem_f2_nc(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ld_dsmem_f_nc(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ld_dsmem_f(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

// ---------------------------------------------------------------- cross-GPU flags (fused all-reduce)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Spin (one thread) until *flag >= (*step + 1) * per_step.
__device__ __forceinline__ void wait_flag(const unsigned long long* flag, const long long* step,
                                          unsigned long long per_step) {
  const unsigned long long target = (static_cast<unsigned long long>(*reinterpret_cast<const volatile long long*>(step)) + 1ull) * per_step;
  while (ld_acquire_sys(flag) < target) __nanosleep(32);
}

// ---------------------------------------------------------------- programmatic dependent launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- launch timeline (DSINF_LAUNCH_TRACE)
// slot[0] = earliest CTA start, slot[kTraceEnd] = latest CTA end of one launch (globaltimer ns).
constexpr int kTraceEnd = 1024;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_begin(unsigned long long* slot) {
  if (slot != nullptr && threadIdx.x == 0) atomicMin(slot, gtimer());
}
__device__ __forceinline__ void trace_end(unsigned long long* slot) {
  if (slot != nullptr && threadIdx.x == 0) atomicMax(slot + kTraceEnd, gtimer());
}
// Phase stamps of SBI-GeMM launches (compiled in with -DDSINF_DIAG, `make DIAG=1`) (thread `tid` of each CTA): slot[2 * kTraceEnd] = earliest
// dependency release (after griddepcontrol.wait), slot[3 * kTraceEnd] = latest prologue end,
// slot[4 * kTraceEnd] = latest main-loop end, slot[5 * kTraceEnd] = longest per-CTA prologue
// (own release -> own prologue end), slot[6 * kTraceEnd] = latest release.
constexpr int kTracePhases = 10;  // + slots 7..9: sub-phase probes (max over CTAs of t - own release)
__device__ __forceinline__ unsigned long long trace_release(unsigned long long* slot, int tid) {
  if (slot == nullptr || threadIdx.x != tid) return 0;
  const unsigned long long t = gtimer();
  atomicMin(slot + 2 * kTraceEnd, t);
  atomicMax(slot + 6 * kTraceEnd, t);
  return t;
}
// Sub-phase probe: max over CTAs of SM clock cycles since `c0` (clock64 at release), read after
// `dep` is available and after every earlier memory operation of the thread (memory clobber).
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}
__device__ __forceinline__ void trace_sub(unsigned long long* slot, int idx, int tid, long long c0, long long dep = 0) {
#ifndef DSINF_DIAG
  return;
#endif
  if (slot == nullptr || threadIdx.x != tid) return;
  long long c;
  asm volatile("{ .reg .u64 d; mov.u64 d, %1; mov.u64 %0, %%clock64; }" : "=l"(c) : "l"(dep) : "memory");
  atomicMax(slot + idx * kTraceEnd, static_cast<unsigned long long>(c - c0));
}
// Same, but the stamp is taken only once `v` has arrived (a branch on it stalls the warp).
__device__ __forceinline__ void trace_sub_after(unsigned long long* slot, int idx, int tid, long long c0, unsigned v) {
#ifndef DSINF_DIAG
  return;
#endif
  if (slot == nullptr || threadIdx.x != tid) return;
  long long c = 0;
  if (v != 0x7f7f7f7fu) c = clock64();
  atomicMax(slot + idx * kTraceEnd, static_cast<unsigned long long>(c - c0));
}
__device__ __forceinline__ void trace_prologue_end(unsigned long long* slot, int tid, unsigned long long t_rel) {
  if (slot == nullptr || threadIdx.x != tid) return;
  const unsigned long long t = gtimer();
  atomicMax(slot + 3 * kTraceEnd, t);
  atomicMax(slot + 5 * kTraceEnd, t - t_rel);
}
__device__ __forceinline__ void trace_phase_max(unsigned long long* slot, int idx, int tid) {
  if (slot != nullptr && threadIdx.x == tid) atomicMax(slot + idx * kTraceEnd, gtimer());
}

// ---------------------------------------------------------------- warp MMA (legacy tensor path)
// D(16x8,f32) += A(16x16,f16,row) * B(16x8,f16,col)
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D(16x8,s32) += A(16x32,s8,row) * B(32x8,s8,col)
__device__ __forceinline__ void mma_s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace ptx
}  // namespace dsinf
