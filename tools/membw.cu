// HBM read-streaming ceiling on this GPU: how fast can one kernel launch stream S bytes, and
// what is the fixed per-launch cost?  Two variants:
//   bulk : one elected thread per CTA issues cp.async.bulk (global -> smem) 16 KB chunks through
//          an mbarrier ring (the SBI-GeMM producer pattern without the MMA consumers);
//   ldg  : every thread issues 16-byte ld.global.nc loads, 8 in flight, summed to defeat DCE.
// Buffers rotate over > 2x L2 capacity so each launch reads from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/membw tools/membw.cu && build/membw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kChunk = 16384;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void bulk_kernel(const char* src, size_t bytes, int stages, unsigned long long* sink) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  char* buf = sm + 1024;
  const size_t chunks = bytes / kChunk;
  const size_t per = (chunks + gridDim.x - 1) / gridDim.x;
  const size_t c0 = blockIdx.x * per, c1 = c0 + per < chunks ? c0 + per : chunks;
  if (threadIdx.x != 0 || c0 >= c1) return;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  size_t issued = c0;
  for (int s = 0; s < stages && issued < c1; ++s, ++issued) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kChunk));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(buf + s * kChunk)), "l"(src + issued * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s])) : "memory");
  }
  unsigned long long acc = 0;
  for (size_t c = c0; c < c1; ++c) {
    const int s = (c - c0) % stages;
    const uint32_t par = ((c - c0) / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(par));
    acc += *reinterpret_cast<volatile int*>(buf + s * kChunk);
    if (issued < c1) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kChunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf + s * kChunk)), "l"(src + issued * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s])) : "memory");
      ++issued;
    }
  }
  if (acc == 0x1234567) *sink = acc;
}

template <int U>
__global__ void ldg_kernel(const int4* src, size_t n16, unsigned long long* sink) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int acc = 0;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc ^= src[i].x;
  if (acc == 0x1234567) *sink = acc;
}

// blocked variant: each CTA streams one contiguous range (like a GEMM tile's weight slab)
template <int U>
__global__ void ldg_blocked_kernel(const int4* src, size_t n16, unsigned long long* sink) {
  const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const size_t b0 = blockIdx.x * per, b1 = min(n16, b0 + per);
  int acc = 0;
  size_t i = b0 + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < b1; i += U * blockDim.x) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * blockDim.x));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < b1; i += blockDim.x) acc ^= src[i].x;
  if (acc == 0x1234567) *sink = acc;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t kRot = 768ull << 20;  // rotate through 768 MB so every launch misses L2
  char* pool;
  CK(cudaMalloc(&pool, kRot));
  CK(cudaMemset(pool, 1, kRot));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 13 * kChunk));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t sizes[] = {33554432ull, 100663296ull, 134217728ull};
  printf("sms=%d\n", sms);
  auto run = [&](const char* name, size_t bytes, int grid, auto&& launch_one) -> int {
    const int nbuf = static_cast<int>(kRot / bytes);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int it = 0; it < 40; ++it) launch_one(pool + (it % nbuf) * bytes);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0, s));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    const double us = best * 1e3 / 40;
    printf("%-28s bytes=%9zu grid=%5d  %7.2f us/launch  %7.1f GB/s\n", name, bytes, grid, us, bytes / us / 1e3);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    return 0;
  };
  for (size_t bytes : sizes) {
    for (int st : {4, 6, 8, 12}) {
      for (int cps : {1, 2}) {
        const int smem = 1024 + st * kChunk;
        if (cps * smem > 227 * 1024) continue;
        char name[64];
        snprintf(name, sizeof name, "bulk st=%d cta/sm=%d", st, cps);
        run(name, bytes, sms * cps, [&](const char* src) { bulk_kernel<<<sms * cps, 32, smem, s>>>(src, bytes, st, sink); });
      }
    }
    for (int mult : {2, 4, 8}) {
      char name[64];
      snprintf(name, sizeof name, "ldg U=4 grid=%dx", mult);
      run(name, bytes, sms * mult, [&](const char* src) { ldg_kernel<4><<<sms * mult, 512, 0, s>>>(reinterpret_cast<const int4*>(src), bytes / 16, sink); });
      snprintf(name, sizeof name, "ldg U=8 grid=%dx", mult);
      run(name, bytes, sms * mult, [&](const char* src) { ldg_kernel<8><<<sms * mult, 512, 0, s>>>(reinterpret_cast<const int4*>(src), bytes / 16, sink); });
      snprintf(name, sizeof name, "ldg-blocked U=8 grid=%dx", mult);
      run(name, bytes, sms * mult, [&](const char* src) { ldg_blocked_kernel<8><<<sms * mult, 256, 0, s>>>(reinterpret_cast<const int4*>(src), bytes / 16, sink); });
      snprintf(name, sizeof name, "ldg-blocked U=16 grid=%dx", mult);
      run(name, bytes, sms * mult, [&](const char* src) { ldg_blocked_kernel<16><<<sms * mult, 256, 0, s>>>(reinterpret_cast<const int4*>(src), bytes / 16, sink); });
    }
  }
  // bigger stage counts / chunk splits for the bulk path at the GEMM sizes
  return 0;
}
