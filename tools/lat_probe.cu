// Dependent-load latency right after griddepcontrol.wait, in a producer -> consumer kernel pair
// shaped like two consecutive decode GEMMs.
//   producer: 148*2 CTAs stream `stream_mb` of a big buffer (ld.global.cg, 16 B/lane), then write a
//             16 KB row (plain stores) and add into 16 stat words (red.add.u64).
//   consumer: launched with programmatic stream serialization; CTAs wait, then time (clock64) one
//             dependent load from the row / the stats / a never-written buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void producer(const int4* big, size_t n16, float* row, unsigned long long* stats, int do_atomics, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldcg(big + i);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
  if (blockIdx.x < 32) row[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (do_atomics && threadIdx.x < 2) atomicAdd(stats + (blockIdx.x % 8) * 2 + threadIdx.x, 1ull);
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void consumer(const float* row, const unsigned long long* stats, const float* cold, int which,
                         long long* lat, int pre_touch, const char* big, int pf_kb) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  long long dep = 0;
  if (pf_kb > 0 && threadIdx.x == 0) {  // TMA-style bulk prefetch into smem before the wait
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(pf_kb * 1024));
    for (int k = 0; k < pf_kb / 16; ++k) {
      const char* src = big + ((size_t)blockIdx.x * pf_kb + k * 16) * 1024 + (size_t)(which + 1) * (300u << 20);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(sm + k * 16384)),
                   "l"(src), "r"(b)
                   : "memory");
    }
  }
  if (pre_touch && threadIdx.x == 0) {  // touch the line before the wait (TLB / L2 warm)
    dep = (long long)__ldcg(row + blockIdx.x % 32) + (long long)__ldcg(stats) + (long long)__ldcg(cold + blockIdx.x);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x != 0) return;
  long long c0 = clock64();
  long long v;
  if (which == 0) v = (long long)__ldcg(row + blockIdx.x % 4096);
  else if (which == 1) v = (long long)__ldcg(stats + (blockIdx.x % 16));
  else v = (long long)__ldcg(cold + blockIdx.x * 32);
  long long c1 = 0;
  if (v + dep != 0x7fffffffffffll) c1 = clock64();  // the branch waits for the load
  lat[blockIdx.x] = c1 - c0;
  if (pf_kb > 0) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(b) : "memory");
  }
}

int main(int argc, char** argv) {
  const size_t big_bytes = (size_t)(argc > 1 ? atoi(argv[1]) : 1) << 30;
  int4* big; float* row; unsigned long long* stats; float* cold; long long* lat; int* sink;
  CK(cudaMalloc(&big, big_bytes));
  CK(cudaMemset(big, 1, big_bytes));
  CK(cudaMalloc(&row, 4096 * 4));
  CK(cudaMalloc(&stats, 16 * 8));
  CK(cudaMalloc(&cold, 1 << 20));
  CK(cudaMemset(cold, 0, 1 << 20));
  CK(cudaMalloc(&lat, 1024 * 8));
  CK(cudaMalloc(&sink, 4));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  const int cgrid = 192;
  const char* names[3] = {"row (plain stores)", "stats (atomics)", "never written"};
  CK(cudaFuncSetAttribute(consumer, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int mb : {64, 256}) {
    for (int pf : {0, 64}) {
      for (int pdl = 0; pdl < 2; ++pdl) {
        for (int which = 0; which < 3; ++which) {
          for (int pre = 0; pre < 1; ++pre) {
            const int atom = 1;
            std::vector<long long> all;
            for (int rep = 0; rep < 20; ++rep) {
              const size_t off16 = ((size_t)rep * 997 * (1 << 20) / 16) % (big_bytes / 16 - (size_t)mb * (1 << 20) / 16);
              producer<<<296, 512, 0, s>>>(big + off16, (size_t)mb * (1 << 20) / 16, row, stats, atom, sink);
              cudaLaunchConfig_t cfg{};
              cfg.gridDim = dim3(cgrid);
              cfg.blockDim = dim3(128);
              cfg.stream = s;
              cfg.dynamicSmemBytes = pf * 1024;
              cudaLaunchAttribute at;
              at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
              at.val.programmaticStreamSerializationAllowed = pdl;
              cfg.attrs = &at;
              cfg.numAttrs = 1;
              CK(cudaLaunchKernelEx(&cfg, consumer, (const float*)row, (const unsigned long long*)stats,
                                    (const float*)cold, which, lat, pre, (const char*)big, pf));
              CK(cudaStreamSynchronize(s));
              std::vector<long long> h(cgrid);
              CK(cudaMemcpy(h.data(), lat, cgrid * 8, cudaMemcpyDeviceToHost));
              if (rep >= 2) all.insert(all.end(), h.begin(), h.end());
            }
            std::sort(all.begin(), all.end());
            printf("stream %4d MB prefetch %3d KB/CTA pdl %d  %-20s  cycles p50 %6lld p90 %6lld max %6lld\n", mb, pf, pdl,
                   names[which], all[all.size() / 2], all[all.size() * 9 / 10], all.back());
          }
        }
      }
    }
  }
  return 0;
}
