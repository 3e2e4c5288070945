// NCCL loaded on first use with dlopen, so the library has no link-time NCCL dependency and
// shares whichever libnccl.so.2 the process already mapped (torch bundles one).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace dsinf {
namespace nccl {

typedef struct ncclComm* Comm;
constexpr int kUniqueIdBytes = 128;
struct UniqueId {
  char internal[kUniqueIdBytes];
};

// Values from nccl.h (ncclDataType_t / ncclRedOp_t).
constexpr int kUint8 = 1;
constexpr int kFloat32 = 7;
constexpr int kSum = 0;

void get_unique_id(UniqueId* id);
Comm init_rank(int nranks, const UniqueId& id, int rank);
void destroy(Comm c);
void allreduce_sum_f32(float* buf, size_t count, Comm c, cudaStream_t s);
void allgather_bytes(const void* send, void* recv, size_t bytes_per_rank, Comm c, cudaStream_t s);

// Symmetric memory (NCCL >= 2.27: ncclMemAlloc + ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)):
// the latency-bound per-layer all-reduce buffers registered as collective windows.  Optional symbols:
// has_windows() is false on an older libnccl, and callers keep plain cudaMalloc buffers.
typedef struct ncclWindow* Window;
constexpr int kWinCollSymmetric = 0x01;
bool has_windows();
void* mem_alloc(size_t bytes);
void mem_free(void* p);
Window window_register(Comm c, void* buf, size_t bytes);  // collective over the communicator
void window_deregister(Comm c, Window w);

}  // namespace nccl
}  // namespace dsinf
