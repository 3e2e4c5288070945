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

}  // namespace nccl
}  // namespace dsinf
