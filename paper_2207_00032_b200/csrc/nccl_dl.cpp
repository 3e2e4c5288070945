#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "common.h"

namespace dsinf {
namespace nccl {

namespace {

typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*CommDestroyFn)(Comm);
typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*AllGatherFn)(const void*, void*, size_t, int, Comm, cudaStream_t);
typedef const char* (*ErrStrFn)(int);
typedef int (*MemAllocFn)(void**, size_t);
typedef int (*MemFreeFn)(void*);
typedef int (*WinRegFn)(Comm, void*, size_t, Window*, int);
typedef int (*WinDeregFn)(Comm, Window);

struct Api {
  void* handle = nullptr;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  AllReduceFn all_reduce = nullptr;
  AllGatherFn all_gather = nullptr;
  ErrStrFn err_str = nullptr;
  MemAllocFn mem_alloc = nullptr;
  MemFreeFn mem_free = nullptr;
  WinRegFn win_reg = nullptr;
  WinDeregFn win_dereg = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  static std::string load_error;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      load_error = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    a.get_unique_id = reinterpret_cast<GetUniqueIdFn>(dlsym(a.handle, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<CommInitRankFn>(dlsym(a.handle, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<CommDestroyFn>(dlsym(a.handle, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<AllReduceFn>(dlsym(a.handle, "ncclAllReduce"));
    a.all_gather = reinterpret_cast<AllGatherFn>(dlsym(a.handle, "ncclAllGather"));
    a.err_str = reinterpret_cast<ErrStrFn>(dlsym(a.handle, "ncclGetErrorString"));
    a.mem_alloc = reinterpret_cast<MemAllocFn>(dlsym(a.handle, "ncclMemAlloc"));
    a.mem_free = reinterpret_cast<MemFreeFn>(dlsym(a.handle, "ncclMemFree"));
    a.win_reg = reinterpret_cast<WinRegFn>(dlsym(a.handle, "ncclCommWindowRegister"));
    a.win_dereg = reinterpret_cast<WinDeregFn>(dlsym(a.handle, "ncclCommWindowDeregister"));
  });
  if (!a.handle || !a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.all_gather)
    throw NcclError(load_error.empty() ? "NCCL symbols missing" : load_error);
  return a;
}

void check(int r, const char* what) {
  if (r != 0) {
    const char* s = api().err_str ? api().err_str(r) : "?";
    throw NcclError(std::string(what) + " failed: " + s);
  }
}

}  // namespace

void get_unique_id(UniqueId* id) { check(api().get_unique_id(id), "ncclGetUniqueId"); }

Comm init_rank(int nranks, const UniqueId& id, int rank) {
  Comm c = nullptr;
  check(api().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void destroy(Comm c) {
  if (c) api().comm_destroy(c);
}

void allreduce_sum_f32(float* buf, size_t count, Comm c, cudaStream_t s) {
  check(api().all_reduce(buf, buf, count, kFloat32, kSum, c, s), "ncclAllReduce");
}

void allgather_bytes(const void* send, void* recv, size_t bytes_per_rank, Comm c, cudaStream_t s) {
  check(api().all_gather(send, recv, bytes_per_rank, kUint8, c, s), "ncclAllGather");
}

bool has_windows() {
  const Api& a = api();
  return a.mem_alloc && a.mem_free && a.win_reg && a.win_dereg;
}

void* mem_alloc(size_t bytes) {
  void* p = nullptr;
  check(api().mem_alloc(&p, bytes), "ncclMemAlloc");
  return p;
}

void mem_free(void* p) {
  if (p) api().mem_free(p);
}

Window window_register(Comm c, void* buf, size_t bytes) {
  Window w = nullptr;
  check(api().win_reg(c, buf, bytes, &w, kWinCollSymmetric), "ncclCommWindowRegister");
  return w;
}

void window_deregister(Comm c, Window w) {
  if (w) api().win_dereg(c, w);
}

}  // namespace nccl
}  // namespace dsinf
