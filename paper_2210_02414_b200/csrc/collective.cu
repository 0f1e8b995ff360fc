// collective.cu — NCCL (dlopen) allreduce for the row-parallel linears.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "collective.h"
#include "common.cuh"

namespace glm {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror();
      return;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!a.AllReduce) fail(GLM_NCCL, "collective", "libnccl.so.2 not loadable: " + err);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(GLM_NCCL, "collective", std::string(what) + ": " + api().GetErrorString(r));
}

__global__ void k_zero_outside(float* logits, int M, int64_t V, int64_t off, int64_t local) {
  const int64_t n = static_cast<int64_t>(M) * V;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i % V;
    if (c < off || c >= off + local) logits[i] = 0.f;
  }
}

}  // namespace

Collective::~Collective() {
  if (comm_) api().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void Collective::unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == kUniqueIdBytes, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

void Collective::init(int rank, int size, const void* id128) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  check(api().CommInitRank(&c, size, id, rank), "ncclCommInitRank");
  comm_ = c;
  rank_ = rank;
  size_ = size;
}

void Collective::allreduce_sum(float* buf, int64_t count, cudaStream_t st) {
  if (!comm_) fail(GLM_NCCL, "collective", "tensor-parallel communicator not initialised (glm_model_init_comm)");
  check(api().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), st),
        "ncclAllReduce(sum)");
}

void Collective::allreduce_max_u64(unsigned long long* buf, int64_t count, cudaStream_t st) {
  if (!comm_) fail(GLM_NCCL, "collective", "tensor-parallel communicator not initialised (glm_model_init_comm)");
  check(api().AllReduce(buf, buf, static_cast<size_t>(count), ncclUint64, ncclMax, static_cast<ncclComm_t>(comm_), st),
        "ncclAllReduce(max)");
}

void Collective::allgather_logits(float* logits, int M, int64_t V, int64_t off, int64_t local, cudaStream_t st) {
  k_zero_outside<<<148 * 4, 256, 0, st>>>(logits, M, V, off, local);
  LAUNCH_CHECK("k_zero_outside");
  allreduce_sum(logits, static_cast<int64_t>(M) * V, st);
}

}  // namespace glm
