// collective.h — cross-rank sums for Megatron tensor parallelism.
//
// NCCL over NVLink/NVSwitch, one process per GPU. libnccl is resolved at run time with
// dlopen("libnccl.so.2") so this library links no NCCL: inside a torch process the
// torch-bundled NCCL already loaded is reused, so one NCCL serves torch.distributed and
// this library. Every call is stream-ordered and CUDA-graph capturable.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace glm {

constexpr int kUniqueIdBytes = 128;  // sizeof(ncclUniqueId)

class Collective {
 public:
  Collective() = default;
  ~Collective();
  static void unique_id(void* out128);
  void init(int rank, int size, const void* id128);
  bool ready() const { return comm_ != nullptr; }
  void allreduce_sum(float* buf, int64_t count, cudaStream_t st);
  void allreduce_max_u64(unsigned long long* buf, int64_t count, cudaStream_t st);
  // logits [M][V]: each rank wrote its vocab slice, the rest is zero -> sum = gather
  void allgather_logits(float* logits, int M, int64_t V, int64_t off, int64_t local, cudaStream_t st);

 private:
  void* comm_ = nullptr;
  int rank_ = 0, size_ = 1;
};

}  // namespace glm
