// collective.h — cross-rank sums for Megatron tensor parallelism.
//
// One process per GPU. Two transports:
//  * NCCL over NVLink/NVSwitch for prefill-sized messages, the vocab-sharded head's argmax /
//    logits and communicator bring-up. libnccl is resolved at run time with
//    dlopen("libnccl.so.2") so this library links no NCCL: inside a torch process the
//    torch-bundled NCCL already loaded is reused. Stream-ordered and CUDA-graph capturable.
//  * the decode sublayer sums (B x hidden fp32, 48 KB at B = 1) skip NCCL: every rank pushes
//    its slice of the row-parallel output straight into every peer's inbox over NVLink
//    (CUDA IPC peer mappings) from inside the DeepNorm LayerNorm kernel, raises a per-slice
//    flag, and sums the t inboxes in rank order once the peers' flags arrive (PeerArgs,
//    block.cu k_deepnorm_ln) — one kernel instead of reduce + ncclAllReduce + LayerNorm.
//
// For tests on a single GPU the same model code runs t rank-models in one process
// (one host thread each) over an emulated group (EmuGroup): the allreduce is a
// stream-ordered sum kernel over the ranks' buffers behind a host barrier plus cross-stream
// events, and the fused decode sum runs its push phase and its consume phase as two
// launches separated by that barrier, so no kernel ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "block.h"

namespace glm {

constexpr int kUniqueIdBytes = 128;  // sizeof(ncclUniqueId)

struct EmuGroup;  // in-process rank group (collective.cu)
EmuGroup* emu_group_create(int size);
void emu_group_destroy(EmuGroup* g);

class Collective {
 public:
  Collective() = default;
  ~Collective();
  static void unique_id(void* out128);
  void init(int rank, int size, const void* id128);  // NCCL communicator
  void init_emulated(EmuGroup* g, int rank);         // in-process test group
  bool ready() const { return comm_ != nullptr || emu_ != nullptr; }
  bool emulated() const { return emu_ != nullptr; }
  int rank() const { return rank_; }
  int size() const { return size_; }
  void allreduce_sum(float* buf, int64_t count, cudaStream_t st);
  void allreduce_max_u64(unsigned long long* buf, int64_t count, cudaStream_t st);
  // logits [M][V]: each rank wrote its vocab slice, the rest is zero -> sum = gather
  void allgather_logits(float* logits, int M, int64_t V, int64_t off, int64_t local, cudaStream_t st);

  // Fused decode sublayer sum (block.cu): inboxes [2][size][max_b][d] fp32 + flags on every
  // rank, mapped into every peer (CUDA IPC over NCCL-exchanged handles, or the emulated
  // group's pointers). Collective call: every rank of the group calls it.
  void setup_peer(int max_b, int64_t d, cudaStream_t st);
  bool peer_ready() const { return peer_.size > 1; }
  PeerArgs peer_args() const { return peer_; }
  // emulated group only: this rank's stream waits until every rank's stream reached this
  // point (host barrier + cross-stream events)
  void barrier(cudaStream_t st);
  // the fused kernel's timeout word (a peer never arrived): throws GLM_NCCL if set
  void check_peer(cudaStream_t st);

 private:
  void* comm_ = nullptr;
  EmuGroup* emu_ = nullptr;
  int rank_ = 0, size_ = 1;
  PeerArgs peer_{};
  void* peer_base_ = nullptr;              // own inbox/flag region (cudaMalloc)
  void* peer_open_[kMaxTp] = {};           // IPC-opened peer regions (NCCL mode)
  float* scratch_ = nullptr;               // emulated allreduce result staging
  int64_t scratch_bytes_ = 0;
};

}  // namespace glm
