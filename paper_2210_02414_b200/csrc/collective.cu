// collective.cu — tensor-parallel sums: NCCL (dlopen), the fused-decode peer inboxes (CUDA
// IPC), and the in-process emulated group used by the single-GPU tests (collective.h).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "collective.h"
#include "common.cuh"

namespace glm {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
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
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
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

struct RankPtrs {
  const void* p[kMaxTp];
};

// out = sum over ranks of p[r] in rank order (identical bits on every rank)
__global__ void k_sum_ranks(RankPtrs in, int size, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < size; ++r) acc += static_cast<const float*>(in.p[r])[i];
    out[i] = acc;
  }
}

__global__ void k_max_ranks(RankPtrs in, int size, unsigned long long* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    unsigned long long m = 0;
    for (int r = 0; r < size; ++r) {
      const unsigned long long v = static_cast<const unsigned long long*>(in.p[r])[i];
      m = v > m ? v : m;
    }
    out[i] = m;
  }
}

int grid_n(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b < kNumSMs * 8 ? b : kNumSMs * 8));
}

// peer region of one rank: inbox [2][size][max_b][d] fp32 | flags [2][size][max_b][slices] u32 |
// gen [max_b][slices] u32 | err int
struct PeerLayout {
  size_t inbox, flags, gen, err, total;
  PeerLayout(int size, int max_b, int64_t d) {
    inbox = 0;
    flags = inbox + sizeof(float) * 2 * size * static_cast<size_t>(max_b) * d;
    gen = flags + sizeof(unsigned) * 2 * size * static_cast<size_t>(max_b) * kPeerSlices;
    err = gen + sizeof(unsigned) * static_cast<size_t>(max_b) * kPeerSlices;
    total = (err + 256 + 255) / 256 * 256;
  }
};

}  // namespace

// ---- in-process rank group (single-GPU tests) -------------------------------------------
struct EmuGroup {
  int size;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  std::vector<void*> ptr;
  std::vector<cudaEvent_t> ev;
  explicit EmuGroup(int n) : size(n), ptr(n, nullptr), ev(n, nullptr) {}
  ~EmuGroup() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  void host_barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = phase;
    if (++arrived == size) {
      arrived = 0;
      ++phase;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return phase != my; });
    }
  }
  // publish this rank's pointer and stream position; returns every rank's pointer once all
  // ranks published, with this rank's stream ordered after every rank's published position
  std::vector<void*> exchange(int rank, void* p, cudaStream_t st) {
    if (!ev[rank]) CUDA_CHECK(cudaEventCreateWithFlags(&ev[rank], cudaEventDisableTiming));
    ptr[rank] = p;
    CUDA_CHECK(cudaEventRecord(ev[rank], st));
    host_barrier();
    std::vector<void*> all = ptr;
    for (int r = 0; r < size; ++r)
      if (r != rank) CUDA_CHECK(cudaStreamWaitEvent(st, ev[r], 0));
    host_barrier();  // nobody re-records its event before every rank enqueued its waits
    return all;
  }
};

EmuGroup* emu_group_create(int size) {
  if (size < 2 || size > kMaxTp) fail(GLM_CONTRACT, "collective", "emulated group size must be in 2..8");
  return new EmuGroup(size);
}
void emu_group_destroy(EmuGroup* g) { delete g; }

// ---- Collective ----------------------------------------------------------------------------
Collective::~Collective() {
  for (int r = 0; r < kMaxTp; ++r)
    if (peer_open_[r]) cudaIpcCloseMemHandle(peer_open_[r]);
  if (peer_base_) cudaFree(peer_base_);
  if (scratch_) cudaFree(scratch_);
  if (comm_) api().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void Collective::unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == kUniqueIdBytes, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

void Collective::init(int rank, int size, const void* id128) {
  if (size > kMaxTp) fail(GLM_CONTRACT, "collective", "tensor-parallel size above 8");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  check(api().CommInitRank(&c, size, id, rank), "ncclCommInitRank");
  comm_ = c;
  rank_ = rank;
  size_ = size;
}

void Collective::init_emulated(EmuGroup* g, int rank) {
  if (!g) fail(GLM_CONTRACT, "collective", "null emulated group");
  if (rank < 0 || rank >= g->size) fail(GLM_CONTRACT, "collective", "rank outside the emulated group");
  emu_ = g;
  rank_ = rank;
  size_ = g->size;
}

void Collective::barrier(cudaStream_t st) {
  if (!emu_) fail(GLM_CONTRACT, "collective", "barrier() is the emulated group's phase separator");
  emu_->exchange(rank_, nullptr, st);
}

void Collective::allreduce_sum(float* buf, int64_t count, cudaStream_t st) {
  if (emu_) {
    if (scratch_bytes_ < count * 4) {
      if (scratch_) CUDA_CHECK(cudaFree(scratch_));
      CUDA_CHECK(cudaMalloc(&scratch_, count * 4));
      scratch_bytes_ = count * 4;
    }
    const std::vector<void*> all = emu_->exchange(rank_, buf, st);  // every rank's buffer is complete
    RankPtrs rp{};
    for (int r = 0; r < size_; ++r) rp.p[r] = all[r];
    k_sum_ranks<<<grid_n(count), 256, 0, st>>>(rp, size_, scratch_, count);
    LAUNCH_CHECK("k_sum_ranks");
    emu_->exchange(rank_, nullptr, st);  // every rank has read every buffer
    CUDA_CHECK(cudaMemcpyAsync(buf, scratch_, count * 4, cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (!comm_) fail(GLM_NCCL, "collective", "tensor-parallel communicator not initialised (glm_model_init_comm)");
  check(api().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), st),
        "ncclAllReduce(sum)");
}

void Collective::allreduce_max_u64(unsigned long long* buf, int64_t count, cudaStream_t st) {
  if (emu_) {
    if (scratch_bytes_ < count * 8) {
      if (scratch_) CUDA_CHECK(cudaFree(scratch_));
      CUDA_CHECK(cudaMalloc(&scratch_, count * 8));
      scratch_bytes_ = count * 8;
    }
    const std::vector<void*> all = emu_->exchange(rank_, buf, st);
    RankPtrs rp{};
    for (int r = 0; r < size_; ++r) rp.p[r] = all[r];
    k_max_ranks<<<grid_n(count), 256, 0, st>>>(rp, size_, reinterpret_cast<unsigned long long*>(scratch_), count);
    LAUNCH_CHECK("k_max_ranks");
    emu_->exchange(rank_, nullptr, st);
    CUDA_CHECK(cudaMemcpyAsync(buf, scratch_, count * 8, cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (!comm_) fail(GLM_NCCL, "collective", "tensor-parallel communicator not initialised (glm_model_init_comm)");
  check(api().AllReduce(buf, buf, static_cast<size_t>(count), ncclUint64, ncclMax, static_cast<ncclComm_t>(comm_), st),
        "ncclAllReduce(max)");
}

void Collective::allgather_logits(float* logits, int M, int64_t V, int64_t off, int64_t local, cudaStream_t st) {
  k_zero_outside<<<kNumSMs * 4, 256, 0, st>>>(logits, M, V, off, local);
  LAUNCH_CHECK("k_zero_outside");
  allreduce_sum(logits, static_cast<int64_t>(M) * V, st);
}

void Collective::setup_peer(int max_b, int64_t d, cudaStream_t st) {
  if (size_ < 2) return;
  if (!ready()) fail(GLM_NCCL, "collective", "setup_peer before the communicator");
  const PeerLayout lay(size_, max_b, d);
  CUDA_CHECK(cudaMalloc(&peer_base_, lay.total));
  CUDA_CHECK(cudaMemsetAsync(peer_base_, 0, lay.total, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  std::vector<void*> bases(size_, nullptr);
  if (emu_) {
    bases = emu_->exchange(rank_, peer_base_, st);
  } else {
    // CUDA IPC handles of every rank's region, exchanged with one NCCL all-gather
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    CUDA_CHECK(cudaIpcGetMemHandle(&h, peer_base_));
    void* dh = nullptr;
    CUDA_CHECK(cudaMalloc(&dh, 64 * (size_ + 1) + 4 * (size_ + 1)));
    CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(dh) + 64 * size_, &h, 64, cudaMemcpyHostToDevice, st));
    if (!api().AllGather) fail(GLM_NCCL, "collective", "ncclAllGather not found in libnccl.so.2");
    check(api().AllGather(static_cast<uint8_t*>(dh) + 64 * size_, dh, 64, ncclUint8, static_cast<ncclComm_t>(comm_), st),
          "ncclAllGather(ipc handles)");
    std::vector<cudaIpcMemHandle_t> hs(size_);
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), dh, 64 * size_, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    // every rank maps every peer, then all agree (min over ranks) before any kernel relies on
    // it: a rank that cannot map a peer turns the fused path off on every rank (NCCL decode)
    int ok = 1;
    std::string why;
    for (int r = 0; r < size_ && ok; ++r) {
      if (r == rank_) {
        bases[r] = peer_base_;
        continue;
      }
      const cudaError_t e = cudaIpcOpenMemHandle(&peer_open_[r], hs[r], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        cudaGetLastError();
        peer_open_[r] = nullptr;
        ok = 0;
        why = cudaGetErrorString(e);
      } else {
        bases[r] = peer_open_[r];
      }
    }
    int* flag = reinterpret_cast<int*>(static_cast<uint8_t*>(dh) + 64 * (size_ + 1));
    CUDA_CHECK(cudaMemcpyAsync(flag, &ok, 4, cudaMemcpyHostToDevice, st));
    check(api().AllReduce(flag, flag, 1, ncclInt32, ncclMin, static_cast<ncclComm_t>(comm_), st), "ncclAllReduce(peer ok)");
    CUDA_CHECK(cudaMemcpyAsync(&ok, flag, 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    CUDA_CHECK(cudaFree(dh));
    if (!ok) {
      for (int r = 0; r < size_; ++r)
        if (peer_open_[r]) {
          cudaIpcCloseMemHandle(peer_open_[r]);
          peer_open_[r] = nullptr;
        }
      cudaFree(peer_base_);
      peer_base_ = nullptr;
      peer_ = PeerArgs{};
      fprintf(stderr, "[collective] rank %d: fused decode allreduce unavailable (%s); decode sums use NCCL\n", rank_,
              why.empty() ? "a peer could not map the inboxes" : why.c_str());
      return;
    }
  }
  PeerArgs p;
  for (int r = 0; r < size_; ++r) {
    p.inbox[r] = reinterpret_cast<float*>(static_cast<uint8_t*>(bases[r]) + lay.inbox);
    p.flags[r] = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(bases[r]) + lay.flags);
  }
  p.gen = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(peer_base_) + lay.gen);
  p.err = reinterpret_cast<int*>(static_cast<uint8_t*>(peer_base_) + lay.err);
  p.rank = rank_;
  p.size = size_;
  p.max_b = max_b;
  p.mode = emu_ ? 1 : 3;
  p.d = d;
  peer_ = p;
}

void Collective::check_peer(cudaStream_t st) {
  if (!peer_ready()) return;
  int err = 0;
  CUDA_CHECK(cudaMemcpyAsync(&err, peer_.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  if (err) fail(GLM_NCCL, "collective", "a tensor-parallel peer did not deliver its decode partial (timeout)");
}

}  // namespace glm
