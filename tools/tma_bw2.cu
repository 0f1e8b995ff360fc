// Bulk-copy streaming with the GEMV's consumer structure: P producer threads, C consumer
// warps each reading 16 B/lane of every 8 KB stage (as the transcode warps do) and arriving
// on the slot's empty barrier (count C).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
template <int RING, int P, int C, int ITEMS_STRIDE>
__global__ void __launch_bounds__(1024, 1) k(const uint8_t* src, int64_t nst, float* sink) {
  constexpr int SB = 8192;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + RING * SB);
  uint64_t* empty = full + RING;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + i)), "r"(C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // CTA b streams the 8 KB blocks b, b + 148*ITEMS_STRIDE... as items of 96 blocks (like row tiles)
  if (warp >= C && warp < C + P) {
    const int pr = warp - C;
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int64_t q = pr; q < nst; q += P) {
        const int slot = q % RING;
        wait(empty + slot, ((q / RING) & 1) ^ 1);
        const int64_t item = blockIdx.x + (q / 96) * 148, st = q % 96;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + slot)), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                         smem_u32(sm + slot * SB)), "l"(src + (item * 96 + st) * SB), "r"(SB), "r"(smem_u32(full + slot)), "l"(pol)
                     : "memory");
      }
    }
  } else if (warp < C) {
    uint32_t acc = 0;
    for (int64_t q = 0; q < nst; ++q) {
      const int slot = q % RING;
      wait(full + slot, (q / RING) & 1);
      const uint4 u = *reinterpret_cast<const uint4*>(sm + slot * SB + (warp % 4) * 2048 + (warp / 4) * 512 + lane * 16);
      acc ^= u.x ^ u.y ^ u.z ^ u.w;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
    }
    if (acc == 12345u) sink[0] = acc;
  }
}
template <int RING, int P, int C, int S>
void run(const uint8_t* src, int64_t bytes, float* sink) {
  const int64_t nst = (bytes / 148 / 8192) / 96 * 96;
  const size_t smem = RING * 8192 + 2 * RING * 8;
  cudaFuncSetAttribute(k<RING, P, C, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = (C + P) * 32;
  k<RING, P, C, S><<<148, threads, smem>>>(src, nst, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) k<RING, P, C, S><<<148, threads, smem>>>(src, nst, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("ring %2d producers %d consumers %2d: %7.0f GB/s (%s)\n", RING, P, C, 5.0 * nst * 8192 * 148 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int64_t bytes = 2ll << 30;
  uint8_t* src; float* sink;
  cudaMalloc(&src, bytes + (256 << 20)); cudaMalloc(&sink, 4);
  cudaMemset(src, 1, bytes);
  run<16, 1, 1, 1>(src, bytes, sink);
  run<16, 4, 1, 1>(src, bytes, sink);
  run<16, 1, 16, 1>(src, bytes, sink);
  run<16, 4, 16, 1>(src, bytes, sink);
  run<24, 4, 16, 1>(src, bytes, sink);
  return 0;
}
