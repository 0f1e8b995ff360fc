// Bulk-copy (cp.async.bulk, 1-D TMA) streaming bandwidth: 1 CTA/SM, ring of RING slots of
// SB bytes, P producer threads (round-robin slots), 1 consumer warp per... releases slots.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
template <int SB, int RING, int P, int COPIES>
__global__ void __launch_bounds__(256, 1) k(const uint8_t* src, int64_t per_cta, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + RING * SB);
  uint64_t* empty = full + RING;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + i)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t nst = per_cta / SB;
  const uint8_t* base = src + blockIdx.x * per_cta;
  if (warp < P) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int64_t q = warp; q < nst; q += P) {
        const int slot = q % RING;
        wait(empty + slot, ((q / RING) & 1) ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + slot)), "r"(SB) : "memory");
        for (int c = 0; c < COPIES; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                           smem_u32(sm + slot * SB + c * (SB / COPIES))),
                       "l"(base + q * SB + c * (SB / COPIES)), "r"(SB / COPIES), "r"(smem_u32(full + slot)), "l"(pol)
                       : "memory");
      }
    }
  } else if (warp == 7) {
    float acc = 0.f;
    for (int64_t q = 0; q < nst; ++q) {
      const int slot = q % RING;
      wait(full + slot, (q / RING) & 1);
      acc += reinterpret_cast<const float*>(sm + slot * SB)[lane];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
    }
    if (acc == 12345.f) sink[0] = acc;
  }
}
template <int SB, int RING, int P, int COPIES>
void run(const uint8_t* src, int64_t bytes, float* sink) {
  const int64_t per_cta = (bytes / 148) / SB * SB;
  const size_t smem = RING * SB + 2 * RING * 8;
  cudaFuncSetAttribute(k<SB, RING, P, COPIES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<SB, RING, P, COPIES><<<148, 256, smem>>>(src, per_cta, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) k<SB, RING, P, COPIES><<<148, 256, smem>>>(src, per_cta, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("slot %6d B ring %2d producers %d copies/slot %d: %7.0f GB/s (%s)\n", SB, RING, P, COPIES,
         5.0 * per_cta * 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int64_t bytes = 2ll << 30;
  uint8_t* src; float* sink;
  cudaMalloc(&src, bytes); cudaMalloc(&sink, 4);
  cudaMemset(src, 1, bytes);
  run<8192, 12, 1, 1>(src, bytes, sink);
  run<8192, 12, 4, 1>(src, bytes, sink);
  run<8192, 24, 4, 1>(src, bytes, sink);
  run<16384, 12, 1, 1>(src, bytes, sink);
  run<16384, 12, 4, 1>(src, bytes, sink);
  run<32768, 6, 1, 1>(src, bytes, sink);
  run<32768, 6, 4, 1>(src, bytes, sink);
  run<32768, 6, 2, 4>(src, bytes, sink);
  run<65536, 3, 1, 1>(src, bytes, sink);
  run<4096, 48, 4, 1>(src, bytes, sink);
  return 0;
}
