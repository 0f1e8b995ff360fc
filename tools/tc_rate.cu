// tcgen05.mma issue/throughput probe: cycles per MMA (kind::f16, K = 16) for A from TMEM (ts)
// or shared memory (ss), M in {64, 128}, N in {16, 64, 256}; one CTA, one issuing thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int M, int N, bool TS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t sb = smem_u32(sm);
    // B (N rows) at sm[0..], A (M rows, ss) at sm[32768..]; K-major interleave, LBO = rows*16, SBO = 128
    const uint64_t bdesc = (uint64_t)((sb >> 4) & 0x3FFF) | ((uint64_t)((N * 16) >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    const uint64_t adesc = (uint64_t)(((sb + 32768) >> 4) & 0x3FFF) | ((uint64_t)((M * 16) >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tb + 256),
                     "r"(tb + (i & 7) * 8), "l"(bdesc), "r"(idesc), "r"(1));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tb + 256),
                     "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
template <int M, int N, bool TS>
void run() {
  long long* d; long long h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  k<M, N, TS><<<1, 128, 65536>>>(d, 64);
  k<M, N, TS><<<1, 128, 65536>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s M=%3d N=%3d: issue %.1f cyc/MMA, completion %.1f cyc/MMA  (%s)\n", TS ? "ts" : "ss", M, N, (double)h[0] / iters,
         (double)h[1] / iters, cudaGetErrorString(e));
}
int main() {
  run<128, 16, true>(); run<128, 64, true>(); run<128, 256, true>();
  run<64, 16, true>(); run<64, 64, true>();
  run<128, 16, false>(); run<128, 64, false>(); run<128, 256, false>(); run<64, 16, false>();
  return 0;
}
