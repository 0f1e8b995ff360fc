// tcgen05.mma small-N rate: unrolled issue with uniform operands, 1 vs 2 issuing warps.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc));
}
template <int N, int ISSUERS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  if (warp < ISSUERS) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t sb = smem_u32(sm);
    const uint64_t bdesc = (uint64_t)((sb >> 4) & 0x3FFF) | ((uint64_t)((N * 16) >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    const uint32_t dcol = tb + 256 + warp * 64, acol = tb + (warp & 1) * 128;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
      if (threadIdx.x % 32 == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ts(dcol, acol + j * 8, bdesc + j * 32, idesc);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x % 32 == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])));
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar[warp])));
      long long t2 = clock64();
      out[warp * 2] = t1 - t0;
      out[warp * 2 + 1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
template <int N, int IS>
void run() {
  long long* d; long long h[8] = {};
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k<N, IS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const int iters = 4096;
  k<N, IS><<<1, 128, 32768>>>(d, 64);
  k<N, IS><<<1, 128, 32768>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < IS; ++i) mx = h[2*i+1] > mx ? h[2*i+1] : mx;
  printf("N=%3d issuers=%d: issue %.1f cyc/MMA/issuer, completion %.1f cyc per MMA (all issuers) (%s)\n", N, IS,
         (double)h[0] / iters, (double)mx / (iters * IS), cudaGetErrorString(e));
}
int main() {
  run<16, 1>(); run<16, 2>(); run<16, 3>(); run<16, 4>(); run<32, 4>(); run<64, 4>();
  return 0;
}
