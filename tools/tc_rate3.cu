// Does concurrent tcgen05.st traffic slow tcgen05.mma (A from TMEM, N = 16)?
// 4 issuer threads issue MMAs over A columns [0,256); 16 writer warps store 16-column chunks.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int WRITERS, int STCOLS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  long long t0 = clock64();
  if (warp < 4) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 17) | (8u << 24);
      const uint32_t sb = smem_u32(sm);
      const uint64_t bdesc = (uint64_t)((sb >> 4) & 0x3FFF) | ((uint64_t)(256 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tb + 256 + warp * 16),
                       "r"(tb + ((i / 8 + warp) % 8) * 32 + (j % 4) * 8), "l"(bdesc + (j % 4) * 32), "r"(idesc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])));
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar[warp])));
      out[warp] = clock64() - t0;
    }
  } else if (warp < 4 + WRITERS) {
    const int quarter = warp & 3;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = 0x3c003c00u + lane + i;
    const int nst = iters / 4;  // stores per writer
    for (int i = 0; i < nst; ++i) {
      const uint32_t addr = tb + ((uint32_t)(quarter * 32) << 16) + ((i * 16 + (warp >> 2) * 64) % 256);
      if (STCOLS == 16)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                     "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    if (lane == 0) out[warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
template <int W, int C>
void run() {
  long long* d; long long h[32] = {};
  cudaMalloc(&d, 256);
  cudaMemset(d, 0, 256);
  cudaFuncSetAttribute(k<W, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  const int iters = 4096;
  k<W, C><<<1, (4 + W) * 32, 16384>>>(d, 64);
  k<W, C><<<1, (4 + W) * 32, 16384>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  long long mm = 0, ws = 0;
  for (int i = 0; i < 4; ++i) mm = h[i] > mm ? h[i] : mm;
  for (int i = 4; i < 4 + W; ++i) ws = h[i] > ws ? h[i] : ws;
  printf("writers %2d: MMA %.1f cyc per MMA (4 issuers); STTM.x16 %.1f cyc per store per SM (%s)\n", W, (double)mm / (4 * iters),
         W ? (double)ws / ((iters / 4) * W) : 0.0, cudaGetErrorString(e));
}
int main() {
  run<0, 16>(); run<4, 16>(); run<16, 16>();
  return 0;
}
