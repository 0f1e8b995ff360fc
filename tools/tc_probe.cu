// Validates the tcgen05 building blocks used by the TMEM-staged GEMV:
// TMEM alloc, tcgen05.st (A operand, 128 rows x K fp16), B (16 x K fp16) in shared memory
// in the K-major no-swizzle canonical layout, tcgen05.mma kind::f16 with A from TMEM,
// tcgen05.commit -> mbarrier, tcgen05.ld of the fp32 accumulator.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int K = 64;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __half* A, const __half* B, float* D) {
  // A: [128][K] row-major, B: [16][K] row-major (tokens x k), D: [128][16]
  __shared__ __align__(1024) __half bs[16 * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B canonical K-major INTERLEAVE: [kstep][kh][rg][row 8][8 k]; LBO = 256 B (kh), SBO = 128 B (rg)
  for (int i = threadIdx.x; i < 16 * K; i += blockDim.x) {
    const int n = i / K, kk = i % K;
    const int ks = kk / 16, kh = (kk % 16) / 8, ke = kk % 8, rg = n / 8, r = n % 8;
    bs[((ks * 2 + kh) * 2 + rg) * 64 + r * 8 + ke] = B[n * K + kk];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  // A -> TMEM columns [0, K/2): lane = row, column j = (k 2j, 2j+1)
  {
    const int row = warp * 32 + lane;
    uint32_t r[K / 2];
    for (int j = 0; j < K / 2; ++j) {
      __half2 h = __halves2half2(A[row * K + 2 * j], A[row * K + 2 * j + 1]);
      r[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dcol = 32;  // D at columns [32, 48)
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint32_t saddr = smem_u32(bs) + ks * 512;
      const uint64_t desc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(256 >> 4) << 16) |
                            ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tbase + dcol),
          "r"(tbase + ks * 8), "l"(desc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[16];
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + dcol;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int n = 0; n < 16; ++n) D[row * 16 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(64));
}

int main() {
  __half hA[128 * K], hB[16 * K];
  float ref[128 * 16], got[128 * 16];
  srand(1);
  for (int i = 0; i < 128 * K; ++i) hA[i] = __float2half((float)(rand() % 15 - 7));
  for (int i = 0; i < 16 * K; ++i) hB[i] = __float2half((float)(rand() % 9 - 4) * 0.25f);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      float s = 0;
      for (int kk = 0; kk < K; ++kk) s += __half2float(hA[m * K + kk]) * __half2float(hB[n * K + kk]);
      ref[m * 16 + n] = s;
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(got));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(got, dD, sizeof(got), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128 * 16; ++i)
    if (got[i] != ref[i]) {
      if (bad < 8) printf("mismatch row %d col %d: got %f ref %f\n", i / 16, i % 16, got[i], ref[i]);
      ++bad;
    }
  printf("%s: %d mismatches of %d\n", bad ? "FAIL" : "PASS", bad, 128 * 16);
  return 0;
}
