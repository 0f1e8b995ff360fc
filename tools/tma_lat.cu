// Latency of bulk-copying an L2-resident activation vector into shared memory (the GEMV
// prologue's x load): 1 or 148 CTAs, same or distinct source, piece size, issuing threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const uint8_t* src, int bytes, int piece, int issuers, int distinct, long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* s = src + (distinct ? static_cast<size_t>(blockIdx.x) * bytes : 0);
  long long t0 = clock64();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
  __syncthreads();
  const int np = bytes / piece;
  if ((int)threadIdx.x < issuers)
    for (int p = threadIdx.x; p < np; p += issuers)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + p * piece)),
                   "l"(s + static_cast<size_t>(p) * piece), "r"(piece), "r"(sa(&bar)) : "memory");
  asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  uint8_t* src; cudaMalloc(&src, 148 * 65536); cudaMemset(src, 1, 148 * 65536);
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int bytes : {24576, 65536})
    for (int grid : {1, 148})
      for (int distinct : {0, 1})
        for (int piece : {16384, 4096, 1024})
          for (int issuers : {1, 8, 32}) {
            if (bytes % piece) continue;
            long long best = 1LL << 60, worst = 0;
            for (int rep = 0; rep < 5; ++rep) {
              k<<<grid, 256, 65536>>>(src, bytes, piece, issuers, distinct, d);
              long long h[148]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
              long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
              if (rep > 0) { best = mx < best ? mx : best; worst = mx > worst ? mx : worst; }
            }
            printf("bytes %6d grid %3d distinct %d piece %5d issuers %2d: max-CTA %6lld cycles (%.2f us at %d MHz; worst %lld)\n",
                   bytes, grid, distinct, piece, issuers, best, best / (clk / 1e3), clk / 1000, worst);
          }
}
