// Does sm_100a run 4-bit mma.sync (m16n8k64 u4 x s4) natively? Throughput in dense MACs/clk/SM
// against m16n8k32 u8 x s8, both with 4 independent accumulators per warp.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int* out, int iters) {
  int acc[4][4] = {};
  uint32_t w = threadIdx.x * 0x9E3779B9u, b0 = threadIdx.x ^ 0x3c00, b1 = threadIdx.x ^ 0x1234;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t a0 = w + c, a1 = w ^ c, a2 = w + 7 * c, a3 = w ^ (3 * c);
      if (MODE == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    w = w * 1664525u + 1013904223u;
  }
  int s = 0;
  for (int c = 0; c < 4; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(const char* name, int warps) {
  int* o; cudaMalloc(&o, 1 << 24);
  const int iters = 8192;
  k<MODE><<<148, warps * 32>>>(o, iters);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE><<<148, warps * 32>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double macs = 148.0 * warps * iters * 4 * 16 * 8 * (MODE == 0 ? 32 : 64);
  printf("%-24s warps %2d: %.3f ms  %.1f TMAC/s (%s)\n", name, warps, ms, macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int w : {4, 8, 16}) { run<0>("m16n8k32 u8.s8", w); run<1>("m16n8k64 u4.s4", w); }
}
