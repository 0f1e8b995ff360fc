// Microbenchmark: per-SM throughput of the instructions in the INT4 transcode on sm_100a.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define REP 8
template <int OP>
__global__ void k(uint32_t* out, int iters) {
  uint32_t v[REP];
  for (int i = 0; i < REP; ++i) v[i] = threadIdx.x * (i + 3) + 0x64006400u;
  const uint32_t c1 = 0x000F000Fu, c2 = 0x64006400u, c3 = 0x2C002C00u, c4 = 0xD480D480u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < REP; ++i) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(c1), "r"(c2));
      if (OP == 1) asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(v[i]) : "r"(c2));
      if (OP == 2) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(c3), "r"(c4));
      if (OP == 3) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(0x01000000u));
      if (OP == 4) asm volatile("shr.b32 %0, %0, 8;" : "+r"(v[i]));
      if (OP == 5) asm volatile("prmt.b32 %0, %0, %1, 0x4140;" : "+r"(v[i]) : "r"(c2));
      if (OP == 6) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(*(float*)&v[i]) : "f"(1.0001f), "f"(0.5f));
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < REP; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char* name) {
  uint32_t* o;
  cudaMalloc(&o, 148 * 1024 * 4);
  int iters = 20000;
  k<OP><<<148, 1024>>>(o, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<148, 1024>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = (double)iters * REP * 32 * 148;  // 32 warps per block
  double per_sm_cycle = warp_instr / 148 / (ms * 1e-3 * 1.9e9);
  printf("%-10s %.3f warp-instr/cycle/SM (assuming 1.9 GHz), %.3f ms\n", name, per_sm_cycle, ms);
}
int main() {
  run<0>("LOP3");
  run<1>("HSUB2");
  run<2>("HFMA2");
  run<3>("IMAD.HI");
  run<4>("SHF");
  run<5>("PRMT");
  run<6>("FFMA");
  return 0;
}
