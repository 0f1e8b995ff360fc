// Microbenchmark: legacy mma.sync m16n8k16 (HMMA.16816.F32) latency and throughput on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void k(float* out, int iters, long long* cyc) {
  float acc[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c) for (int i = 0; i < 4; ++i) acc[c][i] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x1234;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps, int blocks) {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  int iters = 4096;
  k<CH><<<blocks, warps * 32>>>(o, iters, c);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, warps * 32>>>(o, iters, c);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  double hmma = (double)iters * CH * warps * blocks;
  printf("chains %2d warps/blk %2d blocks %4d: %6.2f cyc per HMMA per warp (block0), chip %.3f HMMA/cycle/SM @ %.0f MHz est\n",
         CH, warps, blocks, (double)cyc / (iters * CH), hmma / (ms * 1e-3) / 148 / 1.965e9, 0.0);
}
int main() {
  run<1>(1, 1); run<2>(1, 1); run<4>(1, 1); run<8>(1, 1);
  run<1>(4, 1); run<4>(4, 1); run<8>(4, 1);
  run<4>(16, 148); run<8>(16, 148); run<8>(32, 148); run<4>(32, 148);
  return 0;
}
