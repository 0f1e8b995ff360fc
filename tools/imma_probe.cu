// Microbenchmark: legacy mma.sync m16n8k32 u8 x s8 -> s32 (IMMA.16832) throughput on sm_100a,
// alone and interleaved with the LOP3 nibble unpack the INT4 GEMV would need (4 LOP3 per IMMA),
// against HMMA.16816.F32 with the fp16 transcode (5 ALU/FMA ops per HMMA).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int* out, int iters, long long* cyc) {
  int acc[4][4] = {};
  float facc[4][4] = {};
  uint32_t w = threadIdx.x * 0x9E3779B9u, b0 = threadIdx.x ^ 0x3c00, b1 = threadIdx.x ^ 0x1234;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t a0, a1, a2, a3;
      if (MODE == 0) {  // IMMA alone
        a0 = w; a1 = w + 1; a2 = w + 2; a3 = w + 3;
      } else {          // IMMA + 4 LOP3 (two code words -> lo/hi nibble bytes)
        const uint32_t w0 = w + c, w1 = w ^ c;
        asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, 0, 0xC0;" : "=r"(a0) : "r"(w0));
        asm volatile("lop3.b32 %0, %1, 0xF0F0F0F0, 0, 0xC0;" : "=r"(a1) : "r"(w0));
        asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, 0, 0xC0;" : "=r"(a2) : "r"(w1));
        asm volatile("lop3.b32 %0, %1, 0xF0F0F0F0, 0, 0xC0;" : "=r"(a3) : "r"(w1));
      }
      if (MODE < 2) {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else {  // HMMA reference with the same 4 LOP3
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(facc[c][0]), "+f"(facc[c][1]), "+f"(facc[c][2]), "+f"(facc[c][3])
            : "r"(a0 | 0x64006400u), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
    w = w * 1664525u + 1013904223u;
  }
  long long t1 = clock64();
  int s = 0;
  for (int c = 0; c < 4; ++c)
    for (int i = 0; i < 4; ++i) s += acc[c][i] + static_cast<int>(facc[c][i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  int* o;
  long long* c;
  cudaMalloc(&o, 1 << 24);
  cudaMalloc(&c, 8);
  const int iters = 8192, blocks = 148;
  k<MODE><<<blocks, warps * 32>>>(o, iters, c);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, warps * 32>>>(o, iters, c);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  const double mma = 4.0 * iters * warps;  // per SM
  printf("%-28s warps %2d: %.3f MMA/cycle/SM (clock64 of CTA 0), %.1f cyc/MMA/SMSP, chip %.3f ms (%s)\n", name, warps,
         mma / cyc, cyc / (mma / 4), ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("IMMA.16832 u8.s8", 8);
  run<0>("IMMA.16832 u8.s8", 16);
  run<1>("IMMA.16832 + 4 LOP3", 16);
  run<1>("IMMA.16832 + 4 LOP3", 32);
  run<2>("HMMA.16816 + 4 LOP3", 16);
  return 0;
}
