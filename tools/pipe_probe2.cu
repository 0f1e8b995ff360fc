// Co-issue probe: which pipes do LOP3 / HSUB2 / HFMA2 / HMMA share on sm_100a.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define REP 8
__device__ __forceinline__ void op(int kind, uint32_t& v, uint32_t c1, uint32_t c2) {
  if (kind == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v) : "r"(c1), "r"(c2));
  if (kind == 1) asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(v) : "r"(c2));
  if (kind == 2) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(v) : "r"(c1), "r"(c2));
  if (kind == 3) asm volatile("shr.b32 %0, %0, %1;" : "+r"(v) : "r"(c1 & 7));
}
template <int A, int B, int MMA>
__global__ void k(uint32_t* out, int iters) {
  uint32_t v[REP], w[REP];
  for (int i = 0; i < REP; ++i) v[i] = w[i] = threadIdx.x * (i + 3) + 0x64006400u;
  const uint32_t c1 = 0x000F000Fu + (threadIdx.x & 1), c2 = 0x64006400u;
  float acc[2][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < REP; ++i) {
      op(A, v[i], c1, c2);
      if (B >= 0) op(B, w[i], c1, c2);
    }
    if (MMA) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                     : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(w[0]), "r"(w[1]));
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < REP; ++i) s ^= v[i] ^ w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (uint32_t)(acc[0][0] + acc[1][1]);
}
template <int A, int B, int MMA>
void run(const char* name) {
  uint32_t* o;
  cudaMalloc(&o, 148 * 512 * 4);
  const int iters = 20000;
  k<A, B, MMA><<<148, 512>>>(o, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<A, B, MMA><<<148, 512>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = 16.0;  // per SM
  const double n_alu = REP * (B >= 0 ? 2 : 1);
  const double cyc = ms * 1e-3 * 1.9e9;
  printf("%-24s ops %.2f warp-instr/cycle/SM, mma %.3f/cycle/SM  (%.3f ms)\n", name, iters * n_alu * warps / cyc,
         MMA ? iters * 2 * warps / cyc : 0.0, ms);
}
int main() {
  run<0, -1, 0>("LOP3");
  run<0, 0, 0>("LOP3+LOP3");
  run<0, 1, 0>("LOP3+HSUB2");
  run<0, 2, 0>("LOP3+HFMA2");
  run<1, 2, 0>("HSUB2+HFMA2");
  run<2, 2, 0>("HFMA2+HFMA2");
  run<0, 3, 0>("LOP3+SHF");
  run<0, 2, 1>("LOP3+HFMA2+HMMA");
  run<0, -1, 1>("LOP3+HMMA");
  run<2, -1, 1>("HFMA2+HMMA");
  run<1, -1, 1>("HSUB2+HMMA");
  return 0;
}
