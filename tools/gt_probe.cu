// %globaltimer resolution on this GPU: distinct consecutive values seen by one thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int n = 0;
  for (int i = 0; i < 2000000 && n < 16; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[n++] = t - prev; prev = t; }
  }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8); cudaMemset(d, 0, 128);
  k<<<1, 1>>>(d); unsigned long long h[16]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("globaltimer steps (ns):"); for (int i = 0; i < 16; ++i) printf(" %llu", h[i]); printf("\n");
}
