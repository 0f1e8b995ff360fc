// rowstat.cuh — LayerNorm row statistics shared by the LayerNorm kernels (block.cu) and the
// decode GEMV's fused LayerNorm prologue (gemv.cu).
#pragma once
#include <cuda_runtime.h>

namespace glm {

// Row statistics (mean, biased variance; tensor.cpp:264-267) without the E[z^2] - mean^2
// cancellation: every partial is (count, mean, M2 = sum of squared deviations from its own
// mean) and partials merge with Chan et al.'s pairwise update, so a row whose mean is large
// against its spread (loaded checkpoints with LN biases) keeps full fp32 precision. All merges
// run in a fixed order: identical results on every CTA, rank and run.
struct RowStat {
  float n, mean, m2;
};
__device__ __forceinline__ RowStat stat_merge(RowStat a, RowStat b) {
  const float n = a.n + b.n;
  if (b.n == 0.f) return a;
  if (a.n == 0.f) return b;
  const float d = b.mean - a.mean, f = b.n / n;
  return RowStat{n, fmaf(d, f, a.mean), a.m2 + b.m2 + d * d * a.n * f};
}
// A thread's own values accumulate as shifted sums about the first value it sees (K): within
// a row |z - K| is a few standard deviations, so S2 - S1^2 / n loses only a few bits; the
// per-thread partials then merge exactly (stat_merge).
struct ShiftedSums {
  float k = 0.f, s1 = 0.f, s2 = 0.f, n = 0.f;
  __device__ __forceinline__ void add(float v) {
    if (n == 0.f) k = v;
    const float t = v - k;
    s1 += t;
    s2 = fmaf(t, t, s2);
    n += 1.f;
  }
  __device__ __forceinline__ RowStat stat() const {
    if (n == 0.f) return RowStat{0.f, 0.f, 0.f};
    return RowStat{n, k + s1 / n, fmaxf(s2 - s1 * s1 / n, 0.f)};
  }
};
__device__ __forceinline__ RowStat warp_stat(RowStat a) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    RowStat b{__shfl_xor_sync(0xffffffffu, a.n, o), __shfl_xor_sync(0xffffffffu, a.mean, o),
              __shfl_xor_sync(0xffffffffu, a.m2, o)};
    // merge in lane order so both partners compute the same bits
    a = (threadIdx.x & o) ? stat_merge(b, a) : stat_merge(a, b);
  }
  return a;
}

}  // namespace glm
