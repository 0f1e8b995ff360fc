// digits.cuh — 16-bit fixed-point activation digits shared by the integer-MMA decode GEMVs
// (gemv.cu k_gemv_i4 / k_gemv_mk_i4, gemv_tc.cu k_gemv_tc_i4).
#pragma once
#include <cstdint>

#include <cuda_fp16.h>

namespace glm {
namespace {

constexpr float kDigitQ = 32512.f;  // 127 * 256: keeps the balanced hi digit in [-127, 127]

// One 16-k group of fragment-ordered fp16 activations (32 B, halves [j][2t, 2t+1, 2t+8, 2t+9])
// -> 16 hi digits | 16 lo digits in weight-word byte order ([j][2t, 2t+8, 2t+1, 2t+9]); returns
// the sum of the group's x_int. x_int = rint(x * inv_s) of the exact product (one FFMA onto the
// 1.5 * 2^23 + 128 magic: |x_int| <= 32512 < 2^22, so the sum rounds to the nearest even integer
// and its float bits are 0x4B400000 + x_int + 128); the low 16 bits u = x_int + 128 hold lo + 128
// in the low byte and hi in the next (two's complement), so two PRMT levels gather the 4 lo / 4
// hi bytes of a word and one LOP flips lo's sign bit; the x_int sum is 256 * sum(hi) + sum(lo)
// from two dp4a per word.
__device__ __forceinline__ int digits_regs(const uint4 h0, const uint4 h1, float inv_s, uint4& hi4, uint4& lo4) {
  const uint32_t hw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
  constexpr float kMagic = 12583040.f;  // 1.5 * 2^23 + 128
  uint32_t hi[4], lo[4];
  int shi = 0, slo = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * j]));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * j + 1]));
    const float fq[4] = {f01.x, f23.x, f01.y, f23.y};  // byte order 2t, 2t+8, 2t+1, 2t+9
    uint32_t u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = __float_as_uint(__fmaf_rn(fq[q], inv_s, kMagic));
    const uint32_t t01 = __byte_perm(u[0], u[1], 0x5410), t23 = __byte_perm(u[2], u[3], 0x5410);
    lo[j] = __byte_perm(t01, t23, 0x6420) ^ 0x80808080u;
    hi[j] = __byte_perm(t01, t23, 0x7531);
    shi = __dp4a(static_cast<int>(hi[j]), 0x01010101, shi);
    slo = __dp4a(static_cast<int>(lo[j]), 0x01010101, slo);
  }
  hi4 = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  lo4 = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  return 256 * shi + slo;
}
// in place: p[0] <- hi digits, p[1] <- lo digits
__device__ __forceinline__ int digits_group(uint4* p, float inv_s) {
  uint4 hi, lo;
  const int s = digits_regs(p[0], p[1], inv_s, hi, lo);
  p[0] = hi;
  p[1] = lo;
  return s;
}

}  // namespace
}  // namespace glm
