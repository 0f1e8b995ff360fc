// gen.cuh — counter-based synthetic weights.
//
// GLM-130B-shaped random-init weights (126.8 B parameters) cannot come from the
// reference's serial mt19937_64 stream (rng.hpp:13-63), so the GPU generates
// value(seed, tensor_id, flat) on the fly: Philox4x32-10 over counter
// (flat_lo, flat_hi, tensor_id, 0), Irwin-Hall sum of the eight 16-bit halves,
// centred, scaled to unit variance and by sigma with single IEEE float multiplies
// (explicitly rounded, no FMA contraction), rounded to bf16 (RNE). Every step is
// integer or correctly-rounded float arithmetic, so the CPU oracle
// (oracle/oracle.cpp gen_bf16) reproduces each value bit for bit.
#pragma once
#include <stdint.h>

namespace glm {

__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                         uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// bf16 bits of the synthetic weight at `flat` of tensor `tensor_id`.
__device__ __forceinline__ uint16_t gen_bf16(uint64_t seed, uint32_t tensor_id, uint64_t flat,
                                             float sigma) {
  uint32_t c0 = static_cast<uint32_t>(flat), c1 = static_cast<uint32_t>(flat >> 32), c2 = tensor_id,
           c3 = 0u;
  philox10(c0, c1, c2, c3, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const int32_t s = static_cast<int32_t>((c0 & 0xFFFFu) + (c0 >> 16) + (c1 & 0xFFFFu) + (c1 >> 16) +
                                         (c2 & 0xFFFFu) + (c2 >> 16) + (c3 & 0xFFFFu) + (c3 >> 16));
  const float z = __fmul_rn(static_cast<float>(s - 262140), 0x1.3988e2p-16f);
  const float w = __fmul_rn(z, sigma);
  uint32_t u = __float_as_uint(w);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

__device__ __forceinline__ double bf16_bits_to_double(uint16_t b) {
  return static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16));
}

// Tensor ids (oracle/oracle.cpp or_params_init_philox): layer * 8 + slot, embedding
// 0xFFFF0000; activations used by tests 0xFFFE0000 + k.
constexpr uint32_t kEmbedTensorId = 0xFFFF0000u;

}  // namespace glm
