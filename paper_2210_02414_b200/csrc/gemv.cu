// gemv.cu — W4A16 / W8A16 decode GEMV for M <= 16 tokens.
//
// Replaces `matmul(x, dequantize(q))` (quant.cpp:188-221 + tensor.cpp:135-155) on the
// decode path. HBM-bound: every weight byte is read exactly once per call.
//
//  * weights: one coalesced 512 B warp load (LDG.128 per lane, L1::no_allocate) per
//    64-deep chunk of a 16-feature row tile, in the fragment-ordered device layout of
//    layout.cuh, double-buffered in registers (next chunk group in flight while the
//    current one is transcoded);
//  * dequantisation in registers: INT4 nibbles -> fp16 with one LOP3 (|0x6400 magic)
//    and one HSUB2/HFMA2 per pair of codes, INT8 bytes with PRMT; the codes are exact
//    small integers in fp16;
//  * the K-loop reduction runs on the tensor cores: mma.sync m16n8k16 (f16 x f16 -> f32)
//    with the weights as A (16 features) and the <= 8 tokens as B, fp32 accumulation;
//  * activations arrive pre-permuted in fragment order (x_frag), 32 B per lane per
//    chunk, L1-resident across the warps of an SM;
//  * split-K over `ksplit` static slices balances the 148 SMs; partial sums go to a
//    [ksplit][M][Np] fp32 buffer reduced (with the group scale) by the consumer.
#include "common.cuh"
#include "kernels.h"

namespace glm {

namespace {

constexpr int kWarps = 8;       // warps per CTA
constexpr int kCtasPerSM = 2;   // resident CTAs per SM (128 regs/thread budget)

__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop_or_magic(uint32_t w, uint32_t mask) {
  uint32_t d;
  // d = (w & mask) | 0x64006400  (one LOP3)
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(w), "r"(mask), "r"(0x64006400u));
  return d;
}

// INT4 word -> the 4 fp16x2 A-fragment registers (codes exact).
__device__ __forceinline__ void dq4(uint32_t w, uint32_t (&a)[4]) {
  const uint32_t k1032 = 0x64086408u;                // (1032, 1032): 1024 + 8 offset
  const uint32_t k1_16 = 0x2C002C00u;                // (1/16, 1/16)
  const uint32_t kneg72 = 0xD480D480u;               // (-72, -72) = -(64 + 8)
  const uint32_t w8 = w >> 8;
  a[0] = hsub2_u32(lop_or_magic(w, 0x000F000Fu), k1032);
  a[1] = hfma2_u32(lop_or_magic(w, 0x00F000F0u), k1_16, kneg72);
  a[2] = hsub2_u32(lop_or_magic(w8, 0x000F000Fu), k1032);
  a[3] = hfma2_u32(lop_or_magic(w8, 0x00F000F0u), k1_16, kneg72);
}

// INT8 word pair -> 4 fp16x2 registers.
__device__ __forceinline__ void dq8(uint32_t w0, uint32_t w1, uint32_t (&a)[4]) {
  const uint32_t k1152 = 0x64806480u;  // (1152, 1152): 1024 + 128 offset
  a[0] = hsub2_u32(__byte_perm(w0, 0x64646464u, 0x4140), k1152);
  a[1] = hsub2_u32(__byte_perm(w0, 0x64646464u, 0x4342), k1152);
  a[2] = hsub2_u32(__byte_perm(w1, 0x64646464u, 0x4140), k1152);
  a[3] = hsub2_u32(__byte_perm(w1, 0x64646464u, 0x4342), k1152);
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct GemvArgs {
  const uint4* w;       // device layout
  const uint4* xf;      // x_frag, uint4 view, for row tiles < rt_split
  const uint4* xf2;     // x_frag for row tiles >= rt_split (fused W1|V launch)
  int64_t rt_split;
  float* partial;       // [ksplit][M][Np]
  int64_t nrt, nch, Np;
  int M, ksplit;
};

template <int BITS, int NT>
__device__ __forceinline__ void compute_chunk(const uint4 (&wv)[BITS == 4 ? 1 : 2], const uint4 (&xv)[NT][2],
                                              float (&acc)[NT][4]) {
  const uint32_t ws[4] = {wv[0].x, wv[0].y, wv[0].z, wv[0].w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t a[4];
    if constexpr (BITS == 4) {
      dq4(ws[j], a);
    } else {
      const uint4 v = j < 2 ? wv[0] : wv[1];
      const int jj = j & 1;
      dq8(jj ? v.z : v.x, jj ? v.w : v.y, a);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint4 x = xv[nt][j >> 1];
      const uint32_t b0 = (j & 1) ? x.z : x.x, b1 = (j & 1) ? x.w : x.y;
      mma16816(acc[nt], a, b0, b1);
    }
  }
}

template <int BITS, int NT>
__global__ void __launch_bounds__(kWarps * 32, kCtasPerSM) k_gemv(GemvArgs a) {
  constexpr int WV = BITS == 4 ? 1 : 2;              // uint4 weight loads per chunk per lane
  constexpr int CHUNK_U4 = BITS == 4 ? 32 : 64;      // uint4 per chunk block
  constexpr int kUnroll = BITS == 4 ? 8 : 4;         // chunks per stage: 4 KB per warp in flight
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t nitems = a.nrt * a.ksplit;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kWarps;
  bool xon[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xon[nt] = (nt * 8 + g) < a.M;

  for (int64_t item = static_cast<int64_t>(blockIdx.x) * kWarps + warp; item < nitems; item += wstride) {
    const int64_t rt = item / a.ksplit;
    const int s = static_cast<int>(item % a.ksplit);
    const int64_t c0 = a.nch * s / a.ksplit, c1 = a.nch * (s + 1) / a.ksplit;
    const uint4* wp = a.w + rt * a.nch * CHUNK_U4 + lane;
    const uint4* xfb = rt < a.rt_split ? a.xf : a.xf2;
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[nt][i] = 0.f;

    // Two named register stages (no dynamic indexing -> no local memory): while one
    // stage is transcoded + MMA'd the other stage's LDG.128s are in flight.
    uint4 wa[kUnroll][WV], wb[kUnroll][WV];
    auto load_stage = [&](uint4 (&dst)[kUnroll][WV], int64_t cs) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int v = 0; v < WV; ++v)
          dst[u][v] = (cs + u < c1) ? ld_stream(wp + (cs + u) * CHUNK_U4 + v * 32) : make_uint4(0, 0, 0, 0);
    };
    auto compute_stage = [&](const uint4 (&src)[kUnroll][WV], int64_t cs) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (cs + u < c1) {
          uint4 xv[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (xon[nt]) {
              const uint4* xp = xfb + (((nt * 8 + g) * a.nch + (cs + u)) * 4 + t) * 2;
              xv[nt][0] = ld_nc(xp);
              xv[nt][1] = ld_nc(xp + 1);
            } else {
              xv[nt][0] = make_uint4(0, 0, 0, 0);
              xv[nt][1] = make_uint4(0, 0, 0, 0);
            }
          }
          compute_chunk<BITS, NT>(src[u], xv, acc);
        }
      }
    };
    int64_t c = c0;
    load_stage(wa, c);
    for (; c < c1; c += 2 * kUnroll) {
      if (c + kUnroll < c1) load_stage(wb, c + kUnroll);
      compute_stage(wa, c);
      if (c + kUnroll >= c1) break;
      if (c + 2 * kUnroll < c1) load_stage(wa, c + 2 * kUnroll);
      compute_stage(wb, c + kUnroll);
    }
    // D fragment: rows g, g+8 (features); cols 2t, 2t+1 (tokens) of each n-tile.
    float* out = a.partial + static_cast<int64_t>(s) * a.M * a.Np + rt * kTileN;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = nt * 8 + 2 * t + (i & 1);
        const int row = g + 8 * (i >> 1);
        if (m < a.M) out[static_cast<int64_t>(m) * a.Np + row] = acc[nt][i];
      }
  }
}

__global__ void k_xfrag_from_f32(const float* __restrict__ x, int64_t ldx, int M, int64_t K, int64_t Kp,
                                 int64_t nch, const float* __restrict__ row_scale, __half* __restrict__ xf) {
  // one thread per (m, even k) pair
  const int64_t pairs = static_cast<int64_t>(M) * (Kp / 2);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / (Kp / 2));
    const int64_t k = (i % (Kp / 2)) * 2;
    const float v0 = k < K ? x[m * ldx + k] * row_scale[k] : 0.f;
    const float v1 = k + 1 < K ? x[m * ldx + k + 1] * row_scale[k + 1] : 0.f;
    *reinterpret_cast<__half2*>(xf + xfrag_index(nch, m, k)) = __floats2half2_rn(v0, v1);
  }
}

__global__ void k_gemv_reduce(const float* __restrict__ partial, int ksplit, int M, int64_t N, int64_t Np,
                              const float* __restrict__ col_scale, float* __restrict__ y, int64_t ldy) {
  const int64_t total = static_cast<int64_t>(M) * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / N);
    const int64_t n = i % N;
    float acc = 0.f;
    for (int s = 0; s < ksplit; ++s) acc += partial[(static_cast<int64_t>(s) * M + m) * Np + n];
    y[m * ldy + n] = acc * col_scale[n];
  }
}

}  // namespace

GemvPlan plan_gemv(int64_t nrt, int64_t nch) {
  GemvPlan p;
  const int64_t total_warps = static_cast<int64_t>(kNumSMs) * kCtasPerSM * kWarps;
  double best = -1.0;
  const int64_t max_split = nch < 32 ? nch : 32;
  for (int64_t ks = 1; ks <= max_split; ++ks) {
    if (nch / ks < 4 && ks > 1) break;  // keep >= 4 chunks (2 KB per lane) per item
    const int64_t items = nrt * ks;
    const int64_t waves = (items + total_warps - 1) / total_warps;
    double eff = static_cast<double>(items) / static_cast<double>(waves * total_warps);
    eff -= 0.002 * static_cast<double>(ks);  // small ksplit preferred (partial traffic)
    if (eff > best + 1e-9) {
      best = eff;
      p.ksplit = static_cast<int>(ks);
    }
  }
  const int64_t items = nrt * p.ksplit;
  const int64_t ctas = (items + kWarps - 1) / kWarps;
  const int64_t maxc = static_cast<int64_t>(kNumSMs) * kCtasPerSM;
  p.grid = static_cast<int>(ctas < maxc ? ctas : maxc);
  return p;
}

GemvPlan plan_gemv(const QLayout& L, int M) {
  (void)M;
  return plan_gemv(L.nrt, L.nch);
}

void gemv_launch(const GemvOp& op, int M, float* partial, const GemvPlan& p, cudaStream_t st) {
  if (M < 1 || M > 16) fail(GLM_DIMENSION, "qlinear", "GEMV path takes 1..16 rows, got " + std::to_string(M));
  GemvArgs a{static_cast<const uint4*>(op.codes), reinterpret_cast<const uint4*>(op.xf),
             reinterpret_cast<const uint4*>(op.xf2 ? op.xf2 : op.xf), op.xf2 ? op.rt_split : op.nrt, partial,
             op.nrt, op.nch, op.nrt * kTileN, M, p.ksplit};
  const dim3 grid(p.grid), block(kWarps * 32);
  if (op.bits == 4) {
    if (M <= 8) k_gemv<4, 1><<<grid, block, 0, st>>>(a);
    else k_gemv<4, 2><<<grid, block, 0, st>>>(a);
  } else {
    if (M <= 8) k_gemv<8, 1><<<grid, block, 0, st>>>(a);
    else k_gemv<8, 2><<<grid, block, 0, st>>>(a);
  }
  LAUNCH_CHECK("k_gemv");
}

void gemv_launch(const QWeightDev& w, const __half* xfrag, int M, float* partial, const GemvPlan& p,
                 cudaStream_t st) {
  GemvOp op{w.codes, w.L.bits, w.L.nrt, w.L.nch, xfrag, nullptr, 0};
  gemv_launch(op, M, partial, p, st);
}

void xfrag_from_f32(const float* x, int64_t ldx, int M, const QWeightDev& w, __half* xfrag, cudaStream_t st) {
  const int64_t pairs = static_cast<int64_t>(M) * (w.L.Kp / 2);
  const int grid = static_cast<int>(std::min<int64_t>((pairs + 255) / 256, 148 * 16));
  k_xfrag_from_f32<<<grid, 256, 0, st>>>(x, ldx, M, w.L.K, w.L.Kp, w.L.nch, w.row_scale, xfrag);
  LAUNCH_CHECK("k_xfrag_from_f32");
}

void gemv_reduce(const float* partial, int ksplit, int M, const QWeightDev& w, float* y, int64_t ldy,
                 cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(M) * w.L.N;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_gemv_reduce<<<grid, 256, 0, st>>>(partial, ksplit, M, w.L.N, w.L.Np, w.col_scale, y, ldy);
  LAUNCH_CHECK("k_gemv_reduce");
}

}  // namespace glm
