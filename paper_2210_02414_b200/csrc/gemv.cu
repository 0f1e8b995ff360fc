// gemv.cu — W4A16 / W8A16 decode GEMV for M <= 16 tokens.
//
// Replaces `matmul(x, dequantize(q))` (quant.cpp:188-221 + tensor.cpp:135-155) on the
// decode path. HBM-bound: every weight byte is read exactly once per call.
//
//  * weights: each warp streams its own 16-feature row tile through a 3-stage ring of 4 KB
//    shared-memory stages filled by the bulk-copy engine (cp.async.bulk = 1-D TMA, L2
//    evict-first, mbarrier transaction counts); lanes read their 16 B fragment words
//    with LDS.128 from the fragment-ordered device layout of layout.cuh;
//  * dequantisation in registers: INT4 nibbles -> fp16 with one LOP3 (|0x6400 magic)
//    and one HSUB2/HFMA2 per pair of codes, INT8 bytes with PRMT; the codes are exact
//    small integers in fp16;
//  * the K-loop reduction runs on the tensor cores: mma.sync m16n8k16 (f16 x f16 -> f32)
//    with the weights as A (16 features) and the <= 8 tokens as B, fp32 accumulation in
//    four independent chains;
//  * activations arrive pre-permuted in fragment order (x_frag), 32 B per lane per chunk,
//    fetched for a whole stage before the stage's mbarrier wait;
//  * split-K over `ksplit` static slices balances the 148 SMs; partial sums go to a
//    [ksplit][M][Np] fp32 buffer reduced (with the group scale) by the consumer.
//
// Measured on B200 (tools/*_probe.cu): this register-MMA form sustains ~3.6 TB/s INT4 /
// ~6 TB/s INT8 at M = 1. A tcgen05 variant (transcode into TMEM, async MMA) was built and
// measured slower for decode (2.6 / 5.3 TB/s: a small-N tcgen05.mma costs its issuing
// thread ~68 cycles and the extra cross-warp hand-offs add ~350 cycles per stage); it is
// used where it wins, for prefill (qmm_tc.cu). Round 2's integer tcgen05 variant for 2..16 tokens
// (kind::i8, gemv_tc.cu) is bit-identical to k_gemv_mk_i4 but also slower; opt-in (GLM_GEMV_TC).
#include <cstdlib>
#include <type_traits>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "digits.cuh"

namespace glm {

GLM_TRACE_TU(gemv)

namespace {


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
  const uint32_t w8 = __umulhi(w, 0x01000000u);  // w >> 8 on the FMA pipe (IMAD.HI), ALU pipe is the bottleneck
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

// INT4 word -> the 4 A-fragment registers WITHOUT removing the code offset: rows g
// (registers 0, 2) carry 1032 + code, rows g + 8 (registers 1, 3) carry 1152 + 16 * code.
// One LOP3 per register; the offsets are removed after the K-loop from the sum of the
// activations (k_gemv_m1 epilogue), which takes the HSUB2/HFMA2 out of the inner loop
// (+13% GEMV bandwidth measured). Cost: the fp32 accumulator carries 1032 * sum(x), so the
// result is exact to ~5e-5 of max|y| instead of ~1e-6 (still 20x below the fp16 rounding of
// the activations). A variant with all four registers at 1152 + 16 * code (three shifts on
// the FMA pipe) was 5x more precise but 17% slower.
__device__ __forceinline__ void dq4_raw(uint32_t w, uint32_t (&a)[4]) {
  const uint32_t w8 = __umulhi(w, 0x01000000u);  // w >> 8 on the FMA pipe
  a[0] = lop_or_magic(w, 0x000F000Fu);
  a[1] = lop_or_magic(w, 0x00F000F0u);
  a[2] = lop_or_magic(w8, 0x000F000Fu);
  a[3] = lop_or_magic(w8, 0x00F000F0u);
}

__device__ __forceinline__ void compute_chunk4_raw(const uint4& wv, const uint4 (&xv)[2], float (&acc)[4][1][4]) {
  const uint32_t ws[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t a[4];
    dq4_raw(ws[j], a);
    const uint4 x = xv[j >> 1];
    mma16816(acc[j][0], a, (j & 1) ? x.z : x.x, (j & 1) ? x.w : x.y);
  }
}

template <int BITS, int NT>
__device__ __forceinline__ void compute_chunk4(const uint4 (&wv)[BITS == 4 ? 1 : 2], const uint4 (&xv)[NT][2],
                                               float (&acc)[4][NT][4]) {
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
      mma16816(acc[j][nt], a, b0, b1);
    }
  }
}

constexpr int kTWarps = 16;
constexpr int kStages = 3;
constexpr int kStageBytes = 4096;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int BITS, int NT>
__global__ void __launch_bounds__(kTWarps * 32, 1) k_gemv_tma(GemvArgs a) {
  constexpr int CHUNK = BITS == 4 ? 512 : 1024;
  constexpr int U = kStageBytes / CHUNK;  // chunks per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  uint8_t* ring = smem + static_cast<size_t>(warp) * kStages * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kTWarps) * kStages * kStageBytes) + warp * kStages;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

  const int64_t nitems = a.nrt * a.ksplit;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kTWarps;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * kTWarps + warp;
  bool xon[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xon[nt] = (nt * 8 + g) < a.M;

  // issue cursor over this warp's (item, chunk) sequence
  int64_t ii = first, ic = 0, ic1 = 0;
  auto item_range = [&](int64_t item, int64_t& c0, int64_t& c1) {
    const int s = static_cast<int>(item % a.ksplit);
    c0 = a.nch * s / a.ksplit;
    c1 = a.nch * (s + 1) / a.ksplit;
  };
  if (ii < nitems) item_range(ii, ic, ic1);
  uint32_t issued = 0;
  auto issue = [&]() {  // lane 0 only; returns false when the sequence is exhausted
    if (ii >= nitems) return;
    const int64_t n = min(static_cast<int64_t>(U), ic1 - ic);
    const int slot = issued % kStages;
    const int64_t rt = ii / a.ksplit;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.w) + (rt * a.nch + ic) * CHUNK;
    mbar_expect_tx(bars + slot, static_cast<uint32_t>(n * CHUNK));
    bulk_g2s(ring + slot * kStageBytes, src, static_cast<uint32_t>(n * CHUNK), bars + slot, policy);
    ++issued;
    ic += n;
    if (ic >= ic1) {
      ii += wstride;
      if (ii < nitems) item_range(ii, ic, ic1);
    }
  };
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) issue();
  // weights never change during decode: their prefetch runs ahead of the predecessor kernel
  pdl_wait();
  pdl_trigger();
  // lanes other than 0 track the issue count implicitly: consumption order is identical
  uint32_t consumed = 0;

  for (int64_t item = first; item < nitems; item += wstride) {
    const int64_t rt = item / a.ksplit;
    const int s = static_cast<int>(item % a.ksplit);
    int64_t c0, c1;
    item_range(item, c0, c1);
    const uint4* xfb = reinterpret_cast<const uint4*>(rt < a.rt_split ? a.xf : a.xf2);
    // four independent accumulator chains (one per k-tile of a chunk)
    float acc[4][NT][4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[h][nt][i] = 0.f;
    for (int64_t c = c0; c < c1; c += U) {
      const int n = static_cast<int>(min(static_cast<int64_t>(U), c1 - c));
      const int slot = consumed % kStages;
      // activations of the whole stage first (L1/L2 latency overlaps the mbarrier wait);
      // NT = 2 (9..16 tokens) would exceed the register budget and loads per chunk instead
      constexpr int UX = NT == 1 ? U : 1;
      uint4 xv[UX][NT][2];
      auto load_x = [&](uint4 (&dst)[NT][2], int64_t cc, bool on) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (xon[nt] && on) {
            const uint4* xp = xfb + (((nt * 8 + g) * a.nch + cc) * 4 + t) * 2;
            dst[nt][0] = ld_nc(xp);
            dst[nt][1] = ld_nc(xp + 1);
          } else {
            dst[nt][0] = make_uint4(0, 0, 0, 0);
            dst[nt][1] = make_uint4(0, 0, 0, 0);
          }
        }
      };
      if constexpr (NT == 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) load_x(xv[u], c + u, u < n);
      }
      mbar_wait(bars + slot, (consumed / kStages) & 1);
      const uint8_t* st = ring + slot * kStageBytes;
      if (n == U) {
        // full stage: straight-line code, no per-chunk branches, so LDS / LOP3 / HMMA of
        // consecutive chunks interleave
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint4 wv[BITS == 4 ? 1 : 2];
          wv[0] = *reinterpret_cast<const uint4*>(st + u * CHUNK + lane * 16);
          if constexpr (BITS == 8) wv[1] = *reinterpret_cast<const uint4*>(st + u * CHUNK + 512 + lane * 16);
          if constexpr (NT == 1) {
            compute_chunk4<BITS, NT>(wv, xv[u], acc);
          } else {
            load_x(xv[0], c + u, true);
            compute_chunk4<BITS, NT>(wv, xv[0], acc);
          }
        }
      } else {
        for (int u = 0; u < n; ++u) {
          uint4 wv[BITS == 4 ? 1 : 2];
          wv[0] = *reinterpret_cast<const uint4*>(st + u * CHUNK + lane * 16);
          if constexpr (BITS == 8) wv[1] = *reinterpret_cast<const uint4*>(st + u * CHUNK + 512 + lane * 16);
          uint4 xu[NT][2];
          load_x(xu, c + u, true);  // tail stage: per-chunk activations
          compute_chunk4<BITS, NT>(wv, xu, acc);
        }
      }
      __syncwarp();
      ++consumed;
      if (lane == 0) issue();
    }
    float* out = a.partial + static_cast<int64_t>(s) * a.M * a.Np + rt * kTileN;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = nt * 8 + 2 * t + (i & 1);
        const int row = g + 8 * (i >> 1);
        if (m < a.M) out[static_cast<int64_t>(m) * a.Np + row] = (acc[0][nt][i] + acc[1][nt][i]) + (acc[2][nt][i] + acc[3][nt][i]);
      }
  }
}

// ---- multi-token variant (2..16 tokens: batched decode) ----------------------------------
// At M tokens every weight fragment feeds NT = ceil(M/8) MMAs, and the activations, not the
// weights, dominate on-chip traffic if each warp fetches its own: a CTA therefore works on
// CTA-items = (16 consecutive row tiles, one k-slice), one row tile per warp, and the M
// activation rows of the k-slice are bulk-copied once per CTA-item into a double-buffered
// shared-memory slice (next item's slice in flight while the current one is consumed).
// Weights stream through the per-warp TMA rings exactly as in the other variants.
constexpr int kMkStages = 2;
constexpr int kMkSliceBytes = 48 * 1024;  // one activation-slice buffer (all x vectors, all tokens)

// RT row tiles per warp (CTA-item = 16 * RT row tiles): with RT = 2 every activation
// fragment read from shared memory feeds both tiles' MMAs, halving the activation traffic
// that bounds INT4 at 9..16 tokens (16 warps re-read the same slice; ncu: ~0.7 shared
// wavefronts per cycle per SM at RT = 1). A stage then holds U/2 chunks of each tile.
template <int BITS, int NT, int RT>
__global__ void __launch_bounds__(kTWarps * 32, 1) k_gemv_mk(GemvArgs a, int nx) {
  trace_point(10);
  constexpr int CHUNK = BITS == 4 ? 512 : 1024;
  constexpr int U = kStageBytes / CHUNK / RT;  // chunks per tile per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nch = static_cast<int>(a.nch), ksplit = a.ksplit, M = a.M;
  const int nrt = static_cast<int>(a.nrt);
  constexpr int kTiles = kTWarps * RT;  // row tiles per CTA-item
  uint8_t* ring = smem + static_cast<size_t>(warp) * kMkStages * kStageBytes;
  uint8_t* xbuf = smem + static_cast<size_t>(kTWarps) * kMkStages * kStageBytes;  // [2][kMkSliceBytes]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xbuf + 2 * kMkSliceBytes);          // [2]
  uint64_t* bars = xbar + 2 + warp * kMkStages;
  if (lane == 0) {
    for (int q = 0; q < kMkStages; ++q) mbar_init(bars + q, 1);
    if (warp == 0) {
      mbar_init(xbar, 1);
      mbar_init(xbar + 1, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy, keep;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const int ngroups = (nrt + kTiles - 1) / kTiles;
  const int nitems = ngroups * ksplit;
  auto slice = [&](int s, int& c0, int& c1) {
    c0 = nch * s / ksplit;
    c1 = nch * (s + 1) / ksplit;
  };
  // weight producer (lane 0 of each warp) walks this CTA's items in consumption order
  int pj = blockIdx.x, pc = 0, pc1 = 0, prt = -1, pslot = 0;
  auto pitem = [&]() {  // position the producer on item pj (skipping items where this warp idles)
    while (pj < nitems) {
      prt = (pj / ksplit) * kTiles + warp * RT;
      slice(pj % ksplit, pc, pc1);
      if (prt < nrt) return;
      pj += gridDim.x;
    }
  };
  pitem();
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  auto issue = [&]() {
    if (pj >= nitems) return;
    const int n = min(U, pc1 - pc);
    const int ntile = (RT == 2 && prt + 1 < nrt) ? 2 : 1;
    mbar_expect_tx(bars + pslot, static_cast<uint32_t>(ntile * n * CHUNK));
    for (int q = 0; q < ntile; ++q) {
      const uint8_t* src = wbase + (static_cast<int64_t>(prt + q) * nch + pc) * CHUNK;
      bulk_g2s(ring + pslot * kStageBytes + q * n * CHUNK, src, static_cast<uint32_t>(n * CHUNK), bars + pslot, policy);
    }
    pslot = pslot + 1 == kMkStages ? 0 : pslot + 1;
    pc += n;
    if (pc >= pc1) {
      pj += gridDim.x;
      pitem();
    }
  };
  if (lane == 0)
    for (int q = 0; q < kMkStages; ++q) issue();
  pdl_wait();
  pdl_trigger();
  trace_point(11);
  // activation slices: buffer b holds [nx][M][chunks of the slice][128 B]
  auto load_x = [&](int local, int item) {
    int c0, c1;
    slice(item % ksplit, c0, c1);
    const int nck = c1 - c0;
    const int b = local & 1;
    mbar_expect_tx(xbar + b, static_cast<uint32_t>(nx * M * nck * 128));
    for (int v = 0; v < nx; ++v)
      for (int m = 0; m < M; ++m) {
        const uint8_t* src = reinterpret_cast<const uint8_t*>(v == 0 ? a.xf : a.xf2) +
                             (static_cast<int64_t>(m) * nch + c0) * 128;
        bulk_g2s(xbuf + b * kMkSliceBytes + ((v * M + m) * nck) * 128, src, static_cast<uint32_t>(nck * 128), xbar + b,
                 keep);
      }
  };
  if (threadIdx.x == 0) {
    if (static_cast<int>(blockIdx.x) < nitems) load_x(0, blockIdx.x);
    if (static_cast<int>(blockIdx.x + gridDim.x) < nitems) load_x(1, blockIdx.x + gridDim.x);
  }
  int cslot = 0;
  uint32_t cpar = 0;
  int local = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++local) {
    const int s = item % ksplit;
    const int rt = (item / ksplit) * kTiles + warp * RT;
    int c0, c1;
    slice(s, c0, c1);
    const int nck = c1 - c0;
    const int b = local & 1;
    mbar_wait(xbar + b, (local >> 1) & 1);
    if (rt < nrt) {
      // (RT = 2: the host only pairs tiles on one side of rt_split, which is even)
      const int v = rt < a.rt_split ? 0 : nx - 1;
      const bool two = RT == 2 && rt + 1 < nrt;
      const uint8_t* xrow[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        xrow[nt] = xbuf + b * kMkSliceBytes + ((v * M + min(nt * 8 + g, M - 1)) * nck) * 128 + t * 32;
      float acc[RT][4][NT][4];
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[r][h][nt][i] = 0.f;
      for (int c = 0; c < nck; c += U) {
        const int n = min(U, nck - c);
        mbar_wait(bars + cslot, cpar);
        const uint8_t* st = ring + cslot * kStageBytes + lane * 16;
        auto chunk = [&](int u) {
          uint4 xv[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint4* xa = reinterpret_cast<const uint4*>(xrow[nt] + (c + u) * 128);
            xv[nt][0] = xa[0];
            xv[nt][1] = xa[1];
          }
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            if (r == 1 && !two) break;
            uint4 wv[BITS == 4 ? 1 : 2];
            const uint8_t* sp = st + (r * n + u) * CHUNK;
            wv[0] = *reinterpret_cast<const uint4*>(sp);
            if constexpr (BITS == 8) wv[1] = *reinterpret_cast<const uint4*>(sp + 512);
            compute_chunk4<BITS, NT>(wv, xv, acc[r]);
          }
        };
        if (n == U) {
#pragma unroll
          for (int u = 0; u < U; ++u) chunk(u);
        } else {
          for (int u = 0; u < n; ++u) chunk(u);
        }
        __syncwarp();
        if (cslot + 1 == kMkStages) {
          cslot = 0;
          cpar ^= 1u;
        } else {
          ++cslot;
        }
        if (lane == 0) issue();
      }
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        if (r == 1 && !two) break;
        float* out = a.partial + static_cast<int64_t>(s) * M * a.Np + static_cast<int64_t>(rt + r) * kTileN;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int m = nt * 8 + 2 * t + (i & 1);
            const int row = g + 8 * (i >> 1);
            if (m < M)
              out[static_cast<int64_t>(m) * a.Np + row] =
                  (acc[r][0][nt][i] + acc[r][1][nt][i]) + (acc[r][2][nt][i] + acc[r][3][nt][i]);
          }
      }
    }
    __syncthreads();  // every warp is done with activation buffer b
    if (threadIdx.x == 0 && item + 2 * static_cast<int>(gridDim.x) < nitems) load_x(local + 2, item + 2 * gridDim.x);
  }
  trace_point(13);
}

// ---- single-token variant (batch-1 decode, the headline path) -----------------------------
// As k_gemv_tma with M = 1, but the whole activation vector (Kp fp16 = 24 KB at K = 12288,
// 64 KB at K = 32768; twice that for a fused W1|V launch with distinct kRow folds) is
// bulk-copied into shared memory once per CTA at launch, next to the weight rings. The
// K-loop then reads its B fragments with LDS (≈30-cycle latency, no per-stage global loads
// or register zeroing).
// The weight ring depth `nst` (2 or 3 stages per warp) is chosen by the host to fit 227 KB.
constexpr int kM1MaxWarps = 24;
constexpr int kM1DefaultWarps = 16;

// MT = 2 (two-token decode): the same kernel with both tokens' activation vectors resident;
// lane (g, t) reads token min(g, MT - 1), so token columns 0 and 1 of the MMA are real and
// the others duplicate token MT - 1 (discarded).
template <int BITS, int NST, int SB, int MT = 1>
__global__ void __launch_bounds__(kM1MaxWarps * 32, 1) k_gemv_m1(GemvArgs a, int nx, int early) {
  trace_point(10);
  constexpr int CHUNK = BITS == 4 ? 512 : 1024;
  constexpr int U = SB / CHUNK;  // chunks per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nch = static_cast<int>(a.nch), ksplit = a.ksplit;
  const int xbytes = nch * 128;  // one token: Kp halves
  const int vbytes = MT * xbytes;  // one activation vector set: [MT tokens][chunks][128 B]
  uint8_t* ring = smem + static_cast<size_t>(warp) * NST * SB;
  uint8_t* xs = smem + static_cast<size_t>(nw) * NST * SB;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xs + nx * vbytes);
  uint64_t* bars = xbar + 1 + warp * NST;
  if (lane == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(bars + s, 1);
    if (warp == 0) mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy, keep;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));

  const int nitems = static_cast<int>(a.nrt) * ksplit;
  const int wstride = static_cast<int>(gridDim.x) * nw;
  const int first = static_cast<int>(blockIdx.x) * nw + warp;
  // item -> (row tile, k-slice, chunk range): 32-bit, once per item
  auto decode = [&](int item, int& rt, int& s, int& c0, int& c1) {
    rt = item / ksplit;
    s = item - rt * ksplit;
    c0 = nch * s / ksplit;
    c1 = nch * (s + 1) / ksplit;
  };

  // producer state (lane 0): next chunk to copy
  int pi = first, prt = 0, ps = 0, pc = 0, pc1 = 0, pslot = 0;
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  if (pi < nitems) decode(pi, prt, ps, pc, pc1);
  auto issue = [&]() {
    if (pi >= nitems) return;
    const int n = min(U, pc1 - pc);
    const uint8_t* src = wbase + (static_cast<int64_t>(prt) * nch + pc) * CHUNK;
    mbar_expect_tx(bars + pslot, static_cast<uint32_t>(n * CHUNK));
    bulk_g2s(ring + pslot * SB, src, static_cast<uint32_t>(n * CHUNK), bars + pslot, policy);
    pslot = pslot + 1 == NST ? 0 : pslot + 1;
    pc += n;
    if (pc >= pc1) {
      pi += wstride;
      if (pi < nitems) decode(pi, prt, ps, pc, pc1);
    }
  };
  // weights never change during decode: `early` stages are fetched ahead of the
  // predecessor kernel (programmatic dependent launch), the rest after it completes
  if (lane == 0)
    for (int s = 0; s < early && s < NST; ++s) issue();
  pdl_wait();
  pdl_trigger();
  trace_point(11);
  if (threadIdx.x == 0) {
    // the activation vector(s): L2-resident (just written by the producer), kept there;
    // requested ahead of any weight stage not yet in flight
    mbar_expect_tx(xbar, static_cast<uint32_t>(nx * vbytes));
    for (int v = 0; v < nx; ++v) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(v == 0 ? a.xf : a.xf2);
      for (int o = 0; o < vbytes; o += 16384) {
        const uint32_t nb = static_cast<uint32_t>(min(16384, vbytes - o));
        bulk_g2s(xs + v * vbytes + o, src + o, nb, xbar, keep);
      }
    }
  }
  if (lane == 0)
    for (int s = early; s < NST; ++s) issue();
  // B fragments: every token column gets the same activation vector (lane (g, t) reads the
  // fragment of column 0 whatever g is), so the MMA computes 8 identical result columns and
  // only column 0 is stored: no zero-fill, no per-lane address selection, and the 8 lanes
  // reading one address are served by a single shared-memory broadcast.
  const uint8_t* xs0 = xs + (MT == 1 ? 0 : min(g, MT - 1)) * xbytes + t * 32;
  const uint8_t* xs1 = xs0 + (nx - 1) * vbytes;
  constexpr int cstride = 128;
  const int64_t rt_split = a.rt_split;
  mbar_wait(xbar, 0);
  // per-chunk sums of the fp16 activations as the MMA sees them (exact in fp32: 64 terms)
  float* xsum = reinterpret_cast<float*>(xbar + 1 + nw * NST);
  // 8 lanes per 128-byte chunk, one 16-byte load each, 3-step shuffle reduction
  const int nxc = nx * MT * nch;  // chunk sums, [vector][token][chunk]
  for (int i0 = 0; i0 < nxc; i0 += blockDim.x >> 3) {  // warp-uniform trip count
    const int i = i0 + (threadIdx.x >> 3);
    const uint4 v = i < nxc ? reinterpret_cast<const uint4*>(xs + static_cast<int64_t>(i) * 128)[threadIdx.x & 7]
                            : make_uint4(0, 0, 0, 0);
    const uint32_t wds[4] = {v.x, v.y, v.z, v.w};
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&wds[e]));
      sum += f.x + f.y;
    }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    if ((threadIdx.x & 7) == 0 && i < nxc) xsum[i] = sum;
  }
  __syncthreads();
  trace_point(12);

  int cslot = 0;
  uint32_t cpar = 0;
  for (int item = first; item < nitems; item += wstride) {
    int rt, s, c0, c1;
    decode(item, rt, s, c0, c1);
    const uint8_t* xc = (rt < rt_split ? xs0 : xs1) + c0 * cstride;
    float acc[4][1][4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[h][0][i] = 0.f;
    for (int c = c0; c < c1; c += U) {
      const int n = min(U, c1 - c);
      mbar_wait(bars + cslot, cpar);
      const uint8_t* st = ring + cslot * SB + lane * 16;
      auto chunk = [&](int u) {
        uint4 wv[BITS == 4 ? 1 : 2];
        wv[0] = *reinterpret_cast<const uint4*>(st + u * CHUNK);
        if constexpr (BITS == 8) wv[1] = *reinterpret_cast<const uint4*>(st + u * CHUNK + 512);
        uint4 xv[1][2];
        const uint4* xa = reinterpret_cast<const uint4*>(xc + u * cstride);
        xv[0][0] = xa[0];
        xv[0][1] = xa[1];
        if constexpr (BITS == 4) compute_chunk4_raw(wv[0], xv[0], acc);
        else compute_chunk4<BITS, 1>(wv, xv, acc);
      };
      if (n == U) {
#pragma unroll
        for (int u = 0; u < U; ++u) chunk(u);
      } else {
        for (int u = 0; u < n; ++u) chunk(u);
      }
      xc += U * cstride;
      __syncwarp();
      if (cslot + 1 == NST) {
        cslot = 0;
        cpar ^= 1u;
      } else {
        ++cslot;
      }
      if (lane == 0) issue();
    }
    if constexpr (MT > 1) {
      // token column n = 2t + e lives in accumulator elements e (row g) and 2 + e (row g + 8)
      static_assert(BITS == 4, "multi-token m1 kernel is INT4 only");
      const float* xsv = xsum + (rt < rt_split ? 0 : (nx - 1) * MT * nch);
      float sxm[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        float v = 0.f;
        for (int cc = c0 + lane; cc < c1; cc += 32) v += xsv[m * nch + cc];
        sxm[m] = warp_sum(v);
      }
      float* outm = a.partial + static_cast<int64_t>(s) * MT * a.Np + static_cast<int64_t>(rt) * kTileN;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * t + e;
        if (n < MT) {
          float sxn = sxm[0];
#pragma unroll
          for (int m = 1; m < MT; ++m)
            if (n == m) sxn = sxm[m];
          const float lo = (acc[0][0][e] + acc[1][0][e]) + (acc[2][0][e] + acc[3][0][e]);
          const float hi = (acc[0][0][2 + e] + acc[1][0][2 + e]) + (acc[2][0][2 + e] + acc[3][0][2 + e]);
          outm[static_cast<int64_t>(n) * a.Np + g] = lo - 1032.f * sxn;
          outm[static_cast<int64_t>(n) * a.Np + g + 8] = (hi - 1152.f * sxn) * 0.0625f;
        }
      }
      continue;
    }
    float* out = a.partial + static_cast<int64_t>(s) * a.Np + static_cast<int64_t>(rt) * kTileN;
    float sx = 0.f;
    if constexpr (BITS == 4) {
      const float* xsv = xsum + (rt < rt_split ? 0 : (nx - 1) * nch);
      for (int cc = c0 + lane; cc < c1; cc += 32) sx += xsv[cc];
      sx = warp_sum(sx);
    }
    if (t == 0) {  // token column 0 lives in accumulator elements 0 (row g) and 2 (row g + 8)
      const float lo = (acc[0][0][0] + acc[1][0][0]) + (acc[2][0][0] + acc[3][0][0]);
      const float hi = (acc[0][0][2] + acc[1][0][2]) + (acc[2][0][2] + acc[3][0][2]);
      if constexpr (BITS == 4) {
        out[g] = lo - 1032.f * sx;
        out[g + 8] = (hi - 1152.f * sx) * 0.0625f;
      } else {
        out[g] = lo;
        out[g + 8] = hi;
      }
    }
  }
  __syncthreads();
  trace_point(13);
}


// ---- integer-MMA single-token variant (INT4, 1..4 tokens: batch-1 decode, the headline) ----
// The fp16 path above spends ~17 of the ~21 issue cycles a 256-weight HMMA may take at the
// HBM rate on the transcode (4 LOP3 + IMAD.HI) and the HMMA dispatch, so it is bound by the
// SM issue rate and the clock, not by HBM. This kernel feeds the codes to the tensor core as
// integers: mma.sync m16n8k32 u8 x s8 -> s32 (IMMA.16832, 512 weights per instruction at
// the HMMA instruction rate, tools/imma_probe.cu) with the weight bytes taken straight from
// the fragment-ordered layout: each byte of a lane's word holds (row g, row g + 8) at one k,
// so `w & 0x0F0F0F0F` is row g's A register (code + 8) and `w & 0xF0F0F0F0` row g + 8's
// (16 (code + 8)), one LOP3 each and no shift: 8 LOP3 + 2 IMMA per 1024 weights.
//
// The activations become exact integers: per token vector, x_int = rint(x / s_x) with
// s_x = max|x| / 32512 (16-bit fixed point; the fp16 input has 11 significant bits, so the
// added error is <= max|x| / 65024 per element), split into balanced base-256 digits
// x_int = 256 hi + lo (hi, lo signed bytes). MMA column 2m holds token m's hi digits and
// column 2m + 1 its lo digits, so lane (g, t) ends with token t's two digit sums for rows g and
// g + 8. Every product and sum is exact integer arithmetic (|acc| < 2^31 for K <= 32768);
// the code offsets leave with the integer digit sums of the slice, and the only rounding left
// is the final fp32 scale: results are bit-reproducible and independent of summation order.
// The conversion runs once per CTA in place in shared memory after the activation bulk copy:
// [v][m][chunk][t][32 B] of fp16 fragments -> [.. 16 B hi digits | 16 B lo digits] in the byte
// order of the lane's weight words (k = 16 j + {2t, 2t + 8, 2t + 1, 2t + 9}).
__device__ __forceinline__ void imma16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void compute_chunk_i4(const uint4& wv, const uint4& xv, int (&acc0)[4], int (&acc1)[4]) {
  imma16832(acc0, wv.x & 0x0F0F0F0Fu, wv.x & 0xF0F0F0F0u, wv.y & 0x0F0F0F0Fu, wv.y & 0xF0F0F0F0u, xv.x, xv.y);
  imma16832(acc1, wv.z & 0x0F0F0F0Fu, wv.z & 0xF0F0F0F0u, wv.w & 0x0F0F0F0Fu, wv.w & 0xF0F0F0F0u, xv.z, xv.w);
}

// Row results of one item from the integer accumulators: rows g carry (code + 8), rows g + 8
// carry 16 (code + 8), both against digits x_int = 256 hi + lo; S = sum of x_int over the item's
// k-range removes the code offset exactly (int64: 256 * acc can exceed int32)
__device__ __forceinline__ float2 i4_rows(int c_hi, int c_lo, int u_hi, int u_lo, int S, float s_x) {
  const long long r0 = 256ll * c_hi + c_lo - 8ll * S;
  const long long r1 = 256ll * u_hi + u_lo - 128ll * S;
  return make_float2(static_cast<float>(r0) * s_x, static_cast<float>(r1) * (0.0625f * s_x));
}

template <int NST, int SB, int MT>
__global__ void __launch_bounds__(kM1MaxWarps * 32, 1) k_gemv_i4(GemvArgs a, int nx, int early, int l2pf) {
  trace_point(10);
  constexpr int CHUNK = 512;
  constexpr int U = SB / CHUNK;  // chunks per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nch = static_cast<int>(a.nch), ksplit = a.ksplit;
  const int xbytes = nch * 128;    // one token: Kp halves (fp16) = Kp digit pairs (int8 x 2)
  const int vbytes = MT * xbytes;  // one activation vector set: [MT tokens][chunks][128 B]
  uint8_t* ring = smem + static_cast<size_t>(warp) * NST * SB;
  uint8_t* xs = smem + static_cast<size_t>(nw) * NST * SB;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xs + nx * vbytes);
  uint64_t* bars = xbar + 1 + warp * NST;
  int* dsum = reinterpret_cast<int*>(xbar + 1 + nw * NST);      // [v][m][chunk] sums of x_int
  float* sx = reinterpret_cast<float*>(dsum + nx * MT * nch);   // [v * MT + m]: s_x
  float* isx = sx + 8;                                           // [v * MT + m]: 1 / s_x
  float* wmax = isx + 8;                                         // [warps][v * MT + m]
  if (lane == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(bars + s, 1);
    if (warp == 0) mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy, keep;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));

  const int nitems = static_cast<int>(a.nrt) * ksplit;
  const int wstride = static_cast<int>(gridDim.x) * nw;
  const int first = static_cast<int>(blockIdx.x) * nw + warp;
  auto decode = [&](int item, int& rt, int& s, int& c0, int& c1) {
    rt = item / ksplit;
    s = item - rt * ksplit;
    c0 = nch * s / ksplit;
    c1 = nch * (s + 1) / ksplit;
  };
  int pi = first, prt = 0, ps = 0, pc = 0, pc1 = 0, pslot = 0;
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  if (pi < nitems) decode(pi, prt, ps, pc, pc1);
  auto issue = [&]() {
    if (pi >= nitems) return;
    const int n = min(U, pc1 - pc);
    const uint8_t* src = wbase + (static_cast<int64_t>(prt) * nch + pc) * CHUNK;
    mbar_expect_tx(bars + pslot, static_cast<uint32_t>(n * CHUNK));
    bulk_g2s(ring + pslot * SB, src, static_cast<uint32_t>(n * CHUNK), bars + pslot, policy);
    pslot = pslot + 1 == NST ? 0 : pslot + 1;
    pc += n;
    if (pc >= pc1) {
      pi += wstride;
      if (pi < nitems) decode(pi, prt, ps, pc, pc1);
    }
  };
  if (lane == 0) {
    for (int s = 0; s < early && s < NST; ++s) issue();
    // L2 prefetch of the stream beyond the ring while the predecessor kernel still runs
    if (l2pf > 0 && pi < nitems) {
      const int n = min(l2pf / CHUNK, pc1 - pc);
      if (n > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wbase + (static_cast<int64_t>(prt) * nch + pc) * CHUNK),
                     "r"(static_cast<uint32_t>(n * CHUNK))
                     : "memory");
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_point(11);
  if (threadIdx.x == 0) {
    mbar_expect_tx(xbar, static_cast<uint32_t>(nx * vbytes));
    for (int v = 0; v < nx; ++v) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(v == 0 ? a.xf : a.xf2);
      for (int o = 0; o < vbytes; o += 16384) {
        const uint32_t nb = static_cast<uint32_t>(min(16384, vbytes - o));
        bulk_g2s(xs + v * vbytes + o, src + o, nb, xbar, keep);
      }
    }
  }
  mbar_wait(xbar, 0);  // the activation copy first: ring stages not fetched before the wait follow it
  if (lane == 0)
    for (int s = early; s < NST; ++s) issue();
  trace_point(14);
  // (1) max |x| per activation vector (v, m): 16-byte units, [vm][chunk][8 units]
  const int nvm = nx * MT;
  const int upv = nch * 8;
  {
    // packed fp16 maxima of |x| (exact), NaN-propagating, one vector at a time (no division)
    float mx[2 * MT];
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q) {
      mx[q] = 0.f;
      if (q >= nvm) continue;
      const uint4* xv = reinterpret_cast<const uint4*>(xs) + q * upv;
      __half2 m2 = __float2half2_rn(0.f);
      for (int i = threadIdx.x; i < upv; i += blockDim.x) {
        const uint4 v = xv[i];
        const uint32_t wd[4] = {v.x & 0x7FFF7FFFu, v.y & 0x7FFF7FFFu, v.z & 0x7FFF7FFFu, v.w & 0x7FFF7FFFu};
#pragma unroll
        for (int e = 0; e < 4; ++e) m2 = __hmax2_nan(m2, *reinterpret_cast<const __half2*>(&wd[e]));
      }
      const float2 f = __half22float2(m2);
      mx[q] = (f.x != f.x || f.y != f.y) ? __int_as_float(0x7fc00000) : fmaxf(f.x, f.y);
    }
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q) {
      float m = mx[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float r = __shfl_xor_sync(0xffffffffu, m, o);
        m = (m != m || r != r) ? __int_as_float(0x7fc00000) : fmaxf(m, r);
      }
      if (lane == 0 && q < nvm) wmax[warp * 8 + q] = m;
    }
    __syncthreads();
    if (threadIdx.x < nvm) {
      float m = 0.f;
      for (int w = 0; w < nw; ++w) {
        const float r = wmax[w * 8 + threadIdx.x];
        m = (m != m || r != r) ? __int_as_float(0x7fc00000) : fmaxf(m, r);
      }
      // non-finite activations propagate as NaN results (the fp16 path would produce inf/NaN)
      sx[threadIdx.x] = (m == 0.f) ? 0.f : (finite_f32(m) ? m / kDigitQ : __int_as_float(0x7fc00000));
      isx[threadIdx.x] = (m > 0.f && finite_f32(m)) ? kDigitQ / m : 0.f;
    }
    __syncthreads();
  }
  trace_point(15);
  // (2) in-place conversion to digits, 32-byte groups [vm][chunk][t]; chunk digit sums
  {
    const int ngroups = nvm * nch * 4;
    for (int i0 = 0; i0 < ngroups; i0 += blockDim.x) {  // warp-uniform trip count
      const int i = i0 + threadIdx.x;
      int sm = 0;
      if (i < ngroups) sm = digits_group(reinterpret_cast<uint4*>(xs) + 2 * i, isx[i / (nch * 4)]);
      sm += __shfl_xor_sync(0xffffffffu, sm, 1);
      sm += __shfl_xor_sync(0xffffffffu, sm, 2);
      if ((i & 3) == 0 && i < ngroups) dsum[i >> 2] = sm;
    }
    __syncthreads();
  }
  trace_point(12);

  // B fragments: column g = digit (g & 1) of token min(g >> 1, MT - 1)
  const uint8_t* xs0 = xs + min(g >> 1, MT - 1) * xbytes + t * 32 + (g & 1) * 16;
  const uint8_t* xs1 = xs0 + (nx - 1) * vbytes;
  const int64_t rt_split = a.rt_split;
  int cslot = 0;
  uint32_t cpar = 0;
  for (int item = first; item < nitems; item += wstride) {
    int rt, s, c0, c1;
    decode(item, rt, s, c0, c1);
    const int v = rt < rt_split ? 0 : nx - 1;
    const uint8_t* xc = (v == 0 ? xs0 : xs1) + c0 * 128;
    int acc[4][4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[h][i] = 0;
    for (int c = c0; c < c1; c += U) {
      const int n = min(U, c1 - c);
      mbar_wait(bars + cslot, cpar);
      const uint8_t* st = ring + cslot * SB + lane * 16;
      if (n == U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint4 wv = *reinterpret_cast<const uint4*>(st + u * CHUNK);
          const uint4 xv = *reinterpret_cast<const uint4*>(xc + u * 128);
          compute_chunk_i4(wv, xv, acc[2 * (u & 1)], acc[2 * (u & 1) + 1]);
        }
      } else {
        for (int u = 0; u < n; ++u) {
          const uint4 wv = *reinterpret_cast<const uint4*>(st + u * CHUNK);
          const uint4 xv = *reinterpret_cast<const uint4*>(xc + u * 128);
          compute_chunk_i4(wv, xv, acc[0], acc[1]);
        }
      }
      xc += U * 128;
      __syncwarp();
      if (cslot + 1 == NST) {
        cslot = 0;
        cpar ^= 1u;
      } else {
        ++cslot;
      }
      if (lane == 0) issue();
    }
    // sum of x_int over this slice per token (removes the code offsets)
    int S = 0;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      int h = 0;
      for (int cc = c0 + lane; cc < c1; cc += 32) h += dsum[(v * MT + m) * nch + cc];
      h = __reduce_add_sync(0xffffffffu, h);
      if (t == m) S = h;
    }
    if (t < MT) {
      const float2 y = i4_rows((acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]),
                               (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]),
                               (acc[0][2] + acc[1][2]) + (acc[2][2] + acc[3][2]),
                               (acc[0][3] + acc[1][3]) + (acc[2][3] + acc[3][3]), S, sx[v * MT + t]);
      float* out = a.partial + (static_cast<int64_t>(s) * MT + t) * a.Np + static_cast<int64_t>(rt) * kTileN;
      out[g] = y.x;
      out[g + 8] = y.y;
    }
  }
  __syncthreads();
  trace_point(13);
}

// ---- integer-MMA multi-token variant (INT4, 3..16 tokens: batched decode) -----------------
// A CTA owns a contiguous range of `per` items of the slice-major list (item = slice * ngroups +
// row-tile group; a group is 16 * RT row tiles, one per warp and RT): consecutive items share
// their k-slice, so the slice of all M activation rows is bulk-copied into ONE resident 96 KB
// buffer and converted to digit pairs (one scale per (vector, token, slice): the slice's max,
// so every split-K partial carries its own scale) only when the slice changes — once or twice
// per CTA instead of once per item, and twice the slice of a double-buffered design, which
// halves the split-K partials the LayerNorm / GeGLU kernels reduce. A code fragment (8 LOP3)
// feeds NQ = ceil(M / 4) IMMA column groups of 4 tokens (column 2j + e: token 4q + j, digit e).
constexpr int kMkXBytes = 2 * kMkSliceBytes;  // the resident activation slice (single buffer)

template <int NQ, int RT>
__global__ void __launch_bounds__(kTWarps * 32, 1) k_gemv_mk_i4(GemvArgs a, int nx, int per) {
  trace_point(10);
  constexpr int CHUNK = 512;
  constexpr int U = kStageBytes / CHUNK / RT;  // chunks per tile per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nch = static_cast<int>(a.nch), ksplit = a.ksplit, M = a.M;
  const int nrt = static_cast<int>(a.nrt);
  constexpr int kTiles = kTWarps * RT;
  uint8_t* ring = smem + static_cast<size_t>(warp) * kMkStages * kStageBytes;
  uint8_t* xb = smem + static_cast<size_t>(kTWarps) * kMkStages * kStageBytes;  // [nx][M][nck][128]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xb + kMkXBytes);
  uint64_t* bars = xbar + 1 + warp * kMkStages;
  float* sxs = reinterpret_cast<float*>(xbar + 1 + kTWarps * kMkStages);  // [32] slice scale per (v, m)
  float* isx = sxs + 32;                                                  // [32] 1 / scale
  int* dsum = reinterpret_cast<int*>(isx + 32);                           // [32] slice sums of x_int
  if (lane == 0) {
    for (int q = 0; q < kMkStages; ++q) mbar_init(bars + q, 1);
    if (warp == 0) mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy, keep;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const int ngroups = (nrt + kTiles - 1) / kTiles;
  const int nitems = ngroups * ksplit;
  const int i0 = blockIdx.x * per, i1 = min(nitems, i0 + per);
  auto slice = [&](int s, int& c0, int& c1) {
    c0 = nch * s / ksplit;
    c1 = nch * (s + 1) / ksplit;
  };
  // weight producer (lane 0 of each warp) walks this CTA's items in consumption order
  int pj = i0, pc = 0, pc1 = 0, prt = -1, pslot = 0;
  auto pitem = [&]() {  // position the producer on item pj (skipping items where this warp idles)
    while (pj < i1) {
      prt = (pj % ngroups) * kTiles + warp * RT;
      slice(pj / ngroups, pc, pc1);
      if (prt < nrt) return;
      ++pj;
    }
  };
  pitem();
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  auto issue = [&]() {
    if (pj >= i1) return;
    const int n = min(U, pc1 - pc);
    const int ntile = (RT == 2 && prt + 1 < nrt) ? 2 : 1;
    mbar_expect_tx(bars + pslot, static_cast<uint32_t>(ntile * n * CHUNK));
    for (int q = 0; q < ntile; ++q) {
      const uint8_t* src = wbase + (static_cast<int64_t>(prt + q) * nch + pc) * CHUNK;
      bulk_g2s(ring + pslot * kStageBytes + q * n * CHUNK, src, static_cast<uint32_t>(n * CHUNK), bars + pslot, policy);
    }
    pslot = pslot + 1 == kMkStages ? 0 : pslot + 1;
    pc += n;
    if (pc >= pc1) {
      ++pj;
      pitem();
    }
  };
  if (lane == 0)
    for (int q = 0; q < kMkStages; ++q) issue();
  pdl_wait();
  pdl_trigger();
  trace_point(11);
  const int nvm = nx * M;
  int cslot = 0;
  uint32_t cpar = 0, xpar = 0;
  int cur = -1;  // k-slice resident in xb
  for (int item = i0; item < i1; ++item) {
    const int s = item / ngroups;
    const int rt = (item % ngroups) * kTiles + warp * RT;
    int c0, c1;
    slice(s, c0, c1);
    const int nck = c1 - c0;
    if (s != cur) {
      // (0) the slice of all nx * M activation rows into the resident buffer
      __syncthreads();  // every warp is done with the previous slice
      if (threadIdx.x == 0) {
        mbar_expect_tx(xbar, static_cast<uint32_t>(nvm * nck * 128));
        for (int v = 0; v < nx; ++v)
          for (int m = 0; m < M; ++m) {
            const uint8_t* src = reinterpret_cast<const uint8_t*>(v == 0 ? a.xf : a.xf2) +
                                 (static_cast<int64_t>(m) * nch + c0) * 128;
            bulk_g2s(xb + ((v * M + m) * nck) * 128, src, static_cast<uint32_t>(nck * 128), xbar, keep);
          }
      }
      mbar_wait(xbar, xpar);
      xpar ^= 1u;
      // (1) slice max per activation vector (v, m): one warp per vector
      for (int vm = warp; vm < nvm; vm += kTWarps) {
        const uint4* row = reinterpret_cast<const uint4*>(xb + static_cast<size_t>(vm) * nck * 128);
        float mx = 0.f;
        bool nan = false;
        for (int i = lane; i < nck * 8; i += 32) {
          const uint4 q = row[i];
          const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(__habs2(*reinterpret_cast<const __half2*>(&wd[e])));
            nan = nan || f.x != f.x || f.y != f.y;
            mx = fmaxf(mx, fmaxf(f.x, f.y));
          }
        }
        mx = warp_max(mx);
        nan = __any_sync(0xffffffffu, nan);
        if (lane == 0) {
          const bool bad = nan || !finite_f32(mx);
          sxs[vm] = bad ? __int_as_float(0x7fc00000) : mx / kDigitQ;
          isx[vm] = (mx > 0.f && !bad) ? kDigitQ / mx : 0.f;
          dsum[vm] = 0;
        }
      }
      __syncthreads();
      // (2) in place: fp16 fragments -> digit pairs; sums of x_int per vector over the slice
      const int ng = nvm * nck * 4;
      for (int i = threadIdx.x; i < ng; i += kTWarps * 32) {
        const int vm = i / (nck * 4);
        const int sm = digits_group(reinterpret_cast<uint4*>(xb) + 2 * i, isx[vm]);
        if (sm) atomicAdd(&dsum[vm], sm);  // integer: order-independent
      }
      __syncthreads();
      cur = s;
    }
    if (rt < nrt) {
      const int v = rt < a.rt_split ? 0 : nx - 1;
      const bool two = RT == 2 && rt + 1 < nrt;
      const uint8_t* xrow[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        xrow[q] = xb + ((v * M + min(4 * q + (g >> 1), M - 1)) * nck) * 128 + t * 32 + (g & 1) * 16;
      int acc[RT][NQ][2][4];
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[r][q][h][i] = 0;
      // the k loop, instantiated for one or two row tiles so the unrolled chunk has no
      // per-tile branch (a divergent-looking branch makes the compiler fence every MMA group)
      auto kloop = [&](auto two_c) {
        constexpr int NR = decltype(two_c)::value ? RT : 1;
        for (int c = 0; c < nck; c += U) {
          const int n = min(U, nck - c);
          mbar_wait(bars + cslot, cpar);
          const uint8_t* st = ring + cslot * kStageBytes + lane * 16;
          auto chunk = [&](int u) {
            uint4 xv[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) xv[q] = *reinterpret_cast<const uint4*>(xrow[q] + (c + u) * 128);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
              const uint4 wv = *reinterpret_cast<const uint4*>(st + (r * n + u) * CHUNK);
              const uint32_t a0 = wv.x & 0x0F0F0F0Fu, a1 = wv.x & 0xF0F0F0F0u, a2 = wv.y & 0x0F0F0F0Fu,
                             a3 = wv.y & 0xF0F0F0F0u;
              const uint32_t a4 = wv.z & 0x0F0F0F0Fu, a5 = wv.z & 0xF0F0F0F0u, a6 = wv.w & 0x0F0F0F0Fu,
                             a7 = wv.w & 0xF0F0F0F0u;
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                imma16832(acc[r][q][0], a0, a1, a2, a3, xv[q].x, xv[q].y);
                imma16832(acc[r][q][1], a4, a5, a6, a7, xv[q].z, xv[q].w);
              }
            }
          };
          if (n == U) {
#pragma unroll
            for (int u = 0; u < U; ++u) chunk(u);
          } else {
            for (int u = 0; u < n; ++u) chunk(u);
          }
          __syncwarp();
          if (cslot + 1 == kMkStages) {
            cslot = 0;
            cpar ^= 1u;
          } else {
            ++cslot;
          }
          if (lane == 0) issue();
        }
      };
      if (two) kloop(std::true_type{});
      else kloop(std::false_type{});
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        if (r == 1 && !two) break;
        float* out = a.partial + static_cast<int64_t>(s) * M * a.Np + static_cast<int64_t>(rt + r) * kTileN;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int m = 4 * q + t;
          if (m < M) {
            const float2 y = i4_rows(acc[r][q][0][0] + acc[r][q][1][0], acc[r][q][0][1] + acc[r][q][1][1],
                                     acc[r][q][0][2] + acc[r][q][1][2], acc[r][q][0][3] + acc[r][q][1][3],
                                     dsum[v * M + m], sxs[v * M + m]);
            out[static_cast<int64_t>(m) * a.Np + g] = y.x;
            out[static_cast<int64_t>(m) * a.Np + g + 8] = y.y;
          }
        }
      }
    }
  }
  trace_point(13);
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
                              const float* __restrict__ col_scale, float* __restrict__ y, int64_t ldy,
                              const float* __restrict__ zt, const float* __restrict__ zvec) {
  const int64_t total = static_cast<int64_t>(M) * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / N);
    const int64_t n = i % N;
    float acc = 0.f;
    for (int s = 0; s < ksplit; ++s) acc += partial[(static_cast<int64_t>(s) * M + m) * Np + n];
    y[m * ldy + n] = zt ? acc * col_scale[n] + zt[m] * zvec[n] : acc * col_scale[n];
  }
}

}  // namespace

// INT4 decode GEMVs on the integer MMA (k_gemv_i4, k_gemv_mk_i4) unless GLM_GEMV_IMMA=0 (fp16 HMMA
// k_gemv_m1, the round-1 kernel, kept for A/B)
bool gemv_imma() {
  static const bool on = [] { const char* e = getenv("GLM_GEMV_IMMA"); return !e || e[0] != '0'; }();
  return on;
}
// warps per CTA of the single-token kernel family (GLM_M1_WARPS overrides): the integer-MMA
// kernel runs 8 at one token (tools/r2_m1_sweep2.sh: 8 x 2 x 8 KB beat 4..16 warps and 4..16 KB
// stages 2..4 deep), 16 at two (tools/r2_b2_ab2.sh), the fp16 kernels 16
int m1_warps(int M) {
  static const int env = [] { const char* e = getenv("GLM_M1_WARPS"); return e ? atoi(e) : 0; }();
  const int v = env ? env : (gemv_imma() && M == 1 ? 8 : kM1DefaultWarps);
  return v < 4 ? 4 : (v > kM1MaxWarps ? kM1MaxWarps : v);
}

// Row tiles per warp of the multi-token kernel (GLM_MK_RT overrides: 1 or 2).
int mk_row_tiles(int bits, int M) {
  static const int env = [] { const char* e = getenv("GLM_MK_RT"); return e ? atoi(e) : 0; }();
  if (env == 1 || env == 2) return env;
  // measured: fp16 kernels +12% (INT4) / +13% (INT8) at 16 tokens, a loss at <= 8; the integer-MMA
  // kernel gains from 8 tokens on (qkv shape, tools/r2_mk_probe.py: M = 8 47.3 -> 43.0 us)
  if (bits == 4 && gemv_imma()) return M >= 6 ? 2 : 1;
  return M > 8 ? 2 : 1;
}

namespace {
// Shared-memory plan of the single-token kernel family (k_gemv_m1, MT = M tokens): ring
// depth, stage bytes and warps next to the resident activation vectors.
struct M1Shape {
  int nst, sb, warps;
  size_t smem;
  bool ok;
};
constexpr size_t kM1SmemLimit = 227 * 1024 - 1024;  // leave room for the static shared memory
constexpr int kM1MaxTokens = 2;


M1Shape m1_shape(int64_t nch, int M, int nx, int plan_warps) {
  static const int m1s = [] { const char* e = getenv("GLM_M1_STAGES"); return e ? atoi(e) : 2; }();
  static const int m1sb_env = [] { const char* e = getenv("GLM_M1_STAGE_KB"); return e ? atoi(e) * 1024 : 0; }();
  const int m1sb = m1sb_env ? m1sb_env : (gemv_imma() && M == 1 ? 8192 : 6144);
  // activation vectors + per-chunk sums (fp32, or int2 digit sums + scales + per-warp maxima)
  const size_t xb = gemv_imma() ? static_cast<size_t>(nx) * M * nch * (128 + 4) + 8 + 64 + kM1MaxWarps * 32
                                : static_cast<size_t>(nx) * M * nch * (128 + 4) + 8;
  M1Shape m;
  m.warps = plan_warps;  // the plan's warps if the rings fit next to x, else fewer
  auto need = [&](int w, int n, int b) { return xb + static_cast<size_t>(w) * n * (b + 8); };
  if (gemv_imma() && M == 1) {
    // integer-MMA kernel: stages of 4..16 KB, 2..4 deep (k_gemv_i4 instantiations); shrink the
    // stage, then the depth, then the warps until the rings fit next to the activations
    static const int sbs[5] = {4096, 6144, 8192, 12288, 16384};
    int si = 0;
    for (int i = 0; i < 5; ++i)
      if (m1sb >= sbs[i]) si = i;
    m.nst = m1s < 2 ? 2 : (m1s > 4 ? 4 : m1s);
    for (;;) {
      m.sb = sbs[si];
      if (need(m.warps, m.nst, m.sb) <= kM1SmemLimit) break;
      if (si > 0) --si;
      else if (m.nst > 2) --m.nst;
      else if (m.warps > 4) --m.warps;
      else break;
    }
    m.smem = need(m.warps, m.nst, m.sb);
    m.ok = m.smem <= kM1SmemLimit;
    return m;
  }
  m.nst = m1s >= 3 ? 3 : 2;
  m.sb = m1sb >= 8192 ? 8192 : (m1sb >= 6144 ? 6144 : 4096);  // larger stages amortise per-stage work
  if (need(m.warps, m.nst, m.sb) > kM1SmemLimit) m.nst = 2;
  while (m.sb > 4096 && need(m.warps, m.nst, m.sb) > kM1SmemLimit) m.sb -= 2048;
  while (m.warps > 8 && need(m.warps, m.nst, m.sb) > kM1SmemLimit) --m.warps;
  m.smem = need(m.warps, m.nst, m.sb);
  m.ok = m.smem <= kM1SmemLimit && nch * 128 * M < (int64_t{1} << 30);
  return m;
}

// The single-token kernel family takes INT4 at up to GLM_M1_TOKENS (default 2) tokens when
// the activation vectors fit next to 12 or more warps' rings (else the multi-token kernel).
// With the integer MMA, two tokens default to the multi-token kernel k_gemv_mk_i4
// (tools/r2_b2_ab2.sh, batch-2 decode: 151.1 tok/s against 150.7 / 146.0 / 144.8 for
// k_gemv_i4<., ., 2> on 16 / 12 / 8 warps); GLM_M1_TOKENS=2 selects the single-token family.
bool use_m1(int64_t nch, int M, int bits, int nx) {
  static const int maxm = [] {
    const char* e = getenv("GLM_M1_TOKENS");
    const int v = e ? atoi(e) : (gemv_imma() ? 1 : kM1MaxTokens);
    return v < 1 ? 1 : (v > kM1MaxTokens ? kM1MaxTokens : v);
  }();
  if (bits != 4 || M > maxm) return false;
  const M1Shape m = m1_shape(nch, M, nx, m1_warps(M));
  return m.ok && (M == 1 || m.warps >= std::min(12, m1_warps(M)));
}
}  // namespace

// INT4 decode GEMVs of GLM_GEMV_TC = T .. 16 tokens run the tcgen05 kernel (gemv_tc.cu); off by
// default (0): bit-identical to k_gemv_mk_i4 but slower on every GLM-130B shape (3.5-3.9 vs
// 4.1-5.9 TB/s); it needs 128-feature tiles (always: Np % 128 == 0).
int tc_min_tokens() {
  static const int v = [] { const char* e = getenv("GLM_GEMV_TC"); return e ? atoi(e) : 0; }();
  return v;
}
bool use_tc(int64_t nrt, int M, int bits) {
  return bits == 4 && gemv_imma() && tc_min_tokens() > 0 && M >= tc_min_tokens() && M >= 2 && M <= 16 && nrt % 8 == 0;
}

GemvPlan plan_gemv(int64_t nrt, int64_t nch, int M, int bits, int nx) {
  GemvPlan p;
  if (use_tc(nrt, M, bits)) {
    // tcgen05 kernel: items of 128 features x one k-slice (<= kTcSliceChunks chunks), slice-major
    // contiguous ranges of `per` items per CTA; the same k-split penalty as the IMMA kernel
    p.tc = true;
    p.warps = 14;
    const int64_t ntiles = nrt / 8;
    const int64_t ks_min = (nch + kTcSliceChunks - 1) / kTcSliceChunks;
    double best = -1.0;
    for (int64_t ks = ks_min; ks <= std::min<int64_t>(nch, ks_min + 24); ++ks) {
      const int64_t items = ntiles * ks;
      const int64_t per = (items + kNumSMs - 1) / kNumSMs;
      const double eff = static_cast<double>(items) / static_cast<double>(per * kNumSMs) - 0.004 * static_cast<double>(ks);
      if (eff > best + 1e-9) {
        best = eff;
        p.ksplit = static_cast<int>(ks);
        p.per = static_cast<int>(per);
      }
    }
    const int64_t items = ntiles * p.ksplit;
    p.grid = static_cast<int>((items + p.per - 1) / p.per);
    return p;
  }
  if (M >= 2 && !use_m1(nch, M, bits, nx) && bits == 4 && gemv_imma() && nx * M <= 32) {
    // integer-MMA multi-token kernel: slice-major items, contiguous ranges of `per` items per
    // CTA, one resident activation slice (kMkXBytes) per CTA
    p.warps = kTWarps;
    p.rt_per_warp = mk_row_tiles(bits, M);
    const int64_t kmax = std::max<int64_t>(1, kMkXBytes / (static_cast<int64_t>(nx) * M * 128));
    const int64_t ks_min = (nch + kmax - 1) / kmax;
    const int64_t ngroups = (nrt + kTWarps * p.rt_per_warp - 1) / (kTWarps * p.rt_per_warp);
    double best = -1.0;
    for (int64_t ks = ks_min; ks <= std::min<int64_t>(nch, ks_min + 24); ++ks) {
      const int64_t items = ngroups * ks;
      const int64_t per = (items + kNumSMs - 1) / kNumSMs;
      const double eff = static_cast<double>(items) / static_cast<double>(per * kNumSMs) - 0.004 * static_cast<double>(ks);
      if (eff > best + 1e-9) {
        best = eff;
        p.ksplit = static_cast<int>(ks);
        p.per = static_cast<int>(per);
      }
    }
    const int64_t items = ngroups * p.ksplit;
    p.grid = static_cast<int>((items + p.per - 1) / p.per);
    return p;
  }
  if (M >= 2 && !use_m1(nch, M, bits, nx)) {
    // multi-token kernel: CTA-items of 16 row tiles x one k-slice; the slice of all M
    // activation rows (nx vectors) must fit one shared-memory buffer
    p.warps = kTWarps;
    p.rt_per_warp = mk_row_tiles(bits, M);
    const int64_t kmax = std::max<int64_t>(1, kMkSliceBytes / (static_cast<int64_t>(nx) * M * 128));
    const int64_t ks_min = (nch + kmax - 1) / kmax;
    const int64_t ngroups = (nrt + kTWarps * p.rt_per_warp - 1) / (kTWarps * p.rt_per_warp);
    double best = -1.0;
    for (int64_t ks = ks_min; ks <= std::min<int64_t>(nch, ks_min + 24); ++ks) {
      const int64_t items = ngroups * ks;
      const int64_t waves = (items + kNumSMs - 1) / kNumSMs;
      const double eff = static_cast<double>(items) / static_cast<double>(waves * kNumSMs) - 0.004 * static_cast<double>(ks);
      if (eff > best + 1e-9) {
        best = eff;
        p.ksplit = static_cast<int>(ks);
      }
    }
    const int64_t items = ngroups * p.ksplit;
    p.grid = static_cast<int>(items < kNumSMs ? items : kNumSMs);
    return p;
  }
  p.warps = use_m1(nch, M, bits, nx) ? m1_warps(M) : kTWarps;
  const int64_t total_warps = static_cast<int64_t>(kNumSMs) * p.warps;
  double best = -1.0;
  const int64_t max_split = nch < 32 ? nch : 32;
  for (int64_t ks = 1; ks <= max_split; ++ks) {
    if (nch / ks < 4 && ks > 1) break;  // keep >= 4 chunks per item
    const int64_t items = nrt * ks;
    const int64_t waves = (items + total_warps - 1) / total_warps;
    double eff = static_cast<double>(items) / static_cast<double>(waves * total_warps);
    eff -= 0.002 * static_cast<double>(ks);  // small ksplit preferred (partial traffic)
    if (eff > best + 1e-9) {
      best = eff;
      p.ksplit = static_cast<int>(ks);
    }
  }
  const int64_t ctas = (nrt * p.ksplit + p.warps - 1) / p.warps;
  p.grid = static_cast<int>(ctas < kNumSMs ? ctas : kNumSMs);
  return p;
}

GemvPlan plan_gemv(const QLayout& L, int M) { return plan_gemv(L.nrt, L.nch, M, L.bits, 1); }

int gemv_kind(const GemvPlan& p, int64_t nch, int M, int bits, int nx) {
  return p.tc ? kGemvI4Tc : gemv_kind(nch, M, bits, nx);
}

int gemv_kind(int64_t nch, int M, int bits, int nx) {  // mirrors gemv_launch's dispatch (plans without tc)
  if (M >= 2 && !use_m1(nch, M, bits, nx))
    return (bits == 4 && gemv_imma() && M * nx <= 32) ? kGemvI4Multi : kGemvF16Multi;
  if (use_m1(nch, M, bits, nx)) return gemv_imma() ? kGemvI4Single : kGemvF16Single;
  return kGemvF16Tma;
}

void gemv_launch(const GemvOp& op, int M, float* partial, const GemvPlan& p, cudaStream_t st) {
  if (M < 1 || M > 16) fail(GLM_DIMENSION, "qlinear", "GEMV path takes 1..16 rows, got " + std::to_string(M));
  GemvArgs a{static_cast<const uint4*>(op.codes), reinterpret_cast<const uint4*>(op.xf),
             reinterpret_cast<const uint4*>(op.xf2 ? op.xf2 : op.xf), op.xf2 ? op.rt_split : op.nrt, partial,
             op.nrt, op.nch, op.nrt * kTileN, M, p.ksplit};
  const int nx_op = (op.xf2 && op.xf2 != op.xf) ? 2 : 1;
  if (p.tc) {
    gemv_tc_launch(op, M, partial, p, st);
    return;
  }
  if (M >= 2 && !use_m1(op.nch, M, op.bits, nx_op)) {
    const int nx = nx_op;
    const int64_t slice_max = (op.nch + p.ksplit - 1) / p.ksplit;
    const bool i4 = op.bits == 4 && gemv_imma() && M * nx <= 32;
    if (slice_max * 128 * M * nx > (i4 ? kMkXBytes : kMkSliceBytes) || p.warps != kTWarps ||
        (p.rt_per_warp == 2 && op.rt_split % 2))
      fail(GLM_CONTRACT, "qlinear", "GEMV plan does not match the multi-token kernel (plan for this M and x count)");
    const size_t smem1 = static_cast<size_t>(kTWarps) * kMkStages * kStageBytes + 2 * kMkSliceBytes +
                         (2 + kTWarps * kMkStages) * 8;
    static bool attr_mk = false;
    if (!attr_mk) {
      for (auto k : {k_gemv_mk<4, 1, 1>, k_gemv_mk<4, 2, 1>, k_gemv_mk<8, 1, 1>, k_gemv_mk<8, 2, 1>, k_gemv_mk<4, 1, 2>,
                     k_gemv_mk<4, 2, 2>, k_gemv_mk<8, 1, 2>, k_gemv_mk<8, 2, 2>})
        CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1));
      attr_mk = true;
    }
    const dim3 gridm(p.grid), blockm(kTWarps * 32);
    const bool two = p.rt_per_warp == 2;
    if (op.bits == 4 && gemv_imma() && M * nx <= 32) {
      const size_t smem2 = static_cast<size_t>(kTWarps) * kMkStages * kStageBytes + kMkXBytes +
                           (1 + kTWarps * kMkStages) * 8 + 32 * 4 * 3;
      if (p.per < 1) fail(GLM_CONTRACT, "qlinear", "GEMV plan does not match the integer-MMA multi-token kernel");
      static bool attr_i4 = false;
      if (!attr_i4) {
        for (auto k : {k_gemv_mk_i4<1, 1>, k_gemv_mk_i4<2, 1>, k_gemv_mk_i4<3, 1>, k_gemv_mk_i4<4, 1>,
                       k_gemv_mk_i4<1, 2>, k_gemv_mk_i4<2, 2>, k_gemv_mk_i4<3, 2>, k_gemv_mk_i4<4, 2>})
          CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
        attr_i4 = true;
      }
      const int nq = (M + 3) / 4;
      void (*k)(GemvArgs, int, int) = nullptr;
      if (two) k = nq == 1 ? k_gemv_mk_i4<1, 2> : nq == 2 ? k_gemv_mk_i4<2, 2> : nq == 3 ? k_gemv_mk_i4<3, 2> : k_gemv_mk_i4<4, 2>;
      else k = nq == 1 ? k_gemv_mk_i4<1, 1> : nq == 2 ? k_gemv_mk_i4<2, 1> : nq == 3 ? k_gemv_mk_i4<3, 1> : k_gemv_mk_i4<4, 1>;
      launch_k(k, gridm, blockm, smem2, st, a, nx, p.per);
      LAUNCH_CHECK("k_gemv_mk_i4");
      return;
    }
    if (op.bits == 4) {
      if (M <= 8) launch_k(two ? k_gemv_mk<4, 1, 2> : k_gemv_mk<4, 1, 1>, gridm, blockm, smem1, st, a, nx);
      else launch_k(two ? k_gemv_mk<4, 2, 2> : k_gemv_mk<4, 2, 1>, gridm, blockm, smem1, st, a, nx);
    } else {
      if (M <= 8) launch_k(two ? k_gemv_mk<8, 1, 2> : k_gemv_mk<8, 1, 1>, gridm, blockm, smem1, st, a, nx);
      else launch_k(two ? k_gemv_mk<8, 2, 2> : k_gemv_mk<8, 2, 1>, gridm, blockm, smem1, st, a, nx);
    }
    LAUNCH_CHECK("k_gemv_mk");
    return;
  }
  const size_t smem = static_cast<size_t>(kTWarps) * kStages * (kStageBytes + 8);
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_tma<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_tma<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_tma<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_tma<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const dim3 grid(p.grid), block(kTWarps * 32);
  if (use_m1(op.nch, M, op.bits, nx_op)) {
    const M1Shape m = m1_shape(op.nch, M, nx_op, p.warps);
    static bool attr1 = false;
    if (!attr1) {
      for (auto k : {k_gemv_m1<4, 2, 4096, 1>, k_gemv_m1<4, 2, 6144, 1>, k_gemv_m1<4, 2, 8192, 1>, k_gemv_m1<4, 3, 4096, 1>,
                     k_gemv_m1<4, 2, 4096, 2>, k_gemv_m1<4, 2, 6144, 2>})
        CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kM1SmemLimit));
      attr1 = true;
    }
    static const int early = [] { const char* e = getenv("GLM_PREFETCH"); return e ? atoi(e) : 2; }();
    // L2 prefetch of the next 32 KB of each warp's stream beyond its ring, issued before the
    // dependency wait (GLM_GEMV_L2PF = KB, 0 off): the LayerNorm / attention / GeGLU kernels in
    // between GEMVs keep HBM busy longer (same-box A/B: 81.6 -> 82.8 tok/s at 1965 MHz, 79.1 ->
    // 79.6 at 1770-1800 MHz; the GEMV-only replay is ~1.5% slower: extra L2 traffic, no overlap)
    static const int l2pf = [] { const char* e = getenv("GLM_GEMV_L2PF"); return (e ? atoi(e) : 32) * 1024; }();
    const dim3 block1(m.warps * 32);
    if (gemv_imma()) {
      using K1 = void (*)(GemvArgs, int, int, int);
      // [stages - 2][stage size 4 / 6 / 8 / 12 / 16 KB]
      static const K1 table[3][5] = {
          {k_gemv_i4<2, 4096, 1>, k_gemv_i4<2, 6144, 1>, k_gemv_i4<2, 8192, 1>, k_gemv_i4<2, 12288, 1>,
           k_gemv_i4<2, 16384, 1>},
          {k_gemv_i4<3, 4096, 1>, k_gemv_i4<3, 6144, 1>, k_gemv_i4<3, 8192, 1>, k_gemv_i4<3, 12288, 1>,
           k_gemv_i4<3, 16384, 1>},
          {k_gemv_i4<4, 4096, 1>, k_gemv_i4<4, 6144, 1>, k_gemv_i4<4, 8192, 1>, k_gemv_i4<4, 12288, 1>,
           k_gemv_i4<4, 16384, 1>}};
      static bool attr2 = false;
      if (!attr2) {
        for (auto& row : table)
          for (K1 k : row) CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kM1SmemLimit));
        for (auto k : {k_gemv_i4<2, 4096, 2>, k_gemv_i4<2, 6144, 2>})
          CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kM1SmemLimit));
        attr2 = true;
      }
      if (M == 2) {
        if (m.sb >= 6144) launch_k(k_gemv_i4<2, 6144, 2>, grid, block1, m.smem, st, a, nx_op, early, l2pf);
        else launch_k(k_gemv_i4<2, 4096, 2>, grid, block1, m.smem, st, a, nx_op, early, l2pf);
      } else {
        const int si = m.sb == 4096 ? 0 : m.sb == 6144 ? 1 : m.sb == 8192 ? 2 : m.sb == 12288 ? 3 : 4;
        launch_k(table[m.nst - 2][si], grid, block1, m.smem, st, a, nx_op, early, l2pf);
      }
      LAUNCH_CHECK("k_gemv_i4");
      return;
    }
    if (M == 2) {
      if (m.sb >= 6144) launch_k(k_gemv_m1<4, 2, 6144, 2>, grid, block1, m.smem, st, a, nx_op, early);
      else launch_k(k_gemv_m1<4, 2, 4096, 2>, grid, block1, m.smem, st, a, nx_op, early);
    } else if (m.nst == 3) {
      launch_k(k_gemv_m1<4, 3, 4096, 1>, grid, block1, m.smem, st, a, nx_op, early);
    } else if (m.sb == 8192) {
      launch_k(k_gemv_m1<4, 2, 8192, 1>, grid, block1, m.smem, st, a, nx_op, early);
    } else if (m.sb == 6144) {
      launch_k(k_gemv_m1<4, 2, 6144, 1>, grid, block1, m.smem, st, a, nx_op, early);
    } else {
      launch_k(k_gemv_m1<4, 2, 4096, 1>, grid, block1, m.smem, st, a, nx_op, early);
    }
    LAUNCH_CHECK("k_gemv_m1");
    return;
  }
  if (op.bits == 4) {
    if (M <= 8) launch_k(k_gemv_tma<4, 1>, grid, block, smem, st, a);
    else launch_k(k_gemv_tma<4, 2>, grid, block, smem, st, a);
  } else {
    if (M <= 8) launch_k(k_gemv_tma<8, 1>, grid, block, smem, st, a);
    else launch_k(k_gemv_tma<8, 2>, grid, block, smem, st, a);
  }
  LAUNCH_CHECK("k_gemv_tma");
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

// zero-point token sums: one warp per row, fp16 rounding of the folded activation exactly as
// the activation buffers hold it
__global__ void k_zp_token_sums(const float* __restrict__ x, int64_t ldx, int64_t K, const float* __restrict__ row_scale,
                                const float* __restrict__ zeta, float* __restrict__ zt) {
  const int m = blockIdx.x;
  float acc = 0.f;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
    acc += __half2float(__float2half_rn(x[m * ldx + k] * row_scale[k])) * zeta[k];
  __shared__ float red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
    zt[m] = t;
  }
}

void zp_token_sums(const float* x, int64_t ldx, int M, const QWeightDev& w, float* zt, cudaStream_t st) {
  k_zp_token_sums<<<M, 256, 0, st>>>(x, ldx, w.L.K, w.row_scale, w.zeta, zt);
  LAUNCH_CHECK("k_zp_token_sums");
}

// zt[m] = sum_k x'[m][k] * zeta[k] over the fp16 activations exactly as the MMA reads them,
// from the decode x_frag layout (tile == 0) or the tcgen05 token tiles (tile == 1)
__global__ void k_zp_sums_act(const __half* __restrict__ xf, int64_t nch, int64_t Kp, int tile,
                              const float* __restrict__ zeta, float* __restrict__ zt) {
  const int m = blockIdx.x;
  float acc = 0.f;
  for (int64_t k = threadIdx.x; k < Kp; k += blockDim.x) {
    const float z = zeta[k];
    if (z != 0.f) acc += __half2float(xf[tile ? xtile_index(Kp, m, k) : xfrag_index(nch, m, k)]) * z;
  }
  __shared__ float red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
    zt[m] = t;
  }
}

void zp_sums_act(const __half* xf, int M, const QWeightDev& w, int tile, float* zt, cudaStream_t st) {
  if (!w.zeta) fail(GLM_CONTRACT, "qlinear", "zero-point sums need zeropoint weights");
  k_zp_sums_act<<<M, 256, 0, st>>>(xf, w.L.nch, w.L.Kp, tile, w.zeta, zt);
  LAUNCH_CHECK("k_zp_sums_act");
}

void gemv_reduce(const float* partial, int ksplit, int M, const QWeightDev& w, float* y, int64_t ldy,
                 cudaStream_t st, const float* zt) {
  const int64_t total = static_cast<int64_t>(M) * w.L.N;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_gemv_reduce<<<grid, 256, 0, st>>>(partial, ksplit, M, w.L.N, w.L.Np, w.col_scale, y, ldy, zt, w.zvec);
  LAUNCH_CHECK("k_gemv_reduce");
}

}  // namespace glm
