// qmm_tc.cu — W4A16 / W8A16 quantized GEMM for prefill on the 5th-generation tensor cores.
//
// Replaces `matmul(x, dequantize(q))` (quant.cpp:188-221 + tensor.cpp:135-155) when many
// token rows share the weights (prefill, M > 16): a 128-feature x 256-token output tile per
// CTA item, fp32 accumulator in TMEM, one persistent CTA per SM (all 512 TMEM columns:
// 8 x 32 A-operand columns + one 256-column accumulator).
//
//   warp 18     TMA producer (weights): one tensor-map copy per stage gathers the 8 row
//               tiles' 512 B (INT8: 1 KB) blocks of one 64-k chunk, 64 B swizzle, into a
//               12-stage ring;
//   warps 0-15  transcode: 4 groups x 4 TMEM lane quarters; group g owns the 64-k stages with
//               q % 4 == g. Each thread owns one output feature (TMEM lane): it reads the
//               64 B of fragment-ordered codes that hold its feature (layout.cuh) from the
//               staged chunk, regroups them into fp16 pairs (k, k+1) with LOP3/PRMT
//               magic-number conversion and writes them to its TMEM lane with tcgen05.st
//               (the MMA's A operand); after an item, every group drains a quarter of the
//               accumulator's token columns (epilogue: tcgen05.ld, scale, store);
//   warp 16     TMA producer (activations): one cp.async.bulk per stage brings the 256-token
//               x 64-k activation tile (32 KB, canonical K-major layout) into a 4-stage ring;
//   warp 17     MMA issuer: tcgen05.mma.cta_group::1.kind::f16, A = transcoded weights in TMEM,
//               B = activations in smem, M = 128 features, N = 256 tokens (a 128 x 128 MMA
//               costs ~125 cycles of issue, so the wider N halves the instruction count per
//               FLOP), K = 16 per instruction; tcgen05.commit releases the smem slot / TMEM
//               buffer.
//
// Evidence: UTCHMMA / LDTM / STTM / UBLKCP in `cuobjdump -sass` of this object.
#include <cuda.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace glm {

namespace {

constexpr int NTOK = kQmmTokens;  // token columns per tile (UMMA N)
constexpr int kGroups = 4;
constexpr int kTcWarps = 4 * kGroups;
constexpr int kThreads = (kTcWarps + 3) * 32;  // + activation producer, MMA issuer, weight producer
constexpr int kPK = 64;                          // k per stage = one layout chunk
constexpr int XB = kPK * NTOK * 2;               // activation bytes per stage (32 KB at N = 256)
constexpr int RX = 4;                            // activation ring
constexpr int NA = 8;                            // 32-column A buffers (two per group)
constexpr int NDB = NTOK <= 128 ? 2 : 1;         // accumulator tiles (2: epilogue overlaps the next item)
constexpr uint32_t D_COL = NA * 32;              // 256: accumulators at [256, 512)
template <int BITS>
constexpr int wstage_bytes() { return BITS == 4 ? 4096 : 8192; }
// weight-code ring (one 64-k chunk of 128 features per stage); the GeGLU-paired INT8 launch
// gives 4 stages to the u/v exchange buffer
template <int BITS, bool PAIR>
constexpr int wring_stages() { return PAIR && BITS == 8 ? 8 : 12; }
// GeGLU epilogue exchange: per group, the two v warps' 16-token x 32-feature fp32 slices, x2 buffers
constexpr int kXchFloats = 16 * 32;
constexpr int kXchBytes = kGroups * 2 * 2 * kXchFloats * 4;
template <int BITS, bool PAIR>
constexpr size_t qmm_smem() {
  return static_cast<size_t>(RX) * XB + static_cast<size_t>(wring_stages<BITS, PAIR>()) * wstage_bytes<BITS>() +
         (PAIR ? kXchBytes : 0) + 1024 + 1024;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
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
// 128 features x one 64-k chunk of codes: the 8 row tiles' blocks (layout.cuh), gathered
// by one tensor-map copy with the 64 B swizzle, so that the transcode threads' 16-byte reads
// (lane g reads 16 B of each 64 B row g) hit 8 distinct bank groups.
template <int BITS>
__device__ __forceinline__ void tma_codes(void* dst, const CUtensorMap* map, int c, int rt16, uint64_t* bar,
                                          uint64_t pol) {
  if constexpr (BITS == 4) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(0), "r"(0), "r"(c), "r"(rt16), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(0), "r"(0), "r"(0), "r"(c), "r"(rt16), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t lop_or_magic(uint32_t w, uint32_t mask) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(w), "r"(mask), "r"(0x64006400u));
  return d;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

struct QmmArgs {
  const uint8_t* w;   // fragment-ordered device layout (layout.cuh)
  // GeGLU-paired launch (PAIR): an item is 64 features of W1 (TMEM lanes 0-63) and the same 64
  // features of V (lanes 64-127); the epilogue writes gelu(x.W1 * s1) * (x.V * s2) straight into
  // W2's activation tiles (tensor.cpp:313-318 fused after both matmuls)
  const float* col_scale2;  // V's group scale
  __half* xo;               // W2 activation tiles (xtile_index), Kp = xo_Kp
  const float* xo_rs;       // W2's kRow fold, or null
  int64_t xo_Kp;
  const __half* xt;   // activations, 128-token tiles (xtile_index)
  float* partial;     // [ksplit][M][Np], or the final y [M][ldo] when col_scale is set
  const float* col_scale;  // non-null (ksplit == 1): write y = acc * col_scale, columns < N
  const float *zt, *zvec;  // optional zero-point rank-1 term y += zt[m] * zvec[n] (direct output)
  int64_t ldo, N;
  int64_t nrt16, nch, Np, Kp;
  int M, ksplit, ntt, nrt128;
  int tokgroup;  // token tiles walked together (their activations stay L2-resident)
  int out_half;  // direct output as fp16 (prefill qkv feeding RoPE / the KV cache)
  int wevict;    // weight copies with an L2 evict_first hint
  long long* trace;
};
__device__ __forceinline__ void stamp(const QmmArgs& a, int ev, uint32_t q) {
  if (a.trace && blockIdx.x == 0 && q < 256) a.trace[q * 8 + ev] = clock64();
}

// item -> (128-feature tile, token tile, k split); token tiles innermost so the CTAs working
// at the same time share a few weight row tiles (L2-resident), stages = 64-k chunks.
// Token tiles are walked in groups of a.tokgroup (qmm_token_group: 4 x 256 tokens = 25 MB of activations at
// K = 12288) so that a group's activations stay L2-resident while every row tile passes
// over them; a packed prefill of many samples would otherwise re-read them from HBM.
__device__ __forceinline__ void decode_item(const QmmArgs& a, int64_t item, int64_t& rt, int64_t& tt, int& s,
                                            int64_t& c0, int64_t& c1) {
  const int64_t kTokGroup = a.tokgroup;
  s = static_cast<int>(item % a.ksplit);
  int64_t rest = item / a.ksplit;
  const int64_t full = a.ntt / kTokGroup;              // complete token groups
  const int64_t per_full = static_cast<int64_t>(a.nrt128) * kTokGroup;
  int64_t tg, tgn;
  if (rest < full * per_full) {
    tg = rest / per_full;
    rest -= tg * per_full;
    tgn = kTokGroup;
  } else {
    rest -= full * per_full;
    tg = full;
    tgn = a.ntt - full * kTokGroup;
  }
  tt = tg * kTokGroup + rest % tgn;
  rt = rest / tgn;
  c0 = a.nch * s / a.ksplit;
  c1 = a.nch * (s + 1) / a.ksplit;
}

// The 64 B of codes holding feature (row tile i, g, half h) for chunk c: lanes 4g..4g+3.
template <int BITS>
struct Codes {
  uint4 u[BITS == 4 ? 4 : 8];
};
// This thread's 64 B (INT8: 2 x 64 B) of a staged chunk: row tile i16 of the stage, row g,
// 16-byte unit t stored at unit t ^ (g >> 1) of the 64 B row (64 B swizzle).
template <int BITS>
__device__ __forceinline__ void smem_codes(const uint8_t* stage, int i16, int g, Codes<BITS>& cd) {
  constexpr int TB = BITS == 4 ? 512 : 1024;
  const uint8_t* row = stage + i16 * TB + g * 64;
  const int sw = (g >> 1) & 3;
#pragma unroll
  for (int t = 0; t < 4; ++t) cd.u[t] = *reinterpret_cast<const uint4*>(row + ((t ^ sw) << 4));
  if constexpr (BITS == 8) {
#pragma unroll
    for (int t = 0; t < 4; ++t) cd.u[4 + t] = *reinterpret_cast<const uint4*>(row + 512 + ((t ^ sw) << 4));
  }
}

// Regroup this feature's codes into 32 fp16 pairs (k = 2c, 2c+1 of the chunk, c = column).
template <int BITS>
__device__ __forceinline__ void transcode(const Codes<BITS>& cd, int h, uint32_t (&r)[32]) {
  if constexpr (BITS == 4) {
    // word j of lane t: nibbles (h, h+4) = k (2t, 2t+1), (h+2, h+6) = k (2t+8, 2t+9) of k-tile j
    const uint32_t k1032 = 0x64086408u;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t ws[4] = {cd.u[t].x, cd.u[t].y, cd.u[t].z, cd.u[t].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t w = ws[j] >> (4 * h);
        r[8 * j + t] = hsub2_u32(lop_or_magic(w, 0x000F000Fu), k1032);
        r[8 * j + 4 + t] = hsub2_u32(lop_or_magic(w >> 8, 0x000F000Fu), k1032);
      }
    }
  } else {
    // k-tile j of lane t: word pair (wd0, wd1); bytes (2h, 2h+1) of wd0 = k (2t, 2t+1),
    // of wd1 = k (2t+8, 2t+9)
    const uint32_t k1152 = 0x64806480u;
    const uint32_t sel = h ? 0x4342u : 0x4140u;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 v = cd.u[(j >> 1) * 4 + t];
        const uint32_t wd0 = (j & 1) ? v.z : v.x, wd1 = (j & 1) ? v.w : v.y;
        r[8 * j + t] = hsub2_u32(__byte_perm(wd0, 0x64646464u, sel), k1152);
        r[8 * j + 4 + t] = hsub2_u32(__byte_perm(wd1, 0x64646464u, sel), k1152);
      }
    }
  }
}

template <int BITS, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    k_qmm_tc(QmmArgs a, const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap vmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr int WB = wstage_bytes<BITS>();
  constexpr int NW = wring_stages<BITS, PAIR>();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xring = smem;
  uint8_t* wring = smem + static_cast<size_t>(RX) * XB;
  float* xch = reinterpret_cast<float*>(wring + static_cast<size_t>(NW) * WB);  // PAIR only
  uint64_t* wfull = reinterpret_cast<uint64_t*>(wring + static_cast<size_t>(NW) * WB + (PAIR ? kXchBytes : 0));
  uint64_t* wempty = wfull + NW;
  uint64_t* xfull = wempty + NW;
  uint64_t* xempty = xfull + RX;
  uint64_t* a_full = xempty + RX;
  uint64_t* a_empty = a_full + NA;
  uint64_t* d_full = a_empty + NA;
  uint64_t* d_empty = d_full + NDB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + NDB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < RX; ++i) {
      mbar_init(xfull + i, 1);
      mbar_init(xempty + i, 1);
    }
    for (int i = 0; i < NW; ++i) {
      mbar_init(wfull + i, 1);
      mbar_init(wempty + i, 4);  // the 4 warps of the transcode group that owns the stage
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(a_full + i, 4);
      mbar_init(a_empty + i, 1);
    }
    for (int i = 0; i < NDB; ++i) {
      mbar_init(d_full + i, 1);
      mbar_init(d_empty + i, kTcWarps);  // every transcode warp drains a quarter of the tile
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int64_t nitems = static_cast<int64_t>(a.nrt128) * a.ntt * a.ksplit;

  if (warp == kTcWarps) {
    // ---------------- TMA producer: activation tiles ----------------
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      uint32_t q = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        int64_t rt, tt, c0, c1;
        int s;
        decode_item(a, item, rt, tt, s, c0, c1);
        for (int64_t c = c0; c < c1; ++c, ++q) {
          const int xs = q % RX;
          mbar_wait(xempty + xs, ((q / RX) & 1) ^ 1);
          stamp(a, 0, q);
          mbar_expect_tx(xfull + xs, XB);
          bulk_g2s(xring + xs * XB, a.xt + tt * a.Kp * NTOK + c * kPK * NTOK, XB, xfull + xs, pol);
          stamp(a, 5, q);
        }
      }
    }
  } else if (warp == kTcWarps + 2) {
    // ---------------- TMA producer: weight codes, one 64-k chunk of 128 features per stage ------
    if (lane == 0) {
      // weights are re-read by the G token tiles of a group close together in time; evict_first
      // (GLM_QMM_WEVICT=1) lets the group's activations keep their L2 lines instead
      uint64_t pol;
      if (a.wevict) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      uint32_t q = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        int64_t rt, tt, c0, c1;
        int s;
        decode_item(a, item, rt, tt, s, c0, c1);
        for (int64_t c = c0; c < c1; ++c, ++q) {
          const int ws = q % NW;
          mbar_wait(wempty + ws, ((q / NW) & 1) ^ 1);
          mbar_expect_tx(wfull + ws, WB);
          if constexpr (PAIR) {  // 4 row tiles of W1, then the same 4 of V
            tma_codes<BITS>(wring + static_cast<size_t>(ws) * WB, &wmap, static_cast<int>(c), static_cast<int>(rt * 4),
                            wfull + ws, pol);
            tma_codes<BITS>(wring + static_cast<size_t>(ws) * WB + WB / 2, &vmap, static_cast<int>(c),
                            static_cast<int>(rt * 4), wfull + ws, pol);
          } else {
            tma_codes<BITS>(wring + static_cast<size_t>(ws) * WB, &wmap, static_cast<int>(c), static_cast<int>(rt * 8),
                            wfull + ws, pol);
          }
        }
      }
    }
  } else if (warp == kTcWarps + 1) {
    // ---------------- MMA issuer (whole warp converged; elect.sync issues) ----------------
    const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(NTOK >> 3) << 17) | (8u << 24);
    const uint64_t desc_hi = (static_cast<uint64_t>((NTOK * 16) >> 4) << 16) |
                             (static_cast<uint64_t>(128 >> 4) << 32) | (1ull << 46);
    const uint32_t x0 = smem_u32(xring);
    uint32_t q = 0, it = 0;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
      int64_t rt, tt, c0, c1;
      int s;
      decode_item(a, item, rt, tt, s, c0, c1);
      const int db = it % NDB;
      mbar_wait(d_empty + db, ((it / NDB) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tbase + D_COL + db * NTOK;
      for (int64_t c = c0; c < c1; ++c, ++q) {
        const int xs = q % RX, ab = q % NA;
        mbar_wait(xfull + xs, (q / RX) & 1);
        mbar_wait(a_full + ab, (q / NA) & 1);
        tc_fence_after();
        if (lane == 0) stamp(a, 3, q);
        const uint64_t dbase = desc_hi | static_cast<uint64_t>(((x0 + xs * XB) >> 4) & 0x3FFF);
#pragma unroll
        for (int ks = 0; ks < kPK / 16; ++ks)
          mma_f16_ts_elect(dcol, tbase + ab * 32 + ks * 8, dbase + ((ks * NTOK * 32) >> 4), idesc,
                           (c > c0 || ks > 0) ? 1u : 0u);
        tc_commit_elect(xempty + xs);
        tc_commit_elect(a_empty + ab);
        __syncwarp();
        if (lane == 0) stamp(a, 4, q);
      }
      tc_commit_elect(d_full + db);
      __syncwarp();
    }
  } else {
    // ---------------- transcode (+ epilogue on group 0) ----------------
    const int quarter = warp & 3, group = warp >> 2;
    const int row = quarter * 32 + lane;              // TMEM lane = feature in the 128 tile
    const int i16 = row >> 4, g = row & 7, h = (row >> 3) & 1;
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    uint32_t q = 0, it = 0;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
      int64_t rt, tt, c0, c1;
      int s;
      decode_item(a, item, rt, tt, s, c0, c1);
      // owned stages of this item: chunks with (global chunk index) % kGroups == group
      int64_t c = c0 + ((group - static_cast<int>(q % kGroups)) + kGroups) % kGroups;
      uint32_t qq = q + static_cast<uint32_t>(c - c0);
      for (; c < c1; c += kGroups, qq += kGroups) {
        const int ws = qq % NW, ab = qq % NA;
        mbar_wait(wfull + ws, (qq / NW) & 1);
        if (warp == 0 && lane == 0) stamp(a, 1, qq);
        Codes<BITS> cur;
        smem_codes<BITS>(wring + static_cast<size_t>(ws) * WB, i16, g, cur);
        uint32_t r[32];
        transcode<BITS>(cur, h, r);
        __syncwarp();
        if (lane == 0) mbar_arrive(wempty + ws);
        mbar_wait(a_empty + ab, ((qq / NA) & 1) ^ 1);
        tc_fence_after();
        tmem_st16(lane_base + ab * 32, r);
        tmem_st16(lane_base + ab * 32 + 16, r + 16);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (warp == 0 && lane == 0) stamp(a, 2, qq);
        if (lane == 0) mbar_arrive(a_full + ab);
      }
      q += static_cast<uint32_t>(c1 - c0);
      if constexpr (PAIR) {  // GeGLU epilogue: v warps (quarters 2, 3) hand x.V to the u warps
        const int db = it % NDB;
        mbar_wait(d_full + db, (it / NDB) & 1);
        tc_fence_after();
        const int64_t f = rt * 64 + (quarter & 1) * 32 + lane;  // feature of W1 / V / W2's k
        const bool keep = f < a.N;
        const float cs = keep ? (quarter < 2 ? a.col_scale[f] : a.col_scale2[f]) : 0.f;  // v warps: V's scale
        const float rs = keep && a.xo_rs ? a.xo_rs[f] : 1.f;
        float* xw = xch + (group * 2 + (quarter & 1)) * 2 * kXchFloats + lane;
        const int64_t tile_base = tt * a.xo_Kp * NTOK + ((f % 16) / 8 + (f / 16) * 2) * (8 * NTOK) + f % 8;
#pragma unroll 1
        for (int c16 = group * (NTOK / kGroups), b = 0; c16 < (group + 1) * (NTOK / kGroups); c16 += 16, b ^= 1) {
          uint32_t v[16];
          tmem_ld16(lane_base + D_COL + db * NTOK + c16, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // the u warp computes tokens 0-7 of the chunk, its v partner tokens 8-15: each hands
          // the other half of its operand over (v: tokens 0-7 at +0, u: tokens 8-15 at +256)
          const bool is_u = quarter < 2;  // warp-uniform: both branches index v[] statically
          float* xb = xw + b * kXchFloats;
          float own[8];
          if (is_u) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              xb[256 + m * 32] = __uint_as_float(v[8 + m]) * cs;
              own[m] = __uint_as_float(v[m]) * cs;
            }
          } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              xb[m * 32] = __uint_as_float(v[m]) * cs;
              own[m] = __uint_as_float(v[8 + m]) * cs;
            }
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + group) : "memory");
          const int m0 = c16 + (is_u ? 0 : 8);
          const float* src = xb + (is_u ? 0 : 256);
          if (keep) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              if (tt * NTOK + m0 + m < a.M) {
                const float other = src[m * 32];
                const float u = is_u ? own[m] : other, vv = is_u ? other : own[m];
                const float o = 0.5f * u * (1.f + erff(u * 0.70710678118654752440f)) * vv * rs;
                a.xo[tile_base + ((m0 + m) / 8) * 64 + ((m0 + m) % 8) * 8] = __float2half_rn(o);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty + db);
      } else {  // epilogue: group g drains token columns [g, g + 1) * NTOK / kGroups of the tile
        const int db = it % NDB;
        mbar_wait(d_full + db, (it / NDB) & 1);
        tc_fence_after();
        const int64_t col = rt * 128 + row;
        const bool direct = a.col_scale != nullptr;  // final output, group scale applied here
        const float cs = direct && col < a.N ? a.col_scale[col] : 1.f;
        const float zv = direct && a.zt && col < a.N ? a.zvec[col] : 0.f;
        const int64_t ld = direct ? a.ldo : a.Np;
        float* out = a.partial + (direct ? 0 : static_cast<int64_t>(s) * a.M * a.Np) + col;
        const bool keep = !direct || col < a.N;
#pragma unroll 1
        for (int c16 = group * (NTOK / kGroups); c16 < (group + 1) * (NTOK / kGroups); c16 += 16) {
          uint32_t v[16];
          tmem_ld16(lane_base + D_COL + db * NTOK + c16, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            const int64_t tok = tt * NTOK + c16 + m;
            if (tok < a.M && keep) {
              const float y = zv != 0.f ? __uint_as_float(v[m]) * cs + a.zt[tok] * zv : __uint_as_float(v[m]) * cs;
              if (a.out_half) reinterpret_cast<__half*>(a.partial)[tok * ld + col] = __float2half_rn(y);
              else out[tok * ld] = y;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty + db);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

__global__ void k_xtile_from_f32(const float* __restrict__ x, int64_t ldx, int M, int64_t K, int64_t Kp, int NT,
                                 const float* __restrict__ row_scale, __half* __restrict__ xt) {
  const int64_t pairs = static_cast<int64_t>(NT) * (Kp / 2);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / (Kp / 2));
    const int64_t k = (i % (Kp / 2)) * 2;
    const float v0 = (m < M && k < K) ? x[m * ldx + k] * row_scale[k] : 0.f;
    const float v1 = (m < M && k + 1 < K) ? x[m * ldx + k + 1] * row_scale[k + 1] : 0.f;
    *reinterpret_cast<__half2*>(xt + xtile_index(Kp, m, k)) = __floats2half2_rn(v0, v1);
  }
}

}  // namespace

long long*& qmm_trace_ptr() {
  static long long* p = nullptr;
  return p;
}

// Tensor map of a linear's device-layout codes: [64 B row][8 rows g][(INT8: 2 halves)]
// [nch chunks][nrt16 row tiles], box = one chunk of 8 row tiles, 64 B swizzle. The driver
// entry point comes through the runtime (no libcuda link); maps are cached per buffer.
namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// box_rt: row tiles per copy (8; 4 for the GeGLU-paired launch, which stages W1 and V halves).
EncodeTiledFn tensor_map_encoder() {
  static EncodeTiledFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) fail(GLM_CUDA, "qlinear", "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  return encode;
}

}  // namespace

CUtensorMap codes_tensor_map_raw(const void* codes, int64_t nrt, int64_t nch, int bits, int box_rt, bool wide) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int64_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(codes, ((nrt * 1000003 + nch * 17 + bits) * 16 + box_rt) * 2 + (wide ? 1 : 0));
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  EncodeTiledFn encode = tensor_map_encoder();
  CUtensorMap m;
  const bool i8 = bits == 8;
  const cuuint32_t rank = i8 ? 5 : 4;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
  const cuuint64_t cb = i8 ? 1024 : 512;  // QLayout::chunk_bytes
  if (wide) {
    // INT4, rows of 128 B (two g rows), 128 B swizzle: half the copy rows of the 64 B form
    if (i8) fail(GLM_CONTRACT, "qlinear", "128 B code rows are INT4 only");
    const cuuint64_t d[4] = {128, 4, static_cast<cuuint64_t>(nch), static_cast<cuuint64_t>(nrt)};
    const cuuint64_t sd[3] = {128, 512, static_cast<cuuint64_t>(nch) * cb};
    const cuuint32_t bx[4] = {128, 4, 1, static_cast<cuuint32_t>(box_rt)};
    for (int i = 0; i < 4; ++i) dims[i] = d[i], box[i] = bx[i];
    for (int i = 0; i < 3; ++i) strides[i] = sd[i];
  } else if (i8) {
    const cuuint64_t d[5] = {64, 8, 2, static_cast<cuuint64_t>(nch), static_cast<cuuint64_t>(nrt)};
    const cuuint64_t sd[4] = {64, 512, 1024, static_cast<cuuint64_t>(nch) * cb};
    const cuuint32_t bx[5] = {64, 8, 2, 1, static_cast<cuuint32_t>(box_rt)};
    for (int i = 0; i < 5; ++i) dims[i] = d[i], box[i] = bx[i];
    for (int i = 0; i < 4; ++i) strides[i] = sd[i];
  } else {
    const cuuint64_t d[4] = {64, 8, static_cast<cuuint64_t>(nch), static_cast<cuuint64_t>(nrt)};
    const cuuint64_t sd[3] = {64, 512, static_cast<cuuint64_t>(nch) * cb};
    const cuuint32_t bx[4] = {64, 8, 1, static_cast<cuuint32_t>(box_rt)};
    for (int i = 0; i < 4; ++i) dims[i] = d[i], box[i] = bx[i];
    for (int i = 0; i < 3; ++i) strides[i] = sd[i];
  }
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(codes), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GLM_CUDA, "qlinear", "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  cache[key] = m;
  return m;
}

CUtensorMap rows_tensor_map(const void* base, int64_t inner_bytes, int64_t rows, int64_t row_stride, int64_t groups,
                            int64_t group_stride, int box_rows, int box_groups) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner_bytes), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(groups)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride), static_cast<cuuint64_t>(group_stride)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(inner_bytes), static_cast<cuuint32_t>(box_rows),
                             static_cast<cuuint32_t>(box_groups)};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box,
                                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(GLM_CUDA, "qlinear", "cuTensorMapEncodeTiled (activation rows) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

namespace {
CUtensorMap codes_tensor_map(const QWeightDev& w, int box_rt = 8) {
  return codes_tensor_map_raw(w.codes, w.L.nrt, w.L.nch, w.L.bits, box_rt, false);
}
}  // namespace

// Token tiles per group (GLM_QMM_TOKGROUP overrides). The SMs hold ~148 items at once, so a
// group of G token tiles spans 148 / G row tiles per wave: activations are read once while the
// group's G x 256 x K fp16 tiles stay in L2, weights once per group. Config 3 (8192 tokens,
// ncu DRAM reads per block): G = 16 (100 MB of activations at K = 12288) thrashes L2 —
// 6.8 + 2.3 + 11.9 + 6.3 GB, 23.8 ms; G = 4: 2.3 + 1.0 + 3.5 + 3.5 GB, 22.5 ms (lower DRAM
// traffic also buys SM clock under the power cap: 1.44 -> 1.49 GHz in the qkv GEMM).
int qmm_token_group(int64_t Kp) {
  static const int g = [] { const char* e = getenv("GLM_QMM_TOKGROUP"); return e ? atoi(e) : 4; }();
  (void)Kp;
  return g < 1 ? 1 : g;
}

int qmm_weight_evict_first() {
  static const int v = [] { const char* e = getenv("GLM_QMM_WEVICT"); return e ? atoi(e) : 0; }();
  return v;
}

template <int BITS, bool PAIR>
void launch_qmm(const QmmArgs& a, int grid, const CUtensorMap& wmap, const CUtensorMap& vmap, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_qmm_tc<BITS, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(qmm_smem<BITS, PAIR>())));
    attr = true;
  }
  k_qmm_tc<BITS, PAIR><<<grid, kThreads, qmm_smem<BITS, PAIR>(), st>>>(a, wmap, vmap);
  LAUNCH_CHECK("k_qmm_tc");
}

GemvPlan plan_qmm(const QLayout& L, int M) {
  GemvPlan p;
  const int64_t ntt = (M + NTOK - 1) / NTOK, nrt128 = L.Np / 128;
  const int64_t workers = kNumSMs;
  double best = -1.0;
  const int64_t max_split = L.nch < 16 ? L.nch : 16;
  for (int64_t ks = 1; ks <= max_split; ++ks) {
    if (L.nch / ks < 8 && ks > 1) break;
    const int64_t items = ntt * nrt128 * ks;
    const int64_t waves = (items + workers - 1) / workers;
    // an unsplit K writes the scaled output directly (no partials, no reduce pass)
    double eff = static_cast<double>(items) / static_cast<double>(waves * workers) - 0.01 * static_cast<double>(ks) -
                 (ks > 1 ? 0.04 : 0.0);
    if (eff > best + 1e-9) {
      best = eff;
      p.ksplit = static_cast<int>(ks);
    }
  }
  const int64_t items = ntt * nrt128 * p.ksplit;
  p.grid = static_cast<int>(items < workers ? items : workers);
  return p;
}

void qmm_launch(const QWeightDev& w, const __half* xt, int M, float* partial, const GemvPlan& p, cudaStream_t st,
                float* y, int64_t ldy, const float* zt, bool y_half) {
  if (y_half && !y) fail(GLM_CONTRACT, "qlinear", "fp16 output needs the direct (unsplit) mode");
  if (M < 1) fail(GLM_DIMENSION, "qlinear", "M must be >= 1");
  if (w.L.Np % 128 || w.L.Kp % 64) fail(GLM_DIMENSION, "qlinear", "layout not padded for the tcgen05 path");
  if (y && p.ksplit != 1) fail(GLM_CONTRACT, "qlinear", "direct output needs an unsplit K");
  QmmArgs a{};
  a.w = static_cast<const uint8_t*>(w.codes);
  a.xt = xt;
  a.partial = y ? y : partial;
  a.col_scale = y ? w.col_scale : nullptr;
  a.zt = y ? zt : nullptr;
  a.zvec = w.zvec;
  a.ldo = ldy;
  a.N = w.L.N;
  a.nrt16 = w.L.nrt;
  a.nch = w.L.nch;
  a.Np = w.L.Np;
  a.Kp = w.L.Kp;
  a.M = M;
  a.ksplit = p.ksplit;
  a.ntt = (M + NTOK - 1) / NTOK;
  a.nrt128 = static_cast<int>(w.L.Np / 128);
  a.tokgroup = qmm_token_group(w.L.Kp);
  a.wevict = qmm_weight_evict_first();
  a.out_half = y_half ? 1 : 0;
  a.trace = nullptr;
  static long long* trace_buf = nullptr;
  if (getenv("GLM_QMM_TRACE")) {
    if (!trace_buf) CUDA_CHECK(cudaMalloc(&trace_buf, 256 * 8 * sizeof(long long)));
    CUDA_CHECK(cudaMemsetAsync(trace_buf, 0, 256 * 8 * sizeof(long long), st));
    a.trace = trace_buf;
    qmm_trace_ptr() = trace_buf;
  }
  const CUtensorMap wmap = codes_tensor_map(w);
  if (w.L.bits == 4) launch_qmm<4, false>(a, p.grid, wmap, wmap, st);
  else launch_qmm<8, false>(a, p.grid, wmap, wmap, st);
}

bool qmm_geglu_supported(const QWeightDev& w1, const QWeightDev& v, int M) {
  static const bool off = [] {
    const char* e = getenv("GLM_QMM_GEGLU");
    return e && e[0] == '0';
  }();
  return !off && M > 16 && w1.L.bits == v.L.bits && w1.L.K == v.L.K && w1.L.N == v.L.N && w1.L.Np == v.L.Np &&
         w1.L.nch == v.L.nch && w1.zvec == nullptr && v.zvec == nullptr && w1.L.Np % 128 == 0 && w1.L.Kp % 64 == 0;
}

void qmm_geglu_launch(const QWeightDev& w1, const QWeightDev& v, const __half* xt, int M, __half* xo, int64_t xo_Kp,
                      const float* xo_rs, cudaStream_t st) {
  if (!qmm_geglu_supported(w1, v, M)) fail(GLM_CONTRACT, "qlinear", "W1 / V pair not eligible for the fused GeGLU GEMM");
  QmmArgs a{};
  a.w = static_cast<const uint8_t*>(w1.codes);
  a.xt = xt;
  a.col_scale = w1.col_scale;
  a.col_scale2 = v.col_scale;
  a.xo = xo;
  a.xo_Kp = xo_Kp;
  a.xo_rs = xo_rs;
  a.N = w1.L.N;
  a.nrt16 = w1.L.nrt;
  a.nch = w1.L.nch;
  a.Np = w1.L.Np;
  a.Kp = w1.L.Kp;
  a.M = M;
  a.ksplit = 1;
  a.ntt = (M + NTOK - 1) / NTOK;
  a.nrt128 = static_cast<int>(w1.L.Np / 64);  // 64-feature blocks of the pair
  a.tokgroup = qmm_token_group(w1.L.Kp);
  a.wevict = qmm_weight_evict_first();
  a.trace = nullptr;
  const int64_t items = static_cast<int64_t>(a.nrt128) * a.ntt;
  const int grid = static_cast<int>(items < kNumSMs ? items : kNumSMs);
  const CUtensorMap wmap = codes_tensor_map(w1, 4), vmap = codes_tensor_map(v, 4);
  if (w1.L.bits == 4) launch_qmm<4, true>(a, grid, wmap, vmap, st);
  else launch_qmm<8, true>(a, grid, wmap, vmap, st);
}

void xtile_from_f32(const float* x, int64_t ldx, int M, const QWeightDev& w, __half* xt, cudaStream_t st) {
  const int NT = xtile_tokens(M);
  const int64_t pairs = static_cast<int64_t>(NT) * (w.L.Kp / 2);
  const int grid = static_cast<int>(std::min<int64_t>((pairs + 255) / 256, 148 * 16));
  k_xtile_from_f32<<<grid, 256, 0, st>>>(x, ldx, M, w.L.K, w.L.Kp, NT, w.row_scale, xt);
  LAUNCH_CHECK("k_xtile_from_f32");
}

}  // namespace glm
