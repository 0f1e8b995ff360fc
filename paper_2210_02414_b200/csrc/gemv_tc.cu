// gemv_tc.cu — INT4 multi-token decode GEMV on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8, A = weight codes in TMEM, B = activation digits in shared memory).
//
// Replaces `matmul(x, dequantize(q))` (quant.cpp:188-221 + tensor.cpp:135-155) for 2..16
// decode tokens with exactly the arithmetic of k_gemv_mk_i4 (gemv.cu): per (token, k-slice)
// 16-bit fixed-point activations x_int = 256 hi + lo (digits.cuh), exact int32 products and
// sums of (code + 8) x digit, the code offset removed in int64, one fp32 scale — so its
// partials are bit-identical to the integer-MMA kernel for the same k-split. At 16 tokens the
// mma.sync form needs ~416 T IMMA-MAC/s to keep up with HBM (two digit columns per token) and
// the IMMA pipe tops out near that; one tcgen05 i8 MMA of 128 features x 32 digit columns x
// 32 k costs its issuing thread ~55 cycles (tools/i8_probe.cu), i.e. ~10 TB/s of INT4 codes.
//
// Item = 128 features (8 row tiles) x one k-slice (<= 64 chunks of 64 k); contiguous ranges
// of `per` slice-major items per persistent CTA (one CTA per SM).
//   warps 0-7   transcode, 2 groups of 4 (TMEM lane quarters); group g owns the ring stages
//               with q % 2 == g: each thread reads its feature's 64 B per chunk (layout.cuh:
//               lanes 4g..4g+3 of the row tile; 128 B rows of two g rows, 128 B swizzle, by the
//               tensor map) and masks the nibbles into u8 A words (rows g: code + 8, rows g + 8:
//               16 (code + 8)), written with tcgen05.st. At every new k-slice they also build the
//               B operand: one TMA brings the slice's fp16 activations as [chunk][16 tokens][128 B]
//               (tokens >= M zero-filled), a max pass sets the per-token scale, and each chunk's
//               2 KB is turned into digits IN PLACE by one warp — [token][4 groups][32 B] becomes
//               the K-major core-matrix layout [group][16 hi rows | 16 lo rows][16 B], so the
//               staged slice is the canonical B operand without a copy;
//   warp 8      producer: lanes 0..3 issue one tensor-map copy each (4 chunks = 16 KB of 128
//               features per stage), 4-stage ring;
//   warp 9      MMA issuer: per chunk two M = 128, N = 32, K = 32 MMAs into a double-buffered
//               s32 accumulator;
//   warps 10-13 epilogue: tcgen05.ld, 256 hi + lo - offset * sum(x_int) in int64, x s_x, partials.
//
// Status: correct (bit-identical to k_gemv_mk_i4; tests/test_gpu_qlinear.py) but slower on every
// GLM-130B shape, so opt-in (GLM_GEMV_TC=T: T..16 tokens). Per-CTA timeline at qkv, 16 tokens
// (tools/tc_trace.py): the k-slice's digits are ready ~9.6 us after entry, and the code stream
// then runs at ~33-36 GB/s per SM even with the MMAs, TMEM stores and code reads all skipped
// (GLM_TC_DBG=15) and with 1-D bulk copies instead of the tensor map — below the ~44 GB/s the
// IMMA kernel's 16 warps x 2 x 4 KB rings sustain; deeper rings (8 x 16 KB) and L2 prefetch
// (GLM_TC_PF) did not help (profiles/r2_tc_negative.txt).
#include <cuda.h>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "digits.cuh"
#include "kernels.h"

namespace glm {

GLM_TRACE_TU(gemv_tc)

namespace {

#ifndef GLM_TC_U
#define GLM_TC_U 4
#endif
constexpr int kU = GLM_TC_U;                 // 64-k chunks per ring stage
constexpr int kChunkBytes = 4096;            // 128 features x 64 k of INT4 codes
constexpr int kStageB = kU * kChunkBytes;    // 16 KB
#ifndef GLM_TC_NS
#define GLM_TC_NS 4
#endif
constexpr int kNS = GLM_TC_NS;               // ring stages
constexpr int kSliceChunks = kTcSliceChunks; // max chunks per k-slice
constexpr int kSliceBytes = kSliceChunks * 2048;  // fp16 staging == digit B operand (2 KB per chunk)
constexpr int kNA = 6;                       // A buffers in TMEM (kU x 16 columns each)
constexpr uint32_t kDCol = kNA * kU * 16;    // accumulators (2 x 32 columns) after the A buffers
constexpr int kThreads = 14 * 32;
constexpr int kBarBytes = ((2 * kNS + 2 * kNA + 6) * 8 + 15) / 16 * 16;  // mbarriers
constexpr size_t kSmem = 1024 + kSliceBytes + static_cast<size_t>(kNS) * kStageB + kBarBytes + 4 * 16 * 4 + 16;

struct TcArgs {
  float* partial;  // [ksplit][M][Np]
  int64_t Np;
  int nch, ntiles, ksplit, M, per, split_tiles;  // tiles >= split_tiles read the second x
  int box;  // chunks per activation copy (the longest slice)
  int pf;   // chunks of weight codes prefetched into L2 ahead of the ring
  int dbg;  // diagnostics (GLM_TC_DBG): 1 skip the MMAs, 2 skip the TMEM stores, 4 skip the code
            // reads, 8 weights by 1-D bulk copies per row tile (all: wrong results, timing only)
  const uint8_t* codes;
};

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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void bar_transcode() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ void tma_chunk(void* dst, const CUtensorMap* map, int c, int rt16, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(0), "r"(0), "r"(c), "r"(rt16), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_chunk_prefetch(const CUtensorMap* map, int c, int rt16) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(map), "r"(0), "r"(0), "r"(c),
               "r"(rt16)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_rows(void* dst, const CUtensorMap* map, int g0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(0), "r"(0), "r"(g0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

struct Item {
  int s, tile, c0, c1, key;
};
__device__ __forceinline__ Item item_of(const TcArgs& a, int item) {
  Item it;
  it.s = item / a.ntiles;
  it.tile = item % a.ntiles;
  it.c0 = static_cast<int>(static_cast<int64_t>(a.nch) * it.s / a.ksplit);
  it.c1 = static_cast<int>(static_cast<int64_t>(a.nch) * (it.s + 1) / a.ksplit);
  it.key = 2 * it.s + (it.tile >= a.split_tiles ? 1 : 0);
  return it;
}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemv_tc_i4(TcArgs a, const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                 const __grid_constant__ CUtensorMap xmap2) {
  trace_point(10);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem;                  // the k-slice: fp16 staging, then the digit B operand
  uint8_t* ring = smem + kSliceBytes;  // weight stages
  uint64_t* wfull = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(kNS) * kStageB);
  uint64_t* wempty = wfull + kNS;
  uint64_t* afull = wempty + kNS;
  uint64_t* aempty = afull + kNA;
  uint64_t* dfull = aempty + kNA;
  uint64_t* dempty = dfull + 2;
  uint64_t* xbar = dempty + 2;
  uint64_t* xready = xbar + 1;
  int* amax = reinterpret_cast<int*>(smem + kSliceBytes + static_cast<size_t>(kNS) * kStageB + kBarBytes);
  float* sxs = reinterpret_cast<float*>(amax + 16);
  float* isx = sxs + 16;
  int* dsum = reinterpret_cast<int*>(isx + 16);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dsum + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 8 * 32) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(wfull + i, 1);
      mbar_init(wempty + i, 4);  // the 4 warps of the owning transcode group
    }
    for (int i = 0; i < kNA; ++i) {
      mbar_init(afull + i, 4);
      mbar_init(aempty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(dfull + i, 1);
      mbar_init(dempty + i, 4);  // the 4 epilogue warps
    }
    mbar_init(xbar, 1);
    mbar_init(xready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nitems = a.ntiles * a.ksplit;
  const int i0 = blockIdx.x * a.per, i1 = min(nitems, i0 + a.per);

  if (warp == 8) {
    // ---------------- TMA producer: weight codes (constant: runs ahead of the dependency wait) ----
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    // optional L2 prefetch a.pf chunks ahead of the ring (GLM_TC_PF, off by default: slower)
    int pf_item = i0, pf_c = 0, pf_c1 = 0, pf_tile = 0;
    if (i0 < i1) {
      const Item t = item_of(a, i0);
      pf_c = t.c0, pf_c1 = t.c1, pf_tile = t.tile;
    }
    auto prefetch_one = [&]() {
      if (pf_item >= i1) return;
      tma_chunk_prefetch(&wmap, pf_c, pf_tile * 8);
      if (++pf_c >= pf_c1 && ++pf_item < i1) {
        const Item t = item_of(a, pf_item);
        pf_c = t.c0, pf_c1 = t.c1, pf_tile = t.tile;
      }
    };
    if (a.pf >= 0 && lane == 0)
      for (int i = 0; i < a.pf + kNS * kU; ++i) prefetch_one();
    uint32_t q = 0;
    for (int item = i0; item < i1; ++item) {
      const Item it = item_of(a, item);
      for (int c = it.c0; c < it.c1; c += kU, ++q) {
        const int ws = q % kNS, n = min(kU, it.c1 - c);
        if (lane == 0) {
          mbar_wait(wempty + ws, ((q / kNS) & 1) ^ 1);
          mbar_expect_tx(wfull + ws, static_cast<uint32_t>(n * kChunkBytes));
        }
        __syncwarp();
        if (a.dbg & 8) {  // lanes 0-7: one row tile each
          if (lane < 8)
            bulk_g2s(ring + static_cast<size_t>(ws) * kStageB + lane * n * 512,
                     a.codes + (static_cast<int64_t>(it.tile * 8 + lane) * a.nch + c) * 512, n * 512, wfull + ws, pol);
          continue;
        }
        if (lane < n) {  // lanes 0..n-1: one chunk each
          tma_chunk(ring + static_cast<size_t>(ws) * kStageB + lane * kChunkBytes, &wmap, c + lane, it.tile * 8, wfull + ws, pol);
        }
        if (a.pf >= 0 && lane == 0)
          for (int u = 0; u < n; ++u) prefetch_one();
      }
    }
    pdl_trigger();
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    pdl_trigger();
    // D s32 (bits 4-5 = 2), A u8 (7-9 = 0), B s8 (10-12 = 1), N = 32, M = 128
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    // K-major, no swizzle: LBO = 512 B between the 16-k core-matrix columns, SBO = 128 B between 8-row groups
    const uint64_t desc_hi = (static_cast<uint64_t>(512 >> 4) << 16) | (static_cast<uint64_t>(128 >> 4) << 32) | (1ull << 46);
    const uint32_t x0 = smem_u32(xs);
    uint32_t q = 0, sw = 0;
    int prev = -1;
    for (int item = i0, n_it = 0; item < i1; ++item, ++n_it) {
      const Item it = item_of(a, item);
      if (it.key != prev) {
        mbar_wait(xready, sw & 1);
        ++sw;
        prev = it.key;
      }
      const int db = n_it & 1;
      mbar_wait(dempty + db, ((n_it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tbase + kDCol + db * 32;
      for (int c = it.c0; c < it.c1; c += kU, ++q) {
        const int ab = q % kNA, n = min(kU, it.c1 - c);
        mbar_wait(afull + ab, (q / kNA) & 1);
        tc_fence_after();
        for (int u = 0; u < ((a.dbg & 1) ? 0 : n); ++u) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t bd = desc_hi | static_cast<uint64_t>(((x0 + (c - it.c0 + u) * 2048 + ks * 1024) >> 4) & 0x3FFF);
            mma_i8(dcol, tbase + ab * (kU * 16) + u * 16 + ks * 8, bd, idesc, (c > it.c0 || u > 0 || ks > 0) ? 1u : 0u);
          }
        }
        commit(aempty + ab);
        __syncwarp();
      }
      commit(dfull + db);
      __syncwarp();
    }
  } else if (warp >= 10) {
    // ---------------- epilogue ----------------
    pdl_wait();  // the partial buffer may still be read by the previous kernel
    pdl_trigger();
    const int quarter = warp & 3, row = quarter * 32 + lane;
    const bool h = (row >> 3) & 1;
    uint32_t sw = 0;
    int prev = -1;
    for (int item = i0, n_it = 0; item < i1; ++item, ++n_it) {
      const Item it = item_of(a, item);
      if (it.key != prev) {
        mbar_wait(xready, sw & 1);
        ++sw;
        prev = it.key;
      }
      const int db = n_it & 1;
      mbar_wait(dfull + db, (n_it >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      const uint32_t taddr = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + kDCol + db * 32;
      tmem_ld16(taddr, v);
      tmem_ld16(taddr + 16, v + 16);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float* out = a.partial + static_cast<int64_t>(it.s) * a.M * a.Np + static_cast<int64_t>(it.tile) * 128 + row;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        if (m < a.M) {
          const long long r = 256ll * static_cast<int>(v[m]) + static_cast<int>(v[16 + m]);
          // same rounding as gemv.cu i4_rows: rows g + 8 carry 16 (code + 8)
          const float y = h ? static_cast<float>(r - 128ll * dsum[m]) * (0.0625f * sxs[m])
                            : static_cast<float>(r - 8ll * dsum[m]) * sxs[m];
          out[static_cast<int64_t>(m) * a.Np] = y;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + db);  // also releases the slice scales / sums (read above)
    }
  } else {
    // ---------------- transcode (+ the digit B operand at every new k-slice) ----------------
    pdl_wait();
    pdl_trigger();
    trace_point(11);
    const int tid = threadIdx.x;  // 0..255
    const int group = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane = feature of the 128-feature tile
    // staged chunk = 32 rows of 128 B (row R = 4 i16 + g / 2 holds rows g, g ^ 1), 128 B swizzle:
    // logical 16 B unit v of row R sits at unit v ^ (R & 7)
    const int i16 = row >> 4, g = row & 7, rr = i16 * 4 + (g >> 1), half = g & 1;
    const uint32_t mask = ((row >> 3) & 1) ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    uint32_t q = 0, sw = 0;
    int prev = -1;
    for (int item = i0, n_it = 0; item < i1; ++item, ++n_it) {
      const Item it = item_of(a, item);
      if (it.key != prev) {
        // every previous item's epilogue is done: its MMAs read the old digits, it read the old scales
        if (n_it >= 1) mbar_wait(dempty + ((n_it - 1) & 1), ((n_it - 1) >> 1) & 1);
        if (n_it >= 2) mbar_wait(dempty + ((n_it - 2) & 1), ((n_it - 2) >> 1) & 1);
        const int nck = it.c1 - it.c0;
        if (tid == 0) {
          mbar_expect_tx(xbar, static_cast<uint32_t>(a.box * 2048));
          tma_rows(xs, (it.key & 1) ? &xmap2 : &xmap, it.c0, xbar);
        }
        if (tid < 16) {
          amax[tid] = 0;
          dsum[tid] = 0;
        }
        mbar_wait(xbar, sw & 1);
        trace_point(14);
        bar_transcode();
        // (1) per-token max |x| over the slice (chunk blocks [16 tokens][128 B], one warp per
        // chunk, lane l reads 16 B units l + 32 j = token l / 8 + 4 j): half bits of |x| compare
        // as integers (NaN > inf)
        uint32_t mx2[4] = {0u, 0u, 0u, 0u};
        for (int c = warp; c < nck; c += 8) {
          const uint4* blk = reinterpret_cast<const uint4*>(xs + c * 2048);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 u = blk[lane + 32 * j];
            mx2[j] = __vmaxu2(mx2[j], u.x & 0x7FFF7FFFu);
            mx2[j] = __vmaxu2(mx2[j], u.y & 0x7FFF7FFFu);
            mx2[j] = __vmaxu2(mx2[j], u.z & 0x7FFF7FFFu);
            mx2[j] = __vmaxu2(mx2[j], u.w & 0x7FFF7FFFu);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int mh = static_cast<int>(max(mx2[j] & 0xFFFFu, mx2[j] >> 16));
          mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, 1));
          mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, 2));
          mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, 4));
          if ((lane & 7) == 0 && mh) atomicMax(&amax[(lane >> 3) + 4 * j], mh);
        }
        bar_transcode();
        if (tid < 16) {
          const int hb = amax[tid];
          const bool bad = hb >= 0x7C00;
          const float mxf = __half2float(__ushort_as_half(static_cast<unsigned short>(hb)));
          sxs[tid] = bad ? __int_as_float(0x7fc00000) : mxf / kDigitQ;
          isx[tid] = (mxf > 0.f && !bad) ? kDigitQ / mxf : 0.f;
        }
        bar_transcode();
        trace_point(15);
        // (2) in place, one warp per chunk: the chunk's [16 tokens][4 groups t][32 B] become the B
        // operand's [t][16 hi rows | 16 lo rows][16 B]; lane = (token m, groups 2 tp, 2 tp + 1)
        const int m = lane & 15, tp = lane >> 4;
        const float inv = isx[m];
        int ssum = 0;
        for (int c = warp; c < nck; c += 8) {
          uint4* blk = reinterpret_cast<uint4*>(xs + c * 2048);
          const uint4 a0 = blk[m * 8 + tp * 4 + 0], a1 = blk[m * 8 + tp * 4 + 1];
          const uint4 b0 = blk[m * 8 + tp * 4 + 2], b1 = blk[m * 8 + tp * 4 + 3];
          __syncwarp();
          uint4 hi, lo;
          ssum += digits_regs(a0, a1, inv, hi, lo);
          blk[(2 * tp) * 32 + (m >> 3) * 8 + (m & 7)] = hi;
          blk[(2 * tp) * 32 + (2 + (m >> 3)) * 8 + (m & 7)] = lo;
          ssum += digits_regs(b0, b1, inv, hi, lo);
          blk[(2 * tp + 1) * 32 + (m >> 3) * 8 + (m & 7)] = hi;
          blk[(2 * tp + 1) * 32 + (2 + (m >> 3)) * 8 + (m & 7)] = lo;
          __syncwarp();
        }
        ssum += __shfl_xor_sync(0xffffffffu, ssum, 16);
        if (lane < 16 && ssum) atomicAdd(&dsum[m], ssum);  // integer: order-independent
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_transcode();
        if (tid == 0) mbar_arrive(xready);
        trace_point(12);
        ++sw;
        prev = it.key;
      }
      for (int c = it.c0; c < it.c1; c += kU, ++q) {
        if ((q & 1) != static_cast<uint32_t>(group)) continue;
        const int ws = q % kNS, ab = q % kNA, n = min(kU, it.c1 - c);
        mbar_wait(wfull + ws, (q / kNS) & 1);
        uint32_t r[kU * 16];
        const uint8_t* st = ring + static_cast<size_t>(ws) * kStageB + rr * 128;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (u < n && !(a.dbg & 4)) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint4 w = *reinterpret_cast<const uint4*>(st + u * kChunkBytes + (((half * 4 + t) ^ (rr & 7)) << 4));
              r[u * 16 + 4 * t + 0] = w.x & mask;
              r[u * 16 + 4 * t + 1] = w.y & mask;
              r[u * 16 + 4 * t + 2] = w.z & mask;
              r[u * 16 + 4 * t + 3] = w.w & mask;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(wempty + ws);
        mbar_wait(aempty + ab, ((q / kNA) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (u < n && !(a.dbg & 2)) tmem_st16(lane_base + ab * (kU * 16) + u * 16, r + u * 16);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(afull + ab);
      }
    }
    trace_point(13);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

}  // namespace

void gemv_tc_launch(const GemvOp& op, int M, float* partial, const GemvPlan& p, cudaStream_t st) {
  if (op.bits != 4 || M < 1 || M > 16 || op.nrt % 8 || p.ksplit < 1 || p.per < 1)
    fail(GLM_CONTRACT, "qlinear", "GEMV plan does not match the tcgen05 decode kernel");
  const int64_t slice_max = (op.nch + p.ksplit - 1) / p.ksplit;
  if (slice_max > kSliceChunks) fail(GLM_CONTRACT, "qlinear", "k-slice exceeds the tcgen05 decode kernel's buffer");
  const bool two = op.xf2 && op.xf2 != op.xf;
  if (two && op.rt_split % 8) fail(GLM_CONTRACT, "qlinear", "split activation launch needs 128-feature boundaries");
  TcArgs a;
  a.partial = partial;
  a.Np = op.nrt * kTileN;
  a.nch = static_cast<int>(op.nch);
  a.ntiles = static_cast<int>(op.nrt / 8);
  a.ksplit = p.ksplit;
  a.M = M;
  a.per = p.per;
  a.split_tiles = two ? static_cast<int>(op.rt_split / 8) : a.ntiles;
  a.box = static_cast<int>(slice_max);
  static const int pf = [] { const char* e = getenv("GLM_TC_PF"); return e ? atoi(e) : -1; }();
  a.pf = pf;
  static const int dbg = [] { const char* e = getenv("GLM_TC_DBG"); return e ? atoi(e) : 0; }();
  a.dbg = dbg;
  a.codes = static_cast<const uint8_t*>(op.codes);
  const CUtensorMap wmap = codes_tensor_map_raw(op.codes, op.nrt, op.nch, 4, 8, true);
  // x_frag [M][nch][128 B] viewed as [chunk][token][128 B]
  const CUtensorMap xmap = rows_tensor_map(op.xf, 128, M, op.nch * 128, op.nch, 128, 16, a.box);
  const CUtensorMap xmap2 = two ? rows_tensor_map(op.xf2, 128, M, op.nch * 128, op.nch, 128, 16, a.box) : xmap;
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_tc_i4, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem)));
    attr = true;
  }
  const int nitems = a.ntiles * a.ksplit;
  const int grid = (nitems + a.per - 1) / a.per;
  launch_k(k_gemv_tc_i4, dim3(grid), dim3(kThreads), kSmem, st, a, wmap, xmap, xmap2);
  LAUNCH_CHECK("k_gemv_tc_i4");
}

}  // namespace glm
