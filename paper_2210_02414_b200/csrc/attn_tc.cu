// attn_tc.cu — prefill attention on the 5th-generation tensor cores (head_dim 128).
//
// softmax(q k^T / sqrt(dh) + gMASK) v for one [gMASK] sample (model.cpp:137-152; visibility
// j < max(C, i + 1), corruption.cpp:338-367), flash schedule over 128-key blocks, two
// 128-row query tiles per CTA so the tensor core works on one tile while the other's
// softmax runs:
//
//   warp 9      MMA issuer: S_t(j) = Q_t K_j^T into tile t's TMEM score columns (A = Q_t and
//               B = K_j from shared memory, K-major), then, once softmax t has written P_t(j)
//               over the first half of those columns, O_t += P_t(j) V_j (A = P_t from TMEM,
//               B = V_j from shared memory, MN-major) and at once S_t(j + 1);
//   warp 8      producer: K_j and V_j of the sequence's fp16 cache rows into two shared-
//               memory slots, one tensor-map TMA per tile (box 64 dh x 128 keys x 2 dh
//               halves, 128 B swizzle: the same bytes serve as the K-major B operand of
//               Q K^T and, for V, as the MN-major B operand of P V);
//   warps 0-7   softmax, group t = warps 4t..4t+3, one query row per thread = one TMEM lane:
//               the score row (fp32) from TMEM, gMASK, online max / sum in fp32, P = 2^(s - m)
//               as fp16 back into TMEM, the O_t rescale in TMEM when a row's max rises, and
//               the final O / l store.
//
// TMEM columns: S_t / P_t [128 t, 128 t + 128), O_t [256 + 128 t, 384 + 128 t).
#include <cuda.h>

#include <cfloat>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "block.h"
#include "common.cuh"

namespace glm {

namespace {

constexpr int kUR = 128;   // query rows per CTA (UMMA M)
constexpr int kUK = 128;   // keys per block (UMMA N of S, K of P.V)
constexpr int kUD = 128;   // head dim (UMMA K of S, N of P.V)
constexpr int kTileBytes = kUR * kUD * 2;  // 32 KB: Q, one K block, one V block
constexpr int kUTiles = 2;      // query tiles per CTA: one softmax group each, the tensor core alternates
constexpr int kUSlots = 2;      // K/V block slots (one TMA per tile)
constexpr int kUThreads = (4 * kUTiles + 2) * 32;
constexpr uint32_t kColS = 0, kColO = 256;  // S_t / P_t at 128 t, O_t at 256 + 128 t
constexpr size_t kUSmem = (static_cast<size_t>(kUTiles) + 2 * kUSlots) * kTileBytes + 1024;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void ub_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void ub_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void ub_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(bar))
      : "memory");
}
// D (TMEM) (+)= A (smem desc) * B (smem desc)
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D (TMEM) (+)= A (TMEM) * B (smem desc)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Shared-memory matrix descriptor, no swizzle: start >> 4, leading / stride byte offsets >> 4,
// sm100 descriptor version bit 46.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// 128-byte-swizzled tiles (what a TMA box with a 128 B inner extent writes at full speed):
// a 128-row x 128-element fp16 tile is two 16 KB halves [element/64][row][64 elements],
// each 128 B row with its 16-byte chunks XOR-ed by row % 8. Descriptor layout type 2
// (SWIZZLE_128B), 8-row stride (SBO) 1024 B; for the K-major Q and K the MMA's 16-element
// K step moves 32 B inside a row, for the MN-major V the two 64-element N halves are 16 KB
// apart (LBO) and a 16-key K step moves 2 KB.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return sdesc(addr, lbo, sbo) | (2ull << 61);
}
__device__ __forceinline__ uint32_t sw128_off(int row, int e) {
  return (e >> 6) * 16384 + row * 128 + ((((e & 63) >> 3) ^ (row & 7)) << 4) + (e & 7) * 2;
}


__device__ __forceinline__ void tma_kv(void* dst, const CUtensorMap* map, int key0, int head, int seq, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          su32(dst)),
      "l"(map), "r"(0), "r"(key0), "r"(0), "r"(head), "r"(seq), "r"(su32(bar))
      : "memory");
}  // (box: 64 elements x 128 keys x 2 halves of dh, 128 B swizzle)
__device__ __forceinline__ void ub_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}

// sm_100 three-input max and packed fp32-pair add / subtract (FMNMX3, FADD2)
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float2 add2f(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 sub2f(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n sub.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__global__ void __launch_bounds__(kUThreads, 1) k_attn_prefill_umma(AttnPrefillArgs a, int v_lbo, int v_sbo,
                                                                    const __grid_constant__ CUtensorMap kmap,
                                                                    const __grid_constant__ CUtensorMap vmap) {
  extern __shared__ __align__(1024) uint8_t usm_raw[];
  uint8_t* usm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(usm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = usm;                                          // [kUTiles]
  uint8_t* Ks = usm + kUTiles * kTileBytes;                   // [kUSlots]
  uint8_t* Vs = usm + (kUTiles + kUSlots) * kTileBytes;       // [kUSlots]
  __shared__ __align__(8) uint64_t kv_full[kUSlots], kv_empty[kUSlots], s_full[kUTiles], p_full[kUTiles],
      o_done[kUTiles], q_ready;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y, i0 = blockIdx.x * (kUTiles * kUR);
  const int n = a.n, C = a.context_len;
  const int kend = min(n, max(C, i0 + kUTiles * kUR));  // keys visible to some row of the CTA
  const int nblk = (kend + kUK - 1) / kUK;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < kUSlots; ++i) {
      ub_init(kv_full + i, 1);
      ub_init(kv_empty + i, 1);
    }
    for (int t = 0; t < kUTiles; ++t) {
      ub_init(s_full + t, 1);
      ub_init(p_full + t, 4);
      ub_init(o_done + t, 1);
    }
    ub_init(&q_ready, 4 * kUTiles);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = tmem_slot;

  if (warp < 4 * kUTiles) {
    // ---------------- softmax group t (4 warps): one query row per thread = TMEM lane ----------------
    const int t = warp >> 2, q = warp & 3;
    const int r = q * 32 + lane;
    const int i = i0 + t * kUR + r;
    // Q row -> fp16 scaled by log2(e) / sqrt(dh) into the swizzled K-major tile of group t
    {
      const float qs = 1.4426950408889634f * rsqrtf(static_cast<float>(kUD));
      const float4* qrow = reinterpret_cast<const float4*>(a.q + (static_cast<int64_t>(head) * n + (i < n ? i : 0)) * kUD);
      uint8_t* Qt = Qs + t * kTileBytes;
#pragma unroll
      for (int k = 0; k < kUD; k += 8) {
        const float4 v0 = i < n ? qrow[k / 4] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 v1 = i < n ? qrow[k / 4 + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
        const __half2 h0 = __floats2half2_rn(v0.x * qs, v0.y * qs), h1 = __floats2half2_rn(v0.z * qs, v0.w * qs);
        const __half2 h2 = __floats2half2_rn(v1.x * qs, v1.y * qs), h3 = __floats2half2_rn(v1.z * qs, v1.w * qs);
        *reinterpret_cast<uint4*>(Qt + sw128_off(r, k)) =
            make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                       *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) ub_arrive(&q_ready);
    }
    const int lim = min(max(C, i + 1), n);  // keys j < lim are visible to row i
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t colS = kColS + t * kUK, colO = kColO + t * kUD;  // P_t overwrites S_t's first 64 columns
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      ub_wait(s_full + t, j & 1);  // S_t(j) complete => P.V_t(j - 1) complete as well (in order)
      fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tld32(lane_base + colS + c * 32, sr[c]);
      twait_ld();
      float sv[kUK];
#pragma unroll
      for (int c = 0; c < kUK; ++c) sv[c] = __uint_as_float(sr[c >> 5][c & 31]);
      if (a.prescale > 0.f) {  // half-emulated storage: fp16(score / prescale), log2 units here
        const float to = 0.6931471805599453f / a.prescale, back = a.prescale * 1.4426950408889634f;
#pragma unroll
        for (int c = 0; c < kUK; ++c) sv[c] = half_round(sv[c] * to) * back;
      }
      const int j0 = j * kUK;
      if (!__all_sync(0xffffffffu, j0 + kUK <= lim)) {
#pragma unroll
        for (int c = 0; c < kUK; ++c)
          if (j0 + c >= lim) sv[c] = -INFINITY;
      }
      // row max: 8 chains of three-input max (FMNMX3), half the instructions of fmaxf
      float bm8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) bm8[u] = sv[u];
#pragma unroll
      for (int c = 8; c + 16 <= kUK; c += 16)
#pragma unroll
        for (int u = 0; u < 8; ++u) bm8[u] = max3f(bm8[u], sv[c + u], sv[c + 8 + u]);
#pragma unroll
      for (int u = 0; u < 8; ++u) bm8[u] = fmaxf(bm8[u], sv[kUK - 8 + u]);
      const float bm = max3f(max3f(bm8[0], bm8[1], bm8[2]), max3f(bm8[3], bm8[4], bm8[5]), fmaxf(bm8[6], bm8[7]));
      // lazy max: the exponent reference moves only when a score exceeds it by more than
      // 8 (P <= 2^8 stays exact enough in fp16, l and O accumulate in fp32), so O needs a
      // rescale in TMEM only rarely after the first blocks
      const float mn = bm > m + 8.f ? bm : m;
      const float ms = mn == -INFINITY ? 0.f : mn;  // row with nothing visible yet: p = 0
      const float corr = ex2(m - ms);
      l *= corr;
      // exponent arguments and the row sum on packed fp32 pairs (FADD2): one instruction per
      // two scores instead of two
      uint32_t pw[kUK / 2];
      float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 ms2 = make_float2(ms, ms);
#pragma unroll
      for (int c = 0; c < kUK; c += 2) {
        const float2 x = sub2f(make_float2(sv[c], sv[c + 1]), ms2);
        const float p0 = ex2(x.x), p1 = ex2(x.y);
        ls[(c >> 1) & 3] = add2f(ls[(c >> 1) & 3], make_float2(p0, p1));
        const __half2 hv = __floats2half2_rn(p0, p1);
        pw[c / 2] = *reinterpret_cast<const uint32_t*>(&hv);
      }
      const float2 ls01 = add2f(ls[0], ls[1]), ls23 = add2f(ls[2], ls[3]), lsum = add2f(ls01, ls23);
      l += lsum.x + lsum.y;
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {  // O_t rescale (P.V_t(j - 1) is complete)
#pragma unroll
        for (int h = 0; h < kUD; h += 64) {
          uint32_t v0[32], v1[32];
          tld32(lane_base + colO + h, v0);
          tld32(lane_base + colO + h + 32, v1);
          twait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            v0[e] = __float_as_uint(__uint_as_float(v0[e]) * corr);
            v1[e] = __float_as_uint(__uint_as_float(v1[e]) * corr);
          }
          tst32(lane_base + colO + h, v0);
          tst32(lane_base + colO + h + 32, v1);
        }
      }
      tst32(lane_base + colS, *reinterpret_cast<const uint32_t(*)[32]>(&pw[0]));
      tst32(lane_base + colS + 32, *reinterpret_cast<const uint32_t(*)[32]>(&pw[32]));
      twait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) ub_arrive(p_full + t);
      m = mn;
    }
    // ---- O / l ----
    if (nblk > 0) {
      ub_wait(o_done + t, (nblk - 1) & 1);
      fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int c = 0; c < kUD; c += 32) {
      uint32_t v[32];
      if (nblk > 0) {
        tld32(lane_base + colO + c, v);
        twait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
      }
      if (i < n && a.xo.xf) {  // fp16 activation tiles of the out-proj (16-byte runs of 8 features)
        const int64_t m = a.xrow0 + i;
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          const int64_t k = static_cast<int64_t>(head) * kUD + c + e;
          uint32_t hx[4];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float s0 = a.xo.row_scale ? a.xo.row_scale[k + j] : 1.f;
            const float s1 = a.xo.row_scale ? a.xo.row_scale[k + j + 1] : 1.f;
            const __half2 hv = __floats2half2_rn(__uint_as_float(v[e + j]) * inv * s0, __uint_as_float(v[e + j + 1]) * inv * s1);
            hx[j / 2] = *reinterpret_cast<const uint32_t*>(&hv);
          }
          *reinterpret_cast<uint4*>(a.xo.xf + xtile_index(a.xo.Kp, m, k)) = make_uint4(hx[0], hx[1], hx[2], hx[3]);
        }
      } else if (i < n) {
        float* orow = a.out + static_cast<int64_t>(i) * a.ldout + head * kUD + c;
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(orow + e) = make_float4(__uint_as_float(v[e]) * inv, __uint_as_float(v[e + 1]) * inv,
                                                             __uint_as_float(v[e + 2]) * inv, __uint_as_float(v[e + 3]) * inv);
      }
    }
  } else if (warp == 4 * kUTiles) {
    // ---------------- producer: K_j, V_j into slot j % kUSlots (keys past the cache arrive as zeros) ----------------
    if (lane == 0)
      for (int j = 0; j < nblk; ++j) {
        const int slot = j % kUSlots;
        ub_wait(kv_empty + slot, ((j / kUSlots) & 1) ^ 1);
        ub_expect_tx(kv_full + slot, 2 * kTileBytes);
        tma_kv(Ks + slot * kTileBytes, &kmap, j * kUK, head, a.seq, kv_full + slot);
        tma_kv(Vs + slot * kTileBytes, &vmap, j * kUK, head, a.seq, kv_full + slot);
      }
  } else {
    // ---------------- MMA issuer: S_A(j), S_B(j); then per tile P.V_t(j) and S_t(j + 1) ----------------
    // kind::f16: D f32 (bit 4), A/B f16, N >> 3 at bit 17, M >> 4 at bit 24; bit 16: B MN-major
    const uint32_t idesc_s = (1u << 4) | (static_cast<uint32_t>(kUK >> 3) << 17) | (static_cast<uint32_t>(kUR >> 4) << 24);
    const uint32_t idesc_o = (1u << 4) | (1u << 16) | (static_cast<uint32_t>(kUD >> 3) << 17) | (static_cast<uint32_t>(kUR >> 4) << 24);
    ub_wait(&q_ready, 0);
    auto issue_s = [&](int t, int j) {
      const uint32_t qa = su32(Qs + t * kTileBytes), k0 = su32(Ks + (j % kUSlots) * kTileBytes);
#pragma unroll
      for (int ks = 0; ks < kUD / 16; ++ks)
        mma_ss(tbase + kColS + t * kUK, sdesc_sw128(qa + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024),
               sdesc_sw128(k0 + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
      commit_elect(s_full + t);
    };
    auto issue_pv = [&](int t, int j) {
      const uint32_t v0 = su32(Vs + (j % kUSlots) * kTileBytes);
#pragma unroll
      for (int ks = 0; ks < kUK / 16; ++ks)
        mma_ts(tbase + kColO + t * kUD, tbase + kColS + t * kUK + ks * 8, sdesc_sw128(v0 + ks * 2048, v_lbo, v_sbo),
               idesc_o, (j > 0 || ks > 0) ? 1u : 0u);
      commit_elect(o_done + t);
    };
    if (nblk > 0) {
      ub_wait(kv_full, 0);
      fence_after();
      for (int t = 0; t < kUTiles; ++t) issue_s(t, 0);
      __syncwarp();
    }
    for (int j = 0; j < nblk; ++j) {
      const bool more = j + 1 < nblk;
      if (more) ub_wait(kv_full + (j + 1) % kUSlots, ((j + 1) / kUSlots) & 1);
      for (int t = 0; t < kUTiles; ++t) {
        ub_wait(p_full + t, j & 1);
        fence_after();
        issue_pv(t, j);
        if (t == kUTiles - 1) commit_elect(kv_empty + j % kUSlots);  // every MMA of block j issued
        if (more) issue_s(t, j + 1);
        __syncwarp();
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

}  // namespace

namespace {
// Tensor map of one layer's K or V cache [batch][heads][max_ctx][128] fp16 as the 5-D view
// (64 halves, key, dh half, head, sequence) with strides (256 B, 128 B, ...): a box of
// (64, 128, 2, 1, 1) with the 128 B swizzle lands as [dh half][key][64 halves] (sw128_off).
// Rows beyond the cache read as zeros. Maps are cached per (buffer, shape): a later model may
// reuse an address with another shape.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
CUtensorMap kv_tensor_map(const __half* base, const AttnPrefillArgs& a) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, CUtensorMap> cache;  // (base, max_ctx, heads)
  static EncodeTiledFn encode = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(static_cast<const void*>(base), a.max_ctx, a.heads);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) fail(GLM_CUDA, "attention", "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  // the sequence count is not in the arguments; the map never reads beyond the sequence asked for
  const cuuint64_t dims[5] = {64, static_cast<cuuint64_t>(a.max_ctx), 2, static_cast<cuuint64_t>(a.heads), 65536};
  const cuuint64_t row = kUD * 2;
  const cuuint64_t strides[4] = {row, 128, row * a.max_ctx, row * a.max_ctx * a.heads};
  const cuuint32_t box[5] = {64, kUK, 2, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  CUtensorMap m;
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<__half*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GLM_CUDA, "attention", "K/V tensor map rejected (" + std::to_string(static_cast<int>(r)) + ")");
  cache[key] = m;
  return m;
}
}  // namespace

// The tcgen05 prefill attention takes head_dim 128 (GLM_ATTN_UMMA=0 selects the mma.sync
// flash kernel); V descriptor offsets overridable for bring-up (GLM_ATTN_VLBO / _VSBO; the
// defaults were verified against the oracle: the MN-major V takes the N-half distance as
// LBO and the 8-key stride as SBO).
bool attn_prefill_umma_eligible(int dh) {
  static const int on = [] { const char* e = getenv("GLM_ATTN_UMMA"); return e ? atoi(e) : 1; }();
  return on && dh == kUD;
}

bool launch_attn_prefill_umma(const AttnPrefillArgs& a, cudaStream_t st) {
  if (!attn_prefill_umma_eligible(a.dh)) return false;
  static const int vlbo = [] { const char* e = getenv("GLM_ATTN_VLBO"); return e ? atoi(e) : 16384; }();
  static const int vsbo = [] { const char* e = getenv("GLM_ATTN_VSBO"); return e ? atoi(e) : 1024; }();
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_prefill_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kUSmem)));
    attr = true;
  }
  const CUtensorMap km = kv_tensor_map(a.kcache, a), vm = kv_tensor_map(a.vcache, a);
  const dim3 grid((a.n + kUTiles * kUR - 1) / (kUTiles * kUR), a.heads);
  k_attn_prefill_umma<<<grid, kUThreads, kUSmem, st>>>(a, vlbo, vsbo, km, vm);
  LAUNCH_CHECK("k_attn_prefill_umma");
  return true;
}

}  // namespace glm
