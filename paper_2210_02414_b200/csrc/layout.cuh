// layout.cuh — the B200 device layout of a quantized linear and of its activations.
//
// A reference weight W[K][N] (row-major, y = x.W, model.hpp:41-49) is stored as "row
// tiles" of 16 output features x "chunks" of 64 input features, each tile/chunk a
// contiguous 512 B (INT4) or 1024 B (INT8) block, tiles outermost:
//
//     block(rt, c) at ((rt * nch) + c) * chunk_bytes
//
// Inside a block, lane l = 4g + t of a warp owns exactly the mma.sync.m16n8k16 A
// fragments it needs for the 4 k-tiles of the chunk, so one coalesced 512 B warp load
// (16 B per lane) feeds 4 (INT4) or 2 (INT8) MMAs of the decode GEMV with no shuffles.
// A fragment register r in 0..3 holds rows {g, g+8}[r&1] and k columns
// {2t, 2t+1} + 8*(r>>1) of the 16x16 k-tile (PTX ISA m16n8k16 .f16 A layout).
//
// INT4: word j (k-tile j) of the lane's 16 bytes holds 8 nibbles, offset-binary (code+8):
//   nibble p = r + 4*hi  ->  register r, half hi (hi = odd k column)
//   so (w & 0x000F000F) | 0x6400_6400 is register 0 as fp16 (1024+u), etc.
// INT8: each k-tile takes two words (8 B); the 16 B at +0 hold k-tiles 0,1, the 16 B at
//   +512 hold k-tiles 2,3. Word wd holds registers 2wd, 2wd+1 as bytes
//   [r.lo, r.hi, r'.lo, r'.hi], offset-binary (code+128) for the 0x64 PRMT transcode.
// The prefill kernel (tcgen05, qmm_tc.cu) reads the same blocks through shared memory and
// regroups each feature's codes into TMEM lanes.
//
// Activations have two layouts, chosen by the consumer:
//   * decode GEMV (M <= 16): "fragment order" x_frag[m][c][t][16] fp16 — the 16 halves lane
//     (g = m mod 8, t) needs as B fragments for the 4 k-tiles of chunk c (xfrag_index);
//   * prefill tcgen05 GEMM (M > 16): the tcgen05 K-major no-swizzle canonical layout, core
//     matrices of 8 tokens x 8 k (xtile_index), copied into shared memory as-is by TMA.
#pragma once
#include <stdint.h>

namespace glm {

constexpr int kTileN = 16;   // output features per row tile
constexpr int kChunkK = 64;  // input features per chunk

struct QLayout {
  int64_t K, N;     // logical (reference) shape [K, N]
  int64_t Kp, Np;   // padded: Kp to 128 (two chunks, one tcgen05 stage), Np to 128 (TMEM lanes)
  int64_t nrt, nch; // row tiles, chunks
  int bits;
  __host__ __device__ int64_t chunk_bytes() const { return bits == 4 ? 512 : 1024; }
  __host__ __device__ int64_t bytes() const { return nrt * nch * chunk_bytes(); }
};

inline QLayout make_layout(int64_t K, int64_t N, int bits) {
  QLayout L;
  L.K = K;
  L.N = N;
  L.Kp = (K + 127) / 128 * 128;
  L.Np = (N + 127) / 128 * 128;
  L.nrt = L.Np / kTileN;
  L.nch = L.Kp / kChunkK;
  L.bits = bits;
  return L;
}

// Byte offset (and nibble shift for INT4) of element (k, n) in the device layout.
__host__ __device__ inline int64_t layout_offset(const QLayout& L, int64_t k, int64_t n, int* shift) {
  const int64_t rt = n / kTileN, c = k / kChunkK;
  const int row = static_cast<int>(n % kTileN), kk = static_cast<int>(k % kChunkK);
  const int g = row & 7, rsel = row >> 3;
  const int j = kk >> 4, kc = kk & 15;
  const int hi = kc & 1, t = (kc & 7) >> 1, r = rsel | ((kc >> 3) << 1);
  const int lane = g * 4 + t;
  const int64_t base = (rt * L.nch + c) * L.chunk_bytes();
  if (L.bits == 4) {
    const int p = r + 4 * hi;
    *shift = (p & 1) * 4;
    return base + lane * 16 + j * 4 + (p >> 1);
  }
  *shift = 0;
  const int half = j >> 1, jj = j & 1, wd = r >> 1, b = (r & 1) * 2 + hi;
  return base + half * 512 + lane * 16 + jj * 8 + wd * 4 + b;
}

// Inverse map: element `sub` (nibble 0 = low / 1 = high for INT4, 0 for INT8) of byte `o`.
__host__ __device__ inline void layout_element(const QLayout& L, int64_t o, int sub, int64_t* k, int64_t* n) {
  const int64_t blk = o / L.chunk_bytes();
  const int64_t rt = blk / L.nch, c = blk % L.nch;
  int in = static_cast<int>(o % L.chunk_bytes());
  int lane, j, r, hi;
  if (L.bits == 4) {
    lane = in / 16;
    j = (in % 16) / 4;
    const int p = 2 * (in % 4) + sub;  // nibble position in the word
    r = p & 3;
    hi = p >> 2;
  } else {
    const int half = in / 512;
    in %= 512;
    lane = in / 16;
    const int jj = (in % 16) / 8, wd = (in % 8) / 4, b = in % 4;
    j = half * 2 + jj;
    r = wd * 2 + (b >> 1);
    hi = b & 1;
  }
  const int g = lane >> 2, t = lane & 3;
  *n = rt * kTileN + g + 8 * (r & 1);
  *k = c * kChunkK + j * 16 + 2 * t + 8 * (r >> 1) + hi;
}

// Half index of activation (m, k) in x_frag for a layer with nch chunks.
__host__ __device__ inline int64_t xfrag_index(int64_t nch, int64_t m, int64_t k) {
  const int64_t c = k / kChunkK;
  const int kk = static_cast<int>(k % kChunkK);
  const int j = kk >> 4, kc = kk & 15;
  const int t = (kc & 7) >> 1;
  return ((m * nch + c) * 4 + t) * 16 + j * 4 + (kc >> 3) * 2 + (kc & 1);
}

// Half index of activation (m, k) in a tcgen05 B-operand buffer: T-token tiles (T =
// kXTileTokens, the GEMM's UMMA N), each tile [k/16][k-half][T/8 core-matrix rows of 8
// tokens][8 tokens][8 k] (the K-major no-swizzle canonical layout, LBO = 16·T B, SBO =
// 128 B), so a 64-k stage of a tile is one contiguous 128·T B block for the bulk-copy engine.
constexpr int kXTileTokens = 256;
__host__ __device__ inline int64_t xtile_index(int64_t Kp, int64_t m, int64_t k) {
  constexpr int T = kXTileTokens;
  const int64_t tile = m / T;
  const int mm = static_cast<int>(m % T), kk = static_cast<int>(k % 16);
  return tile * Kp * T + ((k / 16) * 2 + kk / 8) * (8 * T) + (mm / 8) * 64 + (mm % 8) * 8 + kk % 8;
}

}  // namespace glm
