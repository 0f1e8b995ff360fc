// block.h — argument blocks + launchers of the GLM block kernels (block.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "layout.cuh"

namespace glm {

// A sublayer output still in GEMV split-K partial form: value(m, n) =
// scale[n] * sum_s p[s * split_stride + m * ld + n] (scale may be null = 1).
struct SubIn {
  const float* p = nullptr;
  int ksplit = 1;
  int64_t split_stride = 0, ld = 0;
  const float* scale = nullptr;
  // zeropoint weights (quant.cpp:145-186): y[m][n] += zt[m] * zv[n] after the column scale
  // (gemv.cu QWeightDev::zvec / zp_sums_frag); null for absmax
  const float* zt = nullptr;
  const float* zv = nullptr;
};

// Destination activation buffer (fp16) of the next quantized linear, with its kRow
// activation fold (row_scale may be null = 1). xf == null disables the output. Layout per
// consumer (layout.cuh): x_frag for the decode GEMV (tile == 0, nch chunks) or 128-token
// tcgen05 B-operand tiles for the prefill GEMM (tile == 1, padded depth Kp).
struct XOut {
  __half* xf = nullptr;
  int64_t nch = 0, Kp = 0;
  int tile = 0;
  const float* row_scale = nullptr;
};

#if defined(__CUDACC__)
// Store the pair (k, k+1) of row m into the consumer's activation buffer (fp16, with the
// consumer's kRow fold).
__device__ __forceinline__ void store_xfrag_pair(const XOut& xo, int m, int64_t k, float v0, float v1) {
  if (!xo.xf) return;
  const float s0 = xo.row_scale ? xo.row_scale[k] : 1.f, s1 = xo.row_scale ? xo.row_scale[k + 1] : 1.f;
  const int64_t idx = xo.tile ? xtile_index(xo.Kp, m, k) : xfrag_index(xo.nch, m, k);
  *reinterpret_cast<__half2*>(xo.xf + idx) = __floats2half2_rn(v0 * s0, v1 * s1);
}
#endif

// Fused decode allreduce of a row-parallel sublayer output (tensor parallelism, collective.h):
// rank r pushes its [row m][CTA slice c] of the sublayer output into inbox[dst] slot
// (gen & 1, r) of every rank dst, then raises flags[dst][(gen & 1, r, m, c)] = gen; each rank
// sums the t slots of its own inbox in rank order once the t flags read gen, so every rank
// computes bit-identical sums. gen counts the calls per (m, c) (own counters). mode: 1 push
// only, 2 wait + sum only (the two halves of the emulated single-GPU group, separated by a
// host barrier), 3 both (one launch per rank on real multi-GPU).
constexpr int kMaxTp = 8;
constexpr int kPeerSlices = 8;  // one flag per (row, LayerNorm cluster CTA)
struct PeerArgs {
  float* inbox[kMaxTp] = {};     // per destination rank: [2][size][max_b][d] fp32
  unsigned* flags[kMaxTp] = {};  // per destination rank: [2][size][max_b][kPeerSlices]
  unsigned* gen = nullptr;       // own: [max_b][kPeerSlices]
  int* err = nullptr;            // own: set when a peer's flag does not arrive (timeout)
  int rank = 0, size = 1, max_b = 0, mode = 3;
  int64_t d = 0;
};

struct LnArgs {
  SubIn in;
  float* h;                 // [M][d] residual in / LN output out
  const float *gain, *bias;
  float alpha, eps;
  int64_t d;
  XOut x0, x1;              // up to two consumers (ffn_w1 and ffn_v have distinct kRow scales)
  float* tap;               // optional [M][d] copy of the sublayer output
  int zero_sublayer;
  PeerArgs peer{};          // size > 1: sum the sublayer output across tensor-parallel ranks
  int half_store = 0;       // PrecisionPolicy kHalfEmulated: round the sublayer output and h to fp16 (model.cpp:213-223)
};

struct ActArgs {
  SubIn w1, v;
  int M;
  int64_t f;
  XOut xo;
};

struct AttnDecodeArgs {
  SubIn qkv;                // partials of the fused qkv GEMV, local columns [q | k | v]
  int64_t d_local;          // heads_local * dh
  int heads, dh, max_ctx, max_splits;
  const int* positions;     // [B]
  const int* cache_len;     // [B]
  const float2* rope;       // [max_pos][dh/2] (cos, sin)
  __half *kcache, *vcache;  // [B][heads][max_ctx][dh] for this layer
  float* part;              // [B][heads][max_splits][dh + 2]
  int* counters;            // [B][heads], zero-initialised
  XOut xo;                  // x_frag of out_proj
  float* out;               // optional fp32 [B][d_local]
  float prescale = 0.f;     // > 0: PrecisionPolicy kHalfEmulated, scores stored as fp16(score / prescale) (model.cpp:143-148)
  int stage_keys = 0;       // set by launch_attn_decode: keys per CTA staged in shared memory (0: read from L2/HBM)
  int split_keys = 256;     // set by launch_attn_decode: cached keys per CTA (attn_decode_split_keys)
};

struct RopeStoreArgs {
  const float* qkv;         // [n][ldqkv] reduced fp32 (local columns [q | k | v])
  int64_t ldqkv, d_local;
  int n, heads, dh, seq, max_ctx, slot0;
  const int* positions;
  const float2* rope;
  float* q;                 // [heads][n][dh] rotated q
  __half *kcache, *vcache;
  const __half* qkv_h = nullptr;  // fp16 rows instead of qkv (prefill GEMM output, head_dim 128)
};

struct AttnPrefillArgs {
  const float* q;           // [heads][n][dh]
  const __half *kcache, *vcache;
  int n, heads, dh, seq, max_ctx, context_len;
  float* out;               // [n][ldout]
  int64_t ldout;
  // tcgen05 kernel only (attn_prefill_umma_eligible): write O straight into the out-proj's
  // activation tiles at token rows xrow0 + i instead of the fp32 rows
  XOut xo{};
  int xrow0 = 0;
  float prescale = 0.f;     // > 0: PrecisionPolicy kHalfEmulated (see AttnDecodeArgs)
};

struct HeadArgs {
  const void* E;            // [vocab][d] fp32 or bf16 (full table; rows offset below)
  const float* h;           // [M][d]
  int M;
  int64_t d, vocab_offset, vocab_local;
  float* logits;            // optional [M][ld_logits], written at column vocab_offset + v
  int64_t ld_logits;
  unsigned long long* argmax;  // [M] packed (value, ~index), zero-initialised
  __nv_bfloat16* hb = nullptr;  // [M][d] scratch: bf16 copy of h for the tensor-core head
};

// half_store: round h to fp16 (PrecisionPolicy kHalfEmulated, model.cpp:197)
void launch_embed(const void* E, bool bf16, int64_t d, const int* tokens, int M, float* h, const XOut& xo,
                  cudaStream_t st, bool half_store = false);
void launch_deepnorm_ln(const LnArgs& a, int M, cudaStream_t st);
void launch_geglu_act(const ActArgs& a, cudaStream_t st);
// keys per CTA of the decode attention: 256 up to a 256-token cache (no merge), else 64
// (long caches: many small CTAs stream the cache concurrently, deterministic merge)
int attn_decode_split_keys(int max_ctx);
int attn_decode_split_keys(int max_ctx, int batch);
int attn_decode_splits(int max_ctx);  // capacity of the split partial buffer
void launch_attn_decode(const AttnDecodeArgs& a, int B, cudaStream_t st);
void launch_advance(int* cache_len, int B, cudaStream_t st);
void launch_rope_store(const RopeStoreArgs& a, cudaStream_t st);
void launch_attn_prefill(const AttnPrefillArgs& a, cudaStream_t st);
// tcgen05 prefill attention (attn_tc.cu): false if it does not take this call (head_dim != 128)
bool launch_attn_prefill_umma(const AttnPrefillArgs& a, cudaStream_t st);
bool attn_prefill_umma_eligible(int dh);
void launch_rows_to_xfrag(const float* x, int64_t ld, int M, int64_t K, const XOut& xo, cudaStream_t st);
void launch_head(const HeadArgs& a, bool bf16, cudaStream_t st);
// status (optional): set to 1 when a row's winning logit is not finite
void launch_argmax_finish(unsigned long long* keys, int* tokens, int M, cudaStream_t st, int* status = nullptr);

}  // namespace glm
