// kernels.h — host-side launchers shared by the C ABI and the model runner.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "glm130b.h"
#include "layout.cuh"
#include "block.h"

namespace glm {

// ---- quant.cu ----
void quantize_device(const void* w, glm_dtype dtype, int64_t rows, int64_t cols, int bits, int scheme,
                     int axis, int8_t* payload, double* scales, double* zps, uint8_t* constant_group,
                     cudaStream_t st);
void dequantize_device(const int8_t* payload, const double* scales, const double* zps, int64_t rows,
                       int64_t cols, int bits, int scheme, int axis, double* out, cudaStream_t st);
void pack_int4_device(const int8_t* codes, int64_t n, int8_t* packed, cudaStream_t st);
void unpack_int4_device(const int8_t* packed, int64_t n, int8_t* codes, cudaStream_t st);
void repack_device(const int8_t* payload, const QLayout& L, void* dev, cudaStream_t st);
struct ShardSpec;
// canonical FULL payload [Kfull, Nfull] -> device layout of the local shard L
void repack_shard_device(const int8_t* payload, int64_t Nfull, const ShardSpec& shard, const QLayout& L,
                         void* dev, cudaStream_t st);
void unrepack_device(const void* dev, const QLayout& L, int8_t* payload, cudaStream_t st);
void runtime_scales_device(const double* scales, int64_t nscales, const QLayout& L, int axis,
                           float* col_scale, float* row_scale, cudaStream_t st);
double host_unkey(unsigned long long k);
// Host check of a canonical absmax payload (n codes): INT4 nibble -8 / INT8 -128 are outside
// the absmax code range (quant.cpp:19-31) -> GLM_CONTRACT; an odd INT4 count must pad with 0.
void validate_absmax_payload(const int8_t* payload, int64_t payload_bytes, int64_t n, int bits);

// Megatron shard of a [K, N] linear: local column j maps to full column
// (j / col_per_rank_block) * col_block + col_offset + (j % col_per_rank_block);
// local row i maps to full row row_offset + i.
struct ShardSpec {
  int64_t col_block, col_per_rank_block, col_offset, row_offset;
};
void gen_quantize_device(uint64_t seed, uint32_t tensor_id, int64_t K, int64_t N, float s_lo,
                         float s_hi, int64_t split, int bits, int axis, const ShardSpec& shard,
                         const QLayout& L, void* dev, double* scales_full, cudaStream_t st);
void gather_scales_device(const double* full, const ShardSpec& shard, int axis, int64_t n_local,
                          double* local, cudaStream_t st);

// ---- gemv.cu : W4A16 / W8A16 decode GEMV (M <= 16) ----
struct QWeightDev {
  QLayout L;
  int axis = 0;
  void* codes = nullptr;         // device layout
  float* col_scale = nullptr;    // [Np] epilogue scale
  float* row_scale = nullptr;    // [Kp] activation fold (kRow), 1 otherwise
  double* scales64 = nullptr;    // canonical FP64 scales of this (local) matrix
  int64_t nscales = 0;
  // zeropoint scheme (quant.cpp:145-186, dequant :209-216): w = s_eff * (code + z) with
  // s_eff = s (or 1 for constant groups, whose codes are 0 and value is z). The MMA still
  // accumulates x . code; the zero points add a rank-1 term y[m][n] += zt[m] * zvec[n] with
  // zt[m] = sum_k x'_k * zeta_k over the fp16 activations the MMA sees (zp_token_sums).
  const float* zvec = nullptr;   // [Np]: s_eff_n * z_n (kColumn), s_eff * z (kWhole), s_max (kRow)
  const float* zeta = nullptr;   // [Kp]: z_k (kRow), 1 (others); 0 beyond K
};
// zt[m] = sum_k half(x[m][k] * row_scale[k]) * zeta[k]   (the zero-point term of zeropoint weights)
void zp_token_sums(const float* x, int64_t ldx, int M, const QWeightDev& w, float* zt, cudaStream_t st);
// the same sums from the fp16 activations already in the consumer layout (tile 0: decode x_frag,
// 1: tcgen05 token tiles); M rows
void zp_sums_act(const __half* xf, int M, const QWeightDev& w, int tile, float* zt, cudaStream_t st);

struct GemvPlan {
  int ksplit = 1;
  int grid = 1;
  int warps = 16;  // warps per CTA the split-K balance was computed for
  int rt_per_warp = 1;  // multi-token kernel: row tiles per warp (1 or 2)
  int per = 0;          // integer-MMA multi-token kernels: items per CTA (slice-major ranges)
  bool tc = false;      // INT4 2..16 tokens on the tcgen05 kernel (gemv_tc.cu)
};
int mk_row_tiles(int bits, int M);
// Split-K plan for an M-row GEMV; the single-token INT4 kernel runs more warps per SM.
GemvPlan plan_gemv(const QLayout& L, int M);
// nx: activation vectors the launch reads (2 for a fused W1|V launch with distinct kRow folds)
GemvPlan plan_gemv(int64_t nrt, int64_t nch, int M, int bits, int nx = 1);
// One decode-GEMV launch (M <= 16) over nrt row tiles of contiguous device-layout codes;
// row tiles >= rt_split read x_frag xf2 (fused W1|V launch, distinct kRow folds).
struct GemvOp {
  const void* codes;
  int bits;
  int64_t nrt, nch;
  const __half* xf;
  const __half* xf2;
  int64_t rt_split;
};

void gemv_launch(const GemvOp& op, int M, float* partial, const GemvPlan& p, cudaStream_t st);
// ---- gemv_tc.cu : INT4 2..16-token decode GEMV on tcgen05 (kind::i8), bit-identical to k_gemv_mk_i4 ----
#ifndef GLM_TC_SLICE
#define GLM_TC_SLICE 64
#endif
constexpr int kTcSliceChunks = GLM_TC_SLICE;  // longest k-slice (64-k chunks) of one item
void gemv_tc_launch(const GemvOp& op, int M, float* partial, const GemvPlan& p, cudaStream_t st);
// Which decode-GEMV kernel gemv_launch runs for M tokens (diagnostics / parity contracts)
enum GemvKind { kGemvF16Single = 0, kGemvI4Single = 1, kGemvI4Multi = 2, kGemvF16Multi = 3, kGemvF16Tma = 4, kGemvI4Tc = 6 };
int gemv_kind(int64_t nch, int M, int bits, int nx = 1);
int gemv_kind(const GemvPlan& p, int64_t nch, int M, int bits, int nx = 1);
// partial[s][m][n] (fp32, [ksplit][M][Np]) = sum over k-split s of x . W
void gemv_launch(const QWeightDev& w, const __half* xfrag, int M, float* partial, const GemvPlan& p,
                 cudaStream_t st);

// ---- qmm_tc.cu : tcgen05 quantized GEMM for prefill (M > 16 tokens) ----
int qmm_min_rows();
constexpr int kQmmTokens = kXTileTokens;  // token columns per MMA tile (UMMA N)
inline int xtile_tokens(int M) { return (M + kQmmTokens - 1) / kQmmTokens * kQmmTokens; }
// partial[s][m][n] (fp32, [ksplit][M][Np]) from activations xt in the tcgen05 B-operand
// layout (layout.cuh xtile_index) holding NT = xtile_tokens(M) token rows.
GemvPlan plan_qmm(const QLayout& L, int M);
// y (optional, ksplit == 1): write the scaled result y[M][ldy] directly instead of partials
void qmm_launch(const QWeightDev& w, const __half* xt, int M, float* partial, const GemvPlan& p, cudaStream_t st,
                float* y = nullptr, int64_t ldy = 0, const float* zt = nullptr, bool y_half = false);
// Fused W1|V GEMM + GeGLU (prefill): xo (W2's activation tiles, Kp = xo_Kp, kRow fold xo_rs
// or null) = fp16(gelu(x.W1 * s1) * (x.V * s2)) for absmax W1 / V of one shape sharing x.
bool qmm_geglu_supported(const QWeightDev& w1, const QWeightDev& v, int M);
void qmm_geglu_launch(const QWeightDev& w1, const QWeightDev& v, const __half* xt, int M, __half* xo, int64_t xo_Kp,
                      const float* xo_rs, cudaStream_t st);
void xtile_from_f32(const float* x, int64_t ldx, int M, const QWeightDev& w, __half* xt, cudaStream_t st);
long long*& qmm_trace_ptr();
// Tensor maps (cuTensorMapEncodeTiled through the runtime): the device-layout codes of nrt row
// tiles x nch chunks, box = box_rt row tiles of one chunk, 64 B swizzle (wide: INT4 as 128 B
// rows of two g rows, 128 B swizzle) (cached per buffer);
// and a 3-D byte tensor [groups][rows][inner] with free row / group strides (not cached).
CUtensorMap codes_tensor_map_raw(const void* codes, int64_t nrt, int64_t nch, int bits, int box_rt, bool wide);
CUtensorMap rows_tensor_map(const void* base, int64_t inner_bytes, int64_t rows, int64_t row_stride, int64_t groups,
                            int64_t group_stride, int box_rows, int box_groups);  // diagnostics: device buffer of the last traced launch (GLM_QMM_TRACE)

// x fp32 [M][K] (row stride ldx) -> x_frag fp16 with the kRow scale fold
void xfrag_from_f32(const float* x, int64_t ldx, int M, const QWeightDev& w, __half* xfrag, cudaStream_t st);
// y[m][n] (row stride ldy) = col_scale[n] * sum_s partial[s][m][n]
// (zt: per-row zero-point sums for zeropoint weights, else null)
void gemv_reduce(const float* partial, int ksplit, int M, const QWeightDev& w, float* y, int64_t ldy,
                 cudaStream_t st, const float* zt = nullptr);

// diagnostics: bind the timeline trace buffer of each translation unit (common.cuh)
void trace_bind_gemv(unsigned long long* buf, unsigned long long cap);
void trace_bind_block(unsigned long long* buf, unsigned long long cap);
void trace_bind_model(unsigned long long* buf, unsigned long long cap);
void trace_bind_gemv_tc(unsigned long long* buf, unsigned long long cap);

}  // namespace glm
