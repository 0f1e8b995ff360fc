/* glm130b.h — C ABI of the B200-native GLM-130B quantized inference hot path.
 *
 * Drop-in boundary for the glmlab reference's quantization + model-forward operator
 * API (paths relative to /root/reference/proj). Every entry point names the reference
 * interface it replaces. Exceptions never cross this ABI: each call returns a
 * glm_status (the reference's error classes, include/glmlab/common.hpp:28-56) and
 * glm_last_error() returns the thread-local "[module] message" text.
 *
 * All compute runs on the current CUDA device (sm_100a). There is no CPU fallback:
 * without a usable B200 every compute call returns GLM_CUDA.
 *
 * Conventions
 *   - "host" buffers are ordinary CPU memory owned by the caller; "device" buffers are
 *     CUDA device pointers; `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - A weight matrix is the reference's row-major [rows = in (K), cols = out (N)]
 *     (include/glmlab/model.hpp:41-49), used as y = x . W.
 *   - Quantized payloads are the reference's canonical bytes: INT8 codes in flat
 *     row-major order, or INT4 codes packed two per byte, even flat index in the low
 *     nibble (quant.cpp:223-240). Scales are doubles, one per group (quant.hpp:26-42).
 */
#ifndef GLM130B_H_
#define GLM130B_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GLM_OK = 0,
  GLM_CONTRACT = 1,  /* ContractError  (common.hpp:43) */
  GLM_DIMENSION = 2, /* DimensionError (common.hpp:38) */
  GLM_FORMAT = 3,    /* FormatError    (common.hpp:48) */
  GLM_POLICY = 4,    /* PolicyError    (common.hpp:53) */
  GLM_CUDA = 5,      /* CUDA runtime / device failure (no reference equivalent) */
  GLM_NCCL = 6       /* collective failure (no reference equivalent) */
} glm_status;

typedef enum { GLM_AXIS_ROW = 0, GLM_AXIS_COLUMN = 1, GLM_AXIS_WHOLE = 2 } glm_axis; /* quant.hpp:14 */
typedef enum { GLM_ABSMAX = 0, GLM_ZEROPOINT = 1 } glm_scheme;                       /* quant.hpp:13 */
typedef enum { GLM_F64 = 0, GLM_F32 = 1, GLM_BF16 = 2, GLM_F16 = 3 } glm_dtype;

const char* glm_last_error(void);
const char* glm_version(void);

/* ---------------------------------------------------------------------------------
 * Quantization (quantlab, include/glmlab/quant.hpp:44-51)
 * ------------------------------------------------------------------------------- */

/* Number of scale groups: rows (kRow), cols (kColumn) or 1 (kWhole) (quant.cpp:38-48). */
int64_t glm_group_count(int64_t rows, int64_t cols, glm_axis axis);
/* Canonical payload size: rows*cols (INT8) or ceil(rows*cols/2) (INT4). */
int64_t glm_payload_bytes(int64_t rows, int64_t cols, int bits);

/* quantize_absmax / quantize_zeropoint (quant.hpp:44-45, quant.cpp:113-186), computed on
 * the GPU in FP64, bit-exact with the reference. Host buffers. `w` is [rows, cols] of
 * `dtype` (F64 or F32 or BF16). zero_points/constant_group are written for
 * GLM_ZEROPOINT only (may be NULL for GLM_ABSMAX). */
glm_status glm_quantize_weight(const void* w, glm_dtype dtype, int64_t rows, int64_t cols,
                               int bits, glm_scheme scheme, glm_axis axis, int8_t* payload,
                               double* scales, double* zero_points, uint8_t* constant_group);
/* Same, all pointers device pointers, stream-ordered. */
glm_status glm_quantize_weight_device(const void* w, glm_dtype dtype, int64_t rows, int64_t cols,
                                      int bits, glm_scheme scheme, glm_axis axis, int8_t* payload,
                                      double* scales, double* zero_points,
                                      uint8_t* constant_group, void* stream);

/* dequantize (quant.hpp:46, quant.cpp:188-221) on the GPU; host buffers; out [rows, cols]. */
glm_status glm_dequantize(const int8_t* payload, int64_t payload_bytes, const double* scales,
                          const double* zero_points, int64_t rows, int64_t cols, int bits,
                          glm_scheme scheme, glm_axis axis, double* out);

/* pack_int4 / unpack_int4 (quant.hpp:50-51, quant.cpp:223-255) on the GPU; host buffers.
 * pack: codes outside [-7, 7] -> GLM_CONTRACT. unpack: packed_bytes != ceil(count/2) ->
 * GLM_FORMAT. */
glm_status glm_pack_int4(const int8_t* codes, int64_t count, int8_t* packed);
glm_status glm_unpack_int4(const int8_t* packed, int64_t packed_bytes, int64_t count,
                           int8_t* codes);

/* ---------------------------------------------------------------------------------
 * Quantized linear: replaces `matmul(x, dequantize(q))` (quant.cpp:188-221 +
 * tensor.cpp:135-155). The handle holds the codes in the B200 device layout
 * plus runtime scales; the canonical payload can be
 * exported back bit-exactly.
 * ------------------------------------------------------------------------------- */
typedef struct glm_qweight glm_qweight;

/* From the canonical reference payload + FP64 scales (host buffers). Absmax only. */
glm_status glm_qweight_create(const int8_t* payload, const double* scales, int64_t rows,
                              int64_t cols, int bits, glm_axis axis, glm_qweight** out);
/* Any scheme: zeropoint weights (quantize_zeropoint, quant.cpp:145-186) run the same
 * kernels with the zero points applied as a rank-1 epilogue term; zero_points may be NULL
 * for GLM_ABSMAX. Constant groups (scale 0) follow quant.cpp:209-216. */
glm_status glm_qweight_create_ex(const int8_t* payload, const double* scales, const double* zero_points,
                                 int64_t rows, int64_t cols, int bits, glm_scheme scheme, glm_axis axis,
                                 glm_qweight** out);
/* Quantize a [rows, cols] weight (host, dtype F64/F32/BF16) straight into a handle. */
glm_status glm_qweight_quantize(const void* w, glm_dtype dtype, int64_t rows, int64_t cols,
                                int bits, glm_axis axis, glm_qweight** out);
/* A [rows, cols] weight of counter-based synthetic values (DESIGN.md "Synthetic weights":
 * seed, tensor_id, std sigma) generated and quantized on the GPU (config-5 sweeps). */
glm_status glm_qweight_synthetic(uint64_t seed, uint32_t tensor_id, int64_t rows, int64_t cols,
                                 float sigma, int bits, glm_axis axis, glm_qweight** out);
glm_status glm_qweight_destroy(glm_qweight* q);
/* Canonical payload + FP64 scales back out of the device layout (host buffers). */
glm_status glm_qweight_export(const glm_qweight* q, int8_t* payload, double* scales);
/* Device layout bytes (for layout tests), size via glm_qweight_device_bytes. */
int64_t glm_qweight_device_bytes(const glm_qweight* q);
glm_status glm_qweight_device_copy(const glm_qweight* q, uint8_t* host_out);

/* Diagnostics: per-stage clock64 stamps [256][8] of CTA 0 of the last quantized-matmul launch
 * made with the environment variable GLM_QMM_TRACE set. */
glm_status glm_debug_qmm_trace(long long* host_out);

/* Diagnostics: the kernel glm_qlinear runs for M rows of q. out[0]: 0 fp16 single-token GEMV,
 * 1 integer-MMA single-token GEMV, 2 integer-MMA multi-token GEMV, 3 fp16 multi-token GEMV,
 * 4 fp16 TMA GEMV, 5 tcgen05 GEMM (prefill), 6 tcgen05 integer multi-token GEMV (opt-in,
 * GLM_GEMV_TC); out[1]: k-splits (the integer multi-token GEMVs 2 and 6
 * quantize activations per (token, k-split) on 64-element chunk boundaries
 * chunk = nch * s / ksplit); out[2]: nch, the 64-element chunks along K. Host only, no launch. */
glm_status glm_debug_gemv_plan(const glm_qweight* q, int64_t M, int32_t* out);
/* The same plan for a [rows, cols] weight of `bits` without a handle (host only, no device
 * needed): out[0..2] as above, out[3] the launch's CTA count. */
glm_status glm_debug_plan_shape(int64_t rows, int64_t cols, int bits, int64_t M, int32_t* out);

/* Diagnostics: device timeline. While a trace runs, thread 0 of every CTA of the decode
 * kernels appends (globaltimer ns, tag << 32 | block << 8 | smid) pairs; stop copies up to
 * `capacity` pairs (2 * capacity uint64) to host_out and returns the count. */
glm_status glm_debug_trace_start(int64_t capacity);
glm_status glm_debug_trace_stop(uint64_t* host_out, int64_t capacity, int64_t* count);

/* y[M, cols] = x[M, rows] . dequantize(q), fp32 in/out, device pointers. M >= 1. */
glm_status glm_qlinear(const glm_qweight* q, const float* x, int64_t M, float* y, void* stream);
/* Same with host buffers (H2D, kernel, D2H inside). */
glm_status glm_qlinear_host(const glm_qweight* q, const float* x, int64_t M, float* y);
/* Time `iters` back-to-back GEMV launches of the kernel glm_qlinear uses at this M on
 * device-resident inputs (CUDA events on the launching stream). Returns mean us/launch.
 * Inputs are larger than L2 when rows*cols*bits/8 > 126 MB; `flush` writes a 256 MB
 * buffer between launches otherwise. */
glm_status glm_qlinear_bench(const glm_qweight* q, int64_t M, int iters, int flush, double* us);

/* ---------------------------------------------------------------------------------
 * GLM model (glmmodel, include/glmlab/model.hpp:15-101)
 * ------------------------------------------------------------------------------- */
typedef struct {
  int num_layers, hidden, num_heads, ffn_hidden, vocab; /* GLMConfig (model.hpp:15-31) */
  double init_method_std, layernorm_eps, deepnorm_alpha; /* 0 -> reference defaults */
} glm_config;

typedef struct {
  int64_t element_count, quant_payload_bytes, scale_bytes, half_baseline_bytes,
      wide_baseline_bytes; /* MemoryAccounting (quant.hpp:80-86) */
  int64_t device_weight_bytes, device_head_bytes, device_kv_bytes; /* B200 layout */
} glm_memory;

typedef struct glm_model glm_model;

/* Allocates a model for `max_batch` concurrent sequences of up to `max_ctx` positions.
 * bits in {4, 8}; axis GLM_AXIS_ROW (reference default) or GLM_AXIS_COLUMN (per output
 * channel). head_bf16 != 0 stores the tied embedding/head in bf16, else fp32.
 * tp_rank/tp_size: Megatron tensor-parallel shard of this process (1 GPU per rank). */
glm_status glm_model_create(const glm_config* cfg, int bits, glm_axis axis, int max_batch,
                            int max_ctx, int head_bf16, int tp_rank, int tp_size,
                            glm_model** out);
glm_status glm_model_destroy(glm_model* m);
/* The effective configuration (ffn_hidden / alpha resolved to the reference defaults). */
glm_status glm_model_get_config(const glm_model* m, glm_config* out);
/* Tensor parallelism (tp_size > 1): rank 0 calls glm_tp_unique_id, shares the 128 bytes
 * with every rank (e.g. over torch.distributed), then each rank calls
 * glm_model_init_comm before loading weights. No-op at tp_size == 1. */
glm_status glm_tp_unique_id(void* out128);
glm_status glm_model_init_comm(glm_model* m, const void* unique_id);
/* Test hook (single GPU): an in-process group of `size` rank-models (tp_rank 0..size-1 of
 * tp_size = size, all on the current device), each driven by its own host thread. Its
 * collectives are stream-ordered sum kernels behind a host barrier; the fused decode
 * allreduce runs its push and sum phases as two launches split by that barrier, so the same
 * sharded model code runs with no kernel waiting on another rank's kernel. Decode then runs
 * without a CUDA graph. Every rank calls glm_model_init_comm_emulated concurrently. */
typedef struct glm_tp_group glm_tp_group;
glm_status glm_tp_emulated_group_create(int size, glm_tp_group** out);
glm_status glm_tp_emulated_group_destroy(glm_tp_group* g);
glm_status glm_model_init_comm_emulated(glm_model* m, glm_tp_group* g);
/* Reference parameters (host doubles, model.hpp:41-65), quantized on the GPU with the
 * model's policy (quantize_model, quant.cpp:284-311). which: 0 qkv [d,3d], 1 out_proj
 * [d,d], 2 ffn_w1 [d,f], 3 ffn_v [d,f], 4 ffn_w2 [f,d], 5 ln1_gain, 6 ln1_bias,
 * 7 ln2_gain, 8 ln2_bias; embedding [vocab, d] via glm_model_set_embedding. */
glm_status glm_model_set_embedding(glm_model* m, const double* embedding);
/* Rows [row0, row0 + nrows) of the embedding (host doubles [nrows, hidden]): streaming loaders. */
glm_status glm_model_set_embedding_rows(glm_model* m, int64_t row0, int64_t nrows, const double* values);
glm_status glm_model_set_tensor(glm_model* m, int layer, int which, const double* values);
/* A quantized linear given as the reference's canonical QuantizedMatrix (quant.hpp:26-42:
 * payload bytes + FP64 scales of the FULL [K, N] matrix, the model's bits/axis, absmax);
 * stored as this rank's shard without re-quantizing. Wrong lengths -> GLM_FORMAT. */
glm_status glm_model_set_quantized(glm_model* m, int layer, int which, const int8_t* payload,
                                   int64_t payload_bytes, const double* scales, int64_t nscales);
/* load_quantized_model (quant.cpp:450-491): a checkpoint directory written by the reference's
 * save_quantized_model (manifest.json + GLMT tensors, tensor_io.cpp:68-179). Every file is
 * validated before device work (GLM_FORMAT on malformed input); absmax checkpoints only. */
glm_status glm_model_load_quantized(const char* dir, int max_batch, int max_ctx, int head_bf16,
                                    int tp_rank, int tp_size, glm_model** out);
/* QuantPolicy::scheme (quant.hpp:53-58) of every linear: GLM_ABSMAX (default) or
 * GLM_ZEROPOINT (quantize_zeropoint, quant.cpp:145-186). Call before any weight is set;
 * glm_model_set_tensor then quantizes with the scheme, glm_model_set_quantized_zp takes the
 * canonical zeropoint matrix (payload, FP64 scales with 0 marking a constant group, FP64 zero
 * points; dequantization quant.cpp:188-221). */
glm_status glm_model_set_scheme(glm_model* m, glm_scheme scheme);
glm_status glm_model_set_quantized_zp(glm_model* m, int layer, int which, const int8_t* payload,
                                      int64_t payload_bytes, const double* scales,
                                      const double* zero_points, int64_t ngroups);
/* FP64 zero points of one quantized linear of this rank's shard (zeropoint models). */
glm_status glm_model_export_zero_points(const glm_model* m, int layer, int which, double* zero_points);
/* Synthetic random-init weights of the configured shape, generated and quantized on the
 * GPU with the counter-based generator of DESIGN.md (same stds as model.cpp:69-104). */
glm_status glm_model_init_synthetic(glm_model* m, uint64_t seed);
/* Canonical payload/scales of one quantized linear of this rank's shard (host). */
glm_status glm_model_export_linear(const glm_model* m, int layer, int which, int8_t* payload,
                                   double* scales);
glm_status glm_model_memory(const glm_model* m, glm_memory* out);

/* Prefill: runs `n` tokens of sequence `seq` (tokens/positions host arrays) through the
 * model, filling its KV cache from slot 0. Visibility is the GLM blank-infilling rule for
 * a [gMASK] sample: key j visible to query i iff j < max(context_length, i + 1)
 * (corruption.cpp:338-367; context_length = n gives a fully bidirectional prefix).
 * logits (host, optional) receives [n, vocab] fp32. */
glm_status glm_model_prefill(glm_model* m, int seq, const int* tokens, const int* positions,
                             int n, int context_length, float* logits);
/* Packed prefill (pack_samples, corruption.cpp:295-334): nseg samples concatenated row-wise
 * (tokens/positions of sample i at rows [sum_{j<i} lengths[j], ...)) run as one batch through
 * the linears; attention is per sample (segment isolation) with its own context length, and
 * sample i fills the KV cache of sequence seqs[i] (distinct) from slot 0. logits (optional)
 * receives [sum(lengths), vocab]. */
glm_status glm_model_prefill_batch(glm_model* m, int nseg, const int* seqs, const int* lengths,
                                   const int* context_lengths, const int* tokens, const int* positions,
                                   float* logits);
/* One decode step for sequences 0..batch-1: token b at position positions[b] attends to
 * its whole cache plus itself (decode rows are causal-suffix rows, corruption.cpp:349-362).
 * next_tokens (host, optional) = greedy argmax; logits (host, optional) [batch, vocab]. */
glm_status glm_model_decode_step(glm_model* m, int batch, const int* tokens,
                                 const int* positions, int* next_tokens, float* logits);
/* One GLM block (model.cpp:198-224: qkv -> attention -> out_proj -> deepnorm_residual,
 * then geglu -> deepnorm_residual; model.hpp:70-80) of `layer` on caller hidden states:
 * x_io [n, hidden] fp32 DEVICE buffer holds the block input and receives its output;
 * positions [n] int32 device (each in 0..max_ctx). The call is ordered after earlier work on
 * `stream` (cudaStream_t, NULL = legacy stream) and later work on `stream` after it.
 *   GLM_BLOCK_PREFILL: the n rows are one sample of sequence `seq`; they fill this layer's KV
 *     cache of `seq` from slot 0; visibility j < max(context_length, i + 1).
 *   GLM_BLOCK_DECODE: n = batch rows; row b appends one token to sequence b's cache of this
 *     layer and attends over it.
 * The block API tracks its own per-layer cache lengths (glm_model_reset clears them); it
 * shares the KV storage with glm_model_prefill / decode_step, so drive a model through one
 * API at a time. Taps (glm_model_enable_taps) record this layer's sublayer outputs. */
typedef enum { GLM_BLOCK_PREFILL = 0, GLM_BLOCK_DECODE = 1 } glm_block_mode;
glm_status glm_block_forward(glm_model* m, int layer, glm_block_mode mode, int seq, float* x_io,
                             const int* positions, int n, int context_length, void* stream);
/* Same with host buffers (positions validated on the host). */
glm_status glm_block_forward_host(glm_model* m, int layer, glm_block_mode mode, int seq, float* x_io,
                                  const int* positions, int n, int context_length);
/* Sequence length currently cached for `seq`. */
int glm_model_cached_length(const glm_model* m, int seq);
glm_status glm_model_reset(glm_model* m);
/* Sublayer taps: when enabled, the last prefill/decode call records per layer
 * the attention output after out_proj and the GeGLU output after W2 (before the DeepNorm
 * residual), [layers, rows, hidden] fp32, rows = n (prefill) or batch (decode). */
glm_status glm_model_enable_taps(glm_model* m, int enable);
glm_status glm_model_get_taps(const glm_model* m, float* attn, float* ffn);
/* PrecisionPolicy (tensor.hpp:18-29) of later prefill / decode / block calls: half_storage != 0 is
 * Storage::kHalfEmulated — the embedding rows, every DeepNorm output, the attention and GeGLU
 * sublayer outputs, and the attention scores divided by softmax_prescale are rounded to binary16
 * where forward() calls storage_round (model.cpp:148, 197, 213-223); 0 is kWide (the default). */
glm_status glm_model_set_precision(glm_model* m, int half_storage, double softmax_prescale);
/* Test hook: force every sublayer output to zero (the "echo" chain of SURVEY §8c). */
glm_status glm_model_zero_sublayers(glm_model* m, int enable);

/* ---------------------------------------------------------------------------------
 * Op-level block functions (model.hpp:70-80), fp32 in / out. The model's prefill / decode
 * paths use fused kernels; these run the same arithmetic one op at a time.
 * ------------------------------------------------------------------------------- */
/* deepnorm_residual (model.cpp:125-131): out = LayerNorm(alpha * x + y) * gain + bias with
 * the biased variance and eps (tensor.cpp:256-274); x, y, out [rows, d] (out may alias x),
 * gain / bias [d]; d even. Device pointers, stream-ordered. */
glm_status glm_deepnorm_residual(const float* x, const float* y, int64_t rows, int64_t d, double alpha,
                                 const float* gain, const float* bias, double eps, float* out,
                                 void* stream);
glm_status glm_deepnorm_residual_host(const float* x, const float* y, int64_t rows, int64_t d,
                                      double alpha, const float* gain, const float* bias, double eps,
                                      float* out);
/* geglu (model.cpp:133-135): y = (GeLU_erf(x.W1) * (x.V)).W2 with quantized W1, V [d, f] and
 * W2 [f, n]; x [M, d], y [M, n]. */
glm_status glm_geglu(const glm_qweight* w1, const glm_qweight* v, const glm_qweight* w2, const float* x,
                     int64_t M, float* y, void* stream);
glm_status glm_geglu_host(const glm_qweight* w1, const glm_qweight* v, const glm_qweight* w2,
                          const float* x, int64_t M, float* y);
/* attention (model.cpp:137-152), one head, default PrecisionPolicy: RoPE(q) RoPE(k)^T /
 * sqrt(dh), entries with mask[i * n + j] == 0 -> -inf, wide softmax, weights . v. q, k, v,
 * out [n, dh]; positions [n]; mask [n, n] (1 = visible). A row with no visible key ->
 * GLM_POLICY (tensor.cpp:231-234). */
glm_status glm_attention(const float* q, const float* k, const float* v, int64_t n, int64_t dh,
                         const int* positions, const uint8_t* mask, float* out, void* stream);
glm_status glm_attention_host(const float* q, const float* k, const float* v, int64_t n, int64_t dh,
                              const int* positions, const uint8_t* mask, float* out);

/* Decode benchmark: `steps` greedy decode steps for `batch` sequences, starting from the
 * current caches, on device-resident state via the captured CUDA graph. Times the steps
 * with CUDA events on the model stream. ms_per_step receives the mean; gemv_us (optional)
 * the mean duration of the W4/W8 GEMV launches measured with events around each. */
glm_status glm_model_bench_decode(glm_model* m, int batch, int steps, int warmup,
                                  double* ms_per_step, double* gemv_ms_per_step,
                                  int* launches_per_step);

#ifdef __cplusplus
}
#endif
#endif /* GLM130B_H_ */
