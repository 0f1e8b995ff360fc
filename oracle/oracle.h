/* oracle.h — CPU restatement of the glmlab reference path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the B200 product in paper_2210_02414_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it. The product never links, loads or calls it.
 *
 * Every function restates the reference algorithm in plain C++ (double, one
 * deterministic summation order) and cites the reference file:line it follows
 * (paths relative to /root/reference/proj). Parity of this restatement is pinned
 * against the reference's own golden values (tests/golden JSON fixtures, produced by the
 * reference's unmodified sources) and, when oracle/_ref is built, against the
 * reference itself.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GLMConfig (include/glmlab/model.hpp:15-31). ffn_hidden 0 -> default_ffn_hidden,
 * deepnorm_alpha 0 -> sqrt(2N). */
typedef struct {
  int num_layers, hidden, num_heads, ffn_hidden, vocab;
  double init_method_std, layernorm_eps, deepnorm_alpha;
} or_config;

/* CorruptedSample fields the forward consumes (include/glmlab/corruption.hpp:66-81). */
typedef struct {
  int n;
  const int* tokens;
  const int* positions;
  const int* span_id;     /* -1 context, -2 padding, else span index */
  const int* span_offset;
  const int* segment;
  const int* span_rank;   /* per span index */
  int num_spans;
  int unidirectional;     /* AttentionVariant::kUnidirectional (model.cpp:156-162) */
} or_sample;

enum { OR_OK = 0, OR_CONTRACT = 1, OR_DIMENSION = 2, OR_FORMAT = 3, OR_POLICY = 4 };
enum { OR_AXIS_ROW = 0, OR_AXIS_COLUMN = 1, OR_AXIS_WHOLE = 2 };
enum { OR_ABSMAX = 0, OR_ZEROPOINT = 1 };
/* tensor slots of one layer (model.hpp:41-49) */
enum { OR_QKV = 0, OR_OUT = 1, OR_W1 = 2, OR_V = 3, OR_W2 = 4, OR_EMBED = 7 };

const char* or_last_error(void);

/* ---- rng.hpp:13-63 ---- */
void or_rng_normal(uint64_t seed, int64_t n, double mean, double stddev, double* out);
int or_default_ffn_hidden(int hidden, int num_heads);  /* model.cpp:30-37 */
double or_deepnorm_alpha(int num_layers);               /* model.cpp:39 */

/* ---- quant.cpp ---- */
int or_quantize(const double* w, int64_t rows, int64_t cols, int bits, int scheme, int axis,
                int8_t* payload, double* scales, double* zero_points, uint8_t* constant_group);
int or_dequantize(const int8_t* payload, int64_t payload_bytes, const double* scales,
                  const double* zero_points, int64_t rows, int64_t cols, int bits, int scheme,
                  int axis, double* out);
int or_pack_int4(const int8_t* codes, int64_t n, int8_t* packed);
int or_unpack_int4(const int8_t* packed, int64_t packed_bytes, int64_t count, int8_t* codes);
int64_t or_group_count(int64_t rows, int64_t cols, int axis);

/* ---- model.cpp: parameters ---- */
typedef struct or_params or_params;
or_params* or_params_init_reference(const or_config* cfg, uint64_t seed);  /* model.cpp:69-104 */
or_params* or_params_init_philox(const or_config* cfg, uint64_t seed);     /* counter-based */
void or_params_free(or_params* p);
int or_params_shape(const or_params* p, int which, int64_t* rows, int64_t* cols);
const double* or_params_tensor(const or_params* p, int layer, int which);
/* quantize_model + dequantize_model (quant.cpp:284-342) in place: every linear is
 * replaced by dequantize(quantize(w)). Payload/scales are kept for export. */
int or_params_quantize(or_params* p, int bits, int scheme, int axis);
int or_params_qpayload(const or_params* p, int layer, int which, const int8_t** payload,
                       int64_t* payload_bytes, const double** scales, int64_t* nscales);

/* ---- model.cpp:166-226 forward ----
 * logits [n, vocab]; taps (optional) attn_taps/ffn_taps [L, n, d] = the sublayer output
 * (after out_proj / after W2) before the DeepNorm residual; zero_sublayers forces those
 * outputs to 0 (the "echo" chain used for the Delta_ref normalisation). */
int or_forward(const or_params* p, const or_sample* s, double* logits, double* attn_taps,
               double* ffn_taps, int zero_sublayers);
/* Same under PrecisionPolicy (tensor.hpp:18-29): half != 0 = kHalfEmulated storage, scores
 * stored as binary16(score / prescale) and multiplied back inside the softmax. */
int or_forward_policy(const or_params* p, const or_sample* s, int half, double prescale, double* logits,
                      double* attn_taps, double* ffn_taps, int zero_sublayers);

/* ---- ops (tensor.cpp) ---- */
void or_rope_rotate(const double* x, int64_t rows, int64_t d, const int* positions, double* out);
int or_softmax_rows(const double* x, int64_t rows, int64_t cols, double* out);
void or_layer_norm(const double* x, int64_t rows, int64_t cols, const double* gain,
                   const double* bias, double eps, double* out);
void or_gelu(const double* x, int64_t n, double* out);
int or_attention(const double* q, const double* k, const double* v, int64_t n, int64_t dh,
                 const int* positions, const uint8_t* mask, double* out);
int or_build_mask(const or_sample* s, uint8_t* mask);
double or_half_round(double x);

/* ---- counter-based weights shared with the GPU generator ---- */
uint16_t or_philox_bf16(uint64_t seed, uint32_t tensor_id, uint64_t flat, float sigma);
double or_bf16_to_double(uint16_t b);
void or_gen_matrix(uint64_t seed, uint32_t tensor_id, int64_t rows, int64_t cols,
                   float sigma_lo, float sigma_hi, int64_t split_col, double* out);
/* rows [row0, row0 + nrows) of or_gen_matrix's matrix (chunked generation of large tables) */
void or_gen_rows(uint64_t seed, uint32_t tensor_id, int64_t row0, int64_t nrows, int64_t cols,
                 float sigma_lo, float sigma_hi, int64_t split_col, double* out);
/* dequantize (quant.cpp:188-221, absmax) restricted to the columns sel[0..nsel): out [rows, nsel] */
int or_dequantize_cols(const int8_t* payload, const double* scales, int64_t rows, int64_t cols, int bits,
                       int axis, const int64_t* sel, int64_t nsel, double* out);
/* quantized-linear oracle: y[M,N] = x[M,K] . dequantize(q) (quant.cpp:188-221 then
 * tensor.cpp:135-155), restricted to output columns cols[0..ncols) */
int or_qlinear_cols(const double* x, int64_t M, int64_t K, int64_t N, const int8_t* payload,
                    const double* scales, int bits, int axis, const int64_t* cols, int64_t ncols,
                    double* y);

/* Streaming generate + quantize_absmax of a counter-based [K, N] matrix (never
 * materialises the doubles): codes/scales identical to or_quantize(or_gen_matrix(...)). */
int or_gen_quantize(uint64_t seed, uint32_t tensor_id, int64_t K, int64_t N, float sigma_lo, float sigma_hi,
                    int64_t split_col, int bits, int axis, int8_t* payload, double* scales);
/* y[M, N] = x[M, K] . dequantize(q) over all columns, k-outer (row-major streaming). */
int or_qlinear_full(const double* x, int64_t M, int64_t K, int64_t N, const int8_t* payload,
                    const double* scales, int bits, int axis, double* y);

/* FNV-1a-64 running hash (SURVEY §8c golden hashes) */
uint64_t or_fnv1a64(const uint8_t* data, int64_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
