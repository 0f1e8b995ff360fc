// glm130b.hpp — header-only C++ wrapper over the C ABI (glm130b.h) that restores the
// reference's C++ operator API for the quantized inference path: the names, value
// semantics and exception classes of include/glmlab/quant.hpp:26-91,
// include/glmlab/model.hpp:15-95 and include/glmlab/common.hpp:28-56 (paths relative to
// /root/reference/proj). A reference-shaped caller swaps
//     #include <glmlab/quant.hpp>      ->  #include "glm130b.hpp"
//     glmlab::quantize_absmax(w, 4, GroupAxis::kRow)
//                                      ->  glmlab::b200::quantize_absmax(w.data(), K, N, 4, GroupAxis::kRow)
// (the reference takes an Eigen::Ref<const Mat>; this wrapper takes the same row-major
// doubles as a pointer + shape so it has no Eigen dependency).
//
// The C ABI returns glm_status codes; every wrapper call turns a non-OK status into the
// matching exception, so `CHECK_THROWS_AS(..., ContractError)` cases port one to one.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "glm130b.h"

namespace glmlab {
namespace b200 {

// Error hierarchy of common.hpp:28-56 (+ the two device-side classes with no reference
// equivalent). what() carries the "[module] message" text of glm_last_error().
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractError : Error {
  using Error::Error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct FormatError : Error {
  using Error::Error;
};
struct PolicyError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};
struct NcclError : Error {
  using Error::Error;
};

inline void check(glm_status s) {
  if (s == GLM_OK) return;
  const std::string msg = glm_last_error();
  switch (s) {
    case GLM_CONTRACT: throw ContractError(msg);
    case GLM_DIMENSION: throw DimensionError(msg);
    case GLM_FORMAT: throw FormatError(msg);
    case GLM_POLICY: throw PolicyError(msg);
    case GLM_CUDA: throw CudaError(msg);
    case GLM_NCCL: throw NcclError(msg);
    default: throw Error(msg);
  }
}

using Index = std::int64_t;

enum class QuantScheme { kAbsmax = GLM_ABSMAX, kZeropoint = GLM_ZEROPOINT };       // quant.hpp:13
enum class GroupAxis { kRow = GLM_AXIS_ROW, kColumn = GLM_AXIS_COLUMN, kWhole = GLM_AXIS_WHOLE };  // quant.hpp:14

// QuantizedMatrix (quant.hpp:26-42): owns the canonical payload and FP64 scales.
struct QuantizedMatrix {
  int bits = 8;
  QuantScheme scheme = QuantScheme::kAbsmax;
  GroupAxis axis = GroupAxis::kRow;
  Index rows = 0, cols = 0;
  std::vector<std::int8_t> payload;
  std::vector<double> scales;
  std::vector<double> zero_points;          // kZeropoint only
  std::vector<std::uint8_t> constant_group;  // kZeropoint only
};

inline Index group_count(Index rows, Index cols, GroupAxis axis) {
  return glm_group_count(rows, cols, static_cast<glm_axis>(axis));
}

// quantize_absmax / quantize_zeropoint (quant.hpp:44-45): w is row-major [rows, cols].
inline QuantizedMatrix quantize(const double* w, Index rows, Index cols, int bits, QuantScheme scheme,
                                GroupAxis axis) {
  QuantizedMatrix q;
  q.bits = bits;
  q.scheme = scheme;
  q.axis = axis;
  q.rows = rows;
  q.cols = cols;
  const Index pb = glm_payload_bytes(rows, cols, bits);
  const Index g = group_count(rows, cols, axis);
  q.payload.resize(static_cast<size_t>(pb > 0 ? pb : 0));
  q.scales.resize(static_cast<size_t>(g > 0 ? g : 0));
  if (scheme == QuantScheme::kZeropoint) {
    q.zero_points.resize(q.scales.size());
    q.constant_group.resize(q.scales.size());
  }
  check(glm_quantize_weight(w, GLM_F64, rows, cols, bits, static_cast<glm_scheme>(scheme),
                            static_cast<glm_axis>(axis), q.payload.data(), q.scales.data(),
                            q.zero_points.empty() ? nullptr : q.zero_points.data(),
                            q.constant_group.empty() ? nullptr : q.constant_group.data()));
  return q;
}
inline QuantizedMatrix quantize_absmax(const double* w, Index rows, Index cols, int bits, GroupAxis axis) {
  return quantize(w, rows, cols, bits, QuantScheme::kAbsmax, axis);
}
inline QuantizedMatrix quantize_zeropoint(const double* w, Index rows, Index cols, int bits, GroupAxis axis) {
  return quantize(w, rows, cols, bits, QuantScheme::kZeropoint, axis);
}

// dequantize (quant.hpp:46): row-major [rows, cols] doubles.
inline std::vector<double> dequantize(const QuantizedMatrix& q) {
  std::vector<double> out(static_cast<size_t>(q.rows * q.cols));
  check(glm_dequantize(q.payload.data(), static_cast<Index>(q.payload.size()), q.scales.data(),
                       q.zero_points.empty() ? nullptr : q.zero_points.data(), q.rows, q.cols, q.bits,
                       static_cast<glm_scheme>(q.scheme), static_cast<glm_axis>(q.axis), out.data()));
  return out;
}

// pack_int4 / unpack_int4 (quant.hpp:50-51).
inline std::vector<std::int8_t> pack_int4(const std::vector<std::int8_t>& codes) {
  std::vector<std::int8_t> packed(static_cast<size_t>((codes.size() + 1) / 2));
  check(glm_pack_int4(codes.data(), static_cast<Index>(codes.size()), packed.data()));
  return packed;
}
inline std::vector<std::int8_t> unpack_int4(const std::vector<std::int8_t>& packed, Index count) {
  std::vector<std::int8_t> codes(static_cast<size_t>(count > 0 ? count : 0));
  check(glm_unpack_int4(packed.data(), static_cast<Index>(packed.size()), count, codes.data()));
  return codes;
}

// Quantized linear resident on the GPU: replaces matmul(x, dequantize(q)) (tensor.cpp:135-155).
class QLinear {
 public:
  explicit QLinear(const QuantizedMatrix& q) : rows_(q.rows), cols_(q.cols) {
    glm_qweight* h = nullptr;
    check(glm_qweight_create_ex(q.payload.data(), q.scales.data(),
                                q.zero_points.empty() ? nullptr : q.zero_points.data(), q.rows, q.cols, q.bits,
                                static_cast<glm_scheme>(q.scheme), static_cast<glm_axis>(q.axis), &h));
    h_.reset(h);
  }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  // y[M, cols] = x[M, rows] . dequantize(q); host fp32 buffers.
  std::vector<float> operator()(const std::vector<float>& x, Index M) const {
    if (static_cast<Index>(x.size()) != M * rows_) throw DimensionError("[qlinear] x must be [M, rows]");
    std::vector<float> y(static_cast<size_t>(M * cols_));
    check(glm_qlinear_host(h_.get(), x.data(), M, y.data()));
    return y;
  }
  // Device pointers, stream-ordered (stream = cudaStream_t).
  void run_device(const float* x, Index M, float* y, void* stream) const {
    check(glm_qlinear(h_.get(), x, M, y, stream));
  }
  const glm_qweight* handle() const { return h_.get(); }
  QuantizedMatrix export_canonical(int bits, GroupAxis axis) const {
    QuantizedMatrix q;
    q.bits = bits;
    q.axis = axis;
    q.rows = rows_;
    q.cols = cols_;
    q.payload.resize(static_cast<size_t>(glm_payload_bytes(rows_, cols_, bits)));
    q.scales.resize(static_cast<size_t>(group_count(rows_, cols_, axis)));
    check(glm_qweight_export(h_.get(), q.payload.data(), q.scales.data()));
    return q;
  }

 private:
  struct Del {
    void operator()(glm_qweight* p) const { glm_qweight_destroy(p); }
  };
  Index rows_, cols_;
  std::unique_ptr<glm_qweight, Del> h_;
};

// ---- op-level block functions (model.hpp:70-80), host fp32 rows -------------------------
// deepnorm_residual (model.cpp:125-131): LayerNorm(alpha * x + sublayer_output)
inline std::vector<float> deepnorm_residual(const std::vector<float>& x, const std::vector<float>& sublayer_output,
                                            Index rows, Index d, double alpha, const std::vector<float>& gain,
                                            const std::vector<float>& bias, double eps = 1e-5) {
  if (static_cast<Index>(x.size()) != rows * d || x.size() != sublayer_output.size())
    throw DimensionError("[glmmodel] deepnorm_residual operands must share a shape");
  if (static_cast<Index>(gain.size()) != d || static_cast<Index>(bias.size()) != d)
    throw DimensionError("[tensorcore] layer_norm gain/bias must match last dimension");
  std::vector<float> out(x.size());
  check(glm_deepnorm_residual_host(x.data(), sublayer_output.data(), rows, d, alpha, gain.data(), bias.data(), eps,
                                   out.data()));
  return out;
}

// geglu (model.cpp:133-135): (GeLU(x W1) * x V) W2 with quantized weights
inline std::vector<float> geglu(const std::vector<float>& x, Index M, const QLinear& w1, const QLinear& v,
                                const QLinear& w2) {
  if (static_cast<Index>(x.size()) != M * w1.rows()) throw DimensionError("[glmmodel] geglu x must be [M, d]");
  std::vector<float> y(static_cast<size_t>(M * w2.cols()));
  check(glm_geglu_host(w1.handle(), v.handle(), w2.handle(), x.data(), M, y.data()));
  return y;
}

// attention (model.cpp:137-152): one head; mask row-major [n, n], nonzero = visible
inline std::vector<float> attention(const std::vector<float>& q, const std::vector<float>& k,
                                    const std::vector<float>& v, Index n, Index dh, const std::vector<int>& positions,
                                    const std::vector<std::uint8_t>& mask) {
  if (static_cast<Index>(q.size()) != n * dh || k.size() != q.size() || v.size() != q.size() ||
      static_cast<Index>(positions.size()) != n || static_cast<Index>(mask.size()) != n * n)
    throw DimensionError("[tensorcore] attention operands must be [n, dh] with [n] positions and an [n, n] mask");
  std::vector<float> out(q.size());
  check(glm_attention_host(q.data(), k.data(), v.data(), n, dh, positions.data(), mask.data(), out.data()));
  return out;
}

// GLMConfig (model.hpp:15-31); zeros select the reference defaults.
struct GLMConfig {
  int num_layers = 4, hidden = 512, num_heads = 8, ffn_hidden = 0, vocab = 262;
  double init_method_std = 0, layernorm_eps = 0, deepnorm_alpha = 0;
  glm_config c() const {
    return glm_config{num_layers, hidden, num_heads, ffn_hidden, vocab, init_method_std, layernorm_eps,
                      deepnorm_alpha};
  }
};

// QuantizedModel + forward (quant.hpp:61-77, model.hpp:83-91) as a KV-cached GPU model.
class QuantizedModel {
 public:
  QuantizedModel(const GLMConfig& cfg, int bits, GroupAxis axis, int max_batch, int max_ctx,
                 bool head_bf16 = false, int tp_rank = 0, int tp_size = 1,
                 QuantScheme scheme = QuantScheme::kAbsmax)
      : cfg_(cfg) {
    const glm_config c = cfg.c();
    glm_model* m = nullptr;
    check(glm_model_create(&c, bits, static_cast<glm_axis>(axis), max_batch, max_ctx, head_bf16 ? 1 : 0,
                           tp_rank, tp_size, &m));
    m_.reset(m);
    if (scheme != QuantScheme::kAbsmax) check(glm_model_set_scheme(m, static_cast<glm_scheme>(scheme)));
  }
  // load_quantized_model (quant.cpp:450-491): a checkpoint directory written by the reference
  static QuantizedModel load_quantized(const std::string& dir, int max_batch = 1, int max_ctx = 2048,
                                       bool head_bf16 = false, int tp_rank = 0, int tp_size = 1) {
    glm_model* m = nullptr;
    check(glm_model_load_quantized(dir.c_str(), max_batch, max_ctx, head_bf16 ? 1 : 0, tp_rank, tp_size, &m));
    return QuantizedModel(m);
  }
  // a canonical QuantizedMatrix of linear `which` (0 qkv .. 4 ffn_w2) of `layer`
  void set_quantized(int layer, int which, const QuantizedMatrix& q) {
    if (q.scheme == QuantScheme::kZeropoint) {
      if (q.zero_points.size() != q.scales.size()) throw FormatError("[quantlab] zero point count differs from the scale count");
      check(glm_model_set_quantized_zp(m_.get(), layer, which, q.payload.data(), static_cast<Index>(q.payload.size()),
                                       q.scales.data(), q.zero_points.data(), static_cast<Index>(q.scales.size())));
      return;
    }
    check(glm_model_set_quantized(m_.get(), layer, which, q.payload.data(), static_cast<Index>(q.payload.size()),
                                  q.scales.data(), static_cast<Index>(q.scales.size())));
  }
  glm_model* handle() const { return m_.get(); }
  void set_embedding(const std::vector<double>& e) { check(glm_model_set_embedding(m_.get(), e.data())); }
  // which: 0 qkv, 1 out_proj, 2 ffn_w1, 3 ffn_v, 4 ffn_w2, 5..8 LN gains/biases (model.hpp:41-65).
  void set_tensor(int layer, int which, const std::vector<double>& v) {
    check(glm_model_set_tensor(m_.get(), layer, which, v.data()));
  }
  void init_synthetic(std::uint64_t seed) { check(glm_model_init_synthetic(m_.get(), seed)); }
  glm_memory memory_accounting() const {
    glm_memory out{};
    check(glm_model_memory(m_.get(), &out));
    return out;
  }
  // Prefill of one gMASK sample; returns [n, vocab] logits when want_logits.
  std::vector<float> prefill(int seq, const std::vector<int>& tokens, const std::vector<int>& positions,
                             int context_length, bool want_logits = true) {
    const int n = static_cast<int>(tokens.size());
    if (static_cast<int>(positions.size()) != n) throw DimensionError("[model] tokens/positions length mismatch");
    std::vector<float> logits(want_logits ? static_cast<size_t>(n) * cfg_.vocab : 0);
    check(glm_model_prefill(m_.get(), seq, tokens.data(), positions.data(), n, context_length,
                            want_logits ? logits.data() : nullptr));
    return logits;
  }
  // One greedy decode step for sequences 0..B-1; returns next tokens.
  std::vector<int> decode_step(const std::vector<int>& tokens, const std::vector<int>& positions,
                               std::vector<float>* logits = nullptr) {
    const int B = static_cast<int>(tokens.size());
    std::vector<int> next(static_cast<size_t>(B));
    if (logits) logits->resize(static_cast<size_t>(B) * cfg_.vocab);
    check(glm_model_decode_step(m_.get(), B, tokens.data(), positions.data(), next.data(),
                                logits ? logits->data() : nullptr));
    return next;
  }
  void reset() { check(glm_model_reset(m_.get())); }
  // One GLM block (model.cpp:198-224) of `layer` on host hidden states x [n, hidden], in place.
  void block_forward(int layer, glm_block_mode mode, int seq, std::vector<float>& x, const std::vector<int>& positions,
                     int context_length) {
    const int n = static_cast<int>(positions.size());
    if (static_cast<Index>(x.size()) != static_cast<Index>(n) * cfg_.hidden)
      throw DimensionError("[glmmodel] block input must be [n, hidden]");
    check(glm_block_forward_host(m_.get(), layer, mode, seq, x.data(), positions.data(), n, context_length));
  }
  void enable_taps(bool on) { check(glm_model_enable_taps(m_.get(), on ? 1 : 0)); }
  // PrecisionPolicy (tensor.hpp:18-29): Storage::kHalfEmulated and softmax_prescale
  void set_precision(bool half_storage, double softmax_prescale = 1.0) {
    check(glm_model_set_precision(m_.get(), half_storage ? 1 : 0, softmax_prescale));
  }
  // per-layer sublayer outputs of the last call: [layers, rows, hidden] each
  void taps(int rows, std::vector<float>& attn, std::vector<float>& ffn) const {
    attn.resize(static_cast<size_t>(cfg_.num_layers) * rows * cfg_.hidden);
    ffn.resize(attn.size());
    check(glm_model_get_taps(m_.get(), attn.data(), ffn.data()));
  }

 private:
  explicit QuantizedModel(glm_model* m) : m_(m) {
    glm_config c{};
    check(glm_model_get_config(m, &c));
    cfg_.num_layers = c.num_layers;
    cfg_.hidden = c.hidden;
    cfg_.num_heads = c.num_heads;
    cfg_.ffn_hidden = c.ffn_hidden;
    cfg_.vocab = c.vocab;
    cfg_.init_method_std = c.init_method_std;
    cfg_.layernorm_eps = c.layernorm_eps;
    cfg_.deepnorm_alpha = c.deepnorm_alpha;
  }
  struct Del {
    void operator()(glm_model* p) const { glm_model_destroy(p); }
  };
  GLMConfig cfg_;
  std::unique_ptr<glm_model, Del> m_;
};

}  // namespace b200
}  // namespace glmlab
