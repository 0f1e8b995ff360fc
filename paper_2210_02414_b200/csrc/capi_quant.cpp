#include <cmath>
#include <algorithm>
#include <cstdlib>
// capi_quant.cpp — C ABI for quantization and the quantized linear (include/glm130b.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "device_buffer.h"
#include "kernels.h"

namespace glm {

thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }

// Row count from which the quantized linear runs on the tcgen05 GEMM instead of the
// decode GEMV (GLM_QMM_MIN_M, default 17: the GEMV covers M <= 16).
int qmm_min_rows() {
  static const int v = [] {
    const char* e = std::getenv("GLM_QMM_MIN_M");
    const int x = e ? std::atoi(e) : 17;
    return x < 2 ? 2 : (x > 17 ? 17 : x);
  }();
  return v;
}

bool sync_launch_debug() {
  static const bool on = std::getenv("GLM_SYNC_LAUNCH") != nullptr;
  return on;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GLM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int64_t group_count(int64_t rows, int64_t cols, int axis) {
  return axis == GLM_AXIS_ROW ? rows : axis == GLM_AXIS_COLUMN ? cols : 1;
}
int64_t payload_bytes(int64_t rows, int64_t cols, int bits) {
  return bits == 4 ? (rows * cols + 1) / 2 : rows * cols;
}
size_t dtype_size(glm_dtype d) {
  switch (d) {
    case GLM_F64: return 8;
    case GLM_F32: return 4;
    case GLM_BF16: case GLM_F16: return 2;
  }
  fail(GLM_CONTRACT, "quantlab", "unknown dtype");
}

}  // namespace glm

struct glm_qweight {
  glm::QWeightDev w;
  glm::DeviceBuffer codes, col_scale, row_scale, scales64, zvec, zeta;
  int bits = 8;
  int scheme = GLM_ABSMAX;
};

namespace glm {

// Builds a handle from a canonical payload + FP64 scales already on the device.
std::unique_ptr<glm_qweight> make_qweight(const int8_t* d_payload, const double* d_scales, int64_t rows,
                                          int64_t cols, int bits, int axis, cudaStream_t st) {
  auto q = std::make_unique<glm_qweight>();
  q->bits = bits;
  q->w.L = make_layout(rows, cols, bits);
  q->w.axis = axis;
  q->w.nscales = group_count(rows, cols, axis);
  q->codes.alloc(q->w.L.bytes());
  q->col_scale.alloc(q->w.L.Np * sizeof(float));
  q->row_scale.alloc(q->w.L.Kp * sizeof(float));
  q->scales64.alloc(q->w.nscales * sizeof(double));
  q->w.codes = q->codes.ptr;
  q->w.col_scale = q->col_scale.as<float>();
  q->w.row_scale = q->row_scale.as<float>();
  q->w.scales64 = q->scales64.as<double>();
  CUDA_CHECK(cudaMemcpyAsync(q->w.scales64, d_scales, q->w.nscales * 8, cudaMemcpyDeviceToDevice, st));
  repack_device(d_payload, q->w.L, q->w.codes, st);
  runtime_scales_device(q->w.scales64, q->w.nscales, q->w.L, axis, q->w.col_scale, q->w.row_scale, st);
  return q;
}

void check_policy(int bits, int axis) {
  if (bits != 4 && bits != 8) fail(GLM_CONTRACT, "quantlab", "bit width must be 4 or 8, got " + std::to_string(bits));
  if (axis < 0 || axis > 2) fail(GLM_CONTRACT, "quantlab", "unknown group axis");
}

// y = x . dequantize(q) for any M >= 1 (device pointers): the decode GEMV for M <= 16 rows,
// the tcgen05 GEMM (128-token tiles) above; then the split-K reduce with the group scale.
void validate_absmax_payload(const int8_t* payload, int64_t payload_bytes, int64_t n, int bits) {
  if (bits == 4) {
    for (int64_t i = 0; i < payload_bytes; ++i) {
      const uint8_t b = static_cast<uint8_t>(payload[i]);
      if ((b & 0x0F) == 0x08 || (b & 0xF0) == 0x80) fail(GLM_CONTRACT, "quantlab", "INT4 code -8 outside [-7, 7]");
    }
    if (n % 2 && payload_bytes > 0 && (static_cast<uint8_t>(payload[payload_bytes - 1]) >> 4) != 0)
      fail(GLM_FORMAT, "quantlab", "odd INT4 payload must pad its last nibble with 0");
  } else {
    for (int64_t i = 0; i < payload_bytes; ++i)
      if (payload[i] == -128) fail(GLM_CONTRACT, "quantlab", "INT8 code -128 outside [-127, 127]");
  }
}

const QWeightDev& qweight_dev(const glm_qweight* q) {
  if (!q) fail(GLM_CONTRACT, "qlinear", "null weight handle");
  return q->w;
}

void qlinear_device(const glm_qweight* q, const float* x, int64_t M, float* y, cudaStream_t st) {
  const QWeightDev& w = q->w;
  const bool gemv = M < qmm_min_rows();
  const GemvPlan p = gemv ? plan_gemv(w.L, static_cast<int>(M)) : plan_qmm(w.L, static_cast<int>(M));
  const int64_t rows = gemv ? M : xtile_tokens(static_cast<int>(M));
  DeviceBuffer xb(rows * w.L.Kp * 2), part(static_cast<int64_t>(p.ksplit) * M * w.L.Np * 4);
  CUDA_CHECK(cudaMemsetAsync(xb.ptr, 0, xb.bytes, st));
  DeviceBuffer ztb(w.zvec ? M * 4 : 0);
  const float* zt = nullptr;
  if (w.zvec) {  // zeropoint weights: per-row sums of the activations the MMA sees
    zp_token_sums(x, w.L.K, static_cast<int>(M), w, ztb.as<float>(), st);
    zt = ztb.as<float>();
  }
  if (gemv) {
    xfrag_from_f32(x, w.L.K, static_cast<int>(M), w, xb.as<__half>(), st);
    gemv_launch(w, xb.as<__half>(), static_cast<int>(M), part.as<float>(), p, st);
  } else {
    xtile_from_f32(x, w.L.K, static_cast<int>(M), w, xb.as<__half>(), st);
    if (p.ksplit == 1) {  // the tcgen05 epilogue writes the scaled result directly
      qmm_launch(w, xb.as<__half>(), static_cast<int>(M), part.as<float>(), p, st, y, w.L.N, zt);
      CUDA_CHECK(cudaStreamSynchronize(st));
      return;
    }
    qmm_launch(w, xb.as<__half>(), static_cast<int>(M), part.as<float>(), p, st);
  }
  gemv_reduce(part.as<float>(), p.ksplit, static_cast<int>(M), w, y, w.L.N, st, zt);
  CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace glm

using namespace glm;

extern "C" {

const char* glm_last_error(void) { return g_last_error.c_str(); }
const char* glm_version(void) { return "glm130b-b200 0.1 (sm_100a)"; }

int64_t glm_group_count(int64_t rows, int64_t cols, glm_axis axis) { return group_count(rows, cols, axis); }
int64_t glm_payload_bytes(int64_t rows, int64_t cols, int bits) { return payload_bytes(rows, cols, bits); }

glm_status glm_quantize_weight_device(const void* w, glm_dtype dtype, int64_t rows, int64_t cols, int bits,
                                      glm_scheme scheme, glm_axis axis, int8_t* payload, double* scales,
                                      double* zero_points, uint8_t* constant_group, void* stream) {
  return guarded([&] {
    if (scheme == GLM_ZEROPOINT && !zero_points) fail(GLM_CONTRACT, "quantlab", "zeropoint needs zero_points");
    quantize_device(w, dtype, rows, cols, bits, scheme, axis, payload, scales, zero_points, constant_group,
                    static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_quantize_weight(const void* w, glm_dtype dtype, int64_t rows, int64_t cols, int bits,
                               glm_scheme scheme, glm_axis axis, int8_t* payload, double* scales,
                               double* zero_points, uint8_t* constant_group) {
  return guarded([&] {
    check_policy(bits, axis);
    if (rows < 0 || cols < 0) fail(GLM_DIMENSION, "quantlab", "negative shape");
    const int64_t n = rows * cols, g = group_count(rows, cols, axis), pb = payload_bytes(rows, cols, bits);
    if (n == 0) return;
    cudaStream_t st = nullptr;
    DeviceBuffer dw(n * dtype_size(dtype)), dp(pb), ds(g * 8), dz(g * 8), dc(g);
    CUDA_CHECK(cudaMemcpy(dw.ptr, w, dw.bytes, cudaMemcpyHostToDevice));
    quantize_device(dw.ptr, dtype, rows, cols, bits, scheme, axis, dp.as<int8_t>(), ds.as<double>(),
                    dz.as<double>(), dc.as<uint8_t>(), st);
    CUDA_CHECK(cudaMemcpy(payload, dp.ptr, pb, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(scales, ds.ptr, g * 8, cudaMemcpyDeviceToHost));
    if (scheme == GLM_ZEROPOINT) {
      if (zero_points) CUDA_CHECK(cudaMemcpy(zero_points, dz.ptr, g * 8, cudaMemcpyDeviceToHost));
      if (constant_group) CUDA_CHECK(cudaMemcpy(constant_group, dc.ptr, g, cudaMemcpyDeviceToHost));
    }
  });
}

glm_status glm_dequantize(const int8_t* payload, int64_t pbytes, const double* scales, const double* zero_points,
                          int64_t rows, int64_t cols, int bits, glm_scheme scheme, glm_axis axis, double* out) {
  return guarded([&] {
    // header / payload validation (quant.cpp:189-197)
    if (rows < 0 || cols < 0 || (bits != 4 && bits != 8))
      fail(GLM_FORMAT, "quantlab", "corrupt quantized matrix header");
    const int64_t expected = payload_bytes(rows, cols, bits);
    if (pbytes != expected)
      fail(GLM_FORMAT, "quantlab",
           "payload length " + std::to_string(pbytes) + " does not match " + std::to_string(expected));
    if (scheme == GLM_ZEROPOINT && !zero_points) fail(GLM_FORMAT, "quantlab", "zeropoint payload lacks zero points");
    const int64_t n = rows * cols, g = group_count(rows, cols, axis);
    if (n == 0) return;
    DeviceBuffer dp(pbytes), ds(g * 8), dz(g * 8), dout(n * 8);
    CUDA_CHECK(cudaMemcpy(dp.ptr, payload, pbytes, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(ds.ptr, scales, g * 8, cudaMemcpyHostToDevice));
    if (scheme == GLM_ZEROPOINT) CUDA_CHECK(cudaMemcpy(dz.ptr, zero_points, g * 8, cudaMemcpyHostToDevice));
    dequantize_device(dp.as<int8_t>(), ds.as<double>(), dz.as<double>(), rows, cols, bits, scheme, axis,
                      dout.as<double>(), nullptr);
    CUDA_CHECK(cudaMemcpy(out, dout.ptr, n * 8, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_pack_int4(const int8_t* codes, int64_t count, int8_t* packed) {
  return guarded([&] {
    if (count < 0) fail(GLM_DIMENSION, "quantlab", "negative count");
    if (count == 0) return;
    const int64_t nb = (count + 1) / 2;
    DeviceBuffer dc(count), dp(nb);
    CUDA_CHECK(cudaMemcpy(dc.ptr, codes, count, cudaMemcpyHostToDevice));
    pack_int4_device(dc.as<int8_t>(), count, dp.as<int8_t>(), nullptr);
    CUDA_CHECK(cudaMemcpy(packed, dp.ptr, nb, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_unpack_int4(const int8_t* packed, int64_t packed_bytes, int64_t count, int8_t* codes) {
  return guarded([&] {
    if (count < 0 || packed_bytes != (count + 1) / 2)
      fail(GLM_FORMAT, "quantlab", "packed INT4 length does not match the recorded count");
    if (count == 0) return;
    DeviceBuffer dp(packed_bytes), dc(count);
    CUDA_CHECK(cudaMemcpy(dp.ptr, packed, packed_bytes, cudaMemcpyHostToDevice));
    unpack_int4_device(dp.as<int8_t>(), count, dc.as<int8_t>(), nullptr);
    CUDA_CHECK(cudaMemcpy(codes, dc.ptr, count, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_qweight_create(const int8_t* payload, const double* scales, int64_t rows, int64_t cols, int bits,
                              glm_axis axis, glm_qweight** out) {
  return guarded([&] {
    check_policy(bits, axis);
    if (rows <= 0 || cols <= 0) fail(GLM_DIMENSION, "qlinear", "empty weight");
    const int64_t pb = payload_bytes(rows, cols, bits), g = group_count(rows, cols, axis);
    DeviceBuffer dp(pb), ds(g * 8);
    CUDA_CHECK(cudaMemcpy(dp.ptr, payload, pb, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(ds.ptr, scales, g * 8, cudaMemcpyHostToDevice));
    validate_absmax_payload(payload, pb, rows * cols, bits);
    for (int64_t i = 0; i < g; ++i)
      if (!std::isfinite(scales[i]) || scales[i] < 0.0) fail(GLM_FORMAT, "quantlab", "scales must be finite and >= 0");
    auto q = make_qweight(dp.as<int8_t>(), ds.as<double>(), rows, cols, bits, axis, nullptr);
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = q.release();
  });
}

glm_status glm_qweight_create_ex(const int8_t* payload, const double* scales, const double* zero_points,
                                 int64_t rows, int64_t cols, int bits, glm_scheme scheme, glm_axis axis,
                                 glm_qweight** out) {
  if (scheme == GLM_ABSMAX) return glm_qweight_create(payload, scales, rows, cols, bits, axis, out);
  return guarded([&] {
    check_policy(bits, axis);
    if (scheme != GLM_ZEROPOINT) fail(GLM_CONTRACT, "quantlab", "unknown quantization scheme");
    if (!zero_points) fail(GLM_CONTRACT, "quantlab", "zeropoint weights need their zero points");
    if (rows <= 0 || cols <= 0) fail(GLM_DIMENSION, "qlinear", "empty weight");
    const int64_t pb = payload_bytes(rows, cols, bits), g = group_count(rows, cols, axis);
    // s_eff = s, or 1 for constant groups (s == 0: codes 0, value z; quant.cpp:209-216)
    std::vector<double> seff(g);
    for (int64_t i = 0; i < g; ++i) {
      if (!std::isfinite(scales[i]) || !std::isfinite(zero_points[i])) fail(GLM_FORMAT, "quantlab", "non-finite scale");
      seff[i] = scales[i] == 0.0 ? 1.0 : scales[i];
    }
    DeviceBuffer dp(pb), ds(g * 8);
    CUDA_CHECK(cudaMemcpy(dp.ptr, payload, pb, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(ds.ptr, seff.data(), g * 8, cudaMemcpyHostToDevice));
    auto q = make_qweight(dp.as<int8_t>(), ds.as<double>(), rows, cols, bits, axis, nullptr);
    q->scheme = GLM_ZEROPOINT;
    CUDA_CHECK(cudaMemcpy(q->w.scales64, scales, g * 8, cudaMemcpyHostToDevice));  // export the originals
    const QLayout& L = q->w.L;
    std::vector<float> zvec(L.Np, 0.f), zeta(L.Kp, 0.f);
    double smax = 0.0;
    for (int64_t i = 0; i < g; ++i) smax = std::max(smax, seff[i]);
    for (int64_t n = 0; n < cols; ++n)
      zvec[n] = static_cast<float>(axis == GLM_AXIS_ROW ? smax
                                   : axis == GLM_AXIS_COLUMN ? seff[n] * zero_points[n]
                                                             : seff[0] * zero_points[0]);
    for (int64_t k = 0; k < rows; ++k) zeta[k] = axis == GLM_AXIS_ROW ? static_cast<float>(zero_points[k]) : 1.f;
    q->zvec.alloc(L.Np * 4);
    q->zeta.alloc(L.Kp * 4);
    CUDA_CHECK(cudaMemcpy(q->zvec.ptr, zvec.data(), L.Np * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(q->zeta.ptr, zeta.data(), L.Kp * 4, cudaMemcpyHostToDevice));
    q->w.zvec = q->zvec.as<float>();
    q->w.zeta = q->zeta.as<float>();
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = q.release();
  });
}

glm_status glm_qweight_quantize(const void* w, glm_dtype dtype, int64_t rows, int64_t cols, int bits,
                                glm_axis axis, glm_qweight** out) {
  return guarded([&] {
    check_policy(bits, axis);
    if (rows <= 0 || cols <= 0) fail(GLM_DIMENSION, "qlinear", "empty weight");
    const int64_t n = rows * cols, pb = payload_bytes(rows, cols, bits), g = group_count(rows, cols, axis);
    DeviceBuffer dw(n * dtype_size(dtype)), dp(pb), ds(g * 8);
    CUDA_CHECK(cudaMemcpy(dw.ptr, w, dw.bytes, cudaMemcpyHostToDevice));
    quantize_device(dw.ptr, dtype, rows, cols, bits, GLM_ABSMAX, axis, dp.as<int8_t>(), ds.as<double>(), nullptr,
                    nullptr, nullptr);
    auto q = make_qweight(dp.as<int8_t>(), ds.as<double>(), rows, cols, bits, axis, nullptr);
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = q.release();
  });
}

glm_status glm_qweight_synthetic(uint64_t seed, uint32_t tensor_id, int64_t rows, int64_t cols, float sigma, int bits,
                                 glm_axis axis, glm_qweight** out) {
  return guarded([&] {
    check_policy(bits, axis);
    if (axis == GLM_AXIS_WHOLE) fail(GLM_CONTRACT, "qlinear", "synthetic weights use row or column groups");
    if (rows <= 0 || cols <= 0) fail(GLM_DIMENSION, "qlinear", "empty weight");
    auto q = std::make_unique<glm_qweight>();
    q->bits = bits;
    q->w.L = make_layout(rows, cols, bits);
    q->w.axis = axis;
    q->w.nscales = group_count(rows, cols, axis);
    q->codes.alloc(q->w.L.bytes());
    q->col_scale.alloc(q->w.L.Np * sizeof(float));
    q->row_scale.alloc(q->w.L.Kp * sizeof(float));
    q->scales64.alloc(q->w.nscales * sizeof(double));
    q->w.codes = q->codes.ptr;
    q->w.col_scale = q->col_scale.as<float>();
    q->w.row_scale = q->row_scale.as<float>();
    q->w.scales64 = q->scales64.as<double>();
    ShardSpec identity{cols, cols, 0, 0};
    gen_quantize_device(seed, tensor_id, rows, cols, sigma, sigma, cols, bits, axis, identity, q->w.L, q->w.codes,
                        q->w.scales64, nullptr);
    runtime_scales_device(q->w.scales64, q->w.nscales, q->w.L, axis, q->w.col_scale, q->w.row_scale, nullptr);
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = q.release();
  });
}

glm_status glm_qweight_destroy(glm_qweight* q) {
  return guarded([&] { delete q; });
}

glm_status glm_qweight_export(const glm_qweight* q, int8_t* payload, double* scales) {
  return guarded([&] {
    const int64_t pb = payload_bytes(q->w.L.K, q->w.L.N, q->bits);
    DeviceBuffer dp(pb);
    unrepack_device(q->w.codes, q->w.L, dp.as<int8_t>(), nullptr);
    CUDA_CHECK(cudaMemcpy(payload, dp.ptr, pb, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(scales, q->w.scales64, q->w.nscales * 8, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_debug_qmm_trace(long long* host_out) {
  return guarded([&] {
    if (!qmm_trace_ptr()) fail(GLM_CONTRACT, "qlinear", "no traced launch (set GLM_QMM_TRACE)");
    CUDA_CHECK(cudaMemcpy(host_out, qmm_trace_ptr(), 256 * 8 * sizeof(long long), cudaMemcpyDeviceToHost));
  });
}

static void plan_summary(const QLayout& L, int64_t M, int32_t* out) {
  if (M >= qmm_min_rows()) {
    const GemvPlan p = plan_qmm(L, static_cast<int>(M));
    out[0] = 5;
    out[1] = p.ksplit;
    out[3] = p.grid;
  } else {
    const GemvPlan p = plan_gemv(L, static_cast<int>(M));
    out[0] = gemv_kind(p, L.nch, static_cast<int>(M), L.bits);
    out[1] = p.ksplit;
    out[3] = p.grid;
  }
  out[2] = static_cast<int32_t>(L.nch);
}

glm_status glm_debug_gemv_plan(const glm_qweight* q, int64_t M, int32_t* out) {
  return guarded([&] {
    if (!q || !out) fail(GLM_CONTRACT, "qlinear", "null argument");
    if (M < 1) fail(GLM_DIMENSION, "qlinear", "M must be >= 1");
    int32_t o[4];
    plan_summary(q->w.L, M, o);
    for (int i = 0; i < 3; ++i) out[i] = o[i];
  });
}

glm_status glm_debug_plan_shape(int64_t rows, int64_t cols, int bits, int64_t M, int32_t* out) {
  return guarded([&] {
    if (!out) fail(GLM_CONTRACT, "qlinear", "null argument");
    if (M < 1 || rows < 1 || cols < 1) fail(GLM_DIMENSION, "qlinear", "M, rows and cols must be >= 1");
    if (bits != 4 && bits != 8) fail(GLM_CONTRACT, "quantlab", "bit width must be 4 or 8");
    plan_summary(make_layout(rows, cols, bits), M, out);
  });
}

static unsigned long long* g_trace_dev = nullptr;

glm_status glm_debug_trace_start(int64_t capacity) {
  return guarded([&] {
    if (capacity < 1) fail(GLM_CONTRACT, "trace", "capacity must be positive");
    if (g_trace_dev) cudaFree(g_trace_dev);
    CUDA_CHECK(cudaMalloc(&g_trace_dev, (1 + 2 * capacity) * sizeof(unsigned long long)));
    CUDA_CHECK(cudaMemset(g_trace_dev, 0, (1 + 2 * capacity) * sizeof(unsigned long long)));
    trace_bind_gemv(g_trace_dev, capacity);
    trace_bind_block(g_trace_dev, capacity);
    trace_bind_model(g_trace_dev, capacity);
    trace_bind_gemv_tc(g_trace_dev, capacity);
  });
}

glm_status glm_debug_trace_stop(uint64_t* host_out, int64_t capacity, int64_t* count) {
  return guarded([&] {
    if (!g_trace_dev) fail(GLM_CONTRACT, "trace", "no trace running");
    CUDA_CHECK(cudaDeviceSynchronize());
    unsigned long long n = 0;
    CUDA_CHECK(cudaMemcpy(&n, g_trace_dev, sizeof(n), cudaMemcpyDeviceToHost));
    const int64_t m = std::min<int64_t>(static_cast<int64_t>(n), capacity);
    if (host_out && m > 0)
      CUDA_CHECK(cudaMemcpy(host_out, g_trace_dev + 1, 2 * m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (count) *count = m;
    trace_bind_gemv(nullptr, 0);
    trace_bind_block(nullptr, 0);
    trace_bind_model(nullptr, 0);
    trace_bind_gemv_tc(nullptr, 0);
    cudaFree(g_trace_dev);
    g_trace_dev = nullptr;
  });
}

int64_t glm_qweight_device_bytes(const glm_qweight* q) { return q ? q->w.L.bytes() : 0; }

glm_status glm_qweight_device_copy(const glm_qweight* q, uint8_t* host_out) {
  return guarded([&] { CUDA_CHECK(cudaMemcpy(host_out, q->w.codes, q->w.L.bytes(), cudaMemcpyDeviceToHost)); });
}

glm_status glm_qlinear(const glm_qweight* q, const float* x, int64_t M, float* y, void* stream) {
  return guarded([&] {
    if (M < 1) fail(GLM_DIMENSION, "qlinear", "M must be >= 1");
    qlinear_device(q, x, M, y, static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_qlinear_host(const glm_qweight* q, const float* x, int64_t M, float* y) {
  return guarded([&] {
    if (M < 1) fail(GLM_DIMENSION, "qlinear", "M must be >= 1");
    DeviceBuffer dx(M * q->w.L.K * 4), dy(M * q->w.L.N * 4);
    CUDA_CHECK(cudaMemcpy(dx.ptr, x, dx.bytes, cudaMemcpyHostToDevice));
    qlinear_device(q, dx.as<float>(), M, dy.as<float>(), nullptr);
    CUDA_CHECK(cudaMemcpy(y, dy.ptr, dy.bytes, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_qlinear_bench(const glm_qweight* q, int64_t M, int iters, int flush, double* us) {
  return guarded([&] {
    if (M < 1) fail(GLM_DIMENSION, "qlinear", "M must be >= 1");
    const QWeightDev& w = q->w;
    const bool gemv = M < qmm_min_rows();
    const GemvPlan p = gemv ? plan_gemv(w.L, static_cast<int>(M)) : plan_qmm(w.L, static_cast<int>(M));
    const int64_t rows = gemv ? M : xtile_tokens(static_cast<int>(M));
    DeviceBuffer xb(rows * w.L.Kp * 2), part(static_cast<int64_t>(p.ksplit) * M * w.L.Np * 4);
    DeviceBuffer fl(flush ? (256ll << 20) : 0);
    CUDA_CHECK(cudaMemset(xb.ptr, 0, xb.bytes));
    cudaStream_t st;
    CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto launch = [&] {
      if (gemv) gemv_launch(w, xb.as<__half>(), static_cast<int>(M), part.as<float>(), p, st);
      else qmm_launch(w, xb.as<__half>(), static_cast<int>(M), part.as<float>(), p, st);
    };
    for (int i = 0; i < 3; ++i) launch();
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    double total = 0.0;
    if (!flush) {
      // back-to-back launches, as inside the decode graph: no host gaps in the timed region
      CUDA_CHECK(cudaEventRecord(e0, st));
      for (int i = 0; i < iters; ++i) launch();
      CUDA_CHECK(cudaEventRecord(e1, st));
      CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      total = ms;
    }
    for (int i = 0; flush && i < iters; ++i) {
      CUDA_CHECK(cudaMemsetAsync(fl.ptr, i & 0xFF, fl.bytes, st));
      CUDA_CHECK(cudaEventRecord(e0, st));
      launch();
      CUDA_CHECK(cudaEventRecord(e1, st));
      CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    *us = 1000.0 * total / iters;
  });
}

}  // extern "C"
