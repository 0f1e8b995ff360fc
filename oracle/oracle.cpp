// oracle.cpp — CPU restatement of the glmlab hot path. TEST INFRASTRUCTURE ONLY:
// the B200 product never links or calls this file (see oracle.h header).
//
// Citations are file:line under /root/reference/proj.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct OrError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& module, const std::string& msg) {
  throw OrError{code, "[" + module + "] " + msg};
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return OR_OK;
  } catch (const OrError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return OR_CONTRACT;
  }
}

// ---- rng.hpp:13-63 -------------------------------------------------------------
// splitmix64 finalizer seeding an mt19937_64; normal() builds a fresh
// std::normal_distribution per draw (rng.hpp:30-32), which discards the cached
// second polar value, so the draw sequence differs from a reused distribution.
uint64_t splitmix_mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

struct RefRng {
  std::mt19937_64 eng;
  explicit RefRng(uint64_t seed) : eng(splitmix_mix(seed)) {}
  double normal(double mean, double sd) { return std::normal_distribution<double>(mean, sd)(eng); }
};

// ---- quant.cpp:19-73 -----------------------------------------------------------
int max_code(int bits) { return (1 << (bits - 1)) - 1; }  // quant.cpp:19

void check_bits(int bits) {  // quant.cpp:21-25
  if (bits != 4 && bits != 8)
    fail(OR_CONTRACT, "quantlab", "bit width must be 4 or 8, got " + std::to_string(bits));
}

int8_t round_code(double x, int bits) {  // quant.cpp:27-31 (nearbyint = RNE)
  const double r = std::nearbyint(x);
  const double cap = static_cast<double>(max_code(bits));
  return static_cast<int8_t>(std::clamp(r, -cap, cap));
}

struct GroupView {
  int64_t count, size;
};

GroupView group_view(int64_t rows, int64_t cols, int axis) {  // quant.cpp:38-48
  switch (axis) {
    case OR_AXIS_ROW: return {rows, cols};
    case OR_AXIS_COLUMN: return {cols, rows};
    case OR_AXIS_WHOLE: return {1, rows * cols};
  }
  fail(OR_CONTRACT, "quantlab", "unknown group axis");
}

// flat index of element k of group g (quant.cpp:50-59, :135-137)
inline int64_t group_flat(int axis, int64_t cols, int64_t g, int64_t k) {
  return axis == OR_AXIS_COLUMN ? k * cols + g : axis == OR_AXIS_ROW ? g * cols + k : k;
}

std::vector<int8_t> pack4(const int8_t* codes, int64_t n) {  // quant.cpp:223-240
  for (int64_t i = 0; i < n; ++i)
    if (codes[i] < -7 || codes[i] > 7)
      fail(OR_CONTRACT, "quantlab", "INT4 code " + std::to_string(codes[i]) + " outside [-7, 7]");
  std::vector<int8_t> out(static_cast<size_t>((n + 1) / 2), 0);
  for (int64_t i = 0; i < n; ++i) {
    const uint8_t nib = static_cast<uint8_t>(codes[i]) & 0x0f;
    uint8_t& b = reinterpret_cast<uint8_t&>(out[static_cast<size_t>(i / 2)]);
    b = (i % 2 == 0) ? nib : static_cast<uint8_t>(b | (nib << 4));
  }
  return out;
}

std::vector<int8_t> unpack4(const int8_t* packed, int64_t packed_bytes, int64_t count) {
  // quant.cpp:242-255
  if (count < 0 || packed_bytes != (count + 1) / 2)
    fail(OR_FORMAT, "quantlab", "packed INT4 length does not match the recorded count");
  std::vector<int8_t> codes(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    const uint8_t b = static_cast<uint8_t>(packed[i / 2]);
    int v = (i % 2 == 0) ? (b & 0x0f) : (b >> 4);
    if (v >= 8) v -= 16;
    codes[static_cast<size_t>(i)] = static_cast<int8_t>(v);
  }
  return codes;
}

struct QMat {
  int bits = 8, scheme = OR_ABSMAX, axis = OR_AXIS_ROW;
  int64_t rows = 0, cols = 0;
  std::vector<int8_t> payload;
  std::vector<double> scales, zero_points;
  std::vector<uint8_t> constant_group;
};

void check_finite(const double* w, int64_t n) {  // quant.cpp:61-65
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(w[i])) fail(OR_CONTRACT, "quantlab", "quantization requires finite inputs");
}

QMat quantize_absmax(const double* w, int64_t rows, int64_t cols, int bits, int axis) {
  // quant.cpp:113-143
  check_bits(bits);
  check_finite(w, rows * cols);
  QMat q;
  q.bits = bits;
  q.scheme = OR_ABSMAX;
  q.axis = axis;
  q.rows = rows;
  q.cols = cols;
  const GroupView v = group_view(rows, cols, axis);
  const double cap = static_cast<double>(max_code(bits));
  std::vector<int8_t> codes(static_cast<size_t>(rows * cols), 0);
  q.scales.assign(static_cast<size_t>(v.count), 0.0);
  for (int64_t g = 0; g < v.count; ++g) {
    double absmax = 0.0;
    for (int64_t k = 0; k < v.size; ++k)
      absmax = std::max(absmax, std::fabs(w[group_flat(axis, cols, g, k)]));
    const double s = absmax / cap;
    q.scales[static_cast<size_t>(g)] = s;
    if (s == 0.0) continue;
    for (int64_t k = 0; k < v.size; ++k) {
      const int64_t flat = group_flat(axis, cols, g, k);
      codes[static_cast<size_t>(flat)] = round_code(w[flat] / s, bits);
    }
  }
  q.payload = bits == 4 ? pack4(codes.data(), rows * cols) : codes;  // quant.cpp:67-73
  return q;
}

QMat quantize_zeropoint(const double* w, int64_t rows, int64_t cols, int bits, int axis) {
  // quant.cpp:145-186
  check_bits(bits);
  check_finite(w, rows * cols);
  QMat q;
  q.bits = bits;
  q.scheme = OR_ZEROPOINT;
  q.axis = axis;
  q.rows = rows;
  q.cols = cols;
  const GroupView v = group_view(rows, cols, axis);
  std::vector<int8_t> codes(static_cast<size_t>(rows * cols), 0);
  q.scales.assign(static_cast<size_t>(v.count), 0.0);
  q.zero_points.assign(static_cast<size_t>(v.count), 0.0);
  q.constant_group.assign(static_cast<size_t>(v.count), 0);
  for (int64_t g = 0; g < v.count; ++g) {
    double lo = w[group_flat(axis, cols, g, 0)], hi = lo;
    for (int64_t k = 1; k < v.size; ++k) {
      const double x = w[group_flat(axis, cols, g, k)];
      lo = std::min(lo, x);
      hi = std::max(hi, x);
    }
    if (hi == lo) {
      q.zero_points[static_cast<size_t>(g)] = lo;
      q.constant_group[static_cast<size_t>(g)] = 1;
      continue;
    }
    const double s = (hi - lo) / static_cast<double>((1 << bits) - 2);
    const double z = std::nearbyint(lo / s) + static_cast<double>(max_code(bits));
    q.scales[static_cast<size_t>(g)] = s;
    q.zero_points[static_cast<size_t>(g)] = z;
    for (int64_t k = 0; k < v.size; ++k) {
      const int64_t flat = group_flat(axis, cols, g, k);
      codes[static_cast<size_t>(flat)] = round_code(std::nearbyint(w[flat] / s) - z, bits);
    }
  }
  q.payload = bits == 4 ? pack4(codes.data(), rows * cols) : codes;
  return q;
}

std::vector<double> dequantize(const QMat& q) {  // quant.cpp:188-221
  if (q.rows < 0 || q.cols < 0 || (q.bits != 4 && q.bits != 8))
    fail(OR_FORMAT, "quantlab", "corrupt quantized matrix header");
  const int64_t n = q.rows * q.cols;
  const int64_t expected = q.bits == 4 ? (n + 1) / 2 : n;
  if (static_cast<int64_t>(q.payload.size()) != expected)
    fail(OR_FORMAT, "quantlab",
         "payload length " + std::to_string(q.payload.size()) + " does not match " +
             std::to_string(expected));
  const std::vector<int8_t> codes =
      q.bits == 4 ? unpack4(q.payload.data(), static_cast<int64_t>(q.payload.size()), n)
                  : q.payload;
  const GroupView v = group_view(q.rows, q.cols, q.axis);
  std::vector<double> out(static_cast<size_t>(n));
  for (int64_t g = 0; g < v.count; ++g) {
    const double s = q.scales[static_cast<size_t>(g)];
    const double z = q.scheme == OR_ZEROPOINT ? q.zero_points[static_cast<size_t>(g)] : 0.0;
    for (int64_t k = 0; k < v.size; ++k) {
      const int64_t flat = group_flat(q.axis, q.cols, g, k);
      const double code = static_cast<double>(codes[static_cast<size_t>(flat)]);
      double value;
      if (q.scheme == OR_ABSMAX) value = s * code;
      else if (s == 0.0) value = z;
      else value = s * (code + z);
      out[static_cast<size_t>(flat)] = value;
    }
  }
  return out;
}

// ---- tensor.cpp ops --------------------------------------------------------------
// C[m,n] = A[m,k] B[k,n] (tensor.cpp:135-155 computes the same product with Eigen;
// here one fixed i-k-j order, each output row owned by one thread).
void matmul(const double* A, const double* B, double* C, int64_t M, int64_t K, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    double* c = C + i * N;
    std::fill(c, c + N, 0.0);
    for (int64_t k = 0; k < K; ++k) {
      const double a = A[i * K + k];
      const double* b = B + k * N;
      for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
    }
  }
}

void rope(const double* x, int64_t rows, int64_t d, const int* pos, double* out) {
  // tensor.cpp:335-383: adjacent pairs (2j, 2j+1), theta_j = 10000^(-2j/d)
  std::vector<double> th(static_cast<size_t>(d / 2));
  for (int64_t j = 0; j < d / 2; ++j)
    th[static_cast<size_t>(j)] =
        std::pow(10000.0, -2.0 * static_cast<double>(j) / static_cast<double>(d));
  for (int64_t r = 0; r < rows; ++r) {
    const double m = static_cast<double>(pos[r]);
    for (int64_t j = 0; j < d / 2; ++j) {
      const double ang = m * th[static_cast<size_t>(j)];
      const double c = std::cos(ang), s = std::sin(ang);
      const double a = x[r * d + 2 * j], b = x[r * d + 2 * j + 1];
      out[r * d + 2 * j] = c * a - s * b;
      out[r * d + 2 * j + 1] = s * a + c * b;
    }
  }
}

void softmax(const double* x, int64_t rows, int64_t cols, double* out) {
  // tensor.cpp:221-254 with prescale 1 (wide policy)
  for (int64_t r = 0; r < rows; ++r) {
    const double* row = x + r * cols;
    double mx = -std::numeric_limits<double>::infinity();
    for (int64_t c = 0; c < cols; ++c) mx = std::max(mx, row[c]);
    if (mx == -std::numeric_limits<double>::infinity())
      fail(OR_POLICY, "tensorcore",
           "softmax row " + std::to_string(r) + " is entirely -inf; no distribution is defined");
    double total = 0.0;
    for (int64_t c = 0; c < cols; ++c) {
      const double e = std::exp(row[c] - mx);
      out[r * cols + c] = e;
      total += e;
    }
    for (int64_t c = 0; c < cols; ++c) out[r * cols + c] /= total;
  }
}

void layernorm(const double* x, int64_t rows, int64_t cols, const double* gain,
               const double* bias, double eps, double* out) {
  // tensor.cpp:256-274: mean, biased variance, 1/sqrt(var+eps), affine
  for (int64_t r = 0; r < rows; ++r) {
    const double* in = x + r * cols;
    double sum = 0.0;
    for (int64_t c = 0; c < cols; ++c) sum += in[c];
    const double mean = sum / static_cast<double>(cols);
    double sq = 0.0;
    for (int64_t c = 0; c < cols; ++c) sq += (in[c] - mean) * (in[c] - mean);
    const double var = sq / static_cast<double>(cols);
    const double is = 1.0 / std::sqrt(var + eps);
    for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = (in[c] - mean) * is * gain[c] + bias[c];
  }
}

void gelu(const double* x, int64_t n, double* out) {  // tensor.cpp:313-318 (exact erf)
  for (int64_t i = 0; i < n; ++i) out[i] = 0.5 * x[i] * (1.0 + std::erf(x[i] * 0.7071067811865475244));
}

void build_mask(const or_sample* s, uint8_t* mask) {  // corruption.cpp:338-367
  const int n = s->n;
  if (s->unidirectional) {  // model.cpp:156-162
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) mask[i * n + j] = j <= i;
    return;
  }
  for (int i = 0; i < n; ++i) {
    const int seg_i = s->segment[i], span_i = s->span_id[i], off_i = s->span_offset[i];
    for (int j = 0; j < n; ++j) {
      const int seg_j = s->segment[j], span_j = s->span_id[j];
      bool vis;
      if (span_i == -2 || span_j == -2) vis = i == j;
      else if (seg_i != seg_j) vis = false;
      else if (span_i == -1) vis = span_j == -1;
      else if (span_j == -1) vis = true;
      else if (span_i == span_j) vis = s->span_offset[j] <= off_i;
      else vis = s->span_rank[span_j] < s->span_rank[span_i];
      mask[i * n + j] = vis;
    }
  }
}

double half_round(double x) {  // tensor.cpp:97-121
  if (std::isnan(x)) return x;
  const double sign = std::signbit(x) ? -1.0 : 1.0;
  const double a = std::fabs(x);
  if (a == 0.0 || std::isinf(x)) return x;
  if (a >= 65520.0) return sign * std::numeric_limits<double>::infinity();
  if (a <= 0x1p-25) return sign * 0.0;
  double quantum;
  if (a < 0x1p-14) {
    quantum = 0x1p-24;
  } else {
    int e = 0;
    std::frexp(a, &e);
    quantum = std::ldexp(1.0, e - 11);
  }
  return sign * std::nearbyint(a / quantum) * quantum;
}

// half > 0: PrecisionPolicy kHalfEmulated with softmax_prescale `prescale` (tensor.hpp:18-29)
void attention(const double* q, const double* k, const double* v, int64_t n, int64_t dh,
               const int* pos, const uint8_t* mask, double* out, int half = 0, double prescale = 1.0) {
  // model.cpp:137-152: RoPE(q), RoPE(k), scores / (sqrt(dh) * prescale), storage_round,
  // -inf fill, softmax (multiplies the prescale back, tensor.cpp:229), P.V
  std::vector<double> rq(static_cast<size_t>(n * dh)), rk(static_cast<size_t>(n * dh));
  rope(q, n, dh, pos, rq.data());
  rope(k, n, dh, pos, rk.data());
  std::vector<double> sc(static_cast<size_t>(n * n)), p(static_cast<size_t>(n * n));
  const double inv = 1.0 / (std::sqrt(static_cast<double>(dh)) * (half ? prescale : 1.0));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t c = 0; c < dh; ++c) acc += rq[i * dh + c] * rk[j * dh + c];
      double s = acc * inv;
      if (half) s = half_round(s) * prescale;
      sc[i * n + j] = mask[i * n + j] ? s : -std::numeric_limits<double>::infinity();
    }
  softmax(sc.data(), n, n, p.data());
  matmul(p.data(), v, out, n, n, dh);
}

// ---- model.cpp ---------------------------------------------------------------------
int default_ffn(int hidden, int heads) {  // model.cpp:30-37
  if ((8 * hidden) % 3 == 0) return (8 * hidden) / 3;
  const double target = 8.0 * hidden / 3.0;
  const int step = (heads % 2 == 0) ? heads : 2 * heads;
  const int lo = static_cast<int>(std::floor(target / step)) * step;
  const int hi = lo + step;
  return (target - lo <= hi - target && lo > 0) ? lo : hi;
}

double xavier_std(int64_t fan_in, int64_t fan_out) {  // model.cpp:24-26
  return std::sqrt(2.0 / static_cast<double>(fan_in + fan_out));
}

void validate(const or_config& c) {  // model.cpp:45-59
  if (c.num_layers < 1) fail(OR_CONTRACT, "glmmodel", "num_layers must be >= 1");
  if (c.hidden < 1 || c.num_heads < 1 || c.hidden % c.num_heads != 0)
    fail(OR_CONTRACT, "glmmodel", "hidden must be divisible by num_heads");
  if ((c.hidden / c.num_heads) % 2 != 0)
    fail(OR_CONTRACT, "glmmodel", "head dimension must be even for rotary pairs");
  if (c.vocab <= 4) fail(OR_CONTRACT, "glmmodel", "vocabulary must cover the reserved control ids");
}

// ---- counter-based generator ---------------------
// Philox4x32-10 keyed by the seed, counter (flat_lo, flat_hi, tensor_id, 0).
// The 8 16-bit halves are summed (Irwin-Hall, n=8), centred, scaled to unit
// variance and by sigma in float with explicit round-to-nearest, then rounded
// to bf16 (RNE). Only integer ops and single IEEE float multiplies: bit-identical
// to the CUDA generator in paper_2210_02414_b200/csrc/gen.cuh.
inline void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  const uint64_t p = static_cast<uint64_t>(a) * b;
  hi = static_cast<uint32_t>(p >> 32);
  lo = static_cast<uint32_t>(p);
}

void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c[0], hi0, lo0);
    mulhilo(0xCD9E8D57u, c[2], hi1, lo1);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

uint16_t gen_bf16(uint64_t seed, uint32_t tensor_id, uint64_t flat, float sigma) {
  uint32_t c[4] = {static_cast<uint32_t>(flat), static_cast<uint32_t>(flat >> 32), tensor_id, 0u};
  philox(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  int32_t s = 0;
  for (int i = 0; i < 4; ++i) s += static_cast<int32_t>(c[i] & 0xFFFFu) + static_cast<int32_t>(c[i] >> 16);
  volatile float z = static_cast<float>(s - 262140) * 0x1.3988e2p-16f;  // 1/53509.92
  volatile float w = z * sigma;
  return f32_to_bf16_rne(w);
}

double bf16_to_double(uint16_t b) {
  const uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return static_cast<double>(f);
}

}  // namespace

// ---- model parameters ------------------------------------------------------------
struct or_params {
  or_config cfg;
  int64_t d, f;
  std::vector<double> embedding;
  std::vector<std::vector<double>> lin[5];  // [slot][layer]
  std::vector<std::vector<double>> ln1g, ln1b, ln2g, ln2b;
  bool quantized = false;
  std::vector<QMat> q[5];
};

namespace {

or_params* new_params(const or_config* cfg) {
  validate(*cfg);
  auto* p = new or_params();
  p->cfg = *cfg;
  if (p->cfg.ffn_hidden <= 0) p->cfg.ffn_hidden = default_ffn(cfg->hidden, cfg->num_heads);
  if (p->cfg.deepnorm_alpha <= 0.0) p->cfg.deepnorm_alpha = std::sqrt(2.0 * cfg->num_layers);
  if (p->cfg.layernorm_eps <= 0.0) p->cfg.layernorm_eps = 1e-5;
  if (p->cfg.init_method_std <= 0.0) p->cfg.init_method_std = 0.0052;
  p->d = p->cfg.hidden;
  p->f = p->cfg.ffn_hidden;
  const int L = p->cfg.num_layers;
  for (auto& s : p->lin) s.resize(static_cast<size_t>(L));
  p->ln1g.assign(L, std::vector<double>(static_cast<size_t>(p->d), 1.0));
  p->ln2g.assign(L, std::vector<double>(static_cast<size_t>(p->d), 1.0));
  p->ln1b.assign(L, std::vector<double>(static_cast<size_t>(p->d), 0.0));
  p->ln2b.assign(L, std::vector<double>(static_cast<size_t>(p->d), 0.0));
  return p;
}

void shape_of(const or_params* p, int which, int64_t& r, int64_t& c) {
  const int64_t d = p->d, f = p->f;
  switch (which) {
    case OR_QKV: r = d; c = 3 * d; return;
    case OR_OUT: r = d; c = d; return;
    case OR_W1: case OR_V: r = d; c = f; return;
    case OR_W2: r = f; c = d; return;
    case OR_EMBED: r = p->cfg.vocab; c = d; return;
    case 5: case 6: r = 1; c = d; return;  // LN gains (biases are zero at init, model.cpp:92-95)
  }
  fail(OR_CONTRACT, "oracle", "unknown tensor slot");
}

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

void or_rng_normal(uint64_t seed, int64_t n, double mean, double sd, double* out) {
  RefRng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal(mean, sd);
}

int or_default_ffn_hidden(int hidden, int num_heads) { return default_ffn(hidden, num_heads); }
double or_deepnorm_alpha(int num_layers) { return std::sqrt(2.0 * num_layers); }

int64_t or_group_count(int64_t rows, int64_t cols, int axis) {
  return group_view(rows, cols, axis).count;
}

int or_quantize(const double* w, int64_t rows, int64_t cols, int bits, int scheme, int axis,
                int8_t* payload, double* scales, double* zero_points, uint8_t* constant_group) {
  return guarded([&] {
    QMat q = scheme == OR_ABSMAX ? quantize_absmax(w, rows, cols, bits, axis)
                                 : quantize_zeropoint(w, rows, cols, bits, axis);
    std::memcpy(payload, q.payload.data(), q.payload.size());
    std::memcpy(scales, q.scales.data(), q.scales.size() * sizeof(double));
    if (scheme == OR_ZEROPOINT) {
      if (zero_points) std::memcpy(zero_points, q.zero_points.data(), q.zero_points.size() * 8);
      if (constant_group) std::memcpy(constant_group, q.constant_group.data(), q.constant_group.size());
    }
  });
}

int or_dequantize(const int8_t* payload, int64_t payload_bytes, const double* scales,
                  const double* zero_points, int64_t rows, int64_t cols, int bits, int scheme,
                  int axis, double* out) {
  return guarded([&] {
    QMat q;
    q.bits = bits;
    q.scheme = scheme;
    q.axis = axis;
    q.rows = rows;
    q.cols = cols;
    q.payload.assign(payload, payload + payload_bytes);
    const int64_t g = (bits == 4 || bits == 8) ? group_view(rows, cols, axis).count : 0;
    q.scales.assign(scales, scales + g);
    if (scheme == OR_ZEROPOINT) q.zero_points.assign(zero_points, zero_points + g);
    std::vector<double> o = dequantize(q);
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

int or_pack_int4(const int8_t* codes, int64_t n, int8_t* packed) {
  return guarded([&] {
    auto v = pack4(codes, n);
    std::memcpy(packed, v.data(), v.size());
  });
}

int or_unpack_int4(const int8_t* packed, int64_t packed_bytes, int64_t count, int8_t* codes) {
  return guarded([&] {
    auto v = unpack4(packed, packed_bytes, count);
    std::memcpy(codes, v.data(), v.size());
  });
}

or_params* or_params_init_reference(const or_config* cfg, uint64_t seed) {
  // model.cpp:69-104 — draw order: E, then per layer qkv (row-major, std by column
  // block), out_proj, ffn_w1, ffn_v, ffn_w2.
  or_params* p = nullptr;
  int rc = guarded([&] {
    p = new_params(cfg);
    RefRng rng(seed);
    const int64_t d = p->d, f = p->f;
    const double factor = 1.0 / std::sqrt(2.0 * p->cfg.num_layers);
    auto normal_matrix = [&](int64_t r, int64_t c, double sd) {
      std::vector<double> m(static_cast<size_t>(r * c));
      for (auto& x : m) x = rng.normal(0.0, sd);
      return m;
    };
    p->embedding = normal_matrix(p->cfg.vocab, d, p->cfg.init_method_std);
    for (int l = 0; l < p->cfg.num_layers; ++l) {
      const double v_std = xavier_std(d, d) * factor;
      std::vector<double> qkv(static_cast<size_t>(d * 3 * d));
      for (int64_t r = 0; r < d; ++r)
        for (int64_t c = 0; c < 3 * d; ++c)
          qkv[static_cast<size_t>(r * 3 * d + c)] =
              rng.normal(0.0, c < 2 * d ? p->cfg.init_method_std : v_std);
      p->lin[OR_QKV][l] = std::move(qkv);
      p->lin[OR_OUT][l] = normal_matrix(d, d, xavier_std(d, d) * factor);
      p->lin[OR_W1][l] = normal_matrix(d, f, xavier_std(d, f) * factor);
      p->lin[OR_V][l] = normal_matrix(d, f, xavier_std(d, f) * factor);
      p->lin[OR_W2][l] = normal_matrix(f, d, xavier_std(f, d) * factor);
    }
  });
  if (rc != OR_OK) {
    delete p;
    return nullptr;
  }
  return p;
}

uint16_t or_philox_bf16(uint64_t seed, uint32_t tensor_id, uint64_t flat, float sigma) {
  return gen_bf16(seed, tensor_id, flat, sigma);
}
double or_bf16_to_double(uint16_t b) { return bf16_to_double(b); }

void or_gen_matrix(uint64_t seed, uint32_t tensor_id, int64_t rows, int64_t cols, float sigma_lo,
                   float sigma_hi, int64_t split_col, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const uint64_t flat = static_cast<uint64_t>(r * cols + c);
      out[r * cols + c] = bf16_to_double(gen_bf16(seed, tensor_id, flat, c < split_col ? sigma_lo : sigma_hi));
    }
}

void or_gen_rows(uint64_t seed, uint32_t tensor_id, int64_t row0, int64_t nrows, int64_t cols, float sigma_lo,
                 float sigma_hi, int64_t split_col, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const uint64_t flat = static_cast<uint64_t>((row0 + r) * cols + c);
      out[r * cols + c] = bf16_to_double(gen_bf16(seed, tensor_id, flat, c < split_col ? sigma_lo : sigma_hi));
    }
}

int or_dequantize_cols(const int8_t* payload, const double* scales, int64_t rows, int64_t cols, int bits, int axis,
                       const int64_t* sel, int64_t nsel, double* out) {
  // dequantize (quant.cpp:188-221, absmax: W[r][c] = s_g * code, codes unpacked as
  // unpack_int4 does, quant.cpp:242-255) for the selected columns only: out [rows, nsel]
  return guarded([&] {
    check_bits(bits);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t j = 0; j < nsel; ++j) {
        const int64_t c = sel[j];
        if (c < 0 || c >= cols) continue;
        const int64_t flat = r * cols + c;
        int code;
        if (bits == 8) {
          code = payload[flat];
        } else {
          const uint8_t byte = static_cast<uint8_t>(payload[flat / 2]);
          code = (flat % 2 == 0) ? (byte & 0x0f) : (byte >> 4);
          if (code >= 8) code -= 16;
        }
        const double sc = axis == OR_AXIS_ROW ? scales[r] : axis == OR_AXIS_COLUMN ? scales[c] : scales[0];
        out[r * nsel + j] = sc * static_cast<double>(code);
      }
  });
}

or_params* or_params_init_philox(const or_config* cfg, uint64_t seed) {
  // Same stds as model.cpp:69-104, values from the counter-based generator.
  or_params* p = nullptr;
  int rc = guarded([&] {
    p = new_params(cfg);
    const int64_t d = p->d, f = p->f;
    const double factor = 1.0 / std::sqrt(2.0 * p->cfg.num_layers);
    const float s_init = static_cast<float>(p->cfg.init_method_std);
    auto gen = [&](uint32_t id, int64_t r, int64_t c, double sd_lo, double sd_hi, int64_t split) {
      std::vector<double> m(static_cast<size_t>(r * c));
      or_gen_matrix(seed, id, r, c, static_cast<float>(sd_lo), static_cast<float>(sd_hi), split, m.data());
      return m;
    };
    p->embedding = gen(0xFFFF0000u, p->cfg.vocab, d, s_init, s_init, d);
    for (int l = 0; l < p->cfg.num_layers; ++l) {
      const uint32_t base = static_cast<uint32_t>(l) * 8u;
      const double v_std = xavier_std(d, d) * factor;
      p->lin[OR_QKV][l] = gen(base + OR_QKV, d, 3 * d, p->cfg.init_method_std, v_std, 2 * d);
      p->lin[OR_OUT][l] = gen(base + OR_OUT, d, d, xavier_std(d, d) * factor, 0, d);
      p->lin[OR_W1][l] = gen(base + OR_W1, d, f, xavier_std(d, f) * factor, 0, f);
      p->lin[OR_V][l] = gen(base + OR_V, d, f, xavier_std(d, f) * factor, 0, f);
      p->lin[OR_W2][l] = gen(base + OR_W2, f, d, xavier_std(f, d) * factor, 0, d);
    }
  });
  if (rc != OR_OK) {
    delete p;
    return nullptr;
  }
  return p;
}

void or_params_free(or_params* p) { delete p; }

int or_params_shape(const or_params* p, int which, int64_t* rows, int64_t* cols) {
  return guarded([&] { shape_of(p, which, *rows, *cols); });
}

const double* or_params_tensor(const or_params* p, int layer, int which) {
  if (which == OR_EMBED) return p->embedding.data();
  if (which == 5) return p->ln1g[layer].data();
  if (which == 6) return p->ln2g[layer].data();
  return p->lin[which][static_cast<size_t>(layer)].data();
}

int or_params_quantize(or_params* p, int bits, int scheme, int axis) {
  // quantize_model then dequantize_model (quant.cpp:284-342): the five linears of
  // every layer; embedding and LN pass through untouched.
  return guarded([&] {
    check_bits(bits);
    for (int s = 0; s < 5; ++s) {
      p->q[s].resize(static_cast<size_t>(p->cfg.num_layers));
      for (int l = 0; l < p->cfg.num_layers; ++l) {
        int64_t r, c;
        shape_of(p, s, r, c);
        auto& w = p->lin[s][static_cast<size_t>(l)];
        QMat q = scheme == OR_ABSMAX ? quantize_absmax(w.data(), r, c, bits, axis)
                                     : quantize_zeropoint(w.data(), r, c, bits, axis);
        w = dequantize(q);
        p->q[s][static_cast<size_t>(l)] = std::move(q);
      }
    }
    p->quantized = true;
  });
}

int or_params_qpayload(const or_params* p, int layer, int which, const int8_t** payload,
                       int64_t* payload_bytes, const double** scales, int64_t* nscales) {
  return guarded([&] {
    if (!p->quantized) fail(OR_CONTRACT, "oracle", "model is not quantized");
    const QMat& q = p->q[which][static_cast<size_t>(layer)];
    *payload = q.payload.data();
    *payload_bytes = static_cast<int64_t>(q.payload.size());
    *scales = q.scales.data();
    *nscales = static_cast<int64_t>(q.scales.size());
  });
}

int or_forward_policy(const or_params* p, const or_sample* s, int half, double prescale, double* logits,
                      double* attn_taps, double* ffn_taps, int zero_sublayers);

int or_forward(const or_params* p, const or_sample* s, double* logits, double* attn_taps,
               double* ffn_taps, int zero_sublayers) {
  return or_forward_policy(p, s, 0, 1.0, logits, attn_taps, ffn_taps, zero_sublayers);
}

int or_forward_policy(const or_params* p, const or_sample* s, int half, double prescale, double* logits,
                      double* attn_taps, double* ffn_taps, int zero_sublayers) {
  // model.cpp:166-226; half: storage_round points of PrecisionPolicy kHalfEmulated
  // (model.cpp:148, 197, 213-216, 220-223)
  auto sround = [&](std::vector<double>& v) {
    if (half)
      for (double& x : v) x = half_round(x);
  };
  return guarded([&] {
    const or_config& cfg = p->cfg;
    const int64_t n = s->n, d = p->d, f = p->f, dh = d / cfg.num_heads;
    for (int i = 0; i < n; ++i)
      if (s->tokens[i] < 0 || s->tokens[i] >= cfg.vocab)
        fail(OR_CONTRACT, "glmmodel",
             "token id " + std::to_string(s->tokens[i]) + " overflows vocabulary " +
                 std::to_string(cfg.vocab));
    std::vector<uint8_t> mask(static_cast<size_t>(n * n));
    build_mask(s, mask.data());
    const double alpha = cfg.deepnorm_alpha;
    std::vector<double> h(static_cast<size_t>(n * d));
    for (int64_t i = 0; i < n; ++i)  // embedding_rows (tensor.cpp:396-412)
      std::memcpy(&h[i * d], &p->embedding[static_cast<size_t>(s->tokens[i]) * d], d * 8);
    sround(h);
    std::vector<double> qkv(static_cast<size_t>(n * 3 * d)), heads(static_cast<size_t>(n * d)),
        attn(static_cast<size_t>(n * d)), z(static_cast<size_t>(n * d)),
        a(static_cast<size_t>(n * f)), b(static_cast<size_t>(n * f)), ff(static_cast<size_t>(n * d));
    std::vector<double> qh(static_cast<size_t>(n * dh)), kh(qh.size()), vh(qh.size()), oh(qh.size());
    for (int l = 0; l < cfg.num_layers; ++l) {
      matmul(h.data(), p->lin[OR_QKV][l].data(), qkv.data(), n, d, 3 * d);
      for (int hd = 0; hd < cfg.num_heads; ++hd) {  // model.cpp:200-210 column blocks
        for (int64_t i = 0; i < n; ++i)
          for (int64_t c = 0; c < dh; ++c) {
            qh[i * dh + c] = qkv[i * 3 * d + hd * dh + c];
            kh[i * dh + c] = qkv[i * 3 * d + d + hd * dh + c];
            vh[i * dh + c] = qkv[i * 3 * d + 2 * d + hd * dh + c];
          }
        attention(qh.data(), kh.data(), vh.data(), n, dh, s->positions, mask.data(), oh.data(), half, prescale);
        for (int64_t i = 0; i < n; ++i)
          for (int64_t c = 0; c < dh; ++c) heads[i * d + hd * dh + c] = oh[i * dh + c];
      }
      matmul(heads.data(), p->lin[OR_OUT][l].data(), attn.data(), n, d, d);
      if (zero_sublayers) std::fill(attn.begin(), attn.end(), 0.0);
      sround(attn);
      if (attn_taps) std::memcpy(attn_taps + static_cast<int64_t>(l) * n * d, attn.data(), n * d * 8);
      for (int64_t i = 0; i < n * d; ++i) z[i] = alpha * h[i] + attn[i];  // model.cpp:125-131
      layernorm(z.data(), n, d, p->ln1g[l].data(), p->ln1b[l].data(), cfg.layernorm_eps, h.data());
      sround(h);
      // geglu (model.cpp:133-135)
      matmul(h.data(), p->lin[OR_W1][l].data(), a.data(), n, d, f);
      matmul(h.data(), p->lin[OR_V][l].data(), b.data(), n, d, f);
      gelu(a.data(), n * f, a.data());
      for (int64_t i = 0; i < n * f; ++i) a[i] *= b[i];
      matmul(a.data(), p->lin[OR_W2][l].data(), ff.data(), n, f, d);
      if (zero_sublayers) std::fill(ff.begin(), ff.end(), 0.0);
      sround(ff);
      if (ffn_taps) std::memcpy(ffn_taps + static_cast<int64_t>(l) * n * d, ff.data(), n * d * 8);
      for (int64_t i = 0; i < n * d; ++i) z[i] = alpha * h[i] + ff[i];
      layernorm(z.data(), n, d, p->ln2g[l].data(), p->ln2b[l].data(), cfg.layernorm_eps, h.data());
      sround(h);
    }
    // tied head: logits = h . E^T (model.cpp:225)
    const int64_t V = cfg.vocab;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t t = 0; t < V; ++t) {
        double acc = 0.0;
        for (int64_t c = 0; c < d; ++c) acc += h[i * d + c] * p->embedding[t * d + c];
        logits[i * V + t] = acc;
      }
  });
}

void or_rope_rotate(const double* x, int64_t rows, int64_t d, const int* positions, double* out) {
  rope(x, rows, d, positions, out);
}

int or_softmax_rows(const double* x, int64_t rows, int64_t cols, double* out) {
  return guarded([&] { softmax(x, rows, cols, out); });
}

void or_layer_norm(const double* x, int64_t rows, int64_t cols, const double* gain,
                   const double* bias, double eps, double* out) {
  layernorm(x, rows, cols, gain, bias, eps, out);
}

void or_gelu(const double* x, int64_t n, double* out) { gelu(x, n, out); }

int or_attention(const double* q, const double* k, const double* v, int64_t n, int64_t dh,
                 const int* positions, const uint8_t* mask, double* out) {
  return guarded([&] { attention(q, k, v, n, dh, positions, mask, out); });
}

int or_build_mask(const or_sample* s, uint8_t* mask) {
  return guarded([&] { build_mask(s, mask); });
}

double or_half_round(double x) { return half_round(x); }


int or_qlinear_cols(const double* x, int64_t M, int64_t K, int64_t N, const int8_t* payload,
                    const double* scales, int bits, int axis, const int64_t* cols, int64_t ncols,
                    double* y) {
  // y = x . dequantize(q) restricted to the requested output columns: the
  // dequantized value s_g * code is formed exactly as quant.cpp:210-211 does.
  return guarded([&] {
    check_bits(bits);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < ncols; ++j) {
      const int64_t c = cols[j];
      for (int64_t m = 0; m < M; ++m) {
        double acc = 0.0;
        for (int64_t k = 0; k < K; ++k) {
          const int64_t flat = k * N + c;
          int code;
          if (bits == 8) {
            code = payload[flat];
          } else {
            const uint8_t byte = static_cast<uint8_t>(payload[flat / 2]);
            code = (flat % 2 == 0) ? (byte & 0x0f) : (byte >> 4);
            if (code >= 8) code -= 16;
          }
          const double s = axis == OR_AXIS_ROW ? scales[k] : axis == OR_AXIS_COLUMN ? scales[c] : scales[0];
          acc += x[m * K + k] * (s * static_cast<double>(code));
        }
        y[m * ncols + j] = acc;
      }
    }
  });
}

int or_gen_quantize(uint64_t seed, uint32_t tensor_id, int64_t K, int64_t N, float sigma_lo, float sigma_hi,
                    int64_t split_col, int bits, int axis, int8_t* payload, double* scales) {
  // quantize_absmax (quant.cpp:113-143) over generated values, two passes.
  return guarded([&] {
    check_bits(bits);
    if (axis == OR_AXIS_WHOLE) fail(OR_CONTRACT, "oracle", "streaming quantizer covers row/column");
    const double cap = static_cast<double>(max_code(bits));
    auto val = [&](int64_t k, int64_t n) {
      return bf16_to_double(gen_bf16(seed, tensor_id, static_cast<uint64_t>(k * N + n), n < split_col ? sigma_lo : sigma_hi));
    };
    const int64_t groups = axis == OR_AXIS_ROW ? K : N;
    std::vector<double> amax(static_cast<size_t>(groups), 0.0);
    if (axis == OR_AXIS_ROW) {
#pragma omp parallel for schedule(static)
      for (int64_t k = 0; k < K; ++k) {
        double m = 0.0;
        for (int64_t n = 0; n < N; ++n) m = std::max(m, std::fabs(val(k, n)));
        amax[static_cast<size_t>(k)] = m;
      }
    } else {
#pragma omp parallel
      {
        std::vector<double> loc(static_cast<size_t>(N), 0.0);
#pragma omp for schedule(static)
        for (int64_t k = 0; k < K; ++k)
          for (int64_t n = 0; n < N; ++n) loc[static_cast<size_t>(n)] = std::max(loc[static_cast<size_t>(n)], std::fabs(val(k, n)));
#pragma omp critical
        for (int64_t n = 0; n < N; ++n) amax[static_cast<size_t>(n)] = std::max(amax[static_cast<size_t>(n)], loc[static_cast<size_t>(n)]);
      }
    }
    for (int64_t g = 0; g < groups; ++g) scales[g] = amax[static_cast<size_t>(g)] / cap;
    const int64_t nb = bits == 4 ? (K * N + 1) / 2 : K * N;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nb; ++b) {
      auto code = [&](int64_t flat) -> int {
        const int64_t k = flat / N, n = flat % N;
        const double s = scales[axis == OR_AXIS_ROW ? k : n];
        return s == 0.0 ? 0 : round_code(val(k, n) / s, bits);
      };
      if (bits == 8) {
        payload[b] = static_cast<int8_t>(code(b));
      } else {
        const int c0 = code(2 * b), c1 = (2 * b + 1 < K * N) ? code(2 * b + 1) : 0;
        payload[b] = static_cast<int8_t>((c0 & 0xF) | ((c1 & 0xF) << 4));
      }
    }
  });
}

int or_qlinear_full(const double* x, int64_t M, int64_t K, int64_t N, const int8_t* payload,
                    const double* scales, int bits, int axis, double* y) {
  // x . dequantize(q) (quant.cpp:188-221 + tensor.cpp:135-155), W[k][n] = s_g * code formed
  // per element as dequantize does, accumulated k-outer like a row-major GEMM.
  return guarded([&] {
    check_bits(bits);
    const int64_t NB = 2048;
#pragma omp parallel for schedule(dynamic)
    for (int64_t nb = 0; nb < N; nb += NB) {
      const int64_t n1 = std::min(N, nb + NB);
      std::vector<double> acc(static_cast<size_t>((n1 - nb) * M), 0.0);
      for (int64_t k = 0; k < K; ++k) {
        for (int64_t n = nb; n < n1; ++n) {
          const int64_t flat = k * N + n;
          int code;
          if (bits == 8) {
            code = payload[flat];
          } else {
            const uint8_t byte = static_cast<uint8_t>(payload[flat >> 1]);
            code = (flat & 1) ? (byte >> 4) : (byte & 0x0f);
            if (code >= 8) code -= 16;
          }
          const double s = axis == OR_AXIS_ROW ? scales[k] : axis == OR_AXIS_COLUMN ? scales[n] : scales[0];
          const double w = s * static_cast<double>(code);
          for (int64_t m = 0; m < M; ++m) acc[static_cast<size_t>((n - nb) * M + m)] += x[m * K + k] * w;
        }
      }
      for (int64_t n = nb; n < n1; ++n)
        for (int64_t m = 0; m < M; ++m) y[m * N + n] = acc[static_cast<size_t>((n - nb) * M + m)];
    }
  });
}

uint64_t or_fnv1a64(const uint8_t* data, int64_t n, uint64_t h) {
  for (int64_t i = 0; i < n; ++i) h = (h ^ data[i]) * 1099511628211ull;
  return h;
}

}  // extern "C"
