// The GLM block at the C ABI from a C++ caller (include/glm130b.hpp), checked against the CPU
// oracle (oracle/oracle.h, TEST INFRASTRUCTURE linked only into this test binary):
//   * deepnorm_residual / attention / geglu op by op (model.hpp:70-80, model.cpp:125-152)
//   * the layer-by-layer block API (glm_block_forward, model.cpp:198-224) chained over every
//     layer of the tiny config from the embedding rows: each layer's sublayer taps equal the
//     oracle forward's (or_forward taps), prefill rows and teacher-forced decode rows, for an
//     absmax and a zeropoint model (QuantizedModel(..., QuantScheme::kZeropoint))
// Built and run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../../oracle/oracle.h"
#include "glm130b.hpp"

using namespace glmlab::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                 \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(c)) {                                                                  \
      ++g_fail;                                                                  \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                            \
  } while (0)

static double max_abs(const std::vector<double>& v) {
  double m = 0;
  for (double x : v) m = std::fmax(m, std::fabs(x));
  return m;
}
template <typename A, typename B>
static double max_diff(const A& a, const B& b, size_t n, size_t off_a = 0, size_t off_b = 0) {
  double m = 0;
  for (size_t i = 0; i < n; ++i) m = std::fmax(m, std::fabs(static_cast<double>(a[off_a + i]) - static_cast<double>(b[off_b + i])));
  return m;
}

static void deepnorm_op() {
  std::mt19937 gen(3);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (int rows : {3, 40}) {
    const int d = 512;
    const double alpha = 2.8284271247461903;
    std::vector<float> x(rows * d), y(rows * d), g(d), b(d);
    for (auto& v : x) v = nd(gen);
    for (auto& v : y) v = 0.1f * nd(gen);
    for (auto& v : g) v = 1.f + 0.1f * nd(gen);
    for (auto& v : b) v = 0.1f * nd(gen);
    const std::vector<float> out = deepnorm_residual(x, y, rows, d, alpha, g, b);
    std::vector<double> z(rows * d), gd(g.begin(), g.end()), bd(b.begin(), b.end()), ref(rows * d);
    for (int i = 0; i < rows * d; ++i) z[i] = alpha * x[i] + y[i];
    or_layer_norm(z.data(), rows, d, gd.data(), bd.data(), 1e-5, ref.data());
    CHECK(max_diff(out, ref, ref.size()) <= 1e-5 * max_abs(ref));
  }
  bool thrown = false;
  try {
    deepnorm_residual(std::vector<float>(4), std::vector<float>(6), 2, 2, 1.0, {1, 1}, {0, 0});
  } catch (const DimensionError&) {
    thrown = true;
  }
  CHECK(thrown);
}

static void attention_op() {
  const int n = 70, dh = 64, C = 40;
  std::mt19937 gen(5);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> q(n * dh), k(n * dh), v(n * dh);
  for (auto* a : {&q, &k, &v})
    for (auto& x : *a) x = nd(gen);
  std::vector<int> pos(n);
  for (int i = 0; i < n; ++i) pos[i] = i < C ? i : C - 1 + (i - C);
  std::vector<std::uint8_t> mask(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) mask[i * n + j] = j < std::max(C, i + 1);  // gMASK (corruption.cpp:338-367)
  const std::vector<float> out = attention(q, k, v, n, dh, pos, mask);
  std::vector<double> qd(q.begin(), q.end()), kd(k.begin(), k.end()), vd(v.begin(), v.end()), ref(n * dh);
  CHECK(or_attention(qd.data(), kd.data(), vd.data(), n, dh, pos.data(), mask.data(), ref.data()) == 0);
  CHECK(max_diff(out, ref, ref.size()) <= 1e-4 * max_abs(ref));
  mask[5 * n + 0] = 0;  // a row with no visible key: PolicyError (tensor.cpp:231-234)
  for (int j = 0; j < n; ++j) mask[5 * n + j] = 0;
  bool thrown = false;
  try {
    attention(q, k, v, n, dh, pos, mask);
  } catch (const PolicyError&) {
    thrown = true;
  }
  CHECK(thrown);
}

static void geglu_op() {
  const int M = 5, d = 256, f = 680, nout = 256;
  std::mt19937 gen(7);
  std::normal_distribution<double> nd(0.0, 0.02);
  std::vector<double> w1(d * f), wv(d * f), w2(f * nout);
  for (auto* a : {&w1, &wv, &w2})
    for (auto& x : *a) x = nd(gen);
  const QuantizedMatrix q1 = quantize_absmax(w1.data(), d, f, 4, GroupAxis::kColumn);
  const QuantizedMatrix qv = quantize_absmax(wv.data(), d, f, 4, GroupAxis::kColumn);
  const QuantizedMatrix q2 = quantize_absmax(w2.data(), f, nout, 4, GroupAxis::kColumn);
  const QLinear l1(q1), lv(qv), l2(q2);
  std::vector<float> x(M * d);
  std::normal_distribution<float> ndf(0.f, 1.f);
  for (auto& e : x) e = ndf(gen);
  const std::vector<float> y = geglu(x, M, l1, lv, l2);
  // oracle: x . dequantize(q) in double, erf GeLU (tensor.cpp:313-318)
  std::vector<double> d1(d * f), dv(d * f), d2(f * nout);
  CHECK(or_dequantize(q1.payload.data(), q1.payload.size(), q1.scales.data(), nullptr, d, f, 4, OR_ABSMAX, OR_AXIS_COLUMN, d1.data()) == 0);
  CHECK(or_dequantize(qv.payload.data(), qv.payload.size(), qv.scales.data(), nullptr, d, f, 4, OR_ABSMAX, OR_AXIS_COLUMN, dv.data()) == 0);
  CHECK(or_dequantize(q2.payload.data(), q2.payload.size(), q2.scales.data(), nullptr, f, nout, 4, OR_ABSMAX, OR_AXIS_COLUMN, d2.data()) == 0);
  std::vector<double> ref(M * nout, 0.0);
  for (int m = 0; m < M; ++m) {
    std::vector<double> u(f, 0.0), vv(f, 0.0), g(f);
    for (int kk = 0; kk < d; ++kk)
      for (int j = 0; j < f; ++j) {
        u[j] += x[m * d + kk] * d1[kk * f + j];
        vv[j] += x[m * d + kk] * dv[kk * f + j];
      }
    or_gelu(u.data(), f, g.data());
    for (int j = 0; j < f; ++j)
      for (int o = 0; o < nout; ++o) ref[m * nout + o] += g[j] * vv[j] * d2[j * nout + o];
  }
  CHECK(max_diff(y, ref, ref.size()) <= 1e-2 * max_abs(ref));
}

// The block API chained over the layers == the reference forward's per-layer sublayers.
// (scheme: QuantPolicy::scheme of the model and of the oracle's quantize_model)
static void block_chain(QuantScheme scheme) {
  const int L = 4, d = 512, H = 8, V = 262, P = 60, G = 3;
  or_config oc{L, d, H, 0, V, 0.0, 0.0, 0.0};
  or_params* p = or_params_init_reference(&oc, 1234);
  GLMConfig cfg;
  cfg.num_layers = L;
  cfg.hidden = d;
  cfg.num_heads = H;
  cfg.vocab = V;
  QuantizedModel m(cfg, 4, GroupAxis::kColumn, 1, 128, false, 0, 1, scheme);
  int64_t rows = 0, cols = 0;
  or_params_shape(p, OR_EMBED, &rows, &cols);
  const double* E = or_params_tensor(p, 0, OR_EMBED);
  m.set_embedding(std::vector<double>(E, E + rows * cols));
  for (int l = 0; l < L; ++l) {
    for (int w = 0; w < 5; ++w) {
      or_params_shape(p, w, &rows, &cols);
      const double* t = or_params_tensor(p, l, w);
      m.set_tensor(l, w, std::vector<double>(t, t + rows * cols));
    }
    m.set_tensor(l, 5, std::vector<double>(d, 1.0));
    m.set_tensor(l, 6, std::vector<double>(d, 0.0));
    m.set_tensor(l, 7, std::vector<double>(d, 1.0));
    m.set_tensor(l, 8, std::vector<double>(d, 0.0));
  }
  CHECK(or_params_quantize(p, 4, scheme == QuantScheme::kZeropoint ? OR_ZEROPOINT : OR_ABSMAX, OR_AXIS_COLUMN) == 0);
  // gMASK sample (corruption.cpp:249-293): prefix, [gMASK], [sop] + generated tokens
  std::vector<int> toks, pos, span_id, span_off, seg;
  for (int i = 0; i < P; ++i) toks.push_back(6 + (37 * i + 11) % 256), pos.push_back(i), span_id.push_back(-1), span_off.push_back(-1);
  toks.push_back(2), pos.push_back(P), span_id.push_back(-1), span_off.push_back(-1);
  const int gen[G] = {40, 100, 7};
  for (int j = 0; j <= G; ++j)
    toks.push_back(j == 0 ? 3 : gen[j - 1]), pos.push_back(P + std::max(0, j - 1)), span_id.push_back(0), span_off.push_back(j);
  const int n = static_cast<int>(toks.size()), C = P + 1;
  seg.assign(n, 0);
  const int span_rank[1] = {0};
  or_sample s{n, toks.data(), pos.data(), span_id.data(), span_off.data(), seg.data(), span_rank, 1, 0};
  std::vector<double> logits(static_cast<size_t>(n) * V), at(static_cast<size_t>(L) * n * d), ft(at.size());
  CHECK(or_forward(p, &s, logits.data(), at.data(), ft.data(), 0) == 0);

  // prefill rows [0, C) layer by layer from the embedding rows
  std::vector<float> x(static_cast<size_t>(C) * d);
  for (int i = 0; i < C; ++i)
    for (int c = 0; c < d; ++c) x[i * d + c] = static_cast<float>(E[static_cast<int64_t>(toks[i]) * d + c]);
  m.enable_taps(true);
  std::vector<float> ta, tf;
  const std::vector<int> ppos(pos.begin(), pos.begin() + C);
  for (int l = 0; l < L; ++l) {
    m.block_forward(l, GLM_BLOCK_PREFILL, 0, x, ppos, C);
    m.taps(C, ta, tf);
    std::vector<double> ra(at.begin() + static_cast<size_t>(l) * n * d, at.begin() + static_cast<size_t>(l) * n * d + static_cast<size_t>(C) * d);
    std::vector<double> rf(ft.begin() + static_cast<size_t>(l) * n * d, ft.begin() + static_cast<size_t>(l) * n * d + static_cast<size_t>(C) * d);
    const double ea = max_diff(ta, ra, ra.size(), static_cast<size_t>(l) * C * d), ef = max_diff(tf, rf, rf.size(), static_cast<size_t>(l) * C * d);
    std::printf("%s prefill layer %d: attn tap err %.2e (max %.2e), ffn tap err %.2e (max %.2e)\n",
                scheme == QuantScheme::kZeropoint ? "zeropoint" : "absmax", l, ea, max_abs(ra), ef, max_abs(rf));
    CHECK(ea <= 1e-2 * max_abs(ra));
    CHECK(ef <= 1e-2 * max_abs(rf));
  }
  // teacher-forced decode rows C .. n-1, one block call per layer per row
  for (int r = C; r < n; ++r) {
    std::vector<float> xr(d);
    for (int c = 0; c < d; ++c) xr[c] = static_cast<float>(E[static_cast<int64_t>(toks[r]) * d + c]);
    for (int l = 0; l < L; ++l) {
      m.block_forward(l, GLM_BLOCK_DECODE, 0, xr, {pos[r]}, 0);
      m.taps(1, ta, tf);
      const size_t o = (static_cast<size_t>(l) * n + r) * d;
      std::vector<double> ra(at.begin() + o, at.begin() + o + d), rf(ft.begin() + o, ft.begin() + o + d);
      CHECK(max_diff(ta, ra, d, static_cast<size_t>(l) * d) <= 1e-2 * max_abs(ra));
      CHECK(max_diff(tf, rf, d, static_cast<size_t>(l) * d) <= 1e-2 * max_abs(rf));
    }
  }
  or_params_free(p);
}

int main() {
  deepnorm_op();
  attention_op();
  geglu_op();
  block_chain(QuantScheme::kAbsmax);
  block_chain(QuantScheme::kZeropoint);
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
