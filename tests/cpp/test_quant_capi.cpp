// C++ host-side parity checks through the header-only wrapper (include/glm130b.hpp), written
// the way the reference's doctest units are (test_quant.cpp, test_model.cpp), so a reference
// maintainer can see the drop-in from a C++ caller's side.
//
//   test_quant_capi            full run (needs a B200): KATs + a C++ greedy decode loop
//   test_quant_capi --no-gpu   the failure contract without a GPU: compute calls throw CudaError
//
// Built and run by tests/test_capi.py (CPU) and tests/test_gpu_cpp.py (GPU).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "glm130b.hpp"

using namespace glmlab::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)         \
  do {                                   \
    bool thrown = false;                 \
    try {                                \
      (void)(expr);                      \
    } catch (const T&) {                 \
      thrown = true;                     \
    } catch (...) {                      \
    }                                    \
    CHECK(thrown && #T);                 \
  } while (0)

// test_quant.cpp:40-53 — the absmax worked row.
static void absmax_worked_row() {
  const double w[3] = {1.0, -2.0, 0.5};
  QuantizedMatrix q = quantize_absmax(w, 1, 3, 8, GroupAxis::kRow);
  CHECK(q.scales.size() == 1 && std::fabs(q.scales[0] - 2.0 / 127.0) < 1e-15);
  CHECK(q.payload[0] == 64 && q.payload[1] == -127 && q.payload[2] == 32);  // 63.5 -> 64 (RNE)
  const std::vector<double> d = dequantize(q);
  CHECK(std::fabs(d[0] - 1.007874) < 1e-6 && d[1] == -2.0 && std::fabs(d[2] - 0.503937) < 1e-6);
}

// test_quant.cpp:55-75 — zero matrix, on-grid matrix, non-finite and bad bits.
static void absmax_edge_cases() {
  const std::vector<double> z(12, 0.0);
  QuantizedMatrix q = quantize_absmax(z.data(), 3, 4, 4, GroupAxis::kColumn);
  bool zero = true;
  for (double s : q.scales) zero = zero && s == 0.0;
  CHECK(zero && dequantize(q) == z);
  std::vector<double> g(16);
  for (int i = 0; i < 16; ++i) g[i] = 0.03125 * ((i % 15) - 7);
  q = quantize_absmax(g.data(), 4, 4, 4, GroupAxis::kWhole);
  CHECK(q.scales[0] == 0.03125 && dequantize(q) == g);
  std::vector<double> bad = g;
  bad[5] = INFINITY;
  CHECK_THROWS_AS(quantize_absmax(bad.data(), 4, 4, 8, GroupAxis::kRow), ContractError);
  CHECK_THROWS_AS(quantize_absmax(g.data(), 4, 4, 5, GroupAxis::kRow), ContractError);
}

// test_quant.cpp:188-215 — INT4 packing is a bijection on [-7, 7]; +-8 is rejected.
static void int4_packing() {
  for (int a = -7; a <= 7; ++a)
    for (int b = -7; b <= 7; ++b) {
      const std::vector<std::int8_t> c = {static_cast<std::int8_t>(a), static_cast<std::int8_t>(b)};
      CHECK(unpack_int4(pack_int4(c), 2) == c);
    }
  CHECK_THROWS_AS(pack_int4({8}), ContractError);
  CHECK_THROWS_AS(pack_int4({-8}), ContractError);
  CHECK_THROWS_AS(unpack_int4({1, 2, 3}, 2), FormatError);
}

// Round trip bound |deq - w| <= s/2 and the quantized linear against x . dequantize(q).
static void qlinear_matches_dequantized_product() {
  const int K = 192, N = 80, M = 3;
  std::vector<double> w(K * N);
  unsigned s = 12345;
  auto rnd = [&] {
    s = s * 1664525u + 1013904223u;
    return ((s >> 8) & 0xFFFF) / 32768.0 - 1.0;
  };
  for (auto& v : w) v = 0.02 * rnd();
  for (int bits : {4, 8})
    for (GroupAxis ax : {GroupAxis::kRow, GroupAxis::kColumn}) {
      QuantizedMatrix q = quantize_absmax(w.data(), K, N, bits, ax);
      const std::vector<double> d = dequantize(q);
      bool bound = true;
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) {
          const double sg = q.scales[ax == GroupAxis::kRow ? k : n];
          bound = bound && std::fabs(d[k * N + n] - w[k * N + n]) <= sg / 2 + 1e-12;
        }
      CHECK(bound);
      QLinear lin(q);
      const QuantizedMatrix back = lin.export_canonical(bits, ax);
      CHECK(back.payload == q.payload && back.scales == q.scales);
      std::vector<float> x(M * K);
      for (auto& v : x) v = static_cast<float>(rnd());
      const std::vector<float> y = lin(x, M);
      double err = 0, ref_max = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double r = 0;
          for (int k = 0; k < K; ++k) r += static_cast<double>(x[m * K + k]) * d[k * N + n];
          err = std::fmax(err, std::fabs(r - y[m * N + n]));
          ref_max = std::fmax(ref_max, std::fabs(r));
        }
      CHECK(err <= 5e-3 * ref_max);
      CHECK_THROWS_AS(lin(x, M + 1), DimensionError);
    }
}

// A host decode loop in C++: gMASK prefill + greedy decode, then the KV-cache legality
// property of test_model.cpp:313-343 — the decode step's logits equal the last row of a
// prefill over the extended sequence.
static void cpp_decode_loop() {
  GLMConfig cfg;
  cfg.num_layers = 2;
  cfg.hidden = 256;
  cfg.num_heads = 2;
  cfg.vocab = 300;
  QuantizedModel model(cfg, 4, GroupAxis::kRow, 1, 64);
  model.init_synthetic(7);
  const int P = 11;
  std::vector<int> tokens, positions;
  for (int i = 0; i < P; ++i) tokens.push_back(6 + (37 * i + 11) % 250), positions.push_back(i);
  tokens.push_back(2), positions.push_back(P);  // [gMASK]
  const int C = P + 1;
  tokens.push_back(3), positions.push_back(P);  // [sop] at the mask position
  model.prefill(0, tokens, positions, C, false);
  std::vector<int> seq = tokens, pos = positions;
  std::vector<int> cur = {tokens.back()}, p = {positions.back()};
  std::vector<float> step_logits;
  for (int j = 1; j <= 4; ++j) {
    // teacher-forced varied inputs (greedy on random init is an echo)
    cur = {10 + 17 * j};
    p = {P + j};  // any positions work for this self-consistency property
    seq.push_back(cur[0]);
    pos.push_back(p[0]);
    std::vector<int> next = model.decode_step(cur, p, &step_logits);
    CHECK(next[0] >= 0 && next[0] < cfg.vocab);
  }
  model.reset();
  const std::vector<float> full = model.prefill(0, seq, pos, C, true);
  const float* last = full.data() + (seq.size() - 1) * static_cast<size_t>(cfg.vocab);
  double err = 0, mx = 0;
  for (int v = 0; v < cfg.vocab; ++v) {
    err = std::fmax(err, std::fabs(static_cast<double>(last[v]) - step_logits[v]));
    mx = std::fmax(mx, std::fabs(static_cast<double>(last[v])));
  }
  CHECK(err <= 1e-2 * mx);
  std::printf("cpp decode loop: decode vs prefill max|d| %.3g (max|logit| %.3g)\n", err, mx);
}

static void no_gpu_contract() {
  const double w[4] = {1, 2, 3, 4};
  CHECK_THROWS_AS(quantize_absmax(w, 2, 2, 8, GroupAxis::kRow), CudaError);
  CHECK_THROWS_AS(QuantizedModel(GLMConfig{}, 4, GroupAxis::kRow, 1, 16), CudaError);
  CHECK(group_count(3, 5, GroupAxis::kColumn) == 5);
  CHECK(std::string(glm_version()).find("sm_100a") != std::string::npos);
}

// load_quantized_model through the C++ wrapper: a reference-format checkpoint directory
// (written by tests/test_checkpoint.py) serves greedy decode like the constructed model.
static void load_checkpoint(const char* dir) {
  QuantizedModel m = QuantizedModel::load_quantized(dir, 1, 64);
  std::vector<int> toks = {6, 13, 20, 27, 2};
  std::vector<int> pos = {0, 1, 2, 3, 4};
  std::vector<float> logits = m.prefill(0, toks, pos, 5, true);
  CHECK(logits.size() == 5u * 300u);
  std::vector<int> next = m.decode_step({3}, {4});
  CHECK(next[0] >= 0 && next[0] < 300);
}

int main(int argc, char** argv) {
  if (argc > 2 && std::strcmp(argv[1], "--checkpoint") == 0) {
    load_checkpoint(argv[2]);
  } else if (argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0) {
    no_gpu_contract();
  } else {
    absmax_worked_row();
    absmax_edge_cases();
    int4_packing();
    qlinear_matches_dequantized_product();
    cpp_decode_loop();
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
