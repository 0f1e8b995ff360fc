// ref_harness.cpp — C entry points over the REFERENCE's own, unmodified sources
// (/root/reference/proj/src/{tensor,quant,model,corruption,tensor_io}.cpp compiled with the
// Eigen / doctest stand-ins of oracle/ref_shim into oracle/_ref/libglmref.so by
// oracle/build_ref.sh). TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle
// restatement against the reference itself, and by bench.py's CPU baseline / reference arm
// to time the reference's path on the host cores. The product never loads it.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "glmlab/corruption.hpp"
#include "glmlab/model.hpp"
#include "glmlab/quant.hpp"
#include "glmlab/rng.hpp"
#include "glmlab/tensor.hpp"

using namespace glmlab;

extern "C" void or_gen_rows(uint64_t seed, uint32_t tensor_id, int64_t row0, int64_t nrows, int64_t cols,
                            float sigma_lo, float sigma_hi, int64_t split_col, double* out);  // oracle.cpp

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 1;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const PolicyError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

// ---- BLAS-backed product for the stand-in (Eigen's GEMM at tensor.cpp:146) ----------------
using DgemmFn = void (*)(int, int, int, int64_t, int64_t, int64_t, double, const double*, int64_t, const double*,
                         int64_t, double, double*, int64_t);
DgemmFn g_dgemm = nullptr;
void blas_gemm(bool ta, bool tb, Eigen::Index m, Eigen::Index n, Eigen::Index k, double alpha, const double* A,
               Eigen::Index lda, const double* B, Eigen::Index ldb, double beta, double* C, Eigen::Index ldc) {
  constexpr int kRowMajor = 101, kNoTrans = 111, kTrans = 112;
  g_dgemm(kRowMajor, ta ? kTrans : kNoTrans, tb ? kTrans : kNoTrans, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

GLMConfig tiny_cfg(int layers, int hidden, int heads, int vocab) {
  GLMConfig c;
  c.num_layers = layers;
  c.hidden = hidden;
  c.num_heads = heads;
  c.vocab = vocab;
  return c;
}

// A [gMASK] sample as corrupt_gmask lays it out (corruption.cpp:249-293): rows < C are the
// bidirectional context, rows >= C span 0 in order.
CorruptedSample gmask_sample(const int* tokens, const int* positions, int n, int context_length) {
  CorruptedSample s;
  s.kind = SampleKind::kGMask;
  s.input_tokens.assign(tokens, tokens + n);
  s.positions.assign(positions, positions + n);
  s.targets.assign(n, -1);
  s.segment.assign(n, 0);
  s.span_rank = {0};
  s.context_length = context_length;
  for (int i = 0; i < n; ++i) {
    s.span_id.push_back(i < context_length ? -1 : 0);
    s.span_offset.push_back(i < context_length ? -1 : i - context_length);
  }
  return s;
}

uint64_t fnv(const void* p, size_t n, uint64_t h) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// The reference's quantize_absmax + dequantize of a [K, N] matrix, groups split over threads:
// kColumn groups are columns, kRow groups are rows, and quantize_absmax treats every group
// independently (quant.cpp:113-143), so the blocks' codes / scales are the whole matrix's.
Mat quantize_dequantize_parallel(const Mat& w, int bits, GroupAxis axis, int threads) {
  const Index K = w.rows(), N = w.cols();
  Mat out(K, N);
  const Index groups = axis == GroupAxis::kColumn ? N : K;
  const Index per = (groups + threads - 1) / threads;
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    const Index g0 = t * per, g1 = std::min(groups, g0 + per);
    if (g0 >= g1) break;
    ts.emplace_back([&, g0, g1] {
      if (axis == GroupAxis::kColumn) {
        const QuantizedMatrix q = quantize_absmax(w.block(0, g0, K, g1 - g0), bits, axis);
        out.block(0, g0, K, g1 - g0) = dequantize(q);
      } else {
        const QuantizedMatrix q = quantize_absmax(w.block(g0, 0, g1 - g0, N), bits, axis);
        out.block(g0, 0, g1 - g0, N) = dequantize(q);
      }
    });
  }
  for (auto& t : ts) t.join();
  return out;
}

Mat gen_mat(uint64_t seed, uint32_t id, Index rows, Index cols, double lo, double hi, Index split) {
  Mat m(rows, cols);
  or_gen_rows(seed, id, 0, rows, cols, static_cast<float>(lo), static_cast<float>(hi), split, m.data());
  return m;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// dgemm for the stand-in's matrix product from an ILP64 OpenBLAS (numpy's scipy_openblas64_)
int ref_use_blas(const char* path, int threads) {
  return guarded([&] {
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw std::runtime_error(std::string("dlopen: ") + dlerror());
    g_dgemm = reinterpret_cast<DgemmFn>(dlsym(h, "scipy_cblas_dgemm64_"));
    auto set_threads = reinterpret_cast<void (*)(int)>(dlsym(h, "scipy_openblas_set_num_threads64_"));
    if (!g_dgemm) throw std::runtime_error("scipy_cblas_dgemm64_ not found");
    if (set_threads && threads > 0) set_threads(threads);
    Eigen::set_gemm(blas_gemm);
  });
}

// forward(dequantize_model(quantize_model(init_parameters(cfg, Rng(seed)), {bits, absmax, axis})),
// gmask sample) — the reference's quantized forward (test_quant.cpp:250-272); logits [n, vocab].
// bits 0: unquantized forward(init_parameters(...)); half: PrecisionPolicy kHalfEmulated.
int ref_forward(int layers, int hidden, int heads, int vocab, uint64_t seed, int bits, int axis, const int* tokens,
                const int* positions, int n, int context_length, int unidirectional, int half, double prescale,
                double* logits) {
  return guarded([&] {
    GLMConfig cfg = tiny_cfg(layers, hidden, heads, vocab);
    Rng rng(seed);
    ModelParams p = init_parameters(cfg, rng);
    ModelParams q = bits ? dequantize_model(quantize_model(p, QuantPolicy{bits, QuantScheme::kAbsmax,
                                                                          static_cast<GroupAxis>(axis), true}))
                         : p;
    CorruptedSample s = gmask_sample(tokens, positions, n, context_length);
    ForwardOptions opts;
    if (unidirectional) opts.variant_override = AttentionVariant::kUnidirectional;
    if (half) {  // PrecisionPolicy (tensor.hpp:18-29)
      opts.policy.storage = PrecisionPolicy::Storage::kHalfEmulated;
      opts.policy.softmax_prescale = prescale;
    }
    const Tensor out = forward(q, s, opts);
    std::memcpy(logits, out.values().data(), sizeof(double) * static_cast<size_t>(n) * vocab);
  });
}

// FNV-1a-64 of quantize_model's payloads and scales (SURVEY §8c golden hashes)
int ref_quantize_hashes(int layers, int hidden, int heads, int vocab, uint64_t seed, int bits, int axis,
                        uint64_t* payload_hash, uint64_t* scale_hash, int64_t* payload_bytes, int64_t* nscales) {
  return guarded([&] {
    GLMConfig cfg = tiny_cfg(layers, hidden, heads, vocab);
    Rng rng(seed);
    const QuantizedModel qm =
        quantize_model(init_parameters(cfg, rng), QuantPolicy{bits, QuantScheme::kAbsmax, static_cast<GroupAxis>(axis), true});
    uint64_t hp = 1469598103934665603ull, hs = 1469598103934665603ull;
    int64_t pb = 0, ns = 0;
    for (const QuantizedLayer& l : qm.layers)
      for (const QuantizedMatrix* m : {&l.qkv, &l.out_proj, &l.ffn_w1, &l.ffn_v, &l.ffn_w2}) {
        hp = fnv(m->payload.data(), m->payload.size(), hp);
        hs = fnv(m->scales.data(), m->scales.size() * sizeof(double), hs);
        pb += static_cast<int64_t>(m->payload.size());
        ns += static_cast<int64_t>(m->scales.size());
      }
    *payload_hash = hp;
    *scale_hash = hs;
    *payload_bytes = pb;
    *nscales = ns;
  });
}

// CPU baseline on the reference's own ops: one decode token through
// one GLM-130B-shaped layer (hidden 12288, 96 heads, ffn 32768; INT4 / INT8 weights from the
// counter-based generator quantized and dequantized by the reference's quantize_absmax /
// dequantize, as dequantize_model does once per model build). The reference has no KV cache, so
// a token is the layer body of model.cpp:198-224 with the linears applied to the new row only and
// attention() (model.cpp:137-152) over the `ctx` rows of the grown sequence (earlier rows' q / k / v
// precomputed at setup): matmul (tensor.cpp:135-155, Eigen's GEMM -> BLAS dgemm), slice_cols,
// attention per head, concat_cols, deepnorm_residual, geglu. Also times the tied head
// matmul(h, transpose(E)) over a `head_vocab`-row table (0 = skip). Returns seconds per layer-token.
int ref_bench_layer_decode(uint64_t seed, int bits, int axis, int ctx, int warmup, int steps, int threads,
                           int64_t head_vocab, double* seconds_per_step, double* setup_seconds, double* head_seconds) {
  return guarded([&] {
    const double t0 = now();
    const Index d = 12288, H = 96, dh = 128, f = 32768, L = 70;
    const double fac = 1.0 / std::sqrt(2.0 * L);
    auto xav = [](double a, double b) { return std::sqrt(2.0 / (a + b)); };
    const GroupAxis ax = static_cast<GroupAxis>(axis);
    auto lin = [&](uint32_t id, Index K, Index N, double lo, double hi, Index split) {
      Mat w = gen_mat(seed, id, K, N, lo, hi, split);
      return Tensor::from_matrix(quantize_dequantize_parallel(w, bits, ax, threads));
    };
    const Tensor qkv = lin(0, d, 3 * d, 0.0052, xav(d, d) * fac, 2 * d);
    const Tensor out_proj = lin(1, d, d, xav(d, d) * fac, xav(d, d) * fac, d);
    const Tensor w1 = lin(2, d, f, xav(d, f) * fac, xav(d, f) * fac, f);
    const Tensor wv = lin(3, d, f, xav(d, f) * fac, xav(d, f) * fac, f);
    const Tensor w2 = lin(4, f, d, xav(f, d) * fac, xav(f, d) * fac, d);
    const Tensor g1 = Tensor::constant({d}, 1.0), b1 = Tensor::zeros({d}), g2 = Tensor::constant({d}, 1.0),
                 b2 = Tensor::zeros({d});
    const Real alpha = deepnorm_alpha(static_cast<int>(L));
    // the context: ctx - 1 earlier rows of hidden states, their q / k / v computed once
    Mat hx = gen_mat(seed, 0xFFFE0001u, ctx, d, 1.0, 1.0, d);
    const Tensor qkv_ctx = matmul(Tensor::from_matrix(hx.block(0, 0, ctx - 1, d)), qkv);
    std::vector<int> pos(static_cast<size_t>(ctx));
    for (int i = 0; i < ctx; ++i) pos[i] = i;
    BoolMat mask(ctx, ctx);
    for (int i = 0; i < ctx; ++i)
      for (int j = 0; j < ctx; ++j) mask(i, j) = j <= i;  // the new row is the last: causal
    const Tensor x = Tensor::from_matrix(hx.block(ctx - 1, 0, 1, d));
    *setup_seconds = now() - t0;
    double total = 0;
    for (int it = 0; it < warmup + steps; ++it) {
      const double ts = now();
      const Tensor qkv_new = matmul(x, qkv);
      // rows of the grown sequence: [ctx - 1 cached rows ; new row]
      Mat rows(ctx, 3 * d);
      rows.block(0, 0, ctx - 1, 3 * d) = qkv_ctx.matrix();
      rows.block(ctx - 1, 0, 1, 3 * d) = qkv_new.matrix();
      const Tensor seq = Tensor::from_matrix(rows);
      const Tensor q = slice_cols(seq, 0, d), k = slice_cols(seq, d, d), v = slice_cols(seq, 2 * d, d);
      std::vector<Tensor> heads;
      for (Index h = 0; h < H; ++h)
        heads.push_back(attention(slice_cols(q, h * dh, dh), slice_cols(k, h * dh, dh), slice_cols(v, h * dh, dh), pos, mask));
      const Tensor att_last = Tensor::from_matrix(concat_cols(heads).matrix().block(ctx - 1, 0, 1, d));
      const Tensor attn = matmul(att_last, out_proj);
      const Tensor h1 = deepnorm_residual(x, attn, alpha, g1, b1, 1e-5);
      const Tensor ff = geglu(h1, w1, wv, w2);
      const Tensor y = deepnorm_residual(h1, ff, alpha, g2, b2, 1e-5);
      (void)y;
      if (it >= warmup) total += now() - ts;
    }
    *seconds_per_step = total / std::max(steps, 1);
    *head_seconds = 0;
    if (head_vocab > 0) {
      const Tensor table = Tensor::from_matrix(gen_mat(seed, 0xFFFF0000u, head_vocab, d, 0.0052, 0.0052, d));
      const double th = now();
      const Tensor logits = matmul(x, transpose(table));
      *head_seconds = now() - th;
      (void)logits;
    }
  });
}

}  // extern "C"
