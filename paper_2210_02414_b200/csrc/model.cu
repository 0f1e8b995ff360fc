// model.cu — the GLM model runner behind the glm_model_* C ABI.
//
// Follows forward() of model.cpp:166-226 (embedding -> N x {attention + DeepNorm,
// GeGLU + DeepNorm} -> tied head) with the five linears of every layer quantized on the
// GPU exactly as quantize_model does (quant.cpp:284-311), and adds what the reference
// lacks for serving: a KV cache, prefill/decode split and a CUDA-graph decode step.
//
// Megatron tensor parallelism: rank r of t owns heads [r*H/t, (r+1)*H/t)
// (q/k/v column blocks of qkv, rows of out_proj) and ffn columns [r*f/t, ...) (columns of
// ffn_w1/ffn_v, rows of ffn_w2). Quantization runs on the FULL matrix before sharding so
// scale groups that span ranks are identical on every rank. The row-parallel outputs are
// summed across ranks (collective.cu) before the DeepNorm residual.
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "block.h"
#include "collective.h"
#include "common.cuh"
#include "device_buffer.h"
#include "gen.cuh"
#include "kernels.h"

namespace glm {

GLM_TRACE_TU(model)

namespace {

struct Linear {
  QWeightDev w;
  GemvPlan plans[17];  // decode GEMV plan per row count 1..16
  const GemvPlan& plan(int M) const { return plans[M < 1 ? 1 : (M > 16 ? 16 : M)]; }
  int64_t Kfull = 0, Nfull = 0;
  ShardSpec shard{};
  bool loaded = false;
  // zeropoint scheme (quant.cpp:145-186): writable zvec / zeta of w, the local FP64 zero points
  float *zvec = nullptr, *zeta = nullptr;
  double* zps64 = nullptr;
  int role = 0;  // QKV .. W2: index of its zero-point row sums in glm_model::zt_buf
};

struct Layer {
  Linear lin[5];  // qkv, out_proj, ffn_w1, ffn_v, ffn_w2 (model.hpp:41-49)
  float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
};

enum { QKV = 0, OUT = 1, W1 = 2, VV = 3, W2 = 4 };

__global__ void k_fill(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

__global__ void k_f64_to_bf16(const double* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(static_cast<float>(in[i]));
}

__global__ void k_gen_table(uint64_t seed, uint32_t id, int64_t rows, int64_t cols, float sigma, void* out,
                            int bf16) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint16_t b = gen_bf16(seed, id, static_cast<uint64_t>(i), sigma);
    if (bf16) static_cast<uint16_t*>(out)[i] = b;
    else static_cast<float*>(out)[i] = __uint_as_float(static_cast<uint32_t>(b) << 16);
  }
}

// After a decode step: the greedy token becomes the next input, positions advance.
__global__ void k_feed(const int* __restrict__ next, int* __restrict__ tokens, int* __restrict__ positions, int B) {
  pdl_wait();
  pdl_trigger();
  const int b = threadIdx.x;
  if (b < B) {
    tokens[b] = next[b];
    positions[b] += 1;
  }
}

int grid_of(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b < 148 * 16 ? b : 148 * 16));
}

}  // namespace
}  // namespace glm

using namespace glm;

struct glm_model {
  // config (GLMConfig, model.hpp:15-31)
  int L = 0, d = 0, H = 0, dh = 0, f = 0, V = 0;
  double alpha = 0, eps = 1e-5, init_std = 0.0052;
  int bits = 8, axis = 0, max_batch = 1, max_ctx = 1;
  bool head_bf16 = false;
  int scheme = GLM_ABSMAX;  // QuantPolicy::scheme (quant.hpp:53-58) of every linear
  int tp_rank = 0, tp_size = 1;
  int Hl = 0, dl = 0, fl = 0;
  int64_t vocab_offset = 0, vocab_local = 0;

  std::vector<Layer> layers;
  std::vector<DeviceBuffer> pool;
  void* E = nullptr;
  float2* rope = nullptr;
  __half* kv = nullptr;

  // decode state
  int *d_tokens = nullptr, *d_positions = nullptr, *d_len = nullptr, *d_next = nullptr;
  int *h_tokens = nullptr, *h_positions = nullptr, *h_next = nullptr;  // pinned
  int* d_status = nullptr;  // non-finite winning logit (k_argmax_finish)
  int* h_status = nullptr;  // pinned copy
  unsigned long long* d_argmax = nullptr;
  float* attn_part = nullptr;
  int* attn_ctr = nullptr;

  int attn_splits = 1;
  std::vector<int> h_len;

  // row buffers (grown for prefill)
  int64_t rows_cap = 0;
  DeviceBuffer h, h_bf16, xf_qkv, xf_out, xf_w1, xf_v, xf_w2, logits, taps_attn, taps_ffn;
  DeviceBuffer y_qkv, q_rot, attn_out, y_out, y_a, y_b, y_ffn, ar_buf;
  DeviceBuffer partial;
  DeviceBuffer zt_buf;  // zeropoint: [5 roles][rows_cap] zero-point row sums (zp_sums_act)
  int64_t partial_cap = 0;
  int64_t taps_rows = 0;

  bool taps = false, zero_sub = false;
  // PrecisionPolicy (tensor.hpp:18-29): kHalfEmulated storage rounds h, the sublayer outputs and
  // the attention scores (/ prescale) to binary16 at the reference's storage_round points
  bool half_store = false;
  float prescale = 1.f;
  int64_t last_rows = 0;

  cudaStream_t st = nullptr;
  std::map<std::tuple<int, bool, bool, bool>, cudaGraphExec_t> graphs;
  std::unique_ptr<Collective> comm;

  ~glm_model() {
    for (auto& kv_ : graphs) cudaGraphExecDestroy(kv_.second);
    if (h_tokens) cudaFreeHost(h_tokens);
    if (h_positions) cudaFreeHost(h_positions);
    if (h_next) cudaFreeHost(h_next);
    if (h_peer_err) cudaFreeHost(h_peer_err);
    if (h_status) cudaFreeHost(h_status);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (st) cudaStreamDestroy(st);
  }

  template <typename T>
  T* alloc(int64_t count, bool zero = true) {
    pool.emplace_back(count * static_cast<int64_t>(sizeof(T)));
    if (zero && count) CUDA_CHECK(cudaMemsetAsync(pool.back().ptr, 0, pool.back().bytes, st));
    return pool.back().as<T>();
  }


  // ---------------------------------------------------------------------------------
  void setup(const glm_config& c, int bits_, int axis_, int max_batch_, int max_ctx_, bool head_bf16_, int r, int t) {
    if (c.num_layers < 1) fail(GLM_CONTRACT, "glmmodel", "num_layers must be >= 1");
    if (c.hidden < 1 || c.num_heads < 1 || c.hidden % c.num_heads != 0)
      fail(GLM_CONTRACT, "glmmodel", "hidden must be divisible by num_heads");
    if ((c.hidden / c.num_heads) % 2 != 0) fail(GLM_CONTRACT, "glmmodel", "head dimension must be even for rotary pairs");
    if (c.vocab <= 4) fail(GLM_CONTRACT, "glmmodel", "vocabulary must cover the reserved control ids");
    if (bits_ != 4 && bits_ != 8) fail(GLM_CONTRACT, "quantlab", "bit width must be 4 or 8, got " + std::to_string(bits_));
    if (axis_ != GLM_AXIS_ROW && axis_ != GLM_AXIS_COLUMN && axis_ != GLM_AXIS_WHOLE)
      fail(GLM_CONTRACT, "quantlab", "unknown group axis");
    if (max_batch_ < 1 || max_batch_ > 16) fail(GLM_CONTRACT, "glmmodel", "max_batch must be in 1..16");
    if (max_ctx_ < 1) fail(GLM_CONTRACT, "glmmodel", "max_ctx must be >= 1");
    if (t < 1 || r < 0 || r >= t) fail(GLM_CONTRACT, "glmmodel", "bad tensor-parallel rank");
    L = c.num_layers;
    d = c.hidden;
    H = c.num_heads;
    dh = d / H;
    f = c.ffn_hidden > 0 ? c.ffn_hidden : default_ffn(d, H);
    V = c.vocab;
    alpha = c.deepnorm_alpha > 0 ? c.deepnorm_alpha : std::sqrt(2.0 * L);  // model.cpp:39, :65-67
    eps = c.layernorm_eps > 0 ? c.layernorm_eps : 1e-5;
    init_std = c.init_method_std > 0 ? c.init_method_std : 0.0052;
    bits = bits_;
    axis = axis_;
    max_batch = max_batch_;
    max_ctx = max_ctx_;
    head_bf16 = head_bf16_;
    tp_rank = r;
    tp_size = t;
    if (H % t != 0 || f % t != 0) fail(GLM_CONTRACT, "glmmodel", "heads and ffn_hidden must divide by tp_size");
    if (d % 256 != 0) fail(GLM_CONTRACT, "glmmodel", "this build needs hidden % 256 == 0");
    if (dh > 256) fail(GLM_CONTRACT, "glmmodel", "head dimension > 256 unsupported");
    Hl = H / t;
    dl = Hl * dh;
    fl = f / t;
    vocab_local = (V + t - 1) / t;
    vocab_offset = static_cast<int64_t>(r) * vocab_local;
    if (vocab_offset + vocab_local > V) vocab_local = V - vocab_offset;

    CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    layers.resize(L);
    for (int l = 0; l < L; ++l) {
      Layer& ly = layers[l];
      auto mk = [&](Linear& lin, int64_t K, int64_t N, int64_t Kl, int64_t Nl, ShardSpec sh) {
        lin.Kfull = K;
        lin.Nfull = N;
        lin.shard = sh;
        lin.w.L = make_layout(Kl, Nl, bits);
        lin.w.axis = axis;
        lin.w.nscales = axis == GLM_AXIS_ROW ? Kl : axis == GLM_AXIS_COLUMN ? Nl : 1;
        lin.w.col_scale = alloc<float>(lin.w.L.Np);
        lin.w.row_scale = alloc<float>(lin.w.L.Kp);
        lin.w.scales64 = alloc<double>(lin.w.nscales);
        for (int M = 1; M <= 16; ++M) lin.plans[M] = plan_gemv(lin.w.L, M);
      };
      for (int i = 0; i < 5; ++i) ly.lin[i].role = i;
      mk(ly.lin[QKV], d, 3 * d, d, 3 * dl, ShardSpec{d, dl, static_cast<int64_t>(r) * dl, 0});
      mk(ly.lin[OUT], d, d, dl, d, ShardSpec{d, d, 0, static_cast<int64_t>(r) * dl});
      mk(ly.lin[W1], d, f, d, fl, ShardSpec{f, fl, static_cast<int64_t>(r) * fl, 0});
      mk(ly.lin[VV], d, f, d, fl, ShardSpec{f, fl, static_cast<int64_t>(r) * fl, 0});
      mk(ly.lin[W2], f, d, fl, d, ShardSpec{d, d, 0, static_cast<int64_t>(r) * fl});
      // codes: qkv, out, [w1 | v] contiguous (one fused GEMV launch), w2
      ly.lin[QKV].w.codes = alloc<uint8_t>(ly.lin[QKV].w.L.bytes(), false);
      ly.lin[OUT].w.codes = alloc<uint8_t>(ly.lin[OUT].w.L.bytes(), false);
      uint8_t* w1v = alloc<uint8_t>(ly.lin[W1].w.L.bytes() + ly.lin[VV].w.L.bytes(), false);
      ly.lin[W1].w.codes = w1v;
      ly.lin[VV].w.codes = w1v + ly.lin[W1].w.L.bytes();
      ly.lin[W2].w.codes = alloc<uint8_t>(ly.lin[W2].w.L.bytes(), false);
      ly.ln1g = alloc<float>(d);
      ly.ln1b = alloc<float>(d);
      ly.ln2g = alloc<float>(d);
      ly.ln2b = alloc<float>(d);
      k_fill<<<grid_of(d), 256, 0, st>>>(ly.ln1g, d, 1.f);
      k_fill<<<grid_of(d), 256, 0, st>>>(ly.ln2g, d, 1.f);
    }
    for (int M = 1; M <= 16; ++M)
      fused_plans[M] = plan_gemv(layers[0].lin[W1].w.L.nrt + layers[0].lin[VV].w.L.nrt, layers[0].lin[W1].w.L.nch, M,
                                 bits, axis == GLM_AXIS_ROW ? 2 : 1);
    E = head_bf16 ? static_cast<void*>(alloc<__nv_bfloat16>(static_cast<int64_t>(V) * d))
                  : static_cast<void*>(alloc<float>(static_cast<int64_t>(V) * d));
    // RoPE table in double -> float (tensor.cpp:335-341: theta_j = 10000^(-2j/dh))
    const int half = dh / 2;
    std::vector<float2> tab(static_cast<size_t>(max_ctx + 1) * half);
    for (int p = 0; p <= max_ctx; ++p)
      for (int j = 0; j < half; ++j) {
        const double th = std::pow(10000.0, -2.0 * j / static_cast<double>(dh));
        const double ang = static_cast<double>(p) * th;
        tab[static_cast<size_t>(p) * half + j] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
      }
    rope = alloc<float2>(static_cast<int64_t>(tab.size()), false);
    CUDA_CHECK(cudaMemcpyAsync(rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
    kv = alloc<__half>(kv_elems(), true);
    d_tokens = alloc<int>(max_batch);
    d_positions = alloc<int>(max_batch);
    d_len = alloc<int>(max_batch);
    d_next = alloc<int>(max_batch);
    d_status = alloc<int>(1);
    CUDA_CHECK(cudaMallocHost(&h_status, sizeof(int)));
    *h_status = 0;
    attn_splits = attn_decode_splits(max_ctx);
    if (attn_splits > 256) fail(GLM_DIMENSION, "glmmodel", "max_ctx above 16384 tokens is not supported by the decode attention");
    attn_part = alloc<float>(static_cast<int64_t>(max_batch) * Hl * attn_splits * (dh + 2));
    attn_ctr = alloc<int>(static_cast<int64_t>(max_batch) * Hl);
    CUDA_CHECK(cudaMallocHost(&h_tokens, max_batch * sizeof(int)));
    CUDA_CHECK(cudaMallocHost(&h_positions, max_batch * sizeof(int)));
    CUDA_CHECK(cudaMallocHost(&h_next, max_batch * sizeof(int)));
    h_len.assign(max_batch, 0);
    ensure_rows(max_batch);
    ensure_partial(16);
    if (tp_size > 1) {
      comm = std::make_unique<Collective>();
      // NCCL decode path: reduced sublayer rows [max_batch][d] (allocated here: never inside
      // a captured decode step)
      ar_buf.alloc(static_cast<int64_t>(max_batch) * d * 4);
      CUDA_CHECK(cudaMallocHost(&h_peer_err, sizeof(int)));
      *h_peer_err = 0;
    }
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  // Decode sublayer sums across ranks fused into the DeepNorm LayerNorm (collective.h) unless
  // GLM_TP_FUSED=0 (reduce + ncclAllReduce + LayerNorm)
  bool fused_ar() const {
    static const bool on = [] { const char* e = getenv("GLM_TP_FUSED"); return !e || e[0] != '0'; }();
    return on && comm && comm->peer_ready();
  }
  int* h_peer_err = nullptr;  // pinned copy of the fused collective's timeout word

  void init_comm(const void* uid) {
    comm->init(tp_rank, tp_size, uid);
    comm->setup_peer(max_batch, d, st);
  }
  void init_comm_emulated(EmuGroup* g) {
    comm->init_emulated(g, tp_rank);
    if (comm->size() != tp_size) fail(GLM_CONTRACT, "glmmodel", "emulated group size differs from tp_size");
    comm->setup_peer(max_batch, d, st);
  }

  GemvPlan fused_plans[17];
  const GemvPlan& fused_plan(int M) const { return fused_plans[M < 1 ? 1 : (M > 16 ? 16 : M)]; }

  static int default_ffn(int hidden, int heads) {  // model.cpp:30-37
    if ((8 * hidden) % 3 == 0) return (8 * hidden) / 3;
    const double target = 8.0 * hidden / 3.0;
    const int step = (heads % 2 == 0) ? heads : 2 * heads;
    const int lo = static_cast<int>(std::floor(target / step)) * step;
    const int hi = lo + step;
    return (target - lo <= hi - target && lo > 0) ? lo : hi;
  }

  int64_t kv_layer_elems() const { return 2ll * max_batch * Hl * static_cast<int64_t>(max_ctx) * dh; }
  int64_t kv_elems() const { return kv_layer_elems() * L; }
  __half* kcache(int l) { return kv + kv_layer_elems() * l; }
  __half* vcache(int l) { return kv + kv_layer_elems() * l + kv_layer_elems() / 2; }

  void ensure_rows(int64_t rows) {
    if (rows <= rows_cap) return;
    drop_graphs();  // captured graphs hold the old buffer addresses
    const Layer& ly = layers[0];
    const int64_t nt = std::max<int64_t>(rows, xtile_tokens(static_cast<int>(rows)));
    auto zero = [&](DeviceBuffer& b, int64_t bytes) {
      b.alloc(bytes);
      CUDA_CHECK(cudaMemsetAsync(b.ptr, 0, bytes, st));
    };
    zero(h, rows * d * 4);
    zero(xf_qkv, nt * ly.lin[QKV].w.L.Kp * 2);
    zero(xf_out, nt * ly.lin[OUT].w.L.Kp * 2);
    zero(xf_w1, nt * ly.lin[W1].w.L.Kp * 2);
    zero(xf_v, nt * ly.lin[VV].w.L.Kp * 2);
    zero(xf_w2, nt * ly.lin[W2].w.L.Kp * 2);
    zero(logits, rows * V * 4);
    zero(h_bf16, rows * d * 2);
    zero(zt_buf, 5 * rows * 4);
    pool.emplace_back(rows * 8);
    d_argmax_rows = pool.back().as<unsigned long long>();
    CUDA_CHECK(cudaMemsetAsync(d_argmax_rows, 0, rows * 8, st));
    d_argmax = d_argmax_rows;
    pool.emplace_back(rows * 4);
    d_next_rows = pool.back().as<int>();
    rows_cap = rows;
  }
  unsigned long long* d_argmax_rows = nullptr;
  int* d_next_rows = nullptr;

  // split-K partial buffer large enough for every linear at M rows
  void ensure_partial(int64_t M) {
    int64_t need = 0;
    for (int i = 0; i < 5; ++i) {
      const Linear& lin = layers[0].lin[i];
      const GemvPlan p = M <= 16 ? plan_gemv(lin.w.L, static_cast<int>(M)) : plan_qmm(lin.w.L, static_cast<int>(M));
      need = std::max<int64_t>(need, static_cast<int64_t>(p.ksplit) * M * lin.w.L.Np);
    }
    for (int mm = 1; mm <= std::min<int64_t>(M, 16); ++mm) {
      need = std::max<int64_t>(need, static_cast<int64_t>(fused_plans[mm].ksplit) * mm *
                                         (layers[0].lin[W1].w.L.Np + layers[0].lin[VV].w.L.Np));
      for (int i = 0; i < 5; ++i)
        need = std::max<int64_t>(need, static_cast<int64_t>(layers[0].lin[i].plan(mm).ksplit) * mm *
                                           layers[0].lin[i].w.L.Np);
    }
    if (need <= partial_cap) return;
    drop_graphs();
    partial.alloc(need * 4);
    partial_cap = need;
  }

  void ensure_prefill(int64_t n) {
    ensure_rows(n);
    ensure_partial(n);
    if (y_qkv.bytes >= n * 3 * dl * 4) return;
    y_qkv.alloc(n * 3 * dl * 4);
    q_rot.alloc(n * dl * 4);
    attn_out.alloc(n * dl * 4);
    y_out.alloc(n * d * 4);
    y_a.alloc(n * fl * 4);
    y_b.alloc(n * fl * 4);
    y_ffn.alloc(n * d * 4);
  }

  void ensure_taps(int64_t rows) {
    if (taps_rows >= rows) return;
    drop_graphs();
    taps_attn.alloc(static_cast<int64_t>(L) * rows * d * 4);
    taps_ffn.alloc(static_cast<int64_t>(L) * rows * d * 4);
    taps_rows = rows;
  }

  // tile = 1 for prefill activations consumed by the tcgen05 GEMM (M > 16 rows)
  // consumer activation buffer; the kRow fold vector only where it is not all ones
  XOut xout(__half* xf, const Linear& lin, int tile = 0) const {
    return XOut{xf, lin.w.L.nch, lin.w.L.Kp, tile, axis == GLM_AXIS_ROW ? lin.w.row_scale : nullptr};
  }

  // ---- weights -------------------------------------------------------------------------
  void finish_linear(Linear& lin, const double* full_scales) {
    gather_scales_device(full_scales, lin.shard, axis, lin.w.nscales, lin.w.scales64, st);
    runtime_scales_device(lin.w.scales64, lin.w.nscales, lin.w.L, axis, lin.w.col_scale, lin.w.row_scale, st);
    lin.loaded = true;
  }

  // ---- zeropoint scheme --------------------------------------------------------------------
  void set_scheme(int s) {
    if (s != GLM_ABSMAX && s != GLM_ZEROPOINT) fail(GLM_CONTRACT, "quantlab", "unknown quantization scheme");
    for (const Layer& ly : layers)
      for (const Linear& lin : ly.lin)
        if (lin.loaded) fail(GLM_CONTRACT, "glmmodel", "set the quantization scheme before loading weights");
    if (s == GLM_ZEROPOINT && scheme != GLM_ZEROPOINT)
      for (Layer& ly : layers)
        for (Linear& lin : ly.lin) {
          lin.zvec = alloc<float>(lin.w.L.Np);
          lin.zeta = alloc<float>(lin.w.L.Kp);
          lin.zps64 = alloc<double>(lin.w.nscales);
        }
    scheme = s;
    for (Layer& ly : layers)
      for (Linear& lin : ly.lin) {
        lin.w.zvec = s == GLM_ZEROPOINT ? lin.zvec : nullptr;
        lin.w.zeta = s == GLM_ZEROPOINT ? lin.zeta : nullptr;
      }
    drop_graphs();
  }
  float* zt_of(const Linear& lin) { return scheme == GLM_ZEROPOINT ? zt_buf.as<float>() + lin.role * rows_cap : nullptr; }
  // zero-point row sums of M rows of fp16 activations xf in the consumer layout (tile: tcgen05
  // token tiles, else x_frag); null for absmax
  const float* zp_rows(const Linear& lin, const __half* xf, int64_t M, int tile) {
    if (scheme != GLM_ZEROPOINT) return nullptr;
    float* zt = zt_of(lin);
    zp_sums_act(xf, static_cast<int>(M), lin.w, tile, zt, st);
    return zt;
  }
  // Zeropoint weights of this rank's shard from the FULL canonical scales / zero points (host):
  // runtime scales use s_eff = s (1 for constant groups, whose codes are 0 and value is z;
  // quant.cpp:209-216), zvec / zeta carry the zero-point rank-1 term (QWeightDev).
  void finish_linear_zp(Linear& lin, const double* scales, const double* zps) {
    const ShardSpec& sh = lin.shard;
    const int64_t ng = axis == GLM_AXIS_ROW ? lin.Kfull : axis == GLM_AXIS_COLUMN ? lin.Nfull : 1;
    std::vector<double> seff(ng);
    for (int64_t g = 0; g < ng; ++g) {
      if (!std::isfinite(scales[g]) || scales[g] < 0.0 || !std::isfinite(zps[g]))
        fail(GLM_FORMAT, "quantlab", "zeropoint scales must be finite and >= 0, zero points finite");
      seff[g] = scales[g] == 0.0 ? 1.0 : scales[g];
    }
    DeviceBuffer ds(ng * 8), dz(ng * 8), de(ng * 8), le(lin.w.nscales * 8);
    CUDA_CHECK(cudaMemcpyAsync(ds.ptr, scales, ng * 8, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(dz.ptr, zps, ng * 8, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(de.ptr, seff.data(), ng * 8, cudaMemcpyHostToDevice, st));
    gather_scales_device(ds.as<double>(), sh, axis, lin.w.nscales, lin.w.scales64, st);
    gather_scales_device(dz.as<double>(), sh, axis, lin.w.nscales, lin.zps64, st);
    gather_scales_device(de.as<double>(), sh, axis, lin.w.nscales, le.as<double>(), st);
    runtime_scales_device(le.as<double>(), lin.w.nscales, lin.w.L, axis, lin.w.col_scale, lin.w.row_scale, st);
    auto fcol = [&](int64_t j) { return (j / sh.col_per_rank_block) * sh.col_block + sh.col_offset + (j % sh.col_per_rank_block); };
    double smax = 0.0;  // the local kRow fold's S (runtime_scales_device: max over this shard)
    if (axis == GLM_AXIS_ROW)
      for (int64_t i = 0; i < lin.w.L.K; ++i) smax = std::max(smax, seff[sh.row_offset + i]);
    std::vector<float> zv(lin.w.L.Np, 0.f), ze(lin.w.L.Kp, 0.f);
    for (int64_t j = 0; j < lin.w.L.N; ++j)
      zv[j] = static_cast<float>(axis == GLM_AXIS_ROW ? smax
                                 : axis == GLM_AXIS_COLUMN ? seff[fcol(j)] * zps[fcol(j)]
                                                           : seff[0] * zps[0]);
    for (int64_t i = 0; i < lin.w.L.K; ++i) ze[i] = axis == GLM_AXIS_ROW ? static_cast<float>(zps[sh.row_offset + i]) : 1.f;
    CUDA_CHECK(cudaMemcpyAsync(lin.zvec, zv.data(), zv.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(lin.zeta, ze.data(), ze.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    lin.loaded = true;
  }

  void set_linear_quantized_zp(int l, int which, const int8_t* payload, int64_t payload_bytes, const double* scales,
                               const double* zps, int64_t nscales) {
    if (scheme != GLM_ZEROPOINT) fail(GLM_CONTRACT, "glmmodel", "zero points given to an absmax model");
    Linear& lin = layers[l].lin[which];
    const int64_t K = lin.Kfull, N = lin.Nfull, n = K * N;
    const int64_t pb = bits == 4 ? (n + 1) / 2 : n;
    const int64_t ng = axis == GLM_AXIS_ROW ? K : axis == GLM_AXIS_COLUMN ? N : 1;
    if (payload_bytes != pb) fail(GLM_FORMAT, "quantlab", "payload length does not match the linear's shape and bits");
    if (nscales != ng) fail(GLM_FORMAT, "quantlab", "scale count does not match the model's group axis");
    validate_absmax_payload(payload, pb, n, bits);  // zeropoint codes share the [-cap, cap] range (quant.cpp:27-31)
    DeviceBuffer dp(pb);
    CUDA_CHECK(cudaMemcpyAsync(dp.ptr, payload, pb, cudaMemcpyHostToDevice, st));
    repack_shard_device(dp.as<int8_t>(), N, lin.shard, lin.w.L, lin.w.codes, st);
    finish_linear_zp(lin, scales, zps);
  }

  void set_linear_from_host(int l, int which, const double* w) {
    Linear& lin = layers[l].lin[which];
    const int64_t K = lin.Kfull, N = lin.Nfull, n = K * N;
    DeviceBuffer dw(n * 8), dp(bits == 4 ? (n + 1) / 2 : n), ds((axis == GLM_AXIS_ROW ? K : axis == GLM_AXIS_COLUMN ? N : 1) * 8);
    CUDA_CHECK(cudaMemcpyAsync(dw.ptr, w, n * 8, cudaMemcpyHostToDevice, st));
    if (scheme == GLM_ZEROPOINT) {  // quantize_zeropoint (quant.cpp:145-186) on the GPU
      const int64_t ng = ds.bytes / 8;
      DeviceBuffer dz(ng * 8), dc(ng);
      quantize_device(dw.ptr, GLM_F64, K, N, bits, GLM_ZEROPOINT, axis, dp.as<int8_t>(), ds.as<double>(), dz.as<double>(),
                      dc.as<uint8_t>(), st);
      repack_shard_device(dp.as<int8_t>(), N, lin.shard, lin.w.L, lin.w.codes, st);
      std::vector<double> hs(ng), hz(ng);
      CUDA_CHECK(cudaMemcpyAsync(hs.data(), ds.ptr, ng * 8, cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaMemcpyAsync(hz.data(), dz.ptr, ng * 8, cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      finish_linear_zp(lin, hs.data(), hz.data());
      return;
    }
    quantize_device(dw.ptr, GLM_F64, K, N, bits, GLM_ABSMAX, axis, dp.as<int8_t>(), ds.as<double>(), nullptr, nullptr, st);
    repack_shard_device(dp.as<int8_t>(), N, lin.shard, lin.w.L, lin.w.codes, st);
    finish_linear(lin, ds.as<double>());
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  // A quantized linear given as the reference's canonical QuantizedMatrix (quant.hpp:26-42):
  // payload + FP64 scales go to this rank's device layout without re-quantizing.
  void set_linear_quantized(int l, int which, const int8_t* payload, int64_t payload_bytes, const double* scales,
                            int64_t nscales) {
    if (scheme == GLM_ZEROPOINT) fail(GLM_CONTRACT, "glmmodel", "a zeropoint model needs the zero points (glm_model_set_quantized_zp)");
    Linear& lin = layers[l].lin[which];
    const int64_t K = lin.Kfull, N = lin.Nfull, n = K * N;
    const int64_t pb = bits == 4 ? (n + 1) / 2 : n;
    const int64_t ng = axis == GLM_AXIS_ROW ? K : axis == GLM_AXIS_COLUMN ? N : 1;
    if (payload_bytes != pb) fail(GLM_FORMAT, "quantlab", "payload length does not match the linear's shape and bits");
    if (nscales != ng) fail(GLM_FORMAT, "quantlab", "scale count does not match the model's group axis");
    validate_absmax_payload(payload, pb, n, bits);
    for (int64_t g = 0; g < ng; ++g)
      if (!std::isfinite(scales[g]) || scales[g] < 0.0) fail(GLM_FORMAT, "quantlab", "scales must be finite and >= 0");
    DeviceBuffer dp(pb), ds(ng * 8);
    CUDA_CHECK(cudaMemcpyAsync(dp.ptr, payload, pb, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(ds.ptr, scales, ng * 8, cudaMemcpyHostToDevice, st));
    repack_shard_device(dp.as<int8_t>(), N, lin.shard, lin.w.L, lin.w.codes, st);
    finish_linear(lin, ds.as<double>());
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  void set_embedding(const double* e) { set_embedding_rows(0, V, e); }

  // rows [row0, row0 + nrows) of the tied table (streaming loaders: no full f64 copy on host or device)
  void set_embedding_rows(int64_t row0, int64_t nrows, const double* e) {
    if (row0 < 0 || nrows < 0 || row0 + nrows > V) fail(GLM_CONTRACT, "glmmodel", "embedding rows outside the vocabulary");
    const int64_t chunk_rows = std::max<int64_t>(1, (int64_t{256} << 20) / (8 * static_cast<int64_t>(d)));
    DeviceBuffer de(std::min(nrows, chunk_rows) * d * 8);
    for (int64_t r = 0; r < nrows; r += chunk_rows) {
      const int64_t nr = std::min(chunk_rows, nrows - r), n = nr * d, off = (row0 + r) * d;
      CUDA_CHECK(cudaMemcpyAsync(de.ptr, e + r * d, n * 8, cudaMemcpyHostToDevice, st));
      if (head_bf16) k_f64_to_bf16<<<grid_of(n), 256, 0, st>>>(de.as<double>(), static_cast<__nv_bfloat16*>(E) + off, n);
      else k_f64_to_f32<<<grid_of(n), 256, 0, st>>>(de.as<double>(), static_cast<float*>(E) + off, n);
      LAUNCH_CHECK("embedding upload");
      CUDA_CHECK(cudaStreamSynchronize(st));
    }
  }

  void set_vector(int l, int which, const double* v) {
    float* dst = which == 5 ? layers[l].ln1g : which == 6 ? layers[l].ln1b : which == 7 ? layers[l].ln2g : layers[l].ln2b;
    DeviceBuffer dv(static_cast<int64_t>(d) * 8);
    CUDA_CHECK(cudaMemcpyAsync(dv.ptr, v, d * 8, cudaMemcpyHostToDevice, st));
    k_f64_to_f32<<<grid_of(d), 256, 0, st>>>(dv.as<double>(), dst, d);
    LAUNCH_CHECK("ln upload");
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  void init_synthetic(uint64_t seed) {
    if (scheme != GLM_ABSMAX) fail(GLM_CONTRACT, "glmmodel", "synthetic init generates absmax weights");
    // stds of init_parameters (model.cpp:69-104); values from the counter-based generator
    const double factor = 1.0 / std::sqrt(2.0 * L);
    auto xavier = [](double a, double b) { return std::sqrt(2.0 / (a + b)); };
    const float s_init = static_cast<float>(init_std);
    const float s_v = static_cast<float>(xavier(d, d) * factor);
    const float s_out = static_cast<float>(xavier(d, d) * factor);
    const float s_ffn = static_cast<float>(xavier(d, f) * factor);
    const float s_w2 = static_cast<float>(xavier(f, d) * factor);
    for (int l = 0; l < L; ++l) {
      for (int which = 0; which < 5; ++which) {
        Linear& lin = layers[l].lin[which];
        const int64_t groups = axis == GLM_AXIS_ROW ? lin.Kfull : lin.Nfull;
        if (axis == GLM_AXIS_WHOLE) fail(GLM_CONTRACT, "glmmodel", "synthetic init supports row/column axes");
        DeviceBuffer full(groups * 8);
        float lo, hi;
        int64_t split;
        switch (which) {
          case QKV: lo = s_init; hi = s_v; split = 2ll * d; break;
          case OUT: lo = hi = s_out; split = d; break;
          case W1: case VV: lo = hi = s_ffn; split = f; break;
          default: lo = hi = s_w2; split = d; break;
        }
        gen_quantize_device(seed, static_cast<uint32_t>(l) * 8u + which, lin.Kfull, lin.Nfull, lo, hi, split, bits, axis,
                            lin.shard, lin.w.L, lin.w.codes, full.as<double>(), st);
        finish_linear(lin, full.as<double>());
        CUDA_CHECK(cudaStreamSynchronize(st));
      }
    }
    const int64_t n = static_cast<int64_t>(V) * d;
    k_gen_table<<<grid_of(n), 256, 0, st>>>(seed, kEmbedTensorId, V, d, s_init, E, head_bf16 ? 1 : 0);
    LAUNCH_CHECK("k_gen_table");
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  void check_loaded() const {
    for (const Layer& ly : layers)
      for (const Linear& lin : ly.lin)
        if (!lin.loaded) fail(GLM_CONTRACT, "glmmodel", "model weights are not loaded");
  }

  // ---- row-parallel output sum across ranks (identity at t = 1) -------------------------
  // Decode: partials are reduced into ar_buf [M][d], allreduced, then consumed with scale 1.
  SubIn row_parallel_out(const Linear& lin, const GemvPlan& p, int M, const float* zt) {
    SubIn in{partial.as<float>(), p.ksplit, static_cast<int64_t>(M) * lin.w.L.Np, lin.w.L.Np, lin.w.col_scale, zt, lin.w.zvec};
    if (tp_size == 1) return in;
    if (ar_buf.bytes < static_cast<int64_t>(M) * d * 4) fail(GLM_CONTRACT, "glmmodel", "decode batch above max_batch");
    gemv_reduce(partial.as<float>(), p.ksplit, M, lin.w, ar_buf.as<float>(), d, st, zt);
    comm->allreduce_sum(ar_buf.as<float>(), static_cast<int64_t>(M) * d, st);
    return SubIn{ar_buf.as<float>(), 1, 0, d, nullptr};
  }

  // DeepNorm LayerNorm after a row-parallel linear (out_proj, ffn_w2) in decode: at t > 1 the
  // rank partials are summed inside the LayerNorm kernel (PeerArgs); returns our launches.
  int ln_after_row_parallel(LnArgs ln, const Linear& lin, const GemvPlan& p, int M, const float* zt) {
    if (tp_size > 1 && fused_ar()) {
      ln.in = SubIn{partial.as<float>(), p.ksplit, static_cast<int64_t>(M) * lin.w.L.Np, lin.w.L.Np, lin.w.col_scale, zt,
                    lin.w.zvec};
      ln.peer = comm->peer_args();
      if (comm->emulated()) {  // push phase, group barrier, sum phase
        ln.peer.mode = 1;
        launch_deepnorm_ln(ln, M, st);
        comm->barrier(st);
        ln.peer.mode = 2;
        launch_deepnorm_ln(ln, M, st);
        return 2;
      }
      ln.peer.mode = 3;
      launch_deepnorm_ln(ln, M, st);
      return 1;
    }
    ln.in = row_parallel_out(lin, p, M, zt);
    launch_deepnorm_ln(ln, M, st);
    return tp_size > 1 ? 2 : 1;
  }

  // ---- decode step (enqueued; captured into a CUDA graph) --------------------------------
  // with_logits: the caller reads the logits (at t > 1 that adds the vocab all-gather; the
  // greedy token needs only the (value, index) max-reduction)
  int enqueue_decode(int B, bool with_logits = true) {
    int launches = 0;
    const Layer& l0 = layers[0];
    launch_embed(E, head_bf16, d, d_tokens, B, h.as<float>(), xout(xf_qkv.as<__half>(), l0.lin[QKV]), st, half_store);
    ++launches;
    for (int l = 0; l < L; ++l) launches += decode_layer(l, B, d_positions, d_len, l + 1 < L);
    launches += enqueue_head(B, logits.as<float>(), with_logits);
    launch_argmax_finish(d_argmax, d_next, B, st, d_status);
    launch_advance(d_len, B, st);
    launch_k(k_feed, dim3(1), dim3(32), 0, st, d_next, d_tokens, d_positions, B);
    LAUNCH_CHECK("k_feed");
    return launches + 3;
  }

  // One decode block (model.cpp:198-224) for B rows: input x = h (fp32 residual, [B][d]) and
  // its fp16 copy in xf_qkv (layer l's QKV activation layout); output h (and, when next_x, the
  // next layer's QKV activations). Row b appends one token at slot cache_len[b] of layer l's
  // KV cache of sequence b (the caller advances cache_len).
  int decode_layer(int l, int B, const int* positions, const int* cache_len, bool next_x) {
    int launches = 0;
    Layer& ly = layers[l];
    Linear &qkv = ly.lin[QKV], &out = ly.lin[OUT], &w1 = ly.lin[W1], &v = ly.lin[VV], &w2 = ly.lin[W2];
    const int zl = scheme == GLM_ZEROPOINT ? 5 : 0;  // zero-point row-sum launches
    const float* ztq = zp_rows(qkv, xf_qkv.as<__half>(), B, 0);
    gemv_launch(qkv.w, xf_qkv.as<__half>(), B, partial.as<float>(), qkv.plan(B), st);
    AttnDecodeArgs aa;
    aa.qkv = SubIn{partial.as<float>(), qkv.plan(B).ksplit, static_cast<int64_t>(B) * qkv.w.L.Np, qkv.w.L.Np, qkv.w.col_scale,
                   ztq, qkv.w.zvec};
    aa.d_local = dl;
    aa.heads = Hl;
    aa.dh = dh;
    aa.max_ctx = max_ctx;
    aa.max_splits = attn_splits;
    aa.positions = positions;
    aa.cache_len = cache_len;
    aa.rope = rope;
    aa.kcache = kcache(l);
    aa.vcache = vcache(l);
    aa.part = attn_part;
    aa.counters = attn_ctr;
    aa.xo = xout(xf_out.as<__half>(), out);
    aa.out = nullptr;
    aa.prescale = half_store ? prescale : 0.f;
    launch_attn_decode(aa, B, st);
    const float* zto = zp_rows(out, xf_out.as<__half>(), B, 0);
    gemv_launch(out.w, xf_out.as<__half>(), B, partial.as<float>(), out.plan(B), st);
    LnArgs ln;
    ln.h = h.as<float>();
    ln.gain = ly.ln1g;
    ln.bias = ly.ln1b;
    ln.alpha = static_cast<float>(alpha);
    ln.eps = static_cast<float>(eps);
    ln.d = d;
    ln.x0 = xout(xf_w1.as<__half>(), w1);
    ln.x1 = axis == GLM_AXIS_ROW ? xout(xf_v.as<__half>(), v) : XOut{};  // W1 and V share x unless kRow
    ln.tap = taps ? taps_attn.as<float>() + static_cast<int64_t>(l) * B * d : nullptr;
    ln.zero_sublayer = zero_sub;
    ln.half_store = half_store ? 1 : 0;
    launches += ln_after_row_parallel(ln, out, out.plan(B), B, zto);
    const float* zt1 = zp_rows(w1, xf_w1.as<__half>(), B, 0);
    const float* ztv = zp_rows(v, (axis == GLM_AXIS_ROW ? xf_v : xf_w1).as<__half>(), B, 0);
    GemvOp op{w1.w.codes, bits, w1.w.L.nrt + v.w.L.nrt, w1.w.L.nch, xf_w1.as<__half>(),
              axis == GLM_AXIS_ROW ? xf_v.as<__half>() : xf_w1.as<__half>(), w1.w.L.nrt};
    gemv_launch(op, B, partial.as<float>(), fused_plan(B), st);
    ActArgs act;
    const int64_t np_tot = w1.w.L.Np + v.w.L.Np;
    act.w1 = SubIn{partial.as<float>(), fused_plan(B).ksplit, static_cast<int64_t>(B) * np_tot, np_tot, w1.w.col_scale, zt1,
                   w1.w.zvec};
    act.v = SubIn{partial.as<float>() + w1.w.L.Np, fused_plan(B).ksplit, static_cast<int64_t>(B) * np_tot, np_tot, v.w.col_scale,
                  ztv, v.w.zvec};
    act.M = B;
    act.f = fl;
    act.xo = xout(xf_w2.as<__half>(), w2);
    launch_geglu_act(act, st);
    const float* zt2 = zp_rows(w2, xf_w2.as<__half>(), B, 0);
    gemv_launch(w2.w, xf_w2.as<__half>(), B, partial.as<float>(), w2.plan(B), st);
    LnArgs ln2 = ln;
    ln2.gain = ly.ln2g;
    ln2.bias = ly.ln2b;
    ln2.x0 = next_x ? xout(xf_qkv.as<__half>(), layers[l + 1].lin[QKV]) : XOut{};
    ln2.x1 = XOut{};
    ln2.tap = taps ? taps_ffn.as<float>() + static_cast<int64_t>(l) * B * d : nullptr;
    launches += ln_after_row_parallel(ln2, w2, w2.plan(B), B, zt2);
    return launches + 6 + zl;  // + 4 GEMVs, attention, GeGLU activation (+ zero-point sums)
  }

  int enqueue_head(int M, float* logit_out, bool gather = true) {
    HeadArgs ha;
    ha.E = E;
    ha.h = h.as<float>();
    ha.M = M;
    ha.d = d;
    ha.vocab_offset = vocab_offset;
    ha.vocab_local = vocab_local;
    ha.logits = logit_out;
    ha.ld_logits = V;
    ha.argmax = d_argmax;
    ha.hb = h_bf16.as<__nv_bfloat16>();
    launch_head(ha, head_bf16, st);
    if (tp_size > 1) {
      comm->allreduce_max_u64(d_argmax, M, st);
      if (logit_out && gather) comm->allgather_logits(logit_out, M, V, vocab_offset, vocab_local, st);
    }
    return 1;
  }

  cudaGraphExec_t graph_for(int B, bool with_logits = true) {
    with_logits = with_logits || tp_size == 1;  // one graph at t = 1 (its logits cost nothing extra)
    auto key = std::make_tuple(B, taps, zero_sub, with_logits);
    auto it = graphs.find(key);
    if (it != graphs.end()) return it->second;
    if (taps) ensure_taps(B);
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_decode(B, with_logits);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t ge;
    CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    graphs[key] = ge;
    return ge;
  }

  void drop_graphs() {
    for (auto& kv_ : graphs) cudaGraphExecDestroy(kv_.second);
    graphs.clear();
  }

  void decode_step(int B, const int* tokens, const int* positions, int* next_tokens, float* logits_out) {
    check_loaded();
    if (B < 1 || B > max_batch) fail(GLM_CONTRACT, "glmmodel", "batch must be in 1..max_batch");
    for (int b = 0; b < B; ++b) {
      if (tokens[b] < 0 || tokens[b] >= V)  // model.cpp:170-175
        fail(GLM_CONTRACT, "glmmodel", "token id " + std::to_string(tokens[b]) + " overflows vocabulary " + std::to_string(V));
      if (positions[b] < 0 || positions[b] > max_ctx) fail(GLM_CONTRACT, "glmmodel", "position outside the RoPE table");
      if (h_len[b] + 1 > max_ctx) fail(GLM_CONTRACT, "glmmodel", "KV cache of sequence " + std::to_string(b) + " is full");
      h_tokens[b] = tokens[b];
      h_positions[b] = positions[b];
    }
    CUDA_CHECK(cudaMemcpyAsync(d_tokens, h_tokens, B * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(d_positions, h_positions, B * sizeof(int), cudaMemcpyHostToDevice, st));
    static const bool eager = getenv("GLM_EAGER") != nullptr;  // debugging: no graph
    // the emulated single-GPU rank group separates its phases on the host: no graph
    if (eager || (comm && comm->emulated())) enqueue_decode(B, logits_out != nullptr);
    else CUDA_CHECK(cudaGraphLaunch(graph_for(B, logits_out != nullptr), st));
    if (logits_out) CUDA_CHECK(cudaMemcpyAsync(logits_out, logits.ptr, static_cast<int64_t>(B) * V * 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaMemcpyAsync(h_next, d_next, B * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (fused_ar()) CUDA_CHECK(cudaMemcpyAsync(h_peer_err, comm->peer_args().err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaMemcpyAsync(h_status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (h_peer_err && *h_peer_err)
      fail(GLM_NCCL, "collective", "a tensor-parallel peer did not deliver its decode partial (timeout)");
    check_status();
    for (int b = 0; b < B; ++b) {
      if (next_tokens) next_tokens[b] = h_next[b];
      h_len[b] += 1;
    }
    last_rows = B;
  }

  // ---- prefill ---------------------------------------------------------------------------
  // y[M][N] = x . W for M rows: decode GEMV (M <= 16, x_frag) or the tcgen05 GEMM (128-token
  // tiles) + split-K reduce with the group scale.
  void linear_rows(const Linear& lin, const __half* xf, int64_t M, float* y) {
    GemvPlan p;
    const float* zt = zp_rows(lin, xf, M, M > 16 ? 1 : 0);
    if (M <= 16) {
      p = lin.plan(static_cast<int>(M));
      gemv_launch(lin.w, xf, static_cast<int>(M), partial.as<float>(), p, st);
    } else {
      p = plan_qmm(lin.w.L, static_cast<int>(M));
      if (p.ksplit == 1) {  // tcgen05 epilogue writes the scaled result: no reduce pass
        qmm_launch(lin.w, xf, static_cast<int>(M), partial.as<float>(), p, st, y, lin.w.L.N, zt);
        return;
      }
      qmm_launch(lin.w, xf, static_cast<int>(M), partial.as<float>(), p, st);
    }
    gemv_reduce(partial.as<float>(), p.ksplit, static_cast<int>(M), lin.w, y, lin.w.L.N, st, zt);
  }

  // One prefill block (model.cpp:198-224) over the n packed rows: input h (fp32) + its fp16
  // copy in xf_qkv (layer l's QKV layout: tcgen05 tiles when n > 16), output h (+ the next
  // layer's QKV activations when next_x); segment i (rows row0[i].., sequence seqs[i]) fills
  // layer l's KV cache of its sequence from slot 0 and attends only to itself.
  void prefill_layer(int l, int n, int nseg, const int* seqs, const int* lens, const int* ctx, const int* row0,
                     const int* dpos, bool next_x) {
    const int nt = n > 16 ? 1 : 0;  // activation layout of this prefill: tcgen05 tiles or x_frag
    const bool attn_tiles = nt && attn_prefill_umma_eligible(dh);  // attention writes out-proj tiles
    Layer& ly = layers[l];
    Linear &qkv = ly.lin[QKV], &out = ly.lin[OUT], &w1 = ly.lin[W1], &v = ly.lin[VV], &w2 = ly.lin[W2];
    // qkv rows in fp16 straight from the tcgen05 epilogue when RoPE / the KV cache are the only
    // readers (head_dim 128, unsplit K): half the bytes written and re-read
    bool qkv_half = false;
    if (nt && dh == 128) {
      const GemvPlan pq = plan_qmm(qkv.w.L, n);
      if (pq.ksplit == 1) {
        qmm_launch(qkv.w, xf_qkv.as<__half>(), n, partial.as<float>(), pq, st, y_qkv.as<float>(), qkv.w.L.N,
                   zp_rows(qkv, xf_qkv.as<__half>(), n, 1), true);
        qkv_half = true;
      }
    }
    if (!qkv_half) linear_rows(qkv, xf_qkv.as<__half>(), n, y_qkv.as<float>());
    for (int i = 0; i < nseg; ++i) {
      const int r0 = row0[i], ni = lens[i];
      float* qseg = q_rot.as<float>() + static_cast<int64_t>(r0) * dl;  // [heads][ni][dh] of this sample
      RopeStoreArgs rs{y_qkv.as<float>() + static_cast<int64_t>(r0) * 3 * dl, 3ll * dl, dl, ni, Hl, dh, seqs[i],
                       max_ctx, 0, dpos + r0, rope, qseg, kcache(l), vcache(l)};
      if (qkv_half) rs.qkv_h = reinterpret_cast<const __half*>(y_qkv.as<float>()) + static_cast<int64_t>(r0) * 3 * dl;
      launch_rope_store(rs, st);
      AttnPrefillArgs ap{qseg, kcache(l), vcache(l), ni, Hl, dh, seqs[i], max_ctx, ctx[i],
                         attn_out.as<float>() + static_cast<int64_t>(r0) * dl, dl};
      if (attn_tiles) {
        ap.xo = xout(xf_out.as<__half>(), out, nt);
        ap.xrow0 = r0;
      }
      ap.prescale = half_store ? prescale : 0.f;
      launch_attn_prefill(ap, st);
    }
    if (!attn_tiles) launch_rows_to_xfrag(attn_out.as<float>(), dl, n, dl, xout(xf_out.as<__half>(), out, nt), st);
    linear_rows(out, xf_out.as<__half>(), n, y_out.as<float>());
    if (tp_size > 1) comm->allreduce_sum(y_out.as<float>(), static_cast<int64_t>(n) * d, st);
    LnArgs ln;
    ln.in = SubIn{y_out.as<float>(), 1, 0, d, nullptr};
    ln.h = h.as<float>();
    ln.gain = ly.ln1g;
    ln.bias = ly.ln1b;
    ln.alpha = static_cast<float>(alpha);
    ln.eps = static_cast<float>(eps);
    ln.d = d;
    ln.x0 = xout(xf_w1.as<__half>(), w1, nt);
    ln.x1 = axis == GLM_AXIS_ROW ? xout(xf_v.as<__half>(), v, nt) : XOut{};  // W1 and V share x unless kRow
    ln.tap = taps ? taps_attn.as<float>() + static_cast<int64_t>(l) * n * d : nullptr;
    ln.zero_sublayer = zero_sub;
    ln.half_store = half_store ? 1 : 0;
    launch_deepnorm_ln(ln, n, st);
    if (axis != GLM_AXIS_ROW && qmm_geglu_supported(w1.w, v.w, n)) {  // W1|V GEMM with the GeGLU epilogue
      const XOut xo = xout(xf_w2.as<__half>(), w2, nt);
      qmm_geglu_launch(w1.w, v.w, xf_w1.as<__half>(), n, xo.xf, xo.Kp, xo.row_scale, st);
    } else {
      linear_rows(w1, xf_w1.as<__half>(), n, y_a.as<float>());
      linear_rows(v, (axis == GLM_AXIS_ROW ? xf_v : xf_w1).as<__half>(), n, y_b.as<float>());
      ActArgs act;
      act.w1 = SubIn{y_a.as<float>(), 1, 0, fl, nullptr};
      act.v = SubIn{y_b.as<float>(), 1, 0, fl, nullptr};
      act.M = n;
      act.f = fl;
      act.xo = xout(xf_w2.as<__half>(), w2, nt);
      launch_geglu_act(act, st);
    }
    linear_rows(w2, xf_w2.as<__half>(), n, y_ffn.as<float>());
    if (tp_size > 1) comm->allreduce_sum(y_ffn.as<float>(), static_cast<int64_t>(n) * d, st);
    LnArgs ln2 = ln;
    ln2.in = SubIn{y_ffn.as<float>(), 1, 0, d, nullptr};
    ln2.gain = ly.ln2g;
    ln2.bias = ly.ln2b;
    ln2.x0 = next_x ? xout(xf_qkv.as<__half>(), layers[l + 1].lin[QKV], nt) : XOut{};
    ln2.x1 = XOut{};
    ln2.tap = taps ? taps_ffn.as<float>() + static_cast<int64_t>(l) * n * d : nullptr;
    launch_deepnorm_ln(ln2, n, st);
  }

  // ---- block-level API (glm_block_forward): one layer on caller hidden states ------------
  // The KV cache is the model's; the block API keeps its own per-layer cache lengths
  // (blk_len[layer][seq]) so a caller can drive the layers one at a time.
  std::vector<int> h_blen;  // [L][max_batch]
  DeviceBuffer d_blen_buf;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;

  void block_forward(int l, int mode, int seq, float* x, const int* dpos, const int* hpos, int n, int ctx,
                     cudaStream_t user) {
    check_loaded();
    if (l < 0 || l >= L) fail(GLM_CONTRACT, "glmmodel", "layer index out of range");
    if (mode != GLM_BLOCK_PREFILL && mode != GLM_BLOCK_DECODE) fail(GLM_CONTRACT, "glmmodel", "unknown block mode");
    if (h_blen.empty()) {
      h_blen.assign(static_cast<size_t>(L) * max_batch, 0);
      d_blen_buf.alloc(static_cast<int64_t>(L) * max_batch * 4);
      CUDA_CHECK(cudaMemsetAsync(d_blen_buf.ptr, 0, d_blen_buf.bytes, st));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
    }
    int* blen = d_blen_buf.as<int>() + static_cast<int64_t>(l) * max_batch;
    int* hl = h_blen.data() + static_cast<size_t>(l) * max_batch;
    if (mode == GLM_BLOCK_PREFILL) {
      if (seq < 0 || seq >= max_batch) fail(GLM_CONTRACT, "glmmodel", "sequence index outside max_batch");
      if (n < 1 || n > max_ctx) fail(GLM_CONTRACT, "glmmodel", "prefill length must be in 1..max_ctx");
      if (ctx < 0 || ctx > n) fail(GLM_CONTRACT, "glmmodel", "context_length must be in 0..n");
    } else {
      if (n < 1 || n > max_batch) fail(GLM_CONTRACT, "glmmodel", "decode rows must be in 1..max_batch");
      for (int b = 0; b < n; ++b)
        if (hl[b] + 1 > max_ctx) fail(GLM_CONTRACT, "glmmodel", "KV cache of sequence " + std::to_string(b) + " is full");
    }
    if (hpos)
      for (int i = 0; i < n; ++i)
        if (hpos[i] < 0 || hpos[i] > max_ctx) fail(GLM_CONTRACT, "glmmodel", "position outside the RoPE table");
    if (mode == GLM_BLOCK_PREFILL) ensure_prefill(n);
    if (taps) ensure_taps(n);
    CUDA_CHECK(cudaEventRecord(ev_in, user));
    CUDA_CHECK(cudaStreamWaitEvent(st, ev_in, 0));
    const int nt = (mode == GLM_BLOCK_PREFILL && n > 16) ? 1 : 0;
    CUDA_CHECK(cudaMemcpyAsync(h.ptr, x, static_cast<int64_t>(n) * d * 4, cudaMemcpyDeviceToDevice, st));
    launch_rows_to_xfrag(h.as<float>(), d, n, d, xout(xf_qkv.as<__half>(), layers[l].lin[QKV], nt), st);
    if (mode == GLM_BLOCK_PREFILL) {
      const int row0[2] = {0, n};
      prefill_layer(l, n, 1, &seq, &n, &ctx, row0, dpos, false);
      CUDA_CHECK(cudaMemcpyAsync(blen + seq, &n, 4, cudaMemcpyHostToDevice, st));
    } else {
      decode_layer(l, n, dpos, blen, false);
      launch_advance(blen, n, st);
    }
    CUDA_CHECK(cudaMemcpyAsync(x, h.ptr, static_cast<int64_t>(n) * d * 4, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaEventRecord(ev_out, st));
    CUDA_CHECK(cudaStreamWaitEvent(user, ev_out, 0));
    if (mode == GLM_BLOCK_PREFILL) hl[seq] = n;
    else
      for (int b = 0; b < n; ++b) hl[b] += 1;
    last_rows = n;
  }

  void prefill(int seq, const int* tokens, const int* positions, int n, int context_len, float* logits_out) {
    prefill_batch(1, &seq, &n, &context_len, tokens, positions, logits_out);
  }

  // Packed prefill (pack_samples, corruption.cpp:295-334): `nseg` samples concatenated row-wise
  // run through every linear / LayerNorm / GeGLU as one M = sum(n) batch; RoPE, the KV-cache
  // write and attention stay per sample (segment isolation: each sample attends only to its
  // own sequence's cache), each filling sequence seqs[i] from slot 0.
  void prefill_batch(int nseg, const int* seqs, const int* lens, const int* ctx, const int* tokens,
                     const int* positions, float* logits_out) {
    check_loaded();
    if (nseg < 1 || nseg > max_batch) fail(GLM_CONTRACT, "glmmodel", "segment count must be in 1..max_batch");
    std::vector<int> row0(nseg + 1, 0);
    std::vector<bool> used(max_batch, false);
    for (int i = 0; i < nseg; ++i) {
      if (seqs[i] < 0 || seqs[i] >= max_batch) fail(GLM_CONTRACT, "glmmodel", "sequence index outside max_batch");
      if (used[seqs[i]]) fail(GLM_CONTRACT, "glmmodel", "a sequence appears twice in one packed prefill");
      used[seqs[i]] = true;
      if (lens[i] < 1 || lens[i] > max_ctx) fail(GLM_CONTRACT, "glmmodel", "prefill length must be in 1..max_ctx");
      if (ctx[i] < 0 || ctx[i] > lens[i]) fail(GLM_CONTRACT, "glmmodel", "context_length must be in 0..n");
      row0[i + 1] = row0[i] + lens[i];
    }
    const int n = row0[nseg];
    for (int i = 0; i < n; ++i) {
      if (tokens[i] < 0 || tokens[i] >= V)
        fail(GLM_CONTRACT, "glmmodel", "token id " + std::to_string(tokens[i]) + " overflows vocabulary " + std::to_string(V));
      if (positions[i] < 0 || positions[i] > max_ctx) fail(GLM_CONTRACT, "glmmodel", "position outside the RoPE table");
    }
    ensure_prefill(n);
    const int nt = n > 16 ? 1 : 0;  // activation layout of this prefill: tcgen05 tiles or x_frag
    if (taps) ensure_taps(n);
    DeviceBuffer dtok(n * 4), dpos(n * 4);
    CUDA_CHECK(cudaMemcpyAsync(dtok.ptr, tokens, n * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(dpos.ptr, positions, n * 4, cudaMemcpyHostToDevice, st));
    launch_embed(E, head_bf16, d, dtok.as<int>(), n, h.as<float>(), xout(xf_qkv.as<__half>(), layers[0].lin[QKV], nt), st,
                 half_store);
    for (int l = 0; l < L; ++l) prefill_layer(l, n, nseg, seqs, lens, ctx, row0.data(), dpos.as<int>(), l + 1 < L);
    if (logits_out) {
      enqueue_head(n, logits.as<float>());
      launch_argmax_finish(d_argmax, d_next_rows, n, st, d_status);
      CUDA_CHECK(cudaMemcpyAsync(logits_out, logits.ptr, static_cast<int64_t>(n) * V * 4, cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaMemcpyAsync(h_status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
    }
    for (int i = 0; i < nseg; ++i)
      CUDA_CHECK(cudaMemcpyAsync(d_len + seqs[i], &lens[i], 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    for (int i = 0; i < nseg; ++i) h_len[seqs[i]] = lens[i];
    last_rows = n;
    if (logits_out) check_status();
  }

  // a non-finite winning logit (k_argmax_finish): an fp16 activation overflowed (|x| > 65504,
  // e.g. a loaded checkpoint outside the range random init stays in) or the weights are not finite
  void check_status() {
    if (!*h_status) return;
    *h_status = 0;
    CUDA_CHECK(cudaMemsetAsync(d_status, 0, sizeof(int), st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    fail(GLM_POLICY, "glmmodel",
         "non-finite logits: an activation left the fp16 range of the quantized linears (|x| > 65504) or the "
         "parameters are not finite");
  }

};

// ======================================================================================
// C ABI (include/glm130b.h)
// ======================================================================================
namespace {

glm_model* checked(glm_model* m) {
  if (!m) fail(GLM_CONTRACT, "glmmodel", "null model handle");
  return m;
}
const glm_model* checked(const glm_model* m) {
  if (!m) fail(GLM_CONTRACT, "glmmodel", "null model handle");
  return m;
}

int64_t pbytes(int64_t K, int64_t N, int bits) { return bits == 4 ? (K * N + 1) / 2 : K * N; }

}  // namespace

extern "C" {

glm_status glm_tp_unique_id(void* out128) {
  return guarded([&] { Collective::unique_id(out128); });
}

glm_status glm_model_create(const glm_config* cfg, int bits, glm_axis axis, int max_batch, int max_ctx, int head_bf16,
                            int tp_rank, int tp_size, glm_model** out) {
  return guarded([&] {
    if (!cfg || !out) fail(GLM_CONTRACT, "glmmodel", "null argument");
    auto m = std::make_unique<glm_model>();
    m->setup(*cfg, bits, axis, max_batch, max_ctx, head_bf16 != 0, tp_rank, tp_size);
    *out = m.release();
  });
}

glm_status glm_model_init_comm(glm_model* m, const void* unique_id) {
  return guarded([&] {
    checked(m);
    if (m->tp_size == 1) return;
    if (!unique_id) fail(GLM_CONTRACT, "glmmodel", "null unique id");
    m->init_comm(unique_id);
  });
}

glm_status glm_tp_emulated_group_create(int size, glm_tp_group** out) {
  return guarded([&] {
    if (!out) fail(GLM_CONTRACT, "collective", "null output");
    *out = reinterpret_cast<glm_tp_group*>(emu_group_create(size));
  });
}

glm_status glm_tp_emulated_group_destroy(glm_tp_group* g) {
  return guarded([&] { emu_group_destroy(reinterpret_cast<EmuGroup*>(g)); });
}

glm_status glm_model_init_comm_emulated(glm_model* m, glm_tp_group* g) {
  return guarded([&] {
    checked(m);
    if (m->tp_size == 1) return;
    m->init_comm_emulated(reinterpret_cast<EmuGroup*>(g));
  });
}

glm_status glm_model_destroy(glm_model* m) {
  return guarded([&] { delete m; });
}

glm_status glm_model_set_embedding(glm_model* m, const double* e) {
  return guarded([&] { checked(m)->set_embedding(e); });
}

glm_status glm_model_set_embedding_rows(glm_model* m, int64_t row0, int64_t nrows, const double* values) {
  return guarded([&] {
    if (!values && nrows > 0) fail(GLM_CONTRACT, "glmmodel", "null argument");
    checked(m)->set_embedding_rows(row0, nrows, values);
  });
}

glm_status glm_model_set_tensor(glm_model* m, int layer, int which, const double* values) {
  return guarded([&] {
    checked(m);
    if (layer < 0 || layer >= m->L) fail(GLM_CONTRACT, "glmmodel", "layer index out of range");
    if (which >= 0 && which < 5) m->set_linear_from_host(layer, which, values);
    else if (which >= 5 && which < 9) m->set_vector(layer, which, values);
    else fail(GLM_CONTRACT, "glmmodel", "unknown tensor slot");
  });
}

glm_status glm_model_get_config(const glm_model* m, glm_config* out) {
  return guarded([&] {
    checked(m);
    if (!out) fail(GLM_CONTRACT, "glmmodel", "null output");
    *out = glm_config{m->L, m->d, m->H, m->f, m->V, m->init_std, m->eps, m->alpha};
  });
}

glm_status glm_model_set_quantized(glm_model* m, int layer, int which, const int8_t* payload,
                                   int64_t payload_bytes, const double* scales, int64_t nscales) {
  return guarded([&] {
    checked(m);
    if (layer < 0 || layer >= m->L || which < 0 || which > 4) fail(GLM_CONTRACT, "glmmodel", "bad linear index");
    if (!payload || !scales) fail(GLM_CONTRACT, "glmmodel", "null payload or scales");
    m->set_linear_quantized(layer, which, payload, payload_bytes, scales, nscales);
  });
}

glm_status glm_model_set_scheme(glm_model* m, glm_scheme scheme) {
  return guarded([&] { checked(m)->set_scheme(scheme); });
}

glm_status glm_model_set_quantized_zp(glm_model* m, int layer, int which, const int8_t* payload, int64_t payload_bytes,
                                      const double* scales, const double* zero_points, int64_t ngroups) {
  return guarded([&] {
    checked(m);
    if (layer < 0 || layer >= m->L || which < 0 || which > 4) fail(GLM_CONTRACT, "glmmodel", "bad linear index");
    if (!payload || !scales || !zero_points) fail(GLM_CONTRACT, "glmmodel", "null payload, scales or zero points");
    m->set_linear_quantized_zp(layer, which, payload, payload_bytes, scales, zero_points, ngroups);
  });
}

glm_status glm_model_export_zero_points(const glm_model* m, int layer, int which, double* zero_points) {
  return guarded([&] {
    checked(m);
    if (layer < 0 || layer >= m->L || which < 0 || which > 4) fail(GLM_CONTRACT, "glmmodel", "bad linear index");
    if (m->scheme != GLM_ZEROPOINT) fail(GLM_CONTRACT, "glmmodel", "an absmax model has no zero points");
    const Linear& lin = m->layers[layer].lin[which];
    CUDA_CHECK(cudaMemcpyAsync(zero_points, lin.zps64, lin.w.nscales * 8, cudaMemcpyDeviceToHost, m->st));
    CUDA_CHECK(cudaStreamSynchronize(m->st));
  });
}

glm_status glm_model_init_synthetic(glm_model* m, uint64_t seed) {
  return guarded([&] { checked(m)->init_synthetic(seed); });
}

glm_status glm_model_export_linear(const glm_model* m, int layer, int which, int8_t* payload, double* scales) {
  return guarded([&] {
    checked(m);
    if (layer < 0 || layer >= m->L || which < 0 || which > 4) fail(GLM_CONTRACT, "glmmodel", "bad linear index");
    const Linear& lin = m->layers[layer].lin[which];
    const int64_t pb = pbytes(lin.w.L.K, lin.w.L.N, m->bits);
    DeviceBuffer dp(pb);
    unrepack_device(lin.w.codes, lin.w.L, dp.as<int8_t>(), m->st);
    CUDA_CHECK(cudaMemcpyAsync(payload, dp.ptr, pb, cudaMemcpyDeviceToHost, m->st));
    CUDA_CHECK(cudaMemcpyAsync(scales, lin.w.scales64, lin.w.nscales * 8, cudaMemcpyDeviceToHost, m->st));
    CUDA_CHECK(cudaStreamSynchronize(m->st));
  });
}

glm_status glm_model_memory(const glm_model* m, glm_memory* out) {
  return guarded([&] {
    checked(m);
    // memory_accounting (quant.cpp:344-358) over the full (unsharded) model
    glm_memory r{};
    for (const Layer& ly : m->layers)
      for (const Linear& lin : ly.lin) {
        r.element_count += lin.Kfull * lin.Nfull;
        r.quant_payload_bytes += pbytes(lin.Kfull, lin.Nfull, m->bits);
        const int64_t groups = m->axis == GLM_AXIS_ROW ? lin.Kfull : m->axis == GLM_AXIS_COLUMN ? lin.Nfull : 1;
        r.scale_bytes += groups * 8 * (m->scheme == GLM_ZEROPOINT ? 2 : 1);  // + zero points (quant.cpp:352-353)
        r.device_weight_bytes += lin.w.L.bytes();
      }
    r.half_baseline_bytes = 2 * r.element_count;
    r.wide_baseline_bytes = 8 * r.element_count;
    r.device_head_bytes = static_cast<int64_t>(m->V) * m->d * (m->head_bf16 ? 2 : 4);
    r.device_kv_bytes = m->kv_elems() * 2;
    *out = r;
  });
}

glm_status glm_model_prefill(glm_model* m, int seq, const int* tokens, const int* positions, int n, int context_length,
                             float* logits) {
  return guarded([&] { checked(m)->prefill(seq, tokens, positions, n, context_length, logits); });
}

glm_status glm_model_prefill_batch(glm_model* m, int nseg, const int* seqs, const int* lengths,
                                   const int* context_lengths, const int* tokens, const int* positions, float* logits) {
  return guarded([&] {
    if (!seqs || !lengths || !context_lengths || !tokens || !positions) fail(GLM_CONTRACT, "glmmodel", "null argument");
    checked(m)->prefill_batch(nseg, seqs, lengths, context_lengths, tokens, positions, logits);
  });
}

glm_status glm_model_decode_step(glm_model* m, int batch, const int* tokens, const int* positions, int* next_tokens,
                                 float* logits) {
  return guarded([&] { checked(m)->decode_step(batch, tokens, positions, next_tokens, logits); });
}

int glm_model_cached_length(const glm_model* m, int seq) {
  if (!m || seq < 0 || seq >= m->max_batch) return -1;
  return m->h_len[seq];
}

glm_status glm_model_reset(glm_model* m) {
  return guarded([&] {
    checked(m);
    std::fill(m->h_len.begin(), m->h_len.end(), 0);
    CUDA_CHECK(cudaMemsetAsync(m->d_len, 0, m->max_batch * sizeof(int), m->st));
    std::fill(m->h_blen.begin(), m->h_blen.end(), 0);
    if (m->d_blen_buf.bytes) CUDA_CHECK(cudaMemsetAsync(m->d_blen_buf.ptr, 0, m->d_blen_buf.bytes, m->st));
    CUDA_CHECK(cudaStreamSynchronize(m->st));
  });
}

glm_status glm_block_forward(glm_model* m, int layer, glm_block_mode mode, int seq, float* x_io, const int* positions,
                             int n, int context_length, void* stream) {
  return guarded([&] {
    if (!x_io || !positions) fail(GLM_CONTRACT, "glmmodel", "null argument");
    checked(m)->block_forward(layer, mode, seq, x_io, positions, nullptr, n, context_length,
                              static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_block_forward_host(glm_model* m, int layer, glm_block_mode mode, int seq, float* x_io,
                                  const int* positions, int n, int context_length) {
  return guarded([&] {
    if (!x_io || !positions) fail(GLM_CONTRACT, "glmmodel", "null argument");
    checked(m);
    if (n < 1 || n > std::max(m->max_ctx, m->max_batch)) fail(GLM_CONTRACT, "glmmodel", "row count out of range");
    DeviceBuffer dx(static_cast<int64_t>(n) * m->d * 4), dp(static_cast<int64_t>(n) * 4);
    CUDA_CHECK(cudaMemcpy(dx.ptr, x_io, dx.bytes, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dp.ptr, positions, dp.bytes, cudaMemcpyHostToDevice));
    m->block_forward(layer, mode, seq, dx.as<float>(), dp.as<int>(), positions, n, context_length, m->st);
    CUDA_CHECK(cudaMemcpyAsync(x_io, dx.ptr, dx.bytes, cudaMemcpyDeviceToHost, m->st));
    CUDA_CHECK(cudaStreamSynchronize(m->st));
  });
}

glm_status glm_model_enable_taps(glm_model* m, int enable) {
  return guarded([&] { checked(m)->taps = enable != 0; });
}

glm_status glm_model_get_taps(const glm_model* m, float* attn, float* ffn) {
  return guarded([&] {
    checked(m);
    if (!m->taps || m->taps_rows < m->last_rows || m->last_rows == 0)
      fail(GLM_CONTRACT, "glmmodel", "taps were not recorded by the last call");
    const int64_t bytes = static_cast<int64_t>(m->L) * m->last_rows * m->d * 4;
    CUDA_CHECK(cudaMemcpy(attn, m->taps_attn.ptr, bytes, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(ffn, m->taps_ffn.ptr, bytes, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_model_set_precision(glm_model* m, int half_storage, double softmax_prescale) {
  return guarded([&] {
    checked(m);
    if (!(softmax_prescale > 0.0) || !std::isfinite(softmax_prescale))
      fail(GLM_CONTRACT, "tensorcore", "softmax_prescale must be a positive finite number");
    m->drop_graphs();  // captured steps hold the old policy in their kernel arguments
    m->half_store = half_storage != 0;
    m->prescale = static_cast<float>(softmax_prescale);
  });
}

glm_status glm_model_zero_sublayers(glm_model* m, int enable) {
  return guarded([&] { checked(m)->zero_sub = enable != 0; });
}

glm_status glm_model_bench_decode(glm_model* m, int batch, int steps, int warmup, double* ms_per_step,
                                  double* gemv_ms_per_step, int* launches_per_step) {
  return guarded([&] {
    checked(m);
    m->check_loaded();
    if (m->comm && m->comm->emulated()) fail(GLM_CONTRACT, "glmmodel", "bench_decode needs a real communicator (graph replay)");
    if (batch < 1 || batch > m->max_batch) fail(GLM_CONTRACT, "glmmodel", "batch must be in 1..max_batch");
    for (int b = 0; b < batch; ++b)
      if (m->h_len[b] + warmup + steps > m->max_ctx) fail(GLM_CONTRACT, "glmmodel", "bench would overflow the KV cache");
    // counts our kernel launches of one step (capture-free dry count happens in graph_for)
    cudaGraphExec_t ge = m->graph_for(batch, false);
    for (int i = 0; i < warmup; ++i) CUDA_CHECK(cudaGraphLaunch(ge, m->st));
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    CUDA_CHECK(cudaStreamSynchronize(m->st));
    CUDA_CHECK(cudaEventRecord(e0, m->st));
    for (int i = 0; i < steps; ++i) CUDA_CHECK(cudaGraphLaunch(ge, m->st));
    CUDA_CHECK(cudaEventRecord(e1, m->st));
    CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_step = ms / steps;
    for (int b = 0; b < batch; ++b) m->h_len[b] += warmup + steps;
    if (launches_per_step) {
      // count kernel nodes of the step graph
      cudaGraph_t g;
      CUDA_CHECK(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
      m->enqueue_decode(batch, false);
      CUDA_CHECK(cudaStreamEndCapture(m->st, &g));
      size_t nn = 0;
      CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &nn));
      int kernels = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        CUDA_CHECK(cudaGraphNodeGetType(nd, &t));
        if (t == cudaGraphNodeTypeKernel) ++kernels;
      }
      cudaGraphDestroy(g);
      *launches_per_step = kernels;
    }
    if (gemv_ms_per_step) {
      // the GEMV launches of one step alone (same buffers), timed as a graph
      cudaGraph_t g;
      CUDA_CHECK(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
      for (int l = 0; l < m->L; ++l) {
        Layer& ly = m->layers[l];
        gemv_launch(ly.lin[QKV].w, m->xf_qkv.as<__half>(), batch, m->partial.as<float>(), ly.lin[QKV].plan(batch), m->st);
        gemv_launch(ly.lin[OUT].w, m->xf_out.as<__half>(), batch, m->partial.as<float>(), ly.lin[OUT].plan(batch), m->st);
        GemvOp op{ly.lin[W1].w.codes, m->bits, ly.lin[W1].w.L.nrt + ly.lin[VV].w.L.nrt, ly.lin[W1].w.L.nch,
                  m->xf_w1.as<__half>(), m->axis == GLM_AXIS_ROW ? m->xf_v.as<__half>() : m->xf_w1.as<__half>(),
                  ly.lin[W1].w.L.nrt};
        gemv_launch(op, batch, m->partial.as<float>(), m->fused_plan(batch), m->st);
        gemv_launch(ly.lin[W2].w, m->xf_w2.as<__half>(), batch, m->partial.as<float>(), ly.lin[W2].plan(batch), m->st);
      }
      CUDA_CHECK(cudaStreamEndCapture(m->st, &g));
      cudaGraphExec_t gx;
      CUDA_CHECK(cudaGraphInstantiate(&gx, g, 0));
      cudaGraphDestroy(g);
      CUDA_CHECK(cudaGraphLaunch(gx, m->st));
      const int reps = steps < 5 ? 5 : steps;
      CUDA_CHECK(cudaEventRecord(e0, m->st));
      for (int i = 0; i < reps; ++i) CUDA_CHECK(cudaGraphLaunch(gx, m->st));
      CUDA_CHECK(cudaEventRecord(e1, m->st));
      CUDA_CHECK(cudaEventSynchronize(e1));
      CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      *gemv_ms_per_step = ms / reps;
      cudaGraphExecDestroy(gx);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
