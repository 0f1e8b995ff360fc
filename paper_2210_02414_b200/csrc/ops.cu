// ops.cu — the reference's op-level block functions at the C ABI (model.hpp:70-80):
// deepnorm_residual (model.cpp:125-131), geglu (model.cpp:133-135) and single-head attention
// with an arbitrary visibility mask (model.cpp:137-152). The model's own decode / prefill
// paths use the fused kernels of block.cu / attn_tc.cu; these entry points expose the same
// arithmetic one op at a time for reference-shaped callers and for op-level parity tests.
#include <cmath>
#include <string>

#include "block.h"
#include "common.cuh"
#include "device_buffer.h"
#include "kernels.h"

struct glm_qweight;  // capi_quant.cpp

namespace glm {

void qlinear_device(const glm_qweight* q, const float* x, int64_t M, float* y, cudaStream_t st);  // capi_quant.cpp
const QWeightDev& qweight_dev(const glm_qweight* q);                                               // capi_quant.cpp

namespace {

constexpr float kInvSqrt2 = 0.70710678118654752440f;

int grid_for_n(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b < kNumSMs * 16 ? b : kNumSMs * 16));
}

// GeLU(u) * v, exact erf GeLU (tensor.cpp:313-318)
__global__ void k_gelu_mul(const float* __restrict__ u, const float* __restrict__ v, float* __restrict__ g, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    g[i] = 0.5f * u[i] * (1.f + erff(u[i] * kInvSqrt2)) * v[i];
}

// rope_rotate (tensor.cpp:335-394): adjacent pairs (2j, 2j+1), theta_j = 10000^(-2j/d),
// angle = pos * theta_j, evaluated in double like the reference; values in fp32
__global__ void k_rope_rows(const float* __restrict__ x, int64_t n, int64_t dh, const int* __restrict__ pos,
                            float* __restrict__ out) {
  const int64_t half = dh / 2, total = n * half;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / half, j = i % half;
    const double th = pow(10000.0, -2.0 * static_cast<double>(j) / static_cast<double>(dh));
    double s, c;
    sincos(static_cast<double>(pos[r]) * th, &s, &c);
    const float a = x[r * dh + 2 * j], b = x[r * dh + 2 * j + 1];
    out[r * dh + 2 * j] = static_cast<float>(c * a - s * b);
    out[r * dh + 2 * j + 1] = static_cast<float>(s * a + c * b);
  }
}

// One CTA per query row: scores = rq . rk^T / sqrt(dh), invisible -> -inf (masked_fill,
// tensor.cpp:472-482), wide softmax (tensor.cpp:221-254), out = P . v. A row with no visible
// key raises the reference's PolicyError through *err.
constexpr int kAttnOpThreads = 256;
__global__ void __launch_bounds__(kAttnOpThreads) k_attn_op(const float* __restrict__ rq, const float* __restrict__ rk,
                                                            const float* __restrict__ v, int64_t n, int64_t dh,
                                                            const uint8_t* __restrict__ mask, float* __restrict__ out,
                                                            int* err) {
  extern __shared__ float sm[];  // [n] scores | [dh] q row | [32] reduction
  float* sc = sm;
  float* qrow = sm + n;
  float* red = qrow + dh;
  const int64_t i = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kAttnOpThreads / 32;
  for (int64_t k = threadIdx.x; k < dh; k += kAttnOpThreads) qrow[k] = rq[i * dh + k];
  __syncthreads();
  const float inv = 1.f / sqrtf(static_cast<float>(dh));
  for (int64_t j = warp; j < n; j += nw) {
    float s = 0.f;
    for (int64_t k = lane; k < dh; k += 32) s += qrow[k] * rk[j * dh + k];
    s = warp_sum(s);
    if (lane == 0) sc[j] = mask[i * n + j] ? s * inv : -INFINITY;
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += kAttnOpThreads) mx = fmaxf(mx, sc[j]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < nw; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  if (mx == -INFINITY) {
    if (threadIdx.x == 0) atomicMin(err, static_cast<int>(i));
    for (int64_t k = threadIdx.x; k < dh; k += kAttnOpThreads) out[i * dh + k] = 0.f;
    return;
  }
  float tot = 0.f;
  for (int64_t j = threadIdx.x; j < n; j += kAttnOpThreads) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    tot += e;
  }
  tot = warp_sum(tot);
  if (lane == 0) red[warp] = tot;
  __syncthreads();
  tot = 0.f;
  for (int w = 0; w < nw; ++w) tot += red[w];
  const float rt = 1.f / tot;
  for (int64_t k = threadIdx.x; k < dh; k += kAttnOpThreads) {
    float acc = 0.f;
    for (int64_t j = 0; j < n; ++j) acc += sc[j] * v[j * dh + k];
    out[i * dh + k] = acc * rt;
  }
}

void deepnorm_device(const float* x, const float* y, int64_t rows, int64_t d, double alpha, const float* gain,
                     const float* bias, double eps, float* out, cudaStream_t st) {
  if (rows < 1 || d < 2 || d % 2) fail(GLM_DIMENSION, "glmmodel", "deepnorm_residual needs rows >= 1 and an even width");
  if (out != x) CUDA_CHECK(cudaMemcpyAsync(out, x, rows * d * 4, cudaMemcpyDeviceToDevice, st));
  LnArgs ln;
  ln.in = SubIn{y, 1, 0, d, nullptr};
  ln.h = out;
  ln.gain = gain;
  ln.bias = bias;
  ln.alpha = static_cast<float>(alpha);
  ln.eps = static_cast<float>(eps);
  ln.d = d;
  ln.x0 = XOut{};
  ln.x1 = XOut{};
  ln.tap = nullptr;
  ln.zero_sublayer = 0;
  launch_deepnorm_ln(ln, static_cast<int>(rows), st);
}

void geglu_device(const glm_qweight* w1, const glm_qweight* v, const glm_qweight* w2, const float* x, int64_t M,
                  float* y, cudaStream_t st) {
  const QWeightDev &a = qweight_dev(w1), &b = qweight_dev(v), &c = qweight_dev(w2);
  if (a.L.K != b.L.K || a.L.N != b.L.N || c.L.K != a.L.N)
    fail(GLM_DIMENSION, "glmmodel", "geglu needs w1, v [d, f] and w2 [f, n]");
  DeviceBuffer ua(M * a.L.N * 4), ub(M * a.L.N * 4);
  qlinear_device(w1, x, M, ua.as<float>(), st);
  qlinear_device(v, x, M, ub.as<float>(), st);
  k_gelu_mul<<<grid_for_n(M * a.L.N, 256), 256, 0, st>>>(ua.as<float>(), ub.as<float>(), ua.as<float>(), M * a.L.N);
  LAUNCH_CHECK("k_gelu_mul");
  qlinear_device(w2, ua.as<float>(), M, y, st);
}

void attention_device(const float* q, const float* k, const float* v, int64_t n, int64_t dh, const int* positions,
                      const uint8_t* mask, float* out, cudaStream_t st) {
  if (n < 1) fail(GLM_DIMENSION, "tensorcore", "attention needs n >= 1");
  if (dh % 2) fail(GLM_CONTRACT, "tensorcore", "rope_rotate requires an even last dimension, got " + std::to_string(dh));
  const size_t smem = (static_cast<size_t>(n) + dh + 32) * 4;
  if (smem > 220 * 1024) fail(GLM_DIMENSION, "tensorcore", "attention op: n too large for one row per CTA");
  DeviceBuffer rq(n * dh * 4), rk(n * dh * 4), err(4);
  const int big = 0x7fffffff;
  CUDA_CHECK(cudaMemcpyAsync(err.ptr, &big, 4, cudaMemcpyHostToDevice, st));
  k_rope_rows<<<grid_for_n(n * dh / 2, 256), 256, 0, st>>>(q, n, dh, positions, rq.as<float>());
  k_rope_rows<<<grid_for_n(n * dh / 2, 256), 256, 0, st>>>(k, n, dh, positions, rk.as<float>());
  LAUNCH_CHECK("k_rope_rows");
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_op, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  k_attn_op<<<static_cast<unsigned>(n), kAttnOpThreads, smem, st>>>(rq.as<float>(), rk.as<float>(), v, n, dh, mask, out,
                                                                     err.as<int>());
  LAUNCH_CHECK("k_attn_op");
  int row = big;
  CUDA_CHECK(cudaMemcpyAsync(&row, err.ptr, 4, cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  if (row != big)
    fail(GLM_POLICY, "tensorcore", "softmax row " + std::to_string(row) + " is entirely -inf; no distribution is defined");
}

// host staging helper
struct Staged {
  DeviceBuffer b;
  Staged(const void* host, int64_t bytes) : b(bytes) {
    if (host && bytes) CUDA_CHECK(cudaMemcpy(b.ptr, host, bytes, cudaMemcpyHostToDevice));
  }
  template <typename T>
  T* as() { return b.as<T>(); }
};

}  // namespace
}  // namespace glm

using namespace glm;

extern "C" {

glm_status glm_deepnorm_residual(const float* x, const float* y, int64_t rows, int64_t d, double alpha,
                                 const float* gain, const float* bias, double eps, float* out, void* stream) {
  return guarded([&] {
    if (!x || !y || !gain || !bias || !out) fail(GLM_CONTRACT, "glmmodel", "null argument");
    deepnorm_device(x, y, rows, d, alpha, gain, bias, eps, out, static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_deepnorm_residual_host(const float* x, const float* y, int64_t rows, int64_t d, double alpha,
                                      const float* gain, const float* bias, double eps, float* out) {
  return guarded([&] {
    if (!x || !y || !gain || !bias || !out) fail(GLM_CONTRACT, "glmmodel", "null argument");
    Staged dx(x, rows * d * 4), dy(y, rows * d * 4), dg(gain, d * 4), db(bias, d * 4);
    deepnorm_device(dx.as<float>(), dy.as<float>(), rows, d, alpha, dg.as<float>(), db.as<float>(), eps, dx.as<float>(),
                    nullptr);
    CUDA_CHECK(cudaMemcpy(out, dx.b.ptr, rows * d * 4, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_geglu(const glm_qweight* w1, const glm_qweight* v, const glm_qweight* w2, const float* x, int64_t M,
                     float* y, void* stream) {
  return guarded([&] {
    if (!w1 || !v || !w2 || !x || !y) fail(GLM_CONTRACT, "glmmodel", "null argument");
    if (M < 1) fail(GLM_DIMENSION, "glmmodel", "M must be >= 1");
    geglu_device(w1, v, w2, x, M, y, static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_geglu_host(const glm_qweight* w1, const glm_qweight* v, const glm_qweight* w2, const float* x,
                          int64_t M, float* y) {
  return guarded([&] {
    if (!w1 || !v || !w2 || !x || !y) fail(GLM_CONTRACT, "glmmodel", "null argument");
    if (M < 1) fail(GLM_DIMENSION, "glmmodel", "M must be >= 1");
    const QWeightDev &a = qweight_dev(w1), &c = qweight_dev(w2);
    Staged dx(x, M * a.L.K * 4), dy(nullptr, M * c.L.N * 4);
    geglu_device(w1, v, w2, dx.as<float>(), M, dy.as<float>(), nullptr);
    CUDA_CHECK(cudaMemcpy(y, dy.b.ptr, M * c.L.N * 4, cudaMemcpyDeviceToHost));
  });
}

glm_status glm_attention(const float* q, const float* k, const float* v, int64_t n, int64_t dh, const int* positions,
                         const uint8_t* mask, float* out, void* stream) {
  return guarded([&] {
    if (!q || !k || !v || !positions || !mask || !out) fail(GLM_CONTRACT, "tensorcore", "null argument");
    attention_device(q, k, v, n, dh, positions, mask, out, static_cast<cudaStream_t>(stream));
  });
}

glm_status glm_attention_host(const float* q, const float* k, const float* v, int64_t n, int64_t dh,
                              const int* positions, const uint8_t* mask, float* out) {
  return guarded([&] {
    if (!q || !k || !v || !positions || !mask || !out) fail(GLM_CONTRACT, "tensorcore", "null argument");
    Staged dq(q, n * dh * 4), dk(k, n * dh * 4), dv(v, n * dh * 4), dp(positions, n * 4), dm(mask, n * n),
        dout(nullptr, n * dh * 4);
    attention_device(dq.as<float>(), dk.as<float>(), dv.as<float>(), n, dh, dp.as<int>(), dm.as<uint8_t>(),
                     dout.as<float>(), nullptr);
    CUDA_CHECK(cudaMemcpy(out, dout.b.ptr, n * dh * 4, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
