// block.cu — the GLM block around the quantized linears (glmmodel, model.cpp:125-226).
//
// All kernels keep the residual stream, the DeepNorm add and the LayerNorm statistics in
// fp32 (at N = 70 a sublayer is ~1e-5 of the residual, below any 16-bit
// epsilon). Their fp16 outputs are written straight into the tcgen05
// B-operand layout (layout.cuh) of the NEXT quantized linear, with that linear's kRow
// scale fold, so no separate activation-formatting pass exists on the decode path.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "block.h"
#include "rowstat.cuh"
#include "common.cuh"

namespace glm {

GLM_TRACE_TU(block)

namespace {

constexpr float kInvSqrt2 = 0.70710678118654752440f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Sum over ksplit partials of element n of row m, times the group scale.
__device__ __forceinline__ float reduce_partial(const SubIn& in, int m, int64_t n) {
  float acc = 0.f;
#pragma unroll 4
  for (int s = 0; s < in.ksplit; ++s) acc += in.p[static_cast<int64_t>(s) * in.split_stride + m * in.ld + n];
  acc = in.scale ? acc * in.scale[n] : acc;
  return in.zt ? acc + in.zt[m] * in.zv[n] : acc;
}


template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x < 32) {
    s = (l < NT / 32) ? red[l] : 0.f;
    s = warp_sum(s);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// ---- embedding_rows (tensor.cpp:396-412) ---------------------------------------------
template <typename ET>
__global__ void k_embed(const ET* __restrict__ E, int64_t d, const int* __restrict__ tokens, int M,
                        float* __restrict__ h, XOut xo, int half_store) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int64_t row = tokens[m];
  for (int64_t k = 2 * threadIdx.x; k < d; k += 2 * blockDim.x) {
    float v0, v1;
    if constexpr (sizeof(ET) == 4) {
      v0 = E[row * d + k];
      v1 = E[row * d + k + 1];
    } else {
      v0 = __bfloat162float(E[row * d + k]);
      v1 = __bfloat162float(E[row * d + k + 1]);
    }
    if (half_store) {
      v0 = half_round(v0);
      v1 = half_round(v1);
    }
    h[m * d + k] = v0;
    h[m * d + k + 1] = v1;
    store_xfrag_pair(xo, m, k, v0, v1);
  }
}

// Prefill variant writing tcgen05 activation tiles (k_geglu_act_tiles warp mapping: 32
// tokens x 8 features per warp).
template <typename ET>
__global__ void k_embed_tiles(const ET* __restrict__ E, int64_t d, const int* __restrict__ tokens, int M,
                              float* __restrict__ h, XOut xo, int half_store) {
  pdl_wait();
  pdl_trigger();
  constexpr int T = kXTileTokens;
  const int64_t groups = d / 8, subs = T / 32;
  const int64_t warps = (M + T - 1) / T * groups * subs;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < warps;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t sub = w % subs, rest = w / subs;
    const int64_t g = rest % groups, tile = rest / groups;
    const int64_t m = tile * T + sub * 32 + lane;
    if (m >= M) continue;
    const int64_t n = g * 8, row = tokens[m];
    float v[8];
    if constexpr (sizeof(ET) == 4) {
      const float4* p = reinterpret_cast<const float4*>(E + row * d + n);
      const float4 a = p[0], b = p[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
      const uint4 q = *reinterpret_cast<const uint4*>(E + row * d + n);
      const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wd[e]));
        v[2 * e] = f.x;
        v[2 * e + 1] = f.y;
      }
    }
    if (half_store)
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = half_round(v[e]);
    float4* hp = reinterpret_cast<float4*>(h + m * d + n);
    hp[0] = make_float4(v[0], v[1], v[2], v[3]);
    hp[1] = make_float4(v[4], v[5], v[6], v[7]);
    if (!xo.xf) continue;
    uint32_t hx[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float s0 = xo.row_scale ? xo.row_scale[n + e] : 1.f, s1 = xo.row_scale ? xo.row_scale[n + e + 1] : 1.f;
      const __half2 hv = __floats2half2_rn(v[e] * s0, v[e + 1] * s1);
      hx[e / 2] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    *reinterpret_cast<uint4*>(xo.xf + xtile_index(xo.Kp, m, n)) = make_uint4(hx[0], hx[1], hx[2], hx[3]);
  }
}

// ---- deepnorm_residual = LN(alpha * x + y) (model.cpp:125-131, tensor.cpp:256-274) -----
// One thread-block CLUSTER of kLnCluster CTAs per row: each CTA owns a contiguous slice of
// the row (pairs of features kept in registers), the mean / variance partial sums are
// exchanged through distributed shared memory (DSMEM), so a 12288-wide row is spread over
// 8 SMs instead of serialising its L2 latency on one.
constexpr int kLnCluster = 8;
constexpr int kLnThreads = 384;
constexpr int kLnPairs = 4;  // pairs per thread: d <= 2 * 4 * 384 * 8 = 24576

// CTA-wide statistics (NT threads), fixed merge order; `red` holds NT / 32 entries
template <int NT>
__device__ __forceinline__ RowStat block_stat(RowStat a, RowStat* red) {
  a = warp_stat(a);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = a;
  __syncthreads();
  RowStat t = red[0];
  for (int i = 1; i < NT / 32; ++i) t = stat_merge(t, red[i]);
  return t;
}

// Cluster-wide statistics: each CTA pushes its partial into slot[rank] of every CTA of the
// cluster (distributed shared memory stores), one cluster barrier (release/acquire), then
// every CTA merges its local slots in rank order: identical on every CTA and every run.
// One-sided variant (k_deepnorm_ln): the partial goes to every CTA with st.async, which
// completes on the destination's mbarrier; a CTA waits only for the CL arrivals on its own
// barrier (initialised and published by a cluster barrier before the dependency wait), so
// there is no cluster barrier (and no release of every earlier memory operation) on the path.
template <int CL>
__device__ __forceinline__ RowStat cluster_stat_async(RowStat v, RowStat* red, float4* slots, uint64_t* bar) {
  v = warp_stat(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    RowStat t = red[0];
    for (int i = 1; i < kLnThreads / 32; ++i) t = stat_merge(t, red[i]);
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t lbar = smem_addr(bar), lslot = smem_addr(slots + rank);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lbar), "r"(CL * 16) : "memory");
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      uint32_t rslot, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rslot) : "r"(lslot), "r"(r));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lbar), "r"(r));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                       rslot),
                   "r"(__float_as_uint(t.n)), "r"(__float_as_uint(t.mean)), "r"(__float_as_uint(t.m2)), "r"(0u), "r"(rbar)
                   : "memory");
    }
  }
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n" ::"r"(
                   smem_addr(bar))
               : "memory");
  RowStat r = RowStat{slots[0].x, slots[0].y, slots[0].z};
  for (int i = 1; i < CL; ++i) r = stat_merge(r, RowStat{slots[i].x, slots[i].y, slots[i].z});
  return r;
}

template <int CL>
__device__ __forceinline__ RowStat cluster_stat(RowStat v, RowStat* red, RowStat* slots) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  v = warp_stat(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    RowStat t = red[0];
    for (int i = 1; i < kLnThreads / 32; ++i) t = stat_merge(t, red[i]);
    const unsigned rank = cluster.block_rank();
    if (l < CL) *cluster.map_shared_rank(slots + rank, l) = t;
  }
  cluster.sync();
  RowStat r = slots[0];
  for (int i = 1; i < CL; ++i) r = stat_merge(r, slots[i]);
  return r;
}

// Tensor-parallel sum of this CTA's slice [2 p0, 2 p1) of row m (PeerArgs, block.h): push
// the rank's partial into every rank's inbox, raise the slice flag, wait for the t flags of
// this generation and sum the inbox slots in rank order (same bits on every rank). Returns
// false after a push-only launch (mode 1). A flag that does not arrive within ~20 s sets the
// error word (Collective::check_peer) instead of hanging the GPU.
static_assert(kPeerSlices >= kLnCluster, "one peer flag per LayerNorm cluster CTA");
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool peer_allreduce(const PeerArgs& P, int m, int crank, int64_t p0, int64_t p1,
                                               float2 (&y)[kLnPairs]) {
  __shared__ unsigned s_gen;
  const unsigned* genp = P.gen + m * kPeerSlices + crank;
  if (threadIdx.x == 0) s_gen = *genp + 1u;
  __syncthreads();
  const unsigned gen = s_gen;
  const int par = static_cast<int>(gen & 1u);
  const int64_t slot = static_cast<int64_t>(P.max_b) * P.d;  // one (parity, source rank) slot
  if (P.mode & 1) {
    for (int dst = 0; dst < P.size; ++dst) {
      float* box = P.inbox[dst] + static_cast<int64_t>(par * P.size + P.rank) * slot + static_cast<int64_t>(m) * P.d;
#pragma unroll
      for (int i = 0; i < kLnPairs; ++i) {
        const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
        if (p < p1) *reinterpret_cast<float2*>(box + 2 * p) = y[i];
      }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < P.size)
      st_release_sys(P.flags[threadIdx.x] + ((par * P.size + P.rank) * P.max_b + m) * kPeerSlices + crank, gen);
  }
  if (!(P.mode & 2)) return false;
  if (threadIdx.x < P.size) {
    const unsigned* f = P.flags[P.rank] + ((par * P.size + threadIdx.x) * P.max_b + m) * kPeerSlices + crank;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(f) != gen) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 20000000000ull) {
        atomicExch(P.err, 1);
        break;
      }
    }
  }
  __syncthreads();
  const float* own = P.inbox[P.rank] + static_cast<int64_t>(par * P.size) * slot + static_cast<int64_t>(m) * P.d;
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) {
    const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
    float2 acc = make_float2(0.f, 0.f);
    if (p < p1)
      for (int r = 0; r < P.size; ++r) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(own + r * slot + 2 * p));
        acc.x += v.x;
        acc.y += v.y;
      }
    y[i] = acc;
  }
  if (threadIdx.x == 0) P.gen[m * kPeerSlices + crank] = gen;
  return true;
}

// CL CTAs per row: 8 (up to 8 rows: 15 clusters of 8 are co-resident on the 148 SMs) or 4
// (9..16 rows: 16 clusters of 8 would run in two waves, ncu at 16 rows 18-21 us per launch)
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kLnThreads) k_deepnorm_ln(LnArgs a) {
  trace_point(20);
  __shared__ RowStat red[kLnThreads / 32];
  __shared__ float4 slots[CL];
  __shared__ __align__(8) uint64_t sbar;
  namespace cg = cooperative_groups;
  const int rank = static_cast<int>(cg::this_cluster().block_rank());
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cg::this_cluster().sync();  // every CTA's statistics barrier exists before any st.async (pre-wait)
  const int m = blockIdx.x / CL;
  const int64_t npairs = a.d / 2;
  const int64_t per = (npairs + CL - 1) / CL;
  const int64_t p0 = rank * per, p1 = min(npairs, p0 + per);
  // everything that does not depend on the predecessor GEMV (LN parameters, the scale
  // vector, the residual written two kernels ago) is fetched before waiting on it
  const float* __restrict__ hrow = a.h + static_cast<int64_t>(m) * a.d;
  float2 gn[kLnPairs], bs[kLnPairs], sc[kLnPairs], hv[kLnPairs];
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) {
    const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
    if (p < p1) {
      gn[i] = *reinterpret_cast<const float2*>(a.gain + 2 * p);
      bs[i] = *reinterpret_cast<const float2*>(a.bias + 2 * p);
      sc[i] = a.in.scale ? *reinterpret_cast<const float2*>(a.in.scale + 2 * p) : make_float2(1.f, 1.f);
      hv[i] = *reinterpret_cast<const float2*>(hrow + 2 * p);
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_point(21);
  // split-K partials: all loads of the thread issued back to back (4 splits per batch)
  float2 y[kLnPairs];
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) y[i] = make_float2(0.f, 0.f);
  if (!a.zero_sublayer) {
    for (int s0 = 0; s0 < a.in.ksplit; s0 += 8) {
      float2 v[8][kLnPairs];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int i = 0; i < kLnPairs; ++i) {
          const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
          v[u][i] = (s0 + u < a.in.ksplit && p < p1)
                        ? *reinterpret_cast<const float2*>(a.in.p + static_cast<int64_t>(s0 + u) * a.in.split_stride +
                                                           m * a.in.ld + 2 * p)
                        : make_float2(0.f, 0.f);
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int i = 0; i < kLnPairs; ++i) {
          y[i].x += v[u][i].x;
          y[i].y += v[u][i].y;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) {
    y[i].x *= sc[i].x;
    y[i].y *= sc[i].y;
  }
  if (a.in.zt && !a.zero_sublayer) {  // zeropoint weights: rank-1 term of this rank's rows
    const float ztm = a.in.zt[m];
#pragma unroll
    for (int i = 0; i < kLnPairs; ++i) {
      const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
      if (p < p1) {
        const float2 zv = *reinterpret_cast<const float2*>(a.in.zv + 2 * p);
        y[i].x += ztm * zv.x;
        y[i].y += ztm * zv.y;
      }
    }
  }
  if (a.peer.size > 1 && !peer_allreduce(a.peer, m, rank, p0, p1, y)) return;  // push-only launch
  if (a.half_store)
#pragma unroll
    for (int i = 0; i < kLnPairs; ++i) y[i] = make_float2(half_round(y[i].x), half_round(y[i].y));
  float2 z[kLnPairs];
  ShiftedSums st;
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) {
    const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
    z[i] = make_float2(0.f, 0.f);
    if (p < p1) {
      z[i] = make_float2(a.alpha * hv[i].x + y[i].x, a.alpha * hv[i].y + y[i].y);
      if (a.tap) *reinterpret_cast<float2*>(a.tap + static_cast<int64_t>(m) * a.d + 2 * p) = y[i];
      st.add(z[i].x);
      st.add(z[i].y);
    }
  }
  // one cluster reduction of (count, mean, M2); biased variance (tensor.cpp:267)
  trace_point(23);
  const RowStat tot = cluster_stat_async<CL>(st.stat(), red, slots, &sbar);
  trace_point(24);
  const float mean = tot.mean;
  const float var = tot.m2 / static_cast<float>(a.d);
  const float rstd = rsqrtf(var + a.eps);
#pragma unroll
  for (int i = 0; i < kLnPairs; ++i) {
    const int64_t p = p0 + threadIdx.x + static_cast<int64_t>(i) * kLnThreads;
    if (p < p1) {
      const int64_t n = 2 * p;
      float o0 = (z[i].x - mean) * rstd * gn[i].x + bs[i].x;
      float o1 = (z[i].y - mean) * rstd * gn[i].y + bs[i].y;
      if (a.half_store) {
        o0 = half_round(o0);
        o1 = half_round(o1);
      }
      *reinterpret_cast<float2*>(a.h + static_cast<int64_t>(m) * a.d + n) = make_float2(o0, o1);
      store_xfrag_pair(a.x0, m, n, o0, o1);
      store_xfrag_pair(a.x1, m, n, o0, o1);
    }
  }
  trace_point(22);
}

// Many-row variant (prefill): one CTA per row, no cluster; the row's pairs are strided over
// the CTA's threads and the statistics are a CTA reduction (fixed order).
constexpr int kLnRowThreads = 512;

__global__ void __launch_bounds__(kLnRowThreads) k_deepnorm_ln_rows(LnArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ RowStat red[kLnRowThreads / 32];
  const int m = blockIdx.x;
  const int64_t npairs = a.d / 2;
  float* hrow = a.h + static_cast<int64_t>(m) * a.d;
  ShiftedSums acc;
  // pass 1: z = alpha h + y (kept in h), statistics
  for (int64_t p = threadIdx.x; p < npairs; p += kLnRowThreads) {
    const int64_t n = 2 * p;
    float2 y = make_float2(0.f, 0.f);
    if (!a.zero_sublayer) {
      for (int s = 0; s < a.in.ksplit; ++s) {
        const float2 v = *reinterpret_cast<const float2*>(a.in.p + static_cast<int64_t>(s) * a.in.split_stride +
                                                          m * a.in.ld + n);
        y.x += v.x;
        y.y += v.y;
      }
      if (a.in.scale) {
        y.x *= a.in.scale[n];
        y.y *= a.in.scale[n + 1];
      }
      if (a.half_store) y = make_float2(half_round(y.x), half_round(y.y));
    }
    if (a.tap) *reinterpret_cast<float2*>(a.tap + static_cast<int64_t>(m) * a.d + n) = y;
    const float2 hv = *reinterpret_cast<const float2*>(hrow + n);
    const float2 z = make_float2(a.alpha * hv.x + y.x, a.alpha * hv.y + y.y);
    *reinterpret_cast<float2*>(hrow + n) = z;
    acc.add(z.x);
    acc.add(z.y);
  }
  const RowStat tot = block_stat<kLnRowThreads>(acc.stat(), red);
  const float mean = tot.mean;
  const float var = tot.m2 / static_cast<float>(a.d);  // biased (tensor.cpp:267)
  const float rstd = rsqrtf(var + a.eps);
  // pass 2 (same thread -> same pairs, so z is read back from where this thread wrote it)
  for (int64_t p = threadIdx.x; p < npairs; p += kLnRowThreads) {
    const int64_t n = 2 * p;
    const float2 z = *reinterpret_cast<const float2*>(hrow + n);
    float o0 = (z.x - mean) * rstd * a.gain[n] + a.bias[n];
    float o1 = (z.y - mean) * rstd * a.gain[n + 1] + a.bias[n + 1];
    if (a.half_store) {
      o0 = half_round(o0);
      o1 = half_round(o1);
    }
    *reinterpret_cast<float2*>(hrow + n) = make_float2(o0, o1);
    store_xfrag_pair(a.x0, m, n, o0, o1);
    store_xfrag_pair(a.x1, m, n, o0, o1);
  }
}

// 8 features per thread (two float4 per operand, one 16-byte activation-tile store): the
// same two passes with a quarter of the memory instructions (hidden % 8 == 0, aligned rows).
__device__ __forceinline__ void store_x8(const XOut& xo, int m, int64_t n, const float (&o)[8]) {
  if (!xo.xf) return;
  if (!xo.tile) {
#pragma unroll
    for (int e = 0; e < 8; e += 2) store_xfrag_pair(xo, m, n + e, o[e], o[e + 1]);
    return;
  }
  uint32_t hx[4];
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const float s0 = xo.row_scale ? xo.row_scale[n + e] : 1.f, s1 = xo.row_scale ? xo.row_scale[n + e + 1] : 1.f;
    const __half2 hv = __floats2half2_rn(o[e] * s0, o[e + 1] * s1);
    hx[e / 2] = *reinterpret_cast<const uint32_t*>(&hv);
  }
  *reinterpret_cast<uint4*>(xo.xf + xtile_index(xo.Kp, m, n)) = make_uint4(hx[0], hx[1], hx[2], hx[3]);
}
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

template <int MINB>
__global__ void __launch_bounds__(kLnRowThreads, MINB) k_deepnorm_ln_rows8(LnArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ RowStat red[kLnRowThreads / 32];
  const int m = blockIdx.x;
  const int64_t nv = a.d / 8;
  float* hrow = a.h + static_cast<int64_t>(m) * a.d;
  ShiftedSums acc;
  for (int64_t p = threadIdx.x; p < nv; p += kLnRowThreads) {
    const int64_t n = 8 * p;
    float y[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (!a.zero_sublayer) {
      for (int s = 0; s < a.in.ksplit; ++s) {
        float v[8];
        ld8(a.in.p + static_cast<int64_t>(s) * a.in.split_stride + m * a.in.ld + n, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] += v[e];
      }
      if (a.in.scale)
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] *= a.in.scale[n + e];
      if (a.half_store)
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = half_round(y[e]);
    }
    if (a.tap) st8(a.tap + static_cast<int64_t>(m) * a.d + n, y);
    float z[8];
    ld8(hrow + n, z);
#pragma unroll
    for (int e = 0; e < 8; ++e) z[e] = a.alpha * z[e] + y[e];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc.add(z[e]);
    st8(hrow + n, z);
  }
  const RowStat tot = block_stat<kLnRowThreads>(acc.stat(), red);
  const float mean = tot.mean;
  const float var = tot.m2 / static_cast<float>(a.d);  // biased (tensor.cpp:267)
  const float rstd = rsqrtf(var + a.eps);
  for (int64_t p = threadIdx.x; p < nv; p += kLnRowThreads) {
    const int64_t n = 8 * p;
    float z[8], g[8], b[8];
    ld8(hrow + n, z);
    ld8(a.gain + n, g);
    ld8(a.bias + n, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) z[e] = (z[e] - mean) * rstd * g[e] + b[e];
    if (a.half_store)
#pragma unroll
      for (int e = 0; e < 8; ++e) z[e] = half_round(z[e]);
    st8(hrow + n, z);
    store_x8(a.x0, m, n, z);
    store_x8(a.x1, m, n, z);
  }
}

// ---- GeGLU activation: gelu(x W1) * (x V) (model.cpp:133-135, tensor.cpp:313-318) --------
__device__ __forceinline__ float2 reduce_partial2(const SubIn& in, int m, int64_t n) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
  for (int s = 0; s < in.ksplit; ++s) {
    const float2 v = *reinterpret_cast<const float2*>(in.p + static_cast<int64_t>(s) * in.split_stride + m * in.ld + n);
    acc.x += v.x;
    acc.y += v.y;
  }
  if (in.scale) {
    acc.x *= in.scale[n];
    acc.y *= in.scale[n + 1];
  }
  if (in.zt) {
    acc.x += in.zt[m] * in.zv[n];
    acc.y += in.zt[m] * in.zv[n + 1];
  }
  return acc;
}

// scalar form for an odd feature count (e.g. ffn 1368 over 8 ranks = 171 per rank) or odd row
// strides: feature n + 1 == f reads as 0 (the consumer's padded k)
__device__ __forceinline__ float2 reduce_partial2_any(const SubIn& in, int m, int64_t n, int64_t f) {
  return make_float2(reduce_partial(in, m, n), n + 1 < f ? reduce_partial(in, m, n + 1) : 0.f);
}

template <bool V2>
__global__ void k_geglu_act(ActArgs a) {
  trace_point(40);
  pdl_wait();
  pdl_trigger();
  trace_point(41);
  const int64_t half = (a.f + 1) / 2;
  const int64_t pairs = static_cast<int64_t>(a.M) * half;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / half);
    const int64_t n = (i % half) * 2;
    const float2 u = V2 ? reduce_partial2(a.w1, m, n) : reduce_partial2_any(a.w1, m, n, a.f);
    const float2 v = V2 ? reduce_partial2(a.v, m, n) : reduce_partial2_any(a.v, m, n, a.f);
    const float o0 = 0.5f * u.x * (1.f + erff(u.x * kInvSqrt2)) * v.x;  // tensor.cpp:313-318
    const float o1 = 0.5f * u.y * (1.f + erff(u.y * kInvSqrt2)) * v.y;
    store_xfrag_pair(a.xo, m, n, o0, o1);
  }
  trace_point(42);
}

// GeGLU into tcgen05 activation tiles (prefill, xo.tile): a warp covers 32 consecutive tokens
// x one 8-feature group, so each lane reads 32 B runs of its w1 / v rows and the warp
// writes one contiguous 512 B block of the tile layout (the pair-per-thread kernel above
// scatters 4-byte stores 8·T halves apart there: ~3x slower on 8192 x 32768).
__device__ __forceinline__ void load8(const SubIn& in, int m, int64_t n, float (&o)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = 0.f;
  for (int s = 0; s < in.ksplit; ++s) {
    const float4* p = reinterpret_cast<const float4*>(in.p + static_cast<int64_t>(s) * in.split_stride + m * in.ld + n);
    const float4 a = p[0], b = p[1];
    o[0] += a.x; o[1] += a.y; o[2] += a.z; o[3] += a.w;
    o[4] += b.x; o[5] += b.y; o[6] += b.z; o[7] += b.w;
  }
  if (in.scale)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] *= in.scale[n + e];
  if (in.zt)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] += in.zt[m] * in.zv[n + e];
}

__global__ void k_geglu_act_tiles(ActArgs a) {
  pdl_wait();
  pdl_trigger();
  const int T = a.xo.tile ? kXTileTokens : 1;
  const int64_t groups = a.f / 8, subs = T / 32;
  const int64_t tiles = (a.M + T - 1) / T;
  const int64_t warps = tiles * groups * subs;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < warps;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t sub = w % subs, rest = w / subs;
    const int64_t g = rest % groups, tile = rest / groups;
    const int64_t m = tile * T + sub * 32 + lane;
    if (m >= a.M) continue;
    const int64_t n = g * 8;
    float u[8], v[8];
    load8(a.w1, static_cast<int>(m), n, u);
    load8(a.v, static_cast<int>(m), n, v);
    uint32_t h[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      float o0 = 0.5f * u[e] * (1.f + erff(u[e] * kInvSqrt2)) * v[e];  // tensor.cpp:313-318
      float o1 = 0.5f * u[e + 1] * (1.f + erff(u[e + 1] * kInvSqrt2)) * v[e + 1];
      if (a.xo.row_scale) {
        o0 *= a.xo.row_scale[n + e];
        o1 *= a.xo.row_scale[n + e + 1];
      }
      const __half2 hv = __floats2half2_rn(o0, o1);
      h[e / 2] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    *reinterpret_cast<uint4*>(a.xo.xf + xtile_index(a.xo.Kp, m, n)) = make_uint4(h[0], h[1], h[2], h[3]);
  }
}

// ---- decode attention (model.cpp:137-152 for the rows of the generation part) ----------
// grid (heads, batch, splits); each CTA owns split_keys (256, or 64 for caches longer than
// 256 tokens) consecutive keys of its sequence's cache, so up to 256 cached tokens need no
// cross-CTA merge at all. Before the
// programmatic-dependency wait (the qkv GEMV is still running) the CTA prefetches its
// cached K/V rows into L2; after it, q (and the new k, v) are reduced from the GEMV's
// split-K partials and rotated (RoPE), scores use DH/8 lanes per key (one 16-byte load
// each), softmax is fp32, P.V has lanes own DH/32 features with 8 independent row loads in
// flight, and the new key/value enter from shared memory. With several splits, the last
// CTA of a (head, batch) merges them in split order (deterministic).
constexpr int kAttnThreadsFew = 256;  // threads per CTA at batch <= 2 (few CTAs)
constexpr int kAttnThreadsMany = 128;  // larger batches: more resident CTAs per SM
constexpr int kSplitKeys = 256;    // largest split (size of the score buffer)
constexpr int kSplitKeysLong = 64;  // split of caches longer than kSplitKeys

template <int DH, int kAttnThreads>
__global__ void __launch_bounds__(kAttnThreads, kAttnThreads == 128 ? 12 : 1)
    k_attn_decode(AttnDecodeArgs a) {
  trace_point(30);
  constexpr int NW = kAttnThreads / 32;
  constexpr int FPL = DH / 32;          // features per lane in the PV phase
  constexpr int LPK = DH / 8, KPW = 32 / LPK;
  __shared__ float q[DH];
  __shared__ float p[kSplitKeys];
  __shared__ float red[NW];
  __shared__ float opart[NW][DH];
  __shared__ int last;
  __shared__ __align__(8) uint64_t kvbar;
  __shared__ __align__(16) __half knew[DH];       // the new key / value (unstaged mode)
  __shared__ __align__(16) __half vnew[DH];
  extern __shared__ __align__(128) __half kvs[];  // [2][stage_keys][DH]: this split's keys, values
  const bool staged = a.stage_keys > 0;
  __half* kst = kvs;
  __half* vst = kvs + a.stage_keys * DH;
  const int head = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cache length / position were written by earlier steps (complete before our predecessor ran)
  const int len = a.cache_len[b];
  const int total = len + 1;
  const int k0 = split * a.split_keys, k1 = min(total, k0 + a.split_keys);
  const int kold = min(k1, len);  // cached keys of this split: [k0, kold)
  const int pos = a.positions[b];
  const float inv_sqrt = rsqrtf(static_cast<float>(DH));
  __half* kc = a.kcache + ((static_cast<int64_t>(b) * a.heads + head) * a.max_ctx) * DH;
  __half* vc = a.vcache + ((static_cast<int64_t>(b) * a.heads + head) * a.max_ctx) * DH;
  float* part = a.part + ((static_cast<int64_t>(b) * a.heads + head) * a.max_splits + split) * (DH + 2);
  // The cached rows of this split do not depend on the running qkv GEMV: one bulk copy
  // each for K and V into shared memory, issued before the dependency wait.
  const int n_old = max(0, kold - k0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&kvbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (staged && n_old > 0) {
      const uint32_t bytes = static_cast<uint32_t>(n_old) * DH * 2;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&kvbar)), "r"(2 * bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(kst)),
                   "l"(kc + static_cast<int64_t>(k0) * DH), "r"(bytes), "r"(smem_addr(&kvbar))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(vst)),
                   "l"(vc + static_cast<int64_t>(k0) * DH), "r"(bytes), "r"(smem_addr(&kvbar))
                   : "memory");
    }
  }
  __syncthreads();  // the barrier is initialised before any thread waits on it
  // RoPE factors and the qkv column scales do not depend on the running GEMV either
  const int jt = threadIdx.x < DH / 2 ? threadIdx.x : threadIdx.x - DH / 2;
  float2 cs = make_float2(1.f, 0.f), sq = make_float2(1.f, 1.f), sk = sq, sv = sq;
  if (threadIdx.x < DH) {
    cs = a.rope[static_cast<int64_t>(pos) * (DH / 2) + jt];  // (cos, sin), tensor.cpp:357-363
    const int64_t fq = static_cast<int64_t>(head) * DH + 2 * jt;
    if (a.qkv.scale) {
      sq = *reinterpret_cast<const float2*>(a.qkv.scale + fq);
      sk = *reinterpret_cast<const float2*>(a.qkv.scale + a.d_local + fq);
      sv = *reinterpret_cast<const float2*>(a.qkv.scale + 2 * a.d_local + fq);
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_point(31);

  if (k0 < total) {
    const bool has_new = (len >= k0 && len < k1);
    auto raw2 = [&](int64_t f) {  // split-K sum of columns (f, f+1), unscaled; 8 loads in flight
      float2 acc = make_float2(0.f, 0.f);
      for (int s0 = 0; s0 < a.qkv.ksplit; s0 += 8) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = s0 + u < a.qkv.ksplit
                     ? *reinterpret_cast<const float2*>(a.qkv.p + static_cast<int64_t>(s0 + u) * a.qkv.split_stride +
                                                        b * a.qkv.ld + f)
                     : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += v[u].x;
          acc.y += v[u].y;
        }
      }
      return acc;
    };
    // q pairs on threads [0, DH/2), the new key/value pair on threads [DH/2, DH)
    if (threadIdx.x < DH) {
      const int j = threadIdx.x;
      const int jj = jt;
      const int64_t fq = static_cast<int64_t>(head) * DH + 2 * jj;
      // zeropoint weights: y += zt[b] * zv (after the column scale)
      auto zp2 = [&](int64_t f) {
        return a.qkv.zt ? make_float2(a.qkv.zt[b] * a.qkv.zv[f], a.qkv.zt[b] * a.qkv.zv[f + 1]) : make_float2(0.f, 0.f);
      };
      if (j < DH / 2) {
        const float2 qv = raw2(fq), qz = zp2(fq);
        const float qa = qv.x * sq.x + qz.x, qb = qv.y * sq.y + qz.y;
        q[2 * jj] = (cs.x * qa - cs.y * qb) * inv_sqrt;
        q[2 * jj + 1] = (cs.y * qa + cs.x * qb) * inv_sqrt;
      } else if (has_new) {
        const int64_t fk = a.d_local + fq, fv = 2 * a.d_local + fq;
        const float2 kv2 = raw2(fk), vv2 = raw2(fv), kz = zp2(fk), vz = zp2(fv);
        const float ka = kv2.x * sk.x + kz.x, kb = kv2.y * sk.y + kz.y;
        const float va = vv2.x * sv.x + vz.x, vb = vv2.y * sv.y + vz.y;
        const __half2 kh = __floats2half2_rn(cs.x * ka - cs.y * kb, cs.y * ka + cs.x * kb);
        const __half2 vh = __floats2half2_rn(va, vb);
        *reinterpret_cast<__half2*>(kc + static_cast<int64_t>(len) * DH + 2 * jj) = kh;
        *reinterpret_cast<__half2*>(vc + static_cast<int64_t>(len) * DH + 2 * jj) = vh;
        if (staged) {
          *reinterpret_cast<__half2*>(kst + (len - k0) * DH + 2 * jj) = kh;
          *reinterpret_cast<__half2*>(vst + (len - k0) * DH + 2 * jj) = vh;
        } else {
          *reinterpret_cast<__half2*>(knew + 2 * jj) = kh;
          *reinterpret_cast<__half2*>(vnew + 2 * jj) = vh;
        }
      }
    }
    if (staged && n_old > 0)
      asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n" ::"r"(
                       smem_addr(&kvbar))
                   : "memory");
    __syncthreads();
    trace_point(33);
    // ---- scores: LPK lanes per key, one 16-byte load each ----
    const int sub = lane % LPK, kin = lane / LPK;
    float qr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qr[i] = q[sub * 8 + i];
    auto dot8 = [&](uint4 kv) {
      const uint32_t w4[4] = {kv.x, kv.y, kv.z, kv.w};
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[e]));
        acc += qr[2 * e] * f.x + qr[2 * e + 1] * f.y;
      }
      return acc;
    };
    constexpr int SU = 4;  // key groups in flight per warp
    for (int s0 = k0 + warp * KPW; s0 < k1; s0 += NW * KPW * SU) {
      uint4 kv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int s = s0 + u * NW * KPW + kin;
        const __half* kr = staged ? kst + (s - k0) * DH : (s < kold ? kc + static_cast<int64_t>(s) * DH : knew);
        kv[u] = s < k1 ? (staged || s >= kold ? *reinterpret_cast<const uint4*>(kr + sub * 8)
                                             : ld_nc(reinterpret_cast<const uint4*>(kr + sub * 8)))
                       : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int s = s0 + u * NW * KPW + kin;
        float acc = dot8(kv[u]);
#pragma unroll
        for (int o = LPK / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        // half-emulated storage: scores held as fp16(score / prescale), softmax multiplies back
        if (a.prescale > 0.f) acc = half_round(acc / a.prescale) * a.prescale;
        if (sub == 0 && s < k1) p[s - k0] = acc;
      }
    }
    __syncthreads();
    trace_point(34);
    // ---- softmax over the split (fp32) ----
    float mx = -FLT_MAX;
    for (int s = threadIdx.x; s < k1 - k0; s += kAttnThreads) mx = fmaxf(mx, p[s]);
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();
    float sum = 0.f;
    for (int s = threadIdx.x; s < k1 - k0; s += kAttnThreads) {
      const float e = __expf(p[s] - mx);
      p[s] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    sum = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) sum += red[w];
    // ---- P.V: warp w takes keys k0+w, k0+w+NW, ...; lane owns FPL features ----
    float o[FPL];
#pragma unroll
    for (int f = 0; f < FPL; ++f) o[f] = 0.f;
    constexpr int U = 8;
    for (int s0 = k0 + warp; s0 < k1; s0 += NW * U) {
      uint2 vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * NW;
        const __half* vr = (staged ? vst + (s - k0) * DH : (s < kold ? vc + static_cast<int64_t>(s) * DH : vnew)) +
                           lane * FPL;
        if (s < k1) {
          if constexpr (FPL == 4) vv[u] = *reinterpret_cast<const uint2*>(vr);
          else vv[u] = make_uint2(*reinterpret_cast<const uint32_t*>(vr), 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * NW;
        if (s < k1) {
          const float pw = p[s - k0];
          const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&vv[u].x));
          o[0] += pw * f0.x;
          o[1] += pw * f0.y;
          if constexpr (FPL == 4) {
            const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&vv[u].y));
            o[2] += pw * f1.x;
            o[3] += pw * f1.y;
          }
        }
      }
    }
#pragma unroll
    for (int f = 0; f < FPL; ++f) opart[warp][lane * FPL + f] = o[f];
    __syncthreads();
    trace_point(35);
    if (total <= a.split_keys) {
      // single active split: normalise and hand the row to out_proj directly
      const float inv = 1.f / sum;
      for (int c2 = threadIdx.x; c2 < DH / 2; c2 += kAttnThreads) {
        float o0 = 0.f, o1 = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          o0 += opart[w][2 * c2];
          o1 += opart[w][2 * c2 + 1];
        }
        const int64_t k = static_cast<int64_t>(head) * DH + 2 * c2;
        store_xfrag_pair(a.xo, b, k, o0 * inv, o1 * inv);
        if (a.out) {
          a.out[static_cast<int64_t>(b) * a.heads * DH + k] = o0 * inv;
          a.out[static_cast<int64_t>(b) * a.heads * DH + k + 1] = o1 * inv;
        }
      }
      trace_point(32);
      return;
    }
    for (int c = threadIdx.x; c < DH; c += kAttnThreads) {
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += opart[w][c];
      part[c] = acc;
    }
    if (threadIdx.x == 0) {
      part[DH] = mx;
      part[DH + 1] = sum;
    }
  } else {
    return;  // beyond the cache: no keys, not counted (the merge takes the active splits)
  }
  // ---- the last of the active splits of this (head, b) merges them in order ----
  const int nsp = (total + a.split_keys - 1) / a.split_keys;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* ctr = a.counters + b * a.heads + head;
    last = (atomicAdd(ctr, 1) == nsp - 1);
    if (last) *ctr = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* base = a.part + ((static_cast<int64_t>(b) * a.heads + head) * a.max_splits) * (DH + 2);
  // split weights exp(m_s - max) / sum_s l_s exp(m_s - max), one warp, splits in a fixed order
  float* wsp = p;  // the score buffer is free now (nsp <= kSplitKeys)
  if (warp == 0) {
    float gm = -FLT_MAX;
    for (int s = lane; s < nsp; s += 32) gm = fmaxf(gm, __ldcg(base + s * (DH + 2) + DH));
    gm = warp_max(gm);
    float gl = 0.f;
    for (int s = lane; s < nsp; s += 32) {
      const float w = __expf(__ldcg(base + s * (DH + 2) + DH) - gm);
      wsp[s] = w;
      gl += __ldcg(base + s * (DH + 2) + DH + 1) * w;
    }
    gl = warp_sum(gl);
    const float inv = 1.f / gl;
    for (int s = lane; s < nsp; s += 32) wsp[s] *= inv;
  }
  __syncthreads();
  for (int c2 = threadIdx.x; c2 < DH / 2; c2 += kAttnThreads) {
    float o0 = 0.f, o1 = 0.f;
#pragma unroll 8
    for (int s = 0; s < nsp; ++s) {
      const float w = wsp[s];
      const float2 v = __ldcg(reinterpret_cast<const float2*>(base + s * (DH + 2) + 2 * c2));
      o0 += w * v.x;
      o1 += w * v.y;
    }
    const int64_t k = static_cast<int64_t>(head) * DH + 2 * c2;
    store_xfrag_pair(a.xo, b, k, o0, o1);
    if (a.out) {
      a.out[static_cast<int64_t>(b) * a.heads * DH + k] = o0;
      a.out[static_cast<int64_t>(b) * a.heads * DH + k + 1] = o1;
    }
  }
  trace_point(32);
}

// Cache length bookkeeping after a decode step (kept on the device for CUDA graphs).
__global__ void k_advance(int* __restrict__ cache_len, int B) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) cache_len[b] += 1;
}

// ---- prefill attention (model.cpp:137-152 over a whole [gMASK] sample) -------------------
// RoPE + KV-cache write for all rows, then one CTA per (head, query row block) computes
// softmax(q k^T / sqrt(dh) + mask) v with the blank-infilling visibility
// key j visible to query i  <=>  j < max(C, i + 1)   (corruption.cpp:338-367, gMASK).
__global__ void k_rope_store(RopeStoreArgs a) {
  // grid (n rows, heads); threads over pairs
  const int i = blockIdx.x, head = blockIdx.y, half = a.dh / 2;
  const int pos = a.positions[i];
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const float2 cs = a.rope[static_cast<int64_t>(pos) * half + j];
    const int64_t fq = static_cast<int64_t>(head) * a.dh + 2 * j;
    const float* row = a.qkv + static_cast<int64_t>(i) * a.ldqkv;
    const float qa = row[fq], qb = row[fq + 1];
    const float ka = row[a.d_local + fq], kb = row[a.d_local + fq + 1];
    const float va = row[2 * a.d_local + fq], vb = row[2 * a.d_local + fq + 1];
    const int64_t q_off = (static_cast<int64_t>(head) * a.n + i) * a.dh + 2 * j;
    a.q[q_off] = cs.x * qa - cs.y * qb;
    a.q[q_off + 1] = cs.y * qa + cs.x * qb;
    const int64_t c_off = ((static_cast<int64_t>(a.seq) * a.heads + head) * a.max_ctx + a.slot0 + i) * a.dh + 2 * j;
    *reinterpret_cast<__half2*>(a.kcache + c_off) = __floats2half2_rn(cs.x * ka - cs.y * kb, cs.y * ka + cs.x * kb);
    *reinterpret_cast<__half2*>(a.vcache + c_off) = __floats2half2_rn(va, vb);
  }
}

// head_dim 128: one warp per (row, head), a lane owns 4 features (two rotation pairs) of q,
// k and v (16-byte loads, 8-byte cache stores), 8 heads per 256-thread CTA.
__device__ __forceinline__ float4 ld4f(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4f(const __half* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
template <typename T>
__global__ void k_rope_store128(RopeStoreArgs a, const T* __restrict__ qkv) {
  const int i = blockIdx.x, head = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (head >= a.heads) return;
  const int pos = a.positions[i];
  const float4 cs = reinterpret_cast<const float4*>(a.rope + static_cast<int64_t>(pos) * 64)[lane];  // pairs 2l, 2l+1
  const T* row = qkv + static_cast<int64_t>(i) * a.ldqkv + static_cast<int64_t>(head) * 128 + 4 * lane;
  const float4 q = ld4f(row);
  const float4 k = ld4f(row + a.d_local);
  const float4 v = ld4f(row + 2 * a.d_local);
  *reinterpret_cast<float4*>(a.q + (static_cast<int64_t>(head) * a.n + i) * 128 + 4 * lane) =
      make_float4(cs.x * q.x - cs.y * q.y, cs.y * q.x + cs.x * q.y, cs.z * q.z - cs.w * q.w, cs.w * q.z + cs.z * q.w);
  const int64_t c_off = ((static_cast<int64_t>(a.seq) * a.heads + head) * a.max_ctx + a.slot0 + i) * 128 + 4 * lane;
  const __half2 k0 = __floats2half2_rn(cs.x * k.x - cs.y * k.y, cs.y * k.x + cs.x * k.y);
  const __half2 k1 = __floats2half2_rn(cs.z * k.z - cs.w * k.w, cs.w * k.z + cs.z * k.w);
  const __half2 v0 = __floats2half2_rn(v.x, v.y), v1 = __floats2half2_rn(v.z, v.w);
  *reinterpret_cast<uint2*>(a.kcache + c_off) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&k0), *reinterpret_cast<const uint32_t*>(&k1));
  *reinterpret_cast<uint2*>(a.vcache + c_off) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&v0), *reinterpret_cast<const uint32_t*>(&v1));
}

// Tensor-core flash attention for prefill (FA2 schedule on mma.sync.m16n8k16, fp16 in,
// fp32 accumulate): a CTA owns 64 query rows of one head (16 per warp), streams 64-key
// blocks of K and V through double-buffered shared memory (cp.async), keeps S = Q K^T,
// the online-softmax state and O in registers, and feeds P straight from the S
// accumulators into the P.V MMA. Key blocks wholly invisible to the CTA's rows are never
// loaded; the gMASK rule j < max(C, i + 1) is applied element-wise only on blocks that
// straddle it. exp2 with log2(e) folded into the Q scale (same softmax).
constexpr int kFaRows = 64, kFaKeys = 64, kFaThreads = 128;


__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// Occupancy: Q lives in shared memory only until its fragments are in registers, so it
// shares the second V buffer (first filled for key block 1, after the Q fragments are
// loaded) and three 4-warp CTAs fit per SM (registers capped at 170 per thread).
template <int DH>
__global__ void __launch_bounds__(kFaThreads, DH == 128 ? 3 : 4) k_attn_prefill_tc(AttnPrefillArgs a) {
  constexpr int LDS = DH + 8;  // padded row (halves): ldmatrix rows land in distinct banks
  extern __shared__ __align__(16) __half fsm[];
  __half* Ks = fsm;                        // [2][64][LDS]
  __half* Vs = Ks + 2 * kFaKeys * LDS;     // [2][64][LDS]
  __half* Qs = Vs + kFaKeys * LDS;         // [64][LDS], aliases V buffer 1 (kFaRows == kFaKeys)
  const int head = blockIdx.y, i0 = blockIdx.x * kFaRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n = a.n, C = a.context_len;
  const __half* kc = a.kcache + ((static_cast<int64_t>(a.seq) * a.heads + head) * a.max_ctx) * DH;
  const __half* vc = a.vcache + ((static_cast<int64_t>(a.seq) * a.heads + head) * a.max_ctx) * DH;
  // keys visible to some row of this block: j < max(C, i0 + 64) (and j < n)
  const int kend = min(n, max(C, i0 + kFaRows));
  const int nblk = (kend + kFaKeys - 1) / kFaKeys;
  auto load_kv = [&](int blk, int buf) {
    const int j0 = blk * kFaKeys;
    constexpr int CPR = DH / 8;  // 16-byte chunks per row
    for (int c = threadIdx.x; c < kFaKeys * CPR; c += kFaThreads) {
      const int r = c / CPR, cc = (c % CPR) * 8;
      const int j = j0 + r;
      const bool ok = j < kend;
      const int64_t off = static_cast<int64_t>(ok ? j : 0) * DH + cc;
      cp_async16(Ks + (buf * kFaKeys + r) * LDS + cc, kc + off, ok);
      cp_async16(Vs + (buf * kFaKeys + r) * LDS + cc, vc + off, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  static_assert(kFaRows == kFaKeys, "Q aliases one V buffer");
  load_kv(0, 0);
  // Q (fp32, rotated) -> fp16, pre-scaled by log2(e) / sqrt(dh)
  const float qs = 1.4426950408889634f * rsqrtf(static_cast<float>(DH));
  for (int c = threadIdx.x; c < kFaRows * DH / 2; c += kFaThreads) {
    const int r = c / (DH / 2), cc = (c % (DH / 2)) * 2;
    const int i = i0 + r;
    float2 v = make_float2(0.f, 0.f);
    if (i < n) v = *reinterpret_cast<const float2*>(a.q + (static_cast<int64_t>(head) * n + i) * DH + cc);
    *reinterpret_cast<__half2*>(Qs + r * LDS + cc) = __floats2half2_rn(v.x * qs, v.y * qs);
  }
  __syncthreads();
  uint32_t qa[DH / 16][4];
#pragma unroll
  for (int kt = 0; kt < DH / 16; ++kt)
    ldsm_x4(qa[kt][0], qa[kt][1], qa[kt][2], qa[kt][3],
            Qs + (warp * 16 + (lane & 15)) * LDS + kt * 16 + (lane >> 4) * 8);
  __syncthreads();  // every warp holds its Q fragments: V buffer 1 may be filled
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int rowA = i0 + warp * 16 + g, rowB = rowA + 8;
  const int limA = max(C, rowA + 1), limB = max(C, rowB + 1);
  for (int blk = 0; blk < nblk; ++blk) {
    const int buf = blk & 1;
    if (blk + 1 < nblk) {
      load_kv(blk + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const __half* Kb = Ks + buf * kFaKeys * LDS;
    const __half* Vb = Vs + buf * kFaKeys * LDS;
    // ---- S = Q K^T (16 x 64 per warp) ----
    float sc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
    for (int kt = 0; kt < DH / 16; ++kt) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of key n-tiles
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3;
        ldsm_x4(b0, b1, b2, b3, Kb + (np * 16 + (mi >> 1) * 8 + (lane & 7)) * LDS + kt * 16 + (mi & 1) * 8);
        mma_f16(sc[2 * np], qa[kt][0], qa[kt][1], qa[kt][2], qa[kt][3], b0, b1);
        mma_f16(sc[2 * np + 1], qa[kt][0], qa[kt][1], qa[kt][2], qa[kt][3], b2, b3);
      }
    }
    // half-emulated storage: scores (log2 units here) held as fp16(score / prescale)
    if (a.prescale > 0.f) {
      const float to = 0.6931471805599453f / a.prescale, back = a.prescale * 1.4426950408889634f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[nt][e] = half_round(sc[nt][e] * to) * back;
    }
    // ---- gMASK visibility on blocks that straddle it ----
    const int j0 = blk * kFaKeys;
    if (j0 + kFaKeys > min(limA, limB) || j0 + kFaKeys > n) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = j0 + nt * 8 + 2 * t + (e & 1);
          const int lim = (e >> 1) ? limB : limA;
          if (j >= lim || j >= n) sc[nt][e] = -INFINITY;
        }
    }
    // ---- online softmax (rows g and g + 8 of the warp's 16) ----
    float bm[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      bm[0] = fmaxf(bm[0], fmaxf(sc[nt][0], sc[nt][1]));
      bm[1] = fmaxf(bm[1], fmaxf(sc[nt][2], sc[nt][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      bm[r] = fmaxf(bm[r], __shfl_xor_sync(0xffffffffu, bm[r], 1));
      bm[r] = fmaxf(bm[r], __shfl_xor_sync(0xffffffffu, bm[r], 2));
    }
    float corr[2], mnew[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mrow[r], bm[r]);
      corr[r] = exp2f(mrow[r] - mnew[r]);  // 0 on the first block (mrow = -inf)
      mrow[r] = mnew[r];
      lrow[r] *= corr[r];
    }
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    uint32_t pa[4][4];  // P as the A operand of P.V, one k-tile per 16 keys
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(sc[nt][0] - mnew[0]), p1 = exp2f(sc[nt][1] - mnew[0]);
      const float p2 = exp2f(sc[nt][2] - mnew[1]), p3 = exp2f(sc[nt][3] - mnew[1]);
      lrow[0] += p0 + p1;
      lrow[1] += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_h2(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_h2(p2, p3);
    }
    // ---- O += P V ----
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {  // pairs of dh n-tiles
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3;
        ldsm_x4_t(b0, b1, b2, b3, Vb + (kk * 16 + (mi & 1) * 8 + (lane & 7)) * LDS + dp * 16 + (mi >> 1) * 8);
        mma_f16(o[2 * dp], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
        mma_f16(o[2 * dp + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
      }
    }
    __syncthreads();  // buffer `buf` is refilled two blocks later
  }
  // ---- normalise and store ----
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const int c = head * DH + i * 8 + 2 * t;
    if (rowA < n)
      *reinterpret_cast<float2*>(a.out + static_cast<int64_t>(rowA) * a.ldout + c) =
          make_float2(o[i][0] * inv0, o[i][1] * inv0);
    if (rowB < n)
      *reinterpret_cast<float2*>(a.out + static_cast<int64_t>(rowB) * a.ldout + c) =
          make_float2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

// x_frag from an fp32 [M][K] matrix (row stride ld) for the next linear.
__global__ void k_rows_to_xfrag(const float* __restrict__ x, int64_t ld, int M, int64_t K, XOut xo) {
  const int64_t pairs = static_cast<int64_t>(M) * (K / 2);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / (K / 2));
    const int64_t k = (i % (K / 2)) * 2;
    store_xfrag_pair(xo, m, k, x[m * ld + k], x[m * ld + k + 1]);
  }
}

// fp32 rows -> tcgen05 activation tiles with the warp mapping of k_geglu_act_tiles
// (32 consecutive tokens x one 8-feature group per warp: 32 B reads, 512 B of contiguous
// tile per warp store).
__global__ void k_rows_to_xtile(const float* __restrict__ x, int64_t ld, int M, int64_t K, XOut xo) {
  constexpr int T = kXTileTokens;
  const int64_t groups = K / 8, subs = T / 32;
  const int64_t warps = (M + T - 1) / T * groups * subs;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < warps;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t sub = w % subs, rest = w / subs;
    const int64_t g = rest % groups, tile = rest / groups;
    const int64_t m = tile * T + sub * 32 + lane;
    if (m >= M) continue;
    const int64_t n = g * 8;
    const float4* p = reinterpret_cast<const float4*>(x + m * ld + n);
    const float4 a = p[0], b = p[1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t h[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float s0 = xo.row_scale ? xo.row_scale[n + e] : 1.f, s1 = xo.row_scale ? xo.row_scale[n + e + 1] : 1.f;
      const __half2 hv = __floats2half2_rn(v[e] * s0, v[e + 1] * s1);
      h[e / 2] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    *reinterpret_cast<uint4*>(xo.xf + xtile_index(xo.Kp, m, n)) = make_uint4(h[0], h[1], h[2], h[3]);
  }
}

// ---- tied output head logits = h E^T + greedy argmax (model.cpp:225) -----------------------
// HBM-bound stream over the (unquantised, quant.cpp:289) embedding table: one warp per
// vocab row, each lane keeps kHeadU independent 16-byte loads in flight, fp32 FMA against
// up to kHeadRowsPerGroup rows of h held in shared memory. Argmax keys are packed
// (value, ~index) so atomicMax picks the largest logit and, on ties, the smallest id.
constexpr int kHeadThreads = 256;
constexpr int kHeadRowsPerGroup = 4;
constexpr int kHeadU = 6;

__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  // NaN of either sign maps to the top key so a non-finite row always shows up in its winner
  uint32_t u = (v != v) ? 0x7FFFFFFFu : __float_as_uint(v);
  u = (u >> 31) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(idx));
}

template <typename ET, int MG>
__device__ __forceinline__ void head_rows(const HeadArgs& a, const float* hs, int m0, int warp, int lane) {
  constexpr int EPL = 16 / sizeof(ET);            // elements per 16-byte load
  constexpr int STEP = 32 * EPL;                  // k advanced per warp load
  const ET* E = static_cast<const ET*>(a.E);
  unsigned long long best[MG];
#pragma unroll
  for (int r = 0; r < MG; ++r) best[r] = 0ull;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kHeadThreads / 32);
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * (kHeadThreads / 32) + warp; v < a.vocab_local; v += nwarps) {
    float acc[MG];
#pragma unroll
    for (int r = 0; r < MG; ++r) acc[r] = 0.f;
    const uint4* er = reinterpret_cast<const uint4*>(E + (a.vocab_offset + v) * a.d);
    for (int64_t k0 = 0; k0 < a.d; k0 += STEP * kHeadU) {
      uint4 raw[kHeadU];
#pragma unroll
      for (int u = 0; u < kHeadU; ++u) {
        const int64_t k = k0 + u * STEP + lane * EPL;
        raw[u] = k < a.d ? ld_stream(er + k / EPL) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kHeadU; ++u) {
        const int64_t k = k0 + u * STEP + lane * EPL;
        if (k < a.d) {
          const uint32_t ws[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (sizeof(ET) == 2) {
              const float lo = __uint_as_float(ws[e] << 16), hi = __uint_as_float(ws[e] & 0xFFFF0000u);
#pragma unroll
              for (int r = 0; r < MG; ++r) {
                const float2 hv = *reinterpret_cast<const float2*>(hs + r * a.d + k + 2 * e);
                acc[r] += lo * hv.x + hi * hv.y;
              }
            } else {
              const float wv = __uint_as_float(ws[e]);
#pragma unroll
              for (int r = 0; r < MG; ++r) acc[r] += wv * hs[r * a.d + k + e];
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < MG; ++r) {
      const float lv = warp_sum(acc[r]);
      if (lane == 0) {
        if (a.logits) a.logits[static_cast<int64_t>(m0 + r) * a.ld_logits + a.vocab_offset + v] = lv;
        const unsigned long long key = argmax_key(lv, static_cast<int>(a.vocab_offset + v));
        best[r] = key > best[r] ? key : best[r];
      }
    }
  }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < MG; ++r)
      if (best[r]) atomicMax(a.argmax + m0 + r, best[r]);
}

template <typename ET>
__global__ void __launch_bounds__(kHeadThreads) k_head(HeadArgs a) {
  trace_point(50);
  pdl_wait();
  pdl_trigger();
  trace_point(51);
  extern __shared__ float hs[];  // [kHeadRowsPerGroup][d]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m0 = 0; m0 < a.M; m0 += kHeadRowsPerGroup) {
    const int mg = min(kHeadRowsPerGroup, a.M - m0);
    __syncthreads();
    // stage h: 16-byte loads, four in flight per thread (a scalar loop here was ~25 us of L2
    // latency per launch, noticeable on small vocabularies)
    const int64_t n4 = static_cast<int64_t>(mg) * a.d / 4;
    const float4* src = reinterpret_cast<const float4*>(a.h + static_cast<int64_t>(m0) * a.d);
    float4* dst = reinterpret_cast<float4*>(hs);
    for (int64_t i0 = threadIdx.x; i0 < n4; i0 += 4 * blockDim.x) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * blockDim.x;
        if (i < n4) v[u] = src[i];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * blockDim.x;
        if (i < n4) dst[i] = v[u];
      }
    }
    __syncthreads();
    switch (mg) {
      case 1: head_rows<ET, 1>(a, hs, m0, warp, lane); break;
      case 2: head_rows<ET, 2>(a, hs, m0, warp, lane); break;
      case 3: head_rows<ET, 3>(a, hs, m0, warp, lane); break;
      default: head_rows<ET, 4>(a, hs, m0, warp, lane); break;
    }
  }
  trace_point(52);
}

// Tensor-core head for 2..16 rows (bf16 table): logits = h E^T on mma.sync.m16n8k16.bf16.
// A warp owns 16 vocab rows; per 32-wide k block each lane loads 16 contiguous bytes of
// two E rows (A) and of one h row per 8-token tile (B). The k order inside the block is
// permuted identically for A and B (lane t's bytes 8t..8t+7 feed k-tile halves), so every
// load is a plain 16-byte vector load and the dot products are unchanged.
template <int NTT>
__global__ void __launch_bounds__(kHeadThreads) k_head_tc(HeadArgs a) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* E = static_cast<const __nv_bfloat16*>(a.E);
  const int64_t ntile = (a.vocab_local + 15) / 16;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kHeadThreads / 32);
  for (int m0 = 0; m0 < a.M; m0 += 8 * NTT) {
    const int mg = min(8 * NTT, a.M - m0);
    unsigned long long best[NTT][2];
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt) best[nt][0] = best[nt][1] = 0ull;
    // token rows of this lane's B fragments (duplicates beyond the batch are discarded)
    const __nv_bfloat16* hrow[NTT];
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt) hrow[nt] = a.hb + static_cast<int64_t>(m0 + min(nt * 8 + g, mg - 1)) * a.d + 8 * t;
    for (int64_t tile = static_cast<int64_t>(blockIdx.x) * (kHeadThreads / 32) + warp; tile < ntile; tile += nwarps) {
      const int64_t v0 = tile * 16;
      const int64_t va = min(v0 + g, a.vocab_local - 1), vb = min(v0 + g + 8, a.vocab_local - 1);
      const uint4* ea = reinterpret_cast<const uint4*>(E + (a.vocab_offset + va) * a.d + 8 * t);
      const uint4* eb = reinterpret_cast<const uint4*>(E + (a.vocab_offset + vb) * a.d + 8 * t);
      float acc[NTT][4];
#pragma unroll
      for (int nt = 0; nt < NTT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
      constexpr int U = 4;  // 32-wide k blocks in flight
      for (int64_t k0 = 0; k0 < a.d; k0 += 32 * U) {
        uint4 ra[U], rb[U], rh[U][NTT];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t kb = (k0 + 32 * u) / 8;
          const bool ok = k0 + 32 * u < a.d;
          ra[u] = ok ? ld_stream(ea + kb) : make_uint4(0, 0, 0, 0);
          rb[u] = ok ? ld_stream(eb + kb) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int nt = 0; nt < NTT; ++nt)
            rh[u][nt] = ok ? *reinterpret_cast<const uint4*>(hrow[nt] + k0 + 32 * u) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int nt = 0; nt < NTT; ++nt) {
            // k-tile 0: bytes 0..7 of each 16-byte group, k-tile 1: bytes 8..15
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(acc[nt][0]), "+f"(acc[nt][1]), "+f"(acc[nt][2]), "+f"(acc[nt][3])
                : "r"(ra[u].x), "r"(rb[u].x), "r"(ra[u].y), "r"(rb[u].y), "r"(rh[u][nt].x), "r"(rh[u][nt].y));
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(acc[nt][0]), "+f"(acc[nt][1]), "+f"(acc[nt][2]), "+f"(acc[nt][3])
                : "r"(ra[u].z), "r"(rb[u].z), "r"(ra[u].w), "r"(rb[u].w), "r"(rh[u][nt].z), "r"(rh[u][nt].w));
          }
      }
      // acc[nt][0..1]: vocab row v0+g, tokens nt*8+2t+{0,1}; acc[nt][2..3]: row v0+g+8
#pragma unroll
      for (int nt = 0; nt < NTT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int m = nt * 8 + 2 * t + (e & 1);
          const int64_t v = v0 + g + 8 * (e >> 1);
          if (m < mg && v < a.vocab_local) {
            if (a.logits) a.logits[static_cast<int64_t>(m0 + m) * a.ld_logits + a.vocab_offset + v] = acc[nt][e];
            const unsigned long long key = argmax_key(acc[nt][e], static_cast<int>(a.vocab_offset + v));
            best[nt][e & 1] = key > best[nt][e & 1] ? key : best[nt][e & 1];
          }
        }
    }
    // reduce each token's best over the 8 lanes (g) that hold it, then one atomic per token
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        unsigned long long b = best[nt][e];
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
          b = ob > b ? ob : b;
        }
        const int m = nt * 8 + 2 * t + e;
        if (g == 0 && m < mg && b) atomicMax(a.argmax + m0 + m, b);
      }
  }
}

__global__ void k_rows_to_bf16(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 2; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x * 2)
    *reinterpret_cast<__nv_bfloat162*>(y + i) = __floats2bfloat162_rn(x[i], x[i + 1]);
}

// The winning key also guards the fp16 activation path: NaN keys sort above every number and
// +inf above every finite value, so a row whose activations left the fp16 range (inf -> NaN
// through the LayerNorm) always has a non-finite winner; it raises *status (model.cu reports
// GLM_POLICY) instead of returning a token picked from garbage.
__global__ void k_argmax_finish(unsigned long long* __restrict__ keys, int* __restrict__ tokens, int M, int* status) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < M) {
    const unsigned long long k = keys[m];
    tokens[m] = static_cast<int>(~static_cast<uint32_t>(k & 0xFFFFFFFFull));
    const uint32_t u = static_cast<uint32_t>(k >> 32);
    const float v = __uint_as_float((u >> 31) ? (u & 0x7FFFFFFFu) : ~u);
    if (status && !finite_f32(v)) atomicOr(status, 1);
    keys[m] = 0ull;
  }
}

int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

void launch_embed(const void* E, bool bf16, int64_t d, const int* tokens, int M, float* h, const XOut& xo,
                  cudaStream_t st, bool half_store) {
  const int hs = half_store ? 1 : 0;
  if (xo.tile && d % 8 == 0) {
    const int64_t warps = (M + kXTileTokens - 1) / kXTileTokens * (d / 8) * (kXTileTokens / 32);
    const dim3 grid(grid_for(warps * 32, 256, 1 << 30));  // one pass per warp: the row-id -> row load chain is latency-bound
    if (bf16) launch_k(k_embed_tiles<__nv_bfloat16>, grid, dim3(256), 0, st, static_cast<const __nv_bfloat16*>(E), d, tokens, M, h, xo, hs);
    else launch_k(k_embed_tiles<float>, grid, dim3(256), 0, st, static_cast<const float*>(E), d, tokens, M, h, xo, hs);
    LAUNCH_CHECK("k_embed_tiles");
    return;
  }
  if (bf16) launch_k(k_embed<__nv_bfloat16>, dim3(M), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(E), d, tokens, M, h, xo, hs);
  else launch_k(k_embed<float>, dim3(M), dim3(256), 0, st, static_cast<const float*>(E), d, tokens, M, h, xo, hs);
  LAUNCH_CHECK("k_embed");
}

void launch_deepnorm_ln(const LnArgs& a, int M, cudaStream_t st) {
  if (a.d > 2ll * kLnPairs * kLnThreads * kLnCluster || a.d % 2) fail(GLM_DIMENSION, "glmmodel", "hidden unsupported by LN kernel");
  // (the fused tensor-parallel sum keeps 8: its inbox slices and generation flags are per 8-CTA slice)
  const bool cl4 = M > 8 && a.peer.size <= 1 && a.d <= 2ll * kLnPairs * kLnThreads * 4;
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool v8 = a.d % 8 == 0 && a.in.ld % 4 == 0 && a.in.split_stride % 4 == 0 && al(a.in.p) && al(a.h) &&
                  al(a.gain) && al(a.bias) && al(a.tap);
  static const bool rows8 = [] { const char* e = getenv("GLM_LN_ROWS8"); return !e || e[0] != '0'; }();
  // 3 resident 512-thread CTAs per SM (40 registers): the row's two passes are latency-bound,
  // so occupancy sets the bandwidth (ncu, 8192 x 12288: 1 CTA/SM 487/403 us, 2: 328, 3: 341/263,
  // 4 spills: 440/361)
  if (a.peer.size > 1 && M > 16) fail(GLM_CONTRACT, "glmmodel", "fused tensor-parallel LayerNorm is a decode (<= 16 rows) kernel");
  if (a.in.zt && M > 16) fail(GLM_CONTRACT, "glmmodel", "the zero-point term enters the LayerNorm only in decode (<= 16 rows)");
  if (M > 16 && v8 && rows8) launch_k(k_deepnorm_ln_rows8<3>, dim3(M), dim3(kLnRowThreads), 0, st, a);
  else if (M > 16) launch_k(k_deepnorm_ln_rows, dim3(M), dim3(kLnRowThreads), 0, st, a);
  else if (cl4) launch_k(k_deepnorm_ln<4>, dim3(M * 4), dim3(kLnThreads), 0, st, a);
  else launch_k(k_deepnorm_ln<kLnCluster>, dim3(M * kLnCluster), dim3(kLnThreads), 0, st, a);
  LAUNCH_CHECK("k_deepnorm_ln");
}

void launch_geglu_act(const ActArgs& a, cudaStream_t st) {
  auto al4 = [](const SubIn& in) { return in.ld % 4 == 0 && in.split_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(in.p) & 15) == 0; };
  if (a.xo.tile && a.xo.xf && a.f % 8 == 0 && al4(a.w1) && al4(a.v)) {
    const int64_t warps = (a.M + kXTileTokens - 1) / kXTileTokens * (a.f / 8) * (kXTileTokens / 32);
    launch_k(k_geglu_act_tiles, dim3(grid_for(warps * 32, 256)), dim3(256), 0, st, a);
    LAUNCH_CHECK("k_geglu_act_tiles");
    return;
  }
  const auto al2 = [](const SubIn& in) {
    return in.ld % 2 == 0 && in.split_stride % 2 == 0 && (reinterpret_cast<uintptr_t>(in.p) & 7) == 0 &&
           (!in.scale || (reinterpret_cast<uintptr_t>(in.scale) & 7) == 0);
  };
  const bool v2 = a.f % 2 == 0 && al2(a.w1) && al2(a.v);
  launch_k(v2 ? k_geglu_act<true> : k_geglu_act<false>, dim3(grid_for(static_cast<int64_t>(a.M) * ((a.f + 1) / 2), 128)),
           dim3(128), 0, st, a);
  LAUNCH_CHECK("k_geglu_act");
}

// keys per CTA: 256 (no merge) up to a 256-token cache for one or two sequences (staged) and
// for more than 8 (read from L2 / HBM: 96 x B CTAs already fill the SMs); 64-key splits, each
// staged by one bulk copy issued before the dependency wait, for 3..8 sequences and for longer
// caches (batch sweep, same box: B = 4 251 -> 280, B = 8 429 -> 454 tok/s; B = 16 662 -> 643, so
// not there). GLM_ATTN_SPLIT64=0 keeps the 256-key unstaged CTAs at 3..8 sequences.
// ---- long-context decode attention: one CTA streams a long key range -----------------
// grid (heads, batch, splits) with split_keys = a multiple of 64 chosen so a target number of
// CTAs per SM cover the caches (launch_attn_decode): the split's cached keys pass through a ring
// of kRingStages 64-key shared-memory blocks (one bulk copy each, the first ones issued before
// the dependency wait): all K blocks for the scores (kept in shared memory, up to
// kRingMaxKeys), then the V blocks for P.V, so K and V are read once at HBM speed instead of
// 64-key CTAs waiting in waves. q / the new key / value, RoPE, the split partial format and the
// in-order merge are those of k_attn_decode.
constexpr int kRingBlock = 64;
constexpr int kRingMaxKeys = 2048;
constexpr int kRingThreads = 256;

// NS ring stages: 4 for long caches (two CTAs per SM), 2 for short ones (5-6 per SM: many
// (head, sequence) pairs with a few blocks each)
template <int DH, int NS, int MINB>
__global__ void __launch_bounds__(kRingThreads, MINB) k_attn_decode_ring(AttnDecodeArgs a) {
  trace_point(30);
  constexpr int kRingStages = NS;
  constexpr int NW = kRingThreads / 32;
  constexpr int FPL = DH / 32;
  constexpr int LPK = DH / 8, KPW = 32 / LPK;
  constexpr int BLK_BYTES = kRingBlock * DH * 2;
  __shared__ float q[DH];
  __shared__ float red[NW];
  __shared__ int last;
  __shared__ __align__(8) uint64_t bars[kRingStages];
  __shared__ __align__(16) __half knew[DH];
  __shared__ __align__(16) __half vnew[DH];
  extern __shared__ __align__(128) __half ring[];  // [kRingStages][kRingBlock][DH], then p
  float* p = reinterpret_cast<float*>(ring + kRingStages * kRingBlock * DH);  // [split_keys + 1] scores
  // per-warp P.V partials reuse the ring once every block is consumed (NW * DH floats <= one stage)
  static_assert(NW * DH * 4 <= kRingBlock * DH * 2 * NS, "P.V partials fit the ring");
  float (*opart)[DH] = reinterpret_cast<float (*)[DH]>(ring);
  const int head = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = a.cache_len[b];
  const int total = len + 1;
  const int k0 = split * a.split_keys, k1 = min(total, k0 + a.split_keys);
  const int kold = min(k1, len);
  const int n_old = max(0, kold - k0);
  const int nb = (n_old + kRingBlock - 1) / kRingBlock;  // 64-key blocks of cached keys
  const int pos = a.positions[b];
  const float inv_sqrt = rsqrtf(static_cast<float>(DH));
  __half* kc = a.kcache + ((static_cast<int64_t>(b) * a.heads + head) * a.max_ctx) * DH;
  __half* vc = a.vcache + ((static_cast<int64_t>(b) * a.heads + head) * a.max_ctx) * DH;
  float* part = a.part + ((static_cast<int64_t>(b) * a.heads + head) * a.max_splits + split) * (DH + 2);
  // load j < nb: K block j; nb <= j < 2 nb: V block j - nb
  auto issue = [&](int j) {
    if (j >= 2 * nb) return;
    const int blk = j < nb ? j : j - nb;
    const int kk = k0 + blk * kRingBlock;
    const uint32_t bytes = static_cast<uint32_t>(min(kRingBlock, kold - kk)) * DH * 2;
    uint64_t* bar = bars + (j % kRingStages);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(reinterpret_cast<uint8_t*>(ring) + (j % kRingStages) * BLK_BYTES)),
                 "l"((j < nb ? kc : vc) + static_cast<int64_t>(kk) * DH), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
  };
  auto wait = [&](int j) {
    const uint32_t par = static_cast<uint32_t>((j / kRingStages) & 1);
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                     smem_addr(bars + (j % kRingStages))),
                 "r"(par)
                 : "memory");
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRingStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // cached keys do not depend on the running qkv GEMV
    if (k0 < total)
      for (int j = 0; j < kRingStages; ++j) issue(j);
  }
  __syncthreads();
  const int jt = threadIdx.x < DH / 2 ? threadIdx.x : threadIdx.x - DH / 2;
  float2 cs = make_float2(1.f, 0.f), sq = make_float2(1.f, 1.f), sk = sq, sv = sq;
  if (threadIdx.x < DH) {
    cs = a.rope[static_cast<int64_t>(pos) * (DH / 2) + jt];
    const int64_t fq = static_cast<int64_t>(head) * DH + 2 * jt;
    if (a.qkv.scale) {
      sq = *reinterpret_cast<const float2*>(a.qkv.scale + fq);
      sk = *reinterpret_cast<const float2*>(a.qkv.scale + a.d_local + fq);
      sv = *reinterpret_cast<const float2*>(a.qkv.scale + 2 * a.d_local + fq);
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_point(31);
  if (k0 >= total) return;  // beyond the cache: no keys, not counted by the merge
  const bool has_new = len >= k0 && len < k1;
  if (threadIdx.x < DH) {
    auto raw2 = [&](int64_t f) {
      float2 acc = make_float2(0.f, 0.f);
      for (int s0 = 0; s0 < a.qkv.ksplit; ++s0) {
        const float2 v = *reinterpret_cast<const float2*>(a.qkv.p + static_cast<int64_t>(s0) * a.qkv.split_stride +
                                                          b * a.qkv.ld + f);
        acc.x += v.x;
        acc.y += v.y;
      }
      return acc;
    };
    auto zp2 = [&](int64_t f) {
      return a.qkv.zt ? make_float2(a.qkv.zt[b] * a.qkv.zv[f], a.qkv.zt[b] * a.qkv.zv[f + 1]) : make_float2(0.f, 0.f);
    };
    const int64_t fq = static_cast<int64_t>(head) * DH + 2 * jt;
    if (threadIdx.x < DH / 2) {
      const float2 qv = raw2(fq), qz = zp2(fq);
      const float qa = qv.x * sq.x + qz.x, qb = qv.y * sq.y + qz.y;
      q[2 * jt] = (cs.x * qa - cs.y * qb) * inv_sqrt;
      q[2 * jt + 1] = (cs.y * qa + cs.x * qb) * inv_sqrt;
    } else if (has_new) {
      const int64_t fk = a.d_local + fq, fv = 2 * a.d_local + fq;
      const float2 kv2 = raw2(fk), vv2 = raw2(fv), kz = zp2(fk), vz = zp2(fv);
      const float ka = kv2.x * sk.x + kz.x, kb = kv2.y * sk.y + kz.y;
      const float va = vv2.x * sv.x + vz.x, vb = vv2.y * sv.y + vz.y;
      const __half2 kh = __floats2half2_rn(cs.x * ka - cs.y * kb, cs.y * ka + cs.x * kb);
      const __half2 vh = __floats2half2_rn(va, vb);
      *reinterpret_cast<__half2*>(kc + static_cast<int64_t>(len) * DH + 2 * jt) = kh;
      *reinterpret_cast<__half2*>(vc + static_cast<int64_t>(len) * DH + 2 * jt) = vh;
      *reinterpret_cast<__half2*>(knew + 2 * jt) = kh;
      *reinterpret_cast<__half2*>(vnew + 2 * jt) = vh;
    }
  }
  __syncthreads();
  trace_point(33);
  // ---- scores over the K blocks (LPK lanes per key, one 16-byte load each) ----
  const int sub = lane % LPK, kin = lane / LPK;
  float qr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) qr[i] = q[sub * 8 + i];
  auto dot8 = [&](uint4 kv) {
    const uint32_t w4[4] = {kv.x, kv.y, kv.z, kv.w};
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[e]));
      acc += qr[2 * e] * f.x + qr[2 * e + 1] * f.y;
    }
    return acc;
  };
  auto score = [&](float acc) {
    if (a.prescale > 0.f) acc = half_round(acc / a.prescale) * a.prescale;
    return acc;
  };
  for (int j = 0; j < nb; ++j) {
    wait(j);
    const __half* blk = ring + (j % kRingStages) * (kRingBlock * DH);
    const int nk = min(kRingBlock, n_old - j * kRingBlock);
    // the block's kRingBlock / (NW * KPW) key groups of this warp, loads first (independent chains)
    constexpr int KIT = kRingBlock / (NW * KPW);
    float acc[KIT];
#pragma unroll
    for (int i = 0; i < KIT; ++i) {
      const int s = warp * KPW + kin + i * NW * KPW;
      acc[i] = s < nk ? dot8(*reinterpret_cast<const uint4*>(blk + s * DH + sub * 8)) : 0.f;
    }
#pragma unroll
    for (int o = LPK / 2; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < KIT; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
#pragma unroll
    for (int i = 0; i < KIT; ++i) {
      const int s = warp * KPW + kin + i * NW * KPW;
      if (sub == 0 && s < nk) p[j * kRingBlock + s] = score(acc[i]);
    }
    __syncthreads();  // stage j consumed by every warp
    if (threadIdx.x == 0) issue(j + kRingStages);
  }
  if (has_new && warp == 0) {
    float acc = lane < LPK ? dot8(*reinterpret_cast<const uint4*>(knew + lane * 8)) : 0.f;
#pragma unroll
    for (int o = LPK / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) p[n_old] = score(acc);
  }
  __syncthreads();
  trace_point(34);
  const int nk_all = n_old + (has_new ? 1 : 0);
  // ---- softmax over the split (fp32) ----
  float mx = -FLT_MAX;
  for (int s = threadIdx.x; s < nk_all; s += kRingThreads) mx = fmaxf(mx, p[s]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int s = threadIdx.x; s < nk_all; s += kRingThreads) {
    const float e = __expf(p[s] - mx);
    p[s] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) sum += red[w];
  // ---- P.V over the V blocks: warp w takes keys w, w + NW, ...; lane owns FPL features ----
  float o[FPL];
#pragma unroll
  for (int f = 0; f < FPL; ++f) o[f] = 0.f;
  auto pv = [&](const __half* vr, float pw) {
    const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(vr));
    o[0] += pw * f0.x;
    o[1] += pw * f0.y;
    if constexpr (FPL == 4) {
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(vr + 2));
      o[2] += pw * f1.x;
      o[3] += pw * f1.y;
    }
  };
  for (int j = nb; j < 2 * nb; ++j) {
    wait(j);
    const __half* blk = ring + (j % kRingStages) * (kRingBlock * DH);
    const int jb = j - nb, nk = min(kRingBlock, n_old - jb * kRingBlock);
    if (nk == kRingBlock) {
#pragma unroll
      for (int i = 0; i < kRingBlock / NW; ++i) pv(blk + (warp + i * NW) * DH + lane * FPL, p[jb * kRingBlock + warp + i * NW]);
    } else {
      for (int s = warp; s < nk; s += NW) pv(blk + s * DH + lane * FPL, p[jb * kRingBlock + s]);
    }
    __syncthreads();
    if (threadIdx.x == 0) issue(j + kRingStages);
  }
  if (has_new && warp == 0) pv(vnew + lane * FPL, p[n_old]);
#pragma unroll
  for (int f = 0; f < FPL; ++f) opart[warp][lane * FPL + f] = o[f];
  __syncthreads();
  trace_point(35);
  if (total <= a.split_keys) {  // single active split: normalise, hand the row to out_proj
    const float inv = 1.f / sum;
    for (int c2 = threadIdx.x; c2 < DH / 2; c2 += kRingThreads) {
      float o0 = 0.f, o1 = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        o0 += opart[w][2 * c2];
        o1 += opart[w][2 * c2 + 1];
      }
      const int64_t k = static_cast<int64_t>(head) * DH + 2 * c2;
      store_xfrag_pair(a.xo, b, k, o0 * inv, o1 * inv);
      if (a.out) {
        a.out[static_cast<int64_t>(b) * a.heads * DH + k] = o0 * inv;
        a.out[static_cast<int64_t>(b) * a.heads * DH + k + 1] = o1 * inv;
      }
    }
    trace_point(32);
    return;
  }
  for (int c = threadIdx.x; c < DH; c += kRingThreads) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) acc += opart[w][c];
    part[c] = acc;
  }
  if (threadIdx.x == 0) {
    part[DH] = mx;
    part[DH + 1] = sum;
  }
  // ---- the last of the active splits of this (head, b) merges them in order ----
  const int nsp = (total + a.split_keys - 1) / a.split_keys;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* ctr = a.counters + b * a.heads + head;
    last = (atomicAdd(ctr, 1) == nsp - 1);
    if (last) *ctr = 0;
  }
  __syncthreads();
  if (!last) {
    trace_point(32);
    return;
  }
  __threadfence();
  const float* base = a.part + ((static_cast<int64_t>(b) * a.heads + head) * a.max_splits) * (DH + 2);
  float* wsp = p;
  if (warp == 0) {
    float gm = -FLT_MAX;
    for (int s = lane; s < nsp; s += 32) gm = fmaxf(gm, __ldcg(base + s * (DH + 2) + DH));
    gm = warp_max(gm);
    float gl = 0.f;
    for (int s = lane; s < nsp; s += 32) {
      const float w = __expf(__ldcg(base + s * (DH + 2) + DH) - gm);
      wsp[s] = w;
      gl += __ldcg(base + s * (DH + 2) + DH + 1) * w;
    }
    gl = warp_sum(gl);
    const float inv = 1.f / gl;
    for (int s = lane; s < nsp; s += 32) wsp[s] *= inv;
  }
  __syncthreads();
  for (int c2 = threadIdx.x; c2 < DH / 2; c2 += kRingThreads) {
    float o0 = 0.f, o1 = 0.f;
    for (int s = 0; s < nsp; ++s) {
      const float w = wsp[s];
      const float2 v = __ldcg(reinterpret_cast<const float2*>(base + s * (DH + 2) + 2 * c2));
      o0 += w * v.x;
      o1 += w * v.y;
    }
    const int64_t k = static_cast<int64_t>(head) * DH + 2 * c2;
    store_xfrag_pair(a.xo, b, k, o0, o1);
    if (a.out) {
      a.out[static_cast<int64_t>(b) * a.heads * DH + k] = o0;
      a.out[static_cast<int64_t>(b) * a.heads * DH + k + 1] = o1;
    }
  }
  trace_point(32);
}

int attn_decode_split_keys(int max_ctx, int B) {
  static const bool many64 = [] { const char* e = getenv("GLM_ATTN_SPLIT64"); return !e || e[0] != '0'; }();
  if (max_ctx > kSplitKeys) return kSplitKeysLong;
  return (B > 2 && B <= 8 && many64) ? kSplitKeysLong : kSplitKeys;
}
int attn_decode_split_keys(int max_ctx) { return attn_decode_split_keys(max_ctx, 1); }
// capacity of the split partial buffer: 64-key splits of the longest cache
int attn_decode_splits(int max_ctx) { return (max_ctx + kSplitKeysLong - 1) / kSplitKeysLong; }

void launch_attn_decode(const AttnDecodeArgs& in, int B, cudaStream_t st) {
  AttnDecodeArgs a = in;
  // Each CTA bulk-copies its split's cached keys + values into shared memory ahead of the
  // dependency wait (one HBM round trip, overlapping the qkv GEMV): 256-key CTAs for one or
  // two sequences, 64-key CTAs (32 KB of staging, several per SM) otherwise.
  a.split_keys = attn_decode_split_keys(a.max_ctx, B);
  if (a.max_splits != attn_decode_splits(a.max_ctx)) fail(GLM_CONTRACT, "glmmodel", "decode attention split count");
  // GLM_ATTN_RING: 0 off, 1 long caches only, 2 (default) long caches and 3+ sequences, 3 always
  // (same-box: 3+ sequences at ~135 cached tokens B = 4 / 8 / 16 +2.3 / +3.9 / +1.9 %; one or two
  // sequences keep the 256-key staged CTAs: always-ring 80.1 vs 80.6 tok/s at batch 1)
  static const int ring = [] { const char* e = getenv("GLM_ATTN_RING"); return e ? atoi(e) : 2; }();
  if (ring && (a.max_ctx > kSplitKeys || (ring == 2 && B > 2) || ring == 3) && (a.dh == 128 || a.dh == 64)) {
    // long caches: 6-stage rings of 64-key blocks, GLM_ATTN_RING_CPS (2) streaming CTAs per SM
    // (4 / 6 / 8 stages: 0.2054 / 0.2036 / 0.2173 ms at config 2); short caches of many
    // sequences: 2-stage rings, five or six CTAs per SM
    static const int cps_env = [] { const char* e = getenv("GLM_ATTN_RING_CPS"); return e ? atoi(e) : 0; }();
    const bool long_ctx = a.max_ctx > kSplitKeys;
    const int ns = long_ctx ? 6 : 2;
    const int cps = cps_env > 0 ? cps_env : (long_ctx ? 2 : 5);
    const int64_t ctas = static_cast<int64_t>(a.heads) * B;
    const int64_t nsplit = std::max<int64_t>(1, cps * 148 / ctas);
    int64_t sk = (a.max_ctx + nsplit - 1) / nsplit;
    sk = std::min<int64_t>(kRingMaxKeys, (sk + kRingBlock - 1) / kRingBlock * kRingBlock);
    a.split_keys = static_cast<int>(sk);
    a.stage_keys = 0;
    const dim3 grid(a.heads, B, (a.max_ctx + a.split_keys - 1) / a.split_keys);
    // p: the split's scores (sk + 1), later the merge weights of up to ceil(max_ctx / sk) splits
    const int64_t pn = std::max<int64_t>(sk + 1, (a.max_ctx + sk - 1) / sk) + 3;
    const size_t smem = static_cast<size_t>(ns) * kRingBlock * a.dh * 2 + pn * 4;
    static bool attr_r = false;
    if (!attr_r) {
      const int mxl = 6 * kRingBlock * 128 * 2 + (kRingMaxKeys + 260) * 4, mx2 = 2 * kRingBlock * 128 * 2 + (kRingMaxKeys + 260) * 4;
      CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode_ring<128, 6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mxl));
      CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode_ring<64, 6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mxl));
      for (auto k : {k_attn_decode_ring<128, 2, 5>, k_attn_decode_ring<64, 2, 5>, k_attn_decode_ring<128, 2, 6>,
                     k_attn_decode_ring<64, 2, 6>})
        CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx2));
      attr_r = true;
    }
    // short caches: six resident CTAs per SM (40 registers) once the grid exceeds one wave at
    // five (B = 8: +1.5 %); smaller grids keep the five-CTA build (B = 3 / 4: -0.8 / -0.5 % at six)
    const bool six = static_cast<int64_t>(grid.x) * grid.y * grid.z > 5 * 148;
    if (long_ctx) {
      if (a.dh == 128) launch_k(k_attn_decode_ring<128, 6, 2>, grid, dim3(kRingThreads), smem, st, a);
      else launch_k(k_attn_decode_ring<64, 6, 2>, grid, dim3(kRingThreads), smem, st, a);
    } else if (six) {
      if (a.dh == 128) launch_k(k_attn_decode_ring<128, 2, 6>, grid, dim3(kRingThreads), smem, st, a);
      else launch_k(k_attn_decode_ring<64, 2, 6>, grid, dim3(kRingThreads), smem, st, a);
    } else {
      if (a.dh == 128) launch_k(k_attn_decode_ring<128, 2, 5>, grid, dim3(kRingThreads), smem, st, a);
      else launch_k(k_attn_decode_ring<64, 2, 5>, grid, dim3(kRingThreads), smem, st, a);
    }
    LAUNCH_CHECK("k_attn_decode_ring");
    return;
  }
  if (a.max_splits > kSplitKeys)  // the merge keeps one weight per split in the score buffer
    fail(GLM_DIMENSION, "glmmodel", "decode attention supports caches up to 16384 tokens");
  const dim3 grid(a.heads, B, (a.max_ctx + a.split_keys - 1) / a.split_keys);
  const bool many_unstaged = B > 2 && a.split_keys == kSplitKeys;  // GLM_ATTN_SPLIT64=0
  const int stage = many_unstaged ? 0 : std::min(a.split_keys, (a.max_ctx + 15) / 16 * 16);
  a.stage_keys = stage;
  const size_t smem = 2ull * stage * a.dh * sizeof(__half);
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode<128, kAttnThreadsFew>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSplitKeys * 128 * 2));
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode<64, kAttnThreadsFew>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSplitKeys * 64 * 2));
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode<128, kAttnThreadsMany>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSplitKeysLong * 128 * 2));
    CUDA_CHECK(cudaFuncSetAttribute(k_attn_decode<64, kAttnThreadsMany>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSplitKeysLong * 64 * 2));
    attr = true;
  }
  if (stage && a.split_keys == kSplitKeys) {
    if (a.dh == 128) launch_k(k_attn_decode<128, kAttnThreadsFew>, grid, dim3(kAttnThreadsFew), smem, st, a);
    else if (a.dh == 64) launch_k(k_attn_decode<64, kAttnThreadsFew>, grid, dim3(kAttnThreadsFew), smem, st, a);
    else fail(GLM_DIMENSION, "glmmodel", "decode attention supports head_dim 64 or 128");
  } else {  // many sequences, or 64-key splits of a long cache (staged at <= 2 sequences): 128-thread CTAs
    if (a.dh == 128) launch_k(k_attn_decode<128, kAttnThreadsMany>, grid, dim3(kAttnThreadsMany), smem, st, a);
    else if (a.dh == 64) launch_k(k_attn_decode<64, kAttnThreadsMany>, grid, dim3(kAttnThreadsMany), smem, st, a);
    else fail(GLM_DIMENSION, "glmmodel", "decode attention supports head_dim 64 or 128");
  }
  LAUNCH_CHECK("k_attn_decode");
}

void launch_advance(int* cache_len, int B, cudaStream_t st) {
  launch_k(k_advance, dim3(1), dim3(32), 0, st, cache_len, B);
  LAUNCH_CHECK("k_advance");
}

void launch_rope_store(const RopeStoreArgs& a, cudaStream_t st) {
  const bool al = a.ldqkv % 4 == 0 && a.d_local % 4 == 0 && (reinterpret_cast<uintptr_t>(a.qkv) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(a.rope) & 15) == 0;
  if (a.qkv_h) {
    if (a.dh != 128 || a.ldqkv % 4 || a.d_local % 4 || (reinterpret_cast<uintptr_t>(a.qkv_h) & 7))
      fail(GLM_CONTRACT, "glmmodel", "fp16 qkv rows need head_dim 128 and 8-byte aligned rows");
    k_rope_store128<__half><<<dim3(a.n, (a.heads + 7) / 8), 256, 0, st>>>(a, a.qkv_h);
    LAUNCH_CHECK("k_rope_store128");
    return;
  }
  if (a.dh == 128 && al) {
    k_rope_store128<float><<<dim3(a.n, (a.heads + 7) / 8), 256, 0, st>>>(a, a.qkv);
    LAUNCH_CHECK("k_rope_store128");
    return;
  }
  k_rope_store<<<dim3(a.n, a.heads), 64, 0, st>>>(a);
  LAUNCH_CHECK("k_rope_store");
}

void launch_attn_prefill(const AttnPrefillArgs& a, cudaStream_t st) {
  if (launch_attn_prefill_umma(a, st)) return;
  if (a.xo.xf) fail(GLM_CONTRACT, "glmmodel", "activation-tile attention output needs the tcgen05 kernel");
  const dim3 grid((a.n + kFaRows - 1) / kFaRows, a.heads);
  auto go = [&](auto kernel, int dh) {
    const size_t smem = static_cast<size_t>(4 * kFaKeys) * (dh + 8) * sizeof(__half);
    CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kernel<<<grid, kFaThreads, smem, st>>>(a);
  };
  if (a.dh == 128) go(k_attn_prefill_tc<128>, 128);
  else if (a.dh == 64) go(k_attn_prefill_tc<64>, 64);
  else fail(GLM_DIMENSION, "glmmodel", "prefill attention supports head_dim 64 or 128");
  LAUNCH_CHECK("k_attn_prefill_tc");
}

void launch_rows_to_xfrag(const float* x, int64_t ld, int M, int64_t K, const XOut& xo, cudaStream_t st) {
  if (xo.tile && K % 8 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int64_t warps = (M + kXTileTokens - 1) / kXTileTokens * (K / 8) * (kXTileTokens / 32);
    k_rows_to_xtile<<<grid_for(warps * 32, 256), 256, 0, st>>>(x, ld, M, K, xo);
    LAUNCH_CHECK("k_rows_to_xtile");
    return;
  }
  k_rows_to_xfrag<<<grid_for(static_cast<int64_t>(M) * (K / 2), 256), 256, 0, st>>>(x, ld, M, K, xo);
  LAUNCH_CHECK("k_rows_to_xfrag");
}

void launch_head(const HeadArgs& a, bool bf16, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(a.M < kHeadRowsPerGroup ? a.M : kHeadRowsPerGroup) * a.d * sizeof(float);
  static bool attr_set[2] = {false, false};
  if (!attr_set[bf16]) {
    if (bf16) CUDA_CHECK(cudaFuncSetAttribute(k_head<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    else CUDA_CHECK(cudaFuncSetAttribute(k_head<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set[bf16] = true;
  }
  if (smem > 227 * 1024) fail(GLM_DIMENSION, "glmmodel", "hidden too large for head kernel");
  if (a.d % 256 != 0) fail(GLM_DIMENSION, "glmmodel", "head kernel needs hidden % 256 == 0");
  if (bf16 && a.M > 1 && a.hb) {
    // batched rows: tensor cores on a bf16 copy of h
    const int64_t n = static_cast<int64_t>(a.M) * a.d;
    launch_k(k_rows_to_bf16, dim3(static_cast<unsigned>(std::min<int64_t>((n / 2 + 255) / 256, 1184))), dim3(256), 0, st,
             a.h, a.hb, n);
    LAUNCH_CHECK("k_rows_to_bf16");
    const int grid_tc = kNumSMs * 8;
    if (a.M <= 8) launch_k(k_head_tc<1>, dim3(grid_tc), dim3(kHeadThreads), 0, st, a);
    else launch_k(k_head_tc<2>, dim3(grid_tc), dim3(kHeadThreads), 0, st, a);
    LAUNCH_CHECK("k_head_tc");
    return;
  }
  const int per_sm = static_cast<int>(std::min<size_t>(8, (227 * 1024) / (smem + 1024)));
  // one vocabulary row per warp: no more CTAs than rows (each CTA stages h in shared memory,
  // so idle CTAs of a small vocabulary would only add L2 traffic)
  const int64_t need = (a.vocab_local + kHeadThreads / 32 - 1) / (kHeadThreads / 32);
  const int grid = static_cast<int>(std::min<int64_t>(need, kNumSMs * (per_sm < 1 ? 1 : per_sm)));
  if (bf16) launch_k(k_head<__nv_bfloat16>, dim3(grid), dim3(kHeadThreads), smem, st, a);
  else launch_k(k_head<float>, dim3(grid), dim3(kHeadThreads), smem, st, a);
  LAUNCH_CHECK("k_head");
}

void launch_argmax_finish(unsigned long long* keys, int* tokens, int M, cudaStream_t st, int* status) {
  launch_k(k_argmax_finish, dim3(grid_for(M, 32)), dim3(32), 0, st, keys, tokens, M, status);
  LAUNCH_CHECK("k_argmax_finish");
}

}  // namespace glm
