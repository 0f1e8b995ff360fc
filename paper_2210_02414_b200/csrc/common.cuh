// common.cuh — error plumbing and small device helpers shared by every kernel.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "glm130b.h"

namespace glm {

// Error taxonomy of include/glmlab/common.hpp:28-56 carried as a status code; the
// C ABI turns it into glm_status + glm_last_error() ("[module] message").
struct Error : std::runtime_error {
  glm_status code;
  Error(glm_status c, const std::string& module, const std::string& msg)
      : std::runtime_error("[" + module + "] " + msg), code(c) {}
};

[[noreturn]] inline void fail(glm_status c, const char* module, const std::string& msg) {
  throw Error(c, module, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(GLM_CUDA, "cuda", std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_CHECK(x) ::glm::cuda_check((x), #x)
// GLM_SYNC_LAUNCH=1 (debugging, with GLM_EAGER=1): synchronise after every launch so a
// device fault is attributed to the kernel that caused it.
bool sync_launch_debug();
inline void launch_check(const char* what) {
  cuda_check(cudaGetLastError(), what);
  if (sync_launch_debug()) cuda_check(cudaDeviceSynchronize(), what);
}
#define LAUNCH_CHECK(what) ::glm::launch_check(what)

void set_last_error(const std::string& s);

template <typename F>
glm_status guarded(F&& f) {
  try {
    f();
    return GLM_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("[runtime] host allocation failed");
    return GLM_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GLM_CONTRACT;
  }
}

constexpr int kNumSMs = 148;

// Programmatic dependent launch (PDL) for the decode chain: every kernel of the step is
// launched with programmaticStreamSerialization, so kernel k+1 may become resident while
// kernel k runs. Each kernel calls pdl_wait() before touching anything its predecessor
// writes (griddepcontrol.wait: predecessor complete, its memory visible) and pdl_trigger()
// only AFTER that wait, so at most one kernel runs ahead (no resource deadlock). Work that
// depends on nothing (e.g. the GEMV's weight prefetch) goes before the wait.
// GLM_PDL=0 launches everything with plain stream order (A/B switch).
bool pdl_enabled();

// `coop` adds the cooperative attribute: the launch fails instead of deadlocking if the
// grid cannot be fully co-resident (kernels with a grid-wide barrier).
template <typename... KArgs, typename... Args>
inline void launch_k_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool coop,
                        Args&&... args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  launch_k_ex(kernel, grid, block, smem, st, false, std::forward<Args>(args)...);
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

#if defined(__CUDACC__)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Streaming 128-bit load that does not allocate in L1 (weights are read once).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Read-only 128-bit load that may stay in L1 (activations re-read by every warp).
__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Timeline tracer (diagnostics, tools/timeline.py): when a trace buffer is bound, thread 0
// of every CTA appends (globaltimer ns, tag << 32 | block << 8 | smid) records. Each
// translation unit has its own symbol, bound by trace_bind_all() (capi_quant.cpp).
static __constant__ unsigned long long* g_trace_buf = nullptr;  // constant bank: no global load at kernel entry
static __constant__ unsigned long long g_trace_cap = 0;
__device__ __forceinline__ void trace_point(unsigned tag) {
  unsigned long long* buf = g_trace_buf;
  if (buf == nullptr || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const unsigned long long i = atomicAdd(buf, 1ull);
  if (i < g_trace_cap) {
    buf[1 + 2 * i] = t;
    buf[2 + 2 * i] = (static_cast<unsigned long long>(tag) << 32) | (static_cast<unsigned long long>(blockIdx.x) << 8) | smid;
  }
}
#define GLM_TRACE_TU(name)                                                                   \
  void trace_bind_##name(unsigned long long* buf, unsigned long long cap) {                  \
    CUDA_CHECK(cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(buf)));                          \
    CUDA_CHECK(cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap)));                          \
  }

// IEEE finiteness from the exponent bits (NaN and +-inf have an all-ones exponent): explicit
// so no compiler assumption about NaN can turn a check into |x| != inf.
__device__ __forceinline__ bool finite_f32(float x) { return ((__float_as_uint(x) >> 23) & 0xFFu) != 0xFFu; }

// binary16 storage emulation of the reference's PrecisionPolicy (half_round_value,
// tensor.cpp:97-121): round to nearest even fp16, >= 65520 -> +-inf, below 2^-25 -> 0
__device__ __forceinline__ float half_round(float x) { return __half2float(__float2half_rn(x)); }

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#endif  // __CUDACC__

}  // namespace glm
