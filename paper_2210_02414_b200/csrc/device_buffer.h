// device_buffer.h — owning RAII handle for one cudaMalloc allocation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace glm {

struct DeviceBuffer {
  void* ptr = nullptr;
  int64_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(int64_t n) { alloc(n); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(std::exchange(o.ptr, nullptr)), bytes(std::exchange(o.bytes, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      ptr = std::exchange(o.ptr, nullptr);
      bytes = std::exchange(o.bytes, 0);
    }
    return *this;
  }
  ~DeviceBuffer() { reset(); }
  void alloc(int64_t n) {
    reset();
    if (n > 0) {
      cudaError_t e = cudaMalloc(&ptr, static_cast<size_t>(n));
      if (e != cudaSuccess) {
        ptr = nullptr;
        fail(GLM_CUDA, "cuda", "cudaMalloc of " + std::to_string(n) + " bytes: " + cudaGetErrorString(e));
      }
    }
    bytes = n;
  }
  void reset() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

}  // namespace glm
