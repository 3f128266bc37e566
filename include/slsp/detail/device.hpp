#pragma once
// Host<->device plumbing for the C++ drop-in layer: RAII device buffers on the
// CUDA runtime, the element-type map to the C ABI, and status -> exception
// translation with the reference's messages.

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "slsp/pattern.hpp"
#include "slsp_b200.h"

namespace slsp::detail {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string("slsp_b200 CUDA failure in ") + what + ": " + cudaGetErrorString(e));
}

// Device allocations of the drop-in calls come from a small process-wide
// cache of power-of-two blocks: the reference API is called per row / per
// small matrix in loops, and cudaMalloc + cudaFree (a device-wide sync) per
// call would dominate. Blocks are reused per device; at most kPoolBytes are
// kept idle.
class DevicePool {
 public:
  static DevicePool& get() {
    static DevicePool pool;
    return pool;
  }
  void* acquire(std::size_t bytes, std::size_t* cap) {
    const std::size_t c = bucket(bytes);
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    {
      std::lock_guard<std::mutex> g(mu_);
      auto& fl = free_[key(dev, c)];
      if (!fl.empty()) {
        void* p = fl.back();
        fl.pop_back();
        idle_ -= c;
        *cap = c;
        return p;
      }
    }
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, c), "cudaMalloc");
    *cap = c;
    return p;
  }
  void release(void* p, std::size_t c) {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      std::lock_guard<std::mutex> g(mu_);
      if (idle_ + c <= kPoolBytes) {
        free_[key(dev, c)].push_back(p);
        idle_ += c;
        return;
      }
    }
    cudaFree(p);
  }

 private:
  static constexpr std::size_t kPoolBytes = std::size_t{1} << 30;
  static std::size_t bucket(std::size_t b) {
    std::size_t c = 256;
    while (c < b) c <<= 1;
    return c;
  }
  static std::uint64_t key(int dev, std::size_t c) { return (static_cast<std::uint64_t>(dev) << 56) | c; }
  std::mutex mu_;
  std::unordered_map<std::uint64_t, std::vector<void*>> free_;
  std::size_t idle_ = 0;
};

template <typename T>
class DeviceBuffer {
 public:
  explicit DeviceBuffer(std::size_t count) : n_(count) {
    if (n_) p_ = DevicePool::get().acquire(n_ * sizeof(T), &cap_);
  }
  explicit DeviceBuffer(const std::vector<T>& host) : DeviceBuffer(host.size()) { upload(host.data(), host.size()); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p_) DevicePool::get().release(p_, cap_);
  }
  T* get() const { return static_cast<T*>(p_); }
  std::size_t size() const { return n_; }
  void upload(const T* src, std::size_t count) {
    if (count) cuda_check(cudaMemcpy(p_, src, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  std::vector<T> download(std::size_t count) const {
    std::vector<T> out(count);
    if (count) cuda_check(cudaMemcpy(out.data(), p_, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    return out;
  }
  std::vector<T> download() const { return download(n_); }

 private:
  void* p_ = nullptr;
  std::size_t n_ = 0;
  std::size_t cap_ = 0;
};

// Element types the B200 kernels take (the reference is generic in T).
template <typename T>
constexpr int dtype_code() {
  if constexpr (std::is_same_v<T, std::int8_t>) return SLSP_DT_I8;
  else if constexpr (std::is_same_v<T, std::int32_t>) return SLSP_DT_I32;
  else if constexpr (std::is_same_v<T, float>) return SLSP_DT_F32;
  else if constexpr (std::is_same_v<T, double>) return SLSP_DT_F64;
  else return -1;
}

struct StatusScratch {
  DeviceBuffer<std::uint8_t> buf{SLSP_STATUS_WS_BYTES};
  void* get() const { return buf.get(); }
};

// Maps a C-ABI status to the reference's exception (pattern.hpp:24-57).
inline void raise(int status, const std::string& what) {
  switch (status) {
    case SLSP_OK: return;
    case SLSP_ERR_NOT_COMPLIANT: throw NotCompliantError(what);
    case SLSP_ERR_DIMENSION: throw DimensionMismatchError(what);
    case SLSP_ERR_NON_FINITE: throw NonFiniteInputError(what);
    case SLSP_ERR_MALFORMED: throw MalformedMetadataError(what);
    case SLSP_ERR_PLAN: throw AlreadyCompliantError(what);
    case SLSP_ERR_INVALID: throw std::invalid_argument(what);
    case SLSP_ERR_UNSUPPORTED: throw std::invalid_argument("unsupported on the B200 path: " + what);
    default: throw Error(what + ": " + slsp_status_string(status) + " (" + slsp_last_cuda_error() + ")");
  }
}

}  // namespace slsp::detail
