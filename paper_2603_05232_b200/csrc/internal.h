// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>
#include <utility>

#include "../../include/slsp_b200.h"

namespace slsp_host {

// Records the CUDA error text for slsp_last_cuda_error() and returns SLSP_ERR_CUDA.
int cuda_fail(cudaError_t e, const char* what);

#define SLSP_CUDA_TRY(expr)                                  \
  do {                                                       \
    cudaError_t e__ = (expr);                                \
    if (e__ != cudaSuccess) return ::slsp_host::cuda_fail(e__, #expr); \
  } while (0)

#define SLSP_LAUNCH_CHECK() SLSP_CUDA_TRY(cudaGetLastError())

// Window plan for hw 2:4 (pattern.hpp:107-154). Returns SLSP_OK or SLSP_ERR_PLAN/INVALID.
int plan(int z, int l, int* wc);

// Sentinel written into the status scratch before a checking kernel.
constexpr unsigned long long kNoError = ~0ull;

// Clears the status scratch (async).
int status_reset(void* status_ws, cudaStream_t s);
// Synchronises `s`, reads the min-reduced (row << 32 | index) key.
// Returns SLSP_OK when no error was recorded, else `err_code` with the location.
int status_collect(void* status_ws, cudaStream_t s, int err_code, int64_t* row, int64_t* index);

// Current device must be sm_100 (B200); fails loudly otherwise.
int require_sm100();

// Programmatic dependent launch for the hot kernels over `rows` tokens
// (env SLSP_PDL; see runtime.cu). Every PDL-launched kernel waits
// (griddepcontrol.wait) before touching memory a predecessor may write.
bool pdl_enabled(int64_t rows);

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute
// (PDL) when enabled; plain launch semantics otherwise.
template <typename... KArgs, typename... Args>
int launch_pdl(int64_t rows, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
               Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled(rows) ? 1 : 0;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SLSP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return SLSP_OK;
}

// ---- tuning / probing knobs -------------------------------------------------
// SLSP_* environment variables are snapshotted once (first use) and again on
// slsp_reload_knobs(), so an entry point reads a handful of cached pairs
// instead of scanning the process environment on every call.
const char* knob_str(const char* name);  // nullptr when unset
inline uint64_t knob(const char* name, uint64_t dflt) {
  const char* e = knob_str(name);
  return (e && *e) ? static_cast<uint64_t>(std::strtoull(e, nullptr, 0)) : dflt;
}

// ---- per-device host state -------------------------------------------------
// Launch attributes, occupancy-derived grid caps and uploaded tables are
// device properties: a process that drives several GPUs through the C ABI
// computes each once per device (never "once per process").
constexpr int kMaxDevices = 64;

int current_device(int* dev);  // SLSP_OK, or SLSP_ERR_CUDA / SLSP_ERR_UNSUPPORTED

template <typename T>
struct PerDevice {
  std::mutex mu;
  bool done[kMaxDevices] = {};
  T val[kMaxDevices] = {};
  // The current device's value, computed by init(T&) -> status on first use
  // (failures are not cached).
  template <typename F>
  int get(T* out, F&& init) {
    int dev = 0;
    int st = current_device(&dev);
    if (st) return st;
    std::lock_guard<std::mutex> g(mu);
    if (!done[dev]) {
      if ((st = init(val[dev]))) return st;
      done[dev] = true;
    }
    *out = val[dev];
    return SLSP_OK;
  }
};

// Number of SMs of the current device (cached per device); 0 on failure.
int num_sms();

inline int elem_size(int dtype) {
  switch (dtype) {
    case SLSP_DT_I8:
    case SLSP_DT_E4M3:
      return 1;
    case SLSP_DT_BF16:
      return 2;
    case SLSP_DT_F32:
    case SLSP_DT_I32:
      return 4;
    case SLSP_DT_F64:
      return 8;
    default:
      return 0;
  }
}

}  // namespace slsp_host
