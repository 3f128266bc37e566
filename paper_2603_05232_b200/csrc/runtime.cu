#include <cuda.h>
#include <mutex>
// C-ABI plumbing: versioning, status scratch, plan geometry, device checks.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "internal.h"

extern char** environ;

namespace slsp_host {

namespace {
using KnobSnapshot = std::vector<std::pair<std::string, std::string>>;
std::atomic<const KnobSnapshot*> g_knobs{nullptr};
std::mutex g_knobs_mu;

const KnobSnapshot* snapshot_knobs() {
  auto* snap = new KnobSnapshot();
  for (char** e = environ; e && *e; ++e) {
    if (std::strncmp(*e, "SLSP_", 5) != 0) continue;
    const char* eq = std::strchr(*e, '=');
    if (eq) snap->emplace_back(std::string(*e, eq - *e), std::string(eq + 1));
  }
  return snap;
}
}  // namespace

const char* knob_str(const char* name) {
  const KnobSnapshot* k = g_knobs.load(std::memory_order_acquire);
  if (!k) {
    std::lock_guard<std::mutex> g(g_knobs_mu);
    k = g_knobs.load(std::memory_order_acquire);
    if (!k) {
      k = snapshot_knobs();
      g_knobs.store(k, std::memory_order_release);
    }
  }
  for (const auto& kv : *k)
    if (kv.first == name) return kv.second.c_str();
  return nullptr;
}

int current_device(int* dev) {
  SLSP_CUDA_TRY(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= kMaxDevices) return SLSP_ERR_UNSUPPORTED;
  return SLSP_OK;
}

int num_sms() {
  static PerDevice<int> cache;
  int sms = 0;
  if (cache.get(&sms, [](int& v) -> int {
        int dev = 0;
        SLSP_CUDA_TRY(cudaGetDevice(&dev));
        SLSP_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v > 0 ? SLSP_OK : SLSP_ERR_CUDA;
      }))
    return 0;
  return sms;
}

static thread_local char g_last_cuda_error[256] = "";

int cuda_fail(cudaError_t e, const char* what) {
  std::snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", what, cudaGetErrorString(e));
  return SLSP_ERR_CUDA;
}

int plan(int z, int l, int* wc) {
  int starts[64];
  return slsp_plan_decomposition(z, l, 2, 4, wc, starts, 64);
}

int status_reset(void* status_ws, cudaStream_t s) {
  if (!status_ws) return SLSP_OK;
  SLSP_CUDA_TRY(cudaMemsetAsync(status_ws, 0xFF, SLSP_STATUS_WS_BYTES, s));
  return SLSP_OK;
}

int status_collect(void* status_ws, cudaStream_t s, int err_code, int64_t* row, int64_t* index) {
  if (!status_ws) return SLSP_OK;
  unsigned long long key = kNoError;
  SLSP_CUDA_TRY(cudaMemcpyAsync(&key, status_ws, sizeof(key), cudaMemcpyDeviceToHost, s));
  SLSP_CUDA_TRY(cudaStreamSynchronize(s));
  if (key == kNoError) return SLSP_OK;
  if (row) *row = static_cast<int64_t>(key >> 32);
  if (index) *index = static_cast<int64_t>(key & 0xFFFFFFFFull);
  return err_code;
}

int require_sm100() {
  int dev = 0;
  SLSP_CUDA_TRY(cudaGetDevice(&dev));
  if (!slsp_device_supported(dev)) {
    std::snprintf(g_last_cuda_error, sizeof(g_last_cuda_error),
                  "device %d is not an sm_100 (B200) GPU; the slsp_b200 kernels are sm_100a-only", dev);
    return SLSP_ERR_CUDA;
  }
  return SLSP_OK;
}

// Env SLSP_PDL: 1 on, 0 off, unset: on for calls over at most kPdlAutoRows
// tokens — decode / moderate M, where the launch gap and the GEMM prologue
// are a visible share (measured 1.5-2 us per lift + GEMM pair at M <= 64) —
// and off at large M (measured 1% slower on the M=8192 bench step).
bool pdl_enabled(int64_t rows) {
  constexpr int64_t kPdlAutoRows = 1024;
  const int64_t v = static_cast<int64_t>(knob("SLSP_PDL", 2));
  return v == 1 || (v == 2 && rows <= kPdlAutoRows);
}

}  // namespace slsp_host

extern "C" {

int slsp_version(void) { return 200; }

void slsp_reload_knobs(void) {
  // The previous snapshot is leaked on purpose: a concurrent reader may still
  // hold it (knobs are a probing aid, reloaded a handful of times per process).
  std::lock_guard<std::mutex> g(slsp_host::g_knobs_mu);
  slsp_host::g_knobs.store(slsp_host::snapshot_knobs(), std::memory_order_release);
}

const char* slsp_status_string(int status) {
  switch (status) {
    case SLSP_OK: return "ok";
    case SLSP_ERR_NOT_COMPLIANT: return "not compliant";
    case SLSP_ERR_DIMENSION: return "dimension mismatch";
    case SLSP_ERR_PLAN: return "invalid decomposition plan";
    case SLSP_ERR_NON_FINITE: return "non-finite input";
    case SLSP_ERR_INVALID: return "invalid argument";
    case SLSP_ERR_MALFORMED: return "malformed metadata";
    case SLSP_ERR_UNSUPPORTED: return "unsupported shape or type";
    case SLSP_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char* slsp_last_cuda_error(void) { return slsp_host::g_last_cuda_error; }

int slsp_device_supported(int dev) {
  // Cached per device: cudaGetDeviceProperties costs milliseconds and every
  // entry point checks the architecture (kernels are sm_100a-only).
  static int cache[64] = {0};  // 0 unknown, 1 supported, 2 not supported
  if (dev < 0) return 0;
  if (dev < 64 && cache[dev]) return cache[dev] == 1;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int ok = major == 10 && minor == 0;
  if (dev < 64) cache[dev] = ok ? 1 : 2;
  return ok;
}

// pattern.hpp:107-117 plan_status, pattern.hpp:131-154 plan_decomposition.
// density < hw_density is decided exactly by cross-multiplication.
int slsp_plan_decomposition(int z, int l, int hw_m, int hw_n, int* window_count, int* window_starts, int cap) {
  if (z <= 0 || l <= 0 || z > l || hw_m <= 0 || hw_m >= hw_n) return SLSP_ERR_INVALID;
  if (static_cast<int64_t>(z) * hw_n < static_cast<int64_t>(hw_m) * l) return SLSP_ERR_PLAN;
  const int stride = hw_n - hw_m;
  if (l < hw_n || (l - hw_n) % stride != 0) return SLSP_ERR_PLAN;
  const int wc = (l - hw_n) / stride + 1;
  if (static_cast<int64_t>(wc) * hw_m < z) return SLSP_ERR_PLAN;
  if (window_count) *window_count = wc;
  if (window_starts) {
    if (wc > cap) return SLSP_ERR_INVALID;
    for (int j = 0; j < wc; ++j) window_starts[j] = j * stride;
  }
  return SLSP_OK;
}

// Multi-GPU plumbing for the sharded lift: a rank's payload
// buffer is exported as a CUDA IPC handle (64 bytes, exchanged by the host
// over torch.distributed) and opened by every peer on the same node, so the
// lift kernel writes its K-slice into all ranks' payloads over NVLink.
// The handle names the whole cudaMalloc allocation holding ptr (a caching
// allocator hands out sub-ranges), so the byte offset of ptr inside it is
// returned too; the peer adds it to the base slsp_ipc_open_handle maps.
int slsp_ipc_get_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return SLSP_ERR_INVALID;
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<RangeFn>(fp);
  });
  if (!range) return SLSP_ERR_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return SLSP_ERR_CUDA;
  cudaIpcMemHandle_t h;
  SLSP_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return SLSP_OK;
}

int slsp_ipc_open_handle(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return SLSP_ERR_INVALID;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  SLSP_CUDA_TRY(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return SLSP_OK;
}

int slsp_ipc_close(void* ptr) {
  if (!ptr) return SLSP_ERR_INVALID;
  SLSP_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return SLSP_OK;
}

}  // extern "C"
