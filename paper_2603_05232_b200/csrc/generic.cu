// The reference's generic GEMM instantiations (gemm.hpp:142-197) for the C++
// drop-in's Matrix<int> / Matrix<float> calls, on the CUDA cores: int32
// inputs accumulate in int64, float inputs in double, one thread per output
// element in the reference's left-to-right order. Products of two int32 /
// two floats are exact in int64 / double, so each sum rounds exactly as the
// reference's does: the results are bit-identical at any size. The int8 /
// e4m3 / bf16 paths are the tcgen05 kernels (gemm.cu); these exist so the
// drop-in API is complete, not for speed.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace {

template <typename T, typename Acc>
__global__ void generic_dense_kernel(const T* __restrict__ w, int64_t n, int64_t k, const T* __restrict__ x,
                                     int64_t m, Acc* __restrict__ y) {
  const int64_t total = n * m;
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = o / m, t = o - i * m;  // consecutive threads: consecutive tokens (coalesced x reads)
    Acc acc = 0;
    for (int64_t kk = 0; kk < k; ++kk) acc += static_cast<Acc>(w[i * k + kk]) * static_cast<Acc>(x[kk * m + t]);
    y[o] = acc;
  }
}

template <typename T, typename Acc>
__global__ void generic_sparse_kernel(const T* __restrict__ vals, const uint8_t* __restrict__ codes, int64_t rows,
                                      int64_t windows, int hw_m, int hw_n, const T* __restrict__ lifted, int64_t m,
                                      Acc* __restrict__ y, unsigned long long* status) {
  const int64_t total = rows * m;
  const int64_t width = windows * hw_n;
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = o / m, t = o - i * m;
    const T* v = vals + i * windows * hw_m;
    const uint8_t* c = codes + i * windows * hw_m;
    const T* act = lifted + t * width;
    Acc acc = 0;
    for (int64_t wi = 0; wi < windows; ++wi)
      for (int kk = 0; kk < hw_m; ++kk) {
        const int d = c[wi * hw_m + kk];
        if (d >= hw_n) {  // would gather outside the window
          if (status) atomicMin(status, static_cast<unsigned long long>(i) << 32);
          continue;
        }
        acc += static_cast<Acc>(v[wi * hw_m + kk]) * static_cast<Acc>(act[wi * hw_n + d]);
      }
    y[o] = acc;
  }
}

unsigned grid_of(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

extern "C" {

int slsp_generic_dense_gemm(int dtype, const void* w, int64_t n, int64_t k, const void* x, int64_t m, void* y,
                            slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || k < 0 || m < 0) return SLSP_ERR_INVALID;
  if (dtype != SLSP_DT_I32 && dtype != SLSP_DT_F32) return SLSP_ERR_UNSUPPORTED;
  int st;
  if ((st = require_sm100())) return st;
  if (n == 0 || m == 0) return SLSP_OK;
  if (dtype == SLSP_DT_I32)
    generic_dense_kernel<int32_t, long long><<<grid_of(n * m), 256, 0, s>>>(
        static_cast<const int32_t*>(w), n, k, static_cast<const int32_t*>(x), m, static_cast<long long*>(y));
  else
    generic_dense_kernel<float, double><<<grid_of(n * m), 256, 0, s>>>(static_cast<const float*>(w), n, k,
                                                                      static_cast<const float*>(x), m,
                                                                      static_cast<double*>(y));
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

int slsp_generic_sparse_gemm(int dtype, const void* values, const uint8_t* codes, int64_t rows, int64_t windows,
                             int hw_m, int hw_n, const void* lifted, int64_t m, void* y, void* status_ws,
                             int64_t* bad_row, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (rows < 0 || windows < 0 || m < 0 || hw_m <= 0 || hw_n <= 0 || hw_m > hw_n) return SLSP_ERR_INVALID;
  if (dtype != SLSP_DT_I32 && dtype != SLSP_DT_F32) return SLSP_ERR_UNSUPPORTED;
  int st;
  if ((st = require_sm100())) return st;
  if (rows == 0 || m == 0) return SLSP_OK;
  if (status_ws && (st = status_reset(status_ws, s))) return st;
  auto* status = static_cast<unsigned long long*>(status_ws);
  if (dtype == SLSP_DT_I32)
    generic_sparse_kernel<int32_t, long long><<<grid_of(rows * m), 256, 0, s>>>(
        static_cast<const int32_t*>(values), codes, rows, windows, hw_m, hw_n, static_cast<const int32_t*>(lifted), m,
        static_cast<long long*>(y), status);
  else
    generic_sparse_kernel<float, double><<<grid_of(rows * m), 256, 0, s>>>(
        static_cast<const float*>(values), codes, rows, windows, hw_m, hw_n, static_cast<const float*>(lifted), m,
        static_cast<double*>(y), status);
  SLSP_LAUNCH_CHECK();
  return status_ws ? status_collect(status_ws, s, SLSP_ERR_MALFORMED, bad_row, nullptr) : SLSP_OK;
}

}  // extern "C"
