// Microbenchmark: TMEM -> register read throughput per SM on sm_100a
// (perf probing for the GEMM epilogue; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_read tmem_read.cu
// Prints bytes/clock/SM for tcgen05.ld shapes x warp counts.
#include <cstdint>
#include <cstdio>

#define DEVINL __device__ __forceinline__

DEVINL uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int N>
struct Ld;

#define REGS16(r, o)                                                                                       \
  "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]),         \
      "=r"(r[o + 6]), "=r"(r[o + 7]), "=r"(r[o + 8]), "=r"(r[o + 9]), "=r"(r[o + 10]), "=r"(r[o + 11]),   \
      "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]), "=r"(r[o + 15])

template <>
struct Ld<16> {  // 32x32b.x16: 32 lanes x 16 cols
  static DEVINL void run(uint32_t t, uint32_t (&r)[64]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : REGS16(r, 0)
                 : "r"(t));
  }
};
template <>
struct Ld<32> {
  static DEVINL void run(uint32_t t, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : REGS16(r, 0), REGS16(r, 16)
        : "r"(t));
  }
};
template <>
struct Ld<64> {
  static DEVINL void run(uint32_t t, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : REGS16(r, 0), REGS16(r, 16), REGS16(r, 32), REGS16(r, 48)
        : "r"(t));
  }
};
// 16x256b.x8: 16 lanes x 256 bits x 8 -> 32 regs per thread (same bytes as 32x32b.x32)
template <>
struct Ld<-8> {
  static DEVINL void run(uint32_t t, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : REGS16(r, 0), REGS16(r, 16)
        : "r"(t));
  }
};

template <int SHAPE, int REGS>
__global__ void __launch_bounds__(384, 1) bench(int iters, int warps, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  unsigned long long t0 = 0, t1 = 0;
  if (warp < static_cast<uint32_t>(warps)) {
    const uint32_t lane_base = (warp & 3) * 32;
    const uint32_t col_base = (warp >> 2) * 128;  // warps beyond 4 read other columns
    uint32_t r[64];
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 128; c += REGS) {
        Ld<SHAPE>::run(tmem + (lane_base << 16) + ((col_base + c) & 511), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < REGS; ++j) acc ^= r[j];
      }
    }
    t1 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int SHAPE, int REGS>
void run(const char* name, int warps) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  bench<SHAPE, REGS><<<148, 384>>>(10, warps, d, sink);
  bench<SHAPE, REGS><<<148, 384>>>(iters, warps, d, sink);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  // bytes per iteration per SM: warps x 32 lanes x 128 cols x 4 B
  const double bytes = static_cast<double>(iters) * warps * 32 * 128 * 4;
  printf("%-22s warps %2d: %7.1f B/clk/SM  (%s)\n", name, warps, bytes / avg, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 12}) {
    run<16, 16>("32x32b.x16", w);
    run<32, 32>("32x32b.x32", w);
    run<64, 64>("32x32b.x64", w);
  }
  return 0;
}
