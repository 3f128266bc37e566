// TMA L2->SM ingest microbenchmark (perf probing, not a test).
//
// Persistent grid, one CTA per SM, a STAGES-deep shared-memory ring of
// NB x 16 KB boxes (128 rows x 128 B, 128B swizzle — the GEMM's A/B boxes).
// A producer thread issues the boxes, a consumer thread waits for them and
// frees the slot (no compute), so the loop runs at the rate the memory
// system delivers. Modes:
//   0 private   : every CTA streams its own L2-resident region
//   1 shared    : groups of G consecutive clusters stream the SAME region in
//                 lockstep-ish order (the GEMM raster's operand sharing)
//   2 multicast : within a cluster of CL CTAs, CTA r fetches boxes j % CL == r
//                 and multicasts them to every CTA of the cluster
//   3 dram      : private regions far larger than L2
// Prints delivered bytes per second (chip) and per SM clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_bw.cu -o tma_bw
//   ./tma_bw <cl> <mode> <stages> <nb> <ctas> <iters> [G]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
          su32(bar)),
      "r"(ph)
      : "memory");
}

struct P {
  int mode, stages, nb, iters, group, rows_per_cta, kblocks;
  unsigned long long* cyc;
};

template <int CL>
__global__ void __launch_bounds__(64, 1) bw_kernel(const __grid_constant__ CUtensorMap tm, const P p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages, NB = p.nb;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * NB * 16384);
  uint64_t* empty = full + S;
  const uint32_t cr = CL > 1 ? ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(CL));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (CL > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  const int cluster = blockIdx.x / CL;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    // region: rows [r0, r0 + NB*128)
    int region;
    if (p.mode == 1) region = cluster / p.group;
    else if (p.mode == 2) region = cluster;
    else region = blockIdx.x;
    const int r0 = region * p.rows_per_cta;
    uint32_t ph = 0;
    int s = 0;
    for (int it = 0; it < p.iters; ++it) {
      wait(&empty[s], ph ^ 1);
      const int kb = it % p.kblocks;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(NB * 16384)
                   : "memory");
      for (int j = 0; j < NB; ++j) {
        const uint32_t dst = su32(smem + (s * NB + j) * 16384);
        const int c0 = kb * 128, c1 = r0 + j * 128;
        if (p.mode == 2 && CL > 1) {
          if (j % CL == static_cast<int>(cr)) {
            const uint16_t mask = static_cast<uint16_t>((1u << CL) - 1);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&full[s])), "r"(c0), "r"(c1), "h"(mask)
                : "memory");
          }
        } else {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&full[s])), "r"(c0), "r"(c1)
              : "memory");
        }
      }
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    uint32_t ph = 0;
    int s = 0;
    for (int it = 0; it < p.iters; ++it) {
      wait(&full[s], ph);
      for (int r = 0; r < CL; ++r)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(su32(&empty[s]), r)) : "memory");
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p.cyc[blockIdx.x] = clock64() - t0;
  if (CL > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int CL>
void run(int mode, int S, int NB, int ctas, int iters, int group) {
  const int width = mode == 3 ? 5376 : 1024;  // bytes per row
  const int kblocks = width / 128;
  const int rows_per_cta = NB * 128;
  const int regions = ctas;
  const size_t rows = static_cast<size_t>(regions) * rows_per_cta;
  uint8_t* buf;
  CK(cudaMalloc(&buf, rows * width));
  CK(cudaMemset(buf, 1, rows * width));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(width), rows};
  cuuint64_t str[1] = {static_cast<cuuint64_t>(width)};
  cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", r);
    exit(1);
  }
  P p{mode, S, NB, iters, group, rows_per_cta, kblocks, nullptr};
  CK(cudaMalloc(&p.cyc, ctas * 8));
  const int smem = S * NB * 16384 + 2 * S * 8 + 1024;
  CK(cudaFuncSetAttribute(bw_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, bw_kernel<CL>, tm, p));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  std::vector<unsigned long long> cyc(ctas);
  CK(cudaMemcpy(cyc.data(), p.cyc, ctas * 8, cudaMemcpyDeviceToHost));
  unsigned long long mx = 0;
  for (auto c : cyc) mx = c > mx ? c : mx;
  const double bytes = static_cast<double>(ctas) * iters * NB * 16384.0;
  const double l2bytes = mode == 2 ? bytes / CL : bytes;
  printf("cl %d mode %d stages %d nb %d (stage %3d KB, ring %3d KB) ctas %3d group %2d: %7.3f ms  delivered %6.2f TB/s"
         "  L2-read %6.2f TB/s  %6.1f B/clk/SM  (%.0f MHz eff)\n",
         CL, mode, S, NB, NB * 16, S * NB * 16, ctas, group, best, bytes / best / 1e9, l2bytes / best / 1e9,
         bytes / ctas / static_cast<double>(mx), static_cast<double>(mx) / best / 1e3);
  cudaFree(buf);
  cudaFree(p.cyc);
}

int main(int argc, char** argv) {
  if (argc < 7) {
    printf("usage: tma_bw cl mode stages nb ctas iters [group]\n");
    return 1;
  }
  const int cl = atoi(argv[1]), mode = atoi(argv[2]), S = atoi(argv[3]), NB = atoi(argv[4]), ctas = atoi(argv[5]),
            iters = atoi(argv[6]), group = argc > 7 ? atoi(argv[7]) : 1;
  if (cl == 1) run<1>(mode, S, NB, ctas, iters, group);
  else if (cl == 2) run<2>(mode, S, NB, ctas, iters, group);
  else if (cl == 4) run<4>(mode, S, NB, ctas, iters, group);
  else if (cl == 8) run<8>(mode, S, NB, ctas, iters, group);
  return 0;
}
