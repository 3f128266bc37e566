// Which SM does each CTA of a persistent cluster-of-2 grid (one CTA per SM,
// 200 KB smem) land on? Prints blockIdx -> %smid, the cluster's GPC grouping
// hint (%nsmid) — input for die-aware scheduling experiments.
#include <cstdio>
__global__ void __cluster_dims__(2, 1, 1) k(int* out) {
  extern __shared__ char s[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  s[threadIdx.x] = 0;
}
int main() {
  int* d;
  cudaMalloc(&d, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int h[148];
  for (int rep = 0; rep < 2; ++rep) {
    k<<<148, 128, 200 * 1024>>>(d);
    cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    printf("rep %d:", rep);
    for (int i = 0; i < 148; ++i) printf(" %d", h[i]);
    printf("\n");
  }
  return 0;
}
