// Layout probe (perf/design probing, not part of the library): which TMEM
// (lane, column) each thread receives from tcgen05.ld.16x256b.x1, and where
// stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 puts fragment elements.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_layout tmem_layout.cu && ./tmem_layout
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(uint32_t* out_ld, uint16_t* out_st, uint32_t* out_x4) {
  __shared__ uint32_t slot;
  __shared__ __align__(128) uint16_t st[4 * 64];
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = lane * 256 + c;  // lane = TMEM row
    for (int c8 = 0; c8 < 4; ++c8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + c8 * 8),
                   "r"(v[c8 * 8 + 0]), "r"(v[c8 * 8 + 1]), "r"(v[c8 * 8 + 2]), "r"(v[c8 * 8 + 3]), "r"(v[c8 * 8 + 4]),
                   "r"(v[c8 * 8 + 5]), "r"(v[c8 * 8 + 6]), "r"(v[c8 * 8 + 7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; ++i) out_ld[lane * 4 + i] = r[i];
    uint32_t q[16];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                   "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
                 : "r"(tmem + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) out_x4[lane * 16 + i] = q[i];
    // stmatrix: fragment register i of thread T = code (matrix i, T) so the dump shows the mapping
    uint32_t f[4];
    for (int i = 0; i < 4; ++i) f[i] = ((i * 32 + lane) << 16) | 0x8000u | (i * 32 + lane);
    // rows of the stored (transposed) matrices: lanes 8i..8i+7 give matrix i's row addresses, 16 B per row
    const uint32_t addr = smem_u32(st) + (lane >> 3) * 128 + (lane & 7) * 16;
    asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(f[0]),
                 "r"(f[1]), "r"(f[2]), "r"(f[3]));
    __syncwarp();
    for (int i = lane; i < 4 * 64; i += 32) out_st[i] = st[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  uint32_t* d_ld;
  uint16_t* d_st;
  uint32_t* d_x4;
  cudaMalloc(&d_x4, 32 * 16 * 4);
  cudaMalloc(&d_ld, 32 * 4 * 4);
  cudaMalloc(&d_st, 4 * 64 * 2);
  probe<<<1, 32>>>(d_ld, d_st, d_x4);
  uint32_t h_x4[512];
  cudaMemcpy(h_x4, d_x4, sizeof(h_x4), cudaMemcpyDeviceToHost);
  printf("16x256b.x4 at lane 16: thread T -> (row,col) of r0..r15\n");
  for (int t = 0; t < 8; ++t) {
    printf("T%2d:", t);
    for (int i = 0; i < 16; ++i) printf(" (%u,%u)", h_x4[t * 16 + i] >> 8, h_x4[t * 16 + i] & 255);
    printf("\n");
  }
  uint32_t h_ld[128];
  uint16_t h_st[256];
  cudaMemcpy(h_ld, d_ld, sizeof(h_ld), cudaMemcpyDeviceToHost);
  cudaMemcpy(h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("16x256b.x1: thread T -> (row,col) of r0..r3\n");
  for (int t = 0; t < 32; ++t) {
    printf("T%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" (%u,%u)", h_ld[t * 4 + i] >> 8, h_ld[t * 4 + i] & 255);
    printf("\n");
  }
  printf("stmatrix.x4.trans: stored row r (16 B = 8 b16) of matrix m: element j = (reg i, thread T, half h)\n");
  for (int m = 0; m < 4; ++m)
    for (int r = 0; r < 8; ++r) {
      printf("m%d row%d:", m, r);
      for (int j = 0; j < 8; ++j) {
        const uint16_t e = h_st[m * 64 + r * 8 + j];
        const int code = e & 0x7FFF, hi = (e & 0x8000) ? 0 : 1;  // low half carries 0x8000|code, high half code
        printf(" [r%d T%d %s]", code / 32, code % 32, hi ? "hi" : "lo");
      }
      printf("\n");
    }
  return 0;
}
