// Offline weight transform Φ on sm_100a: Sliding Window Decomposition packer,
// compressor and magnitude pruner.
//
// Memory-bound integer/byte work: one thread per l-element source block
// ("group"); the greedy placement depends only on the block's l-bit nonzero
// mask, so it runs in registers on bit masks. Outputs are staged in shared
// memory per 256-group chunk and written back with 32-bit coalesced stores.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace slsp_dev;

constexpr int kThreads = 256;
constexpr int kMaxL = 32;

// matrix.hpp:63-67 is_nonzero (v != T{}): -0.0 is zero, NaN is nonzero.
// e4m3 codes are judged by decoded value: 0x00 and 0x80 are zero.
template <int ESZ>
SLSP_DEVINL bool nonzero_bits(uint64_t bits, int dtype) {
  if constexpr (ESZ == 1) return dtype == SLSP_DT_E4M3 ? (bits & 0x7Fu) != 0 : (bits & 0xFFu) != 0;
  if constexpr (ESZ == 2) return (bits & 0x7FFFu) != 0;
  if constexpr (ESZ == 4) return dtype == SLSP_DT_I32 ? (bits & 0xFFFFFFFFu) != 0 : (bits & 0x7FFFFFFFu) != 0;
  return (bits & 0x7FFFFFFFFFFFFFFFull) != 0;
}

template <int ESZ>
SLSP_DEVINL uint64_t load_elem(const uint8_t* base, int64_t idx) {
  if constexpr (ESZ == 1) return __ldg(base + idx);
  if constexpr (ESZ == 2) return __ldg(reinterpret_cast<const uint16_t*>(base) + idx);
  if constexpr (ESZ == 4) return __ldg(reinterpret_cast<const uint32_t*>(base) + idx);
  return __ldg(reinterpret_cast<const unsigned long long*>(base) + idx);
}

template <int ESZ>
SLSP_DEVINL void store_elem(uint8_t* base, int64_t idx, uint64_t v) {
  if constexpr (ESZ == 1) base[idx] = static_cast<uint8_t>(v);
  if constexpr (ESZ == 2) reinterpret_cast<uint16_t*>(base)[idx] = static_cast<uint16_t>(v);
  if constexpr (ESZ == 4) reinterpret_cast<uint32_t*>(base)[idx] = static_cast<uint32_t>(v);
  if constexpr (ESZ == 8) reinterpret_cast<unsigned long long*>(base)[idx] = v;
}

SLSP_DEVINL void record_error(unsigned long long* status, int64_t row, int64_t index) {
  if (status) atomicMin(status, (static_cast<unsigned long long>(row) << 32) | static_cast<unsigned long long>(index));
}

// Block-cooperative copy smem -> global: 32-bit stores when the destination
// is 4-byte aligned, bytes otherwise.
SLSP_DEVINL void copy_out(uint8_t* dst, const uint8_t* src, int64_t nbytes) {
  if ((reinterpret_cast<uintptr_t>(dst) & 3u) == 0) {
    const int64_t nw = nbytes >> 2;
    for (int64_t i = threadIdx.x; i < nw; i += blockDim.x)
      reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
    for (int64_t i = (nw << 2) + threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
  } else {
    for (int64_t i = threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
  }
}

struct PackArgs {
  const uint8_t* w;
  int64_t rows, cols;
  int z, l, wc, dtype;
  int64_t groups_real;  // ceil(cols / l)
  int64_t group_slots;  // groups covering the output width
  int64_t out_windows;  // windows written per row
  uint8_t* out_a;       // MODE 0: slided; MODE 1: values
  uint8_t* out_meta;    // MODE 1: packed codes
  int64_t ld_a_bytes;   // row stride of out_a in bytes
  int64_t ld_meta;      // row stride of out_meta in bytes
  unsigned long long* status;
};

// MODE 0: pack_matrix (pack.hpp:171-204) -> slided rows of wc*4 per group.
// MODE 1: pack + compress fused (pack.hpp:83-122 + gemm.hpp:70-110) ->
//         values (2 per window) + packed 2-bit codes (container.hpp:330-336).
template <int ESZ, int MODE>
__global__ void __launch_bounds__(kThreads) pack_kernel(PackArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int wc = a.wc;
  const int64_t chunk = blockIdx.x;
  const int64_t gs = chunk * kThreads + threadIdx.x;
  const int64_t win0 = chunk * kThreads * wc;  // first window of this chunk
  const int64_t chunk_windows = imin64(static_cast<int64_t>(kThreads) * wc, a.out_windows - win0);
  // MODE 1 staging: values [kThreads*wc*2*ESZ] then meta words; MODE 0: slided.
  uint8_t* s_vals = smem;
  uint32_t* s_meta = reinterpret_cast<uint32_t*>(smem + kThreads * wc * 2 * ESZ);
  const int meta_words = (kThreads * wc + 7) / 8;

  for (int64_t row = blockIdx.y; row < a.rows; row += gridDim.y) {
    if (MODE == 1)
      for (int i = threadIdx.x; i < meta_words; i += kThreads) s_meta[i] = 0;
    __syncthreads();
    if (gs < a.group_slots) {
      const uint8_t* src = a.w + (row * a.cols) * ESZ;
      const int64_t col0 = gs * a.l;
      uint32_t mask = 0;
      if (gs < a.groups_real) {
        for (int k = 0; k < a.l; ++k) {
          const int64_t col = col0 + k;
          if (col < a.cols && nonzero_bits<ESZ>(load_elem<ESZ>(src, col), a.dtype)) mask |= 1u << k;
        }
      }
      if (__popc(mask) > a.z) {
        record_error(a.status, row, gs);  // first_overfull_block, pack.hpp:124-133
      }
      // greedy_pack_row (pack.hpp:94-111): windows in order, offsets in order,
      // accept an unused nonzero while the window holds < 2.
      uint32_t used = 0;
      for (int w = 0; w < wc; ++w) {
        const int s = 2 * w;
        int p[2] = {-1, -1};
        int cnt = 0;
        for (int d = 0; d < 4; ++d) {
          const int k = s + d;
          if (((mask >> k) & 1u) && !((used >> k) & 1u) && cnt < 2) {
            used |= 1u << k;
            p[cnt++] = d;
          }
        }
        const int64_t wl = static_cast<int64_t>(threadIdx.x) * wc + w;  // window index within chunk
        if (wl >= chunk_windows) continue;
        if (MODE == 0) {
          uint8_t* dst = s_vals + wl * 4 * ESZ;
          for (int d = 0; d < 4; ++d) {
            const bool take = (p[0] == d) || (p[1] == d);
            store_elem<ESZ>(dst, d, take ? load_elem<ESZ>(src, col0 + s + d) : 0ull);
          }
        } else {
          // compress canonical padding (gemm.hpp:99-102): fill with the
          // smallest unused positions, then sort; padded values are T{}.
          uint64_t v0 = 0, v1 = 0;
          int c0, c1;
          if (cnt == 2) {
            c0 = p[0];
            c1 = p[1];
            v0 = load_elem<ESZ>(src, col0 + s + c0);
            v1 = load_elem<ESZ>(src, col0 + s + c1);
          } else if (cnt == 1) {
            const uint64_t v = load_elem<ESZ>(src, col0 + s + p[0]);
            if (p[0] == 0) {
              c0 = 0; c1 = 1; v0 = v;
            } else {
              c0 = 0; c1 = p[0]; v1 = v;
            }
          } else {
            c0 = 0;
            c1 = 1;
          }
          store_elem<ESZ>(s_vals, wl * 2, v0);
          store_elem<ESZ>(s_vals, wl * 2 + 1, v1);
          const uint32_t nib = static_cast<uint32_t>(c0 | (c1 << 2));
          atomicOr(&s_meta[wl >> 3], nib << (4 * (wl & 7)));
        }
      }
      if (mask & ~used) record_error(a.status, row, gs);  // leftover, pack.hpp:112-119
    }
    __syncthreads();
    if (chunk_windows > 0) {
      if (MODE == 0) {
        copy_out(a.out_a + row * a.ld_a_bytes + win0 * 4 * ESZ, s_vals, chunk_windows * 4 * ESZ);
      } else {
        copy_out(a.out_a + row * a.ld_a_bytes + win0 * 2 * ESZ, s_vals, chunk_windows * 2 * ESZ);
        copy_out(a.out_meta + row * a.ld_meta + win0 / 2, reinterpret_cast<const uint8_t*>(s_meta),
                 (chunk_windows + 1) / 2);
      }
    }
    __syncthreads();
  }
}

// gemm.hpp:70-110 compress: one thread per 4-window of a slided row.
template <int ESZ>
__global__ void compress_kernel(const uint8_t* slided, int64_t rows, int64_t wpr, int dtype, uint8_t* values,
                                uint8_t* codes, unsigned long long* status) {
  const int64_t total = rows * wpr;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t v[4];
    int pos[4], np = 0;
    for (int d = 0; d < 4; ++d) {
      v[d] = load_elem<ESZ>(slided, i * 4 + d);
      if (nonzero_bits<ESZ>(v[d], dtype)) pos[np++] = d;
    }
    if (np > 2) {
      record_error(status, i / wpr, i % wpr);
      continue;
    }
    for (int d = 0; np < 2; ++d) {
      bool found = false;
      for (int j = 0; j < np; ++j) found |= pos[j] == d;
      if (!found) pos[np++] = d;
    }
    if (pos[0] > pos[1]) {
      const int t = pos[0];
      pos[0] = pos[1];
      pos[1] = t;
    }
    store_elem<ESZ>(values, i * 2, v[pos[0]]);
    store_elem<ESZ>(values, i * 2 + 1, v[pos[1]]);
    codes[i * 2] = static_cast<uint8_t>(pos[0]);
    codes[i * 2 + 1] = static_cast<uint8_t>(pos[1]);
  }
}

// pack.hpp:238-261 magnitude_prune: zero the l-z smallest |v| per block,
// ties pruned lower-index first (stable_sort order). One thread per block.
template <int ESZ>
SLSP_DEVINL double magnitude(uint64_t bits, int dtype) {
  if constexpr (ESZ == 1) {
    if (dtype == SLSP_DT_E4M3) return fabs(static_cast<double>(fp8_e4m3_decode(static_cast<uint8_t>(bits))));
    return fabs(static_cast<double>(static_cast<int8_t>(bits)));
  }
  if constexpr (ESZ == 2) return fabs(static_cast<double>(__uint_as_float(static_cast<uint32_t>(bits) << 16)));
  if constexpr (ESZ == 4) {
    if (dtype == SLSP_DT_I32) return fabs(static_cast<double>(static_cast<int32_t>(static_cast<uint32_t>(bits))));
    return fabs(static_cast<double>(__uint_as_float(static_cast<uint32_t>(bits))));
  }
  return fabs(__longlong_as_double(static_cast<long long>(bits)));
}

template <int ESZ>
__global__ void prune_kernel(const uint8_t* w, int64_t rows, int64_t cols, int z, int l, int dtype, uint8_t* out) {
  const int64_t groups = cols / l;
  const int64_t total = rows * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t base = i * l;  // rows are contiguous blocks of cols = groups*l
    double mag[kMaxL];
    for (int k = 0; k < l; ++k) mag[k] = magnitude<ESZ>(load_elem<ESZ>(w, base + k), dtype);
    const int prune = l - z;
    for (int k = 0; k < l; ++k) {
      int rank = 0;
      for (int j = 0; j < l; ++j) rank += (mag[j] < mag[k]) || (mag[j] == mag[k] && j < k);
      store_elem<ESZ>(out, base + k, rank < prune ? 0ull : load_elem<ESZ>(w, base + k));
    }
  }
}

// ---------------------------------------------------------------------------
// 6:8 fast path. The greedy placement (pack.hpp:94-111) plus compress's
// canonical padding (gemm.hpp:99-102) is a pure function of the block's 8-bit
// nonzero mask, so it is tabulated once on the host (build_lut8, the same
// greedy) into 256 entries: per window w, bits [16w, 16w+12) hold the 2-bit
// code pair (4 bits) and the source offsets of the two value slots (4 bits
// each, 8 = padding zero). A thread packs 8 consecutive blocks from 4*ESZ
// 16-byte loads into 48*ESZ value bytes and 12 metadata bytes (vector stores).
struct Lut8 {
  unsigned long long e[256];
};

Lut8 build_lut8() {
  Lut8 t{};
  for (int mask = 0; mask < 256; ++mask) {
    unsigned used = 0;
    unsigned long long entry = 0;
    for (int w = 0; w < 3; ++w) {
      int p[2] = {-1, -1}, cnt = 0;
      for (int d = 0; d < 4; ++d) {
        const int k = 2 * w + d;
        if (((mask >> k) & 1) && !((used >> k) & 1) && cnt < 2) {
          used |= 1u << k;
          p[cnt++] = d;
        }
      }
      int c0, c1, s0 = 8, s1 = 8;  // codes and value sources (8 = zero)
      if (cnt == 2) {
        c0 = p[0], c1 = p[1], s0 = 2 * w + p[0], s1 = 2 * w + p[1];
      } else if (cnt == 1) {
        if (p[0] == 0) c0 = 0, c1 = 1, s0 = 2 * w;
        else c0 = 0, c1 = p[0], s1 = 2 * w + p[0];
      } else {
        c0 = 0, c1 = 1;
      }
      const unsigned long long f = static_cast<unsigned long long>((c0 | (c1 << 2)) | (s0 << 4) | (s1 << 8));
      entry |= f << (16 * w);
    }
    t.e[mask] = entry;
  }
  return t;
}

template <int ESZ>
__global__ void __launch_bounds__(256) pack68_kernel(const uint8_t* __restrict__ w, int64_t rows, int64_t cols,
                                                     int z, int dtype, Lut8 lut, uint8_t* __restrict__ values,
                                                     int64_t ld_vals, uint8_t* __restrict__ meta, int64_t ld_meta,
                                                     unsigned long long* status) {
  __shared__ unsigned long long s_lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = lut.e[i];
  __syncthreads();
  const int64_t octs = cols / 64;  // 8 blocks of 8 per thread
  const int64_t total = rows * octs;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx / octs, q = idx - row * octs;
    const uint4* src = reinterpret_cast<const uint4*>(w + (row * cols + q * 64) * ESZ);
    uint4 v[4 * ESZ];
#pragma unroll
    for (int i = 0; i < 4 * ESZ; ++i) v[i] = __ldg(src + i);
    const unsigned long long* x = reinterpret_cast<const unsigned long long*>(v);  // 8*ESZ bytes per block
    uint32_t ov[12 * ESZ];
    uint32_t om[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < 12 * ESZ; ++i) ov[i] = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      uint32_t mask = 0;
      if constexpr (ESZ == 1) {
        // byte b nonzero (e4m3: ignoring the sign bit) -> bit b
        const unsigned long long m7 = 0x7F7F7F7F7F7F7F7Full;
        const unsigned long long b = dtype == SLSP_DT_E4M3 ? (x[g] & m7) : x[g];
        const unsigned long long t = (((b & m7) + m7) | b) & 0x8080808080808080ull;
        mask = static_cast<uint32_t>(((t >> 7) * 0x0102040810204080ull) >> 56);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const unsigned long long h = x[2 * g + (e >> 2)] >> (16 * (e & 3));
          mask |= ((h & 0x7FFFull) != 0 ? 1u : 0u) << e;
        }
      }
      if (__popc(mask) > z) record_error(status, row, q * 8 + g);  // first_overfull_block
      const unsigned long long ent = s_lut[mask];
#pragma unroll
      for (int wi = 0; wi < 3; ++wi) {
        const uint32_t f = static_cast<uint32_t>(ent >> (16 * wi));
        const int ni = g * 3 + wi;  // nibble index within the thread's 24 windows
        om[ni >> 3] |= (f & 0xFu) << (4 * (ni & 7));
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const uint32_t so = (f >> (4 + 4 * s)) & 0xFu;
          uint32_t val = 0;
          if constexpr (ESZ == 1) {
            if (so < 8) val = static_cast<uint32_t>(x[g] >> (8 * so)) & 0xFFu;
          } else {
            if (so < 8) val = static_cast<uint32_t>(x[2 * g + (so >> 2)] >> (16 * (so & 3))) & 0xFFFFu;
          }
          const int vi = (g * 6 + wi * 2 + s) * ESZ;  // byte index in the thread's value run
          ov[vi >> 2] |= val << (8 * (vi & 3));
        }
      }
    }
    uint4* dv = reinterpret_cast<uint4*>(values + row * ld_vals + q * 48 * ESZ);
#pragma unroll
    for (int i = 0; i < 3 * ESZ; ++i) dv[i] = make_uint4(ov[4 * i], ov[4 * i + 1], ov[4 * i + 2], ov[4 * i + 3]);
    uint32_t* dm = reinterpret_cast<uint32_t*>(meta + row * ld_meta + q * 12);
    dm[0] = om[0];
    dm[1] = om[1];
    dm[2] = om[2];
  }
}

// 8-bit weights, byte-permute form of the same table: per mask, PRMT
// selectors placing the window values (output bytes 0-3 and 4-5 of a block)
// from the block's 8 bytes, a keep-mask that zeroes the padding slots (a -0
// e4m3 byte is "zero" to the packer but not the 0x00 padding value, so the
// padding is masked, not selected), and the 12 code bits. ~2.5 instructions
// per weight byte instead of ~6 (the table-walk form was issue-bound: 64%
// issue-active, math-pipe throttle, ncu profiles/r01_ncu_full.txt).
struct Lut8p {
  unsigned long long sel[256];   // bits 0-15 bytes 0-3, 16-23 bytes 4-5, 32-43 codes
  unsigned long long keep[256];  // bytes 0-3 mask (bits 0-31), bytes 4-5 mask (bits 32-47)
};

Lut8p build_lut8p(const Lut8& t) {
  Lut8p p{};
  for (int mask = 0; mask < 256; ++mask) {
    unsigned long long sel = 0, keep = 0, codes = 0;
    for (int w = 0; w < 3; ++w) {
      const uint32_t f = static_cast<uint32_t>(t.e[mask] >> (16 * w));
      codes |= static_cast<unsigned long long>(f & 0xFu) << (4 * w);
      for (int sl = 0; sl < 2; ++sl) {
        const int ob = 2 * w + sl;  // output byte 0..5 of the block
        const uint32_t so = (f >> (4 + 4 * sl)) & 0xFu;
        const unsigned long long nib = so < 8 ? so : 0;  // any byte; masked below
        const int shift = ob < 4 ? 4 * ob : 16 + 4 * (ob - 4);
        sel |= nib << shift;
        if (so < 8) keep |= 0xFFull << (ob < 4 ? 8 * ob : 32 + 8 * (ob - 4));
      }
    }
    p.sel[mask] = sel | (codes << 32);
    p.keep[mask] = keep;
  }
  return p;
}

__global__ void __launch_bounds__(256) pack68b_kernel(const uint8_t* __restrict__ w, int64_t rows, int64_t cols, int z,
                                                      int dtype, const Lut8p* __restrict__ lut, uint8_t* __restrict__ values,
                                                      int64_t ld_vals, uint8_t* __restrict__ meta, int64_t ld_meta,
                                                      unsigned long long* status) {
  __shared__ unsigned long long s_sel[256], s_keep[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_sel[i] = lut->sel[i];
    s_keep[i] = lut->keep[i];
  }
  __syncthreads();
  const int64_t octs = cols / 64;  // 8 blocks of 8 per thread
  const int64_t total = rows * octs;
  const unsigned long long m7 = 0x7F7F7F7F7F7F7F7Full;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx / octs, q = idx - row * octs;
    const uint4* src = reinterpret_cast<const uint4*>(w + row * cols + q * 64);
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __ldg(src + i);
    const uint32_t* x = reinterpret_cast<const uint32_t*>(v);  // block g = words 2g, 2g+1
    uint32_t ov[12];
    uint32_t om[3] = {0, 0, 0};
#pragma unroll
    for (int g = 0; g < 8; g += 2) {
      uint32_t P[2], Q[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t lo = x[2 * (g + h)], hi = x[2 * (g + h) + 1];
        const unsigned long long b64 = (static_cast<unsigned long long>(hi) << 32) | lo;
        const unsigned long long b = dtype == SLSP_DT_E4M3 ? (b64 & m7) : b64;
        const unsigned long long t = (((b & m7) + m7) | b) & 0x8080808080808080ull;
        const uint32_t mask = static_cast<uint32_t>(((t >> 7) * 0x0102040810204080ull) >> 56);
        if (__popc(mask) > z) record_error(status, row, q * 8 + g + h);  // first_overfull_block
        const unsigned long long sel = s_sel[mask], keep = s_keep[mask];
        P[h] = __byte_perm(lo, hi, static_cast<uint32_t>(sel) & 0xFFFFu) & static_cast<uint32_t>(keep);
        Q[h] = __byte_perm(lo, hi, static_cast<uint32_t>(sel >> 16) & 0xFFu) & static_cast<uint32_t>(keep >> 32);
        const uint32_t c = static_cast<uint32_t>(sel >> 32) & 0xFFFu;  // 12 code bits of block g+h
        const int bit = 12 * (g + h);
        om[bit >> 5] |= c << (bit & 31);
        if ((bit & 31) > 20) om[(bit >> 5) + 1] |= c >> (32 - (bit & 31));
      }
      // blocks A, B (6 bytes each) -> 3 words: [A0-3] [A4 A5 B0 B1] [B2-5]
      ov[3 * (g >> 1)] = P[0];
      ov[3 * (g >> 1) + 1] = __byte_perm(Q[0], P[1], 0x5410);
      ov[3 * (g >> 1) + 2] = __byte_perm(P[1], Q[1], 0x5432);
    }
    uint4* dv = reinterpret_cast<uint4*>(values + row * ld_vals + q * 48);
#pragma unroll
    for (int i = 0; i < 3; ++i) dv[i] = make_uint4(ov[4 * i], ov[4 * i + 1], ov[4 * i + 2], ov[4 * i + 3]);
    uint32_t* dm = reinterpret_cast<uint32_t*>(meta + row * ld_meta + q * 12);
    dm[0] = om[0];
    dm[1] = om[1];
    dm[2] = om[2];
  }
}

// Row-major 2-bit codes -> MMA-tiled metadata (see slsp_tile_meta in the
// header): one 16-byte chunk per thread, coalesced on the tiled side.
// F16 (16-bit A, kind::f16) variant: the 2 KB metadata atom of 128 rows x
// 128 logical k is CUTLASS's TensorEAtom_MMA_F16 ((8,2,8),(16,2,4)) :
// ((128,16,2048),(1,1024,32)) in logical elements, 8 per byte — the 8-bit
// kinds' row-major atom with byte-offset bits 1 and 7 exchanged (row bit 3 <->
// bit 1 of the byte within the row's 16). One destination chunk per thread,
// gathered from rows r and r^8 of the row-major codes.
__global__ void tile_meta_f16_kernel(const uint8_t* __restrict__ meta, int64_t rows, int64_t kp, uint8_t* tiled) {
  const int64_t ld = kp / 8;
  const int64_t chunks_per_block = kp / 128;  // 128-logical atoms per 128-row block
  const int64_t total = (rows + 127) / 128 * 128 * ld / 16;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rd = i & 127;   // destination row slot within the atom
    const int64_t at = i >> 7;    // b * chunks_per_block + c
    const int64_t b = at / chunks_per_block, c = at % chunks_per_block;
    uint8_t out[16];
#pragma unroll
    for (int jd = 0; jd < 16; ++jd) {
      const int64_t rs = (rd & ~int64_t{8}) | (static_cast<int64_t>((jd >> 1) & 1) << 3);
      const int js = (jd & ~2) | static_cast<int>(((rd >> 3) & 1) << 1);
      const int64_t row = b * 128 + rs;
      out[jd] = row < rows ? meta[row * ld + c * 16 + js] : 0x44;
    }
    reinterpret_cast<uint4*>(tiled)[i] = *reinterpret_cast<const uint4*>(out);
  }
}

__global__ void tile_meta_kernel(const uint8_t* __restrict__ meta, int64_t rows, int64_t kp, uint8_t* tiled) {
  const int64_t ld = kp / 8;
  const int64_t stages = kp / 256;
  const int64_t total = (rows + 127) / 128 * 128 * ld / 16;  // 16-byte chunks
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i & 127;        // row within the 128-row block
    const int64_t c = (i >> 7) & 1;   // atom within the stage
    const int64_t bs = i >> 8;        // b * stages + s
    const int64_t b = bs / stages, s = bs % stages;
    const int64_t row = b * 128 + r;
    uint4 v = make_uint4(0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    if (row < rows) v = *reinterpret_cast<const uint4*>(meta + row * ld + s * 32 + c * 16);
    reinterpret_cast<uint4*>(tiled)[i] = v;
  }
}

// slsp_gemm_order (6:8): output window i of a row, period P = i / 192,
// o = i % 192: o < 128 -> block 64P + o/2, window 2*(o & 1); else block
// 64P + o - 128, window 1. One thread per 16 output windows (2*ESZ value
// bytes and one 4-bit code pair each). Offline, one pass over the weights.
template <int ESZ>
__global__ void gemm_order_kernel(const uint8_t* __restrict__ vals, const uint8_t* __restrict__ codes, int64_t rows,
                                  int64_t nblk, int64_t kp_ref, uint8_t* __restrict__ vout, uint8_t* __restrict__ cout,
                                  int64_t kp_out) {
  const int64_t per_row = kp_out / 64;  // 16-window groups per output row
  const int64_t total = rows * per_row;
  const int64_t wref = kp_ref / 4;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / per_row;
    const int64_t i0 = (t - row * per_row) * 16;
    const uint8_t* vr = vals + row * (kp_ref / 2) * ESZ;
    const uint8_t* cr = codes + row * (kp_ref / 8);
    uint8_t v[32 * ESZ];
    uint32_t c[2] = {0u, 0u};
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t i = i0 + u;
      const int64_t P = i / 192, o = i - P * 192;
      const int64_t blk = o < 128 ? 64 * P + (o >> 1) : 64 * P + (o - 128);
      const int64_t w = o < 128 ? 2 * (o & 1) : 1;
      const int64_t j = blk * 3 + w;
      uint32_t nib = 0x4u;  // padding window: values 0, codes (0,1)
      if (blk < nblk && j < wref) {
#pragma unroll
        for (int b = 0; b < 2 * ESZ; ++b) v[u * 2 * ESZ + b] = vr[j * 2 * ESZ + b];
        nib = (cr[j >> 1] >> (4 * (j & 1))) & 0xFu;
      } else {
#pragma unroll
        for (int b = 0; b < 2 * ESZ; ++b) v[u * 2 * ESZ + b] = 0;
      }
      c[u >> 3] |= nib << (4 * (u & 7));
    }
    uint4* dv = reinterpret_cast<uint4*>(vout + (row * (kp_out / 2) + i0 * 2) * ESZ);
#pragma unroll
    for (int q = 0; q < 2 * ESZ; ++q) dv[q] = reinterpret_cast<const uint4*>(v)[q];
    *reinterpret_cast<uint2*>(cout + row * (kp_out / 8) + i0 / 2) = make_uint2(c[0], c[1]);
  }
}

// container.hpp kind-2 payload -> MMA-ready operands: values [rows][W][2]
// (elem bytes each) -> [rows][kp/2] zero-padded; the codes stream (2-bit codes
// packed four per byte over the whole matrix, container.hpp:330-336, so a
// row's windows start at nibble r*W) -> row-major [rows][kp/8] with canonical
// codes (0,1) for the padding windows. One thread per output metadata byte
// (two windows) plus its values.
template <int ESZ>
__global__ void load_compressed_kernel(const uint8_t* __restrict__ vals, const uint8_t* __restrict__ stream,
                                       int64_t rows, int64_t W, int64_t kp, uint8_t* __restrict__ vout,
                                       uint8_t* __restrict__ mout) {
  const int64_t per_row = kp / 8;  // output metadata bytes per row = windows / 2
  const int64_t total = rows * per_row;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / per_row, b = t - r * per_row;
    uint32_t byte = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = 2 * b + h;  // window
      uint32_t nib = 0x4u;
      uint8_t* vo = vout + (r * (kp / 2) + 2 * j) * ESZ;
      if (j < W) {
        const int64_t q = r * W + j;  // nibble index in the stream
        nib = (stream[q >> 1] >> (4 * (q & 1))) & 0xFu;
        const uint8_t* vi = vals + (r * W + j) * 2 * ESZ;
#pragma unroll
        for (int e = 0; e < 2 * ESZ; ++e) vo[e] = vi[e];
      } else {
#pragma unroll
        for (int e = 0; e < 2 * ESZ; ++e) vo[e] = 0;
      }
      byte |= nib << (4 * h);
    }
    mout[t] = static_cast<uint8_t>(byte);
  }
}

// The byte-permute table lives in device memory (4 KB, too large for a
// kernel parameter), uploaded once per device and kept for the process. Env
// SLSP_PACK_PATH=1 selects the table-walk kernel (perf probing).
int device_lut8p(const Lut8& t, const Lut8p** out) {
  static const Lut8p host = build_lut8p(t);
  static slsp_host::PerDevice<const Lut8p*> cache;
  return cache.get(out, [](const Lut8p*& v) -> int {
    void* d = nullptr;
    SLSP_CUDA_TRY(cudaMalloc(&d, sizeof(Lut8p)));
    SLSP_CUDA_TRY(cudaMemcpy(d, &host, sizeof(Lut8p), cudaMemcpyHostToDevice));
    v = static_cast<const Lut8p*>(d);
    return SLSP_OK;
  });
}

int pack_path() { return static_cast<int>(slsp_host::knob("SLSP_PACK_PATH", 2)); }

template <int MODE>
int launch_pack(int esz, PackArgs& a, cudaStream_t s) {
  const int64_t chunks = (a.group_slots + kThreads - 1) / kThreads;
  if (chunks == 0 || a.rows == 0) return SLSP_OK;
  size_t smem = MODE == 0 ? static_cast<size_t>(kThreads) * a.wc * 4 * esz
                          : static_cast<size_t>(kThreads) * a.wc * 2 * esz + ((kThreads * a.wc + 7) / 8) * 4;
  dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(a.rows < 65535 ? a.rows : 65535));
  if (chunks > 0x7fffffff) return SLSP_ERR_UNSUPPORTED;
#define SLSP_PACK_LAUNCH(E)                                                                  \
  do {                                                                                       \
    auto k = pack_kernel<E, MODE>;                                                           \
    static slsp_host::PerDevice<int> attr_set; /* the smem opt-in is per device */           \
    int ok_ = 0;                                                                             \
    int st_ = attr_set.get(&ok_, [&](int& v) -> int {                                               \
      SLSP_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024)); \
      v = 1;                                                                                 \
      return SLSP_OK;                                                                        \
    });                                                                                      \
    if (st_) return st_;                                                                     \
    k<<<grid, kThreads, smem, s>>>(a);                                                       \
  } while (0)
  switch (esz) {
    case 1: SLSP_PACK_LAUNCH(1); break;
    case 2: SLSP_PACK_LAUNCH(2); break;
    case 4: SLSP_PACK_LAUNCH(4); break;
    case 8: SLSP_PACK_LAUNCH(8); break;
    default: return SLSP_ERR_INVALID;
  }
#undef SLSP_PACK_LAUNCH
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 64) b = 148 * 64;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

extern "C" {

int slsp_pack_matrix(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, void* slided,
                     void* status_ws, int64_t* err_row, int64_t* err_block, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  const int esz = elem_size(dtype);
  if (!esz || l > kMaxL || rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  if (cols % l != 0) return SLSP_ERR_DIMENSION;  // pack.hpp:174-177
  if (!status_ws) return SLSP_ERR_INVALID;       // pack_matrix always reports violations
  if ((st = require_sm100())) return st;
  if ((st = status_reset(status_ws, s))) return st;
  PackArgs a{};
  a.w = static_cast<const uint8_t*>(w);
  a.rows = rows;
  a.cols = cols;
  a.z = z;
  a.l = l;
  a.wc = wc;
  a.dtype = dtype;
  a.groups_real = cols / l;
  a.group_slots = a.groups_real;
  a.out_windows = a.groups_real * wc;
  a.out_a = static_cast<uint8_t*>(slided);
  a.ld_a_bytes = a.out_windows * 4 * esz;
  a.status = static_cast<unsigned long long*>(status_ws);
  if ((st = launch_pack<0>(esz, a, s))) return st;
  return status_collect(status_ws, s, SLSP_ERR_NOT_COMPLIANT, err_row, err_block);
}

int slsp_pack_compress(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, int64_t kp, void* values,
                       uint8_t* meta, void* status_ws, int64_t* err_row, int64_t* err_block, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  const int esz = elem_size(dtype);
  if (!esz || esz > 2 || l > kMaxL || rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  const int64_t groups = (cols + l - 1) / l;
  const int64_t kprime = groups * wc * 4;
  if (kp < kprime || kp % 8 != 0) return SLSP_ERR_DIMENSION;
  if ((st = require_sm100())) return st;
  if ((st = status_reset(status_ws, s))) return st;
  unsigned long long* status = static_cast<unsigned long long*>(status_ws);  // may be null: no report
  // 6:8 fast path (table-driven greedy, 8 blocks per thread, vector I/O)
  const int64_t ld_vals = kp / 2 * esz, ld_meta = kp / 8;
  if (l == 8 && cols % 64 == 0 && ld_vals % 16 == 0 && ld_meta % 4 == 0 && rows > 0 &&
      !((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(values) | reinterpret_cast<uintptr_t>(meta)) &
        15u)) {
    static const Lut8 lut = build_lut8();
    const int64_t threads = rows * (cols / 64);
    if (threads > 0) {
      const unsigned grid = grid_for(threads, 256);
      const auto* in = static_cast<const uint8_t*>(w);
      auto* out = static_cast<uint8_t*>(values);
      if (esz == 1)
        if (pack_path() == 1) {
          pack68_kernel<1><<<grid, 256, 0, s>>>(in, rows, cols, z, dtype, lut, out, ld_vals, meta, ld_meta, status);
        } else {
          const Lut8p* dlut = nullptr;
          if ((st = device_lut8p(lut, &dlut))) return st;
          pack68b_kernel<<<grid, 256, 0, s>>>(in, rows, cols, z, dtype, dlut, out, ld_vals, meta, ld_meta, status);
        }
      else
        pack68_kernel<2><<<grid, 256, 0, s>>>(in, rows, cols, z, dtype, lut, out, ld_vals, meta, ld_meta, status);
      SLSP_LAUNCH_CHECK();
    }
    const int64_t kprime_b = kprime / 2 * esz;  // padding windows past K': zero values, codes (0,1)
    if (ld_vals > kprime_b) {
      SLSP_CUDA_TRY(cudaMemset2DAsync(static_cast<uint8_t*>(values) + kprime_b, ld_vals, 0, ld_vals - kprime_b,
                                      rows, s));
      SLSP_CUDA_TRY(cudaMemset2DAsync(meta + kprime / 8, ld_meta, 0x44, ld_meta - kprime / 8, rows, s));
    }
    return status_collect(status_ws, s, SLSP_ERR_NOT_COMPLIANT, err_row, err_block);
  }
  PackArgs a{};
  a.w = static_cast<const uint8_t*>(w);
  a.rows = rows;
  a.cols = cols;
  a.z = z;
  a.l = l;
  a.wc = wc;
  a.dtype = dtype;
  a.groups_real = groups;
  a.out_windows = kp / 4;
  a.group_slots = (a.out_windows + wc - 1) / wc;
  a.out_a = static_cast<uint8_t*>(values);
  a.out_meta = meta;
  a.ld_a_bytes = kp / 2 * esz;
  a.ld_meta = kp / 8;
  a.status = status;
  if ((st = launch_pack<1>(esz, a, s))) return st;
  return status_collect(status_ws, s, SLSP_ERR_NOT_COMPLIANT, err_row, err_block);
}

int slsp_gemm_order(int dtype, const void* values, const uint8_t* codes, int64_t rows, int64_t cols, int64_t kp_ref,
                    void* values_out, uint8_t* codes_out, int64_t kp_out, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int esz = elem_size(dtype);
  if ((esz != 1 && esz != 2) || rows < 0 || cols <= 0 || kp_ref <= 0 || kp_ref % 4 != 0) return SLSP_ERR_INVALID;
  if (rows == 0) return SLSP_OK;
  if (!values || !codes || !values_out || !codes_out) return SLSP_ERR_INVALID;
  const int64_t nblk = (cols + 7) / 8;
  if (kp_ref < nblk * 12) return SLSP_ERR_DIMENSION;  // the reference width must hold every real window
  if (kp_out != (cols + 511) / 512 * 768) return SLSP_ERR_DIMENSION;
  if ((reinterpret_cast<uintptr_t>(values_out) & 15u) || (reinterpret_cast<uintptr_t>(codes_out) & 7u))
    return SLSP_ERR_INVALID;
  int st;
  if ((st = require_sm100())) return st;
  const int64_t total = rows * (kp_out / 64);
  if (total == 0) return SLSP_OK;
  const auto* v = static_cast<const uint8_t*>(values);
  auto* vo = static_cast<uint8_t*>(values_out);
  if (esz == 1) gemm_order_kernel<1><<<grid_for(total, 256), 256, 0, s>>>(v, codes, rows, nblk, kp_ref, vo, codes_out, kp_out);
  else gemm_order_kernel<2><<<grid_for(total, 256), 256, 0, s>>>(v, codes, rows, nblk, kp_ref, vo, codes_out, kp_out);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

int slsp_load_compressed(int dtype, const void* values, const uint8_t* codes_stream, int64_t rows, int64_t windows,
                         int64_t kp, void* values_out, uint8_t* meta_out, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int esz = elem_size(dtype);
  if ((esz != 1 && esz != 2) || rows < 0 || windows < 0) return SLSP_ERR_INVALID;
  if (rows == 0) return SLSP_OK;
  if (!values || !codes_stream || !values_out || !meta_out) return SLSP_ERR_INVALID;
  if (kp % 8 != 0 || kp / 4 < windows) return SLSP_ERR_DIMENSION;
  int st;
  if ((st = require_sm100())) return st;
  const int64_t total = rows * (kp / 8);
  if (total == 0) return SLSP_OK;
  const auto* v = static_cast<const uint8_t*>(values);
  auto* vo = static_cast<uint8_t*>(values_out);
  if (esz == 1) load_compressed_kernel<1><<<grid_for(total, 256), 256, 0, s>>>(v, codes_stream, rows, windows, kp, vo, meta_out);
  else load_compressed_kernel<2><<<grid_for(total, 256), 256, 0, s>>>(v, codes_stream, rows, windows, kp, vo, meta_out);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

int64_t slsp_tiled_meta_bytes(int64_t rows, int64_t kp) { return (rows + 127) / 128 * 128 * (kp / 8); }

int slsp_tile_meta(const uint8_t* meta, int64_t rows, int64_t kp, uint8_t* tiled, slsp_stream_t stream) {
  return slsp_tile_meta_ex(meta, rows, kp, SLSP_DT_I8, tiled, stream);
}

int slsp_tile_meta_ex(const uint8_t* meta, int64_t rows, int64_t kp, int dtype, uint8_t* tiled, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (rows < 0 || kp <= 0) return SLSP_ERR_INVALID;
  if (kp % 256 != 0) return SLSP_ERR_DIMENSION;
  if (rows == 0) return SLSP_OK;
  if (!meta || !tiled) return SLSP_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(meta) | reinterpret_cast<uintptr_t>(tiled)) & 15u) return SLSP_ERR_INVALID;
  int st;
  if ((st = require_sm100())) return st;
  const int64_t chunks = slsp_tiled_meta_bytes(rows, kp) / 16;
  if (chunks == 0) return SLSP_OK;
  if (dtype == SLSP_DT_BF16) tile_meta_f16_kernel<<<grid_for(chunks, 256), 256, 0, s>>>(meta, rows, kp, tiled);
  else tile_meta_kernel<<<grid_for(chunks, 256), 256, 0, s>>>(meta, rows, kp, tiled);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

int slsp_compress(int dtype, const void* slided, int64_t rows, int64_t cols_exp, void* values, uint8_t* codes,
                  void* status_ws, int64_t* err_row, int64_t* err_window, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int esz = elem_size(dtype);
  if (!esz || rows < 0 || cols_exp < 0 || !status_ws) return SLSP_ERR_INVALID;
  if (cols_exp % 4 != 0) return SLSP_ERR_DIMENSION;  // gemm.hpp:78-80
  int st;
  if ((st = require_sm100())) return st;
  if ((st = status_reset(status_ws, s))) return st;
  const int64_t wpr = cols_exp / 4;
  const unsigned grid = grid_for(rows * wpr, 256);
  auto* status = static_cast<unsigned long long*>(status_ws);
  const auto* in = static_cast<const uint8_t*>(slided);
  auto* out = static_cast<uint8_t*>(values);
  switch (esz) {
    case 1: compress_kernel<1><<<grid, 256, 0, s>>>(in, rows, wpr, dtype, out, codes, status); break;
    case 2: compress_kernel<2><<<grid, 256, 0, s>>>(in, rows, wpr, dtype, out, codes, status); break;
    case 4: compress_kernel<4><<<grid, 256, 0, s>>>(in, rows, wpr, dtype, out, codes, status); break;
    case 8: compress_kernel<8><<<grid, 256, 0, s>>>(in, rows, wpr, dtype, out, codes, status); break;
  }
  SLSP_LAUNCH_CHECK();
  return status_collect(status_ws, s, SLSP_ERR_NOT_COMPLIANT, err_row, err_window);
}

int slsp_magnitude_prune(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, void* out,
                         slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int esz = elem_size(dtype);
  if (!esz || z <= 0 || l <= 0 || z > l || l > kMaxL || rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  if (cols % l != 0) return SLSP_ERR_DIMENSION;  // pack.hpp:240-243
  int st;
  if ((st = require_sm100())) return st;
  const unsigned grid = grid_for(rows * (cols / l), 256);
  const auto* in = static_cast<const uint8_t*>(w);
  auto* o = static_cast<uint8_t*>(out);
  switch (esz) {
    case 1: prune_kernel<1><<<grid, 256, 0, s>>>(in, rows, cols, z, l, dtype, o); break;
    case 2: prune_kernel<2><<<grid, 256, 0, s>>>(in, rows, cols, z, l, dtype, o); break;
    case 4: prune_kernel<4><<<grid, 256, 0, s>>>(in, rows, cols, z, l, dtype, o); break;
    case 8: prune_kernel<8><<<grid, 256, 0, s>>>(in, rows, cols, z, l, dtype, o); break;
  }
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

}  // extern "C"
