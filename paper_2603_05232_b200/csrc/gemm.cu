// Structured-sparse and dense GEMMs on sm_100a 5th-gen tensor cores
// (SURVEY.md §8a rows a13-a15, a18).
//
//   Y[n][t] = sum_k W[n][k] * X[t][k]       (gemm.hpp:142-233 orientation)
//
// One persistent kernel template, warp-specialised, CTA pair (cluster of 2,
// tcgen05 cta_group::2):
//   warp 0      TMA producer (both CTAs): A (weights, compressed for .sp),
//               B (lifted activations), E (2-bit metadata) into a STAGES-deep
//               smem ring; completion bytes land on the leader's barrier.
//   warp 1      leader CTA: one elected thread issues tcgen05.cp (E -> TMEM)
//               and tcgen05.mma[.sp] (M=256 across the pair, N=BN tokens);
//               both CTAs: TMEM allocation.
//   warps 2-5   epilogue (both CTAs): tcgen05.ld the accumulator lanes,
//               optional per-channel x per-token dequant to BF16, swizzled
//               smem staging, TMA bulk tensor stores.
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps
// the mainloop of tile i+1. The weight (sparse) operand is A: MMA-M = output
// features, MMA-N = tokens.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace slsp_dev;

constexpr int kNumThreads = 192;

// Debug knobs (env SLSP_GEMM_DEBUG, read once): bit0 skip output stores,
// bit1 skip operand loads (MMA on stale smem), bit2 load k-block 0 of tile 0
// only (L2-resident operands). Results are garbage when set; perf probing only.
enum : uint32_t { kDbgNoStore = 1u, kDbgNoLoad = 2u, kDbgSameTile = 4u, kDbgNoMeta = 8u };
// L2 cache-policy hints (env SLSP_GEMM_HINTS overrides kDefaultHints).
enum : uint32_t { kHintBLast = 1u, kHintAFirst = 2u, kHintOutFirst = 4u };
constexpr uint32_t kDefaultHints = kHintBLast | kHintOutFirst;

template <bool SPARSE_, MmaKind KIND_, int BN_, int STAGES_, int OUT_, int CL_ = 2, int MSUB_ = 1>
struct Cfg {
  static constexpr bool SPARSE = SPARSE_;
  static constexpr MmaKind KIND = KIND_;
  static constexpr int BN = BN_;          // tokens per pair tile (MMA N)
  static constexpr int STAGES = STAGES_;
  static constexpr int OUT = OUT_;
  // Cluster: CL CTAs = CL/2 CTA pairs on adjacent weight tiles of the same
  // token tile; with 2 pairs each activation (B) box is fetched once from L2
  // and multicast to both pairs (each pair loads one half of every B box).
  static constexpr int CL = CL_;
  static constexpr int NPAIR = CL / 2;
  static_assert(CL == 2 || CL == 4, "cluster of 1 or 2 CTA pairs");
  // M-subtiles: the pair runs MSUB UMMAs (M=256 each) per k-step against the
  // same activation stage, so B traffic per MAC drops by MSUB. TMEM then holds
  // MSUB accumulators per tile; with MSUB=2 they are single-buffered and
  // 4*MSUB epilogue warps drain them in parallel.
  static constexpr int MSUB = MSUB_;
  static_assert(MSUB == 1 || MSUB == 2, "one or two M-subtiles per pair");
  static constexpr int ACC_STAGES = MSUB == 1 ? 2 : 1;
  static constexpr int EPI_WARPS = 4 * MSUB;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int BM = 256 * MSUB;   // weight rows per pair tile
  static constexpr int A_ROWS = 128;      // per CTA per M-subtile
  static constexpr int B_ROWS = BN / 2;   // tokens per CTA
  static constexpr int A_SUB = 128 * 128;                    // one 128B-swizzle atom column
  static constexpr int A_STAGE = MSUB * A_SUB;
  static constexpr int B_ATOMS = SPARSE ? 2 : 1;             // B bytes per stage = 2x A bytes for .sp
  static constexpr int B_ATOM = B_ROWS * 128;
  static constexpr int B_STAGE = B_ATOM * B_ATOMS;
  static constexpr int B_PART = B_ROWS / NPAIR;  // rows of each B box one pair fetches (multicast)
  static_assert(B_PART % 8 == 0, "multicast slices must be whole 128B-swizzle atoms");
  static constexpr int E_SUB = SPARSE ? 2 * 128 * 16 : 0;    // two 128x128b metadata atoms
  static constexpr int E_STAGE = MSUB * E_SUB;
  static constexpr int STAGE_TX = A_STAGE + B_STAGE + E_STAGE;
  static constexpr int K_BYTES_B = 128 * B_ATOMS;            // activation bytes consumed per stage
  static constexpr int MMAS = 4;                             // k-steps per stage
  static constexpr int ACC_COLS = BN;                        // 32-bit TMEM columns per accumulator
  static constexpr int E_COL = ACC_STAGES * MSUB * BN;       // metadata columns after the accumulators
  static constexpr int TMEM_COLS = 512;
  static_assert(!SPARSE || E_COL + 8 * MSUB <= TMEM_COLS, "TMEM budget: accumulators + metadata");
  static_assert(SPARSE || E_COL <= TMEM_COLS, "TMEM budget: accumulators");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "cta_group::2 N");
  // epilogue: chunks of 32 rows x EPI_COLS columns, double-buffered smem
  // staging per warp (a TMA store reads one buffer while the next is filled)
  static constexpr int OUT_ESZ = OUT == SLSP_OUT_RAW_NM ? 4 : 2;
  static constexpr int EPI_COLS = MSUB == 2 ? 16 : 32;
  static constexpr int EPI_BUFS = 2;
  static constexpr int EPI_BUF = 32 * EPI_COLS * OUT_ESZ;
  static constexpr int EPI_ROW = EPI_COLS * OUT_ESZ;  // staging row bytes (NM layout) = swizzle span
  static constexpr int EPI_WARP = EPI_BUFS * EPI_BUF;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_STAGE;
  static constexpr int OFF_E = OFF_B + STAGES * B_STAGE;
  static constexpr int OFF_EPI = OFF_E + STAGES * E_STAGE;
  static constexpr int OFF_BAR = OFF_EPI + EPI_WARPS * EPI_WARP;
  static constexpr int NUM_BARS = 2 * STAGES + 4;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // + alignment slack
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static constexpr uint32_t C_FMT = KIND == MmaKind::I8 ? 2u : 1u;
  static constexpr uint32_t AB_FMT = KIND == MmaKind::F8 ? 0u : 1u;
  static constexpr uint32_t IDESC = make_idesc(SPARSE, C_FMT, AB_FMT, AB_FMT, 256, BN);
  using Acc = typename std::conditional<KIND == MmaKind::I8, int32_t, float>::type;
};

struct Params {
  int64_t n, m;       // weight rows, tokens
  int num_kb;         // k-blocks (stages) per tile
  int m_tiles, n_tiles;
  const float* s_ch;  // per weight row
  const float* s_tok; // per token
  void* out;
  int64_t ldo;
  int tma_store;      // 1: swizzled smem staging + TMA store; 0: direct stores
  int direct_vec;     // with tma_store == 0: rows are 16-byte aligned, use vector stores
  uint32_t debug;
  uint32_t hints;     // kHint* L2 policies
  int group;          // weight tiles per raster band
};

// Raster: bands of `group` weight tiles; within a band the weight tile varies
// fastest, so the clusters running concurrently share activation tiles (B)
// and each band's weight tiles stay L2-resident while the band sweeps tokens.
SLSP_DEVINL void tile_coords(int tile, const Params& p, int m_count, int& mt, int& nt) {
  const int per_group = p.group * p.n_tiles;
  const int g = tile / per_group;
  const int first = g * p.group;
  const int gsize = min(p.group, m_count - first);
  const int r = tile - g * per_group;
  mt = first + r % gsize;
  nt = r / gsize;
}

// a18: y = bf16((acc * s_ch[n]) * s_tok[t]) — fp32, this exact operation order
// (restated by oracle/slsp_oracle.c orc_dequant_bf16).
template <typename Acc>
SLSP_DEVINL float dequant(uint32_t raw, float sc, float st) {
  float a;
  if constexpr (std::is_same<Acc, int32_t>::value) a = __int2float_rn(static_cast<int32_t>(raw));
  else a = __uint_as_float(raw);
  return __fmul_rn(__fmul_rn(a, sc), st);
}

SLSP_DEVINL uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// One 32-row x EPI_COLS-column chunk of the accumulator (lane = row) to its
// output. TMA path: the chunk is staged in smem in the output's 128B/64B/32B
// swizzle (chunk index ^= row bits, conflict-free 16-byte stores) and written
// with one bulk tensor store.
template <typename C>
SLSP_DEVINL void epilogue_chunk(const Params& p, const CUtensorMap* tmOut, uint8_t* stage,
                                uint32_t (&r)[C::EPI_COLS], int64_t row0, int64_t t0, float sc) {
  constexpr int NC = C::EPI_COLS;
  constexpr int NW = C::OUT == SLSP_OUT_RAW_NM ? NC : NC / 2;  // 32-bit output words per lane
  const uint32_t lane = lane_id();
  const int64_t row = row0 + lane;
  // per-token scales: one coalesced load, shuffled to every lane
  float st_lane = 0.f;
  if constexpr (C::OUT != SLSP_OUT_RAW_NM)
    st_lane = (lane < NC && t0 + lane < p.m) ? __ldg(p.s_tok + t0 + lane) : 0.f;
  uint32_t w[NW];
  if constexpr (C::OUT == SLSP_OUT_RAW_NM) {
#pragma unroll
    for (int i = 0; i < NC; ++i) w[i] = r[i];
  } else {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const float lo = dequant<typename C::Acc>(r[2 * i], sc, __shfl_sync(0xffffffffu, st_lane, 2 * i));
      const float hi = dequant<typename C::Acc>(r[2 * i + 1], sc, __shfl_sync(0xffffffffu, st_lane, 2 * i + 1));
      w[i] = pack_bf16(lo, hi);
    }
  }
  if (p.debug & kDbgNoStore) return;

  if (p.tma_store) {
    const uint32_t sb = smem_u32(stage);
    if constexpr (C::OUT == SLSP_OUT_BF16_MN) {
      // token-major tile [NC tokens][32 features] bf16: 64B rows, 64B swizzle
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const uint32_t chunk = (lane >> 3) ^ ((i >> 1) & 3);
        st_shared_u16(sb + i * 64 + chunk * 16 + (lane & 7) * 2, static_cast<uint16_t>(w[i >> 1] >> (16 * (i & 1))));
      }
    } else {
      // [32 rows][NC columns]: EPI_ROW-byte rows, EPI_ROW-byte swizzle
      constexpr int CH = C::EPI_ROW / 16;                      // 16-byte chunks per row
      constexpr int SH = C::EPI_ROW == 128 ? 0 : (C::EPI_ROW == 64 ? 1 : 2);
#pragma unroll
      for (int j = 0; j < CH; ++j)
        st_shared_v4(sb + lane * C::EPI_ROW + ((j ^ ((lane >> SH) & (CH - 1))) << 4), w[4 * j], w[4 * j + 1],
                     w[4 * j + 2], w[4 * j + 3]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      const uint64_t pol = (p.hints & kHintOutFirst) ? policy_evict_first() : policy_evict_normal();
      if constexpr (C::OUT == SLSP_OUT_BF16_MN)
        tma_store_2d_hint(tmOut, stage, static_cast<int>(row0), static_cast<int>(t0), pol);
      else
        tma_store_2d_hint(tmOut, stage, static_cast<int>(t0), static_cast<int>(row0), pol);
      bulk_commit();
    }
    return;
  }
  if (row >= p.n) return;
  const int64_t valid = imin64(NC, p.m - t0);
  if constexpr (C::OUT != SLSP_OUT_BF16_MN) {
    // direct 16-byte vector stores of this lane's row segment (NM layouts,
    // 16-byte aligned rows): no staging, no store-completion waits
    if (p.direct_vec && valid == NC) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.out) + (row * p.ldo + t0) * C::OUT_ESZ);
#pragma unroll
      for (int j = 0; j < NW / 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      return;
    }
  }
  // direct stores (unaligned output strides / tails): predicated, register-resident
  if constexpr (C::OUT == SLSP_OUT_RAW_NM) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(p.out) + row * p.ldo + t0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if (i < valid) dst[i] = w[i];
  } else if constexpr (C::OUT == SLSP_OUT_BF16_NM) {
    uint16_t* dst = reinterpret_cast<uint16_t*>(p.out) + row * p.ldo + t0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if (i < valid) dst[i] = static_cast<uint16_t>(w[i >> 1] >> (16 * (i & 1)));
  } else {
    uint16_t* dst = reinterpret_cast<uint16_t*>(p.out) + t0 * p.ldo + row;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if (i < valid) dst[i * p.ldo] = static_cast<uint16_t>(w[i >> 1] >> (16 * (i & 1)));
  }
}

template <typename C>
__global__ void __launch_bounds__(C::THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmOut,
                const Params p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + C::OFF_A;
  uint8_t* sB = smem + C::OFF_B;
  uint8_t* sE = smem + C::OFF_E;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();     // rank in the cluster
  const uint32_t pair = crank >> 1;             // CTA pair within the cluster
  const uint32_t rank = crank & 1;              // rank within the pair (cta_group::2 peer)
  const uint32_t lead = crank & ~1u;            // cluster rank of this pair's leader
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / C::CL;
  const int num_clusters = gridDim.x / C::CL;
  const int m_super = (p.m_tiles + C::NPAIR - 1) / C::NPAIR;  // weight tiles per cluster step
  const int num_tiles = m_super * p.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NPAIR);  // every pair's MMA must be done with a stage (multicast B)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::EPI_WARPS);  // every epilogue warp of both CTAs of the pair
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (C::SPARSE) tma_prefetch(&tmE);
    if (p.tma_store) tma_prefetch(&tmOut);
  }
  if (warp == 1) tmem_alloc<2>(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer ----
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const bool no_load = p.debug & kDbgNoLoad;
      const bool same = p.debug & kDbgSameTile;
      // L2 policy: activations (B) are re-read by every weight tile -> keep
      // them (evict_last); weights stream through a raster band.
      const uint64_t pol_b = (p.hints & kHintBLast) ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_a = (p.hints & kHintAFirst) ? policy_evict_first() : policy_evict_normal();
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int ms, nt;
        tile_coords(tile, p, m_super, ms, nt);
        int mt = ms * C::NPAIR + static_cast<int>(pair);
        if (same) mt = nt = 0;
        const int a_row = mt * C::BM + static_cast<int>(rank) * C::A_ROWS;
        const int b_row = nt * C::BN + static_cast<int>(rank) * C::B_ROWS;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          const int kl = same ? 0 : kb;
          mbar_wait(&empty[stage], phase ^ 1);
          if (no_load) {
            if (leader) mbar_arrive(&full[stage]);
          } else {
            const bool skip_e = p.debug & kDbgNoMeta;
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (C::STAGE_TX - (skip_e ? C::E_STAGE : 0)));
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), lead);
#pragma unroll
            for (int h = 0; h < C::MSUB; ++h)
              tma_load_2d_cg2_hint(sA + stage * C::A_STAGE + h * C::A_SUB, &tmA, bar, kl * 128, a_row + h * 256,
                                   pol_a);
#pragma unroll
            for (int at = 0; at < C::B_ATOMS; ++at) {
              uint8_t* dst = sB + stage * C::B_STAGE + at * C::B_ATOM;
              if constexpr (C::NPAIR == 1) {
                tma_load_2d_cg2_hint(dst, &tmB, bar, kl * C::K_BYTES_B + at * 128, b_row, pol_b);
              } else {  // this pair fetches slice `pair` of the box for the same-rank CTA of every pair
                const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
                tma_load_2d_cg2_mc(dst + pair * C::B_PART * 128, &tmB, bar, kl * C::K_BYTES_B + at * 128,
                                   b_row + static_cast<int>(pair) * C::B_PART, mask, pol_b);
              }
            }
            if constexpr (C::SPARSE)  // one contiguous 4 KB tiled-metadata block per stage and subtile
              if (!skip_e)
#pragma unroll
                for (int h = 0; h < C::MSUB; ++h)
                  tma_load_2d_cg2_hint(sE + stage * C::E_STAGE + h * C::E_SUB, &tmE, bar, 0,
                                       (((a_row + h * 256) >> 7) * p.num_kb + kl) * 16, pol_a);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer ----
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
        const int acc = C::ACC_STAGES == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = C::ACC_STAGES == 2 ? ((it >> 1) & 1) : (it & 1);
        // MSUB=1: double-buffered accumulators, tempty[acc]. MSUB=2: one
        // buffer per subtile and a barrier per subtile, so subtile 0 of this
        // tile starts while the epilogue is still draining subtile 1 of the last.
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * C::MSUB * C::ACC_COLS;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * C::A_STAGE);
          const uint32_t b_base = smem_u32(sB + stage * C::B_STAGE);
          if constexpr (C::SPARSE) {
            const uint32_t e_base = smem_u32(sE + stage * C::E_STAGE);
#pragma unroll
            for (int h = 0; h < C::MSUB; ++h)
#pragma unroll
              for (int c = 0; c < 2; ++c)
                tmem_cp_128x128b_cg2(tmem + C::E_COL + 8 * h + 4 * c,
                                     smem_desc(e_base + h * C::E_SUB + c * 2048, 2048, 128, 0));
          }
#pragma unroll
          for (int h = 0; h < C::MSUB; ++h) {
            if (C::MSUB == 2 && h == 1 && kb == 0) {  // subtile 1's accumulator must be drained too
              mbar_wait(&tempty[1], acc_phase ^ 1);
              tc_fence_after();
            }
#pragma unroll
            for (int j = 0; j < C::MMAS; ++j) {
              const uint32_t acc_flag = (kb | j) != 0;
              const uint64_t adesc = smem_desc(a_base + h * C::A_SUB + j * 32, 16, 1024, 2);
              const uint32_t d = d_tmem + h * C::ACC_COLS;
              if constexpr (C::SPARSE) {
                const uint64_t bdesc = smem_desc(b_base + (j >> 1) * C::B_ATOM + (j & 1) * 64, 16, 1024, 2);
                umma_sparse_cg2<C::KIND>(d, adesc, bdesc, tmem + C::E_COL + 8 * h + 2 * j, C::IDESC, acc_flag);
              } else {
                const uint64_t bdesc = smem_desc(b_base + j * 32, 16, 1024, 2);
                umma_dense_cg2<C::KIND>(d, adesc, bdesc, C::IDESC, acc_flag);
              }
            }
          }
          tc_commit_mc(&empty[stage], static_cast<uint16_t>((1u << C::CL) - 1));  // every CTA of the cluster
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_mc(&tfull[acc], static_cast<uint16_t>(0x3u << lead));  // this pair's epilogues
      }
    }
  } else {
    // ------------------------------------------------ epilogue ----
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t sub = (warp - 2) >> 2;  // MSUB=2: which alternate chunks of a subtile this warp drains
    const uint32_t lane = lane_id();
    uint8_t* stage_base = smem + C::OFF_EPI + (warp - 2) * C::EPI_WARP;
    int buf = 0;
    int it = 0;
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
      int ms, nt;
      tile_coords(tile, p, m_super, ms, nt);
      const int mt = ms * C::NPAIR + static_cast<int>(pair);
      const int acc = C::ACC_STAGES == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = C::ACC_STAGES == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      // MSUB=2: all 8 warps drain subtile 0 (two warps per lane quarter,
      // alternating chunks), release it, then subtile 1.
#pragma unroll 1
      for (int h = 0; h < C::MSUB; ++h) {
        const int64_t row0 = static_cast<int64_t>(mt) * C::BM + h * 256 + rank * C::A_ROWS + quarter * 32;
        float sc = 0.f;
        if constexpr (C::OUT != SLSP_OUT_RAW_NM) sc = (row0 + lane < p.n) ? __ldg(p.s_ch + row0 + lane) : 0.f;
        const uint32_t t_base = tmem + ((quarter * 32) << 16) + (acc * C::MSUB + h) * C::ACC_COLS;
#pragma unroll 1
        for (int c = static_cast<int>(sub); c < C::BN / C::EPI_COLS; c += C::MSUB) {
          const int64_t t0 = static_cast<int64_t>(nt) * C::BN + c * C::EPI_COLS;
          if (t0 >= p.m) break;  // warp-uniform
          uint32_t r[C::EPI_COLS];
          tmem_ld_cols(t_base + c * C::EPI_COLS, r);
          tmem_ld_wait();
          if (p.tma_store) {
            if (lane == 0) bulk_wait_read<C::EPI_BUFS - 1>();  // staging buffer free again
            __syncwarp();
          }
          epilogue_chunk<C>(p, &tmOut, stage_base + buf * C::EPI_BUF, r, row0, t0, sc);
          if (C::EPI_BUFS == 2) buf ^= 1;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[C::MSUB == 2 ? h : acc]), lead));
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<2>(tmem, C::TMEM_COLS);
#endif
}

// ---------------------------------------------------------------- host --
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

uint32_t debug_flags() {
  static uint32_t flags = [] {
    const char* e = std::getenv("SLSP_GEMM_DEBUG");
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 0)) : 0u;
  }();
  return flags;
}

// Tuning knob from the environment (read per call: cheap, and lets probes vary it).
uint32_t env_knob(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? static_cast<uint32_t>(std::strtoul(e, nullptr, 0)) : dflt;
}

// Byte-addressed 2D map (uint8 elements): rows x row_bytes, box rows x 128 B, 128B swizzle.
int make_map_2d(CUtensorMap* map, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SLSP_ERR_CUDA;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SLSP_OK : SLSP_ERR_CUDA;
}

// Metadata map over the slsp_tile_meta layout: a flat byte stream viewed as
// 256-byte rows; one box {256, 16} is the contiguous 4 KB block of a stage
// (two canonical 128x16B tcgen05.cp atoms) — 16 wide requests instead of 256
// 16-byte ones.
int make_map_meta(CUtensorMap* map, const void* base, uint64_t rows, uint64_t kp) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SLSP_ERR_CUDA;
  const uint64_t bytes = static_cast<uint64_t>(slsp_tiled_meta_bytes(static_cast<int64_t>(rows), static_cast<int64_t>(kp)));
  cuuint64_t dims[2] = {256, bytes / 256};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {256, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SLSP_OK : SLSP_ERR_CUDA;
}

// Output map for the TMA-store epilogue: 32x32 element boxes.
//   NM: (cols = tokens m, rows = n); MN: (cols = n, rows = tokens m).
int make_map_out(CUtensorMap* map, void* base, int out_mode, int64_t n, int64_t m, int64_t ldo, int cols,
                 int* use_tma) {
  const int esz = out_mode == SLSP_OUT_RAW_NM ? 4 : 2;
  *use_tma = 0;
  std::memset(map, 0, sizeof(*map));
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (ldo * esz) % 16) return SLSP_OK;  // direct-store path
  EncodeTiledFn enc = get_encode();
  if (!enc) return SLSP_ERR_CUDA;
  const bool mn = out_mode == SLSP_OUT_BF16_MN;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(mn ? n : m), static_cast<cuuint64_t>(mn ? m : n)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldo * esz)};
  // NM: box {cols tokens, 32 rows}, swizzle = row bytes; MN: box {32 features, cols tokens}, 64B rows
  cuuint32_t box[2] = {static_cast<cuuint32_t>(mn ? 32 : cols), static_cast<cuuint32_t>(mn ? cols : 32)};
  cuuint32_t estr[2] = {1, 1};
  const int row_bytes = mn ? 64 : cols * esz;
  const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                  : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return SLSP_ERR_CUDA;
  *use_tma = 1;
  return SLSP_OK;
}

// Epilogue store path: TMA staging (1) or direct 16-byte vector stores (2);
// env SLSP_GEMM_EPI overrides the default (0 = auto: vectors for the
// 2-subtile tiles' narrow chunks, TMA otherwise). MN output always uses TMA.
void select_epilogue(Params& p, int out_mode, uint32_t msub) {
  const uint32_t epi = env_knob("SLSP_GEMM_EPI", 0);
  const bool aligned = p.tma_store != 0;  // make_map_out enables TMA iff rows are 16-byte aligned
  if (out_mode != SLSP_OUT_BF16_MN && aligned && (epi == 2 || (epi == 0 && msub == 2))) {
    p.tma_store = 0;
    p.direct_vec = 1;
  }
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <typename C>
int run(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o, Params p,
        cudaStream_t s) {
  static int max_clusters = 0;
  auto kern = gemm_kernel<C>;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!max_clusters) {  // how many clusters of this shape are co-resident (GPC packing)
    SLSP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    cfg.gridDim = dim3(C::CL * (num_sms() / C::CL));
    int n = 0;
    SLSP_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    max_clusters = n > 0 ? n : num_sms() / C::CL;
  }
  p.m_tiles = static_cast<int>((p.n + C::BM - 1) / C::BM);
  p.n_tiles = static_cast<int>((p.m + C::BN - 1) / C::BN);
  const int tiles = (p.m_tiles + C::NPAIR - 1) / C::NPAIR * p.n_tiles;
  if (tiles == 0) return SLSP_OK;
  int clusters = max_clusters;
  const int cluster_cap = static_cast<int>(env_knob("SLSP_GEMM_CLUSTERS", 0));  // perf probing
  if (cluster_cap > 0 && clusters > cluster_cap) clusters = cluster_cap;
  if (clusters > tiles) clusters = tiles;
  cfg.gridDim = dim3(C::CL * clusters);
  SLSP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, b, e, o, p));
  return SLSP_OK;
}

// Pipeline depth that fits 227 KB of smem for each configuration.
constexpr int stages_for(bool sparse, int msub, bool raw) {
  if (msub == 1) return sparse ? 4 : 6;
  return sparse ? (raw ? 2 : 3) : (raw ? 3 : 4);
}

template <bool SPARSE, MmaKind K, int BN, int CL, int MSUB>
int run_out_cl(int out_mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o,
               const Params& p, cudaStream_t s) {
  constexpr int SR = stages_for(SPARSE, MSUB, true), SB = stages_for(SPARSE, MSUB, false);
  switch (out_mode) {
    case SLSP_OUT_RAW_NM: return run<Cfg<SPARSE, K, BN, SR, SLSP_OUT_RAW_NM, CL, MSUB>>(a, b, e, o, p, s);
    case SLSP_OUT_BF16_NM: return run<Cfg<SPARSE, K, BN, SB, SLSP_OUT_BF16_NM, CL, MSUB>>(a, b, e, o, p, s);
    case SLSP_OUT_BF16_MN: return run<Cfg<SPARSE, K, BN, SB, SLSP_OUT_BF16_MN, CL, MSUB>>(a, b, e, o, p, s);
  }
  return SLSP_ERR_INVALID;
}

// Tile shape knobs: cluster 2 (one CTA pair) or 4 (two pairs sharing
// activation tiles by TMA multicast), and 1 or 2 M-subtiles per pair; env
// SLSP_GEMM_CLUSTER / SLSP_GEMM_MSUB override the per-kernel defaults.
template <bool SPARSE, MmaKind K, int BN>
int run_out(int out_mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o,
            const Params& p, cudaStream_t s, uint32_t cluster, uint32_t msub) {
  if (cluster == 4)
    return msub == 2 ? run_out_cl<SPARSE, K, BN, 4, 2>(out_mode, a, b, e, o, p, s)
                     : run_out_cl<SPARSE, K, BN, 4, 1>(out_mode, a, b, e, o, p, s);
  return msub == 2 ? run_out_cl<SPARSE, K, BN, 2, 2>(out_mode, a, b, e, o, p, s)
                   : run_out_cl<SPARSE, K, BN, 2, 1>(out_mode, a, b, e, o, p, s);
}

constexpr int kSparseBN = 224;
constexpr int kDenseBN = 256;
constexpr uint32_t kSparseCluster = 2;
constexpr uint32_t kDenseCluster = 2;
constexpr uint32_t kSparseMsub = 1;
constexpr uint32_t kDenseMsub = 1;
constexpr uint32_t kRasterGroup = 16;  // measured best of {4, 8, 16, 32, 148} on Qwen2.5-7B shapes

int check_out(int out_mode, const float* s_ch, const float* s_tok, void* out, int64_t ldo, int64_t n, int64_t m) {
  if (!out) return SLSP_ERR_INVALID;
  if (out_mode == SLSP_OUT_RAW_NM || out_mode == SLSP_OUT_BF16_NM) {
    if (ldo < m) return SLSP_ERR_INVALID;
  } else if (out_mode == SLSP_OUT_BF16_MN) {
    if (ldo < n) return SLSP_ERR_INVALID;
  } else {
    return SLSP_ERR_INVALID;
  }
  if (out_mode != SLSP_OUT_RAW_NM && (!s_ch || !s_tok)) return SLSP_ERR_INVALID;
  return SLSP_OK;
}

}  // namespace

extern "C" {

int slsp_sparse_gemm(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                     int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                     slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || kp <= 0) return SLSP_ERR_INVALID;
  if (kp % 256 != 0) return SLSP_ERR_DIMENSION;
  if (kp > (int64_t{1} << 23)) return SLSP_ERR_INVALID;  // gemm.hpp:56 int8 accumulator bound
  if (n > (int64_t{1} << 31) - 256 || m > (int64_t{1} << 31) - 256) return SLSP_ERR_UNSUPPORTED;
  int st = check_out(out_mode, s_ch, s_tok, out, ldo, n, m);
  if (st) return st;
  if (dtype != SLSP_DT_I8 && dtype != SLSP_DT_E4M3) return SLSP_ERR_UNSUPPORTED;
  if ((st = require_sm100())) return st;
  if (n == 0 || m == 0) return SLSP_OK;
  CUtensorMap ta, tb, te, to;
  Params p{};
  if ((st = make_map_2d(&ta, values, kp / 2, n, 128))) return st;
  // activation box: the CTA's half of the N tile, split once more across the
  // pairs of a 4-CTA cluster (each pair fetches one slice and multicasts it)
  const uint32_t cluster = env_knob("SLSP_GEMM_CLUSTER", kSparseCluster) == 4 ? 4 : 2;
  const uint32_t msub = env_knob("SLSP_GEMM_MSUB", kSparseMsub) == 2 ? 2 : 1;
  if ((st = make_map_2d(&tb, act, kp, m, kSparseBN / 2 / (cluster / 2)))) return st;
  if ((st = make_map_meta(&te, meta, n, kp))) return st;
  if ((st = make_map_out(&to, out, out_mode, n, m, ldo, msub == 2 ? 16 : 32, &p.tma_store))) return st;
  select_epilogue(p, out_mode, msub);
  p.n = n;
  p.m = m;
  p.num_kb = static_cast<int>(kp / 256);
  p.s_ch = s_ch;
  p.s_tok = s_tok;
  p.out = out;
  p.ldo = ldo;
  p.debug = debug_flags();
  p.hints = env_knob("SLSP_GEMM_HINTS", kDefaultHints);
  p.group = static_cast<int>(env_knob("SLSP_GEMM_GROUP", kRasterGroup));
  if (dtype == SLSP_DT_I8)
    return run_out<true, MmaKind::I8, kSparseBN>(out_mode, ta, tb, te, to, p, s, cluster, msub);
  return run_out<true, MmaKind::F8, kSparseBN>(out_mode, ta, tb, te, to, p, s, cluster, msub);
}

int slsp_dense_gemm(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m, const float* s_ch,
                    const float* s_tok, int out_mode, void* out, int64_t ldo, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || k <= 0) return SLSP_ERR_INVALID;
  const int esz = elem_size(dtype);
  if (dtype != SLSP_DT_I8 && dtype != SLSP_DT_E4M3 && dtype != SLSP_DT_BF16) return SLSP_ERR_UNSUPPORTED;
  if ((k * esz) % 128 != 0) return SLSP_ERR_DIMENSION;
  if (dtype == SLSP_DT_I8 && k > (int64_t{1} << 23)) return SLSP_ERR_INVALID;  // gemm.hpp:147-149
  if (n > (int64_t{1} << 31) - 256 || m > (int64_t{1} << 31) - 256) return SLSP_ERR_UNSUPPORTED;
  int st = check_out(out_mode, s_ch, s_tok, out, ldo, n, m);
  if (st) return st;
  if ((st = require_sm100())) return st;
  if (n == 0 || m == 0) return SLSP_OK;
  CUtensorMap ta, tb, to;
  Params p{};
  if ((st = make_map_2d(&ta, w, k * esz, n, 128))) return st;
  const uint32_t cluster = env_knob("SLSP_GEMM_CLUSTER", kDenseCluster) == 4 ? 4 : 2;
  const uint32_t msub = env_knob("SLSP_GEMM_MSUB", kDenseMsub) == 2 ? 2 : 1;
  if ((st = make_map_2d(&tb, act, k * esz, m, kDenseBN / 2 / (cluster / 2)))) return st;
  if ((st = make_map_out(&to, out, out_mode, n, m, ldo, msub == 2 ? 16 : 32, &p.tma_store))) return st;
  select_epilogue(p, out_mode, msub);
  p.n = n;
  p.m = m;
  p.num_kb = static_cast<int>(k * esz / 128);
  p.s_ch = s_ch;
  p.s_tok = s_tok;
  p.out = out;
  p.ldo = ldo;
  p.debug = debug_flags();
  p.hints = env_knob("SLSP_GEMM_HINTS", kDefaultHints);
  p.group = static_cast<int>(env_knob("SLSP_GEMM_GROUP", kRasterGroup));
  if (dtype == SLSP_DT_I8)
    return run_out<false, MmaKind::I8, kDenseBN>(out_mode, ta, tb, ta, to, p, s, cluster, msub);
  if (dtype == SLSP_DT_E4M3)
    return run_out<false, MmaKind::F8, kDenseBN>(out_mode, ta, tb, ta, to, p, s, cluster, msub);
  return run_out<false, MmaKind::F16, kDenseBN>(out_mode, ta, tb, ta, to, p, s, cluster, msub);
}

}  // extern "C"
