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
// only (L2-resident operands), bit3 skip metadata loads, bit4 skip the MMAs
// (load pipeline alone). Results are garbage when set; perf probing only.
// bit5 skips the activation (B) load of every third k-block (in-SM lifting
// emulation: the L2 traffic of a kernel that builds those stages in smem).
// bit6 (LIFT) skips the C-block build, bit7 (LIFT) skips its proxy fence.
enum : uint32_t { kDbgNoStore = 1u, kDbgNoLoad = 2u, kDbgSameTile = 4u, kDbgNoMeta = 8u, kDbgNoMma = 16u,
                  kDbgSkipB3 = 32u, kDbgNoBuild = 64u, kDbgNoFence = 128u, kDbgNoAmaxAtomic = 256u,
                  kDbgNoSts = 512u };
// L2 cache-policy hints (env SLSP_GEMM_HINTS overrides kDefaultHints).
enum : uint32_t { kHintBLast = 1u, kHintAFirst = 2u, kHintOutFirst = 4u };
constexpr uint32_t kDefaultHints = kHintBLast | kHintOutFirst;

// Epilogue chunk width (columns per tcgen05.ld + TMA store box).
constexpr int epi_cols(int msub, int bn, int out) {
  // msub 2: the register-staged BF16 [N][M] epilogue stores 32-column boxes;
  // the generic path drains 16-column chunks
  return msub == 2 ? (out != SLSP_OUT_RAW_NM ? 32 : 16) : (out == SLSP_OUT_RAW_NM || bn % 64 != 0) ? 32 : 64;
}

template <bool SPARSE_, MmaKind KIND_, int BN_, int STAGES_, int OUT_, int MSUB_ = 1, int LIFT_ = 0, int KH_ = 0,
          int NPAIR_ = 1, int AMAX_ = 0>
struct Cfg {
  // §8f #3: the token |y|max fold compiled in (slsp_sparse_gemm_amax only; the
  // plain kernels carry none of its registers)
  static constexpr bool AMAX = AMAX_ != 0;
  static constexpr bool SPARSE = SPARSE_;
  static constexpr MmaKind KIND = KIND_;
  static constexpr int BN = BN_;          // tokens per pair tile (MMA N)
  static constexpr int OUT = OUT_;
  // Weight multicast: NPAIR CTA pairs per cluster run the SAME weight tile on
  // NPAIR consecutive token tiles. Each weight subtile (A + metadata) of a
  // stage is fetched from L2 once, by one pair, and TMA-multicast into the
  // same ring slot of every pair (the rank-r CTAs of all pairs); activations
  // stay per pair. L2->SM bytes per stage and pair drop from A+E+B to
  // (A+E)/NPAIR+B; the pairs' rings run in lockstep (a slot is refilled once
  // every pair's MMAs released it).
  static constexpr int NPAIR = NPAIR_;
  static constexpr int CL = 2 * NPAIR;    // CTAs per cluster
  // M-subtiles: the pair runs MSUB UMMAs (M=256 each) per k-step against the
  // same activation stage, so B traffic per MAC drops by MSUB. TMEM then holds
  // MSUB accumulators per tile; with MSUB=2 they are single-buffered and
  // 4*MSUB epilogue warps drain them in parallel.
  static constexpr int MSUB = MSUB_;
  static_assert(MSUB == 1 || MSUB == 2, "one or two M-subtiles per pair");
  static_assert(NPAIR == 1 || (MSUB == 2 && NPAIR == 2), "weight multicast: two pairs, one subtile each");
  // In-SM lifting (sparse, (2N-2):2N with 8 | 2N... here 6:8): the activation
  // operand arrives UNLIFTED (quantized X, K bytes per token) and the lifted
  // K' is consumed in the GEMM window order of slsp_gemm_order: per 512
  // source bytes, two "X" k-blocks whose B tile is X itself (windows 0 and 2
  // of each 8-block are its bytes 0-3 and 4-7) and one "C" k-block holding
  // window 1 (bytes 2-5) of those 64 blocks, which LIFT_WARPS build in shared
  // memory from the two X tiles. The lifted activation never exists in HBM
  // or L2, and a third of the B operand's L2->SM traffic disappears.
  static constexpr bool LIFT = LIFT_ == 1;
  static_assert(!LIFT || SPARSE, "in-SM lifting feeds the sparse kernel");
  // GLIFT (LIFT_ == 2, decode-shaped BF16): the lift happens inside the
  // GEMM — four lift warps build each ring stage's B tile (the lifted
  // activations of this CTA's tokens) straight from the unlifted BF16 X in
  // global memory (L2-resident at decode M), so no lift kernel runs at all.
  static constexpr bool GLIFT = LIFT_ == 2;
  static_assert(!GLIFT || (SPARSE && KIND == MmaKind::F16 && MSUB == 1), "in-GEMM lift: BF16 one-subtile tiles");
  static constexpr int GLIFT_GROUPS = 4, GLIFT_GW = 2;  // stage groups x warps per group
  static constexpr int LIFT_WARPS = LIFT ? 2 : GLIFT ? GLIFT_GROUPS * GLIFT_GW : 0;
  // lift-warp arrivals per CTA on a stage's full barrier
  static constexpr int LIFT_ARRIVE = LIFT ? LIFT_WARPS : GLIFT ? GLIFT_GW : 0;
  // double-buffered accumulators where two (and the sparse metadata
  // columns) fit the 512 TMEM columns: one-subtile tiles up to 224 tokens
  // (sparse) / 256 (dense); 256-token sparse tiles drain in between
  static constexpr int ACC_STAGES = MSUB == 1 && 2 * BN + (SPARSE ? 8 : 0) <= 512 ? 2 : 1;
  static constexpr int EPI_WARPS = 4 * MSUB;
  static constexpr int THREADS = 64 + 32 * (EPI_WARPS + LIFT_WARPS);
  static constexpr int BM = 256 * MSUB;   // weight rows per pair tile
  static constexpr int A_ROWS = 128;      // per CTA per M-subtile
  static constexpr int B_ROWS = BN / 2;   // tokens per CTA
  static_assert(!LIFT || B_ROWS % (8 * (LIFT ? LIFT_WARPS : 1)) == 0, "lift warps own whole 8-row swizzle groups");
  // Half k-stages (sparse 8-bit kinds): 128 lifted bytes per stage instead of
  // 256 — A rows of 64 B (64B swizzle), one B atom, one metadata atom, 2 MMAs
  // per subtile — so the same ring holds twice as many, half-size stages
  // (6 x 34 KB for MSUB=2 instead of 3 x 68 KB): more latency cover per byte.
  static constexpr bool KH = KH_ != 0;
  static_assert(!KH || (SPARSE && KIND != MmaKind::F16 && !LIFT), "half k-stages: sparse 8-bit kinds");
  static constexpr int A_ROW = KH ? 64 : 128;                // A bytes per row per stage
  static constexpr uint32_t A_LAYOUT = KH ? 4u : 2u;         // UMMA desc: SWIZZLE_64B / SWIZZLE_128B
  static constexpr int A_SUB = 128 * A_ROW;                  // one swizzle-atom column of 128 rows
  static constexpr int A_STAGE = MSUB * A_SUB;
  static constexpr int B_ATOMS = SPARSE && !KH ? 2 : 1;      // B bytes per stage = 2x A bytes for .sp
  static constexpr int B_ATOM = B_ROWS * 128;
  static constexpr int B_STAGE = B_ATOM * B_ATOMS;
  // 128x128b metadata atoms per stage and subtile: a stage is 128 bytes of
  // compressed A per row = 256 logical k for 8-bit kinds (2 atoms, 2 TMEM
  // columns per K=64 MMA) and 128 logical k for BF16 (1 atom, 1 column per
  // K=32 MMA); 1 metadata bit per logical k either way
  static constexpr int E_ATOMS = (KIND == MmaKind::F16 || KH) ? 1 : 2;
  static constexpr int E_PER_MMA = KIND == MmaKind::F16 ? 1 : 2;
  static constexpr int E_SUB = SPARSE ? E_ATOMS * 128 * 16 : 0;
  static constexpr int E_STAGE = MSUB * E_SUB;
  static constexpr int STAGE_TX = A_STAGE + B_STAGE + E_STAGE;
  static constexpr int K_BYTES_B = 128 * B_ATOMS;            // activation bytes consumed per stage
  static constexpr int MMAS = KH ? 2 : 4;                    // k-steps per stage
  static constexpr int ACC_COLS = BN;                        // 32-bit TMEM columns per accumulator
  static constexpr int E_COL = ACC_STAGES * MSUB * BN;       // metadata columns after the accumulators
  static constexpr int TMEM_COLS = 512;
  static_assert(!SPARSE || E_COL + 8 * MSUB <= TMEM_COLS, "TMEM budget: accumulators + metadata");
  static_assert(SPARSE || E_COL <= TMEM_COLS, "TMEM budget: accumulators");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "cta_group::2 N");
  // epilogue: chunks of 32 rows x EPI_COLS columns, double-buffered smem
  // staging per warp (a TMA store reads one buffer while the next is filled)
  static constexpr int OUT_ESZ = OUT == SLSP_OUT_RAW_NM ? 4 : 2;
  // MSUB=1: 128-byte staging rows (64 BF16 / 32 int32 columns), so every TMA
  // store writes whole 128-byte lines (measured: L2 write cost is per request)
  static constexpr int EPI_COLS = epi_cols(MSUB, BN, OUT);
  // (LIFT with two subtiles: one staging buffer, so the ring keeps 3 stages)
  static constexpr int EPI_BUFS = LIFT && MSUB == 2 ? 1 : 2;
  static constexpr int EPI_BUF = 32 * EPI_COLS * OUT_ESZ;
  static constexpr int EPI_ROW = EPI_COLS * OUT_ESZ;  // staging row bytes (NM layout) = swizzle span
  // MSUB=2 with BF16 [N][M] output: register-staged epilogue (each subtile is
  // dequantised into registers and its TMEM released before any store), no
  // smem staging.
  // (token-major [M][N] output too: the same drain, the staged boxes
  // transposed in shared memory before the TMA store)
  static constexpr bool REG_EPI = MSUB == 2 && OUT != SLSP_OUT_RAW_NM && !(LIFT && OUT == SLSP_OUT_BF16_MN);
  static constexpr int H0 = (BN / 2 + 31) / 32 * 32;  // REG: columns of the first warp of a lane quarter
  // REG: s_tok slice + one 32x32 BF16 staging box per warp
  static constexpr int EPI_WARP = REG_EPI ? H0 * 4 + 32 * 64 : EPI_BUFS * EPI_BUF;
  // cluster split-K (Params::ksc): one-subtile decode tiles whose per-warp
  // staging area holds the warp's 32 rows x BN raw accumulators
  static constexpr bool KSC_OK = MSUB == 1 && NPAIR == 1 && !AMAX && !LIFT && !REG_EPI && BN <= 64 &&
                                 EPI_WARP >= 32 * BN * 4;
  // smem ring depth: STAGES_ if given, else as many stages as fit (<= 8)
  static constexpr int FIXED_SMEM0 = EPI_WARPS * EPI_WARP + 4 * 8 + 16 + 1024;
  static constexpr int FIT0 = (227 * 1024 - FIXED_SMEM0) / (STAGE_TX + 16);
  // §8f #3 token |y|max fold (BF16 outputs): a per-CTA [2][BN] merge buffer
  // where it costs no ring stage; otherwise the fold goes to global atomics
  // per warp
  static constexpr int AMAX_CAND = AMAX && SPARSE && OUT != SLSP_OUT_RAW_NM ? 2 * BN * 4 : 0;
  static constexpr bool AMAX_SM =
      AMAX_CAND > 0 && (227 * 1024 - FIXED_SMEM0 - AMAX_CAND) / (STAGE_TX + 16) >= (FIT0 < 8 ? FIT0 : 8);
  static constexpr int AMAX_BYTES = AMAX_SM ? AMAX_CAND : 0;
  static constexpr int FIXED_SMEM = FIXED_SMEM0 + AMAX_BYTES;
  static constexpr int FIT = (227 * 1024 - FIXED_SMEM) / (STAGE_TX + 16);
  static constexpr int STAGES = STAGES_ ? STAGES_ : (FIT < 8 ? FIT : 8);
  static_assert(STAGES >= 2, "pipeline depth");
  // LIFT: an X block, its partner and their C block are in the ring at once
  static_assert(!LIFT || STAGES >= 3, "in-SM lifting needs >= 3 ring stages");
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_STAGE;
  static constexpr int OFF_E = OFF_B + STAGES * B_STAGE;
  static constexpr int OFF_EPI = OFF_E + STAGES * E_STAGE;
  static constexpr int OFF_AMAX = OFF_EPI + EPI_WARPS * EPI_WARP;
  static constexpr int OFF_BAR = OFF_AMAX + AMAX_BYTES;
  // Two-subtile stages signal subtile 1's operands (A1, E1) on a second
  // barrier, so subtile 0's MMAs start once B, A0 and E0 have landed.
  static constexpr bool SPLIT = MSUB == 2 && SPARSE && !LIFT;
  // full, empty, xfull, full1 per stage; tfull, tempty; red_full, red_empty (cluster split-K)
  static constexpr int NUM_BARS = 4 * STAGES + 6;
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
  int direct_vec;     // direct stores: 0 scalar, 1 rows 16-byte aligned (v4), 2 rows 32-byte aligned (v8)
  int stok_vec;       // s_tok is 16-byte aligned (float4 loads)
  uint32_t debug;
  unsigned long long* trace;  // perf probing: per-tile clock64 stamps of CTA 0 (env SLSP_GEMM_TRACE = device ptr)
  uint32_t hints;     // kHint* L2 policies
  int group;          // weight tiles per raster band
  // split-K (decode-shaped M): each (weight tile, token tile) is cut into
  // ksplit k-ranges; slice s stores its raw partial accumulators (int32 /
  // fp32) into ws[s][n][m] and a finishing kernel sums the slices in order
  // (deterministic; exact for int32) and applies the epilogue. ksplit == 1:
  // the normal epilogue.
  int splitbar;  // SPLIT configs: per-subtile full barriers (env SLSP_GEMM_SPLITBAR, default 1)
  // MSUB=2: issue subtile 0's MMAs of the last `tail0` k-blocks of a tile
  // before subtile 1's and commit them to their own barrier (tfull[1]), so the
  // epilogue drains subtile 0 while subtile 1 finishes and the next tile's
  // subtile-0 MMAs start sooner (env SLSP_GEMM_TAIL0: 0 = one commit per tile
  // after both subtiles, 1 = early subtile-0 commit only, 2 = + last two
  // k-blocks reordered)
  int tail0;
  int ksplit;
  int pf_stages;  // L2-prefetch the next tile's first pf_stages k-blocks (env SLSP_GEMM_PF)
  int pf_at;      // ... when this tile's k-block pf_at is issued (env SLSP_GEMM_PFAT)
  int pace_ns;   // REG epilogue: sleep between output boxes (env SLSP_GEMM_PACE, perf probing)
  void* ws;
  int64_t ws_cap;  // workspace bytes (bounds ksplit)
  // SURVEY §8f #3 (lift fused upstream): BF16 outputs also fold max |y| of
  // every token (over this launch's output features) into amax[t] (float
  // bits; atomicMax on the bit pattern is exact for non-negative values, and
  // a NaN |y| (0x7FC0.. > Inf) wins, so the consumer sees the row as
  // non-finite). The next layer's lift then needs no |x|max pass of its own.
  uint32_t* amax;
  // GLIFT: the unlifted BF16 X (m x k, row stride x_ld elements) and the
  // pattern's window geometry (l, windows per block, lifted windows per row)
  const void* x;
  int64_t x_ld;
  int lift_l, lift_wc;
  int64_t lift_windows;
  // cluster split-K (decode tiles, Cfg::KSC_OK): the cluster holds ksc CTA
  // pairs that take consecutive k-ranges of ONE tile (the same ranges as a
  // ksc-way workspace split); each pair parks its raw partial accumulators in
  // its epilogue staging smem, and every CTA then sums a 1/ksc row share of
  // the tile over the pairs' buffers through distributed shared memory (in
  // slice order: the finishing kernel's arithmetic) and applies the epilogue.
  // No workspace, no finishing launch. 0/1: none.
  int ksc;
};

// Fold |bf16| of 2*NW token columns (packed in w, token i = half i&1 of
// w[i>>1]) over the warp's 32 rows (lanes): sm != 0 -> max into the CTA's
// shared [BN] merge buffer at column c0 + i (flushed to p.amax once per tile
// by fold_flush), else straight into p.amax[t0 + i]. Lanes whose rows are
// past n hold zeros (their scale is 0), so they are neutral.
template <int NW>
SLSP_DEVINL void fold_token_amax(const Params& p, const uint32_t (&w)[NW], int64_t t0, uint32_t sm = 0,
                                 int c0 = 0) {
  constexpr int NC = 2 * NW;
  const uint32_t lane = lane_id();
  if constexpr (NW == 8) {
    // 16 tokens: transposing butterfly on packed |bf16| pairs (9 shuffles +
    // 9 per-halfword max) instead of 16 warp reductions; afterwards lane L
    // holds the column max of token pair (L >> 2) & 7, four lanes each
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = w[i] & 0x7FFF7FFFu;
    const bool b4 = lane & 16u, b3 = lane & 8u, b2 = lane & 4u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t keep = b4 ? v[i + 4] : v[i], send = b4 ? v[i] : v[i + 4];
      v[i] = __vmaxu2(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t keep = b3 ? v[i + 2] : v[i], send = b3 ? v[i] : v[i + 2];
      v[i] = __vmaxu2(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    uint32_t x;
    {
      const uint32_t keep = b2 ? v[1] : v[0], send = b2 ? v[0] : v[1];
      x = __vmaxu2(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    x = __vmaxu2(x, __shfl_xor_sync(0xffffffffu, x, 2));
    x = __vmaxu2(x, __shfl_xor_sync(0xffffffffu, x, 1));
    if ((lane & 3u) < 2u && !(p.debug & kDbgNoAmaxAtomic)) {
      const int col = 2 * static_cast<int>((lane >> 2) & 7u) + static_cast<int>(lane & 1u);
      const uint32_t val = (lane & 1u) ? (x & 0xFFFF0000u) : (x << 16);
      if (t0 + col < p.m) {
        if (sm) asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(sm + 4u * (c0 + col)), "r"(val) : "memory");
        else atomicMax(p.amax + t0 + col, val);
      }
    }
    return;
  }
  uint32_t mine[(NC + 31) / 32];
#pragma unroll
  for (int j = 0; j < (NC + 31) / 32; ++j) mine[j] = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const uint32_t h = (w[i >> 1] >> (16 * (i & 1))) & 0x7FFFu;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, h);
    if (lane == static_cast<uint32_t>(i & 31)) mine[i >> 5] = mx;
  }
#pragma unroll
  for (int j = 0; j < (NC + 31) / 32; ++j) {
    const int64_t t = t0 + 32 * j + lane;
    if (32 * j + static_cast<int>(lane) < NC && t < p.m && !(p.debug & kDbgNoAmaxAtomic)) {
      if (sm) asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(sm + 4u * (c0 + 32 * j + lane)), "r"(mine[j] << 16)
                           : "memory");
      else atomicMax(p.amax + t, mine[j] << 16);
    }
  }
}

// Epilogue warps only (named barrier 1).
template <int NT>
SLSP_DEVINL void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// After every epilogue warp folded tile `it` into merge buffer it&1: one
// warp moves the BN column maxima to p.amax (one atomic per token per CTA)
// and clears the buffer for tile it+2 (tile it+1 uses the other one).
template <int BN, int NT>
SLSP_DEVINL void fold_flush(const Params& p, uint32_t* buf, int64_t tcol0, bool first_warp) {
  epi_bar<NT>();
  if (first_warp) {
    for (int c = static_cast<int>(lane_id()); c < BN; c += 32) {
      const uint32_t v = buf[c];
      if (v && tcol0 + c < p.m && !(p.debug & kDbgNoAmaxAtomic)) atomicMax(p.amax + tcol0 + c, v);
      buf[c] = 0;
    }
  }
}

// Perf probing: slot `slot` of tile iteration `it` on CTA 0 (16 slots per tile;
// 8/9 hold the MMA's full-wait and the producer's empty-wait cycles of the tile).
#define SLSP_TRACE(it, slot)                                                          \
  do {                                                                                \
    if (p.trace && blockIdx.x == 0) p.trace[(it) * 16 + (slot)] = clock64();           \
  } while (0)

// Raster: bands of `group` weight tiles; within a band the weight tile varies
// fastest, so the clusters running concurrently share activation tiles (B)
// and each band's weight tiles stay L2-resident while the band sweeps tokens.
// n_count: token super-tiles (NPAIR token tiles each).
SLSP_DEVINL void tile_coords(int tile, const Params& p, int m_count, int n_count, int& mt, int& nt, int& kb0,
                             int& kb1, uint32_t kslice = 0, int ksc = 1) {
  const int ks = tile % p.ksplit;  // split-K slice (innermost: the slices of a tile run concurrently)
  tile /= p.ksplit;
  kb0 = ks * p.num_kb / p.ksplit;
  kb1 = (ks + 1) * p.num_kb / p.ksplit;
  if (ksc > 1) {  // cluster split-K: this pair's k-range (same bounds as a ksc-way workspace split)
    kb0 = static_cast<int>(kslice) * p.num_kb / ksc;
    kb1 = (static_cast<int>(kslice) + 1) * p.num_kb / ksc;
  }
  const int per_group = p.group * n_count;
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

// Compiler barrier on 8 registers: the values are materialised at this point
// in program order (asm volatile is not reordered against the mbarrier ops).
SLSP_DEVINL void reg_pin(uint32_t (&w)[8]) {
  asm volatile("" : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7]));
}

// Element-wise BF16 stores of the first `valid` values of a packed row segment.
__device__ __noinline__ void store_tail_u16(uint16_t* dst, const uint32_t* w, int valid) {
  for (int i = 0; i < valid; ++i) dst[i] = static_cast<uint16_t>(w[i >> 1] >> (16 * (i & 1)));
}

// a18 for 16 consecutive tokens whose scales sit in shared memory.
template <typename Acc>
SLSP_DEVINL void dequant16_smem(const uint32_t (&r)[16], float sc, uint32_t st_sm, uint32_t (&w)[8]) {
  float st[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 v = ld_shared_f4(st_sm + 16 * q);
    st[4 * q] = v.x;
    st[4 * q + 1] = v.y;
    st[4 * q + 2] = v.z;
    st[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 a;
    if constexpr (std::is_same<Acc, int32_t>::value) {
      a.x = __int2float_rn(static_cast<int32_t>(r[2 * i]));
      a.y = __int2float_rn(static_cast<int32_t>(r[2 * i + 1]));
    } else {
      a.x = __uint_as_float(r[2 * i]);
      a.y = __uint_as_float(r[2 * i + 1]);
    }
    a = fmul2_rn(fmul2_rn(a, make_float2(sc, sc)), make_float2(st[2 * i], st[2 * i + 1]));
    w[i] = pack_bf16(a.x, a.y);
  }
}

// a18 for 16 consecutive tokens of one row, packed FMUL2 (same two rn
// products per element as dequant()), BF16 pairs out.
template <typename Acc>
SLSP_DEVINL void dequant16(const Params& p, const uint32_t (&r)[16], float sc, int64_t t0, uint32_t (&w)[8]) {
  float st[16];
  if (p.stok_vec && t0 + 16 <= p.m) {
    // volatile loads: issued here, in chunk order (not hoisted for all chunks
    // up front, which would spill)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(st[4 * q]), "=f"(st[4 * q + 1]), "=f"(st[4 * q + 2]), "=f"(st[4 * q + 3])
                   : "l"(p.s_tok + t0 + 4 * q));
  } else {  // token tail: int32 bound, one base pointer
    const int valid = static_cast<int>(imin64(16, p.m - t0));
    const float* base = p.s_tok + t0;
#pragma unroll
    for (int i = 0; i < 16; ++i) st[i] = i < valid ? __ldg(base + i) : 0.f;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 a;
    if constexpr (std::is_same<Acc, int32_t>::value) {
      a.x = __int2float_rn(static_cast<int32_t>(r[2 * i]));
      a.y = __int2float_rn(static_cast<int32_t>(r[2 * i + 1]));
    } else {
      a.x = __uint_as_float(r[2 * i]);
      a.y = __uint_as_float(r[2 * i + 1]);
    }
    a = fmul2_rn(fmul2_rn(a, make_float2(sc, sc)), make_float2(st[2 * i], st[2 * i + 1]));
    w[i] = pack_bf16(a.x, a.y);
  }
}

// One 32-row x EPI_COLS-column chunk of the accumulator (lane = row) to its
// output. TMA path: the chunk is staged in smem in the output's 128B/64B/32B
// swizzle (chunk index ^= row bits, conflict-free 16-byte stores) and written
// with one bulk tensor store.
template <typename C>
SLSP_DEVINL void epilogue_chunk(const Params& p, const CUtensorMap* tmOut, uint8_t* stage,
                                uint32_t (&r)[C::EPI_COLS], int64_t row0, int64_t t0, float sc, uint32_t amax_sm,
                                int c0) {
  constexpr int NC = C::EPI_COLS;
  constexpr int NW = C::OUT == SLSP_OUT_RAW_NM ? NC : NC / 2;  // 32-bit output words per lane
  const uint32_t lane = lane_id();
  const int64_t row = row0 + lane;
  // per-token scales: coalesced loads (32 tokens per load), shuffled to every lane
  constexpr int NST = NC > 32 ? NC / 32 : 1;
  float st_lane[NST];
#pragma unroll
  for (int j = 0; j < NST; ++j) {
    st_lane[j] = 0.f;
    if constexpr (C::OUT != SLSP_OUT_RAW_NM)
      st_lane[j] = (32 * j + lane < NC && t0 + 32 * j + lane < p.m) ? __ldg(p.s_tok + t0 + 32 * j + lane) : 0.f;
  }
  uint32_t w[NW];
  if constexpr (C::OUT == SLSP_OUT_RAW_NM) {
#pragma unroll
    for (int i = 0; i < NC; ++i) w[i] = r[i];
  } else {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const float s0 = __shfl_sync(0xffffffffu, st_lane[(2 * i) >> 5], (2 * i) & 31);
      const float s1 = __shfl_sync(0xffffffffu, st_lane[(2 * i + 1) >> 5], (2 * i + 1) & 31);
      const float lo = dequant<typename C::Acc>(r[2 * i], sc, s0);
      const float hi = dequant<typename C::Acc>(r[2 * i + 1], sc, s1);
      w[i] = pack_bf16(lo, hi);
    }
  }
  if constexpr (C::AMAX && C::OUT != SLSP_OUT_RAW_NM)
    if (p.amax) fold_token_amax<NW>(p, w, t0, amax_sm, c0);
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
  uint64_t* xfull = empty + C::STAGES;  // LIFT: this CTA's X tile of a stage has landed
  uint64_t* full1 = xfull + C::STAGES;  // SPLIT: subtile 1's A/E of a stage have landed
  uint64_t* tfull = full1 + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* red_full = tempty + 2;   // cluster split-K: every pair's partials of this tile are parked
  uint64_t* red_empty = tempty + 3;  // ... and every CTA has read this CTA's partials
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();     // rank in the cluster
  const uint32_t pair = crank >> 1;             // CTA pair within the cluster
  const uint32_t rank = crank & 1;              // rank within the pair (cta_group::2 peer)
  const uint32_t lead = crank & ~1u;            // cluster rank of this pair's leader
  const bool leader = rank == 0;
  // cluster split-K: the cluster is ksc pairs, pair index = k-slice
  const int ksc = C::KSC_OK && p.ksc > 1 ? p.ksc : 1;
  const uint32_t kslice = ksc > 1 ? pair : 0u;
  // token tile within a weight-multicast super-tile (pair is 0 unless NPAIR > 1 or ksc > 1)
  const uint32_t npair_idx = C::KSC_OK && C::NPAIR == 1 ? 0u : pair;
  const int cluster_id = blockIdx.x / (C::CL * ksc);
  const int num_clusters = gridDim.x / (C::CL * ksc);
  // a cluster tile = one weight tile x NPAIR consecutive token tiles (pair p
  // takes token tile ns * NPAIR + p; past the last one it recomputes token
  // tile 0 — its loads stay in bounds — and stores nothing)
  const int n_super = (p.n_tiles + C::NPAIR - 1) / C::NPAIR;
  const int num_tiles = p.m_tiles * n_super * p.ksplit;

#ifdef SLSP_WATCHDOG
  if (threadIdx.x == 0 && blockIdx.x < 2)
    printf("SLSP layout block %d: smem %u A %u B %u E %u EPI %u full %u empty %u xfull %u tfull %u stages %d threads %d\n",
           blockIdx.x, smem_u32(smem), smem_u32(sA), smem_u32(sB), smem_u32(sE), smem_u32(smem + C::OFF_EPI),
           smem_u32(full), smem_u32(empty), smem_u32(xfull), smem_u32(tfull), C::STAGES, C::THREADS);
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      // LIFT: + one arrival per lift warp of both CTAs ("X present" / "C built")
      mbar_init(&full[s], 1 + 2 * C::LIFT_ARRIVE);
      // MMA commit (+ LIFT: each local lift warp is done reading the stage's X tile)
      mbar_init(&empty[s], C::NPAIR + (C::LIFT ? C::LIFT_WARPS : 0));
      mbar_init(&xfull[s], 1);
      mbar_init(&full1[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::EPI_WARPS);  // every epilogue warp of both CTAs of the pair
    }
    if constexpr (C::KSC_OK) {
      mbar_init(red_full, C::EPI_WARPS * ksc);  // the epilogue warps of the ksc same-rank CTAs
      mbar_init(red_empty, C::EPI_WARPS * ksc);
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
  if constexpr (C::AMAX_SM)
    for (int i = threadIdx.x; i < 2 * C::BN; i += C::THREADS) reinterpret_cast<uint32_t*>(smem + C::OFF_AMAX)[i] = 0;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above overlapped the previous kernel's tail; from here
  // on every role touches memory that kernel may have produced or read
  pdl_wait();
  pdl_trigger();

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
      // weight multicast: the rank-r CTA of every pair
      uint16_t mc_mask = 0;
#pragma unroll
      for (int q = 0; q < C::NPAIR; ++q) mc_mask |= static_cast<uint16_t>(1u << (2 * q + rank));
      int it = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
        int mt, ns, kb0, kb1;
        tile_coords(tile, p, p.m_tiles, n_super, mt, ns, kb0, kb1, kslice, ksc);
        int nt = ns * C::NPAIR + static_cast<int>(npair_idx);
        if (nt >= p.n_tiles) nt = 0;  // idle pair of the last super-tile: in-bounds loads, no stores
        if (same) mt = nt = 0;
        long long wait_cycles = 0;
        const int a_row = mt * C::BM + static_cast<int>(rank) * C::A_ROWS;
        const int b_row = nt * C::BN + static_cast<int>(rank) * C::B_ROWS;
        for (int kb = kb0; kb < kb1; ++kb) {
          const int kl = same ? 0 : kb;
          if (p.pf_stages && kb == kb0 + p.pf_at && tile + num_clusters < num_tiles) {
            // warm L2 with the next tile's first k-blocks: at a tile start the
            // ring's first stages are new weight / token tiles whose loads miss
            int mt2, ns2, kc0, kc1;
            tile_coords(tile + num_clusters, p, p.m_tiles, n_super, mt2, ns2, kc0, kc1, kslice, ksc);
            int nt2 = ns2 * C::NPAIR + static_cast<int>(npair_idx);
            if (nt2 >= p.n_tiles) nt2 = 0;
            const int a2 = mt2 * C::BM + static_cast<int>(rank) * C::A_ROWS;
            const int b2 = nt2 * C::BN + static_cast<int>(rank) * C::B_ROWS;
            const int kend = min(kc1, kc0 + p.pf_stages);
            for (int k2 = kc0; k2 < kend; ++k2) {
#pragma unroll
              for (int h = 0; h < C::MSUB; ++h) {
                tma_prefetch_l2_2d(&tmA, k2 * C::A_ROW, a2 + h * 256);
                if constexpr (C::SPARSE)
                  tma_prefetch_l2_2d(&tmE, 0, (((a2 + h * 256) >> 7) * p.num_kb + k2) * 8 * C::E_ATOMS);
              }
              if constexpr (!C::LIFT && !C::GLIFT)
#pragma unroll
                for (int at = 0; at < C::B_ATOMS; ++at) tma_prefetch_l2_2d(&tmB, k2 * C::K_BYTES_B + at * 128, b2);
            }
          }
          if (p.trace) {
            const long long t0 = clock64();
            mbar_wait(&empty[stage], phase ^ 1);
            wait_cycles += clock64() - t0;
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
          }
          // LIFT: k-blocks come in periods of 3 (X, X, C); C blocks load no activations
          const bool xstage = !C::LIFT || kb % 3 != 2;
          if (no_load) {
            if (leader) mbar_arrive(&full[stage]);
            if (C::LIFT) mbar_arrive(&xfull[stage]);
            if (C::SPLIT && leader) mbar_arrive(&full1[stage]);
          } else {
            const bool skip_e = p.debug & kDbgNoMeta;
            if (p.trace && blockIdx.x == 0 && it < 16 && kb < 256) p.trace[65536 + (it * 256 + kb) * 2] = clock64();
            const bool skip_b = !C::LIFT && (p.debug & kDbgSkipB3) && kb % 3 == 2;
            const bool split = C::SPLIT && p.splitbar;
            const uint32_t tx_all = 2 * (C::STAGE_TX - (skip_e ? C::E_STAGE : 0) -
                                         ((skip_b || C::LIFT || C::GLIFT) ? C::B_STAGE : 0));
            const uint32_t tx1 = split ? 2 * (C::A_SUB + (skip_e ? 0 : C::E_SUB)) : 0;
            if (leader) {
              mbar_arrive_expect_tx(&full[stage], tx_all - tx1);
              if constexpr (C::SPLIT) {
                if (split) mbar_arrive_expect_tx(&full1[stage], tx1);
                else mbar_arrive(&full1[stage]);
              }
            }
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), lead);
            const uint32_t bar1 = split ? mapa_shared(smem_u32(&full1[stage]), lead) : bar;
#pragma unroll
            for (int h = 0; h < C::MSUB; ++h) {
              if constexpr (C::NPAIR == 1) {
                tma_load_2d_cg2_hint(sA + stage * C::A_STAGE + h * C::A_SUB, &tmA, h ? bar1 : bar, kl * C::A_ROW,
                                     a_row + h * 256, pol_a);
              } else if (h % C::NPAIR == static_cast<int>(pair)) {
                // subtile h: fetched once by pair h, multicast to the rank-r CTA of every pair;
                // each destination reports the bytes to its own pair leader's barrier
                tma_load_2d_cg2_mc(sA + stage * C::A_STAGE + h * C::A_SUB, &tmA, h ? bar1 : bar, kl * C::A_ROW,
                                   a_row + h * 256, mc_mask, pol_a);
              }
            }
            if constexpr (C::LIFT) {
              // X block j of period q: source bytes [512q + 256j, +256) into this CTA (local barrier)
              // xfull completes once per ring lap (slots alternate between X
              // and C blocks when STAGES % 3 != 0): C blocks arrive without bytes
              if (!xstage) mbar_arrive(&xfull[stage]);
              if (xstage) {
                mbar_arrive_expect_tx(&xfull[stage], C::B_STAGE);
                const int k0 = (kl / 3) * 512 + (kl % 3) * 256;
#pragma unroll
                for (int at = 0; at < C::B_ATOMS; ++at)
                  tma_load_2d_hint(sB + stage * C::B_STAGE + at * C::B_ATOM, &tmB, smem_u32(&xfull[stage]),
                                   k0 + at * 128, b_row, pol_b);
              }
            } else if constexpr (!C::GLIFT) {
#pragma unroll
              for (int at = 0; at < C::B_ATOMS; ++at) {
                if (skip_b) break;
                tma_load_2d_cg2_hint(sB + stage * C::B_STAGE + at * C::B_ATOM, &tmB, bar, kl * C::K_BYTES_B + at * 128,
                                     b_row, pol_b);
              }
            }
            if constexpr (C::SPARSE)  // one contiguous 4 KB tiled-metadata block per stage and subtile
              if (!skip_e)
#pragma unroll
                for (int h = 0; h < C::MSUB; ++h) {
                  const int erow = (((a_row + h * 256) >> 7) * p.num_kb + kl) * 8 * C::E_ATOMS;
                  if constexpr (C::NPAIR == 1)
                    tma_load_2d_cg2_hint(sE + stage * C::E_STAGE + h * C::E_SUB, &tmE, h ? bar1 : bar, 0, erow, pol_a);
                  else if (h % C::NPAIR == static_cast<int>(pair))
                    tma_load_2d_cg2_mc(sE + stage * C::E_STAGE + h * C::E_SUB, &tmE, h ? bar1 : bar, 0, erow, mc_mask,
                                       pol_a);
                }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (p.trace && blockIdx.x == 0) p.trace[it * 16 + 9] = wait_cycles;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer ----
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      // ring slots are freed in every CTA whose TMA fills them: the pair, or
      // with weight multicast every pair of the cluster
      const uint16_t all_ctas = C::NPAIR > 1  ? static_cast<uint16_t>((1u << C::CL) - 1)
                                : C::KSC_OK ? static_cast<uint16_t>(0x3u << lead)
                                            : static_cast<uint16_t>(0x3u);
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
        int mt_, ns_, kb0, kb1;
        tile_coords(tile, p, p.m_tiles, n_super, mt_, ns_, kb0, kb1, kslice, ksc);
        const int acc = C::ACC_STAGES == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = C::ACC_STAGES == 2 ? ((it >> 1) & 1) : (it & 1);
        // MSUB=1: double-buffered accumulators, tempty[acc]. MSUB=2: one
        // buffer per subtile and a barrier per subtile; subtile 0 of this tile
        // starts as soon as the epilogue has released it, and subtile 1's MMAs
        // for the first (up to STAGES) k-blocks are deferred until its drain
        // completes, so the drains hide behind the mainloop.
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        SLSP_TRACE(it, 0);
        if (p.trace && blockIdx.x == 0) {  // wall clock beside clock64: the SM clock the tile ran at
          unsigned long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          p.trace[it * 16 + 10] = gt;
        }
        const uint32_t d_tmem = tmem + acc * C::MSUB * C::ACC_COLS;
        // subtile h's metadata copy + 4 MMAs for k-block kb held in ring stage st
        const bool no_mma = p.debug & kDbgNoMma;
        auto issue = [&](int h, int st, int kb) {
          if (no_mma) return;
          const uint32_t a_base = smem_u32(sA + st * C::A_STAGE + h * C::A_SUB);
          const uint32_t b_base = smem_u32(sB + st * C::B_STAGE);
          // KH: alternate halves of the subtile's 8 metadata columns between stages
          const uint32_t e_col = C::E_COL + 8 * h + (C::KH ? 4 * (kb & 1) : 0);
          if constexpr (C::SPARSE) {
            const uint32_t e_base = smem_u32(sE + st * C::E_STAGE + h * C::E_SUB);
#pragma unroll
            for (int c = 0; c < C::E_ATOMS; ++c)
              tmem_cp_128x128b_cg2(tmem + e_col + 4 * c, smem_desc(e_base + c * 2048, 2048, 128, 0));
          }
#pragma unroll
          for (int j = 0; j < C::MMAS; ++j) {
            const uint32_t acc_flag = (kb != kb0 || j != 0) ? 1u : 0u;
            const uint64_t adesc = smem_desc(a_base + j * 32, 16, 8 * C::A_ROW, C::A_LAYOUT);
            const uint32_t d = d_tmem + h * C::ACC_COLS;
            if constexpr (C::SPARSE) {
              const uint64_t bdesc = smem_desc(b_base + (j >> 1) * C::B_ATOM + (j & 1) * 64, 16, 1024, 2);
              // 16-bit kinds: metadata column j is addressed as the even column
              // j & ~1 plus the instruction descriptor's sparse_id2 = j & 1
              // (bits 0-1); 8-bit kinds use two columns per MMA, id2 = 0
              const uint32_t ecol = C::E_PER_MMA == 1 ? (j & ~1) : 2 * j;
              const uint32_t idesc = C::E_PER_MMA == 1 ? (C::IDESC | static_cast<uint32_t>(j & 1)) : C::IDESC;
              umma_sparse_cg2<C::KIND>(d, adesc, bdesc, tmem + e_col + ecol, idesc, acc_flag);
            } else {
              const uint64_t bdesc = smem_desc(b_base + j * 32, 16, 1024, 2);
              umma_dense_cg2<C::KIND>(d, adesc, bdesc, C::IDESC, acc_flag);
            }
          }
        };
        bool sub1_ready = C::MSUB == 1;
        long long wait_cycles = 0;
        int lag = 0, lag_stage = 0, lag_kb = 0;  // deferred subtile-1 k-blocks (consecutive ring stages)
        uint32_t lag_phase = 0;
        auto wait_full1 = [&](int st, uint32_t ph) {
          if constexpr (C::SPLIT) {
            mbar_wait(&full1[st], ph);
            tc_fence_after();
          }
        };
        const uint16_t pair_epi = static_cast<uint16_t>(0x3u << lead);  // this pair's epilogues
        for (int kb = kb0; kb < kb1; ++kb) {
          if (p.trace) {
            const long long t0 = clock64();
            mbar_wait(&full[stage], phase);
            const long long t1 = clock64();
            wait_cycles += t1 - t0;
            if (blockIdx.x == 0 && it < 16 && kb < 256) p.trace[65536 + (it * 256 + kb) * 2 + 1] = t1;
          } else {
            mbar_wait(&full[stage], phase);
          }
          tc_fence_after();
          if constexpr (C::MSUB == 2) {
            if (p.tail0 == 2 && sub1_ready && kb == kb1 - 2) {
              // last two k-blocks: sub0(k-1), sub0(k) | commit sub0 | sub1(k-1), sub1(k)
              int st2 = stage + 1;
              uint32_t ph2 = phase;
              if (st2 == C::STAGES) {
                st2 = 0;
                ph2 ^= 1u;
              }
              issue(0, stage, kb);
              mbar_wait(&full[st2], ph2);
              tc_fence_after();
              issue(0, st2, kb + 1);
              tc_commit_mc(&tfull[1], pair_epi);
              wait_full1(stage, phase);
              issue(1, stage, kb);
              tc_commit_mc(&empty[stage], all_ctas);
              wait_full1(st2, ph2);
              issue(1, st2, kb + 1);
              tc_commit_mc(&empty[st2], all_ctas);
              stage = st2 + 1;
              phase = ph2;
              if (stage == C::STAGES) {
                stage = 0;
                phase ^= 1u;
              }
              ++kb;
              continue;
            }
          }
          issue(0, stage, kb);
          // subtile 0 complete for this tile: its own commit (tfull[1]) ahead of subtile 1's last MMAs
          if (C::MSUB == 2 && p.tail0 && kb == kb1 - 1) tc_commit_mc(&tfull[1], pair_epi);
          if constexpr (C::MSUB == 1) {
            tc_commit_mc(&empty[stage], all_ctas);  // every CTA of the cluster
          } else if (sub1_ready) {
            wait_full1(stage, phase);
            issue(1, stage, kb);
            tc_commit_mc(&empty[stage], all_ctas);
          } else {
            if (lag++ == 0) {
              lag_stage = stage;
              lag_kb = kb;
              lag_phase = phase;
            }
            // catch up once subtile 1 is drained; block when the ring is
            // exhausted or the tile's k-loop ends
            if (lag == C::STAGES || kb == kb1 - 1 || mbar_test(&tempty[1], acc_phase ^ 1)) {
              mbar_wait(&tempty[1], acc_phase ^ 1);
              tc_fence_after();
              SLSP_TRACE(it, 1);
              sub1_ready = true;
              int st = lag_stage;
              uint32_t ph = lag_phase;
              for (int i = 0; i < lag; ++i) {
                wait_full1(st, ph);
                issue(1, st, lag_kb + i);
                tc_commit_mc(&empty[st], all_ctas);
                if (++st == C::STAGES) {
                  st = 0;
                  ph ^= 1u;
                }
              }
              lag = 0;
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        SLSP_TRACE(it, 2);
        if (p.trace && blockIdx.x == 0) p.trace[it * 16 + 8] = wait_cycles;
        tc_commit_mc(&tfull[acc], pair_epi);
      }
    }
  } else if (C::GLIFT && warp >= 2 + C::EPI_WARPS) {
    // ------------------------------------------- in-GEMM lift warps ----
    // GLIFT_GROUPS groups of GLIFT_GW warps; group g takes every
    // GLIFT_GROUPS-th stage of the producer's sequence, so that many stages'
    // L2 reads are in flight at once. GLIFT_GROUPS <= STAGES keeps every
    // empty-barrier wait within one phase of the barrier: the group's
    // previous stage q - G needed stage q - G - STAGES consumed, so the slot's
    // occupant before q - STAGES is gone (parity waits cannot tell phases two
    // apart). Per stage: wait for the ring slot,
    // build the stage's B tile for this CTA's tokens — lifted BF16 element e
    // (window j = e/4: source elements l*(j/wc) + 2*(j%wc) + 0..3,
    // quantize.hpp:72-89 lift_row; windows past the real ones are the zero
    // padding up to kp) — as 16-byte chunks of two windows in the 128B
    // swizzle the UMMA descriptor expects, fence the generic-proxy writes to
    // the async proxy, and arrive on the leader's full barrier. Rows of
    // tokens past m are left as they are: their accumulator columns are
    // never stored.
    if constexpr (C::GLIFT) {
      const uint32_t lw = warp - 2 - C::EPI_WARPS;
      const uint32_t grp = lw / C::GLIFT_GW;
      const uint32_t gt = (lw % C::GLIFT_GW) * 32 + lane_id();  // thread within the group
      const uint32_t full_lead = mapa_shared(smem_u32(&full[0]), lead);
      constexpr int CHUNKS = C::B_ATOMS * 8;  // 16-byte chunks per token row per stage
      constexpr int ITER = C::B_ROWS * CHUNKS / (C::GLIFT_GW * 32);
      static_assert(ITER * C::GLIFT_GW * 32 == C::B_ROWS * CHUNKS, "lift group covers the B tile exactly");
      static_assert(C::GLIFT_GROUPS <= C::STAGES, "lift groups run at most one ring lap apart");
      const uint16_t* X = static_cast<const uint16_t*>(p.x);
      const bool no_ldg = p.debug & kDbgNoBuild, no_sts = p.debug & kDbgNoSts;  // perf probing
      // 6:8 path geometry: 8 lanes per token row, RPI rows per iteration
      constexpr int RPI = 4 * C::GLIFT_GW;
      constexpr int IT = C::B_ROWS / RPI;
      static_assert(IT * RPI == C::B_ROWS, "6:8 path: whole rows per iteration");
      const int tl = static_cast<int>(lane_id() & 7);  // triple lane
      const int rsub = static_cast<int>(gt >> 3);      // row within an iteration
      const int wrow0 = static_cast<int>((gt & ~31u) >> 3);  // this warp's first row within an iteration
      const int groups = static_cast<int>(p.lift_windows / 3);
      int stage = 0, cnt = 0;
      uint32_t phase = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int mt_, ns, kb0, kb1;
        tile_coords(tile, p, p.m_tiles, n_super, mt_, ns, kb0, kb1, kslice, ksc);
        const int64_t t_first = static_cast<int64_t>(ns) * C::BN + rank * C::B_ROWS;
        const int rows = static_cast<int>(imin64(C::B_ROWS, p.m - t_first));  // valid token rows (may be <= 0)
        const uint16_t* rp[IT];  // this thread's token rows (6:8 path)
#pragma unroll
        for (int i = 0; i < IT; ++i) rp[i] = X + (t_first + i * RPI + rsub) * p.x_ld;
        for (int kb = kb0; kb < kb1; ++kb) {
          if (cnt == static_cast<int>(grp)) {
          const uint32_t dst = smem_u32(sB + stage * C::B_STAGE);
          if (p.lift_l == 8) {
            // 6:8 on 16-byte aligned rows, by "triples": chunks 3t..3t+2
            // (windows 6t..6t+5) are exactly source blocks 2t and 2t+1:
            //   chunk 3t   = x[0..3]  x[2..5]   of block 2t
            //   chunk 3t+1 = x[4..7] of 2t,  x[0..3] of 2t+1
            //   chunk 3t+2 = x[2..5]  x[4..7]   of block 2t+1
            // so lane tl of a row loads two blocks (2 x LDG.128, 32
            // contiguous bytes) and stores the triple's chunks that fall in
            // this stage (16 chunks: <= 7 triples) — fixed selects, no
            // shuffles. Blocks past the row's last are zero (padding windows).
            const int c0 = kb * CHUNKS;
            const int t = c0 / 3 + tl;
            const bool act = 3 * t < c0 + CHUNKS;
            const bool va = act && 2 * t < groups && !no_ldg, vb = act && 2 * t + 1 < groups && !no_ldg;
            uint4 va4[IT], vb4[IT];
#pragma unroll
            for (int i = 0; i < IT; ++i) {
              const bool live = i * RPI + rsub < rows;
              const uint4* src = reinterpret_cast<const uint4*>(rp[i] + 16 * t);
              va4[i] = (live && va) ? __ldg(src) : make_uint4(0u, 0u, 0u, 0u);
              vb4[i] = (live && vb) ? __ldg(src + 1) : make_uint4(0u, 0u, 0u, 0u);
            }
            mbar_wait(&empty[stage], phase ^ 1);
            const int cc0 = 3 * t - c0;  // stage-local chunk of the triple's first chunk (may be < 0)
#pragma unroll
            for (int i = 0; i < IT; ++i) {
              if (i * RPI + wrow0 >= rows || no_sts) break;  // warp-uniform: no valid row left for this warp
              const int r = i * RPI + rsub;
              const uint32_t rb = dst + r * 128;
              const uint32_t sw = static_cast<uint32_t>(r & 7);
              const uint4 A = va4[i], B = vb4[i];
              if (act && cc0 >= 0)
                st_shared_v4(rb + (cc0 >> 3) * C::B_ATOM + (((cc0 & 7) ^ sw) << 4), A.x, A.y, A.y, A.z);
              if (act && cc0 + 1 >= 0 && cc0 + 1 < CHUNKS)
                st_shared_v4(rb + ((cc0 + 1) >> 3) * C::B_ATOM + ((((cc0 + 1) & 7) ^ sw) << 4), A.z, A.w, B.x, B.y);
              if (act && cc0 + 2 >= 0 && cc0 + 2 < CHUNKS)
                st_shared_v4(rb + ((cc0 + 2) >> 3) * C::B_ATOM + ((((cc0 + 2) & 7) ^ sw) << 4), B.y, B.z, B.z, B.w);
            }
          } else {
            const int lift_l = p.lift_l < 0 ? -p.lift_l : p.lift_l;  // -8: 6:8 on unaligned rows
            uint32_t w[ITER][4];
#pragma unroll
            for (int i = 0; i < ITER; ++i) {
              const int u = static_cast<int>(gt) + i * C::GLIFT_GW * 32;
              const int r = u / CHUNKS, cc = u % CHUNKS;
              const int64_t j0 = (static_cast<int64_t>(kb) * (C::B_ATOMS * 64) + cc * 8) >> 2;  // first window
              const uint16_t* xr = X + (t_first + r) * p.x_ld;
#pragma unroll
              for (int h = 0; h < 2; ++h) {  // two windows per chunk
                const int64_t j = j0 + h;
                w[i][2 * h] = 0u;
                w[i][2 * h + 1] = 0u;
                if (r < rows && j < p.lift_windows && !no_ldg) {
                  const int64_t g = j / p.lift_wc;
                  const uint32_t* src = reinterpret_cast<const uint32_t*>(xr + g * lift_l + 2 * (j - g * p.lift_wc));
                  w[i][2 * h] = __ldg(src);
                  w[i][2 * h + 1] = __ldg(src + 1);
                }
              }
            }
            mbar_wait(&empty[stage], phase ^ 1);
#pragma unroll
            for (int i = 0; i < ITER; ++i) {
              const int u = static_cast<int>(gt) + i * C::GLIFT_GW * 32;
              const int r = u / CHUNKS, cc = u % CHUNKS;
              st_shared_v4(dst + (cc >> 3) * C::B_ATOM + r * 128 + (((cc & 7) ^ (r & 7)) << 4), w[i][0], w[i][1],
                           w[i][2], w[i][3]);
            }
          }
          if (!(p.debug & kDbgNoFence)) fence_async_smem();  // generic-proxy writes -> visible to the tensor core
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_cluster(full_lead + 8u * stage);
          }
          if (++cnt == C::GLIFT_GROUPS) cnt = 0;
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (C::LIFT && warp >= 2 + C::EPI_WARPS) {
    // ------------------------------------------------ lift warps ----
    // Follow the producer's stage sequence. X block (j = kb % 3 < 2): relay
    // "X present" to the MMA issuer (leader's full barrier), then build C atom
    // j of the period's C block from it: for each token row and 4-block chunk
    // q, window 1 of blocks 4q..4q+3 = bytes 2-5 of each 8-byte block, read as
    // two 16-byte X chunks, written as one 16-byte C chunk, both in the 128B
    // swizzle the UMMA descriptor expects (chunk index ^= row & 7). C block:
    // relay "C built" (after both atoms). Each warp owns B_ROWS / LIFT_WARPS
    // rows; a quarter-warp touches 8 consecutive rows of one chunk column, so
    // every 16-byte access is bank-conflict free.
    if constexpr (C::LIFT) {
      const uint32_t lw = warp - 2 - C::EPI_WARPS;
      const uint32_t lane = lane_id();
      const uint32_t full_lead = mapa_shared(smem_u32(&full[0]), lead);
      constexpr int ROWS = C::B_ROWS / C::LIFT_WARPS;
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        for (int kb = 0; kb < p.num_kb; ++kb) {
          const int j = kb % 3;
          if (j < 2) {
            mbar_wait(&xfull[stage], phase);
            __syncwarp();
            // (plain arrive: the relay publishes no data of its own; a
            // .release.cluster arrive costs a MEMBAR.GPU per stage)
            if (lane == 0) mbar_arrive_cluster(full_lead + 8u * stage);  // this CTA's X tile present
            int cs = stage + 2 - j;  // ring slot of this period's C block
            uint32_t cph = phase;
            if (cs >= C::STAGES) {
              cs -= C::STAGES;
              cph ^= 1u;
            }
            if (j == 0) mbar_wait(&empty[cs], cph ^ 1u);  // C slot's previous occupant consumed
            const uint32_t src = smem_u32(sB + stage * C::B_STAGE);
            const uint32_t dst = smem_u32(sB + cs * C::B_STAGE + j * C::B_ATOM);
#pragma unroll
            for (int i = 0; i < ROWS / 8 * 2; ++i) {
              if (p.debug & kDbgNoBuild) break;
              const uint32_t r = lw * ROWS + (i >> 1) * 8 + (lane & 7);
              const uint32_t q = (i & 1) * 4 + (lane >> 3);  // C chunk: blocks 4q..4q+3 of the X tile
              const uint32_t sw = r & 7;
              const uint32_t xa = src + (q >> 2) * C::B_ATOM + r * 128;  // X chunks 2q, 2q+1 live in atom q / 4
              const uint4 x0 = ld_shared_u4(xa + (((2 * q) & 7) ^ sw) * 16);
              const uint4 x1 = ld_shared_u4(xa + (((2 * q + 1) & 7) ^ sw) * 16);
              st_shared_v4(dst + r * 128 + ((q ^ sw) << 4), __byte_perm(x0.x, x0.y, 0x5432),
                           __byte_perm(x0.z, x0.w, 0x5432), __byte_perm(x1.x, x1.y, 0x5432),
                           __byte_perm(x1.z, x1.w, 0x5432));
            }
            if (!(p.debug & kDbgNoFence)) fence_async_smem();  // generic-proxy writes -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);  // done reading this X tile
          } else {
            mbar_wait(&xfull[stage], phase);  // keeps this slot's xfull phase in step (no bytes for C blocks)
            __syncwarp();
            if (lane == 0) {
              // the C writes were fenced to the async proxy after each atom
              mbar_arrive_cluster(full_lead + 8u * stage);  // C block built (both atoms)
              mbar_arrive(&empty[stage]);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if constexpr (C::REG_EPI) {
    // ------------------------------------ register-staged epilogue ----
    // 8 warps: two per TMEM lane quarter; the first owns columns [0, H0) of
    // the tile, the second [H0, BN) (H0 = BN/2 rounded up to a 32-column
    // box). Per subtile: tcgen05.ld (software-pipelined, 16 columns at a time)
    // -> dequant -> BF16 pairs in registers -> release the subtile's TMEM to
    // the MMA warp. Both subtiles are drained before any store, so the MMA
    // waits only for the TMEM reads. Stores: 32-row x 32-column TMA boxes
    // through a warp-private 2 KB staging buffer (64-byte swizzled rows) —
    // per-lane 32-byte global stores cost measurably more L2 throughput.
    // Scales are fetched before the accumulator wait: s_ch into registers,
    // the warp's s_tok slice into a warp-private smem slice (LDS.128 broadcast).
    const uint32_t quarter = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t lane = lane_id();
    const uint64_t pol = (p.hints & kHintOutFirst) ? policy_evict_first() : policy_evict_normal();
    float* stok_sm = reinterpret_cast<float*>(smem + C::OFF_EPI + (warp - 2) * C::EPI_WARP);
    uint8_t* stage = smem + C::OFF_EPI + (warp - 2) * C::EPI_WARP + C::H0 * 4;
    constexpr int NCH = C::H0 / 16;
    const int ncols = half ? C::BN - C::H0 : C::H0;  // warp-uniform
    const int nch = ncols / 16;
    int it = 0;
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
      int mt, ns, kb0_, kb1_;
      tile_coords(tile, p, p.m_tiles, n_super, mt, ns, kb0_, kb1_, kslice, ksc);
      const int nt = ns * C::NPAIR + static_cast<int>(npair_idx);  // >= n_tiles: idle pair, tcol0 >= m stores nothing
      const int64_t tcol0 = static_cast<int64_t>(nt) * C::BN + half * C::H0;
      const int64_t rowq = static_cast<int64_t>(mt) * C::BM + rank * C::A_ROWS + quarter * 32;  // lane 0's row
      const int64_t row0 = rowq + lane;
      const float sc0 = row0 < p.n ? __ldg(p.s_ch + row0) : 0.f;
      const float sc1 = row0 + 256 < p.n ? __ldg(p.s_ch + row0 + 256) : 0.f;
      for (int i = static_cast<int>(lane); i < ncols; i += 32)
        stok_sm[i] = tcol0 + i < p.m ? __ldg(p.s_tok + tcol0 + i) : 0.f;
      __syncwarp();
      // subtile 0 is committed on its own barrier (tfull[1]) when p.tail0
      mbar_wait(&tfull[p.tail0 ? 1 : 0], it & 1);
      tc_fence_after();
      if (warp == 2 && lane == 0) SLSP_TRACE(it, 3);

      auto drain = [&](int h, float sc, uint32_t (&pk)[NCH][8]) __attribute__((always_inline)) {
        const uint32_t t_base = tmem + ((quarter * 32) << 16) + h * C::ACC_COLS + half * C::H0;
        uint32_t r[2][16];
        tmem_ld_32x32b_x16(t_base, r[0]);
        tmem_ld_wait_regs(r[0]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c < nch) {
            if (c + 1 < nch) tmem_ld_32x32b_x16(t_base + (c + 1) * 16, r[(c + 1) & 1]);
            dequant16_smem<typename C::Acc>(r[c & 1], sc, smem_u32(stok_sm) + c * 64, pk[c]);
            reg_pin(pk[c]);  // keep the math before the TMEM release (no sinking into the stores)
            if (c + 1 < nch) tmem_ld_wait_regs(r[(c + 1) & 1]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[h]), lead));
        if (warp == 2 && lane == 0) SLSP_TRACE(it, 4 + 2 * h);
      };
      auto store = [&](int h, const uint32_t (&pk)[NCH][8]) __attribute__((always_inline)) {
        const int64_t rq = rowq + h * 256;
        if (rq >= p.n) return;  // warp-uniform
        if (p.debug & kDbgNoStore) return;
        if (p.tma_store) {
          const uint32_t sb = smem_u32(stage);
#pragma unroll
          for (int b = 0; b < NCH / 2; ++b) {
            const int64_t t0 = tcol0 + 32 * b;
            if (2 * b >= nch || t0 >= p.m) break;  // warp-uniform
            if (p.pace_ns && (h || b)) __nanosleep(p.pace_ns);
            if (lane == 0) bulk_wait_read<0>();  // staging buffer read by the previous box's store
            __syncwarp();
            // [32 rows][64 B] staging in the map's 64-byte swizzle (16-byte chunk ^= (row >> 1) & 3)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t(&w)[8] = pk[2 * b + (j >> 1)];
              const int o = 4 * (j & 1);
              st_shared_v4(sb + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), w[o], w[o + 1], w[o + 2], w[o + 3]);
            }
            if constexpr (C::OUT == SLSP_OUT_BF16_MN) {
              // transpose the [32 features][32 tokens] box in place into the
              // [M][N] map's [32 tokens][32 features] box (64-byte rows, 64B
              // swizzle): ldmatrix reads 8x8 blocks with features as rows,
              // stmatrix.trans writes them back with tokens as rows
              __syncwarp();
              uint32_t q[4][4];
#pragma unroll
              for (int tb = 0; tb < 4; ++tb)  // token block: 8 tokens = one 16-byte chunk of a feature row
                ldmatrix_x4(sb + lane * 64 + ((tb ^ ((lane >> 1) & 3)) << 4), q[tb]);
              __syncwarp();
#pragma unroll
              for (int tb = 0; tb < 4; ++tb) {
                const uint32_t tr = tb * 8 + (lane & 7);  // token row written by this lane, feature chunk lane / 8
                stmatrix_x4_trans(sb + tr * 64 + (((lane >> 3) ^ ((tr >> 1) & 3)) << 4), q[tb][0], q[tb][1], q[tb][2],
                                  q[tb][3]);
              }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              if constexpr (C::OUT == SLSP_OUT_BF16_MN)
                tma_store_2d_hint(&tmOut, stage, static_cast<int>(rq), static_cast<int>(t0), pol);
              else
                tma_store_2d_hint(&tmOut, stage, static_cast<int>(t0), static_cast<int>(rq), pol);
              bulk_commit();
            }
          }
          return;
        }
        const int64_t row = row0 + h * 256;
        if (row >= p.n) return;
        if constexpr (C::OUT == SLSP_OUT_BF16_MN) {  // direct 2-byte stores, coalesced across the lanes' features
          uint16_t* out16 = reinterpret_cast<uint16_t*>(p.out);
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            if (c < nch)
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int64_t t = tcol0 + 16 * c + i;
                if (t < p.m) out16[t * p.ldo + row] = static_cast<uint16_t>(pk[c][i >> 1] >> (16 * (i & 1)));
              }
          return;
        }
        uint8_t* dst_row = reinterpret_cast<uint8_t*>(p.out) + (row * p.ldo + tcol0) * 2;
        if (p.direct_vec == 2 && tcol0 + ncols <= p.m) {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            if (c < nch) st_global_v8_hint(dst_row + c * 32, pk[c], pol);
        } else {  // token tail or unaligned rows: element stores from a local copy (cold path)
          uint32_t tmp[NCH * 8];
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 8; ++i) tmp[c * 8 + i] = pk[c][i];
          store_tail_u16(reinterpret_cast<uint16_t*>(dst_row), tmp, static_cast<int>(imin64(ncols, p.m - tcol0)));
        }
      };
      uint32_t pk0[NCH][8], pk1[NCH][8];
      drain(0, sc0, pk0);
      if (p.tail0) {
        mbar_wait(&tfull[0], it & 1);
        tc_fence_after();
      }
      drain(1, sc1, pk1);
      if (C::AMAX && p.amax) {  // §8f #3: both subtiles' rows, then across lanes and warps
        const uint32_t sm = C::AMAX_SM ? smem_u32(smem + C::OFF_AMAX) + (it & 1) * C::BN * 4 : 0u;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c < nch) {
            uint32_t mx[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) mx[i] = __vmaxu2(pk0[c][i] & 0x7FFF7FFFu, pk1[c][i] & 0x7FFF7FFFu);
            fold_token_amax<8>(p, mx, tcol0 + 16 * c, sm, static_cast<int>(half) * C::H0 + 16 * c);
          }
        }
        if constexpr (C::AMAX_SM)
          fold_flush<C::BN, C::EPI_WARPS * 32>(p, reinterpret_cast<uint32_t*>(smem + C::OFF_AMAX) + (it & 1) * C::BN,
                                               static_cast<int64_t>(nt) * C::BN, warp == 2);
      }
      store(0, pk0);
      if (warp == 2 && lane == 0) SLSP_TRACE(it, 5);
      store(1, pk1);
      if (warp == 2 && lane == 0) SLSP_TRACE(it, 7);
    }
    if (lane == 0) bulk_wait<0>();
  } else {
    // ------------------------------------------------ epilogue ----
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t sub = (warp - 2) >> 2;  // MSUB=2: which alternate chunks of a subtile this warp drains
    const uint32_t lane = lane_id();
    uint8_t* stage_base = smem + C::OFF_EPI + (warp - 2) * C::EPI_WARP;
    int buf = 0;
    int it = 0;
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
      int mt, ns, kb0_, kb1_;
      tile_coords(tile, p, p.m_tiles, n_super, mt, ns, kb0_, kb1_, kslice, ksc);
      const int nt = ns * C::NPAIR + static_cast<int>(npair_idx);  // >= n_tiles: idle pair, t0 >= m stores nothing
      const int acc = C::ACC_STAGES == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = C::ACC_STAGES == 2 ? ((it >> 1) & 1) : (it & 1);
      // MSUB=2: all 8 warps drain subtile 0 (two warps per lane quarter,
      // alternating chunks), release it, then subtile 1; with p.tail0
      // subtile 0 has its own barrier (tfull[1]), tfull[0] covers both
      // cluster split-K: every CTA of the cluster has read this CTA's
      // previous partials before they are overwritten
      if (C::KSC_OK && ksc > 1 && it > 0) mbar_wait_cluster_acquire(red_empty, (it - 1) & 1);
#pragma unroll 1
      for (int h = 0; h < C::MSUB; ++h) {
        if (C::MSUB == 2 && p.tail0) {
          mbar_wait(&tfull[h == 0 ? 1 : 0], acc_phase);
          tc_fence_after();
        } else if (h == 0) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
        }
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
          if (C::KSC_OK && ksc > 1) {
            // cluster split-K: park this slice's raw partials (row = lane) in
            // the warp's staging area, 16-byte chunk j of the row at j ^ (lane & 15)
            const uint32_t rowp = smem_u32(stage_base) + lane * (C::BN * 4);
#pragma unroll
            for (int i = 0; i < C::EPI_COLS; i += 4) {
              const uint32_t j = static_cast<uint32_t>(c * C::EPI_COLS + i) >> 2;
              st_shared_v4(rowp + ((j ^ (lane & 15u)) << 4), r[i], r[i + 1], r[i + 2], r[i + 3]);
            }
            continue;
          }
          if (p.ksplit > 1) {  // split-K: this slice's raw partial sums -> ws[slice][row][t]
            const int64_t row = row0 + lane;
            if (row < p.n && !(p.debug & kDbgNoStore)) {
              uint32_t* dst = static_cast<uint32_t*>(p.ws) + (static_cast<int64_t>(tile % p.ksplit) * p.n + row) * p.m + t0;
              const int64_t valid = imin64(C::EPI_COLS, p.m - t0);
              if (valid == C::EPI_COLS && (p.m & 3) == 0) {
#pragma unroll
                for (int i = 0; i < C::EPI_COLS; i += 4)
                  *reinterpret_cast<uint4*>(dst + i) = make_uint4(r[i], r[i + 1], r[i + 2], r[i + 3]);
              } else {
#pragma unroll
                for (int i = 0; i < C::EPI_COLS; ++i)
                  if (i < valid) dst[i] = r[i];
              }
            }
            continue;
          }
          if (p.tma_store) {
            if (lane == 0) bulk_wait_read<C::EPI_BUFS - 1>();  // staging buffer free again
            __syncwarp();
          }
          epilogue_chunk<C>(p, &tmOut, stage_base + buf * C::EPI_BUF, r, row0, t0, sc,
                            C::AMAX_SM ? smem_u32(smem + C::OFF_AMAX) + (it & 1) * C::BN * 4 : 0u,
                            c * C::EPI_COLS);
          if (C::EPI_BUFS == 2) buf ^= 1;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[C::MSUB == 2 ? h : acc]), lead));
      }
      if constexpr (C::KSC_OK) {
        if (ksc > 1) {
          // publish the partials to the same-rank CTA of every pair, wait for theirs
          fence_acq_rel_cluster();
          __syncwarp();
          // (the cluster-scope fence above is the release; plain remote
          // arrives — .release.cluster would fence again per arrive)
          if (lane == 0)
            for (int q = 0; q < ksc; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(red_full), 2 * q + rank));
          mbar_wait_cluster_acquire(red_full, it & 1);
          // this CTA's share: rows [lo, hi) of its 128 (lane quarter w/32 lives
          // in epilogue warp (w/32 + 2) & 3's staging area), 16-byte chunks
          // (4 tokens) as units: [N][M] outputs take chunks fastest (a warp
          // stores whole rows, coalesced), [M][N] rows fastest. Each thread
          // keeps 4 units' DSMEM loads of a slice in flight, sums in slice
          // order (the finishing kernel's arithmetic), applies the epilogue.
          static_assert(C::BN == 64 && C::EPI_WARPS == 4, "cluster split-K: 64-token tiles, 128 epilogue threads");
          constexpr bool kRowsFast = C::OUT == SLSP_OUT_BF16_MN;
          const int lo = 128 * static_cast<int>(kslice) / ksc, hi = 128 * (static_cast<int>(kslice) + 1) / ksc;
          const int tid = static_cast<int>((warp - 2) * 32 + lane);
          const int64_t tt0 = static_cast<int64_t>(nt) * C::BN;
          const int tcols = static_cast<int>(imin64(C::BN, p.m - tt0));  // valid tokens of the tile
          const int64_t row_base = static_cast<int64_t>(mt) * C::BM + rank * C::A_ROWS;
          const uint32_t epi0 = smem_u32(smem + C::OFF_EPI);
          constexpr int ESZ = C::OUT == SLSP_OUT_RAW_NM ? 4 : 2;
          const bool vec = (reinterpret_cast<uintptr_t>(p.out) % 16 == 0) && ((p.ldo * ESZ) % 16 == 0);
#pragma unroll 1
          for (int u0 = 0; u0 < 1024; u0 += 4 * 128) {  // 64 rows x 16 chunks, 4 units per thread per batch
            uint32_t acc[4][4];
            int rr[4], jj[4];
            bool ok[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int u = u0 + b * 128 + tid;
              const int ro = kRowsFast ? (u & 63) : (u >> 4);
              jj[b] = kRowsFast ? (u >> 6) : (u & 15);
              rr[b] = lo + ro;
              ok[b] = rr[b] < hi && 4 * jj[b] < tcols && row_base + rr[b] < p.n;
            }
            for (int q = 0; q < ksc; ++q) {
              uint4 x[4];
#pragma unroll
              for (int b = 0; b < 4; ++b)
                if (ok[b])
                  x[b] = ld_shared_cluster_v4(mapa_shared(
                      epi0 + ((((rr[b] >> 5) + 2) & 3) * C::EPI_WARP) + (rr[b] & 31) * (C::BN * 4) +
                          ((static_cast<uint32_t>(jj[b]) ^ (static_cast<uint32_t>(rr[b]) & 15u)) << 4),
                      2 * q + rank));
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                if (!ok[b]) continue;
                const uint32_t y[4] = {x[b].x, x[b].y, x[b].z, x[b].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  if (q == 0)
                    acc[b][e] = y[e];
                  else if constexpr (std::is_same<typename C::Acc, int32_t>::value)
                    acc[b][e] = static_cast<uint32_t>(static_cast<int32_t>(acc[b][e]) + static_cast<int32_t>(y[e]));
                  else
                    acc[b][e] = __float_as_uint(__fadd_rn(__uint_as_float(acc[b][e]), __uint_as_float(y[e])));
                }
              }
            }
            if (p.debug & kDbgNoStore) continue;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (!ok[b]) continue;
              const int64_t row = row_base + rr[b];
              const int64_t t = tt0 + 4 * jj[b];
              const int ne = tcols - 4 * jj[b];  // >= 1
              if constexpr (C::OUT == SLSP_OUT_RAW_NM) {
                uint32_t* dst = static_cast<uint32_t*>(p.out) + row * p.ldo + t;
                if (ne >= 4 && vec) {
                  *reinterpret_cast<uint4*>(dst) = make_uint4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
                } else {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    if (e < ne) dst[e] = acc[b][e];
                }
              } else {
                const float sc = __ldg(p.s_ch + row);
                uint16_t h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const __nv_bfloat16 v = __float2bfloat16_rn(
                      dequant<typename C::Acc>(acc[b][e], sc, e < ne ? __ldg(p.s_tok + t + e) : 0.f));
                  h[e] = *reinterpret_cast<const uint16_t*>(&v);
                }
                uint16_t* o = static_cast<uint16_t*>(p.out);
                if (C::OUT == SLSP_OUT_BF16_NM && ne >= 4 && vec) {
                  *reinterpret_cast<uint2*>(o + row * p.ldo + t) =
                      make_uint2(h[0] | (static_cast<uint32_t>(h[1]) << 16), h[2] | (static_cast<uint32_t>(h[3]) << 16));
                } else {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    if (e < ne) o[C::OUT == SLSP_OUT_BF16_MN ? (t + e) * p.ldo + row : row * p.ldo + t + e] = h[e];
                }
              }
            }
          }
          // reads done: release every peer's buffer for its next tile
          fence_acq_rel_cluster();
          __syncwarp();
          if (lane == 0)
            for (int q = 0; q < ksc; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(red_empty), 2 * q + rank));
        }
      }
      if constexpr (C::AMAX_SM)
        if (C::AMAX && p.amax)
          fold_flush<C::BN, C::EPI_WARPS * 32>(p, reinterpret_cast<uint32_t*>(smem + C::OFF_AMAX) + (it & 1) * C::BN,
                                               static_cast<int64_t>(nt) * C::BN, warp == 2);
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

uint32_t debug_flags() { return static_cast<uint32_t>(slsp_host::knob("SLSP_GEMM_DEBUG", 0)); }

// Tuning knob (SLSP_* environment snapshot, slsp_reload_knobs re-reads it).
uint32_t env_knob(const char* name, uint32_t dflt) { return static_cast<uint32_t>(slsp_host::knob(name, dflt)); }

uintptr_t env_ptr(const char* name) { return static_cast<uintptr_t>(slsp_host::knob(name, 0)); }

// Byte-addressed 2D map (uint8 elements): rows x row_bytes, box rows x box_bytes
// (128 B: 128B swizzle, 64 B: 64B swizzle).
int make_map_2d(CUtensorMap* map, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_rows,
                uint32_t box_bytes = 128) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SLSP_ERR_CUDA;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SLSP_OK : SLSP_ERR_CUDA;
}

// Metadata map over the slsp_tile_meta layout: a flat byte stream viewed as
// 256-byte rows; one box {256, 16} is the contiguous 4 KB block of a stage
// (two canonical 128x16B tcgen05.cp atoms) — 16 wide requests instead of 256
// 16-byte ones.
int make_map_meta(CUtensorMap* map, const void* base, uint64_t rows, uint64_t kp, uint32_t box_rows = 16) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SLSP_ERR_CUDA;
  const uint64_t bytes = static_cast<uint64_t>(slsp_tiled_meta_bytes(static_cast<int64_t>(rows), static_cast<int64_t>(kp)));
  cuuint64_t dims[2] = {256, bytes / 256};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {256, box_rows};  // 16: a 256-wide k-stage, 8: a half stage
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
void select_epilogue(Params& p, int out_mode, uint32_t msub, const void* out, int64_t ldo, const float* s_tok) {
  const uint32_t epi = env_knob("SLSP_GEMM_EPI", 0);
  const int esz = out_mode == SLSP_OUT_RAW_NM ? 4 : 2;
  const uintptr_t base = reinterpret_cast<uintptr_t>(out);
  const int64_t row_bytes = ldo * esz;
  p.direct_vec = (base % 32 == 0 && row_bytes % 32 == 0) ? 2 : (base % 16 == 0 && row_bytes % 16 == 0) ? 1 : 0;
  p.stok_vec = (reinterpret_cast<uintptr_t>(s_tok) % 16) == 0;
  // TMA staging where rows are 16-byte aligned (make_map_out enables it),
  // direct vector stores when SLSP_GEMM_EPI=2 (perf probing)
  (void)msub;
  if (out_mode != SLSP_OUT_BF16_MN && p.tma_store && epi == 2) p.tma_store = 0;
}

using slsp_host::num_sms;

// Split-K factor for decode-shaped M: the S minimising the estimated time
// (S = 1 unless a split strictly helps), at most `cap` (workspace slices) and
// at least 2 k-blocks per slice. Env SLSP_GEMM_KSPLIT forces it (within the
// same bounds).
// split-K applies up to this many tokens (where the tiles can leave SMs
// idle: decode and moderate prefill chunks); above 256 tokens the workspace
// is capped at kSplitWsCap bytes (8 slices below that).
constexpr int64_t kSplitMaxM = 1024;
constexpr int64_t kSplitWsCap = int64_t{64} << 20;

int choose_ksplit(int tiles, int num_kb, int clusters, int cap, int64_t slice_bytes) {
  const int hi = cap < num_kb / 2 ? cap : num_kb / 2;
  const int forced = static_cast<int>(env_knob("SLSP_GEMM_KSPLIT", 0));
  if (forced > 0) return forced < hi ? forced : (hi > 1 ? hi : 1);
  // cost in k-block (ring stage) times (~0.27 us each): waves x k-blocks per
  // slice, plus the measured price of splitting — a fixed ~kSplitCostKb
  // k-blocks (finish kernel, more tile prologues) and the slices' write +
  // read traffic at ~5 TB/s, ~kSliceBytesPerKb bytes per k-block time.
  // Measured on the Qwen2.5-7B shapes: the K = 3584 layers
  // (21 INT8 / 42 BF16 k-blocks) lose with any split at M <= 256, K = 18944
  // (111 / 222) gains 1.3-1.6x at M <= 256, ~1.1x at M = 512, and loses at
  // M = 768 (a 3-way split there cost 1.5x).
  const int kSplitCostKb = static_cast<int>(env_knob("SLSP_GEMM_SPLITCOST", 16));
  constexpr double kSliceBytesPerKb = 1.35e6;
  int best = 1;
  double best_cost = static_cast<double>((tiles + clusters - 1) / clusters) * num_kb;
  for (int sp = 2; sp <= hi; ++sp) {
    const double cost = static_cast<double>((tiles * sp + clusters - 1) / clusters) * ((num_kb + sp - 1) / sp) +
                        kSplitCostKb + 2.0 * sp * static_cast<double>(slice_bytes) / kSliceBytesPerKb;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

// Cluster split-K for the decode tiles (Params::ksc): ksc pairs per cluster
// share one tile's k-range and reduce through distributed shared memory.
constexpr int kMaxKsc = 4;  // clusters of <= 8 CTAs (portable size)
constexpr int kKscDefault = 0;

// Decode tiles: one model over {unsplit, workspace split sp, cluster split
// k}, in k-block times per CTA pair: waves x k-blocks per slice + a fixed
// price (4 for either split: the finishing kernel is PDL-launched beside the
// GEMM and starts the moment the slices land) + for the workspace split its
// slices' write + read traffic, weighted 3x the moderate-M model's (fitted to
// the Llama-3.1-8B decode shapes and config 1: o / down keep
// the 4-way workspace split at M = 1 and take the cluster split at M = 64,
// qkv likewise, config 1 the cluster split, gate_up 7-way / unsplit).
void choose_decode_split(int tiles, int num_kb, int clusters, int ws_cap, int64_t slice_bytes, const int* avail,
                         int& ksplit, int& ksc) {
  auto waves = [](int t, int c) { return c > 0 ? (t + c - 1) / c : 1 << 30; };
  constexpr double kPrice = 4.0, kSliceBytesPerKb = 1.35e6 / 3.0;
  double best = static_cast<double>(waves(tiles, clusters)) * num_kb;
  ksplit = 1;
  ksc = 1;
  const int hi = ws_cap < num_kb / 2 ? ws_cap : num_kb / 2;
  for (int sp = 2; sp <= hi; ++sp) {
    const double c = static_cast<double>(waves(tiles * sp, clusters)) * ((num_kb + sp - 1) / sp) + kPrice +
                     2.0 * sp * static_cast<double>(slice_bytes) / kSliceBytesPerKb;
    if (c < best - 1e-9) {
      best = c;
      ksplit = sp;
    }
  }
  for (int k = 2; k <= kMaxKsc; ++k) {
    if (avail[k] <= 0 || num_kb < 2 * k) continue;
    const double c = static_cast<double>(waves(tiles, avail[k])) * ((num_kb + k - 1) / k) + kPrice;
    if (c < best - 1e-9) {
      best = c;
      ksplit = 1;
      ksc = k;
    }
  }
}

// After a split-K GEMM: sum the slices in slice order (exact for int32,
// deterministic for fp32), then the epilogue's exact arithmetic — a18 for
// BF16 outputs (bf16((acc * s_ch[n]) * s_tok[t])), the raw sum for RAW_NM.
template <typename Acc, int OUT>
__global__ void splitk_finish_kernel(const Acc* __restrict__ ws, int slices, int64_t n, int64_t m,
                                     const float* __restrict__ s_ch, const float* __restrict__ s_tok, void* out,
                                     int64_t ldo) {
  // PDL: the blocks are resident beside the GEMM's CTAs (no shared memory)
  // and start the moment its slices are complete and visible
  pdl_wait();
  pdl_trigger();
  const int64_t total = n * m;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Acc acc = ws[i];
    for (int sl = 1; sl < slices; ++sl) acc += ws[sl * total + i];
    const int64_t row = i / m, t = i - row * m;
    if constexpr (OUT == SLSP_OUT_RAW_NM) {
      static_cast<Acc*>(out)[row * ldo + t] = acc;
    } else {
      uint32_t raw;
      if constexpr (std::is_same<Acc, int32_t>::value) raw = static_cast<uint32_t>(acc);
      else raw = __float_as_uint(acc);
      const __nv_bfloat16 b = __float2bfloat16_rn(dequant<Acc>(raw, s_ch[row], s_tok[t]));
      static_cast<uint16_t*>(out)[OUT == SLSP_OUT_BF16_MN ? t * ldo + row : row * ldo + t] =
          *reinterpret_cast<const uint16_t*>(&b);
    }
  }
}

template <typename C>
int run(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o, Params p,
        cudaStream_t s, slsp_gemm_config* query) {
  // co-resident clusters of this shape (GPC packing) and the >48 KB smem
  // opt-in: properties of the device, computed once per device
  static slsp_host::PerDevice<int> max_clusters_cache;
  auto kern = gemm_kernel<C>;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = slsp_host::pdl_enabled(p.m) ? 1 : 0;
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int max_clusters = 0;
  int st = max_clusters_cache.get(&max_clusters, [&](int& v) -> int {
    SLSP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    cfg.gridDim = dim3(C::CL * (num_sms() / C::CL));
    int n = 0;
    SLSP_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    v = n > 0 ? n : num_sms() / C::CL;
    return SLSP_OK;
  });
  if (st) return st;
  p.m_tiles = static_cast<int>((p.n + C::BM - 1) / C::BM);
  p.n_tiles = static_cast<int>((p.m + C::BN - 1) / C::BN);
  int tiles = p.m_tiles * ((p.n_tiles + C::NPAIR - 1) / C::NPAIR);
  int clusters = max_clusters;
  const int cluster_cap = static_cast<int>(env_knob("SLSP_GEMM_CLUSTERS", 0));  // perf probing
  if (cluster_cap > 0 && clusters > cluster_cap) clusters = cluster_cap;
  // split-K where the tiles do not fill the machine (decode-shaped M): needs
  // an accumulation target (the int32/fp32 output itself, or a workspace)
  p.ksplit = 1;
  p.ksc = 1;
  const int64_t slice = p.n * p.m * 4;
  if constexpr (!C::REG_EPI && !C::LIFT) {
    const int cap = p.ws && slice > 0 ? static_cast<int>(p.ws_cap / slice < 16 ? p.ws_cap / slice : 16) : 1;
    if (tiles > 0 && p.m <= kSplitMaxM && cap > 1) p.ksplit = choose_ksplit(tiles, p.num_kb, clusters, cap, slice);
  }
  // cluster split-K (decode tiles): preferred over a workspace split when its
  // estimated cost is lower; SLSP_GEMM_KSPLIT (forced workspace split) turns it off
  int ksc_clusters = clusters;
  if constexpr (C::KSC_OK) {
    static slsp_host::PerDevice<int> ksc_cache[kMaxKsc + 1];
    const int forced_ws = static_cast<int>(env_knob("SLSP_GEMM_KSPLIT", 0));
    const int forced = static_cast<int>(env_knob("SLSP_GEMM_KSC", kKscDefault));
    if (tiles > 0 && forced_ws == 0 && forced != 1) {
      int avail[kMaxKsc + 1] = {0, clusters};
      for (int k = 2; k <= kMaxKsc; ++k) {
        int v = 0;
        int st2 = ksc_cache[k].get(&v, [&](int& out) -> int {
          cudaLaunchConfig_t c2 = cfg;
          cudaLaunchAttribute a2[2] = {attr[0], attr[1]};
          a2[0].val.clusterDim.x = C::CL * k;
          c2.attrs = a2;
          c2.gridDim = dim3(C::CL * k * (num_sms() / (C::CL * k)));
          int nc = 0;
          if (cudaOccupancyMaxActiveClusters(&nc, kern, &c2) != cudaSuccess) {
            (void)cudaGetLastError();
            nc = 0;
          }
          out = nc;
          return SLSP_OK;
        });
        if (st2) return st2;
        avail[k] = cluster_cap > 0 && v > cluster_cap ? cluster_cap : v;
      }
      if (forced > 1) {  // forced cluster split (when it fits)
        const int k = forced < kMaxKsc ? forced : kMaxKsc;
        if (avail[k] > 0 && p.num_kb >= 2 * k) {
          p.ksc = k;
          p.ksplit = 1;
        }
      } else {
        const int cap = p.ws && slice > 0 ? static_cast<int>(p.ws_cap / slice < 16 ? p.ws_cap / slice : 16) : 1;
        choose_decode_split(tiles, p.num_kb, clusters, cap, slice, avail, p.ksplit, p.ksc);
      }
      if (p.ksc > 1) ksc_clusters = avail[p.ksc];
    }
  }
  if (query) {
    query->tokens_per_tile = C::BN;
    query->weight_rows_per_tile = C::BM;
    query->subtiles = C::MSUB;
    query->half_k_stages = C::KH ? 1 : 0;
    query->stages = C::STAGES;
    query->cluster_ctas = C::CL * p.ksc;
    query->ksplit = p.ksplit * p.ksc;
    query->cluster_ksplit = p.ksc;
    query->epilogue = C::REG_EPI ? 1 : 0;
    query->clusters = p.ksc > 1 ? (ksc_clusters < tiles ? ksc_clusters : tiles)
                                : (clusters < tiles * p.ksplit ? clusters : tiles * p.ksplit);
    query->workspace_bytes = p.ksplit > 1 ? p.ksplit * slice : 0;
    return SLSP_OK;
  }
  if (tiles == 0) return SLSP_OK;
  if (p.ksplit > 1) tiles *= p.ksplit;
  if (p.ksc > 1) {
    clusters = ksc_clusters;
    attr[0].val.clusterDim.x = C::CL * p.ksc;
  }
  if (clusters > tiles) clusters = tiles;
  cfg.gridDim = dim3(C::CL * p.ksc * clusters);
  SLSP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, b, e, o, p));
  if (p.ksplit > 1) {
    const int64_t total = p.n * p.m;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    const int st2 = slsp_host::launch_pdl(p.m, splitk_finish_kernel<typename C::Acc, C::OUT>, dim3(grid), dim3(256), 0,
                                          s, static_cast<const typename C::Acc*>(p.ws), p.ksplit, p.n, p.m, p.s_ch,
                                          p.s_tok, p.out, p.ldo);
    if (st2) return st2;
  }
  return SLSP_OK;
}

// The amax-folding instantiations (slsp_sparse_gemm_amax): BF16 outputs, no
// half k-stages, no weight multicast, no in-SM lifting.
template <MmaKind K, int BN>
int run_amax(int out_mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o,
             const Params& p, cudaStream_t s, uint32_t msub, slsp_gemm_config* q) {
  constexpr bool two_sub = BN >= 128 && BN <= 224;
  if (out_mode == SLSP_OUT_BF16_NM) {
    if constexpr (two_sub)
      if (msub == 2) return run<Cfg<true, K, BN, 0, SLSP_OUT_BF16_NM, 2, 0, 0, 1, 1>>(a, b, e, o, p, s, q);
    return run<Cfg<true, K, BN, 0, SLSP_OUT_BF16_NM, 1, 0, 0, 1, 1>>(a, b, e, o, p, s, q);
  }
  if (out_mode == SLSP_OUT_BF16_MN) {
    if constexpr (two_sub)
      if (msub == 2) return run<Cfg<true, K, BN, 0, SLSP_OUT_BF16_MN, 2, 0, 0, 1, 1>>(a, b, e, o, p, s, q);
    return run<Cfg<true, K, BN, 0, SLSP_OUT_BF16_MN, 1, 0, 0, 1, 1>>(a, b, e, o, p, s, q);
  }
  return SLSP_ERR_INVALID;
}

template <bool SPARSE, MmaKind K, int BN, int MSUB, int LIFT, int KH, int NPAIR = 1>
int run_out_cl(int out_mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o,
               const Params& p, cudaStream_t s, slsp_gemm_config* q) {
  switch (out_mode) {  // STAGES = 0: as many as fit
    case SLSP_OUT_RAW_NM:
      return run<Cfg<SPARSE, K, BN, 0, SLSP_OUT_RAW_NM, MSUB, LIFT, KH, NPAIR>>(a, b, e, o, p, s, q);
    case SLSP_OUT_BF16_NM:
      return run<Cfg<SPARSE, K, BN, 0, SLSP_OUT_BF16_NM, MSUB, LIFT, KH, NPAIR>>(a, b, e, o, p, s, q);
    case SLSP_OUT_BF16_MN:
      return run<Cfg<SPARSE, K, BN, 0, SLSP_OUT_BF16_MN, MSUB, LIFT, KH, NPAIR>>(a, b, e, o, p, s, q);
  }
  return SLSP_ERR_INVALID;
}

// Tile shape: 1 or 2 M-subtiles per CTA pair (env SLSP_GEMM_MSUB for the
// sparse kernel, SLSP_DGEMM_MSUB for the dense one; decode tiles: 1), and
// for two-subtile 8-bit sparse tiles optionally two pairs per cluster sharing
// the weight tile by multicast (npair = 2).
template <bool SPARSE, MmaKind K, int BN, int LIFT = 0>
int run_out(int out_mode, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& e, const CUtensorMap& o,
            const Params& p, cudaStream_t s, uint32_t msub, uint32_t kh, slsp_gemm_config* q, uint32_t npair = 1) {
  constexpr bool two_sub = BN >= 128 && !(SPARSE && BN > 224);  // two accumulators fit TMEM
  if constexpr (BN >= 128 && SPARSE && !LIFT && K != MmaKind::F16) {
    if (kh && msub == 1) return run_out_cl<SPARSE, K, BN, 1, 0, 1>(out_mode, a, b, e, o, p, s, q);
    if constexpr (two_sub) {
      if (kh && msub == 2 && out_mode == SLSP_OUT_BF16_NM)
        return run_out_cl<SPARSE, K, BN, 2, 0, 1>(out_mode, a, b, e, o, p, s, q);
      if (!kh && msub == 2 && npair == 2) return run_out_cl<SPARSE, K, BN, 2, 0, 0, 2>(out_mode, a, b, e, o, p, s, q);
    }
  }
  if constexpr (two_sub)
    if (msub == 2) return run_out_cl<SPARSE, K, BN, 2, LIFT, 0>(out_mode, a, b, e, o, p, s, q);
  return run_out_cl<SPARSE, K, BN, 1, LIFT, 0>(out_mode, a, b, e, o, p, s, q);
}

constexpr int kSparseBN = 224;
constexpr int kDenseBN = 256;
// Decode-shaped M (<= 64 tokens): 64-token tiles, so the smem ring holds
// mostly weight bytes (8 stages instead of 4) for the HBM-bound weight stream.
constexpr int kDecodeBN = 64;
constexpr uint32_t kSparseKHalf = 0;  // env SLSP_GEMM_KHALF
constexpr int64_t kDecodeM = 64;
// 64 < M <= 128: the 64-token tiles too, when they at most fill the machine
// once (2 token tiles per weight tile) and K is short (<= 8 KB of original
// weight row): the larger tile count beats re-streaming the weights twice
// (Qwen2.5-7B qkv/o and 4096x4096 at M = 96/128: 16.5 vs 20.5 us, sparse and
// dense alike); long-K or wide layers keep the 224/256-token tiles.
constexpr int64_t kDecodeM2 = 128;
constexpr int64_t kDecodeKBytes = 8192;

bool decode_tiles(int64_t n, int64_t m, int64_t k_bytes, const char* env) {
  const int64_t lim = static_cast<int64_t>(env_knob(env, kDecodeM));
  if (m <= lim) return true;
  if (m > kDecodeM2 || lim != kDecodeM) return false;
  return k_bytes <= kDecodeKBytes && (n + 255) / 256 * ((m + kDecodeBN - 1) / kDecodeBN) <= num_sms() / 2;
}
// Moderate M: 256-token sparse tiles (one subtile, single-buffered
// accumulator) where they need fewer token tiles than 224-token ones — each
// token tile re-streams the whole weight matrix (M = 256: 1 tile instead of
// 2; M = 512: 2 instead of 3) — and there are at most two waves of them (the
// accumulator drain between a cluster's tiles is exposed). Measured on the
// Qwen2.5-7B shapes at M = 256-2048, DESIGN.md §6. Env SLSP_GEMM_BN256_MAXM.
constexpr int64_t kBn256MaxM = 1024;
constexpr int kSparseBN256 = 256;
// half k-stages on one-subtile tiles up to M = 1024 (env SLSP_GEMM_KHALF1):
// measured 6-16% faster at M = 256-1000 on the Qwen2.5-7B shapes,
// bit-identical; at M = 8192 one-subtile tiles lose 10-20% with them
constexpr uint32_t kSparseKHalf1 = 1;
constexpr uint32_t kDenseMsub = 1;
constexpr uint32_t kTail0 = 1;     // early subtile-0 commit (Params::tail0; 2 = + reorder, measured slower)
constexpr uint32_t kSparseMc = 1;  // two pairs sharing the weight tile (two-subtile 8-bit tiles)
constexpr uint32_t kRasterGroup = 16;  // measured best of {4, 8, 16, 32, 148} on Qwen2.5-7B shapes

// M-subtiles for the sparse kernel: two subtiles (512 weight rows per pair,
// activation tile shared) move 29% fewer operand bytes per MAC but halve the
// tile count; use them unless that leaves a partial last wave the one-subtile
// grid would not have (measured on Qwen2.5-7B shapes).
uint32_t sparse_msub(int64_t n, int64_t m) {
  if (m <= 256) return 1;  // decode shapes: more weight tiles (split-K runs on one-subtile tiles)
  // wave quantization: a two-subtile tile costs ~1.8 one-subtile tiles
  // (measured); take one-subtile tiles only when their waves are clearly
  // cheaper (Qwen2.5-7B qkv at M = 2048: 90 two-subtile tiles = 1.2 waves on
  // 74 clusters, 0.041 ms, vs 180 one-subtile tiles 0.039 ms); otherwise two
  // (faster or equal on every Qwen2.5-7B shape at M = 8192)
  const int64_t clusters = num_sms() / 2;
  const int64_t nt = (m + kSparseBN - 1) / kSparseBN;
  const int64_t w2 = ((n + 511) / 512 * nt + clusters - 1) / clusters;
  const int64_t w1 = ((n + 255) / 256 * nt + clusters - 1) / clusters;
  return 10 * w1 < 9 * 18 * w2 / 10 ? 1 : 2;
}


int check_out(int out_mode, const float* s_ch, const float* s_tok, void* out, int64_t ldo, int64_t n, int64_t m) {
  if (n == 0 || m == 0) return SLSP_OK;  // empty result (the reference returns an empty matrix)
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

// Shared body of slsp_sparse_gemm (lifted activations, kp bytes per token)
// and slsp_sparse_gemm_x (unlifted X, kx = 2kp/3 bytes per token, lifted in
// shared memory; values/metadata in slsp_gemm_order's window order). With
// `q` set nothing is launched: the chosen configuration is reported.
template <bool LIFT>
int sparse_entry(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                 int64_t act_row, int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out,
                 int64_t ldo, slsp_stream_t stream, void* ws, int64_t ws_bytes, slsp_gemm_config* q = nullptr,
                 float* tok_amax = nullptr) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || kp <= 0) return SLSP_ERR_INVALID;
  if (kp % 256 != 0) return SLSP_ERR_DIMENSION;
  if (tok_amax && out_mode == SLSP_OUT_RAW_NM) return SLSP_ERR_INVALID;  // |y| max of the BF16 outputs
  if (kp > (int64_t{1} << 23)) return SLSP_ERR_INVALID;  // gemm.hpp:56 int8 accumulator bound
  if (n > (int64_t{1} << 31) - 256 || m > (int64_t{1} << 31) - 256) return SLSP_ERR_UNSUPPORTED;
  int st = SLSP_OK;
  if (out_mode != SLSP_OUT_RAW_NM && out_mode != SLSP_OUT_BF16_NM && out_mode != SLSP_OUT_BF16_MN)
    return SLSP_ERR_INVALID;
  if (!q && (st = check_out(out_mode, s_ch, s_tok, out, ldo, n, m))) return st;
  if (dtype != SLSP_DT_I8 && dtype != SLSP_DT_E4M3 && !(dtype == SLSP_DT_BF16 && !LIFT)) return SLSP_ERR_UNSUPPORTED;
  if ((st = require_sm100())) return st;
  if (!q && (n == 0 || m == 0)) return SLSP_OK;
  const int esz = dtype == SLSP_DT_BF16 ? 2 : 1;
  CUtensorMap ta{}, tb{}, te{}, to{};
  Params p{};

  const bool decode = !LIFT && decode_tiles(n, m, kp * esz * 2 / 3, "SLSP_GEMM_DECODE_M");
  const bool wide = !LIFT && !decode && m <= static_cast<int64_t>(env_knob("SLSP_GEMM_BN256_MAXM", kBn256MaxM)) &&
                    (m + kSparseBN256 - 1) / kSparseBN256 < (m + kSparseBN - 1) / kSparseBN &&
                    (n + 255) / 256 * ((m + kSparseBN256 - 1) / kSparseBN256) <=
                        static_cast<int64_t>(env_knob("SLSP_GEMM_BN256_WAVES", 2)) * (num_sms() / 2);
  const int bn = decode ? kDecodeBN : wide ? kSparseBN256 : kSparseBN;
  const uint32_t msub =
      (decode || wide) ? 1u : env_knob("SLSP_GEMM_MSUB", sparse_msub(n, m)) == 2 ? 2u : 1u;
  // half k-stages: the two-subtile BF16 [N][M] config (off by default), and
  // every one-subtile 8-bit config below the large-M regime (on: a 7-8
  // stage ring instead of 3-4 for the weight-stream-heavy moderate M)
  const uint32_t kh = !LIFT && !decode && esz == 1 && !tok_amax &&
                              ((msub == 2 && out_mode == SLSP_OUT_BF16_NM &&
                                env_knob("SLSP_GEMM_KHALF", kSparseKHalf)) ||
                               (msub == 1 && m <= kBn256MaxM && env_knob("SLSP_GEMM_KHALF1", kSparseKHalf1)))
                          ? 1u
                          : 0u;
  if (ws && ws_bytes >= 2 * n * m * 4 && !tok_amax) {  // split-K partial-sum slices (not with the amax fold)
    p.ws = ws;
    p.ws_cap = ws_bytes;
  }
  if (tok_amax && !q) {  // the fold max-accumulates into zeros
    SLSP_CUDA_TRY(cudaMemsetAsync(tok_amax, 0, static_cast<size_t>(m) * sizeof(float), s));
    p.amax = reinterpret_cast<uint32_t*>(tok_amax);
  }
  if (!q) {
    if ((st = make_map_2d(&tb, act, act_row * esz, m, bn / 2))) return st;
    if ((st = make_map_2d(&ta, values, kp / 2 * esz, n, 128, kh ? 64 : 128))) return st;
    // BF16 and half k-stages: a stage is 128 logical k -> one 2 KB metadata atom
    if ((st = make_map_meta(&te, meta, n, kp, (esz == 2 || kh) ? 8 : 16))) return st;
    if ((st = make_map_out(&to, out, out_mode, n, m, ldo, epi_cols(msub, bn, out_mode), &p.tma_store))) return st;
    select_epilogue(p, out_mode, msub, out, ldo, s_tok);
  }
  p.n = n;
  p.m = m;
  p.num_kb = static_cast<int>(kp * esz / (kh ? 128 : 256));
  p.s_ch = s_ch;
  p.s_tok = s_tok;
  p.out = out;
  p.ldo = ldo;
  p.debug = debug_flags();
  p.trace = reinterpret_cast<unsigned long long*>(env_ptr("SLSP_GEMM_TRACE"));
  p.hints = env_knob("SLSP_GEMM_HINTS", kDefaultHints);
  p.group = static_cast<int>(env_knob("SLSP_GEMM_GROUP", kRasterGroup));
  p.splitbar = static_cast<int>(env_knob("SLSP_GEMM_SPLITBAR", 1));
  p.tail0 = static_cast<int>(env_knob("SLSP_GEMM_TAIL0", kTail0));
  p.pace_ns = static_cast<int>(env_knob("SLSP_GEMM_PACE", 0));
  p.pf_stages = static_cast<int>(env_knob("SLSP_GEMM_PF", 0));
  p.pf_at = static_cast<int>(env_knob("SLSP_GEMM_PFAT", 8));
  constexpr int L = LIFT ? 1 : 0;
  if constexpr (!LIFT) {
    if (tok_amax) {  // the fold variants: 8-bit kinds (the next layer quantizes), no half k-stages
      if (dtype == SLSP_DT_BF16) return SLSP_ERR_UNSUPPORTED;
      const bool i8 = dtype == SLSP_DT_I8;
      if (decode)
        return i8 ? run_amax<MmaKind::I8, kDecodeBN>(out_mode, ta, tb, te, to, p, s, 1, q)
                  : run_amax<MmaKind::F8, kDecodeBN>(out_mode, ta, tb, te, to, p, s, 1, q);
      if (wide)
        return i8 ? run_amax<MmaKind::I8, kSparseBN256>(out_mode, ta, tb, te, to, p, s, 1, q)
                  : run_amax<MmaKind::F8, kSparseBN256>(out_mode, ta, tb, te, to, p, s, 1, q);
      return i8 ? run_amax<MmaKind::I8, kSparseBN>(out_mode, ta, tb, te, to, p, s, msub, q)
                : run_amax<MmaKind::F8, kSparseBN>(out_mode, ta, tb, te, to, p, s, msub, q);
    }
    if (decode) {
      if (dtype == SLSP_DT_I8) return run_out<true, MmaKind::I8, kDecodeBN>(out_mode, ta, tb, te, to, p, s, 1, 0, q);
      if (dtype == SLSP_DT_BF16)
        return run_out<true, MmaKind::F16, kDecodeBN>(out_mode, ta, tb, te, to, p, s, 1, 0, q);
      return run_out<true, MmaKind::F8, kDecodeBN>(out_mode, ta, tb, te, to, p, s, 1, 0, q);
    }
    if (wide) {
      if (dtype == SLSP_DT_I8)
        return run_out<true, MmaKind::I8, kSparseBN256>(out_mode, ta, tb, te, to, p, s, 1, kh, q);
      if (dtype == SLSP_DT_BF16)
        return run_out<true, MmaKind::F16, kSparseBN256>(out_mode, ta, tb, te, to, p, s, 1, 0, q);
      return run_out<true, MmaKind::F8, kSparseBN256>(out_mode, ta, tb, te, to, p, s, 1, kh, q);
    }
    if (dtype == SLSP_DT_BF16)
      return run_out<true, MmaKind::F16, kSparseBN>(out_mode, ta, tb, te, to, p, s, msub, 0, q);
  }
  // weight multicast across two pairs (env SLSP_GEMM_MC: 1 = off, 2 = on)
  const uint32_t npair = !LIFT && msub == 2 && !kh && env_knob("SLSP_GEMM_MC", kSparseMc) == 2 ? 2u : 1u;
  if (dtype == SLSP_DT_I8)
    return run_out<true, MmaKind::I8, kSparseBN, L>(out_mode, ta, tb, te, to, p, s, msub, kh, q, npair);
  return run_out<true, MmaKind::F8, kSparseBN, L>(out_mode, ta, tb, te, to, p, s, msub, kh, q, npair);
}

// slsp_sparse_gemm_lift: the BF16 sparse GEMM on the UNLIFTED activations
// (x: m x cols BF16, row stride x_ld elements); the kernel's lift warps build
// every B stage from x (Cfg::GLIFT). Decode tiles (64 tokens, one subtile) at
// every m; split-K as for sparse_gemm. Equals
// sparse_gemm(values, lift_rows(x, z, l, kp)) bit for bit.
int glift_entry(const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* x, int64_t x_ld, int64_t m,
                int64_t cols, int z, int l, const float* s_ch, const float* s_tok, int out_mode, void* out,
                int64_t ldo, void* ws, int64_t ws_bytes, slsp_stream_t stream, slsp_gemm_config* q = nullptr) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || kp <= 0 || cols < 0) return SLSP_ERR_INVALID;
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  if (kp % 256 != 0 || cols % l != 0) return SLSP_ERR_DIMENSION;  // quantize.hpp:78-81
  const int64_t windows = cols / l * wc;
  if (kp < windows * 4) return SLSP_ERR_DIMENSION;
  if (n > (int64_t{1} << 31) - 256 || m > (int64_t{1} << 31) - 256) return SLSP_ERR_UNSUPPORTED;
  if (out_mode != SLSP_OUT_RAW_NM && out_mode != SLSP_OUT_BF16_NM && out_mode != SLSP_OUT_BF16_MN)
    return SLSP_ERR_INVALID;
  if (!q && (st = check_out(out_mode, s_ch, s_tok, out, ldo, n, m))) return st;
  if (!q && m > 0 && (!x || x_ld < cols || (x_ld & 1) || (reinterpret_cast<uintptr_t>(x) & 3)))
    return SLSP_ERR_INVALID;  // window loads are 4-byte aligned pairs of BF16
  if ((st = require_sm100())) return st;
  if (!q && (n == 0 || m == 0)) return SLSP_OK;
  CUtensorMap ta{}, tb{}, te{}, to{};
  Params p{};
  if (ws && ws_bytes >= 2 * n * m * 4) {
    p.ws = ws;
    p.ws_cap = ws_bytes;
  }
  if (!q) {
    if ((st = make_map_2d(&ta, values, kp, n, 128, 128))) return st;  // kp/2 BF16 values per row
    if ((st = make_map_meta(&te, meta, n, kp, 8))) return st;
    if ((st = make_map_out(&to, out, out_mode, n, m, ldo, epi_cols(1, kDecodeBN, out_mode), &p.tma_store))) return st;
    select_epilogue(p, out_mode, 1, out, ldo, s_tok);
    tb = ta;  // unused: no B loads
  }
  p.n = n;
  p.m = m;
  p.num_kb = static_cast<int>(kp / 128);
  p.s_ch = s_ch;
  p.s_tok = s_tok;
  p.out = out;
  p.ldo = ldo;
  p.debug = debug_flags();
  p.trace = reinterpret_cast<unsigned long long*>(env_ptr("SLSP_GEMM_TRACE"));
  p.hints = env_knob("SLSP_GEMM_HINTS", kDefaultHints);
  p.group = static_cast<int>(env_knob("SLSP_GEMM_GROUP", kRasterGroup));
  p.splitbar = static_cast<int>(env_knob("SLSP_GEMM_SPLITBAR", 1));
  p.tail0 = static_cast<int>(env_knob("SLSP_GEMM_TAIL0", kTail0));
  p.x = x;
  p.x_ld = x_ld;
  p.lift_l = l;
  // the 6:8 path loads whole 16-byte source blocks: rows 16-byte aligned
  // (and the triple layout assumes windows at 0, 2, 4 of each 8-block)
  if (l == 8 && ((reinterpret_cast<uintptr_t>(x) & 15) || (x_ld & 7) || wc != 3)) p.lift_l = -8;
  p.lift_wc = wc;
  p.lift_windows = windows;
  return run_out_cl<true, MmaKind::F16, kDecodeBN, 1, 2, 0>(out_mode, ta, tb, te, to, p, s, q);
}

int dense_entry(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m, const float* s_ch,
                const float* s_tok, int out_mode, void* out, int64_t ldo, void* workspace, int64_t ws_bytes,
                slsp_stream_t stream, slsp_gemm_config* q = nullptr) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || k <= 0) return SLSP_ERR_INVALID;
  const int esz = elem_size(dtype);
  if (dtype != SLSP_DT_I8 && dtype != SLSP_DT_E4M3 && dtype != SLSP_DT_BF16) return SLSP_ERR_UNSUPPORTED;
  if ((k * esz) % 128 != 0) return SLSP_ERR_DIMENSION;
  if (dtype == SLSP_DT_I8 && k > (int64_t{1} << 23)) return SLSP_ERR_INVALID;  // gemm.hpp:147-149
  if (n > (int64_t{1} << 31) - 256 || m > (int64_t{1} << 31) - 256) return SLSP_ERR_UNSUPPORTED;
  if (out_mode != SLSP_OUT_RAW_NM && out_mode != SLSP_OUT_BF16_NM && out_mode != SLSP_OUT_BF16_MN)
    return SLSP_ERR_INVALID;
  int st = SLSP_OK;
  if (!q && (st = check_out(out_mode, s_ch, s_tok, out, ldo, n, m))) return st;
  if ((st = require_sm100())) return st;
  if (!q && (n == 0 || m == 0)) return SLSP_OK;
  CUtensorMap ta{}, tb{}, to{};
  Params p{};
  const bool decode = decode_tiles(n, m, k * esz, "SLSP_DGEMM_DECODE_M");
  const int bn = decode ? kDecodeBN : kDenseBN;
  const uint32_t msub = decode ? 1u : env_knob("SLSP_DGEMM_MSUB", kDenseMsub) == 2 ? 2u : 1u;
  if (workspace && ws_bytes >= 2 * n * m * 4) {  // split-K partial-sum slices
    p.ws = workspace;
    p.ws_cap = ws_bytes;
  }
  if (!q) {
    if ((st = make_map_2d(&ta, w, k * esz, n, 128))) return st;
    if ((st = make_map_2d(&tb, act, k * esz, m, bn / 2))) return st;
    if ((st = make_map_out(&to, out, out_mode, n, m, ldo, epi_cols(msub, bn, out_mode), &p.tma_store))) return st;
    select_epilogue(p, out_mode, msub, out, ldo, s_tok);
  }
  p.n = n;
  p.m = m;
  p.num_kb = static_cast<int>(k * esz / 128);
  p.s_ch = s_ch;
  p.s_tok = s_tok;
  p.out = out;
  p.ldo = ldo;
  p.debug = debug_flags();
  p.trace = reinterpret_cast<unsigned long long*>(env_ptr("SLSP_GEMM_TRACE"));
  p.hints = env_knob("SLSP_GEMM_HINTS", kDefaultHints);
  p.group = static_cast<int>(env_knob("SLSP_GEMM_GROUP", kRasterGroup));
  p.splitbar = static_cast<int>(env_knob("SLSP_GEMM_SPLITBAR", 1));
  if (dtype == SLSP_DT_I8)
    return decode ? run_out<false, MmaKind::I8, kDecodeBN>(out_mode, ta, tb, ta, to, p, s, 1, 0, q)
                  : run_out<false, MmaKind::I8, kDenseBN>(out_mode, ta, tb, ta, to, p, s, msub, 0, q);
  if (dtype == SLSP_DT_E4M3)
    return decode ? run_out<false, MmaKind::F8, kDecodeBN>(out_mode, ta, tb, ta, to, p, s, 1, 0, q)
                  : run_out<false, MmaKind::F8, kDenseBN>(out_mode, ta, tb, ta, to, p, s, msub, 0, q);
  return decode ? run_out<false, MmaKind::F16, kDecodeBN>(out_mode, ta, tb, ta, to, p, s, 1, 0, q)
                : run_out<false, MmaKind::F16, kDenseBN>(out_mode, ta, tb, ta, to, p, s, msub, 0, q);
}

}  // namespace

extern "C" {

int slsp_sparse_gemm(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                     int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                     slsp_stream_t stream) {
  return sparse_entry<false>(dtype, values, meta, n, kp, act, kp, m, s_ch, s_tok, out_mode, out, ldo, stream, nullptr,
                             0);
}

int slsp_sparse_gemm_ws(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                        int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                        void* workspace, int64_t ws_bytes, slsp_stream_t stream) {
  return sparse_entry<false>(dtype, values, meta, n, kp, act, kp, m, s_ch, s_tok, out_mode, out, ldo, stream, workspace,
                             ws_bytes);
}

int slsp_sparse_gemm_amax(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                          int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                          float* tok_amax, slsp_stream_t stream) {
  if (!tok_amax) return SLSP_ERR_INVALID;
  return sparse_entry<false>(dtype, values, meta, n, kp, act, kp, m, s_ch, s_tok, out_mode, out, ldo, stream, nullptr,
                             0, nullptr, tok_amax);
}

int64_t slsp_gemm_workspace_bytes(int64_t n, int64_t m) {
  if (m > kSplitMaxM || n <= 0 || m <= 0) return 0;
  const int64_t slice = n * m * 4;
  const int64_t full = 8 * slice;  // 8 slices, capped at kSplitWsCap (0 if that holds < 2 slices)
  return full <= kSplitWsCap ? full : (kSplitWsCap / slice >= 2 ? kSplitWsCap / slice * slice : 0);
}

int slsp_sparse_gemm_config(int dtype, int64_t n, int64_t kp, int64_t m, int out_mode, int64_t ws_bytes,
                            slsp_gemm_config* cfg) {
  if (!cfg) return SLSP_ERR_INVALID;
  *cfg = slsp_gemm_config{};
  // a non-null sentinel stands for "a workspace of ws_bytes will be passed"
  void* ws = ws_bytes > 0 ? reinterpret_cast<void*>(uintptr_t{256}) : nullptr;
  return sparse_entry<false>(dtype, nullptr, nullptr, n, kp, nullptr, kp, m, nullptr, nullptr, out_mode, nullptr, 0,
                             nullptr, ws, ws_bytes, cfg);
}

int slsp_dense_gemm_config(int dtype, int64_t n, int64_t k, int64_t m, int out_mode, int64_t ws_bytes,
                           slsp_gemm_config* cfg) {
  if (!cfg) return SLSP_ERR_INVALID;
  *cfg = slsp_gemm_config{};
  void* ws = ws_bytes > 0 ? reinterpret_cast<void*>(uintptr_t{256}) : nullptr;
  return dense_entry(dtype, nullptr, n, k, nullptr, m, nullptr, nullptr, out_mode, nullptr, 0, ws, ws_bytes, nullptr,
                     cfg);
}

int slsp_sparse_gemm_x(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kx, const void* act,
                       int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                       slsp_stream_t stream) {
  if (kx <= 0) return SLSP_ERR_INVALID;
  if (kx % 512 != 0) return SLSP_ERR_DIMENSION;
  return sparse_entry<true>(dtype, values, meta, n, kx / 2 * 3, act, kx, m, s_ch, s_tok, out_mode, out, ldo, stream,
                            nullptr, 0);
}

int slsp_dense_gemm(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m, const float* s_ch,
                    const float* s_tok, int out_mode, void* out, int64_t ldo, slsp_stream_t stream) {
  return dense_entry(dtype, w, n, k, act, m, s_ch, s_tok, out_mode, out, ldo, nullptr, 0, stream);
}

int slsp_dense_gemm_ws(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m, const float* s_ch,
                       const float* s_tok, int out_mode, void* out, int64_t ldo, void* workspace, int64_t ws_bytes,
                       slsp_stream_t stream) {
  return dense_entry(dtype, w, n, k, act, m, s_ch, s_tok, out_mode, out, ldo, workspace, ws_bytes, stream);
}

int slsp_sparse_gemm_lift(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* x,
                          int64_t x_ld, int64_t m, int64_t cols, int z, int l, const float* s_ch, const float* s_tok,
                          int out_mode, void* out, int64_t ldo, void* workspace, int64_t ws_bytes,
                          slsp_stream_t stream) {
  if (dtype != SLSP_DT_BF16) return SLSP_ERR_UNSUPPORTED;
  return glift_entry(values, meta, n, kp, x, x_ld, m, cols, z, l, s_ch, s_tok, out_mode, out, ldo, workspace, ws_bytes,
                     stream);
}

int slsp_sparse_gemm_lift_config(int dtype, int64_t n, int64_t kp, int64_t m, int64_t cols, int z, int l,
                                 int out_mode, int64_t ws_bytes, slsp_gemm_config* out) {
  if (!out) return SLSP_ERR_INVALID;
  if (dtype != SLSP_DT_BF16) return SLSP_ERR_UNSUPPORTED;
  *out = slsp_gemm_config{};
  // a non-null dummy so the config reflects a call that can split
  void* ws = ws_bytes > 0 ? reinterpret_cast<void*>(uintptr_t{256}) : nullptr;
  return glift_entry(nullptr, nullptr, n, kp, nullptr, cols, m, cols, z, l, nullptr, nullptr, out_mode, nullptr, 0, ws,
                     ws_bytes, nullptr, out);
}

}  // extern "C"
