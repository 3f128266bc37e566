// Shared sm_100a device helpers: mbarriers, TMA, tcgen05 (TMEM / UMMA), and
// small numeric utilities. Inline PTX only; no CUTLASS/CuTe dispatch.
#pragma once

#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SLSP_DEVINL __device__ __forceinline__

namespace slsp_dev {

// ---------------------------------------------------------------- basics --
SLSP_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SLSP_DEVINL uint32_t lane_id() { return threadIdx.x & 31u; }

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

SLSP_DEVINL uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

SLSP_DEVINL void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Address of the same shared-memory object in CTA `rank` of the cluster.
SLSP_DEVINL uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

SLSP_DEVINL bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// -------------------------------------------------------------- mbarrier --
SLSP_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

SLSP_DEVINL void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

SLSP_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SLSP_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Arrive on a barrier that may live in another CTA of the cluster. Default
// (.release.cta) semantics: used to hand TMEM back to the MMA warp, which
// reads no memory the arriving threads wrote (the tcgen05 fences order the
// TMEM loads); .release.cluster would add MEMBAR.GPU + ERRBAR per arrive.
SLSP_DEVINL void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Release at cluster scope: orders this thread's prior shared-memory writes
// (already fenced to the async proxy) before the remote barrier's completion.
SLSP_DEVINL void mbar_arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Distributed shared memory: 16 bytes from a shared::cluster address (mapa).
SLSP_DEVINL uint4 ld_shared_cluster_v4(uint32_t cluster_addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

SLSP_DEVINL void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

#ifdef SLSP_WATCHDOG
// Debug build (build.py --watchdog): a wait that spins ~seconds reports the
// barrier (smem offset, parity) of the first stuck thread and traps.
SLSP_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (long long n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (n == (1ll << 21)) {
      printf("SLSP WATCHDOG block %d warp %d lane %d: barrier smem+%u parity %u\n", blockIdx.x, threadIdx.x / 32,
             threadIdx.x % 32, smem_u32(bar), parity);
      asm volatile("trap;");
    }
  }
}
#else
SLSP_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif

SLSP_DEVINL void mbar_wait_cluster_acquire(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------- TMA --
SLSP_DEVINL void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// L2 prefetch of one tensor box (no shared-memory destination, no completion).
SLSP_DEVINL void tma_prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

// 2-CTA (cta_group::2) tensor loads: data lands in the issuing CTA's smem,
// completion bytes are reported to `bar_cluster` (the leader CTA's barrier).
SLSP_DEVINL void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

SLSP_DEVINL void tma_load_3d_cg2(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Same, with an L2 eviction-priority policy (createpolicy).
SLSP_DEVINL void tma_load_2d_cg2_hint(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1,
                                      uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// Plain (one-CTA) tensor load into this CTA's smem, completion on a local barrier.
SLSP_DEVINL void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// cta_group::2 load multicast to the CTAs in `mask` (same smem offset in each);
// completion bytes go to each destination pair's leader barrier.
SLSP_DEVINL void tma_load_2d_cg2_mc(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1,
                                    uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
      : "memory");
}

SLSP_DEVINL void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1, uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
               : "memory");
}

SLSP_DEVINL uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// smem -> global tensor store (bulk async group), used by the GEMM epilogue.
SLSP_DEVINL void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
SLSP_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
SLSP_DEVINL void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
SLSP_DEVINL void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Make generic-proxy smem writes visible to the async (TMA) proxy.
SLSP_DEVINL void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

SLSP_DEVINL void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
SLSP_DEVINL void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

SLSP_DEVINL uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SLSP_DEVINL uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// --------------------------------------------------------------- tcgen05 --
template <int CG>
SLSP_DEVINL void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  if constexpr (CG == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  } else {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
}

template <int CG>
SLSP_DEVINL void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
  else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

SLSP_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SLSP_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Commit all prior tcgen05 async ops of this thread to an mbarrier, multicast
// to the CTAs in `cta_mask` (same smem offset in each).
SLSP_DEVINL void tc_commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
SLSP_DEVINL void tc_commit_1cta(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// UMMA shared-memory matrix descriptor (K-major).
//   layout: 0 = no swizzle (interleave), 2 = 128B swizzle.
SLSP_DEVINL uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// Instruction descriptor (kind::i8 / f8f6f4 / f16), both operands K-major.
//   c_fmt: 1 = F32, 2 = S32; a/b_fmt per kind (i8: 1 = signed; e4m3: 0; bf16: 1).
__host__ __device__ constexpr uint32_t make_idesc(bool sparse, uint32_t c_fmt, uint32_t a_fmt, uint32_t b_fmt,
                                                  uint32_t M, uint32_t N) {
  return (sparse ? (1u << 2) : 0u) | (c_fmt << 4) | (a_fmt << 7) | (b_fmt << 10) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

enum class MmaKind { I8 = 0, F8 = 1, F16 = 2 };

template <MmaKind K>
SLSP_DEVINL void umma_dense_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  if constexpr (K == MmaKind::I8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
  else if constexpr (K == MmaKind::F8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <MmaKind K>
SLSP_DEVINL void umma_sparse_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t e_tmem, uint32_t idesc,
                                 uint32_t acc) {
  if constexpr (K == MmaKind::I8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(e_tmem));
  else if constexpr (K == MmaKind::F8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.sp.cta_group::2.kind::f8f6f4 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(e_tmem));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(e_tmem));
}

// smem -> TMEM copy of a 128-lane x 128-bit tile (the sparse metadata atom).
SLSP_DEVINL void tmem_cp_128x128b_cg2(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

// TMEM -> registers: 32 lanes x 32 columns of 32-bit (one warp, its lane quarter).
SLSP_DEVINL void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

SLSP_DEVINL void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int N>
SLSP_DEVINL void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 64) {
    tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
    tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
  } else if constexpr (N == 32) {
    tmem_ld_32x32b_x32(taddr, r);
  } else {
    tmem_ld_32x32b_x16(taddr, r);
  }
}

SLSP_DEVINL void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// tcgen05.ld.16x256b.x1: 16 TMEM lanes x 8 columns; thread T receives
// r0 = (lane T/4, col 2(T%4)), r1 = (lane T/4, col 2(T%4)+1),
// r2 = (lane 8+T/4, col 2(T%4)), r3 = (lane 8+T/4, col 2(T%4)+1) — measured
// (tests/micro/tmem_layout.cu); the mma.sync C-fragment layout.
SLSP_DEVINL void tmem_ld_16x256b_x1(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
// .x2: two consecutive 8-column blocks, registers [4i, 4i+4) = block i (measured)
SLSP_DEVINL void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
SLSP_DEVINL void tmem_ld_wait_regs16(uint32_t (&a)[8], uint32_t (&b)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
               :
               : "memory");
}
SLSP_DEVINL void tmem_ld_wait_regs8(uint32_t (&a)[4], uint32_t (&b)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3])
               :
               : "memory");
}

// stmatrix.m8n8.x4.trans: stored row r of matrix m (16 bytes at the address
// lane 8m + r supplies) = for j = 0..7 the (r & 1) half of register m of
// thread 4j + r/2 (measured, tests/micro/tmem_layout.cu). With register m of
// thread T = (feature 8m + T/4: tokens 2(T%4), 2(T%4)+1) that is row = token r,
// 8 consecutive features — the transpose the token-major epilogue needs.
// ldmatrix.m8n8.x4 (no transpose): register i of thread T = (row T/4, cols
// 2(T%4), 2(T%4)+1) of matrix i, whose row j is read at the address lane 8i+j
// supplies (16 bytes = 8 b16).
SLSP_DEVINL void ldmatrix_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr)
               : "memory");
}

SLSP_DEVINL void stmatrix_x4_trans(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0),
               "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}

// wait::ld that also orders every later use of r after the wait (the
// registers of an in-flight tcgen05.ld are read-write operands of the wait).
SLSP_DEVINL void tmem_ld_wait_regs(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])
               :
               : "memory");
}

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start its prologue
// while the previous kernel in the stream drains; pdl_wait() blocks until that
// kernel has completed and its memory is visible, pdl_trigger() lets the next
// kernel launch. Both are no-ops for kernels launched without the attribute.
SLSP_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SLSP_DEVINL void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

SLSP_DEVINL uint4 ld_shared_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

SLSP_DEVINL float2 ld_shared_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

SLSP_DEVINL float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// Non-blocking probe of an mbarrier phase.
SLSP_DEVINL bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Packed fp32 pair multiply (sm_100 FMUL2): two IEEE round-to-nearest products,
// bit-identical to two __fmul_rn.
SLSP_DEVINL float2 fmul2_rn(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a2, b2, d2;\n\t"
      "mov.b64 a2, {%2, %3};\n\tmov.b64 b2, {%4, %5};\n\t"
      "mul.rn.f32x2 d2, a2, b2;\n\tmov.b64 {%0, %1}, d2;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

SLSP_DEVINL float2 fadd2_rn(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a2, b2, d2;\n\t"
      "mov.b64 a2, {%2, %3};\n\tmov.b64 b2, {%4, %5};\n\t"
      "add.rn.f32x2 d2, a2, b2;\n\tmov.b64 {%0, %1}, d2;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

SLSP_DEVINL float2 fsub2_rn(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a2, b2, d2;\n\t"
      "mov.b64 a2, {%2, %3};\n\tmov.b64 b2, {%4, %5};\n\t"
      "sub.rn.f32x2 d2, a2, b2;\n\tmov.b64 {%0, %1}, d2;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// 32-byte global store (sm_100 STG.256) with an L2 cache-policy hint.
SLSP_DEVINL void st_global_v8_hint(void* p, const uint32_t (&w)[8], uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "l"(pol)
               : "memory");
}

// ------------------------------------------------------------- numerics --
// fp8.hpp:25-52 (reference) restated for the device: e4m3fn, RNE in double,
// saturating at +-448, sign kept for tiny negatives (0x80).
SLSP_DEVINL uint8_t fp8_e4m3_encode(double x) {
  if (isnan(x)) return 0x7F;
  const uint8_t sign = signbit(x) ? 0x80 : 0x00;
  const double a = fabs(x);
  if (a == 0.0) return sign;
  if (a >= 448.0) return sign | 0x7E;
  int exp2 = 0;
  frexp(a, &exp2);
  int e = exp2 - 1;
  if (e < -6) {
    const double m = rint(ldexp(a, 9));
    if (m >= 8.0) return sign | 0x08;
    return sign | static_cast<uint8_t>(m);
  }
  double q = rint(ldexp(a, 3 - e));
  if (q >= 16.0) {
    q = 8.0;
    ++e;
  }
  if (e > 8) return sign | 0x7E;
  const uint8_t ef = static_cast<uint8_t>(e + 7);
  const uint8_t mant = static_cast<uint8_t>(q) & 0x7;
  if (ef == 15 && mant == 7) return sign | 0x7E;
  return sign | static_cast<uint8_t>(ef << 3) | mant;
}

SLSP_DEVINL float fp8_e4m3_decode(uint8_t code) {
  const int exp_field = (code >> 3) & 0xF;
  const int mant = code & 0x7;
  if (exp_field == 15 && mant == 7) return __int_as_float(0x7fc00000);
  float v = exp_field == 0 ? ldexpf(static_cast<float>(mant) / 8.0f, -6)
                           : ldexpf(1.0f + static_cast<float>(mant) / 8.0f, exp_field - 7);
  return (code & 0x80) ? -v : v;
}

// quantize.hpp:30-37: int8 = clamp(rne(s), +-127); fp8: 0 -> 0x00 else encode(clamp(s, +-448)).
SLSP_DEVINL uint8_t quantize_value(double scaled, int kind) {
  if (kind == 0) {
    double q = rint(scaled);
    q = fmin(fmax(q, -127.0), 127.0);
    return static_cast<uint8_t>(static_cast<int8_t>(q));
  }
  if (scaled == 0.0) return 0;
  return fp8_e4m3_encode(fmin(fmax(scaled, -448.0), 448.0));
}

}  // namespace slsp_dev
