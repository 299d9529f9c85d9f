// tc_ptx.cuh — PTX wrappers shared by the tcgen05 kernels (hv_tc.cu,
// grad_tc.cu): mbarriers, TMA, tcgen05 MMA / commit / TMEM ld-st, UMMA
// descriptors.  Internal linkage per translation unit.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace wgp {
namespace {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t addr = smem_u32(b);
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) break;
  }
}
// Non-blocking phase test (whole warp, uniform).
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// One try_wait probe: suspends the warp for up to a hardware time limit
// while the phase is incomplete (no issue-slot spinning), then reports.
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// MMA issue helpers are called by a whole converged warp with warp-uniform
// operands (so descriptors live in uniform registers); one lane, chosen by
// elect.sync, issues.
// The three 3xTF32 partial products of one K step from a single asm block
// (one elect): D (+)= A_hi B_hi + A_hi B_lo + A_lo B_hi.
__device__ __forceinline__ void mma3_ss(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, t, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %6, 0;\n"
      " setp.eq.u32 t, 0, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %3, %5, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %4, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, t;\n}\n" ::"r"(d),
      "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma3_ts(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, t, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %6, 0;\n"
      " setp.eq.u32 t, 0, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, t;\n}\n" ::"r"(d),
      "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
// TMA issue by one elected lane of a converged warp.
__device__ __forceinline__ void tma_load_2d_warp(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                                 int c1) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_warp(uint64_t* b, uint32_t bytes) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(b)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_warp(uint64_t* b) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(smem_u32(b))
      : "memory");
}

#define R8(i) "=r"(r[i + 0]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), \
              "=r"(r[i + 5]), "=r"(r[i + 6]), "=r"(r[i + 7])
#define W8(i) "r"(r[i + 0]), "r"(r[i + 1]), "r"(r[i + 2]), "r"(r[i + 3]), "r"(r[i + 4]), \
              "r"(r[i + 5]), "r"(r[i + 6]), "r"(r[i + 7])

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R8(0), R8(8), R8(16), R8(24)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : R8(0)
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      W8(0), W8(8), W8(16), W8(24)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 bytes (SBO), version 1 (sm_100), LBO unused for swizzled K-major.
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  return static_cast<uint64_t>((a >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// kind::f16 instruction descriptor: D f32, A/B fp16 (a/b format 0), both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : R8(0), R8(8)
      : "r"(taddr));
}
// 1D bulk copy global -> shared completing tx bytes on `bar` (one elected lane).
__device__ __forceinline__ void bulk_load_warp(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The 12 MMAs of one MMA-1 group (Gram, 4 K steps of 3xTF32, A and B from
// shared memory) from one asm block and one elect: per-k descriptors by
// immediate adds.  Per-k-step helper calls cost the issuing warp ~45
// instructions each (elect, uniform-register moves, descriptor math), taken
// from the epilogue warps of the same SMSP (measured in grad_tc).
__device__ __forceinline__ void mma1_group_tf32(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                                uint32_t idesc) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b64 xh, xl, yh, yl;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.s64 xh, %1, 0;\n"
      " add.s64 xl, %2, 0;\n"
      " add.s64 yh, %3, 0;\n"
      " add.s64 yl, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yh, %5, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xl, yh, %5, t;\n"
      " add.s64 xh, %1, 2;\n"
      " add.s64 xl, %2, 2;\n"
      " add.s64 yh, %3, 2;\n"
      " add.s64 yl, %4, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xl, yh, %5, t;\n"
      " add.s64 xh, %1, 4;\n"
      " add.s64 xl, %2, 4;\n"
      " add.s64 yh, %3, 4;\n"
      " add.s64 yl, %4, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xl, yh, %5, t;\n"
      " add.s64 xh, %1, 6;\n"
      " add.s64 xl, %2, 6;\n"
      " add.s64 yh, %3, 6;\n"
      " add.s64 yl, %4, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xh, yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], xl, yh, %5, t;\n"
      "}\n"
      ::"r"(d), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc));
}
// Packed Gram (small d): the three 3xTF32 passes concatenated along K,
// a' = [a_hi | a_hi | a_lo], b' = [b_hi | b_lo | b_hi] (each d + 2 wide), so
// a'.b' = hi.hi + hi.lo + lo.hi in nk = ceil(3 (d + 2) / 8) <= 8 K steps
// instead of 12 MMAs.  K columns 0..31 live in the "hi" plane, 32..63 in
// the "lo" plane; steps past nk are predicated off (one elect, one block).
#define WGP_PACKED_PREDS                                  \
  " setp.ne.b32 f, 0, 0;\n"                               \
  " setp.eq.b32 t, 0, 0;\n"                               \
  " elect.sync _|e, 0xffffffff;\n"                        \
  " setp.gt.u32 q, %6, 1;\n and.pred p1, e, q;\n"         \
  " setp.gt.u32 q, %6, 2;\n and.pred p2, e, q;\n"         \
  " setp.gt.u32 q, %6, 3;\n and.pred p3, e, q;\n"         \
  " setp.gt.u32 q, %6, 4;\n and.pred p4, e, q;\n"         \
  " setp.gt.u32 q, %6, 5;\n and.pred p5, e, q;\n"         \
  " setp.gt.u32 q, %6, 6;\n and.pred p6, e, q;\n"         \
  " setp.gt.u32 q, %6, 7;\n and.pred p7, e, q;\n"
__device__ __forceinline__ void mma1_packed_tf32(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                                 uint32_t idesc, uint32_t nk) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t, q, p1, p2, p3, p4, p5, p6, p7;\n"
      " .reg .b64 x, y;\n" WGP_PACKED_PREDS
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %3, %5, f;\n"
      " add.s64 x, %1, 2;\n add.s64 y, %3, 2;\n"
      " @p1 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      " add.s64 x, %1, 4;\n add.s64 y, %3, 4;\n"
      " @p2 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      " add.s64 x, %1, 6;\n add.s64 y, %3, 6;\n"
      " @p3 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      " @p4 tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %4, %5, t;\n"
      " add.s64 x, %2, 2;\n add.s64 y, %4, 2;\n"
      " @p5 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      " add.s64 x, %2, 4;\n add.s64 y, %4, 4;\n"
      " @p6 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      " add.s64 x, %2, 6;\n add.s64 y, %4, 6;\n"
      " @p7 tcgen05.mma.cta_group::1.kind::tf32 [%0], x, y, %5, t;\n"
      "}\n" ::"r"(d),
      "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(nk));
}
// As mma1_packed_tf32 with A_I in TMEM: K column k at TMEM column a0 + k.
__device__ __forceinline__ void mma1_packed_tf32_ts(uint32_t d, uint32_t a0, uint64_t bh, uint64_t bl,
                                                    uint32_t idesc, uint32_t nk) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t, q, p1, p2, p3, p4, p5, p6, p7;\n"
      " .reg .b32 x;\n"
      " .reg .b64 y;\n" WGP_PACKED_PREDS
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, f;\n"
      " add.u32 x, %1, 8;\n add.s64 y, %3, 2;\n"
      " @p1 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      " add.u32 x, %1, 16;\n add.s64 y, %3, 4;\n"
      " @p2 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      " add.u32 x, %1, 24;\n add.s64 y, %3, 6;\n"
      " @p3 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      " add.u32 x, %1, 32;\n"
      " @p4 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], %4, %5, t;\n"
      " add.u32 x, %1, 40;\n add.s64 y, %4, 2;\n"
      " @p5 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      " add.u32 x, %1, 48;\n add.s64 y, %4, 4;\n"
      " @p6 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      " add.u32 x, %1, 56;\n add.s64 y, %4, 6;\n"
      " @p7 tcgen05.mma.cta_group::1.kind::tf32 [%0], [x], y, %5, t;\n"
      "}\n" ::"r"(d),
      "r"(a0), "l"(0ull), "l"(bh), "l"(bl), "r"(idesc), "r"(nk));
}
#undef WGP_PACKED_PREDS
// MMA-1 group with A_I in TMEM (hi at column ah, lo at al): 12 MMAs, one
// asm block and one elect, as mma1_group_tf32.
__device__ __forceinline__ void mma1_group_tf32_ts(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                                   uint32_t idesc) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 xh, xl;\n"
      " .reg .b64 yh, yl;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 xh, %1, 0;\n"
      " add.u32 xl, %2, 0;\n"
      " add.s64 yh, %3, 0;\n"
      " add.s64 yl, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yh, %5, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xl], yh, %5, t;\n"
      " add.u32 xh, %1, 8;\n"
      " add.u32 xl, %2, 8;\n"
      " add.s64 yh, %3, 2;\n"
      " add.s64 yl, %4, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xl], yh, %5, t;\n"
      " add.u32 xh, %1, 16;\n"
      " add.u32 xl, %2, 16;\n"
      " add.s64 yh, %3, 4;\n"
      " add.s64 yl, %4, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xl], yh, %5, t;\n"
      " add.u32 xh, %1, 24;\n"
      " add.u32 xl, %2, 24;\n"
      " add.s64 yh, %3, 6;\n"
      " add.s64 yl, %4, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yh, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xh], yl, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [xl], yh, %5, t;\n"
      "}\n"
      ::"r"(d), "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc));
}
// The 12 MMAs of one MMA-2 tile (K.V, 4 K steps of 3xTF32: k_hi / k_lo in
// TMEM at kcol / kcol + 64, V hi / lo descriptors vh / vl) from one asm block
// and one elect; acc = 0 starts the accumulator (first tile of a chunk).
__device__ __forceinline__ void mma2_tile_tf32(uint32_t o, uint32_t kcol, uint64_t vh, uint64_t vl, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n"
      " .reg .pred e, p, t;\n"
      " .reg .b32 ah, al;\n"
      " .reg .b64 yh, yl;\n"
      " setp.ne.b32 p, %5, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 ah, %1, 0;\n"
      " add.u32 al, %1, 64;\n"
      " add.s64 yh, %2, 0;\n"
      " add.s64 yl, %3, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yh, %4, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], yh, %4, t;\n"
      " add.u32 ah, %1, 8;\n"
      " add.u32 al, %1, 72;\n"
      " add.s64 yh, %2, 2;\n"
      " add.s64 yl, %3, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], yh, %4, t;\n"
      " add.u32 ah, %1, 16;\n"
      " add.u32 al, %1, 80;\n"
      " add.s64 yh, %2, 4;\n"
      " add.s64 yl, %3, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], yh, %4, t;\n"
      " add.u32 ah, %1, 24;\n"
      " add.u32 al, %1, 88;\n"
      " add.s64 yh, %2, 6;\n"
      " add.s64 yl, %3, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], yh, %4, t;\n"
      "}\n"
      ::"r"(o), "r"(kcol), "l"(vh), "l"(vl), "r"(idesc), "r"(acc));
}
// The 12 MMAs of one fp16 MMA-2 tile (64 points, 4 K steps of 16 in fp16 x 3):
// per 32-column half h of the tile's TMEM columns, k1 pairs in [32h, 32h+16)
// and k2 pairs in [32h+16, 32h+32) (8 columns per K step); V hi / lo
// descriptors advance 32 bytes per K step.  One asm block, one elect.
__device__ __forceinline__ void mma2_tile_f16(uint32_t o, uint32_t kcol, uint64_t vh, uint64_t vl, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n"
      " .reg .pred e, p, t;\n"
      " .reg .b32 a1, a2;\n"
      " .reg .b64 yh, yl;\n"
      " setp.ne.b32 p, %5, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 a1, %1, 0;\n"
      " add.u32 a2, %1, 16;\n"
      " add.s64 yh, %2, 0;\n"
      " add.s64 yl, %3, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yh, %4, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], yh, %4, t;\n"
      " add.u32 a1, %1, 8;\n"
      " add.u32 a2, %1, 24;\n"
      " add.s64 yh, %2, 2;\n"
      " add.s64 yl, %3, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], yh, %4, t;\n"
      " add.u32 a1, %1, 32;\n"
      " add.u32 a2, %1, 48;\n"
      " add.s64 yh, %2, 4;\n"
      " add.s64 yl, %3, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], yh, %4, t;\n"
      " add.u32 a1, %1, 40;\n"
      " add.u32 a2, %1, 56;\n"
      " add.s64 yh, %2, 6;\n"
      " add.s64 yl, %3, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], yl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], yh, %4, t;\n"
      "}\n"
      ::"r"(o), "r"(kcol), "l"(vh), "l"(vl), "r"(idesc), "r"(acc));
}
// TMA 2D load multicast to the CTAs of `mask` in the cluster: the box lands at
// the same shared-memory offset in each and completes tx bytes on the
// mbarrier at the same offset in each (one elected lane).
__device__ __forceinline__ void tma_load_2d_mc_warp(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                    uint16_t mask) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// MMA completion arrive on the mbarrier at this offset in every CTA of `mask`.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// All threads of all CTAs of the cluster.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 32-bit load of `p` (this CTA's shared variable) in the shared memory of
// cluster CTA `rank` (distributed shared memory).
__device__ __forceinline__ uint32_t ld_shared_cluster_u32(const void* p, uint32_t rank) {
  uint32_t a, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

}  // namespace
}  // namespace wgp
