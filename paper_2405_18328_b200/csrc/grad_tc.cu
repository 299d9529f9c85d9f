// grad_tc.cu — gradient contraction on the tensor core (the
// derivative_contractions of proj/src/kernel.cpp:199-262).
//
// Per entry (i, j) the gradient needs
//   W^B_ij = sum_c L_ic R_jc            (an s-long dot product: GEMM-shaped)
//   u_ij, decay 2^-u, k_ij, (x_ik - x_jk)^2 per lengthscale   (O(d) CUDA-core work)
// and accumulates, per lengthscale k and for the signal,
//   A_k = sum W^A decay dx_k^2,  B_k = sum W^B decay dx_k^2,
//   A_s = sum W^A k,             B_s = sum W^B k,   W^A = vy_i vy_j / 2.
// The SIMT kernel (grad_rff.cu) spends ~64 of its ~100 FP ops per entry on
// W^B.  Here the tensor core forms W^B (3xTF32, ~2^-21 per product: L_I from
// TMEM, R_J from shared memory, fp32 accumulation over s <= 64 terms) and the
// epilogue warps do only the O(d) part: ~5d + 6 FP ops and 2 MUFU per entry.
// The distances are formed from direct coordinate differences (not a Gram),
// exactly as the SIMT kernel does: they are needed for the per-lengthscale
// terms anyway and keep r^2 >= 0 and bit-identical to grad_simt.
//
// CTA = 128 rows (TMEM lanes) x a J range in 64-point tiles.  Warps 0..11:
// three epilogue groups (group w takes tiles t = w mod 3; warp w % 4 owns
// TMEM lanes 32 (w % 4) .. +31 = its 32 rows); warp 12 TMA / bulk producer;
// warp 13 MMA issuer; warp 14 TMEM allocator.  TMEM: six W buffers of 64
// fp32 columns [0, 384), L_I hi [384, 448), L_I lo [448, 512).  Rings:
// R_J planes (consumed by the MMA, freed by its commit) and the epilogue's
// per-point data x_j | vy_j (freed by the epilogue).  Reductions: fp32 per
// row over 4 tiles (256 entries), then a per-row fp64 sum in shared memory,
// fp64 warp / CTA sums in fixed order, one fp64 partial per CTA -- the
// [2 (d + 1)] partial format grad_finalize sums (bitwise deterministic).
#include "common.cuh"
#include "hv_tc.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace wgp {
namespace {

constexpr int gTI = 128;             // rows per CTA (MMA M, TMEM lanes)
constexpr int gTJ = 64;              // points per J tile (MMA N)
constexpr int gThreads = 512;
constexpr int gEpiGroups = 3, gEpiWarps = 12, gEpiThreads = 384;
// Warp roles.  Every SMSP (warp % 4) runs three epilogue warps (4..15; warp
// w reads TMEM lanes 32 (w % 4) .. +31) and one issuer warp (0..3): issuer q
// loads and multiplies the tiles t = q (mod 4).  The issue work of the loads
// and MMAs costs the hosting SMSP's epilogue warps issue slots, and each
// epilogue group advances at the pace of its slowest lane quarter, so it is
// spread evenly (measured with WGP_GRAD_TRACE: a single issuer warp left its
// SMSP's epilogue warps the bottleneck of the whole pipeline).
constexpr int gEpiBase = 4;
constexpr int gIssuers = 4;
constexpr int gWarpAlloc = 1;
constexpr int gBufs = 6;                    // W buffers (64 TMEM columns each)
constexpr uint32_t gLhi = 384, gLlo = 448;  // L_I planes, <= 64 columns each
constexpr int gNM = 4;                      // R_J ring: stage t % 4, owned by issuer t % 4
constexpr int gMaxNE = 8;                   // epilogue-data ring: 8 (or 4 when shared memory is short)
constexpr int gFlushTiles = 4;              // fp32 row sums span 4 tiles (256 entries)
constexpr int gSmemLimit = 232448 - 4096;   // 227 KB opt-in minus static smem
constexpr uint32_t gTfMask = 0xFFFFE000u;

// Epilogue stage of one tile: [d + 1][64] fp32, coordinate-major (rows 0..d-1:
// -x_jk, row d: vy_j), so one 16-byte shared load yields 4 points of one
// coordinate (two float2 pairs) and x_ik - x_jk is one FADD2.
__host__ __device__ constexpr int ep_of(int d) { return d + 1; }

// After tcgen05.wait::ld: the registers of the completed load are redefined
// here for the compiler, so no use or copy of them is scheduled before the wait.
__device__ __forceinline__ void pin(uint32_t (&r)[16]) {
  asm volatile("" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
               "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
               "+r"(r[14]), "+r"(r[15]));
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

// Per-entry work of two points j, j+1 (one row i per lane) in packed fp32x2
// (FADD2 / FMUL2 / FFMA2 halve the issue slots of the FMA-pipe work, which
// bounds this epilogue): nx[k] = -x_jk pair, vy pair, w = W^B pair.
template <int D>
__device__ __forceinline__ void entry_pair(const float2 (&xi)[D], const float2 (&nx)[D], float2 vy, float2 w,
                                           float2 sf2, float2 ac, float2 (&A)[D + 1], float2 (&B)[D + 1]) {
  float2 dq[D];
  float2 r2;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float2 df = __fadd2_rn(xi[k], nx[k]);
    dq[k] = __fmul2_rn(df, df);
    r2 = k == 0 ? dq[0] : __fadd2_rn(r2, dq[k]);
  }
  float2 u, dec;
  u.x = sqrt_approx(r2.x);
  u.y = sqrt_approx(r2.y);
  dec.x = ex2_approx(-u.x);
  dec.y = ex2_approx(-u.y);
  const float2 pk = __ffma2_rn(ac, u, sf2);  // k = pk * dec
  const float2 dA = __fmul2_rn(dec, vy), dB = __fmul2_rn(dec, w);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    A[k] = __ffma2_rn(dq[k], dA, A[k]);
    B[k] = __ffma2_rn(dq[k], dB, B[k]);
  }
  A[D] = __ffma2_rn(pk, dA, A[D]);
  B[D] = __ffma2_rn(pk, dB, B[D]);
}

// W(t) = L_I R_J^T in 3xTF32 over K = 32 (4 K steps): all 12 MMAs of a tile from one
// asm block and one elect (per-k A / B addresses by immediate adds), so the
// issuing warp costs its SMSP ~34 instructions per tile instead of ~180.
// a: TMEM address of L_I hi column 0 (lo 64 columns further); bh / bl: B
// descriptors of the stage's hi / lo plane (boxes of 32 K, 8192 bytes apart).
__device__ __forceinline__ void mma_w_k32(uint32_t d, uint32_t a, uint64_t bh, uint64_t bl, uint32_t idesc) {
  asm volatile(
      "{\n .reg .pred e, f, t;\n .reg .b32 ah, al;\n .reg .b64 dh, dl;\n"
      " setp.ne.b32 f, 0, 0;\n setp.eq.b32 t, 0, 0;\n elect.sync _|e, 0xffffffff;\n"
      " add.u32 ah, %1, 0;\n add.u32 al, %1, 64;\n add.s64 dh, %2, 0;\n add.s64 dl, %3, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 8;\n add.u32 al, %1, 72;\n add.s64 dh, %2, 2;\n add.s64 dl, %3, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 16;\n add.u32 al, %1, 80;\n add.s64 dh, %2, 4;\n add.s64 dl, %3, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 24;\n add.u32 al, %1, 88;\n add.s64 dh, %2, 6;\n add.s64 dl, %3, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      "}\n"
      ::"r"(d), "r"(a), "l"(bh), "l"(bl), "r"(idesc));
}
// W(t) = L_I R_J^T in 3xTF32 over K = 64 (8 K steps): all 24 MMAs of a tile from one
// asm block and one elect (per-k A / B addresses by immediate adds), so the
// issuing warp costs its SMSP ~62 instructions per tile instead of ~360.
// a: TMEM address of L_I hi column 0 (lo 64 columns further); bh / bl: B
// descriptors of the stage's hi / lo plane (boxes of 32 K, 8192 bytes apart).
__device__ __forceinline__ void mma_w_k64(uint32_t d, uint32_t a, uint64_t bh, uint64_t bl, uint32_t idesc) {
  asm volatile(
      "{\n .reg .pred e, f, t;\n .reg .b32 ah, al;\n .reg .b64 dh, dl;\n"
      " setp.ne.b32 f, 0, 0;\n setp.eq.b32 t, 0, 0;\n elect.sync _|e, 0xffffffff;\n"
      " add.u32 ah, %1, 0;\n add.u32 al, %1, 64;\n add.s64 dh, %2, 0;\n add.s64 dl, %3, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 8;\n add.u32 al, %1, 72;\n add.s64 dh, %2, 2;\n add.s64 dl, %3, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 16;\n add.u32 al, %1, 80;\n add.s64 dh, %2, 4;\n add.s64 dl, %3, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 24;\n add.u32 al, %1, 88;\n add.s64 dh, %2, 6;\n add.s64 dl, %3, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 32;\n add.u32 al, %1, 96;\n add.s64 dh, %2, 512;\n add.s64 dl, %3, 512;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 40;\n add.u32 al, %1, 104;\n add.s64 dh, %2, 514;\n add.s64 dl, %3, 514;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 48;\n add.u32 al, %1, 112;\n add.s64 dh, %2, 516;\n add.s64 dl, %3, 516;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      " add.u32 ah, %1, 56;\n add.u32 al, %1, 120;\n add.s64 dh, %2, 518;\n add.s64 dl, %3, 518;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dh, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], dl, %4, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], dh, %4, t;\n"
      "}\n"
      ::"r"(d), "r"(a), "l"(bh), "l"(bl), "r"(idesc));
}

struct GradTcArgs {
  int64_t n;
  int64_t r0, r1;  // rows [r0, r1)
  int d, dp, s, spk;  // spk: K extent of W^B (32 or 64: multiples of one 128-byte swizzle row)
  int num_jt, splits, ne;
  int cs, rt_pad;     // cluster size (CTAs sharing each R_J stage by TMA multicast), row tiles padded to cs
  uint32_t mstage, estage, acc_off;
  const float* xs;   // prepared points [n][dp]
  const float* vy;   // [n]
  const float* xv;   // [n_pad / 64][d + 1][64]: -x_jk rows, vy_j row (zero past n)
  const float* L;
  int64_t ld;
  float sf2, a, coef_b;
  double* part;      // [gridDim.x][2 (d + 1)]
  int dbg;           // WGP_GRAD_DEBUG ablation bits: 1 no MMA, 2 no epilogue math, 4 no R loads
  unsigned long long* trace;  // WGP_GRAD_TRACE: per warp {total, wait A, wait B, wait C} clk, summed over CTAs
};

template <int D>
__global__ void __launch_bounds__(gThreads, 1)
    grad_tc_kernel(const __grid_constant__ CUtensorMap mRhi, const __grid_constant__ CUtensorMap mRlo,
                   const GradTcArgs p) {
  constexpr int EP = ep_of(D);
  constexpr int NW = 2 * (D + 1);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // rfull[s]: R_J planes of stage s landed (all cs slices); rempty[s]: the
  // MMAs of all cs CTAs of the cluster released stage s; efull[s]: x_j | vy_j
  // of stage s landed; mdone[b]: W of the tile in buffer b ready; wfree[b]:
  // the epilogue read W buffer b; efree[s]: the epilogue read stage s;
  // lready: L_I in TMEM.  mdone shares the W-buffer ring: MMA(t) completes
  // phase t / 6 of mdone[t % 6] only after the epilogue of t - 6 consumed the
  // previous one, so no waiter can miss a phase whatever the issue order.
  __shared__ __align__(8) uint64_t bar_rfull[gNM], bar_rempty[gNM], bar_efull[gMaxNE], bar_mdone[gBufs],
      bar_wfree[gBufs], bar_efree[gMaxNE], bar_lready;
  __shared__ double wacc[gEpiWarps][NW];
  __shared__ uint32_t tmem_slot;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sR = smem;                                                 // nm x [R_hi | R_lo]
  const float* sE = reinterpret_cast<const float*>(sR + static_cast<size_t>(gNM) * p.mstage);  // ne x [EP][64]
  double* sAcc = reinterpret_cast<double*>(smem + p.acc_off);        // [NW][384] per-row fp64 sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // clusters of cs consecutive row tiles share one J range (and its R_J stream)
  const int rt = blockIdx.x % p.rt_pad, sp = blockIdx.x / p.rt_pad;
  const int CS = p.cs;
  const uint32_t crank = CS > 1 ? cluster_ctarank() : 0u;
  const uint16_t cmask = static_cast<uint16_t>((1u << CS) - 1u);
  const int jt_begin = static_cast<int>(static_cast<int64_t>(p.num_jt) * sp / p.splits);
  const int jt_end = static_cast<int>(static_cast<int64_t>(p.num_jt) * (sp + 1) / p.splits);
  const int T = jt_end - jt_begin;
  const int NE = p.ne;

  if (threadIdx.x == 0) {
    for (int i = 0; i < gNM; ++i) {
      mbar_init(&bar_rfull[i], 1);
      mbar_init(&bar_rempty[i], CS);
    }
    for (int i = 0; i < NE; ++i) {
      mbar_init(&bar_efull[i], 1);
      mbar_init(&bar_efree[i], 4);
    }
    for (int i = 0; i < gBufs; ++i) {
      mbar_init(&bar_mdone[i], 1);
      mbar_init(&bar_wfree[i], 4);
    }
    mbar_init(&bar_lready, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == gWarpAlloc) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers multicast into this CTA's ring and barriers
  tc_after();
  const uint32_t tmem = tmem_slot;

  if (warp < gIssuers) {
    // ------------------------------------------------------------ issuer q
    // Tiles t = q, q + 4, ...: R_J stage t % 4 and W buffer t % 6.  R_J stage
    // = nbox boxes of 64 points x 128 bytes (hi / lo planes x spk / 32); CTA
    // rank r of the cluster loads boxes r, r + cs, ... multicast to every
    // CTA, so the cluster reads R once.  The next own tile's loads are issued
    // as soon as every CTA's MMA released the stage (3 tiles of lead).
    const int q = warp;
    constexpr uint32_t idesc = idesc_tf32(gTI, gTJ);
    const uint32_t plane = p.mstage / 2;
    const int nbox = 2 * (p.spk / 32);
    long long tw1 = 0, tw2 = 0;
    const long long tstart = clock64();
    auto load = [&](int t) {
      const int sm = t & (gNM - 1);
      const int pt = (jt_begin + t) * gTJ;
      uint8_t* rb = sR + static_cast<size_t>(sm) * p.mstage;
      if (p.dbg & 4) {
        mbar_arrive_warp(&bar_rfull[sm]);
      } else {
        mbar_expect_tx_warp(&bar_rfull[sm], p.mstage);
        for (int bi = static_cast<int>(crank); bi < nbox; bi += CS) {
          const int kb = bi >> 1;
          uint8_t* dst = rb + (bi & 1) * plane + kb * 8192;
          const CUtensorMap* map = (bi & 1) ? &mRlo : &mRhi;
          if (CS > 1)
            tma_load_2d_mc_warp(dst, map, &bar_rfull[sm], 32 * kb, pt, cmask);
          else
            tma_load_2d_warp(dst, map, &bar_rfull[sm], 32 * kb, pt);
        }
      }
      const int se = t % NE;
      const long long c1 = p.trace ? clock64() : 0;
      if (t >= NE) mbar_wait(&bar_efree[se], ((t - NE) / NE) & 1);
      if (p.trace) tw2 += clock64() - c1;
      mbar_expect_tx_warp(&bar_efull[se], p.estage);
      bulk_load_warp(const_cast<float*>(sE) + se * (p.estage / 4), p.xv + static_cast<int64_t>(pt) * EP, p.estage,
                     &bar_efull[se]);
    };
    if (q < T) {
      load(q);
      mbar_wait(&bar_lready, 0);
      tc_after();
    }
    for (int t = q; t < T; t += gIssuers) {
      const int sm = t & (gNM - 1), b = t % gBufs;
      const long long c0 = p.trace ? clock64() : 0;
      if (t >= gBufs) mbar_wait(&bar_wfree[b], ((t - gBufs) / gBufs) & 1);
      mbar_wait(&bar_rfull[sm], (t >> 2) & 1);
      if (p.trace) tw1 += clock64() - c0;
      tc_after();
      if (!(p.dbg & 1)) {
        const uint8_t* rb = sR + static_cast<size_t>(sm) * p.mstage;
        const uint64_t dh = umma_desc(rb), dl = umma_desc(rb + plane);
        const uint32_t dcol = tmem + static_cast<uint32_t>(b) * gTJ;
        if (p.spk == 64)
          mma_w_k64(dcol, tmem + gLhi, dh, dl, idesc);
        else
          mma_w_k32(dcol, tmem + gLhi, dh, dl, idesc);
      }
      mma_commit(&bar_mdone[b]);
      if (CS > 1)
        mma_commit_mc(&bar_rempty[sm], cmask);
      else
        mma_commit(&bar_rempty[sm]);
      // the stage's next use (own tile t + 4) once all cs CTAs released it;
      // after the last own tile this wait drains the peers' arrivals before exit
      mbar_wait(&bar_rempty[sm], (t >> 2) & 1);
      if (t + gIssuers < T) load(t + gIssuers);
    }
    if (p.trace && lane == 0) {
      unsigned long long* tr = p.trace + warp * 4;
      atomicAdd(tr + 0, static_cast<unsigned long long>(clock64() - tstart));
      atomicAdd(tr + 1, static_cast<unsigned long long>(tw1));
      atomicAdd(tr + 2, static_cast<unsigned long long>(tw2));
    }
  } else if (warp >= gEpiBase) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - gEpiBase;  // epilogue warp index 0..11
    const int q = warp & 3, w = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int64_t gi = p.r0 + static_cast<int64_t>(rt) * gTI + row;
    const bool valid = gi < p.r1;
    float2 xi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float v = valid ? p.xs[gi * p.dp + k] : 0.f;
      xi[k] = make_float2(v, v);
    }
    const float hvy = valid ? 0.5f * p.vy[gi] : 0.f;
    if (w == 0 && T > 0) {
      // L_I (row gi, columns [0, spk), zero past s and past n) -> TMEM hi / lo planes
      for (int kb = 0; kb < p.spk / 32; ++kb) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int col = 32 * kb + c;
          const float v = (valid && col < p.s) ? p.L[gi + static_cast<int64_t>(col) * p.ld] : 0.f;
          hi[c] = __float_as_uint(v) & gTfMask;
          lo[c] = __float_as_uint(v - __uint_as_float(hi[c]));
        }
        __syncwarp();
        tmem_st32(tmem + lanes + gLhi + 32 * kb, hi);
        tmem_st32(tmem + lanes + gLlo + 32 * kb, lo);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_lready);
    }
    double* acc64 = sAcc + ew * 32 + lane;  // slot k at acc64[k * 384]
#pragma unroll
    for (int k = 0; k < NW; ++k) acc64[k * gEpiThreads] = 0.0;
    const float2 sf2 = make_float2(p.sf2, p.sf2), ac = make_float2(p.a, p.a);
    float2 A[D + 1], B[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) A[k] = B[k] = make_float2(0.f, 0.f);
    auto flush = [&]() {
#pragma unroll
      for (int k = 0; k <= D; ++k) {
        acc64[k * gEpiThreads] += static_cast<double>(A[k].x) + static_cast<double>(A[k].y);
        acc64[(D + 1 + k) * gEpiThreads] += static_cast<double>(B[k].x) + static_cast<double>(B[k].y);
        A[k] = B[k] = make_float2(0.f, 0.f);
      }
    };
    // points per shared load: 4 (two pairs) while the registers allow it
    constexpr int QP = D <= 6 ? 4 : 2;
    const uint32_t sE_u32 = smem_u32(sE);
    int since = 0;
    long long tw1 = 0, tw2 = 0, tw3 = 0;
    const long long tstart = clock64();
    for (int t = w; t < T; t += gEpiGroups) {
      const int b = t % gBufs, se = t % NE;
      long long c0 = p.trace ? clock64() : 0;
      mbar_wait(&bar_mdone[b], (t / gBufs) & 1);
      long long c1 = p.trace ? clock64() : 0;
      mbar_wait(&bar_efull[se], (t / NE) & 1);
      if (p.trace) {
        const long long c2 = clock64();
        tw1 += c1 - c0;
        tw2 += c2 - c1;
      }
      tc_after();
      const uint32_t ev = sE_u32 + static_cast<uint32_t>(se) * p.estage;  // [D + 1][64] fp32
      // 16-column chunks of W(t); the TMEM load of chunk h + 1 is in flight
      // while chunk h is processed (tcgen05.wait::ld waits for all loads, so
      // two register buffers alternate)
      auto chunk = [&](int h, const uint32_t(&wr)[16]) {
        if (p.dbg & 2) {
          A[0].x += __uint_as_float(wr[h]);
          return;
        }
#pragma unroll
        for (int e = 0; e < 16; e += QP) {
          const uint32_t col = ev + static_cast<uint32_t>(16 * h + e) * 4u;  // warp-uniform: broadcast loads
          if constexpr (QP == 4) {
            float2 n0[D], n1[D];
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const float4 v = lds128(col + k * 256);
              n0[k] = make_float2(v.x, v.y);
              n1[k] = make_float2(v.z, v.w);
            }
            const float4 vy = lds128(col + D * 256);
            entry_pair<D>(xi, n0, make_float2(vy.x, vy.y),
                          make_float2(__uint_as_float(wr[e]), __uint_as_float(wr[e + 1])), sf2, ac, A, B);
            entry_pair<D>(xi, n1, make_float2(vy.z, vy.w),
                          make_float2(__uint_as_float(wr[e + 2]), __uint_as_float(wr[e + 3])), sf2, ac, A, B);
          } else {
            float2 n0[D];
#pragma unroll
            for (int k = 0; k < D; ++k) n0[k] = lds64(col + k * 256);
            entry_pair<D>(xi, n0, lds64(col + D * 256),
                          make_float2(__uint_as_float(wr[e]), __uint_as_float(wr[e + 1])), sf2, ac, A, B);
          }
        }
      };
      const uint32_t wcol = tmem + lanes + static_cast<uint32_t>(b * gTJ);
      uint32_t w0[16], w1[16];
      __syncwarp();
      const long long c3 = p.trace ? clock64() : 0;
      tmem_ld16(wcol, w0);
      tmem_wait_ld();
      if (p.trace) tw3 += clock64() - c3;
      tmem_ld16(wcol + 16, w1);
      chunk(0, w0);
      tmem_wait_ld();
      pin(w1);
      tmem_ld16(wcol + 32, w0);
      chunk(1, w1);
      tmem_wait_ld();
      pin(w0);
      tmem_ld16(wcol + 48, w1);
      chunk(2, w0);
      tmem_wait_ld();
      pin(w1);
      chunk(3, w1);
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_wfree[b]);
        mbar_arrive(&bar_efree[se]);
      }
      if (++since == gFlushTiles) {
        flush();
        since = 0;
      }
    }
    flush();
    if (p.trace && lane == 0) {
      unsigned long long* tr = p.trace + warp * 4;
      atomicAdd(tr + 0, static_cast<unsigned long long>(clock64() - tstart));
      atomicAdd(tr + 1, static_cast<unsigned long long>(tw1));
      atomicAdd(tr + 2, static_cast<unsigned long long>(tw2));
      atomicAdd(tr + 3, static_cast<unsigned long long>(tw3));
    }
    // row scale (W^A = vy_i vy_j / 2: the vy_i / 2 factor; coef_b for W^B),
    // then the fixed-order warp sums
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      double v = acc64[k * gEpiThreads] * (k <= D ? static_cast<double>(hvy) : static_cast<double>(p.coef_b));
      v = warp_sum(v);
      if (lane == 0) wacc[ew][k] = v;
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x < NW) {
    double s = 0.0;
    for (int w = 0; w < gEpiWarps; ++w) s += wacc[w][threadIdx.x];
    p.part[static_cast<int64_t>(blockIdx.x) * NW + threadIdx.x] = s;
  }
  if (CS > 1) cluster_sync_all();
  if (warp == gWarpAlloc) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// R (column-major, ld) -> tf32 hi / lo planes [n_pad][spk] (point-major, K
// contiguous: the MMA's K-major B operand), and the epilogue stages xv.
// 32 points per CTA through a shared-memory transpose (coalesced both ways).
__global__ void grad_tc_prep_kernel(const float* R, int64_t ld, int s, const float* xs, int dp, int d,
                                    const float* vy, int64_t n, int spk, int ep, float* rhi, float* rlo, float* xv) {
  __shared__ float tile[64][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 x 32
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int c = ty; c < spk; c += 8) tile[c][tx] = (i0 + tx < n && c < s) ? R[i0 + tx + static_cast<int64_t>(c) * ld] : 0.f;
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    for (int c = tx; c < spk; c += 32) {
      const float v = tile[c][r];
      const float h = __uint_as_float(__float_as_uint(v) & gTfMask);
      rhi[(i0 + r) * spk + c] = h;
      rlo[(i0 + r) * spk + c] = v - h;
    }
  }
  // epilogue stage: tile-major [n_pad / 64][ep][64], rows -x_jk (k < d) and vy_j
  for (int k = ty; k < ep; k += 8) {
    const int64_t i = i0 + tx;
    float v = 0.f;
    if (i < n) v = k < d ? -xs[i * dp + k] : vy[i];
    xv[(i / 64) * (ep * 64) + k * 64 + (i % 64)] = v;
  }
}

// min_sp: the smallest split count whose J range fits the L2 budget (the
// grid is split-major, as hv_tc's: see choose_splits there).
int choose_grad_splits(int64_t row_tiles, int jt, int sms, int min_sp = 1) {
  constexpr double kCtaOverheadTiles = 8.0;
  int best = 1;
  double best_cost = 1e300;
  for (int sp = 1; sp <= 64; ++sp) {
    if (sp > 1 && jt / sp < 8) break;
    if (sp < min_sp) continue;
    const double waves = std::ceil(static_cast<double>(row_tiles * sp) / sms);
    const double cost = waves * (std::ceil(static_cast<double>(jt) / sp) + kCtaOverheadTiles);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

template <int D>
void launch_grad_tc(const CUtensorMap& mh, const CUtensorMap& ml, const GradTcArgs& a, unsigned grid, int smem,
                    cudaStream_t st) {
  WGP_SMEM_ATTR(grad_tc_kernel<D>, gSmemLimit);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(a.cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  WGP_CUDA(cudaLaunchKernelEx(&cfg, grad_tc_kernel<D>, mh, ml, a));
  WGP_LAUNCH_CHECK();
}

}  // namespace

bool grad_tc_supported(int d, int s) { return d >= 1 && d <= 12 && s >= 1 && s <= 64; }

GradTcPlan grad_tc_plan(int64_t n, int64_t m, int d, int s) {
  GradTcPlan pl;
  pl.n_pad = round_up(std::max<int64_t>(n, 1), gTJ);
  pl.spk = s <= 32 ? 32 : 64;
  pl.ep = ep_of(d);
  // cluster size: CTAs sharing the R_J stream (<= boxes per stage)
  static const int env_cs = [] {
    const char* e = getenv("WGP_GRAD_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  const int nbox = 2 * (pl.spk / 32);
  pl.cs = std::min(nbox, env_cs == 1 || env_cs == 2 || env_cs == 4 ? env_cs : 2);
  const int64_t row_tiles = ceil_div(m, gTI);
  if (row_tiles < pl.cs) pl.cs = 1;
  pl.rt_pad = static_cast<int>(round_up(row_tiles, pl.cs));
  const int jt = static_cast<int>(ceil_div(n, gTJ));
  static const int force = [] {
    const char* e = getenv("WGP_GRAD_SPLITS");
    return e ? atoi(e) : 0;
  }();
  // L2 rasterisation: the R_J / coordinate planes of a split's J range
  // (4 (2 spk + ep) bytes per point) within a 48 MB budget
  static const double l2_budget = [] {
    const char* e = getenv("WGP_TC_L2MB");
    return (e ? atof(e) : 48.0) * 1e6;
  }();
  int min_sp = 1;
  if (l2_budget > 0)
    min_sp = std::max(1, std::min(64, static_cast<int>(std::ceil(static_cast<double>(pl.n_pad) * 4.0 *
                                                                 (2 * pl.spk + pl.ep) / l2_budget))));
  pl.splits = force > 0 ? std::min(force, jt) : choose_grad_splits(pl.rt_pad, jt, tc_sm_count(), min_sp);
  pl.nblk = static_cast<int>(pl.rt_pad * pl.splits);
  pl.ws_bytes = sizeof(float) * static_cast<size_t>(pl.n_pad) * (2 * pl.spk + pl.ep);
  return pl;
}

void grad_tc(const GradParams& p, const GradTcPlan& pl, void* ws, cudaStream_t st) {
  if (!grad_tc_supported(p.d, p.s)) throw std::invalid_argument("grad_tc: needs 1 <= d <= 12 and 1 <= s <= 64");
  float* rhi = static_cast<float*>(ws);
  float* rlo = rhi + pl.n_pad * pl.spk;
  float* xv = rlo + pl.n_pad * pl.spk;
  grad_tc_prep_kernel<<<static_cast<unsigned>(pl.n_pad / 32), 256, 0, st>>>(p.R, p.ld, p.s, p.xs, p.dp, p.d, p.vy,
                                                                             p.n, pl.spk, pl.ep, rhi, rlo, xv);
  WGP_LAUNCH_CHECK();
  const CUtensorMap mh = tc_tensor_map(rhi, pl.spk, pl.n_pad, pl.spk * 4, 32, gTJ);
  const CUtensorMap ml = tc_tensor_map(rlo, pl.spk, pl.n_pad, pl.spk * 4, 32, gTJ);
  GradTcArgs a{};
  a.n = p.n;
  a.r0 = p.r0;
  a.r1 = p.r0 + (p.m < 0 ? p.n : p.m);
  a.d = p.d;
  a.dp = p.dp;
  a.s = p.s;
  a.spk = pl.spk;
  a.num_jt = static_cast<int>(ceil_div(p.n, gTJ));
  a.splits = pl.splits;
  a.cs = pl.cs;
  a.rt_pad = pl.rt_pad;
  a.mstage = 2u * static_cast<uint32_t>(pl.spk / 32) * 8192u;
  a.estage = static_cast<uint32_t>(gTJ * pl.ep * 4);
  const int acc_bytes = 2 * (p.d + 1) * gEpiThreads * 8;
  a.ne = gMaxNE;
  if (gNM * static_cast<int>(a.mstage) + a.ne * static_cast<int>(a.estage) + acc_bytes + 1024 > gSmemLimit) a.ne = 4;
  a.acc_off = gNM * a.mstage + static_cast<uint32_t>(a.ne) * a.estage;
  const int smem = static_cast<int>(a.acc_off) + acc_bytes + 1024;
  if (smem > gSmemLimit) throw DeviceError("grad_tc: shared memory too small");
  a.xs = p.xs;
  a.vy = p.vy;
  a.xv = xv;
  a.L = p.L;
  a.ld = p.ld;
  a.sf2 = p.sf2;
  a.a = p.a;
  a.coef_b = p.coef_b;
  a.part = p.part;
  static const int dbg = [] {
    const char* e = getenv("WGP_GRAD_DEBUG");
    return e ? atoi(e) : 0;
  }();
  a.dbg = dbg;
  static const bool tracing = getenv("WGP_GRAD_TRACE") != nullptr;
  static unsigned long long* trace = nullptr;
  a.trace = nullptr;
  if (tracing) {
    if (!trace) WGP_CUDA(cudaMalloc(&trace, sizeof(unsigned long long) * 64));
    WGP_CUDA(cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 64, st));
    a.trace = trace;
  }
  const unsigned grid = static_cast<unsigned>(pl.nblk);
  switch (p.d) {
#define WGP_GRAD_CASE(D) \
  case D:                \
    launch_grad_tc<D>(mh, ml, a, grid, smem, st); \
    break;
    WGP_GRAD_CASE(1)
    WGP_GRAD_CASE(2)
    WGP_GRAD_CASE(3)
    WGP_GRAD_CASE(4)
    WGP_GRAD_CASE(5)
    WGP_GRAD_CASE(6)
    WGP_GRAD_CASE(7)
    WGP_GRAD_CASE(8)
    WGP_GRAD_CASE(9)
    WGP_GRAD_CASE(10)
    WGP_GRAD_CASE(11)
    WGP_GRAD_CASE(12)
#undef WGP_GRAD_CASE
    default:
      throw std::invalid_argument("grad_tc: unsupported d");
  }
  if (tracing) {
    // per warp: {total, wait A, wait B, wait C} clk summed over CTAs.  Epilogue
    // warps: A = mdone (W ready), B = efull (x_j | vy_j), C = first TMEM load;
    // MMA warp: A = wfree, B = rfull; producer: A = rempty, B = efree.
    unsigned long long h[64];
    WGP_CUDA(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    for (int w = 0; w < 16; ++w) {
      const double tot = static_cast<double>(h[4 * w]);
      if (tot <= 0) continue;
      fprintf(stderr, "[grad_tc trace] warp %2d: total %.3e clk  waitA %5.1f%%  waitB %5.1f%%  waitC %5.1f%%\n", w, tot,
              100.0 * h[4 * w + 1] / tot, 100.0 * h[4 * w + 2] / tot, 100.0 * h[4 * w + 3] / tot);
    }
  }
}

}  // namespace wgp
